"""L2-resident vs HBM read bandwidth on one B200 (torch sum reductions and copies), for the
roofline of the neighbour-tile loads of dg_apply (profiles/r01_ab.md)."""
import torch

torch.cuda.init()
for mb in (8, 16, 32, 64, 96, 512, 2048):
    n = mb * 1024 * 1024 // 8
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    for _ in range(5):
        x.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    a.record()
    for _ in range(reps):
        x.sum()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps * 1e-3
    y = torch.empty_like(x)
    y.copy_(x)
    a.record()
    for _ in range(reps):
        y.copy_(x)
    b.record()
    torch.cuda.synchronize()
    tc = a.elapsed_time(b) / reps * 1e-3
    print(f"{mb:5d} MB: sum read {x.numel()*8/t/1e9:8.0f} GB/s   copy r+w {2*x.numel()*8/tc/1e9:8.0f} GB/s")
