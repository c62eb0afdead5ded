import torch, time
n=262144000//8
h=torch.empty(n, dtype=torch.float64).pin_memory(); h2=torch.empty(n, dtype=torch.float64).pin_memory()
d=torch.empty(n, dtype=torch.float64, device='cuda'); d2=torch.empty_like(d)
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
for mode in ('1 stream 2x262MB','2 streams','d2h','h2d+d2h'):
    torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    if mode=='1 stream 2x262MB':
        d.copy_(h, non_blocking=True); d2.copy_(h2, non_blocking=True)
    elif mode=='2 streams':
        s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    elif mode=='d2h':
        h.copy_(d, non_blocking=True)
    else:
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
        d2.copy_(h2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
    b.record(); torch.cuda.synchronize()
    ms=a.elapsed_time(b); gb=(2 if mode!='d2h' else 1)*n*8/1e9
    print(mode, round(ms,2),'ms', round(gb/(ms/1e3),1),'GB/s')
