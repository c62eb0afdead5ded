import sys, os
sys.path.insert(0, os.getcwd())
import torch, json
import bench
print(json.dumps({k: v for k, v in bench.extras_single_gpu(torch.device("cuda", 0), 37.22, skip="C3").items() if k.startswith("C1")}))
