"""One X·V and one Xᵀ·U block product between cudaProfilerStart/Stop (for ncu DRAM-traffic captures):
python scripts/traffic_products.py c2 fft 32"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1309_5050_b200 import Plan
cfg, path = sys.argv[1], sys.argv[2]
w = synth.get(cfg)
k = int(sys.argv[3]) if len(sys.argv) > 3 else w.block_k
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, path=path)
td = torch.float64 if w.dtype == "f64" else torch.float32
V = torch.randn(p.K, k, device="cuda", dtype=td)
U = torch.randn(p.L, k, device="cuda", dtype=td)
p.matmul(V); p.matmul(U, transpose=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
p.matmul(V)
torch.cuda.synchronize()
p.matmul(U, transpose=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(cfg, path, k, "done")
