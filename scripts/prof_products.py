"""Run a few block products of one config (for ncu captures): python scripts/prof_products.py c3 fft [k] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_1309_5050_b200 import Plan
cfg = sys.argv[1]; path = sys.argv[2] if len(sys.argv) > 2 else "fft"
w = synth.get(cfg)
k = int(sys.argv[3]) if len(sys.argv) > 3 else w.block_k
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, path=path)
td = torch.float64 if w.dtype == "f64" else torch.float32
V = torch.randn(p.K, k, device="cuda", dtype=td)
U = torch.randn(p.L, k, device="cuda", dtype=td)
for _ in range(reps):
    p.matmul(V)
    p.matmul(U, transpose=True)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    p.matmul(V)
    p.matmul(U, transpose=True)
e1.record(); torch.cuda.synchronize()
print(cfg, path, "k", k, f"avg block product {e0.elapsed_time(e1) / (2 * reps):.3f} ms")
