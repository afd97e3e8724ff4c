"""Time (and, under ncu, capture) block products of one config:
python scripts/prof_products.py c5 fft [k] [reps]
Inputs are column-major device tensors and the outputs preallocated, so only the library's kernels run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1309_5050_b200 import Plan
cfg = sys.argv[1]; path = sys.argv[2] if len(sys.argv) > 2 else "fft"
w = synth.get(cfg)
k = int(sys.argv[3]) if len(sys.argv) > 3 else w.block_k
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, path=path)
td = torch.float64 if w.dtype == "f64" else torch.float32
V = torch.randn(k, p.K, device="cuda", dtype=td).t()      # column-major K x k
U = torch.randn(k, p.L, device="cuda", dtype=td).t()
oU = torch.empty(k, p.L, device="cuda", dtype=td)
oV = torch.empty(k, p.K, device="cuda", dtype=td)
def run(which):
    if which == "xv":
        p.matmul(V, out=oU)
    else:
        p.matmul(U, transpose=True, out=oV)
for _ in range(reps):
    run("xv"); run("xtu")
torch.cuda.synchronize()
for which in ("xv", "xtu"):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run(which)
    e1.record(); torch.cuda.synchronize()
    print(cfg, path, which, "k", k, f"avg block product {e0.elapsed_time(e1) / reps:.3f} ms")
