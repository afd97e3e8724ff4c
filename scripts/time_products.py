"""Device time of one X·V and one Xᵀ·U block product through the C ABI, in the solver's layout
(column-major blocks, leading dimension rounded up to 32 elements), CUDA events, median of reps:
    python scripts/time_products.py c5 [k] [reps]      (SSA_FFT_STOCKHAM=1: round-1 FFT passes)
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1309_5050_b200 import Plan, _lib

cfg = sys.argv[1]
w = synth.get(cfg)
k = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else w.block_k
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
path = os.environ.get("PATH_SEL", "fft")
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, path=path)
L = _lib.load()
td = torch.float64 if w.dtype == "f64" else torch.float32
ldq, ldp = (p.K + 31) // 32 * 32, (p.L + 31) // 32 * 32
Q = torch.randn(k, ldq, device="cuda", dtype=td)
P = torch.randn(k, ldp, device="cuda", dtype=td)
OutP = torch.empty(k, ldp, device="cuda", dtype=td)
OutQ = torch.empty(k, ldq, device="cuda", dtype=td)
st = torch.cuda.current_stream()
out = {"cfg": cfg, "k": k, "path": [p.path_xv, p.path_xtu], "stockham": bool(os.environ.get("SSA_FFT_STOCKHAM"))}
for name, tr, src, dst, ldi, ldo in (("xv", 0, Q, OutP, ldq, ldp), ("xtu", 1, P, OutQ, ldp, ldq)):
    def f():
        _lib.check(L.ssa_matmul(p._h, tr, src.data_ptr(), ldi, dst.data_ptr(), ldo, k, 1))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name + "_ms"] = float(np.median(ts))
print(json.dumps(out))
