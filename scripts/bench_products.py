"""Time X·V and Xᵀ·U block products per path (CUDA events, median of reps):
    python scripts/bench_products.py c2 tc,fft,direct [k] [reps]
Prints one line per (path, product): ms, useful TFLOP/s (2·L·K·k) and the path actually used."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1309_5050_b200 import Plan

cfg = sys.argv[1]
paths = (sys.argv[2] if len(sys.argv) > 2 else "tc,fft").split(",")
w = synth.get(cfg)
k = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else w.block_k
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
td = torch.float64 if w.dtype == "f64" else torch.float32
for path in paths:
    try:
        p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, path=path)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"cfg": cfg, "path": path, "error": str(e)}))
        continue
    V = torch.randn(p.K, k, device="cuda", dtype=td)
    U = torch.randn(p.L, k, device="cuda", dtype=td)
    for name, fn, used in (("xv", lambda: p.matmul(V), p.path_xv), ("xtu", lambda: p.matmul(U, transpose=True), p.path_xtu)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        fl = 2.0 * p.L * p.K * k
        print(json.dumps({"cfg": cfg, "req": path, "product": name, "used": used, "k": k, "ms": round(ms, 4),
                          "useful_tflops": round(fl / ms / 1e9, 2)}))
    p.close()
