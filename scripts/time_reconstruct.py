"""Host wall time vs device time of the reconstruction phase (c5 by default): a fresh plan per run,
decompose, then reconstruct #1 (computes V = XᵀU/σ) and #2 (V cached: diagonal averaging only), each
bracketed by device synchronisations; prints host ms, CUDA-event ms and the library launch counts.
    python scripts/time_reconstruct.py [c5] [runs]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1309_5050_b200 import Plan, launch_count

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = synth.get(cfg)
x = torch.as_tensor(w.data, dtype=torch.float64 if w.dtype == "f64" else torch.float32, device="cuda")
for run in range(runs):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = Plan(x, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    p.decompose(w.r, allow_not_converged=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = []
    for rep in range(2):
        launch_count(reset=True)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter(); e0.record()
        p.reconstruct(w.groups, device=True)
        e1.record(); torch.cuda.synchronize(); h1 = time.perf_counter()
        res.append((round((h1 - h0) * 1e3, 3), round(e0.elapsed_time(e1), 3), launch_count()))
    print(f"run {run}: plan {1e3 * (t1 - t0):.2f} ms, decompose {1e3 * (t2 - t1):.2f} ms, "
          f"reconstruct #1 (host, events, launches) {res[0]}, #2 (V cached) {res[1]}", flush=True)
    p.close()
