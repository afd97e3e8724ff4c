"""Plan-creation time per config (warm): python scripts/time_plan.py c4"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1309_5050_b200 import Plan
for cfg in sys.argv[1:]:
    w = synth.get(cfg)
    ts = []
    for i in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
        del p
    print(cfg, "plan ms", [round(x, 2) for x in ts], "K", Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype).K)
