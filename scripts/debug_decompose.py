import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_1309_5050_b200 import Plan
cfg = sys.argv[1]; path = sys.argv[2] if len(sys.argv) > 2 else "auto"
kw = {}
w = synth.get(cfg)
if len(sys.argv) > 3: w.block_k = int(sys.argv[3])
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k, path=path)
t = time.time(); info = p.decompose(w.r, allow_not_converged=True); t = time.time() - t
print(cfg, path, "k", w.block_k, "L", p.L, "K", p.K, f"{t*1e3:.1f} ms", info)
print("sigma", np.array2string(p.sigma[:8], precision=6), "...", p.sigma[-3:])
