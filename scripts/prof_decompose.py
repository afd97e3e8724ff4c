"""One warm decomposition of a config between cudaProfilerStart/Stop (for ncu --profile-from-start off):
python scripts/prof_decompose.py c2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import torch
import synth
from paper_1309_5050_b200 import Plan
cfg = sys.argv[1]
w = synth.get(cfg)
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k)
p.decompose(w.r, allow_not_converged=True)      # warm-up (path autotune, lazy module loading)
p.close()
# a fresh plan: a second decomposition on the same plan would be warm-started from its eigenvectors
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t = time.perf_counter()
info = p.decompose(w.r, allow_not_converged=True)
torch.cuda.synchronize()
t = time.perf_counter() - t
torch.cuda.cudart().cudaProfilerStop()
print(cfg, f"warm decompose {t * 1e3:.2f} ms", {k: info[k] for k in ("n_block_products", "n_restarts", "ms_ritz")})
