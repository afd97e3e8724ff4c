"""Decompose time vs block width k and blocks per restart cycle (SSA_MCYC), second call of each."""
import os, sys, time, itertools, subprocess, json
cfg = sys.argv[1]
ks = [int(v) for v in sys.argv[2].split(",")]
ms = sys.argv[3].split(",")
for k, m in itertools.product(ks, ms):
    env = dict(os.environ, SSA_MCYC=m)
    code = f"""
import sys, time; sys.path.insert(0, '.')
import numpy as np, synth
from paper_1309_5050_b200 import Plan
w = synth.get('{cfg}')
best = 1e9
for rep in range(3):
    p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k={k})
    t = time.perf_counter(); info = p.decompose(w.r, allow_not_converged=True); t = time.perf_counter() - t
    best = min(best, t)
print({k}, {m}, round(best * 1e3, 2), info['n_block_products'], info['n_restarts'], info['n_converged'], round(info['ms_ritz'], 2), '%.1e' % info['max_rel_residual'])
"""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
