"""Reading Q10: measure the σ floor τ of each product path on the noiseless c5 twin (4096²,
window 256², rank 48, σ spread 1.2e-7) against the closed-form spectrum (pin P7):
τ = the smallest σ_i/σ_1 down to which every σ_j >= τ·σ_1 meets the σ bar (relative error
<= 1e-4; DESIGN.md §3 reading Q10).

    python scripts/measure_tau.py [fft,tc,direct] > profiles/r02/tau.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import closed_form as cf
import synth
from paper_1309_5050_b200 import Plan

paths = (sys.argv[1] if len(sys.argv) > 1 else "fft,tc,direct").split(",")
w = synth.config5(noise=False)
s_cf = cf.sigma_rect(w.terms, 256, 256, 3841, 3841)
out = {"config": "c5 noiseless twin", "rank": len(s_cf), "sigma_cf_rel": list(s_cf / s_cf[0]), "paths": {}}
for path in paths:
    try:
        t0 = time.time()
        p = Plan(w.data, w.window, dtype="f32", block_k=64, path=path)
        info = p.decompose(50, allow_not_converged=True)
        s = p.sigma[:len(s_cf)]
        err = np.abs(s - s_cf) / s_cf
        tau = 1.0
        for i in range(len(s_cf)):
            if np.all(err[:i + 1] <= 1e-4):
                tau = s_cf[i] / s_cf[0]
            else:
                break
        out["paths"][path] = {"tau": float(tau), "rel_err": [float(e) for e in err],
                              "n_converged": info["n_converged"], "n_block_products": info["n_block_products"],
                              "path_xv": p.path_xv, "path_xtu": p.path_xtu, "seconds": time.time() - t0}
        p.close()
    except Exception as e:  # noqa: BLE001
        out["paths"][path] = {"error": str(e)}
    print(json.dumps({path: out["paths"][path].get("tau", out["paths"][path].get("error"))}), file=sys.stderr, flush=True)
print(json.dumps(out))
