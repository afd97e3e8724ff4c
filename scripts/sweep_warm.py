"""Warm-decompose sweep of the restart parameters: python scripts/sweep_warm.py c2,c3 2,3,4,5 8,16,32"""
import os, sys, subprocess
cfgs = sys.argv[1].split(","); mcycs = sys.argv[2].split(","); extras = sys.argv[3].split(",")
for cfg in cfgs:
    for extra in extras:
        for mcyc in mcycs:
            env = dict(os.environ)
            if mcyc != "d": env["SSA_MCYC"] = mcyc
            if extra != "d": env["SSA_PK_EXTRA"] = extra
            out = subprocess.run([sys.executable, "scripts/prof_decompose.py", cfg], env=env, capture_output=True,
                                 text=True).stdout.strip().splitlines()
            print(f"{cfg} extra={extra:>2} mcyc={mcyc}: {out[-1] if out else 'FAILED'}", flush=True)
