"""Sweep restart parameters: python scripts/sweep_solver.py c3 fft"""
import os, sys, subprocess, json
cfg, path = sys.argv[1], sys.argv[2]
ks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "32").split(",")]
for k in ks:
    for extra in ("4", "8", "16", "32"):
        for mcyc in ("2", "3", "4", "6", "8"):
            env = dict(os.environ, SSA_PK_EXTRA=extra, SSA_MCYC=mcyc)
            out = subprocess.run([sys.executable, "scripts/debug_decompose.py", cfg, path, str(k)], env=env,
                                 capture_output=True, text=True).stdout.splitlines()
            line = [l for l in out if l.startswith(cfg)]
            if line:
                l = line[0]
                info = eval(l[l.index("{"):])
                print(f"k={k} extra={extra:>2} mcyc={mcyc}: {l.split()[8]} ms  prod={info['n_block_products']:4d} "
                      f"restarts={info['n_restarts']:3d} ritz={info['ms_ritz']:.1f} prodms={info['ms_products']:.1f} conv={info['n_converged']}", flush=True)
