"""TMA streaming probe: boxes {32 rows, bc cols, rg row groups} of a column-major M x n block."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
for (M, n) in [(201601, 32), (201601, 224)]:
    for bc in (32, 64, 128):
        for rg in (1, 2, 4, 8):
            if bc * 128 * rg * 8 > 200 * 1024 or bc > n and bc != 32: continue
            ms = C.c_double(); ck = C.c_double()
            st = L.ssa_bench_tall(4, M, n, bc + 256 * rg, 5, C.byref(ms), C.byref(ck))
            if st != 0: print("err", L.ssa_last_error()); continue
            print(f"M={M} n={n} box cols={bc:3d} rg={rg}: {ms.value * 1e3:7.1f} us {4 * M * n / ms.value / 1e6:6.0f} GB/s")
