"""Read bandwidth of a column-major M x n block streamed in row chunks (ssa_bench_tall which=2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
for (M, n) in [(201601, 224), (201601, 32), (1844160, 64)]:
    for rch32 in (1, 2, 4, 8, 16, 32, 64):
        if rch32 > 64: continue
        ms = C.c_double(); ck = C.c_double()
        assert L.ssa_bench_tall(2, M, n, rch32, 5, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
        print(f"M={M} n={n} chunk={32 * rch32:5d} rows: {ms.value * 1e3:8.1f} us {4 * M * n / ms.value / 1e6:7.0f} GB/s")
