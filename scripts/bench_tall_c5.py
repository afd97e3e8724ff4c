"""Live timing of the solver's tall-skinny kernels at the c5 K-side size (M = 14,753,281, ld rounded to 32):
self Gram WᵀW (n = 64), Gram [A W]ᵀW (n1 = 128, 192), update W -= A·C (m = 64, 128, 192)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
M = 14753281
for which, n1, n2 in [(3, 64, 64), (0, 128, 64), (0, 192, 64), (5, 128, 64), (5, 192, 64), (1, 64, 64), (1, 128, 64), (1, 192, 64)]:
    ms = C.c_double(); ck = C.c_double()
    st = L.ssa_bench_tall(which, M, n1, n2, 5, C.byref(ms), C.byref(ck))
    if st != 0:
        print("error", L.ssa_last_error()); continue
    byts = 4 * M * n1 if which in (3, 5) else (4 * M * (n1 + n2) if which == 0 else 4 * M * (n1 + 2 * n2))
    name = {3: "self-gram", 0: "gram", 1: "update", 5: "tail-gram"}[which]
    print(f"{name:9s} M={M} n1={n1:3d} n2={n2:2d}: {ms.value * 1e3:8.1f} us  {byts / ms.value / 1e6:7.0f} GB/s", flush=True)
