"""One shape of ssa_bench_tall (for ncu): python scripts/bench_tall1.py which M n1 n2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
w, M, n1, n2 = (int(x) for x in sys.argv[1:5])
ms = C.c_double(); ck = C.c_double()
assert L.ssa_bench_tall(w, M, n1, n2, 2, C.byref(ms), C.byref(ck)) == 0
print(w, M, n1, n2, f"{ms.value * 1e3:.1f} us")
