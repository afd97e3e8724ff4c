"""One call of a solver tall-skinny kernel at the c5 K-side size, for ncu:
python scripts/prof_tall.py which n1 n2   (which: 3 self-Gram, 0 Gram, 1 update; see ssa_bench_tall)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
which, n1, n2 = (int(a) for a in sys.argv[1:4])
ms = C.c_double(); ck = C.c_double()
st = L.ssa_bench_tall(which, 14753281, n1, n2, 2, C.byref(ms), C.byref(ck))
print(which, n1, n2, st, ms.value * 1e3, "us")
