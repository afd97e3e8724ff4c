"""TMA streaming probe at the c5 K-side size: bandwidth of box shapes (ssa_bench_tall which = 4;
n2 = rows per box, 32 = 128-B swizzled, -32 = the same box unswizzled; n1 = columns + 1000 x the
distance in stages of a 128-row L2 prefetch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
M = 14753281
for n, brow in [(64, 32), (64, 64), (-1064, 32), (-2064, 32)]:
    ms = C.c_double(); ck = C.c_double()
    st = L.ssa_bench_tall(4, M, n, brow, 5, C.byref(ms), C.byref(ck))
    if st != 0:
        print("error", n, brow, L.ssa_last_error()); continue
    nn = abs(n) % 1000
    print(f"probe n={nn:3d} pd={n // 1000 if n > 0 else -(-n // 1000)} box rows={brow:4d}: {ms.value * 1e3:8.1f} us  {4 * M * nn / ms.value / 1e6:7.0f} GB/s", flush=True)
