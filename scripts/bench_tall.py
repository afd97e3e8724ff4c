"""Micro-benchmark of the solver's tall-skinny fp32 kernels (ssa_bench_tall): Gram AᵀB and update W -= A·C."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1309_5050_b200 import _lib
L = _lib.load()
shapes = [(1024, 32, 32), (1024, 224, 32), (4096, 32, 32), (4096, 224, 32), (201601, 32, 32), (201601, 96, 32), (201601, 192, 32), (201601, 224, 32), (24584, 192, 32), (4096, 192, 32),
          (14753281 // 8, 64, 64), (14753281 // 8, 356, 64)]
for (M, n1, n2) in [(201601, 32, 32), (1844160, 64, 64)]:
    ms = C.c_double(); ck = C.c_double()
    assert L.ssa_bench_tall(3, M, n1, n2, 5, C.byref(ms), C.byref(ck)) == 0
    print(f"self M={M:9d} n1={n1:3d} n2={n2:2d}: {ms.value * 1e3:8.1f} us  {4 * M * n1 / ms.value / 1e6:7.0f} GB/s  check {ck.value:.3e}")
for which in (0, 1):
    for (M, n1, n2) in shapes:
        ms = C.c_double(); ck = C.c_double()
        st = L.ssa_bench_tall(which, M, n1, n2, 5, C.byref(ms), C.byref(ck))
        if st != 0:
            print("error", L.ssa_last_error()); continue
        byts = 4 * M * (n1 + n2) if which == 0 else 4 * M * (n1 + 2 * n2)
        fl = 2.0 * M * n1 * n2
        print(f"{'gram' if which == 0 else 'upd '} M={M:9d} n1={n1:3d} n2={n2:2d}: {ms.value * 1e3:8.1f} us  "
              f"{byts / ms.value / 1e6:7.0f} GB/s  {fl / ms.value / 1e9:6.1f} TFLOP/s  check {ck.value:.3e}")
