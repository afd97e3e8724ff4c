for v in 1 2; do for ka in 4 2; do echo "V=$v KA=$ka"; SSA_GRAM_V=$v SSA_GRAM_KA=$ka timeout 300 python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
for which, (M, n1, n2) in [(0, (20001, 300, 64)), (0, (8200, 65, 33)), (3, (12345, 64, 64)), (0, (9001, 33, 64)), (0, (201601, 224, 32)), (0, (201601, 96, 32)), (0, (201601, 32, 32)), (3, (201601, 32, 32)), (0, (1844160, 64, 64)), (0, (1844160, 356, 64)), (3, (1844160, 64, 64)), (0, (1844160, 548, 64))]:
    ms = C.c_double(); ck = C.c_double()
    assert L.ssa_bench_tall(which, M, n1, n2, 5, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
    print(f"{which} M={M:8d} n1={n1:3d} n2={n2:2d}: {ms.value*1e3:8.1f} us {4*M*(n1+(n2 if which==0 else 0))/ms.value/1e6:6.0f} GB/s check {ck.value:.3e}", flush=True)
PY
done; done
SSA_GRAM_V2NM2=1 SSA_GRAM_V=2 timeout 300 python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
for which, (M, n1, n2) in [(0, (20001, 300, 32)), (0, (201601, 224, 32))]:
    ms = C.c_double(); ck = C.c_double()
    assert L.ssa_bench_tall(which, M, n1, n2, 5, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
    print(f"NM2 {which} M={M:8d} n1={n1:3d} n2={n2:2d}: {ms.value*1e3:8.1f} us {4*M*(n1+(n2 if which==0 else 0))/ms.value/1e6:6.0f} GB/s check {ck.value:.3e}", flush=True)
PY
SSA_GRAM_TRACE=1 SSA_GRAM_V=2 timeout 120 python - 0 <<'PY' 2>&1 | tail -16
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
ms = C.c_double(); ck = C.c_double()
assert L.ssa_bench_tall(0, 1844160, 64, 64, 1, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
print(ms.value * 1e3, "us")
PY
