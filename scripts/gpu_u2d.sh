for d in 0 3; do echo "UPD_DBG=$d"; SSA_UPD_DBG=$d timeout 120 python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
for (M, n1, n2) in [(201601, 224, 32), (1844160, 64, 64), (1844160, 356, 64)]:
    ms = C.c_double(); ck = C.c_double()
    assert L.ssa_bench_tall(1, M, n1, n2, 5, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
    print(f"upd M={M:8d} n1={n1:3d} n2={n2:2d}: {ms.value*1e3:8.1f} us {4*M*(n1+2*n2)/ms.value/1e6:6.0f} GB/s", flush=True)
PY
done
