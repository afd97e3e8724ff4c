for cfg in "2 1"; do set -- $cfg; echo "UPD_V=$1 UPD_TC=$2"; SSA_UPD_V=$1 SSA_UPD_TC=$2 timeout 120 python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
for (M, n1, n2) in [(8200, 65, 33), (8200, 100, 64), (20001, 300, 64), (9001, 33, 17), (70000, 512, 64), (201601, 32, 32), (201601, 96, 32), (201601, 224, 32), (1844160, 64, 64), (1844160, 356, 64), (1844160, 548, 64)]:
    ms = C.c_double(); ck = C.c_double()
    st = L.ssa_bench_tall(1, M, n1, n2, 5, C.byref(ms), C.byref(ck))
    if st != 0: print("err", L.ssa_last_error()); continue
    print(f"upd M={M:8d} n1={n1:3d} n2={n2:2d}: {ms.value*1e3:8.1f} us {4*M*(n1+2*n2)/ms.value/1e6:6.0f} GB/s check {ck.value:.3e}", flush=True)
PY
done
