timeout 300 python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
for (M, n) in [(1844160, 64), (1844160, 128), (201601*4, 224)]:
    for bc in (32, 64, 128):
        for rg in (1, 2, 4):
            if bc * 128 * rg * 8 > 200 * 1024 or bc > n: continue
            ms = C.c_double(); ck = C.c_double()
            st = L.ssa_bench_tall(4, M, n, bc + 256 * rg, 5, C.byref(ms), C.byref(ck))
            if st != 0: print("err", L.ssa_last_error()); continue
            print(f"probe M={M} n={n} box cols={bc:3d} rg={rg}: {ms.value * 1e3:7.1f} us {4 * M * n / ms.value / 1e6:6.0f} GB/s", flush=True)
PY
for w in 3 0; do SSA_GRAM_TRACE=1 timeout 120 python - $w <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_5050_b200 import _lib
L = _lib.load()
ms = C.c_double(); ck = C.c_double()
w = int(sys.argv[1])
assert L.ssa_bench_tall(w, 1844160, 64, 64, 1, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
print(w, ms.value * 1e3, "us")
PY
done 2>&1 | grep -v "^\[gram trace\] M=20" | head -60
