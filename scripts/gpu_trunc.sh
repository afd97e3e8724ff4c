timeout 300 python scripts/bench_tall.py 2>&1 | grep "gram M=   201601"
echo TRUNC; SSA_TF32_TRUNC=1 timeout 300 python scripts/bench_tall.py 2>&1 | grep "gram M=   201601"
SSA_TF32_TRUNC=1 timeout 500 python -m pytest tests/test_gpu_tall.py -q 2>&1 | tail -5
SSA_TF32_TRUNC=1 python - <<'PY'
import ctypes as C, sys
sys.path.insert(0,'.')
from paper_1309_5050_b200 import _lib
L=_lib.load()
for (M,n1,n2) in [(8200,65,33),(20001,300,64),(12345,64,64)]:
    ms=C.c_double(); ck=C.c_double(); L.ssa_bench_tall(0,M,n1,n2,1,C.byref(ms),C.byref(ck)); print("trunc gram err", M,n1,n2, ck.value)
PY
python - <<'PY'
import ctypes as C, sys
sys.path.insert(0,'.')
from paper_1309_5050_b200 import _lib
L=_lib.load()
for (M,n1,n2) in [(8200,65,33),(20001,300,64),(12345,64,64)]:
    ms=C.c_double(); ck=C.c_double(); L.ssa_bench_tall(0,M,n1,n2,1,C.byref(ms),C.byref(ck)); print("rna gram err", M,n1,n2, ck.value)
PY
