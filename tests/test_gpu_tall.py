"""The solver's tall-skinny fp32 kernels (Gram AᵀB and update W −= A·C) on odd shapes that reach every
dispatch branch — tensor-core (tcgen05 3xTF32, M >= 8192: narrow / wide / two-M-tile Grams, AᵀA from
one tile, MN-major update with ragged row tiles and column chunks), cp.async FFMA and thread-per-row
kernels — against an fp64 host evaluation of the same fp32 data (ssa_bench_tall's check).
Bar: 3xTF32 / fp32 accumulation, relative to the largest entry: 2e-6 (SURVEY's 1e-5 product bar with
margin for the k-long sums)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-6


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1309_5050_b200 import _lib, build
    build.build()
    return _lib.load()


def _run(lib, which, M, n1, n2):
    ms, ck = C.c_double(), C.c_double()
    st = lib.ssa_bench_tall(which, M, n1, n2, 1, C.byref(ms), C.byref(ck))
    assert st == 0, lib.ssa_last_error()
    return ck.value


@pytest.mark.parametrize("M,n1,n2", [(8200, 65, 33), (8200, 200, 17), (20001, 300, 64), (9001, 33, 64),
                                     (5000, 100, 32), (1000, 224, 32)])
def test_gram_matches_fp64(lib, M, n1, n2):
    assert _run(lib, 0, M, n1, n2) <= TOL


@pytest.mark.parametrize("M,n1,n2", [(8200, 40, 32), (12345, 64, 64)])
def test_self_gram_matches_fp64(lib, M, n1, n2):
    assert _run(lib, 3, M, n1, n2) <= TOL


@pytest.mark.parametrize("M,n1,n2", [(12345, 128, 64), (20001, 192, 64), (9001, 96, 32), (8200, 320, 64),
                                     (10007, 64, 64)])
def test_tail_gram_matches_fp64(lib, M, n1, n2):
    """[A W]ᵀW with W the last n2 columns of A (the projection Gram of the solver): W read from A's tiles."""
    assert _run(lib, 5, M, n1, n2) <= TOL


@pytest.mark.parametrize("M,n1,n2", [(8200, 65, 33), (8200, 100, 64), (20001, 300, 64), (9001, 33, 17),
                                     (70000, 512, 64), (3000, 224, 32)])
def test_update_matches_fp64(lib, M, n1, n2):
    assert _run(lib, 1, M, n1, n2) <= TOL


_V1_SCRIPT = r"""
import ctypes as C, sys
sys.path.insert(0, sys.argv[1])
from paper_1309_5050_b200 import _lib
L = _lib.load()
worst = 0.0
for which, (M, n1, n2) in [(0, (8200, 65, 33)), (0, (20001, 300, 64)), (3, (12345, 64, 64)), (1, (8200, 100, 64)),
                           (1, (20001, 300, 64))]:
    ms, ck = C.c_double(), C.c_double()
    assert L.ssa_bench_tall(which, M, n1, n2, 1, C.byref(ms), C.byref(ck)) == 0, L.ssa_last_error()
    worst = max(worst, ck.value)
print(worst)
"""


@pytest.mark.parametrize("env", [{"SSA_UPD_TC": "2"}])
def test_kernel_variants_match_fp64(lib, env):
    """The env-selected variant (tensor-core update for narrow m) stays correct: the switches are read once per process, so each runs in
    a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _V1_SCRIPT, root], env={**os.environ, **env}, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= TOL
