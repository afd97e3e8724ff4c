"""Micro-benchmark of the device Jacobi SVD (ssa_small_svd) vs numpy on shapes the solver uses."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
from paper_1309_5050_b200 import _lib

L = _lib.load()
rng = np.random.default_rng(0)
for (m, n, kind) in [(160, 128, "rand"), (176, 144, "rand"), (176, 144, "graded"), (144, 144, "restart"), (288, 256, "rand"), (576, 544, "graded")]:
    A = rng.normal(size=(m, n))
    if kind == "graded":
        A = A * np.logspace(0, -4, n)[None, :]
    if kind == "restart":  # diag(theta) block + coupling, as after a thick restart
        A = np.zeros((m, n)); pk = 48
        A[:pk, :pk] = np.diag(np.linspace(100, 10, pk)); A[:, pk:] = rng.normal(size=(m, n - pk))
    Af = np.asfortranarray(A.copy())
    sw = C.c_int32(); ms = C.c_double()
    st = L.ssa_small_svd(m, n, Af.ctypes.data, C.byref(sw), C.byref(ms))
    assert st == 0, L.ssa_last_error()
    s = np.sort(np.linalg.norm(Af, axis=0))[::-1]
    s_ref = np.linalg.svd(A, compute_uv=False)
    print(f"{kind:8s} {m}x{n}: {ms.value:8.3f} ms, {sw.value} sweeps, max rel err {np.max(np.abs(s - s_ref) / s_ref):.2e}")
