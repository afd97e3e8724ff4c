"""One small TC product (mssa_ragged-like), prints the error or the relative error vs a float64 numpy reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_1309_5050_b200 import Plan
w = synth.config2(seed=21, n=777, s=3, L=300)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = Plan(w.data, w.window, dtype="f32", path="tc", block_k=32)
rng = np.random.default_rng(0)
V = rng.normal(size=(p.K, k)).astype(np.float32)
try:
    U = p.matmul(V)
    x = np.asarray(w.data, np.float32).astype(np.float64)
    L = 300; Kp = 777 - 300 + 1
    ref = np.zeros((L, k))
    for s_ in range(3):
        H = np.array([x[i:i + Kp, s_] for i in range(L)])
        ref += H @ V[s_ * Kp:(s_ + 1) * Kp].astype(np.float64)
    print("ok relerr", np.linalg.norm(U - ref) / np.linalg.norm(ref))
except Exception as e:
    print("ERR", e)
