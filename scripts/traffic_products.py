"""One X·V or one Xᵀ·U block product (solver layout, C ABI) between cudaProfilerStart/Stop, for the ncu
DRAM-traffic capture behind roofline.traffic:
    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --csv --log-file gpurun_out/traffic_c5_xv.csv python scripts/traffic_products.py c5 xv
    python scripts/traffic_summary.py gpurun_out/traffic_c*_*.csv > profiles/r02/traffic.json
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1309_5050_b200 import Plan, _lib

cfg = sys.argv[1]
which = sys.argv[2] if len(sys.argv) > 2 else "xv"
path = sys.argv[3] if len(sys.argv) > 3 else "auto"
w = synth.get(cfg)
k = int(sys.argv[4]) if len(sys.argv) > 4 else w.block_k
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, path=path)
L = _lib.load()
td = torch.float64 if w.dtype == "f64" else torch.float32
ldq, ldp = (p.K + 31) // 32 * 32, (p.L + 31) // 32 * 32
Q = torch.randn(k, ldq, device="cuda", dtype=td)
P = torch.randn(k, ldp, device="cuda", dtype=td)
OutP = torch.empty(k, ldp, device="cuda", dtype=td)
OutQ = torch.empty(k, ldq, device="cuda", dtype=td)
for _ in range(2):
    _lib.check(L.ssa_matmul(p._h, 0, Q.data_ptr(), ldq, OutP.data_ptr(), ldp, k, 1))
    _lib.check(L.ssa_matmul(p._h, 1, P.data_ptr(), ldp, OutQ.data_ptr(), ldq, k, 1))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
if which == "xv":
    _lib.check(L.ssa_matmul(p._h, 0, Q.data_ptr(), ldq, OutP.data_ptr(), ldp, k, 1))
else:
    _lib.check(L.ssa_matmul(p._h, 1, P.data_ptr(), ldp, OutQ.data_ptr(), ldq, k, 1))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(cfg, which, p.path_xv if which == "xv" else p.path_xtu, k, "done", file=sys.stderr)
