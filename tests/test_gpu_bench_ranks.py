"""The N > 1 code path of bench.py rehearsed on ONE GPU.

`bench.py --gpus N` under torch.distributed.run shards ONE decomposition over the ranks by
window-position bands: each rank plans its sub-image (band + (Ly−1)-column halo) and the library's
communicator hook (dist.TorchComm) all-reduces the X·V partials, the K-side Grams and the
reconstruction numerators through the process group.  A multi-GPU box is not available to the tests,
so `--one-gpu-rehearsal` puts every rank on cuda:0 with a gloo group (the all-reduce of the device
buffers is synchronised by the host; no kernel waits on another rank's kernel).  The check is
correctness only: the launcher, the rendezvous, the callback on real device pointers and the JSON
contract, and that the sharded decomposition finds the singular values of the one-rank decomposition
(north star: top-r σ at relative error ≤ 1e-4 where the relative gap is ≥ 1e-3).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(args, world):
    env = dict(os.environ, PYTHONPATH=ROOT)
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
               "--gpus", str(world), "--one-gpu-rehearsal"] + args
    else:
        cmd = [sys.executable, "bench.py", "--gpus", "1", "--shard"] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]        # rank 0 alone prints, one line
    return json.loads(lines[0])


@pytest.mark.parametrize("config,world", [("c3", 2), ("c4", 3), ("c5", 2)])
def test_sharded_bench_matches_one_rank(config, world):
    args = ["--steps", "1", "--warmup", "1", "--config", config, "--no-cpu-baseline"]
    one = _bench(args, 1)
    many = _bench(args, world)
    assert many["n_gpus"] == world and many["scaling"] == "strong" and "rehearsal" in many
    for key in ("metric", "value", "unit", "ms_per_step", "e2e", "gpu_launches", "roofline", "clocks", "config"):
        assert key in many, key
    assert many["gpu_launches"] > 0 and many["config"]["workload"] == config
    assert many["e2e"]["h2d_bytes_per_step"] > 0 and many["e2e"]["d2h_bytes_per_step"] > 0
    assert 0.0 < many["roofline"]["frac"] < 1.0
    s1, sn = np.array(one["sigma_head"]), np.array(many["sigma_head"])
    np.testing.assert_allclose(sn, s1, rtol=1e-4)
    assert many["decomposition"]["n_converged"] > 0
