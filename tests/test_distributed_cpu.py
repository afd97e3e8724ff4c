"""World-size-2/3 gloo tests (CPU) of the multi-GPU band partition.

Each rank holds only its sub-image, the global columns [y0, y1 + Ly − 1) of its origin band plus
the (Ly−1)-column halo.  Checked with real collectives (the same `ssa_comm.allreduce_sum` callback
the C library calls, invoked through its ctypes function pointer on host buffers):
  * the sub-image's own 𝔎 (Alg. 6) is exactly the band of the global 𝔎;
  * the bands' X·V partials sum to the global X·V, Xᵀ·U is band-local, K-side Grams sum;
  * the reconstruction: the bands' diagonal-averaging numerators and hit counts, placed at their
    global columns and summed (the halos overlap), divide to the global X̃ (Alg. 4).
Products and averaging come from the fp64 oracle (no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1309_5050_b200.dist import band_bounds, band_slices, halo_columns, TorchComm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_band_bounds_cover_disjointly():
    for ky in (2, 7, 449, 3841):
        for world in (1, 2, 3, 8):
            if ky < world:
                continue
            b = [band_bounds(ky, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == ky
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [y1 - y0 for y0, y1 in b]
            assert max(sizes) - min(sizes) <= 1
    assert halo_columns(10, 20, 5) == (10, 24)
    with pytest.raises(ValueError):
        band_bounds(3, 4, 0)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.small_shaped(seed=41, nx=30, ny=26, window=(6, 5), wmask_drop=2)
        x = np.asarray(w.data, dtype=np.float64)
        sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)      # global (for the checks)
        (y0, y1), (c0, c1) = band_slices(sh.ny, sh.ly, world, rank)
        # this rank's own data: the sub-image and its mask
        xs = x[:, c0:c1]
        ms = None if w.mask is None else w.mask[:, c0:c1]
        sb = oracle.shapes(xs, w.window, mask=ms, wmask=w.wmask)
        kband = np.asarray(sh.kmask[:, y0:y1], dtype=np.uint8)
        ok_k = np.array_equal(np.asarray(sb.kmask), kband)
        rng = np.random.default_rng(7)           # identical full blocks on every rank
        k = 3
        V = rng.normal(size=(sh.K, k))
        U = rng.normal(size=(sh.L, k))
        kx_all, ky_all = sh.kpos()
        sel = (ky_all >= y0) & (ky_all < y1)
        Vb = np.asfortranarray(V[sel])
        comm = TorchComm(device="cpu")
        fn = comm.struct().allreduce_sum
        # X·V partial of the band (from the sub-image alone), summed with the library's callback
        part = np.asfortranarray(oracle.xv(xs, sb, Vb))
        assert fn(None, part.ctypes.data, part.size, 1, None) == 0
        full = oracle.xv(x, sh, V)
        err_xv = np.abs(part - full).max() / np.abs(full).max()
        # Xᵀ·U is band-local
        vb = oracle.xtu(xs, sb, U)
        err_xtu = np.abs(vb - oracle.xtu(x, sh, U)[sel]).max()
        # K-side Gram: sum of band Grams = full Gram
        G = np.asfortranarray(Vb.T @ Vb)
        assert fn(None, G.ctypes.data, G.size, 1, None) == 0
        err_g = np.abs(G - V.T @ V).max() / np.abs(V.T @ V).max()
        # reconstruction: numerators and hit counts of the sub-image at their global columns, summed
        s, Uo, Vo, _ = oracle.svd_dense(x, sh, 4)
        num = np.zeros((sh.nx, sh.ny))
        num[:, c0:c1] = oracle.diagsums(sb, Uo, Vo[sel], s)
        wts = np.zeros((sh.nx, sh.ny))
        wts[:, c0:c1] = sb.weights
        num = np.asfortranarray(num)
        wts = np.asfortranarray(wts)
        assert fn(None, num.ctypes.data, num.size, 1, None) == 0
        assert fn(None, wts.ctypes.data, wts.size, 1, None) == 0
        ok_w = np.array_equal(wts.astype(np.int64), sh.weights.astype(np.int64))
        rec = np.full((sh.nx, sh.ny), np.nan)
        m = wts > 0
        rec[m] = num[m] / wts[m]
        ref = oracle.reconstruct(x, sh, s, Uo, Vo, [[0, 1, 2, 3]])[0]
        err_rec = np.nanmax(np.abs(rec - ref)) / np.nanmax(np.abs(ref))
        ok_nan = np.array_equal(np.isnan(rec), np.isnan(ref))
        q.put((rank, err_xv, err_xtu, err_g, int(sel.sum()), ok_k, ok_w, err_rec, ok_nan))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_partition_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, e_xv, e_xtu, e_g, nk, ok_k, ok_w, e_rec, ok_nan in res:
        assert ok_k, rank                     # the sub-image's 𝔎 is the band of the global 𝔎
        assert e_xv < 1e-12, (rank, e_xv)
        assert e_xtu < 1e-12, (rank, e_xtu)
        assert e_g < 1e-12, (rank, e_g)
        assert nk > 0
        assert ok_w, rank                     # summed band hit counts = global 𝕎
        assert e_rec < 1e-12 and ok_nan, (rank, e_rec)
