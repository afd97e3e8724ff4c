"""World-size-2 gloo tests (CPU) of the multi-GPU band partition.

Each rank owns a band of origin columns; the partial X·V of the bands, summed through the
same `ssa_comm.allreduce_sum` callback the C library calls (invoked here through its ctypes
function pointer on host buffers), must equal the full product; Xᵀ·U is band-local; K-side
Grams sum to the full Gram.  Products come from the fp64 oracle (no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1309_5050_b200.dist import band_bounds, halo_columns, TorchComm


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
        sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
        y0, y1 = band_bounds(sh.ky, world, rank)
        band = oracle.Shapes(sh.nx, sh.ny, sh.lx, sh.ly, sh.nmask, sh.wmask, sh.kmask.copy(order="F"),
                             sh.weights)
        band.kmask[:, :y0] = 0
        band.kmask[:, y1:] = 0
        rng = np.random.default_rng(7)           # identical full blocks on every rank
        k = 3
        V = rng.normal(size=(sh.K, k))
        U = rng.normal(size=(sh.L, k))
        kx_all, ky_all = sh.kpos()
        sel = (ky_all >= y0) & (ky_all < y1)
        Vb = np.asfortranarray(V[sel])
        # X·V partial of the band, summed with the library's allreduce callback
        part = np.asfortranarray(oracle.xv(x, band, Vb))
        comm = TorchComm(device="cpu")
        fn = comm.struct().allreduce_sum
        assert fn(None, part.ctypes.data, part.size, 1, None) == 0
        full = oracle.xv(x, sh, V)
        err_xv = np.abs(part - full).max() / np.abs(full).max()
        # Xᵀ·U is band-local
        vb = oracle.xtu(x, band, U)
        err_xtu = np.abs(vb - oracle.xtu(x, sh, U)[sel]).max()
        # K-side Gram: sum of band Grams = full Gram
        G = np.asfortranarray(Vb.T @ Vb)
        assert fn(None, G.ctypes.data, G.size, 1, None) == 0
        err_g = np.abs(G - V.T @ V).max() / np.abs(V.T @ V).max()
        q.put((rank, err_xv, err_xtu, err_g, int(sel.sum())))
    finally:
        dist.destroy_process_group()


def test_band_partition_gloo_world2():
    world = 2
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
    for rank, e_xv, e_xtu, e_g, nk in res:
        assert e_xv < 1e-12, (rank, e_xv)
        assert e_xtu < 1e-12, (rank, e_xtu)
        assert e_g < 1e-12, (rank, e_g)
        assert nk > 0
