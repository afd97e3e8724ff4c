"""Multi-GPU plumbing for the window-position (𝔎) band partition.

Each rank owns a contiguous band of origin columns κ_y ∈ [y0, y1) (reading Q13: bands along
the slow axis of the x-fastest layout) and holds only the image columns [y0, y1 + Ly − 1) — its
band plus the (Ly−1)-column halo — so its FFT grid, spectrum and K-side basis are those of the
sub-image.  Xᵀ·U is local to the band; the L x k partials of X·V and the k x k K-side Grams are
summed across ranks through the `ssa_comm.allreduce_sum` callback that the C library calls
(stream-ordered, in place); the reconstruction sums the bands' diagonal-averaging numerators and
hit counts (the halos overlap) and divides once.  This module provides the band bounds, the
sub-image slicing and a torch.distributed implementation of that callback (NCCL on GPUs; the same
code path works on host buffers with gloo, which is what the CPU tests exercise).
"""
from __future__ import annotations

import ctypes as C

from . import _lib as lib


def band_bounds(ky: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of the ky origin columns: the first (ky % world) ranks get one more."""
    if not (0 <= rank < world) or ky < world:
        raise ValueError(f"cannot split {ky} origin columns over {world} ranks")
    base, extra = divmod(ky, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def halo_columns(y0: int, y1: int, ly: int) -> tuple[int, int]:
    """Image columns a band needs: [y0, y1 + ly - 1) (the (Ly-1)-column halo)."""
    return y0, y1 + ly - 1


def band_slices(ny: int, ly: int, world: int, rank: int):
    """(y0, y1) origin band and the image columns [c0, c1) = [y0, y1 + ly − 1) of this rank."""
    y0, y1 = band_bounds(ny - ly + 1, world, rank)
    c0, c1 = halo_columns(y0, y1, ly)
    return (y0, y1), (c0, c1)


def band_plan(x, window, comm, mask=None, **kw):
    """The plan of this rank's band: the sub-image x[:, y0 : y1 + Ly − 1] (and mask), with the
    communicator and the band's global position."""
    from .api import Plan
    ny = x.shape[1]
    (y0, y1), (c0, c1) = band_slices(ny, int(window[1]), comm.world, comm.rank)
    sub = x[:, c0:c1]
    msk = None if mask is None else mask[:, c0:c1]
    return Plan(sub, window, mask=msk, comm=comm, band=(y0, y1), ny_global=ny, **kw)


_DTYPES = {0: "float32", 1: "float64"}


class TorchComm:
    """`ssa_comm` backed by a torch.distributed process group.

    The callback wraps the raw buffer the library hands over (device pointer for NCCL, host
    pointer for gloo) as a tensor and all-reduces it in place with SUM."""

    def __init__(self, group=None, device: str = "cuda"):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.device = device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._fn = lib.ALLREDUCE_FN(self._allreduce)
        self._struct = None

    def _tensor(self, ptr: int, count: int, dtype: int):
        import torch
        tdt = torch.float32 if dtype == 0 else torch.float64
        if self.device == "cuda":
            class _Cai:
                __cuda_array_interface__ = {"shape": (count,), "typestr": "<f4" if dtype == 0 else "<f8",
                                            "data": (ptr, False), "version": 3, "strides": None}
            return torch.as_tensor(_Cai(), device="cuda")
        buf = (C.c_float if dtype == 0 else C.c_double) * count
        return torch.frombuffer(buf.from_address(ptr), dtype=tdt)

    def _allreduce(self, user, ptr, count, dtype, stream):
        try:
            t = self._tensor(ptr, count, dtype)
            if self.device == "cuda":
                import torch
                s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
                with torch.cuda.stream(s):
                    self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
            else:
                self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
            return 0
        except Exception:  # errors must not cross the C ABI
            return 1

    def struct(self) -> lib.ssa_comm:
        if self._struct is None:
            self._struct = lib.ssa_comm(self.rank, self.world, None, self._fn)
        return self._struct


class LocalComm:
    """A stand-in `ssa_comm` for one process that plays rank `rank` of `world` with an identity
    all-reduce: the library then computes exactly the band-local operator (X·V partial of the
    band, band-local Xᵀ·U), which is what the single-GPU band tests check against the oracle."""

    def __init__(self, rank: int = 0, world: int = 2):
        self.rank, self.world = rank, world
        self._fn = lib.ALLREDUCE_FN(lambda user, ptr, count, dtype, stream: 0)
        self._struct = None

    def struct(self) -> lib.ssa_comm:
        if self._struct is None:
            self._struct = lib.ssa_comm(self.rank, self.world, None, self._fn)
        return self._struct
