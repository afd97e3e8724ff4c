"""Test helper: an `ssa_comm` for `world` host threads of ONE process on one GPU.  Each thread owns
a band plan on its own CUDA stream; the library calls allreduce_sum from inside its decomposition /
reconstruction, and the threads meet at a barrier where thread 0 sums the device buffers.  No kernel
ever waits on another rank's kernel (the host threads synchronise), so this checks the band
partition's arithmetic end to end on one GPU — not its timing."""
import threading

from paper_1309_5050_b200 import _lib as lib


class ThreadGroup:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world, timeout=600)
        self.bufs = [None] * world
        self.failed = False


class ThreadComm:
    def __init__(self, group: ThreadGroup, rank: int):
        self.group, self.rank, self.world = group, rank, group.world
        self._fn = lib.ALLREDUCE_FN(self._allreduce)
        self._struct = None
        self.calls = 0

    def _allreduce(self, user, ptr, count, dtype, stream):
        import torch
        g = self.group
        try:
            s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            s.synchronize()

            class _Cai:
                __cuda_array_interface__ = {"shape": (count,), "typestr": "<f4" if dtype == 0 else "<f8",
                                            "data": (ptr, False), "version": 3, "strides": None}
            g.bufs[self.rank] = torch.as_tensor(_Cai(), device="cuda")
            g.barrier.wait()
            if self.rank == 0:
                tot = g.bufs[0].clone()
                for b in g.bufs[1:]:
                    tot += b
                for b in g.bufs:
                    b.copy_(tot)
                torch.cuda.synchronize()
            g.barrier.wait()
            self.calls += 1
            return 0
        except Exception:  # noqa: BLE001 — errors must not cross the C ABI
            g.failed = True
            try:
                g.barrier.abort()
            except Exception:  # noqa: BLE001
                pass
            return 1

    def struct(self):
        if self._struct is None:
            self._struct = lib.ssa_comm(self.rank, self.world, None, self._fn)
        return self._struct


def run_threads(world, fn):
    """Run fn(rank) on `world` threads; returns the results, re-raising the first exception."""
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
