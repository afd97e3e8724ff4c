"""Thin Python façade over the C ABI (argument marshalling only — every step of the
path runs in libssa_b200's CUDA kernels).

    plan = Plan(img, window=(Lx, Ly), mask=None, wmask=None)   # step 1 (embedding)
    info = plan.decompose(r)                                    # step 2 (SVD)
    recs = plan.reconstruct([[0, 1], [2, 3]], add_rest=True)    # steps 3-4

Arrays: numpy (host) or torch CUDA tensors.  Images are indexed ``img[x, y]``
(shape (Nx, Ny)); MSSA systems are (N, s) with the series as columns and window
(L, 1).  L-side blocks are (L, k), K-side blocks (K, k).
"""
from __future__ import annotations

import ctypes as C

import time

import numpy as np

from . import _lib as lib


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _torch():
    import torch
    return torch


def _cur_stream():
    try:
        torch = _torch()
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:
        pass
    return None


class Plan:
    """An embedding of one array (step 1) with its device-side operator data."""

    def __init__(self, x, window, mask=None, wmask=None, *, dtype=None, path="auto", block_k=0,
                 tol=0.0, max_products=0, seed=0, stream=None, comm=None, band=None, ny_global=None,
                 precision=None, svd_method="lanczos"):
        """`comm`/`band`/`ny_global`: a band plan of the window-position partition (see
        dist.band_plan): x is this rank's sub-image = global columns [band[0], band[1] + Ly − 1)."""
        self._L = lib.load()
        self._h = C.c_void_p()
        lx, ly = int(window[0]), int(window[1])
        self._keep = []
        arr = lib.ssa_array()
        if _is_torch(x) and x.is_cuda:
            torch = _torch()
            if dtype is None:
                dtype = "f64" if x.dtype == torch.float64 else "f32"
            td = torch.float64 if dtype == "f64" else torch.float32
            xs = x.to(td).t().contiguous()          # storage with x fastest
            self._keep.append(xs)
            arr.nx, arr.ny = x.shape[0], x.shape[1]
            arr.data = xs.data_ptr()
            arr.on_device = 1
        else:
            xa = x.cpu().numpy() if _is_torch(x) else np.asarray(x)
            if dtype is None:
                dtype = "f64" if xa.dtype == np.float64 else "f32"
            xa = np.asfortranarray(xa, dtype=np.float64 if dtype == "f64" else np.float32)
            self._keep.append(xa)
            arr.nx, arr.ny = xa.shape
            arr.data = xa.ctypes.data
            arr.on_device = 0
        arr.ld = 0
        arr.dtype = lib.SSA_F64 if dtype == "f64" else lib.SSA_F32
        self.dtype = dtype
        self._np_dtype = np.float64 if dtype == "f64" else np.float32
        win = lib.ssa_window(lx, ly, None)
        if wmask is not None:
            wm = np.asfortranarray(np.asarray(wmask, dtype=np.uint8))
            assert wm.shape == (lx, ly), "wmask must be Lx x Ly"
            self._keep.append(wm)
            win.wmask = wm.ctypes.data
        mptr = None
        if mask is not None:
            m = np.asfortranarray(np.asarray(mask.cpu().numpy() if _is_torch(mask) else mask, dtype=np.uint8))
            assert m.shape == (arr.nx, arr.ny), "mask must be Nx x Ny"
            self._keep.append(m)
            mptr = m.ctypes.data
        o = lib.ssa_opts()
        o.stream = stream if stream is not None else _cur_stream()
        o.path = lib.PATHS[path] if isinstance(path, str) else int(path)
        o.block_k = int(block_k)
        o.tol = float(tol)
        o.max_products = int(max_products)
        o.seed = int(seed)
        # arithmetic type of the plan when it differs from the input's ("f32" / "f64")
        o.precision = {None: 0, "f32": 1, "f64": 2}[precision]
        o.svd_method = {"lanczos": 0, "eigen": 1}[svd_method]
        if precision is not None:
            self.dtype = precision
            self._np_dtype = np.float64 if precision == "f64" else np.float32
        if comm is not None:
            self._comm = comm
            o.comm = C.pointer(comm.struct())
            o.band_y0, o.band_y1 = band
            o.ny_global = int(ny_global) if ny_global is not None else 0
        self._opts = o
        lib.check(self._L.ssa_plan_create(C.byref(arr), C.byref(win), mptr, C.byref(o), C.byref(self._h)))
        self._keep = []  # the plan deep-copied its inputs
        inf = lib.ssa_plan_info_t()
        lib.check(self._L.ssa_plan_info(self._h, C.byref(inf)))
        self.nx, self.ny, self.lx, self.ly = inf.nx, inf.ny, inf.lx, inf.ly
        self.kx, self.ky, self.L, self.K = inf.kx, inf.ky, inf.L, inf.K
        self.n_valid, self.n_excluded = inf.n_valid, inf.n_excluded
        self.path = lib.PATH_NAMES.get(inf.path, str(inf.path))
        self.path_xv = lib.PATH_NAMES.get(inf.path_xv, str(inf.path_xv))
        self.path_xtu = lib.PATH_NAMES.get(inf.path_xtu, str(inf.path_xtu))
        self.full_window, self.full_kshape = bool(inf.full_window), bool(inf.full_kshape)
        self.decomp_info = None
        # band plans reconstruct the global image (the ranks' bands assembled)
        self.band = tuple(band) if (comm is not None and comm.world > 1) else None
        self.ny_out = int(ny_global) if self.band else self.ny

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._L.ssa_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------ shapes
    def weights(self) -> np.ndarray:
        w = np.zeros((self.nx, self.ny), dtype=np.int32, order="F")
        lib.check(self._L.ssa_get_weights(self._h, w.ctypes.data, 0))
        return w

    def kmask(self) -> np.ndarray:
        k = np.zeros((self.kx, self.ky), dtype=np.uint8, order="F")
        lib.check(self._L.ssa_get_kmask(self._h, k.ctypes.data, 0))
        return k.astype(bool)

    # ------------------------------------------------------------ products
    def matmul(self, v, transpose=False, out=None):
        """transpose=False: X·v (v: K x k -> L x k); transpose=True: Xᵀ·v (L x k -> K x k)."""
        nin, nout = (self.L, self.K) if transpose else (self.K, self.L)
        if _is_torch(v) and v.is_cuda:
            torch = _torch()
            td = torch.float64 if self.dtype == "f64" else torch.float32
            vv = v.reshape(nin, -1)
            k = vv.shape[1]
            vs = vv.to(td).t().contiguous()       # (k, nin) storage = column-major (nin, k)
            if out is None:
                o = torch.empty((k, nout), dtype=td, device=v.device)
            else:
                # the library writes k columns of nout values at out.data_ptr() (validate)
                if not (_is_torch(out) and out.is_cuda and out.dtype == td and tuple(out.shape) == (k, nout)
                        and out.is_contiguous() and out.device == v.device):
                    raise ValueError(f"out must be a contiguous CUDA tensor of shape ({k}, {nout}) and dtype {td}")
                o = out
            lib.check(self._L.ssa_matmul(self._h, int(transpose), vs.data_ptr(), nin, o.data_ptr(), nout, k, 1))
            return o.t()
        if out is not None:
            raise ValueError("out= is supported for CUDA tensor inputs only")
        va = np.asarray(v)
        squeeze = va.ndim == 1
        va = np.asfortranarray(va.reshape(nin, -1), dtype=self._np_dtype)
        k = va.shape[1]
        o = np.zeros((nout, k), dtype=self._np_dtype, order="F")
        lib.check(self._L.ssa_matmul(self._h, int(transpose), va.ctypes.data, nin, o.ctypes.data, nout, k, 0))
        return o[:, 0] if squeeze else o

    # ------------------------------------------------------------ decomposition
    def decompose(self, r, allow_not_converged=False):
        info = lib.ssa_decomp_info()
        st = self._L.ssa_decompose(self._h, int(r), C.byref(info))
        lib.check(st, allow=(5,) if allow_not_converged else ())
        self.decomp_info = {f: getattr(info, f) for f, _ in info._fields_}
        self.decomp_info["status"] = lib.STATUS[st]
        return self.decomp_info

    @property
    def r(self):
        v = C.c_int32()
        lib.check(self._L.ssa_get_rank(self._h, C.byref(v)))
        return v.value

    @property
    def sigma(self) -> np.ndarray:
        s = np.zeros(self.r, dtype=np.float64)
        lib.check(self._L.ssa_get_sigma(self._h, s.ctypes.data))
        return s

    @property
    def residuals(self) -> np.ndarray:
        """Residual bounds ||Xᵀu_i − σ_i v_i|| of the last decomposition (absolute)."""
        s = np.zeros(self.r, dtype=np.float64)
        lib.check(self._L.ssa_get_residuals(self._h, s.ctypes.data))
        return s

    def _getter(self, fn, n, device):
        if device:
            torch = _torch()
            td = torch.float64 if self.dtype == "f64" else torch.float32
            o = torch.empty((self.r, n), dtype=td, device="cuda")
            lib.check(fn(self._h, o.data_ptr(), 1))
            return o.t()
        o = np.zeros((n, self.r), dtype=self._np_dtype, order="F")
        lib.check(fn(self._h, o.ctypes.data, 0))
        return o

    def U(self, device=False):
        """Eigenvectors U (L x r, 𝔏-lex order); a CUDA tensor with device=True."""
        return self._getter(self._L.ssa_get_u, self.L, device)

    def V(self, device=False):
        """Factor vectors V_i = Xᵀ U_i / σ_i (K x r, 𝔎-lex order)."""
        return self._getter(self._L.ssa_get_v, self.K, device)

    def set_triples(self, sigma, U, V=None):
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        u = np.asfortranarray(U, dtype=self._np_dtype)
        v = None if V is None else np.asfortranarray(V, dtype=self._np_dtype)
        lib.check(self._L.ssa_set_triples(self._h, len(s), s.ctypes.data, u.ctypes.data,
                                          None if v is None else v.ctypes.data, 0))

    # ------------------------------------------------------------ reconstruction
    @staticmethod
    def _csr(groups):
        off = np.zeros(len(groups) + 1, dtype=np.int32)
        for g, idx in enumerate(groups):
            off[g + 1] = off[g] + len(idx)
        idx = np.array([i for g in groups for i in g], dtype=np.int32)
        if idx.size == 0:
            idx = np.zeros(1, dtype=np.int32)
        return off, idx

    def reconstruct(self, groups, add_rest=False, device=False, out=None):
        """List of (Nx, Ny) arrays X̃_g (NaN off 𝔑′); with add_rest a final residual array.
        Host results go to `out` when given: a C-contiguous (n, Ny, Nx) array of the plan's dtype
        (e.g. the numpy view of a pinned torch tensor), otherwise to a new array."""
        off, idx = self._csr(groups)
        n = len(groups) + (1 if add_rest else 0)
        if out is not None and not device:
            assert out.shape == (n, self.ny_out, self.nx) and out.dtype == self._np_dtype and out.flags["C_CONTIGUOUS"]
            lib.check(self._L.ssa_reconstruct(self._h, off.ctypes.data, idx.ctypes.data, len(groups),
                                              int(add_rest), out.ctypes.data, 0))
            return [out[g].T for g in range(n)]
        if device:
            torch = _torch()
            td = torch.float64 if self.dtype == "f64" else torch.float32
            t0 = time.perf_counter()
            o = torch.empty((n, self.ny_out, self.nx), dtype=td, device="cuda")
            t1 = time.perf_counter()
            lib.check(self._L.ssa_reconstruct(self._h, off.ctypes.data, idx.ctypes.data, len(groups),
                                              int(add_rest), o.data_ptr(), 1))
            # host ms of (output allocation by torch, the ABI call): diagnostics for bench.py
            self.last_reconstruct_host_ms = ((t1 - t0) * 1e3, (time.perf_counter() - t1) * 1e3)
            return [o[g].t() for g in range(n)]
        o = np.zeros((n, self.ny_out, self.nx), dtype=self._np_dtype)
        lib.check(self._L.ssa_reconstruct(self._h, off.ctypes.data, idx.ctypes.data, len(groups),
                                          int(add_rest), o.ctypes.data, 0))
        return [o[g].T for g in range(n)]

    def wcor(self, groups, contributions=False):
        """w-correlation matrix of the groups' reconstructions; with contributions=True
        also returns ||X̃_g||²_w / ||X||²_w per group."""
        off, idx = self._csr(groups)
        ng = len(groups)
        rho = np.zeros((ng, ng), dtype=np.float64, order="F")
        con = np.zeros(ng, dtype=np.float64)
        lib.check(self._L.ssa_wcor(self._h, off.ctypes.data, idx.ctypes.data, ng, rho.ctypes.data,
                                   con.ctypes.data))
        return (rho, con) if contributions else rho


    # ------------------------------------------------------------ parameters / forecast (rows f2, f3)
    def esprit(self, idx):
        """LS-ESPRIT / 2D-ESPRIT pairs (λ_k, μ_k) of the eigentriples idx."""
        ii = np.ascontiguousarray(list(idx), dtype=np.int32)
        lam = np.zeros(2 * len(ii)); mu = np.zeros(2 * len(ii))
        lib.check(self._L.ssa_esprit(self._h, ii.ctypes.data, len(ii), lam.ctypes.data, mu.ctypes.data))
        return lam[0::2] + 1j * lam[1::2], mu[0::2] + 1j * mu[1::2]

    def forecast(self, idx, M):
        """Vector forecast (Alg. 7) of the group idx, M steps: an (nx + M, s) array, series
        p holding z_1 .. z_{N_p + M} (updated reconstruction, then the forecast) and NaN below."""
        ii = np.ascontiguousarray(list(idx), dtype=np.int32)
        out = np.zeros((self.ny, self.nx + M), dtype=self._np_dtype)
        lib.check(self._L.ssa_forecast(self._h, ii.ctypes.data, len(ii), int(M), out.ctypes.data, self.nx + M, 0))
        return out.T


def version() -> str:
    return lib.load().ssa_version().decode()


def launch_count(reset: bool = False) -> int:
    return int(lib.load().ssa_launch_count(int(reset)))


def release_workspace() -> None:
    """Free the calling thread's cached solver workspace (ssa_release_workspace)."""
    lib.check(lib.load().ssa_release_workspace())
