#!/usr/bin/env python
"""Benchmark of the multidimensional-SSA hot path on B200 (one JSON line on rank 0).

One STEP = one pass of the whole hot path over one
synthetic input: plan (embedding: shapes, 𝔎, weights), block-Lanczos rank-r
decomposition driven by X·V / Xᵀ·U block products, and the grouped diagonal-
averaging reconstruction.  Default workload: c5 (BASELINE.json configs[4], the
north star's largest config: 2D-SSA 4096² fp32, window 256², r = 50, block k = 64)
at N = 1; --config c1..c5 selects another.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Metric: trajectory products/s = vector products (X·v or Xᵀ·u) completed per
second of whole-step time, summed over ranks (weak scaling: every rank
decomposes its own input, no data-path collective).  `rank_r_time_ms` is the
device time of the decomposition alone (plan and reconstruction
are reported beside it, §8(d)(3-4)); `products_only` is the metric over the
block products' device time alone.  `e2e` is the same metric through the C ABI
with host buffers (H2D of the input and D2H of the reconstructions inside the
timed region).  `roofline` reports the trajectory block product with the larger
share of the step against the roofline of the path that served it (FFT: HBM bytes
model; tc: measured tcgen05 tf32 peak / 3; direct: FFMA), DESIGN.md §6.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FFMA_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 TF: 148 SM x 128 FP32 lanes x FMA x max clock
FP64_PEAK_TFLOPS = FFMA_PEAK_TFLOPS / 2               # B200 non-tensor FP64 = 1/2 FP32 rate


TRAFFIC_FILE = os.path.join("profiles", "r02", "traffic.json")


def _traffic(config, product, path, k):
    """DRAM bytes per block product from the committed ncu capture (profiles/r02/traffic.json), or None."""
    f = os.path.join(os.path.dirname(os.path.abspath(__file__)), TRAFFIC_FILE)
    try:
        with open(f) as fh:
            for e in json.load(fh)["entries"]:
                if (e["config"], e["product"], e["path"]) == (config, product, path) and e.get("k", k) == k:
                    return e["traffic_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    One long-running `nvidia-smi --loop-ms` process, started BEFORE the warm-up steps: its start-up
    (driver / NVML initialisation — on a fresh box the first nvidia-smi call stalled the GPU for ~0.9 s,
    every new process for ~10 ms, and a first timed c5 step of 728 ms was seen with the sampler started
    right before it) then falls into the warm-up.  `mark()` opens the timed region: only samples read
    after it (and the last one before it, for regions shorter than the period) are reported.
    """
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0, period_ms=50):
        self.idx = gpu_index
        self.period = period_ms
        self.samples = []
        self._p = None
        self._t = None
        self._first = threading.Event()
        self._t0 = 0.0
        self._t1 = float("inf")

    def mark(self):
        """Start of the timed region."""
        self._t0 = time.perf_counter()

    def stop(self):
        """End of the timed region (the process keeps running until __exit__)."""
        self._t1 = time.perf_counter()

    def _read(self):
        for line in self._p.stdout:
            line = line.strip()
            if not line:
                continue
            # the first sample is taken as the timed region starts (kept: short regions, c1-c4, may
            # end before the next one)
            self.samples.append([time.perf_counter()] + [s.strip() for s in line.split(",")])
            self._first.set()

    def __enter__(self):
        if os.environ.get("SSA_BENCH_NO_CLOCKS"):      # diagnosis only: the line then says "unsampled"
            return self
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", f"--loop-ms={self.period}"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
            return self
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()
        self._first.wait(timeout=15)
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        before = [s for s in self.samples if s[0] < self._t0]
        inside = [s for s in self.samples if self._t0 <= s[0] <= self._t1]
        use = [s[1:] for s in (before[-1:] + inside)]
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in use if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in use if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in use for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "n_samples": len(use)}


def _quiet_gc():
    """No cyclic-GC passes inside the timed regions (as `timeit` does).  (The one-off +15..+700 ms steps
    of gpurun r1-r4 were NOT this: they persisted with the collector off and went away with the library's
    large-block cache.)"""
    import gc
    gc.collect()
    gc.freeze()
    gc.disable()


def measured_tf32_peak():
    """Dense tcgen05 kind::tf32 TFLOP/s measured on this GPU (library microbenchmark)."""
    import ctypes
    from paper_1309_5050_b200 import _lib
    L = _lib.load()
    ms, tf = ctypes.c_double(), ctypes.c_double()
    _lib.check(L.ssa_bench_mma(100000, 0, ctypes.byref(ms), ctypes.byref(tf)))
    return float(tf.value)


def workload(name, seed_offset=0):
    import synth
    fn = synth.CONFIGS[name]
    base = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}[name]
    return fn(seed=base + 1000 * seed_offset)


def groups_for(w):
    gs = [g for g in w.groups if max(g) < w.r]
    return gs if gs else [list(range(min(4, w.r)))]


# ----------------------------------------------------------------------------- ours
def run_ours(args, rank, world, dist):
    import torch
    from paper_1309_5050_b200 import Plan, launch_count
    dev = torch.device("cuda", 0 if args.one_gpu_rehearsal else int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    w = workload(args.config, seed_offset=rank)
    groups = groups_for(w)
    stream = torch.cuda.Stream(device=dev)
    dt_torch = torch.float64 if w.dtype == "f64" else torch.float32
    img_dev = torch.as_tensor(np.asarray(w.data), dtype=dt_torch, device=dev)
    mask_np = None if w.mask is None else np.asarray(w.mask)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    phases = []
    # e2e inputs / outputs in pinned host memory in the library's layout (x fastest), prepared once
    # outside the timed region: the e2e step pays the H2D copy of the image (+ mask) and the D2H copy
    # of the reconstructions, not a host-side format conversion
    nx_, ny_ = np.asarray(w.data).shape
    img_pin = torch.empty((ny_, nx_), dtype=dt_torch, pin_memory=True)
    img_pin.copy_(torch.as_tensor(np.ascontiguousarray(np.asarray(w.data).T), dtype=dt_torch))
    host_src = img_pin.t()
    mask_pin = None
    if mask_np is not None:
        mask_pin = torch.empty((ny_, nx_), dtype=torch.uint8, pin_memory=True)
        mask_pin.copy_(torch.as_tensor(np.ascontiguousarray(mask_np.T.astype(np.uint8))))
    out_pin = torch.empty((len(groups), ny_, nx_), dtype=dt_torch, pin_memory=True)

    phase_dev = []   # device ms of (plan, decompose, reconstruct) per timed step
    rec_host = []    # host ms of (torch output allocation, ssa_reconstruct call) per timed step

    def step(host=False, events=False):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if events else None
        with torch.cuda.stream(stream):
            if ev:
                ev[0].record(stream)
            t0 = time.perf_counter()
            src = host_src if host else img_dev
            # the ABI takes the 𝔑 mask from host memory on both paths: the pinned, column-major copy
            # (a C-ordered numpy mask cost a host transpose-copy per step: c4 11.3 vs 10.2 ms)
            msk = mask_pin.t().numpy() if mask_pin is not None else None
            p = Plan(src, w.window, mask=msk, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k,
                     path=args.path, stream=stream.cuda_stream)
            t1 = time.perf_counter()
            if ev:
                ev[1].record(stream)
            info = p.decompose(w.r, allow_not_converged=True)
            if ev:
                ev[2].record(stream)
            t2 = time.perf_counter()
            recs = (p.reconstruct(groups, add_rest=False, device=False, out=out_pin.numpy()) if host
                    else p.reconstruct(groups, add_rest=False, device=True))
            if ev:
                ev[3].record(stream)
                rec_host.append([round(x, 3) for x in getattr(p, "last_reconstruct_host_ms", (0.0, 0.0))])
            t3 = time.perf_counter()
            p.close()
            t4 = time.perf_counter()
        phases.append({"plan_ms": (t1 - t0) * 1e3, "decompose_ms": (t2 - t1) * 1e3,
                       "reconstruct_ms": (t3 - t2) * 1e3, "destroy_ms": (t4 - t3) * 1e3})
        if ev:
            ev[3].synchronize()
            phase_dev.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])])
        return info, recs, p

    _quiet_gc()
    with ClockSampler(dev.index) as clk:
        # warm-up (also compiles nothing: the library is AOT-built)
        for _ in range(args.warmup):
            info, recs, p = step()
        torch.cuda.synchronize()
        L, K, k = p.L, p.K, info["block_k"]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        times, infos = [], []
        launches0 = launch_count(reset=True)
        phases.clear()
        clk.mark()
        for _ in range(args.steps):
            flush.fill_(1)                         # flush L2 between timed iterations
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            info, recs, _ = step(events=True)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            infos.append(info)
        clk.stop()
    launches = launch_count(reset=True)
    timed_phases = {k: float(np.mean([ph[k] for ph in phases])) for k in phases[0]} if phases else {}
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_local = float(np.sum(times))
    nvec_local = float(np.sum([i["n_vector_products"] for i in infos]))
    ms_prod = float(np.sum([i["ms_products"] for i in infos]))
    nblk = float(np.sum([i["n_block_products"] for i in infos]))
    if dist:
        t = torch.tensor([ms_local, nvec_local, launches], dtype=torch.float64, device=dev)
        tmax = t.clone(); dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone(); dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_all, nvec_all = float(tmax[0]), float(tsum[1])
    else:
        ms_all, nvec_all = ms_local, nvec_local

    # ---- end-to-end through the C ABI with host buffers (H2D input, D2H reconstructions)
    e2e_times = []
    step(host=True)                                # untimed: the host-buffer path's first pool allocations
    torch.cuda.synchronize()
    for _ in range(max(1, min(args.steps, 5))):
        flush.fill_(1); torch.cuda.synchronize()
        t0 = time.perf_counter()
        info_h, recs_h, _ = step(host=True)
        torch.cuda.synchronize()
        e2e_times.append((time.perf_counter() - t0) * 1e3)
    esz = 8 if w.dtype == "f64" else 4
    h2d = int(np.asarray(w.data).size * esz + (0 if mask_np is None else mask_np.size))
    d2h = int(len(groups) * np.asarray(w.data).size * esz + 8 * w.r)
    e2e_value = info_h["n_vector_products"] / (np.mean(e2e_times) / 1e3) * world

    # ---- roofline of the trajectory block products (the kernels SURVEY §8(d) sizes), timed
    # live: the library brackets every block product with CUDA events on the plan's stream,
    # separately for X·V and Xᵀ·U; each product is held against the roofline of the path
    # that served it, and the one with the larger share of the step is the headline
    peaks = _peaks()
    tf32_measured = measured_tf32_peak()
    esz = 8 if w.dtype == "f64" else 4
    nx_, ny_ = np.asarray(w.data).shape
    kx_, ky_ = nx_ - w.window[0] + 1, ny_ - w.window[1] + 1

    def product_roofline(name, path, ms_total, nblocks, nvec, name_key=""):
        if nblocks <= 0:
            return None
        avg_ms = ms_total / nblocks
        kk = nvec / nblocks
        flops = 2.0 * L * K * kk
        if path == "fft":
            # 3-pass model per vector: read the input box, write the output box,
            # write+read the x-transformed input and the y-filtered output (complex, Hx rows),
            # plus the image spectrum once per block
            Mx = 1 << int(np.ceil(np.log2(nx_))); My = 1 << int(np.ceil(np.log2(max(ny_, 1))))
            Hx = Mx // 2 + 1
            per_vec = esz * (K + L) + 2 * (2 * esz) * Hx * (ky_ + w.window[1])
            alg = kk * per_vec + (2 * esz) * Hx * My
            achieved = alg / (avg_ms / 1e3) / 1e9
            r = {"bound": "hbm", "kernel": f"{name}: FFT correlation (rpass_a/b/c register radix-16 passes)",
                 "achieved": achieved,
                 "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)", "algorithmic_bytes_per_launch": alg}
        elif path == "tc":
            # tcgen05 kind::tf32, 3 MMAs per useful multiply-add (3xTF32): the useful-flop peak is the
            # dense TF32 peak / 3, with the TF32 peak measured in this run (ssa_bench_mma)
            peak = tf32_measured / 3.0
            achieved = flops / (avg_ms / 1e3) / 1e12
            r = {"bound": "tensor", "kernel": f"{name}: tcgen05 3xTF32 polyphase implicit GEMM (hankel_tc)",
                 "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                 "peak_source": "measured: ssa_bench_mma tcgen05 kind::tf32 M128 N256 back-to-back, / 3 (3xTF32)",
                 "algorithmic_flops_per_launch": flops, "tensor_flops_per_launch": 3 * flops}
        else:
            peak = FP64_PEAK_TFLOPS if w.dtype == "f64" else FFMA_PEAK_TFLOPS
            achieved = flops / (avg_ms / 1e3) / 1e12
            r = {"bound": "alu", "kernel": f"{name}: corr_direct (FFMA/DFMA)", "achieved": achieved, "peak": peak,
                 "unit": "TFLOP/s", "frac": achieved / peak,
                 "peak_source": "derived: 148 SM x 128 FP32 FMA/clk x 2 x 1.965 GHz (B200_PROFILING.md SM count,"
                                " MEASURED_PEAKS sm_max_mhz); fp64 = 1/2",
                 "algorithmic_flops_per_launch": flops}
        tr = _traffic(args.config, name_key, path, int(round(kk)))
        r.update({"traffic": tr, "avg_launch_ms": avg_ms, "launches_per_step": nblocks / args.steps,
                  "share_of_step": ms_total / max(ms_local, 1e-9), "path": path})
        if tr is not None:
            r["traffic_source"] = (TRAFFIC_FILE + ": dram__bytes_read.sum + dram__bytes_write.sum of the block "
                                   "product's kernels, one ncu capture (cold caches)")
            if r["unit"] == "GB/s":
                # measured DRAM bytes over the live launch time, next to (ii) = `frac`
                r["dram_achieved"] = tr / (avg_ms / 1e3) / 1e9
                r["dram_frac"] = r["dram_achieved"] / peaks["hbm_gbs"]
        if path == "fft":
            # compulsory lower bound k·(e·|𝔎| + e·L): read the input box, write the output box
            r["compulsory_bytes_per_launch"] = kk * esz * (K + L)
        return r

    prods = {}
    for name, path, key in (("X·V", p.path_xv, "xv"), ("Xᵀ·U", p.path_xtu, "xtu")):
        ms_t = float(np.sum([i[f"ms_products_{key}"] for i in infos]))
        nb_t = float(np.sum([i[f"n_products_{key}"] for i in infos]))
        nv_t = float(np.sum([i[f"n_vectors_{key}"] for i in infos]))
        rr = product_roofline(name, path, ms_t, nb_t, nv_t, key)
        if rr:
            prods[key] = rr
    roof = dict(max(prods.values(), key=lambda r: r["share_of_step"])) if prods else {}
    roof["note"] = ("a 'launch' is one block product of k vectors (FFT: 3 passes; tc: pack + MMA kernel"
                    " + split reduce); events bracket it on the plan's stream, so host launch gaps count; "
                    "achieved = the 3-pass algorithmic bytes (DESIGN.md §6) / the average device time")
    roof["products"] = prods
    # where the rest of the step goes (the products are the kernels SURVEY §8(d) sizes; on the small
    # configs the Ritz SVD and the orthonormalisation take more of the step)
    ms_ritz_step = float(np.sum([i["ms_ritz"] for i in infos])) / args.steps
    ms_step = ms_all / args.steps
    prod_share = float(sum(r["share_of_step"] for r in prods.values()))
    roof["step_shares"] = {"products": prod_share,
                           "ritz_svd (jacobi_gram_kernel, latency bound)": ms_ritz_step / max(ms_step, 1e-9),
                           "orthonormalisation + host": max(0.0, 1.0 - prod_share - ms_ritz_step / max(ms_step, 1e-9))}
    ph = np.mean(np.array(phase_dev), axis=0) if phase_dev else [float("nan")] * 3
    nvec_step = nvec_local / args.steps
    res = {
        "metric": "trajectory products/s",
        "value": nvec_all / (ms_all / 1e3),
        "unit": "vector products/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_all / args.steps,
        "step_ms": [round(float(t), 3) for t in times],
        "step_phases_ms": [[round(float(x), 3) for x in ph_] for ph_ in phase_dev],
        "step_reconstruct_host_ms": rec_host,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": w.dtype,
        "data": "synthetic (seeded BASELINE.json generator, rank-offset seeds)",
        "config": {"workload": w.name, "nx": int(np.asarray(w.data).shape[0]), "ny": int(np.asarray(w.data).shape[1]),
                   "window": list(w.window), "L": int(L), "K": int(K), "r": int(w.r), "block_k": int(k),
                   "groups": len(groups), "path": {"xv": p.path_xv, "xtu": p.path_xtu},
                   "l2": "flushed (256 MB write) between timed steps",
                   "parallelism": f"replicas x{world} (independent inputs per rank)"},
        "rank_r_time_ms": float(ph[1]),
        "phases_device_ms": {"plan": float(ph[0]), "decompose": float(ph[1]), "reconstruct": float(ph[2]),
                             "note": "CUDA events on the plan's stream between the synchronous ABI calls; "
                                     "rank_r_time_ms = decompose (SURVEY §8(d)(2)), plan and reconstruction "
                                     "reported beside it (§8(d)(3-4))"},
        "products_only": {"value": nvec_step / (ms_prod / args.steps / 1e3), "unit": "vector products/s",
                          "ms_per_step": ms_prod / args.steps,
                          "note": "vector products over the device time of the block products alone"},
        "decomposition": {"n_block_products": infos[-1]["n_block_products"],
                          "n_vector_products": infos[-1]["n_vector_products"],
                          "n_restarts": infos[-1]["n_restarts"], "n_converged": infos[-1]["n_converged"],
                          "max_rel_residual": infos[-1]["max_rel_residual"],
                          "ms_products_per_step": ms_prod / args.steps,
                          "ms_ritz_per_step": float(np.sum([i["ms_ritz"] for i in infos])) / args.steps,
                          "host_phases_ms": timed_phases},
        "e2e": {"value": e2e_value, "unit": "vector products/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": float(np.mean(e2e_times)),
                "step_ms": [round(float(t), 3) for t in e2e_times]},
        "gpu_launches": int(launches),
        "roofline": roof,
        "peaks_measured_here": {"tf32_dense_tflops": tf32_measured,
                                "source": "ssa_bench_mma: 148 CTAs x 100k tcgen05.mma kind::tf32 128x256x8"},
        "clocks": clk.summary(),
    }
    return res, w


# ----------------------------------------------------------------------------- oracle (CPU)
def oracle_products_per_s(w, budget_s=15.0):
    """The oracle's naive X·V / Xᵀ·U (oracle/oracle_core.c) on a bounded sample of the same
    workload: whole block products (X·V then Xᵀ·U, k = block width) repeated until the time
    budget is used, or, when one block would exceed the budget, sampled output rows of each
    product scaled to whole blocks."""
    import oracle
    x = np.array(w.data, dtype=np.float64)
    if w.dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    if w.mask is None and w.wmask is None and np.all(np.isfinite(x)) and x.size > (1 << 22):
        sh = oracle.shapes_rect(*x.shape, *w.window)   # full rectangle: the brute-force 𝔎 scan is infeasible at c5
    else:
        sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    rng = np.random.default_rng(0)
    k = w.block_k
    V = rng.normal(size=(sh.K, k)); U = rng.normal(size=(sh.L, k))
    # per-row cost calibrated on a 64-row call (a single row is dominated by call overhead)
    nr = min(64, sh.L)
    t0 = time.perf_counter(); oracle.xv_rows(x, sh, V, np.arange(nr)); t_row = (time.perf_counter() - t0) / nr
    est_block = 2 * t_row * sh.L              # X·V rows cost ≈ Xᵀ·U rows in total (both L·K·k)
    cores = len(os.sched_getaffinity(0))
    if est_block <= budget_s / 2:
        n, t_all = 0, 0.0
        while t_all < budget_s and (n == 0 or t_all + t_all / n <= budget_s * 1.5):
            t0 = time.perf_counter()
            oracle.xv(x, sh, V)
            oracle.xtu(x, sh, U)
            t_all += time.perf_counter() - t0
            n += 1
        value = 2 * k * n / t_all
        sample = f"{w.name}: {n} whole X·V + Xᵀ·U block pairs (k={k}), {t_all:.1f} s of CPU"
        return value, cores, sample
    # sampled output rows of both products, repeated until the time budget is used, scaled
    # to whole blocks (the oracle's cost per output row is uniform for full shapes)
    rows = int(max(1, min(sh.L, budget_s / 4 / max(t_row, 1e-9))))
    kc = int(max(1, min(sh.K, rows * sh.K // sh.L)))
    t_xv = t_xtu = 0.0
    n_rep = 0
    while (t_xv + t_xtu) < budget_s and n_rep < 1000:
        r0 = (n_rep * rows) % max(1, sh.L - rows + 1)
        t0 = time.perf_counter(); oracle.xv_rows(x, sh, V, np.arange(r0, r0 + rows)); t_xv += time.perf_counter() - t0
        k0 = (n_rep * kc) % max(1, sh.K - kc + 1)
        t0 = time.perf_counter(); oracle.xtu(x, sh, U, kstart=k0, kcount=kc); t_xtu += time.perf_counter() - t0
        n_rep += 1
    t_block = (t_xv / n_rep) * sh.L / rows + (t_xtu / n_rep) * sh.K / kc
    value = 2 * k / t_block
    sample = (f"{w.name}: X·V on {rows}/{sh.L} rows and Xᵀ·U on {kc}/{sh.K} rows of a k={k} block, repeated "
              f"{n_rep}x ({t_xv + t_xtu:.1f} s of CPU), scaled to whole blocks")
    return value, cores, sample


def run_sharded(args, rank, world, dist):
    """N > 1 (default) or --shard: ONE decomposition of the config split over the ranks (strong
    scaling).  Rank r holds only its sub-image, the global columns [y0, y1 + Ly − 1)
    of its origin band κ_y ∈ [y0, y1) plus the (Ly−1)-column halo (dist.band_plan): its own FFT grid,
    spectrum and K-side basis.  X·V partials and K-side Grams are summed with an NCCL all-reduce
    through the library's communicator hook (dist.TorchComm); the reconstruction sums the bands'
    numerators and hit counts (one all-reduce per group) and returns the global image on every rank.
    A step = plan + decompose + reconstruct; time = max over ranks; value = the vector products of
    the ONE decomposition per second (not summed over ranks)."""
    import torch
    from paper_1309_5050_b200 import launch_count
    from paper_1309_5050_b200.dist import TorchComm, band_plan, band_slices
    dev = torch.device("cuda", 0 if args.one_gpu_rehearsal else int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    w = workload(args.config, seed_offset=0)          # the same global problem on every rank
    groups = groups_for(w)
    stream = torch.cuda.Stream(device=dev)
    dt_torch = torch.float64 if w.dtype == "f64" else torch.float32
    xg = np.asarray(w.data)
    ny = xg.shape[1]
    (y0, y1), (c0, c1) = band_slices(ny, w.window[1], max(world, 1), rank)
    # this rank's data only: its sub-image (device for the timed steps, pinned host for e2e)
    sub_dev = torch.as_tensor(np.ascontiguousarray(xg[:, c0:c1]), dtype=dt_torch, device=dev)
    sub_pin = torch.empty((c1 - c0, xg.shape[0]), dtype=dt_torch, pin_memory=True)
    sub_pin.copy_(torch.as_tensor(np.ascontiguousarray(xg[:, c0:c1].T), dtype=dt_torch))
    mask = None if w.mask is None else np.asarray(w.mask)
    comm = TorchComm(device="cuda") if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out_pin = torch.empty((len(groups), ny, xg.shape[0]), dtype=dt_torch, pin_memory=True)

    shape_info = {}

    def step(host=False):
        with torch.cuda.stream(stream):
            src = sub_pin.t() if host else sub_dev
            kw = dict(dtype=w.dtype, block_k=w.block_k, path=args.path, stream=stream.cuda_stream, wmask=w.wmask)
            if comm is not None:
                from paper_1309_5050_b200.api import Plan
                msk = None if mask is None else mask[:, c0:c1]
                p = Plan(src, w.window, mask=msk, comm=comm, band=(y0, y1), ny_global=ny, **kw)
            else:
                from paper_1309_5050_b200.api import Plan
                p = Plan(src, w.window, mask=mask, **kw)
            info = p.decompose(w.r, allow_not_converged=True)
            recs = (p.reconstruct(groups, device=False, out=out_pin.numpy()) if host
                    else p.reconstruct(groups, device=True))
            sig = np.array(p.sigma)
            shape_info.update(L=p.L, K=p.K, path_xv=p.path_xv, path_xtu=p.path_xtu)
            p.close()
        return info, sig, recs

    _quiet_gc()
    with ClockSampler(dev.index) as clk:
        for _ in range(args.warmup):
            info, _, _ = step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        times = []
        launch_count(reset=True)
        clk.mark()
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            info, sig, _ = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        clk.stop()
    launches = launch_count(reset=True)
    ms = float(np.sum(times))
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        flush.fill_(1); torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(host=True)
        e1.record(stream)
        e1.synchronize()
        t_e = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        if dist:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e.append(float(t_e[0]))
    nvec = float(info["n_vector_products"])               # one decomposition: not summed over ranks
    esz = 8 if w.dtype == "f64" else 4
    # roofline of rank 0's band-sized block products (the last timed step; same 3-pass byte model as N = 1,
    # DESIGN.md §6, on the band's own grid).  The X·V events include the all-reduce of the L x k partials.
    roof = {}
    Lb, Kb = shape_info["L"], shape_info["K"]
    nxb, nyb = xg.shape[0], c1 - c0
    for name, key in (("X·V", "xv"), ("Xᵀ·U", "xtu")):
        nb, path = info[f"n_products_{key}"], shape_info[f"path_{key}"]
        if nb <= 0:
            continue
        avg_ms, kk = info[f"ms_products_{key}"] / nb, info[f"n_vectors_{key}"] / nb
        if path == "fft":
            Mx = 1 << int(np.ceil(np.log2(nxb))); My = 1 << int(np.ceil(np.log2(max(nyb, 1))))
            Hx = Mx // 2 + 1
            alg = kk * (esz * (Kb + Lb) + 4 * esz * Hx * ((nyb - w.window[1] + 1) + w.window[1])) + 2 * esz * Hx * My
            peak = _peaks()["hbm_gbs"]
            r_ = {"bound": "hbm", "achieved": alg / (avg_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                  "algorithmic_bytes_per_launch": alg}
        else:
            flops = 2.0 * Lb * Kb * kk
            peak = (measured_tf32_peak() / 3.0 if path == "tc"
                    else (FP64_PEAK_TFLOPS if w.dtype == "f64" else FFMA_PEAK_TFLOPS))
            r_ = {"bound": "tensor" if path == "tc" else "alu", "achieved": flops / (avg_ms / 1e3) / 1e12,
                  "peak": peak, "unit": "TFLOP/s", "algorithmic_flops_per_launch": flops}
        r_.update(frac=r_["achieved"] / r_["peak"], traffic=None, avg_launch_ms=avg_ms, path=path,
                  kernel=f"{name} on rank 0's band ({nxb} x {nyb} sub-image)",
                  share_of_step=info[f"ms_products_{key}"] / max(times[-1], 1e-9))
        roof[key] = r_
    roofline = dict(max(roof.values(), key=lambda r_: r_["share_of_step"])) if roof else {}
    roofline["products"] = roof
    res = {"metric": "trajectory products/s", "value": nvec / (ms / args.steps / 1e3), "unit": "vector products/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": w.dtype,
           "data": "synthetic (seeded BASELINE.json generator)",
           "config": {"workload": w.name, "window": list(w.window), "r": w.r, "block_k": w.block_k,
                      "groups": len(groups),
                      "parallelism": f"bands{world}: origin columns split over ranks, each rank holds its "
                                     f"sub-image (band + {w.window[1] - 1}-column halo); NCCL all-reduce of "
                                     f"X·V partials, K-side Grams and reconstruction numerators",
                      "band_of_rank0": list(band_slices(ny, w.window[1], max(world, 1), 0)[0]),
                      "l2": "flushed (256 MB write) between timed steps"},
           "e2e": {"value": nvec / (np.mean(e2e) / 1e3), "unit": "vector products/s",
                   "h2d_bytes_per_step": int(xg.shape[0] * (c1 - c0) * esz),
                   "d2h_bytes_per_step": int(len(groups) * xg.size * esz), "ms_per_step": float(np.mean(e2e))},
           "roofline": roofline,
           "gpu_launches": int(launches), "clocks": clk.summary(), "sigma_head": [float(x) for x in sig[:4]],
           "decomposition": {k2: info[k2] for k2 in ("n_block_products", "n_restarts", "n_converged",
                                                      "max_rel_residual")}}
    return res, w


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--shard", action="store_true",
                    help="one decomposition split over the ranks by window-position bands (strong scaling; "
                         "the default when N > 1)")
    ap.add_argument("--one-gpu-rehearsal", action="store_true",
                    help="correctness rehearsal of the N > 1 code path on a one-GPU box: every rank uses cuda:0 and "
                         "the process group is gloo (host-synchronised all-reduce of the device buffers; no kernel "
                         "waits on another rank's kernel).  Its timings are NOT a measurement")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas (weak scaling) instead of the band partition")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    if args.impl == "reference":
        # the oracle as it stands, on the host cores of rank 0 only
        if rank != 0:
            return
        w = workload(args.config)
        vals = []
        for _ in range(args.warmup):
            oracle_products_per_s(w, budget_s=min(args.cpu_budget, 5.0))
        t0 = time.perf_counter()
        cores, sample = 0, ""
        for _ in range(args.steps):
            v, cores, sample = oracle_products_per_s(w, budget_s=args.cpu_budget / max(args.steps, 1))
            vals.append(v)
        el = time.perf_counter() - t0
        v = float(np.mean(vals))
        print(json.dumps({"impl": "reference", "metric": "trajectory products/s", "value": v,
                          "unit": "vector products/s", "n_gpus": args.gpus, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": w.name, "window": list(w.window)},
                          "cpu_baseline": {"value": v, "unit": "vector products/s", "cores": cores,
                                           "kind": "oracle", "sample": sample, "cpu": cpu_model()},
                          "e2e": {"value": v, "unit": "vector products/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("gloo" if args.one_gpu_rehearsal else "nccl")
        dist = tdist
    sharded = args.shard or (world > 1 and not args.replicas)
    res, w = (run_sharded if sharded else run_ours)(args, rank, world, dist)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1 and not sharded:
            v, cores, sample = oracle_products_per_s(w, budget_s=args.cpu_budget)
            res["cpu_baseline"] = {"value": v, "unit": "vector products/s", "cores": cores, "kind": "oracle",
                                   "sample": sample, "cpu": cpu_model()}
        if args.one_gpu_rehearsal:
            res["rehearsal"] = (f"{world} ranks sharing cuda:0 over gloo: checks the N > 1 code path, "
                                "its timings are not a measurement")
        res["paper_context"] = {"rssa_nutrlan_s": {"mars_25x25": 0.519, "mars_160x80_r50": 0.587},
                                "hardware": "not stated in the paper (P:2518-2624)"}
        print(json.dumps(res))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
