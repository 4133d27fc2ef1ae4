#!/usr/bin/env python
"""Benchmark: Fresnel point x pixel updates/s and ms/hologram on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

One step = one saliency-gated progressive hologram of BASELINE.json
configs[1] (512^2 seeded Gaussian-blob object, 25% smooth-threshold mask,
3-level Haar DWT, centred on a 1024^2 complex64 hologram, lambda 532 nm,
pitch 8 um, z 0.2 m, direct point-source accumulation): DWT + gating +
compaction + accumulation (+ NCCL row-tile all-gather for N > 1), inputs
resident in HBM. `e2e` repeats the step through the C ABI with pinned HOST
buffers: H2D of the object and mask, the step, D2H of the hologram.
For N > 1 launch with torchrun; each rank computes a contiguous row band.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Fresnel point×pixel updates/s and ms/hologram at 1/2/4/8 B200, % of FP32/SFU peak"
UNIT = "updates/s"
SM_COUNT = 148
MUFU_PER_CLK_SM = 16.0
CANON_SFU_PER_UPDATE = 3.0  # rsqrt, sin, cos


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--method", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0, "note": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for name, v in zip(names, s[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own code path, bounded sample

class ReferenceTimer:
    """Times the UNMODIFIED reference (oracle/_ref) on this workload.

    The reference's synthesize_progressive requires object == plane size, so
    the object and mask are zero-padded to the centre of the hologram
    (SURVEY.md §8(c)); a multi-depth scene is the per-layer sum. Each timed
    sample is either the reference's whole synthesize_progressive
    (LutSet::build excluded, like its lut_build precompute) when that fits
    the per-sample budget, or — for holograms that take minutes to hours on
    the CPU — an extrapolation: the reference's own multi-threaded refine()
    (synthesis.cpp:171-178 -> accumulate_deterministic, parallel.cpp:49-98)
    on two contiguous windows of the real gated full-resolution cells
    (K1 < K2 real block applications), fitted as t(K) = a + b K and scaled to
    this scene's exact nonzero-weight operation count (each operation is one
    Nh^2 sweep, synthesis.cpp:28-34; zero weights return early, :20).
    Without _ref the fp64 C restatement is timed instead (kind "port").
    """

    def __init__(self, scene):
        from oracle import oracle as O

        self.O = O
        self.scene = scene
        c = scene.config
        self.n, self.no = c.plane_size, c.object_size
        self.off = (self.n - self.no) // 2
        self.L = c.n_layers
        xs, ys, amps, lay, ops = O.scene_points(scene.objects.astype(np.float64),
                                                scene.masks * (1.0 / 255.0), self.n)
        self.pts = (xs, ys, amps, lay)
        self.points = len(xs)
        self.updates = float(self.points) * self.n * self.n
        nz_ops = 0
        full_cells = None
        for l in range(self.L):
            an = O.analysis(scene.objects[l].astype(np.float64), scene.masks[l] * (1.0 / 255.0))
            approx, det = O.split_pyramid(an["pyramid"], self.no)
            no = self.no
            m_ll, m_l, m_f = np.split(an["masks"], [(no // 4) ** 2, (no // 4) ** 2 + (no // 2) ** 2])
            r_ll = O.expand_residual(*det[2]).ravel()
            r_l = O.expand_residual(*det[1]).ravel()
            r_f = O.expand_residual(*det[0]).ravel()
            nz_ops += int((approx != 0).sum()) + int(((m_ll != 0) & (r_ll != 0)).sum()) + \
                int(((m_l != 0) & (r_l != 0)).sum()) + int(((m_f != 0) & (r_f != 0)).sum())
            if l == 0:
                full_cells = (det[0], np.flatnonzero((m_f != 0) & (r_f != 0)))
        self.nz_ops = nz_ops
        if c.method == "lut":
            # LUT configs count (nonzero gated cell, pixel) updates on both arms
            self.updates = float(nz_ops) * self.n * self.n
        self.full_cells = full_cells
        self.kind = "reference" if O.ref_available() else "port"
        self.lutsets = None
        self.fit = None

    def _luts(self):
        if self.lutsets is None:
            c = self.scene.config
            w = self.O.ref_default_workers()
            self.workers = w
            self.lutsets = [self.O.ref().ref_lutset_build(c.wavelength, c.pitch, z, self.n, w)
                            for z in c.depths]
        return self.lutsets

    def close(self):
        if self.lutsets:
            for h in self.lutsets:
                self.O.ref().ref_lutset_free(h)
        self.lutsets = None

    def _refine_window(self, k, rng):
        import ctypes

        O, n, no, off = self.O, self.n, self.no, self.off
        (h, v, d), cells = self.full_cells
        hp = np.zeros((n // 2, n // 2))
        vp = np.zeros_like(hp)
        dp = np.zeros_like(hp)
        o2 = off // 2
        hp[o2:o2 + no // 2, o2:o2 + no // 2] = h
        vp[o2:o2 + no // 2, o2:o2 + no // 2] = v
        dp[o2:o2 + no // 2, o2:o2 + no // 2] = d
        cy, cx = np.divmod(cells, no)
        padded = (cy + off) * n + (cx + off)
        k = min(k, len(padded))
        s = int(rng.integers(0, max(1, len(padded) - k)))
        gate = np.zeros(n * n)
        gate[padded[s:s + k]] = 1.0
        secs, opsc = ctypes.c_double(), ctypes.c_uint64()
        rc = O.ref().ref_time_refine(self._luts()[0], hp.ctypes.data, vp.ctypes.data,
                                     dp.ctypes.data, n // 2, gate.ctypes.data, 0.5, self.workers,
                                     ctypes.byref(secs), ctypes.byref(opsc))
        assert rc == 0, O.ref().ref_last_error()
        return secs.value, int(opsc.value)

    def estimate(self, budget_s: float):
        """Extrapolated seconds per hologram from a sample of ~budget_s."""
        rng = np.random.default_rng(1234)
        t0, k0 = self._refine_window(64, rng)
        per_op = max(t0 / max(k0, 1), 1e-6)
        k2 = int(max(256, 0.6 * budget_s / per_op))
        k1 = max(64, k2 // 5)
        t1, o1 = self._refine_window(k1, rng)
        t2, o2 = self._refine_window(k2, rng)
        b = (t2 - t1) / max(o2 - o1, 1)
        a = max(t1 - b * o1, 0.0)
        est = 4 * a * self.L + b * self.nz_ops
        self.fit = (a, b, o1, o2)
        return est, (f"reference refine() on {o1}+{o2} real full-res block applications "
                     f"(Nh={self.n}, workers={self.workers}), t(K)=a+bK fit a={a:.3g}s "
                     f"b={b:.3g}s/op, extrapolated to {self.nz_ops} nonzero-weight ops "
                     f"({self.L} layer(s), 4 stages)")

    def full(self):
        """Seconds for the reference's whole synthesize_progressive (sum over layers)."""
        import ctypes

        O, n, no, off = self.O, self.n, self.no, self.off
        total = 0.0
        for l, h in enumerate(self._luts()):
            objp = np.zeros((n, n))
            salp = np.zeros((n, n))
            objp[off:off + no, off:off + no] = self.scene.objects[l]
            salp[off:off + no, off:off + no] = self.scene.masks[l] * (1.0 / 255.0)
            th = np.array([0.5, 0.7, 0.9])
            en = np.array([1, 1, 1], np.int32)
            secs = ctypes.c_double()
            opsr = np.zeros(5, np.uint64)
            rc = O.ref().ref_time_progressive(h, objp.ctypes.data, salp.ctypes.data,
                                              th.ctypes.data, en.ctypes.data, self.workers,
                                              ctypes.byref(secs), None, opsr.ctypes.data)
            assert rc == 0, O.ref().ref_last_error()
            total += secs.value
        return total, (f"reference synthesize_progressive, whole hologram ({self.L} layer(s)): "
                       f"object zero-padded to the {n}^2 plane, default plan, "
                       f"workers={self.workers}, LutSet::build excluded (precompute)")

    def port(self):
        O, c, n = self.O, self.scene.config, self.n
        rng = np.random.default_rng(7)
        npix = 64
        px = rng.integers(0, n, npix)
        py = rng.integers(0, n, npix)
        t0 = time.perf_counter()
        O.direct_pixels(*self.pts, [(c.wavelength, c.pitch, z) for z in c.depths], px, py)
        dt = time.perf_counter() - t0
        return dt * (n * n) / npix, (f"oracle direct Eq.(1) fp64 on {npix} pixels x "
                                     f"{self.points} points, extrapolated")

    def sample(self, budget_s: float, full_if_below: float | None = None):
        """One timed sample: (seconds per hologram, description, cores)."""
        if self.kind == "port":
            s, d = self.port()
            return s, d, os.cpu_count() or 1
        if getattr(self, "use_full", None) is None:
            est, desc = self.estimate(min(budget_s, 10.0))
            limit = budget_s if full_if_below is None else full_if_below
            self.use_full = est <= limit
            if not self.use_full:
                return est, desc, self.workers
        if self.use_full:
            s, d = self.full()
            return s, d, self.workers
        est, desc = self.estimate(min(budget_s, 10.0))
        return est, desc, self.workers


def reference_direct_rate():
    """The reference's own direct Eq.(1) (pointwise_hologram_reference,
    tests/support/oracles.cpp:12-36 — the formula K3 evaluates), single
    thread, on a seeded 64^2 object: updates/s (SURVEY.md §8(d) direct-formula
    baseline)."""
    from oracle import oracle as O

    if not O.ref_available():
        return None
    n = 64
    amp = np.random.default_rng(64).random((n, n))
    t0 = time.perf_counter()
    O.ref_pointwise_hologram_reference(amp, 532e-9, 8e-6, 0.2)
    dt = time.perf_counter() - t0
    upd = float(np.count_nonzero(amp)) * n * n
    return {"value": upd / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"pointwise_hologram_reference on a {n}^2 object / {n}^2 plane, 1 thread, "
                      f"{dt:.2f} s"}


def reference_cpu_sample(scene, target_seconds: float = 10.0):
    t = ReferenceTimer(scene)
    try:
        secs, desc, cores = t.sample(target_seconds, full_if_below=3 * target_seconds)
    finally:
        t.close()
    return {"value": t.updates / secs, "unit": UNIT, "cores": int(cores), "kind": t.kind,
            "sample": desc, "ms_per_hologram": secs * 1e3, "points": t.points}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation on the box's
    host cores (rank 0 only), same metric/config as our arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2211_09938_b200 import scenes

    sc = scenes.make_scene(args.config)
    t = ReferenceTimer(sc)
    per_step = max(2.0, 150.0 / max(1, args.steps + min(args.warmup, 1)))
    secs = []
    try:
        for i in range(min(args.warmup, 1) + args.steps):
            s, desc, cores = t.sample(per_step)
            if i >= min(args.warmup, 1):
                secs.append(s)
    finally:
        t.close()
    ms = float(np.mean(secs)) * 1e3
    v = t.updates / (ms * 1e-3)
    out = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": sc.config.name, "object": sc.config.object_size,
                   "plane": sc.config.plane_size, "points": t.points,
                   "method": "reference LUT synthesize_progressive (CPU)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": int(cores), "kind": t.kind,
                         "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_2211_09938_b200 import _lib, scenes, tiles
    from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the multi-rank path on a single GPU only (numbers
    # from such a run are not measurements): all ranks on device 0, gloo
    if os.environ.get("WCGH_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("WCGH_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    sc = scenes.make_scene(args.config)
    c = sc.config
    row0, rows = tiles.band(rank, world, c.plane_size)
    ctx = _lib.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    torch.cuda.synchronize()
    t_pre = time.perf_counter()
    job = HologramJob(spec_for_scene(sc, method=args.method, row0=row0, rows=rows), ctx)
    torch.cuda.synchronize()
    precompute_ms = (time.perf_counter() - t_pre) * 1e3  # LUT / fringe-spectrum build + buffers

    # resident inputs (device) for the device-timed `value`
    obj_d = torch.from_numpy(sc.objects).cuda()
    sal_d = torch.from_numpy(sc.masks).cuda()
    # pinned host buffers for e2e
    obj_h = torch.from_numpy(sc.objects).pin_memory()
    sal_h = torch.from_numpy(sc.masks).pin_memory()
    full_h = torch.empty((c.plane_size, 2 * c.plane_size), dtype=torch.float32).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # multi-GPU: the row-tile all-gather is fused into the band's final kernel
    # (NVLink P2P stores into CUDA-IPC-mapped peer planes); NCCL all-gather
    # only if the IPC mapping cannot be set up on this box
    gathered, exchange, gather_mode = None, None, "none (1 GPU)"
    if world > 1:
        try:
            exchange = tiles.PeerPlaneExchange(world, rank, c.plane_size, local)
            exchange.register(job)
            gather_mode = "fused: band epilogue stores into CUDA-IPC peer planes over NVLink"
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            gather_mode = f"NCCL all_gather_into_tensor (IPC peer planes unavailable: {e})"
            gathered = torch.empty((c.plane_size, 2 * c.plane_size), dtype=torch.float32,
                                   device="cuda")

    def step():
        job.run()
        if world > 1:
            if exchange is not None:
                dist.barrier()  # every rank's band has landed in every plane
            else:
                tiles.gather_tiles(tiles.tile_tensor(job), world, c.plane_size, out=gathered)

    job.upload_dev(obj_d.data_ptr(), sal_d.data_ptr())
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    synth_ms, launches, stats = [], 0, None
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the timed interval)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
        stats = job.stats()
        synth_ms.append(stats["ms_synthesis"])
        launches += stats["total_launches"]
    torch.cuda.synchronize()
    in_region = len(clocks.samples)
    # a timed region shorter than nvidia-smi's start-up (config 0) has no
    # sample: keep the same load running, untimed, until one arrives (<= 3 s;
    # single rank only — ranks' samplers differ and step() holds barriers)
    t_hold = time.perf_counter()
    while (world == 1 and not clocks.samples and clocks.proc is not None
           and time.perf_counter() - t_hold < 3.0):
        for _ in range(8):
            step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    clk["samples_in_timed_region"] = in_region
    step_ms = [s.elapsed_time(e) for s, e in ev]
    t_rank = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([t_rank], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_rank = float(t.item())
    ms_per_step = t_rank / args.steps
    points = stats["n_points"]
    updates = float(points) * c.plane_size * c.plane_size
    value = updates / (ms_per_step * 1e-3)

    # e2e through the C ABI with pinned host buffers
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        job.upload(obj_h.numpy(), sal_h.numpy())
        job.run()
        if world > 1:
            if exchange is not None:
                dist.barrier()
                if rank == 0:
                    full_h.copy_(exchange.plane_tensor())
            else:
                tiles.gather_tiles(tiles.tile_tensor(job), world, c.plane_size, out=gathered)
                if rank == 0:
                    full_h.copy_(gathered)
        else:
            job.download(full_h.numpy().view(np.complex64))
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_t = float(np.sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_t], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_value = updates / (e2e_t / args.steps * 1e-3)
    h2d = int(sc.objects.nbytes + sc.masks.nbytes)
    d2h = int(c.plane_size * c.plane_size * 8) if rank == 0 else 0

    out = None
    if rank == 0:
        peaks = measured_peaks()
        f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        f_meas = (clk.get("sm_mhz") or 0) * 1e6
        # dominant kernel, timed by CUDA events around its launches on this
        # stream inside wcgh_job_run; per-rank algorithmic updates per step
        k_ms = float(np.mean(synth_ms))
        rank_updates = float(points) * rows * c.plane_size
        achieved = rank_updates / (k_ms * 1e-3)
        if job.spec.method == "direct":
            per_clk, kernel = MUFU_PER_CLK_SM / CANON_SFU_PER_UPDATE, "k_direct_fixed (K3)"
            basis = (f"canonical SFU roofline {SM_COUNT} SMs x {f_max/1e6:.0f} MHz (MEASURED_PEAKS "
                     "sm_max_mhz) x 16 MUFU/clk/SM / 3 MUFU per update (SURVEY.md §8(d)); the kernel "
                     "issues 2 MUFU + ~8.5 packed-fp32x2/ALU issue slots per update, so its own "
                     "bound is 2 MUFU per update (frac_of_2mufu_bound); not an HBM or "
                     "tensor-core kernel")
            bound = "sfu"
            dram = int(points * 16 + rows * c.plane_size * 8)
        elif job.spec.method == "lut":
            per_clk, kernel = 128.0 / 2.0, "k_lut_stage (K4), 4 stage launches"
            basis = (f"FP32 roofline {SM_COUNT} SMs x {f_max/1e6:.0f} MHz x 128 FFMA/clk/SM / 2 FFMA per "
                     "(nonzero cell, pixel) update (SURVEY.md §8(d))")
            bound = "fp32"
            dram = int(4 * (2 * c.plane_size - 1) ** 2 * 8 + rows * c.plane_size * 8)
        else:  # fft: cuFFT transforms dominate (library code, like cuBLAS)
            per_clk, kernel = None, "cuFFT C2C on the 2Nh grid + k_spec_mul/k_scatter/k_extract"
            basis = ("FFT method: the transforms are cuFFT (library); no hand-written-kernel roofline "
                     "is claimed — `value` keeps the direct method's numerator")
            bound = "hbm"
            dram = int(3 * (2 * c.plane_size) ** 2 * 8 * c.n_layers + rows * c.plane_size * 8)
        peak = SM_COUNT * f_max * per_clk if per_clk else None
        # dram__bytes_read + dram__bytes_write per launch from the committed
        # `ncu --set full` capture (profiles/, tools/profile_round.sh)
        traffic = None
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists():
            tj = json.loads(tp.read_text())
            traffic = tj.get({"sfu": "k_direct_fixed", "fp32": "k_lut_stage"}.get(bound, ""))
        roof = {
            "bound": bound, "achieved": achieved if peak else None, "peak": peak, "unit": UNIT,
            "frac": achieved / peak if peak else None, "traffic": traffic, "kernel": kernel,
            "kernel_ms": k_ms,
            "traffic_note": ("bytes per launch from profiles/ncu_traffic.json (config-1 capture for K3; "
                             "config-2 stage average for K4); dominated by the fixed-order "
                             "partial-sum planes, not by point/LUT reads"),
            "peak_basis": basis,
            "frac_at_measured_clock": (achieved / (SM_COUNT * f_meas * per_clk)
                                       if f_meas and per_clk else None),
            "dram_bytes_per_step_algorithmic": dram,
        }
        if bound == "sfu":  # the XU bound of the kernel's actual 2-MUFU instruction mix
            roof["frac_of_2mufu_bound"] = achieved / (SM_COUNT * f_max * MUFU_PER_CLK_SM / 2.0)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian-blob objects, smooth-threshold masks; SURVEY.md §8(d))",
            "config": {"workload": c.name, "object": c.object_size, "plane": c.plane_size,
                       "layers": c.n_layers, "points": points, "updates_per_hologram": updates,
                       "method": job.spec.method, "phase": "fixed-point quadratic + fp32 series",
                       "ops": stats["ops"], "parallelism": f"row tiles x{world}",
                       "gather": gather_mode,
                       "l2": "flushed between timed steps (256 MiB write, outside the step interval)"},
            "ms_per_hologram": ms_per_step,
            "precompute_ms": precompute_ms,
            "precompute_note": ("job creation outside the timed steps: LUT build (K5) for the LUT "
                                "method, fringe spectra for FFT, buffers (the reference's lut_build "
                                "is likewise excluded)"),
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_t / args.steps},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world == 1 and c.n_layers == 1:
            # the same hologram through the other synthesis method (direct Eq.(1)
            # vs the reference's block-LUT superposition), timed the same way
            out["alt_methods"] = []
            h_main = job.download()
            for alt in [m for m in ("direct", "lut", "fft") if m != job.spec.method]:
                try:
                    torch.cuda.synchronize()
                    t_pre = time.perf_counter()
                    ajob = HologramJob(spec_for_scene(sc, method=alt), ctx)
                    torch.cuda.synchronize()
                    a_pre = (time.perf_counter() - t_pre) * 1e3
                    ajob.upload_dev(obj_d.data_ptr(), sal_d.data_ptr())
                    for _ in range(args.warmup):
                        ajob.run()
                    aev = []
                    for _ in range(args.steps):
                        flush.zero_()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        ajob.run()
                        e1.record(stream)
                        aev.append((e0, e1))
                    torch.cuda.synchronize()
                    a_ms = float(np.mean([s.elapsed_time(e) for s, e in aev]))
                    h_alt = ajob.download()
                    ast = ajob.stats()
                    out["alt_methods"].append({
                        "method": alt, "ms_per_hologram": a_ms,
                        "value": updates / (a_ms * 1e-3), "unit": UNIT,
                        "note": ("same hologram (after_full), same numerator as `value`; "
                                 + {"direct": "Eq.(1) per point x pixel on the SFU (K3)",
                                    "lut": "the reference's block-LUT superposition (K4)",
                                    "fft": "correlation with the point fringe via cuFFT, O(Nh^2 log Nh)"}[alt]),
                        "algorithmic_updates": ast["updates"],
                        "precompute_ms": a_pre,
                        "rel_l2_vs_main": float(np.linalg.norm(h_alt - h_main) / np.linalg.norm(h_main)),
                    })
                    ajob.close()
                except Exception as e:
                    out["alt_methods"].append({"method": alt, "error": str(e)})
        if world == 1 and not args.no_cpu_baseline:
            try:
                cb = reference_cpu_sample(sc, target_seconds=args.cpu_seconds)
                out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
                out["cpu_baseline"]["ms_per_hologram"] = cb["ms_per_hologram"]
                out["cpu_baseline_direct_formula"] = reference_direct_rate()
            except Exception as e:  # the baseline is reported, never required
                out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                                       "sample": f"failed: {e}"}
        print(json.dumps(out))
    if world > 1:
        dist.barrier()  # no rank unmaps / frees a plane another rank still writes
    if exchange is not None:
        exchange.close()
    job.close()
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
