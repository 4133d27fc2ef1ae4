#!/usr/bin/env python
"""Benchmark: Fresnel point x pixel updates/s and ms/hologram on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One step = one saliency-gated progressive hologram of BASELINE.json
configs[4] by default — the largest single-GPU configuration the metric's
1/2/4/8-GPU numbers and the >=85% scaling target are quoted on: a 2048^2
seeded Gaussian-blob uint8 object, 25% smooth-threshold mask, 3-level Haar
DWT, centred on a 4096^2 complex64 hologram, lambda 532 nm, pitch 4 um,
z 0.2 m, direct point-source accumulation. The step is DWT + gating +
compaction + accumulation (+ the fused row-tile gather for N > 1) with
inputs resident in HBM. `e2e` repeats the step through the C ABI with pinned
HOST buffers: H2D of the object and mask, the step, D2H of the hologram.
`extra_configs.cfg1` is the same measurement on configs[1] (512^2 on 1024^2,
round 1's headline), with the reference's whole CPU hologram beside it.

--gpus N without a torchrun environment re-launches this script under
`torch.distributed.run` with N ranks (one process per GPU); each rank
computes a contiguous row band and stores it into every rank's plane from
the band's final kernel (CUDA-IPC peer planes over NVLink).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
# K3 as built (k_direct_chirp, NC = 3, point loop unrolled by 2): FMA-pipe lane
# operations per update counted from the SASS of the point loop (2 points x 32
# pixels = 64 updates per trip): multiplier held for 1 / 2 / 4 steps = 308 / 282 /
# 266 packed fp32x2 instructions + 28 / 28 / 27 scalar FMA-pipe ones
# (profiles/sass/k3_direct_chirp_NC3_AMP1_RU2[_HOLD2|_HOLD4].sass).
K3_KERNEL = "k_direct_chirp (K3, chirp-factored angle-addition recurrence)"
K3_LANE_OPS_BY_HOLD = {1: 10.06, 2: 9.25, 4: 8.73}
# packed FFMA2 with the scalar operand in a uniform register (K4's parameter-block form),
# measured by tools/microbench_operands.cu: profiles/s4_microbench_operands.txt (116 of 128;
# 111 with the weight in a regular register, 125-127 straight from the constant bank)
FFMA2_CEILING_LANE_FMA_PER_CLK = 116.0
# one whole reference hologram at a 4096^2 config, timed on the GPU box's
# host against the extrapolation model (tools/ref_full_check.py)
REF_FULL_CHECK = ("config 4 whole reference synthesize_progressive on 16 host cores: 1361 s "
                  "measured vs 1197-1218 s extrapolated by this model (x1.12-1.14, the model "
                  "favours the reference); profiles/s3_reference_full_cfg4.json")
E2E_SECONDS = 60.0          # e2e / alt-method step budget at large configs
ALT_SECONDS = 10.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--method", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip extra_configs / alt_methods")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0, "note": "fallback (B200_PROFILING.md)"}


def host_cpu():
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """--gpus N with no torchrun environment: run N ranks of this script."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    print(f"[bench] --gpus {args.gpus}: launching {args.gpus} ranks: {' '.join(cmd)}",
          file=sys.stderr, flush=True)
    return subprocess.call(cmd)


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
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples), "sm_min_mhz": min(sm) if sm else None,
                "power_w_median": float(np.median(pw)) if pw else None}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own code path

class ReferenceTimer:
    """Times the UNMODIFIED reference (oracle/_ref) on this workload.

    The reference's synthesize_progressive requires object == plane size, so
    the object and mask are zero-padded to the centre of the hologram
    (SURVEY.md §8(c)); a multi-depth scene is the per-layer sum.
    * full(): the reference's whole synthesize_progressive (synthesis.cpp:
      180-253; LutSet::build excluded, like its lut_build precompute) — used
      for configs 0-2 ("full end-to-end runs").
    * estimate(): for the 4096^2 configs, whose CPU hologram takes 15-20
      minutes: the reference's own multi-threaded refine() (synthesis.cpp:
      171-178 -> accumulate_deterministic, parallel.cpp:49-98) on two windows
      of the real gated full-resolution cells (K1 < K2 real block
      applications), fitted t(K) = a + b K and extrapolated by this scene's
      exact nonzero-weight operation count (each op is one Nh^2 sweep,
      synthesis.cpp:28-34; zero weights return early, :20). Labelled
      "extrapolated".
    Without _ref the fp64 C restatement is timed instead (kind "port")."""

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
        self.ops = [int(v) for v in ops]
        nz_ops = 0
        nz_by_stage = [0, 0, 0, 0]
        full_cells = None
        for l in range(self.L):
            an = O.analysis(scene.objects[l].astype(np.float64), scene.masks[l] * (1.0 / 255.0))
            approx, det = O.split_pyramid(an["pyramid"], self.no)
            no = self.no
            m_ll, m_l, m_f = np.split(an["masks"], [(no // 4) ** 2, (no // 4) ** 2 + (no // 2) ** 2])
            r_ll = O.expand_residual(*det[2]).ravel()
            r_l = O.expand_residual(*det[1]).ravel()
            r_f = O.expand_residual(*det[0]).ravel()
            st = [int((approx != 0).sum()), int(((m_ll != 0) & (r_ll != 0)).sum()),
                  int(((m_l != 0) & (r_l != 0)).sum()), int(((m_f != 0) & (r_f != 0)).sum())]
            nz_by_stage = [a + b for a, b in zip(nz_by_stage, st)]
            nz_ops += sum(st)
            if l == 0:
                full_cells = (det[0], np.flatnonzero((m_f != 0) & (r_f != 0)))
        self.nz_ops = nz_ops
        self.nz_by_stage = nz_by_stage
        if c.method == "lut":
            # LUT configs count (nonzero gated cell, pixel) updates on both arms
            self.updates = float(nz_ops) * self.n * self.n
        self.full_cells = full_cells
        self.kind = "reference" if O.ref_available() else "port"
        self.lutsets = None
        self.fit = None
        self.workers = None

    def _luts(self):
        if self.lutsets is None:
            c = self.scene.config
            self.workers = self.O.ref_default_workers()
            self.lutsets = [self.O.ref().ref_lutset_build(c.wavelength, c.pitch, z, self.n, self.workers)
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
        # k cells spread over the whole gated set (contiguous runs of cells
        # gave the same per-op cost). Validation: one whole reference
        # hologram at config 4 on the GPU box's 16 host cores took 1361 s
        # against 1197-1218 s extrapolated this way (ratio 1.12-1.14; the
        # model favours the reference), profiles/s3_reference_full_cfg4.json
        pick = np.sort(rng.choice(len(padded), size=k, replace=False))
        gate = np.zeros(n * n)
        gate[padded[pick]] = 1.0
        secs, opsc = ctypes.c_double(), ctypes.c_uint64()
        rc = O.ref().ref_time_refine(self._luts()[0], hp.ctypes.data, vp.ctypes.data,
                                     dp.ctypes.data, n // 2, gate.ctypes.data, 0.5, self.workers,
                                     ctypes.byref(secs), ctypes.byref(opsc))
        assert rc == 0, O.ref().ref_last_error()
        return secs.value, int(opsc.value)

    def estimate(self, budget_s: float):
        """Extrapolated seconds per hologram from a bounded sample. At Nh = 4096
        a refine() call carries a ~4 s fixed cost (whole-plane residual
        expansion, gating, plane allocation) next to ~2-4 ms per block
        application, so the intercept is measured directly (a one-op window)
        and the slope over a window large enough that b*K dominates the
        intercept's run-to-run noise (K = min(cells, 2048), ~5-10 s)."""
        rng = np.random.default_rng(1234)
        t1, o1 = self._refine_window(1, rng)
        k2 = int(min(len(self.full_cells[1]), max(256, 2048 * budget_s / 10.0)))
        t2, o2 = self._refine_window(k2, rng)
        b = max((t2 - t1) / max(o2 - o1, 1), 1e-7)
        a = max(t1 - b * o1, 0.0)
        est = 4 * a * self.L + b * self.nz_ops
        self.fit = {"a_s": a, "b_s_per_op": b, "window_ops": [o1, o2],
                    "sample_wall_s": t1 + t2}
        return est, (f"EXTRAPOLATED: reference refine() on {o1}+{o2} real full-res block "
                     f"applications (Nh={self.n}, workers={self.workers}), t(K)=a+bK fit "
                     f"a={a:.3g}s b={b:.3g}s/op, scaled to {self.nz_ops} nonzero-weight ops "
                     f"(per stage {self.nz_by_stage}; {self.L} layer(s), 4 stages)")

    def step_sample(self, k: int, rng):
        """One bounded step after estimate(): a real refine() window of k
        block applications; the hologram estimate keeps the fitted per-call
        intercept a and takes the per-op cost from this window."""
        a = self.fit["a_s"]
        t, o = self._refine_window(k, rng)
        b = max(t - a, 0.0) / max(o, 1)
        est = 4 * a * self.L + b * self.nz_ops
        return est, (f"EXTRAPOLATED: reference refine() on {o} real full-res block applications "
                     f"per step (Nh={self.n}, workers={self.workers}), per-call intercept "
                     f"a={a:.3g}s from a two-window fit (windows {self.fit['window_ops']}), "
                     f"scaled to {self.nz_ops} nonzero-weight ops (per stage {self.nz_by_stage}; "
                     f"{self.L} layer(s), 4 stages)")

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
        return dt * (n * n) / npix, (f"EXTRAPOLATED: oracle direct Eq.(1) fp64 on {npix} pixels x "
                                     f"{self.points} points")

    def use_full(self) -> bool:
        return self.scene.config.cfg in (0, 1, 2)


def reference_direct_rate():
    """SURVEY.md §8(d)'s two further CPU baselines, on BASELINE config 0
    (128^2 blob object, z 0.2 m, pitch 8 um), whole holograms: the
    reference's own direct Eq.(1) (pointwise_hologram_reference,
    tests/support/oracles.cpp:12-36 — the formula K3 evaluates; single
    thread) and its production point-wise hologram synthesize_pointwise_oracle
    (synthesis.cpp:255-286: the B = 1 LUT at every pixel, workers = nproc; its
    LUT build excluded). updates = nonzero object pixels x plane pixels."""
    from oracle import oracle as O
    from paper_2211_09938_b200 import scenes

    if not O.ref_available():
        return None
    sc = scenes.make_scene(0)
    obj = sc.objects[0].astype(np.float64)
    n = obj.shape[0]
    upd = float(np.count_nonzero(obj)) * n * n
    t0 = time.perf_counter()
    O.ref_pointwise_hologram_reference(obj, 532e-9, 8e-6, 0.2)
    dt = time.perf_counter() - t0
    direct = {"value": upd / dt, "unit": UNIT, "cores": 1, "kind": "reference",
              "sample": f"pointwise_hologram_reference, whole config-0 hologram ({n}^2), 1 thread, "
                        f"{dt:.2f} s", **host_cpu()}
    t0 = time.perf_counter()
    O.ref_pointwise_oracle(obj, 532e-9, 8e-6, 0.2, workers=0)
    dt2 = time.perf_counter() - t0
    direct["pointwise_oracle"] = {
        "value": upd / dt2, "unit": UNIT, "cores": O.ref_default_workers(), "kind": "reference",
        "sample": (f"synthesize_pointwise_oracle, whole config-0 hologram ({n}^2, B=1 LUT built "
                   f"inside the timed call), {dt2:.3f} s")}
    return direct


def reference_cpu_sample(scene, budget_s: float = 10.0):
    """One bounded reference sample for our arm's `cpu_baseline` (rank 0, N=1)."""
    t = ReferenceTimer(scene)
    try:
        if t.kind == "port":
            secs, desc = t.port()
            cores, extrap = 1, True
        elif t.use_full():
            secs, desc = t.full()
            cores, extrap = t.workers, False
        else:
            secs, desc = t.estimate(budget_s)
            cores, extrap = t.workers, True
    finally:
        t.close()
    out = {"value": t.updates / secs, "unit": UNIT, "cores": int(cores), "kind": t.kind,
           "sample": desc, "ms_per_hologram": secs * 1e3, "extrapolated": extrap,
           "points": t.points, **host_cpu()}
    if extrap and t.fit:
        out["fit"] = t.fit
        out["extrapolation_check"] = REF_FULL_CHECK
        out["nonzero_ops_used"] = t.nz_ops
        out["nonzero_ops_per_stage"] = t.nz_by_stage
    return out


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation on the box's
    host cores (rank 0 only), same metric/config/unit as our arm. Configs
    0-2: each step is the reference's whole synthesize_progressive (as many
    whole holograms as fit a ~4 min budget, >= 1). 4096^2 configs: each step
    is a bounded sample (real refine() windows, ~budget s of wall), the
    hologram time extrapolated from it by the exact op count (labelled)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2211_09938_b200 import scenes

    sc = scenes.make_scene(args.config)
    t = ReferenceTimer(sc)
    holo_s, wall_s, desc, cores, runs = [], [], "", 1, 0
    budget_total = 240.0
    t_start = time.perf_counter()
    try:
        if t.kind == "port":
            for i in range(1 + args.steps):
                w0 = time.perf_counter()
                s, desc = t.port()
                if i >= 1:
                    holo_s.append(s)
                    wall_s.append(time.perf_counter() - w0)
            extrap = True
        elif t.use_full():
            extrap = False
            n_warm = 1 if args.warmup > 0 else 0
            for i in range(n_warm + args.steps):
                w0 = time.perf_counter()
                s, desc = t.full()
                runs += 1
                if i >= n_warm:
                    holo_s.append(s)
                    wall_s.append(time.perf_counter() - w0)
                elapsed = time.perf_counter() - t_start
                if holo_s and elapsed + s > budget_total:
                    break  # bounded: whole holograms only, as many as fit
            cores = t.workers
        else:
            extrap = True
            # warm-up = the two-window fit; then each step one real window
            # sized so the K steps take ~150 s of reference work in total
            t.estimate(10.0)
            a, b = t.fit["a_s"], max(t.fit["b_s_per_op"], 1e-6)
            per_step = max(2.0, 150.0 / max(1, args.steps))
            k = int(max(64, (per_step - a) / b))
            rng = np.random.default_rng(4321)
            for i in range(args.steps):
                w0 = time.perf_counter()
                s, desc = t.step_sample(k, rng)
                holo_s.append(s)
                wall_s.append(time.perf_counter() - w0)
            cores = t.workers
    finally:
        t.close()
    ms_holo = float(np.mean(holo_s)) * 1e3
    v = t.updates / (ms_holo * 1e-3)
    out = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(wall_s)) * 1e3,
        "ms_per_hologram": ms_holo,
        "extrapolated": extrap,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian-blob objects, smooth-threshold masks; SURVEY.md §8(d))",
        "config": {"workload": sc.config.name, "object": sc.config.object_size,
                   "plane": sc.config.plane_size, "layers": sc.config.n_layers,
                   "points": t.points, "updates_per_hologram": t.updates,
                   "method": "reference LUT synthesize_progressive (CPU)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": int(cores), "kind": t.kind,
                         "sample": desc, **host_cpu()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if extrap:
        out["ms_per_step_note"] = ("wall time of each step's bounded sample (real reference work); "
                                   "ms_per_hologram is the extrapolated whole-hologram time `value` "
                                   "is computed from")
        out["nonzero_ops_used"] = t.nz_ops
        out["nonzero_ops_per_stage"] = t.nz_by_stage
        out["op_counts"] = t.ops
        if t.fit:
            out["fit"] = t.fit
        out["extrapolation_check"] = REF_FULL_CHECK
    else:
        out["whole_holograms_timed"] = len(holo_s)
        out["ms_per_step_note"] = "each step = one whole reference hologram"
        if len(holo_s) < args.steps:
            out["steps_timed"] = len(holo_s)
            out["steps_note"] = (f"bounded: {len(holo_s)} of {args.steps} whole-hologram steps fit "
                                 f"the {budget_total:.0f} s budget")
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

def _roofline(job, c, points, rows, k_ms, f_max, f_meas, workload):
    rank_updates = float(points) * rows * c.plane_size
    achieved = rank_updates / (k_ms * 1e-3) if k_ms > 0 else None
    if job.spec.method == "direct":
        per_clk, kernel = MUFU_PER_CLK_SM / CANON_SFU_PER_UPDATE, K3_KERNEL
        form, hold = job.direct_form()
        lane_ops = K3_LANE_OPS_BY_HOLD.get(hold if form == 2 else 1, 10.06)
        basis = (f"canonical SFU roofline {SM_COUNT} SMs x {f_max/1e6:.0f} MHz (MEASURED_PEAKS "
                 "sm_max_mhz) x 16 MUFU/clk/SM / 3 MUFU per update (SURVEY.md §8(d)). K3 "
                 "evaluates exp(ikr)/r by angle addition along 16-pixel runs (2 MUFU per run "
                 "seed, 4 per 32 updates), so it is bound by the FP32 pipe instead: "
                 "frac_of_fp32_bound = achieved / (148 x f x 128 lane-ops/clk/SM / "
                 f"{lane_ops} lane-ops per update at hold = {hold}, counted from the SASS in "
                 "profiles/sass/k3_direct_chirp_NC3_AMP1_RU2*.sass); not an HBM or tensor-core kernel")
        bound, key = "sfu", "k_direct_chirp"
        dram = int(points * 16 + rows * c.plane_size * 8)
    elif job.spec.method == "lut":
        per_clk, kernel = 128.0 / 2.0, ("k_lut_chunk (K4): run-list chunks of the 4 stages as kernel "
                           "parameter blocks, 16x2 register window")
        basis = (f"FP32 roofline {SM_COUNT} SMs x {f_max/1e6:.0f} MHz x 128 FFMA/clk/SM / 2 FFMA per "
                 "(nonzero cell, pixel) update (SURVEY.md §8(d))")
        bound, key = "fp32", "k_lut_chunk"
        dram = int(4 * (2 * c.plane_size - 1) ** 2 * 8 + rows * c.plane_size * 8)
        rank_updates = job.stats()["updates"]
        achieved = rank_updates / (k_ms * 1e-3) if k_ms > 0 else None
    else:
        per_clk, kernel = None, "hand-written row FFTs + transposes on the 2Nh grid (wcgh_fftk.cu)"
        basis = ("FFT method: O(L^2 log L) hand-written Stockham row FFTs, HBM/shared-memory bound; "
                 "no SFU/FP32 roofline applies — `value` keeps the direct method's numerator")
        bound, key = "hbm", None
        dram = int(3 * (2 * c.plane_size) ** 2 * 8 * c.n_layers + rows * c.plane_size * 8)
    peak = SM_COUNT * f_max * per_clk if per_clk else None
    traffic, traffic_src = None, None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists() and key:
        ent = json.loads(tp.read_text()).get(key)
        if isinstance(ent, dict):
            rec = ent.get(workload)
            if rec:
                traffic, traffic_src = rec.get("bytes_per_launch"), rec.get("source")
    roof = {
        "bound": bound, "achieved": achieved if peak else None, "peak": peak, "unit": UNIT,
        "frac": achieved / peak if (peak and achieved) else None, "traffic": traffic,
        "kernel": kernel, "kernel_ms": k_ms, "peak_basis": basis,
        "frac_at_measured_clock": (achieved / (SM_COUNT * f_meas * per_clk)
                                   if (f_meas and per_clk and achieved) else None),
        "dram_bytes_per_step_algorithmic": dram,
    }
    if traffic_src:
        roof["traffic_source"] = traffic_src
        n_launch = max(1, (job.stats().get("synth_launches") or 1))
        roof["achieved_dram_gbs"] = traffic * n_launch / (k_ms * 1e-3) / 1e9 if k_ms > 0 else None
        roof["traffic_note"] = ("dram__bytes_read+write per K3/K4 launch from one `ncu --set full` "
                                "capture; dominated by the fixed-order fp32 partial-sum planes "
                                "(compute-bound kernel, < 1% DRAM utilisation)")
    if bound == "fp32" and achieved:
        # the packed-FFMA2 ceiling measured by tools/microbench_operands.cu on this
        # pool for K4's operand form (uniform-register weight, no loads)
        ceil = SM_COUNT * f_max * FFMA2_CEILING_LANE_FMA_PER_CLK / 2.0
        roof["measured_ffma2_ceiling"] = ceil
        roof["frac_of_measured_ffma2_ceiling"] = achieved / ceil
        roof["ffma2_ceiling_source"] = "profiles/s4_microbench_operands.txt"
    if bound == "sfu" and achieved:
        fp32_peak = SM_COUNT * f_max * 128.0 / lane_ops
        roof["fp32_bound"] = fp32_peak
        roof["frac_of_fp32_bound"] = achieved / fp32_peak
        roof["fp32_lane_ops_per_update"] = lane_ops
        roof["k3_form"] = {"form": form, "hold": hold}
    return roof


class Runner:
    """One workload on this rank: a job over its row band, resident device
    inputs, pinned host buffers, and the fused row-tile gather for N > 1."""

    def __init__(self, sc, method, ctx, stream, world, rank, local):
        import torch

        from paper_2211_09938_b200 import tiles
        from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene

        self.sc, self.c = sc, sc.config
        self.world, self.rank, self.stream = world, rank, stream
        row0, self.rows = tiles.band(rank, world, self.c.plane_size)
        torch.cuda.synchronize()
        t_pre = time.perf_counter()
        self.job = HologramJob(spec_for_scene(sc, method=method, row0=row0, rows=self.rows), ctx)
        torch.cuda.synchronize()
        self.precompute_ms = (time.perf_counter() - t_pre) * 1e3
        self.obj_d = torch.from_numpy(sc.objects).cuda()
        self.sal_d = torch.from_numpy(sc.masks).cuda()
        self.obj_h = torch.from_numpy(sc.objects).pin_memory()
        self.sal_h = torch.from_numpy(sc.masks).pin_memory()
        n = self.c.plane_size
        self.full_h = torch.empty((n, 2 * n), dtype=torch.float32).pin_memory()
        self.exchange, self.gathered, self.gather_mode = None, None, "none (1 GPU)"
        if world > 1:
            try:
                self.exchange = tiles.PeerPlaneExchange(world, rank, n, local)
                self.exchange.register(self.job)
                self.gather_mode = ("fused: band epilogue stores into double-buffered CUDA-IPC "
                                    "peer planes over NVLink")
            except Exception as e:  # noqa: BLE001 - reported in the JSON line
                self.gather_mode = f"NCCL all_gather_into_tensor (IPC peer planes unavailable: {e})"
                self.gathered = torch.empty((n, 2 * n), dtype=torch.float32, device="cuda")
        self.job.upload_dev(self.obj_d.data_ptr(), self.sal_d.data_ptr())

    def step(self):
        import torch.distributed as dist

        from paper_2211_09938_b200 import tiles

        if self.world == 1:
            self.job.run()
        elif self.exchange is not None:
            self.exchange.run()
            dist.barrier()  # every rank's band has landed in every plane
        else:
            self.job.run()
            tiles.gather_tiles(tiles.tile_tensor(self.job), self.world, self.c.plane_size,
                               out=self.gathered)

    def step_e2e(self):
        """The step through the public API with host buffers: H2D of the
        object and mask, run, D2H of the assembled hologram (rank 0)."""
        import torch.distributed as dist

        from paper_2211_09938_b200 import tiles

        self.job.upload(self.obj_h.numpy(), self.sal_h.numpy())
        if self.world == 1:
            self.job.run()
            self.job.download(self.full_h.numpy().view(np.complex64))
        elif self.exchange is not None:
            self.exchange.run()
            dist.barrier()
            if self.rank == 0:  # this epoch's buffer; peers now write the other one
                self.full_h.copy_(self.exchange.plane_tensor())
        else:
            self.job.run()
            tiles.gather_tiles(tiles.tile_tensor(self.job), self.world, self.c.plane_size,
                               out=self.gathered)
            if self.rank == 0:
                self.full_h.copy_(self.gathered)

    def close(self):
        import torch.distributed as dist

        if self.world > 1:
            dist.barrier()  # no rank unmaps / frees a plane another rank still writes
        if self.exchange is not None:
            self.exchange.close()
        self.job.close()


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure(sc, method, args, ctx, stream, world, rank, local, flush, extras):
    """Device-timed `value`, e2e and roofline of one workload (all ranks)."""
    import torch
    import torch.distributed as dist

    c = sc.config
    r = Runner(sc, method, ctx, stream, world, rank, local)
    for _ in range(args.warmup):
        r.step()
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
        r.step()
        ev[i][1].record(stream)
        stats = r.job.stats()
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
            r.step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    clk["samples_in_timed_region"] = in_region
    step_ms = [s.elapsed_time(e) for s, e in ev]
    t_rank = _max_over_ranks(float(np.sum(step_ms)), world)
    ms_per_step = t_rank / args.steps
    points = stats["n_points"]
    updates = float(points) * c.plane_size * c.plane_size
    value = updates / (ms_per_step * 1e-3)

    # e2e through the C ABI with pinned host buffers; at large configs a
    # bounded number of steps (>= 3, ~E2E_SECONDS), all of them timed whole
    e2e_steps = int(min(args.steps, max(3, math.ceil(E2E_SECONDS / max(ms_per_step * 1e-3, 1e-9)))))
    e2e_warm = min(args.warmup, 1 if e2e_steps < args.steps else args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    e2e_clocks = ClockSampler(local)
    e2e_clocks.start()
    for i in range(e2e_warm + e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r.step_e2e()
        torch.cuda.synchronize()
        if i >= e2e_warm:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_clk = e2e_clocks.stop()
    e2e_t = _max_over_ranks(float(np.sum(e2e_ms)), world)
    e2e_value = updates / (e2e_t / e2e_steps * 1e-3)
    h2d = int(sc.objects.nbytes + sc.masks.nbytes)
    d2h = int(c.plane_size * c.plane_size * 8)

    peaks = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    f_meas = (clk.get("sm_mhz") or 0) * 1e6
    # dominant kernel, timed by CUDA events around its launches on this
    # stream inside wcgh_job_run; per-rank algorithmic updates per step
    k_ms = _max_over_ranks(float(np.mean(synth_ms)), world)
    roof = _roofline(r.job, c, points, r.rows, k_ms, f_max, f_meas, c.name)
    out = {
        "value": value, "ms_per_step": ms_per_step, "ms_per_hologram": ms_per_step,
        "config": {"workload": c.name, "object": c.object_size, "plane": c.plane_size,
                   "layers": c.n_layers, "saliency_frac": c.saliency_frac, "points": points,
                   "updates_per_hologram": updates, "method": r.job.spec.method,
                   "phase": "fixed-point quadratic + fp32 series", "ops": stats["ops"],
                   "parallelism": f"row tiles x{world}", "rows_per_rank": r.rows,
                   "gather": r.gather_mode,
                   "l2": "flushed between timed steps (256 MiB write, outside the step interval)"},
        "precompute_ms": r.precompute_ms,
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_t / e2e_steps, "steps": e2e_steps,
                "step_ms": [round(v, 3) for v in e2e_ms], "clocks": e2e_clk,
                "warmup": e2e_warm,
                "path": ("HologramJob.upload (H2D from pinned host) -> run -> download (D2H of the "
                         "whole assembled plane, rank 0) through the C ABI")},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if extras and world == 1 and c.n_layers == 1:
        out["alt_methods"] = alt_methods(sc, r, args, ctx, stream, flush, updates)
    r.close()
    return out


def alt_methods(sc, r, args, ctx, stream, flush, updates):
    """The same hologram through the other synthesis methods (N=1)."""
    import torch

    from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene

    res = []
    h_main = r.job.download()
    for alt in [m for m in ("direct", "lut", "fft") if m != r.job.spec.method]:
        try:
            torch.cuda.synchronize()
            t_pre = time.perf_counter()
            ajob = HologramJob(spec_for_scene(sc, method=alt), ctx)
            torch.cuda.synchronize()
            a_pre = (time.perf_counter() - t_pre) * 1e3
            ajob.upload_dev(r.obj_d.data_ptr(), r.sal_d.data_ptr())
            t0 = time.perf_counter()
            ajob.run()
            torch.cuda.synchronize()
            one = time.perf_counter() - t0
            steps = int(min(args.steps, max(3, math.ceil(ALT_SECONDS / max(one, 1e-9)))))
            for _ in range(min(args.warmup, 2)):
                ajob.run()
            aev = []
            for _ in range(steps):
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
            res.append({
                "method": alt, "ms_per_hologram": a_ms, "steps": steps,
                "value": updates / (a_ms * 1e-3), "unit": UNIT,
                "note": ("same hologram (after_full), same numerator as `value`; "
                         + {"direct": "Eq.(1) per point x pixel on the SFU (K3)",
                            "lut": "the reference's block-LUT superposition (K4)",
                            "fft": "correlation with the point fringe by hand-written FFTs, O(Nh^2 log Nh)"}[alt]),
                "algorithmic_updates": ast["updates"],
                "precompute_ms": a_pre,
                "rel_l2_vs_main": float(np.linalg.norm(h_alt - h_main) / np.linalg.norm(h_main)),
            })
            ajob.close()
        except Exception as e:  # noqa: BLE001
            res.append({"method": alt, "error": str(e)})
    return res


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_2211_09938_b200 import _lib, scenes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    # functional check of the multi-rank path on a single GPU only (numbers
    # from such a run are not measurements): all ranks on device 0
    same_dev = os.environ.get("WCGH_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL refuses two ranks on one device, so the same-device check
        # rendezvouses over gloo unless told otherwise
        backend = os.environ.get("WCGH_BENCH_BACKEND", "gloo" if same_dev else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    peers = [d for d in range(torch.cuda.device_count())
             if d != local and torch.cuda.can_device_access_peer(local, d)]
    props = torch.cuda.get_device_properties(local)
    print(f"[bench rank {rank}/{world}] cuda:{local} {props.name} ({props.multi_processor_count} SMs, "
          f"uuid {getattr(props, 'uuid', '?')}), peer access to {peers}"
          f"{' (WCGH_BENCH_SAME_DEVICE: functional check only)' if same_dev else ''}",
          file=sys.stderr, flush=True)
    ctx = _lib.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    sc = scenes.make_scene(args.config)
    head = measure(sc, args.method, args, ctx, stream, world, rank, local, flush,
                   extras=not args.no_extra)
    extra = {}
    if not args.no_extra and args.config != 1:
        sc1 = scenes.make_scene(1)
        extra["cfg1"] = measure(sc1, None, args, ctx, stream, world, rank, local, flush,
                                extras=False)
    if rank == 0:
        out = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian-blob objects, smooth-threshold masks; SURVEY.md §8(d))",
            **{k: v for k, v in head.items() if k not in ("value", "ms_per_step")},
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                out["cpu_baseline"] = reference_cpu_sample(sc, budget_s=args.cpu_seconds)
                out["cpu_baseline_direct_formula"] = reference_direct_rate()
            except Exception as e:  # the baseline is reported, never required
                out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                                       "sample": f"failed: {e}"}
        if extra:
            ex = {}
            for name, m in extra.items():
                e = {"value": m["value"], "unit": UNIT, "ms_per_hologram": m["ms_per_step"],
                     "config": m["config"], "roofline": m["roofline"], "e2e": m["e2e"],
                     "gpu_launches": m["gpu_launches"], "clocks": m["clocks"]}
                if world == 1 and not args.no_cpu_baseline:
                    try:
                        e["cpu_baseline"] = reference_cpu_sample(scenes.make_scene(1))
                    except Exception as err:  # noqa: BLE001
                        e["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(err)}
                ex[name] = e
            out["extra_configs"] = ex
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
