"""Hologram jobs over the C ABI (wcgh_job_*): resident inputs, device plane.

This is the call a user (or bench.py) makes to synthesize a saliency-gated
progressive hologram on one GPU; multi-GPU row tiles are in `tiles.py`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass
class JobSpec:
    object_size: int
    plane_size: int
    layers: list[tuple[float, float, float]]  # (wavelength, pitch, z) per layer
    t_ll: float = 0.5
    t_l: float = 0.7
    t_full: float = 0.9
    enable_ll: bool = True
    enable_l: bool = True
    enable_full: bool = True
    method: str = "direct"        # "direct" | "lut" | "fft"
    phase: str = "fixed"          # "fixed" | "fp64"
    row0: int = 0
    rows: int | None = None
    obj_dtype: str = "u8"         # "u8" | "f32" | "f64" | "c128" (complex object)
    obj_scale: float = 1.0
    sal_dtype: str = "u8"


_DT = {"u8": L.U8, "f32": L.F32, "f64": L.F64, "c128": L.C128}
_NP = {"u8": np.uint8, "f32": np.float32, "f64": np.float64, "c128": np.complex128}


def _make_desc(spec: JobSpec):
    """wcgh_desc for a spec (and the layer array it points to, kept alive by the caller)."""
    layers = (L.Layer * len(spec.layers))(*[L.Layer(*t) for t in spec.layers])
    d = L.Desc()
    d.object_size = spec.object_size
    d.plane_size = spec.plane_size
    d.n_layers = len(spec.layers)
    d.layers = C.cast(layers, C.POINTER(L.Layer))
    d.plan = L.Plan(spec.t_ll, spec.t_l, spec.t_full, int(spec.enable_ll),
                    int(spec.enable_l), int(spec.enable_full))
    methods = {"direct": L.METHOD_DIRECT, "lut": L.METHOD_LUT, "fft": L.METHOD_FFT}
    if spec.method not in methods:
        raise L.ValidationError(f"unknown method {spec.method!r}")
    d.method = methods[spec.method]
    d.phase_mode = L.PHASE_FIXED if spec.phase == "fixed" else L.PHASE_FP64
    d.row0 = spec.row0
    d.rows = spec.rows if spec.rows is not None else spec.plane_size - spec.row0
    d.obj_dtype = _DT[spec.obj_dtype]
    d.obj_scale = spec.obj_scale
    d.sal_dtype = _DT[spec.sal_dtype]
    return d, layers


class HologramJob:
    def __init__(self, spec: JobSpec, ctx: L.Context | None = None):
        self.ctx = ctx or L.default_context()
        self.spec = spec
        self.rows = spec.rows if spec.rows is not None else spec.plane_size - spec.row0
        d, self._layers = _make_desc(spec)
        self.desc = d
        h = C.c_void_p()
        L.check(self.ctx.lib.wcgh_job_create(self.ctx.h, C.byref(d), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.wcgh_job_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_inputs(self, objects: np.ndarray, saliency: np.ndarray):
        n = self.spec.object_size
        nl = len(self.spec.layers)
        if objects.size != nl * n * n or saliency.size != nl * n * n:
            raise L.ValidationError("synthesize_progressive: object/saliency size does not match the scene")
        if objects.dtype != _NP[self.spec.obj_dtype] or saliency.dtype != _NP[self.spec.sal_dtype]:
            raise L.ValidationError("object/saliency dtype does not match the job spec")

    def upload(self, objects: np.ndarray, saliency: np.ndarray) -> None:
        objects = np.ascontiguousarray(objects)
        saliency = np.ascontiguousarray(saliency)
        self._check_inputs(objects, saliency)
        L.check(self.ctx.lib.wcgh_job_upload(self.h, L.ptr(objects), L.ptr(saliency)))

    def upload_dev(self, obj_ptr: int, sal_ptr: int) -> None:
        L.check(self.ctx.lib.wcgh_job_upload_dev(self.h, C.c_void_p(obj_ptr), C.c_void_p(sal_ptr)))

    def run(self) -> None:
        L.check(self.ctx.lib.wcgh_job_run(self.h))

    def analyze(self) -> dict:
        """Front end only (K1/K2): op counts, point / cell count, ms_analysis."""
        L.check(self.ctx.lib.wcgh_job_analyze(self.h))
        return self.stats()

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        n = self.spec.plane_size
        if out is None:
            out = np.empty((self.rows, n), np.complex64)
        assert out.dtype == np.complex64 and out.flags.c_contiguous and out.size == self.rows * n
        L.check(self.ctx.lib.wcgh_job_download(self.h, L.ptr(out)))
        return out

    def download_a_eff(self) -> np.ndarray:
        """A_eff of the last run/analyze, (n_layers, No, No) fp32 (complex64
        for a "c128" object)."""
        no = self.spec.object_size
        out = np.empty((len(self.spec.layers), no, no), np.float32)
        L.check(self.ctx.lib.wcgh_job_download_a_eff(self.h, L.ptr(out)))
        if self.spec.obj_dtype != "c128":
            return out
        im = np.empty_like(out)
        L.check(self.ctx.lib.wcgh_job_download_a_eff_im(self.h, L.ptr(im)))
        return (out + 1j * im).astype(np.complex64)

    def download_points_im(self) -> np.ndarray:
        """Imaginary amplitudes of download_points()' records ("c128" objects)."""
        n = self.stats()["n_points"]
        out = np.empty(n, np.float32)
        L.check(self.ctx.lib.wcgh_job_download_points_im(self.h, L.ptr(out), n))
        return out

    def download_points(self) -> np.ndarray:
        """Compacted point records of the last direct-method run/analyze."""
        n = C.c_int64(0)
        L.check(self.ctx.lib.wcgh_job_download_points(self.h, None, 0, C.byref(n)))
        out = np.empty(n.value, L.POINT_DTYPE)
        L.check(self.ctx.lib.wcgh_job_download_points(self.h, L.ptr(out), n.value, C.byref(n)))
        return out

    def download_stages(self) -> np.ndarray:
        n = self.spec.plane_size
        out = np.empty((4, self.rows, n), np.complex64)
        L.check(self.ctx.lib.wcgh_job_download_stages(self.h, L.ptr(out)))
        return out

    def reconstruct(self, layer=None, intensity: bool = False) -> np.ndarray:
        """reconstruct (angular_spectrum.cpp:47-61) of the last run's plane on the
        device (whole-plane jobs); layer = (wavelength, pitch, z), default layer 0."""
        n = self.spec.plane_size
        lay = L.Layer(*(layer if layer is not None else self.spec.layers[0]))
        out = np.empty((n, n))
        L.check(self.ctx.lib.wcgh_job_reconstruct(self.h, C.byref(lay), int(bool(intensity)),
                                                  L.ptr(out)))
        return out

    def load_lut(self, layer: int, block: int, lut: np.ndarray) -> None:
        """LUT method: use caller LUT samples (e.g. a CGHL cache) for (layer, block)."""
        lut = np.ascontiguousarray(lut, np.complex64)
        L.check(self.ctx.lib.wcgh_job_load_lut(self.h, int(layer), int(block), L.ptr(lut)))

    def use_lut(self, layer: int, lut) -> None:
        """LUT method: superpose a device LUT (stages.DeviceLut — e.g. the
        caller's FringeLut samples) for `layer` at its block size."""
        L.check(self.ctx.lib.wcgh_job_use_lut(self.h, int(layer), lut.h))

    def set_peer_planes(self, ptrs) -> None:
        """Fused row-tile gather: device pointers of full planes (this rank's and
        the IPC-mapped peers') that every run also writes its band into."""
        arr = (C.c_void_p * max(1, len(ptrs)))(*[C.c_void_p(int(p)) for p in ptrs])
        L.check(self.ctx.lib.wcgh_job_set_peer_planes(self.h, arr, len(ptrs)))

    def plane_dev_ptr(self) -> int:
        return int(self.ctx.lib.wcgh_job_plane_dev(self.h) or 0)

    def stats(self) -> dict:
        s = L.Stats()
        L.check(self.ctx.lib.wcgh_job_stats(self.h, C.byref(s)))
        return {
            "ops": [int(v) for v in s.ops], "n_points": int(s.n_points), "updates": float(s.updates),
            "ms_analysis": s.ms_analysis, "ms_synthesis": s.ms_synthesis, "ms_reduce": s.ms_reduce,
            "ms_total": s.ms_total, "synth_launches": s.synth_launches,
            "total_launches": s.total_launches,
        }

    def direct_form(self) -> tuple:
        """(form, hold) of the K3 kernel the last direct-method run launched
        (0 per-pixel, 1 recurrence, 2 chirp-factored recurrence, 3 fp64 phase)."""
        f, h = C.c_int(-1), C.c_int(0)
        L.check(self.ctx.lib.wcgh_job_direct_form(self.h, C.byref(f), C.byref(h)))
        return int(f.value), int(h.value)

    def __call__(self, objects: np.ndarray, saliency: np.ndarray) -> np.ndarray:
        self.upload(objects, saliency)
        self.run()
        return self.download()


def spec_for_scene(scene, method: str | None = None, phase: str = "fixed", row0: int = 0,
                   rows: int | None = None, **plan) -> JobSpec:
    c = scene.config
    return JobSpec(object_size=c.object_size, plane_size=c.plane_size,
                   layers=[(c.wavelength, c.pitch, z) for z in c.depths],
                   method=method or c.method, phase=phase, row0=row0, rows=rows, **plan)


def write_job_cgh1(job: HologramJob, path, stage: int = -1) -> None:
    """The job's last plane (stage < 0) or LUT stage snapshot as a CGH1 file."""
    L.check(job.ctx.lib.wcgh_job_write_cgh1(job.h, str(path).encode(), int(stage)))


def synthesize_multi(spec: JobSpec, objects: np.ndarray, masks: np.ndarray, devices) -> tuple:
    """wcgh_synthesize_multi: the whole plane as row bands over `devices` (one
    host thread and context each, a device may repeat) -> (plane, stats)."""
    d, layers = _make_desc(spec)
    objects = np.ascontiguousarray(objects, _NP[spec.obj_dtype])
    masks = np.ascontiguousarray(masks, _NP[spec.sal_dtype])
    n = spec.plane_size
    out = np.empty((n, n), np.complex64)
    devs = (C.c_int * len(devices))(*devices)
    st = L.Stats()
    L.check(L.load().wcgh_synthesize_multi(len(devices), devs, C.byref(d), L.ptr(objects),
                                           L.ptr(masks), L.ptr(out), C.byref(st)))
    del layers
    return out, {"ops": [int(v) for v in st.ops], "n_points": int(st.n_points),
                 "updates": float(st.updates), "ms_total": st.ms_total}
