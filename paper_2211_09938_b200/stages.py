"""numpy-level wrappers of the C-ABI stage entry points (include/wcgh.h).

Each function runs on the GPU through libwcgh.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

_DT = {np.dtype(np.uint8): L.U8, np.dtype(np.float32): L.F32, np.dtype(np.float64): L.F64}


def _dtype(a: np.ndarray) -> int:
    try:
        return _DT[a.dtype]
    except KeyError:
        raise L.ValidationError(f"unsupported sample dtype {a.dtype}") from None


def _ctx(ctx):
    return ctx or L.default_context()


def haar_analyze(image: np.ndarray, levels: int = 3, scale: float = 1.0, ctx=None) -> np.ndarray:
    """Flat pyramid: approx, then (h, v, d) per level, finest first."""
    image = np.ascontiguousarray(image)
    n = image.shape[0]
    if image.ndim != 2 or image.shape[1] != n:
        raise L.ValidationError("haar_analyze: image must be square")
    t, s = 0, n
    for _ in range(max(levels, 0)):
        s //= 2
        t += 3 * s * s
    out = np.empty(max(t + s * s, 1))
    c = _ctx(ctx)
    L.check(c.lib.wcgh_haar_analyze(c.h, L.ptr(image), _dtype(image), scale, n, levels, L.ptr(out)))
    return out


def expand_residual(h, v, d, ctx=None) -> np.ndarray:
    h, v, d = (np.ascontiguousarray(a, np.float64) for a in (h, v, d))
    if not (h.shape == v.shape == d.shape):
        raise L.ValidationError("expand_residual: detail subbands differ in size")
    m = h.shape[0]
    out = np.empty((2 * m, 2 * m))
    c = _ctx(ctx)
    L.check(c.lib.wcgh_expand_residual(c.h, L.ptr(h), L.ptr(v), L.ptr(d), m, L.ptr(out)))
    return out


def quantize_saliency(sal: np.ndarray, ctx=None) -> np.ndarray:
    sal = np.ascontiguousarray(sal)
    n = sal.shape[0]
    if sal.ndim != 2 or sal.shape[1] != n:
        raise L.ValidationError("quantize_saliency: map must be square")
    out = np.empty(n * n // 4 + n * n // 16 + n * n // 64)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_quantize_saliency(c.h, L.ptr(sal), _dtype(sal), n, L.ptr(out)))
    return out


def analyze(obj: np.ndarray, sal: np.ndarray, t=(0.5, 0.7, 0.9), en=(1, 1, 1), offset: int = 0,
            layer: int = 0, obj_scale: float = 1.0, want_points=True, want_cells=True, ctx=None):
    obj = np.ascontiguousarray(obj)
    sal = np.ascontiguousarray(sal)
    n = obj.shape[0]
    n2 = n * n
    pyr = np.empty(n2 // 64 + 3 * (n2 // 4 + n2 // 16 + n2 // 64))
    sp = np.empty(n2 // 4 + n2 // 16 + n2 // 64)
    masks = np.empty(n2 // 16 + n2 // 4 + n2, np.uint8)
    a_eff = np.empty((n, n), np.float32)
    cells = np.empty(n2 // 16 + n2 // 4 + n2, np.uint32) if want_cells else None
    pts = np.empty(n2, L.POINT_DTYPE) if want_points else None
    a = L.Analysis()
    a.pyramid = pyr.ctypes.data_as(C.POINTER(C.c_double))
    a.sal_pyr = sp.ctypes.data_as(C.POINTER(C.c_double))
    a.masks = masks.ctypes.data_as(C.POINTER(C.c_uint8))
    a.a_eff = a_eff.ctypes.data_as(C.POINTER(C.c_float))
    if cells is not None:
        a.cells = cells.ctypes.data_as(C.POINTER(C.c_uint32))
    if pts is not None:
        a.points = pts.ctypes.data_as(C.POINTER(L.Point))
    plan = L.Plan(t[0], t[1], t[2], int(en[0]), int(en[1]), int(en[2]))
    c = _ctx(ctx)
    L.check(c.lib.wcgh_analyze(c.h, L.ptr(obj), _dtype(obj), obj_scale, L.ptr(sal), _dtype(sal), n,
                               C.byref(plan), offset, layer, C.byref(a)))
    out = {"pyramid": pyr, "sal_pyr": sp, "masks": masks, "a_eff": a_eff,
           "ops": np.array(list(a.ops), np.uint64), "n_points": int(a.n_points)}
    if pts is not None:
        out["points"] = pts[: a.n_points].copy()
    if cells is not None:
        cc = list(a.cell_counts)
        out["cell_counts"] = cc
        out["cells"] = [cells[: cc[0]].copy(), cells[cc[0]: cc[0] + cc[1]].copy(),
                        cells[cc[0] + cc[1]: cc[0] + cc[1] + cc[2]].copy()]
    return out


def synth_points(points: np.ndarray, layers, nh: int, row0: int = 0, rows: int | None = None,
                 phase: str = "fixed", ctx=None) -> np.ndarray:
    points = np.ascontiguousarray(points, L.POINT_DTYPE)
    rows = nh - row0 if rows is None else rows
    lay = (L.Layer * len(layers))(*[L.Layer(*t) for t in layers])
    out = np.empty((rows, nh), np.complex64)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_synth_points(c.h, L.ptr(points), len(points), lay, len(layers), nh, row0,
                                    rows, L.PHASE_FIXED if phase == "fixed" else L.PHASE_FP64,
                                    L.ptr(out)))
    return out


def build_block_lut(layer, n: int, block: int, ctx=None) -> np.ndarray:
    span = 2 * n - 1
    out = np.empty((span, span), np.complex64)
    lay = L.Layer(*layer)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_build_block_lut(c.h, C.byref(lay), n, block, L.ptr(out)))
    return out


def apply_blocks(plane: np.ndarray, layer, block: int, cells, weights, ctx=None) -> int:
    """plane (n x n complex64, in place) += sum_i w_i crop(S_B at cell_i)."""
    assert plane.dtype == np.complex64 and plane.flags.c_contiguous
    n = plane.shape[0]
    cells = np.ascontiguousarray(cells, np.uint32)
    weights = np.ascontiguousarray(weights, np.float32)
    lay = L.Layer(*layer)
    ops = C.c_uint64(0)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_apply_blocks(c.h, C.byref(lay), n, block, L.ptr(cells), L.ptr(weights),
                                    len(cells), L.ptr(plane), C.byref(ops)))
    return int(ops.value)


def refine(plane: np.ndarray, layer, h, v, d, saliency_finer, threshold: float, ctx=None):
    assert plane.dtype == np.complex64 and plane.flags.c_contiguous
    n = plane.shape[0]
    h, v, d = (np.ascontiguousarray(a, np.float64) for a in (h, v, d))
    sal = np.ascontiguousarray(saliency_finer, np.float64)
    m = h.shape[0]
    if v.shape != h.shape or d.shape != h.shape:
        raise L.ValidationError("refine: residual components differ in size")
    if sal.shape != (2 * m, 2 * m):
        raise L.ValidationError("refine: saliency level does not match the residual resolution")
    mask = np.empty((2 * m, 2 * m), np.uint8)
    lay = L.Layer(*layer)
    ops = C.c_uint64(0)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_refine(c.h, C.byref(lay), n, L.ptr(h), L.ptr(v), L.ptr(d), m, L.ptr(sal),
                              float(threshold), L.ptr(plane), L.ptr(mask), C.byref(ops)))
    return mask, int(ops.value)


def haar_synthesize(pyramid_flat: np.ndarray, n: int, levels: int = 3, ctx=None) -> np.ndarray:
    """haar_synthesize (haar.cpp:76-86) on the device from the flat pyramid of
    haar_analyze: n x n doubles, bit-identical to the reference."""
    flat = np.ascontiguousarray(pyramid_flat, np.float64)
    out = np.empty((n, n))
    c = _ctx(ctx)
    L.check(c.lib.wcgh_haar_synthesize(c.h, L.ptr(flat), int(n), int(levels), L.ptr(out)))
    return out


def upsample_replicate(coarse: np.ndarray, factor: int, ctx=None) -> np.ndarray:
    """upsample_replicate (haar.cpp:98-109) on the device."""
    c_in = np.ascontiguousarray(coarse, np.float64)
    h, w = c_in.shape
    out = np.empty((h * factor, w * factor))
    c = _ctx(ctx)
    L.check(c.lib.wcgh_upsample_replicate(c.h, L.ptr(c_in), w, h, int(factor), L.ptr(out)))
    return out


def point_fringe(layer, dx: int, dy: int, ctx=None) -> complex:
    """point_fringe (fringe_lut.cpp:27-32) in fp64 on the device."""
    out = np.empty(2)
    lay = L.Layer(*layer)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_point_fringe(c.h, C.byref(lay), int(dx), int(dy), L.ptr(out)))
    return complex(out[0], out[1])


_CPLX = {np.dtype(np.complex64): L.F32, np.dtype(np.complex128): L.F64}


class DevicePlane:
    """wcgh_plane: an n x n complex64 hologram resident on the device; stage
    calls (DeviceLut.apply_blocks / refine) accumulate into it with no host
    round trip."""

    def __init__(self, n: int, ctx=None):
        self.ctx = _ctx(ctx)
        self.n = int(n)
        h = C.c_void_p()
        L.check(self.ctx.lib.wcgh_plane_create(self.ctx.h, self.n, C.byref(h)))
        self.h = h

    def zero(self) -> "DevicePlane":
        L.check(self.ctx.lib.wcgh_plane_zero(self.h))
        return self

    def upload(self, plane: np.ndarray) -> "DevicePlane":
        a = np.ascontiguousarray(plane)
        if a.shape != (self.n, self.n) or a.dtype not in _CPLX:
            raise L.ValidationError("plane_upload: need an n x n complex64/complex128 array")
        L.check(self.ctx.lib.wcgh_plane_upload(self.h, L.ptr(a), _CPLX[a.dtype]))
        return self

    def download(self, dtype=np.complex64) -> np.ndarray:
        out = np.empty((self.n, self.n), dtype)
        L.check(self.ctx.lib.wcgh_plane_download(self.h, L.ptr(out), _CPLX[np.dtype(dtype)]))
        return out

    def dev_ptr(self) -> int:
        return int(self.ctx.lib.wcgh_plane_dev(self.h) or 0)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.wcgh_plane_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceLut:
    """wcgh_lut: a block LUT S_B resident on the device — the caller's samples
    (a FringeLut's support, complex64 or complex128) uploaded once, or built
    on the device when samples is None."""

    def __init__(self, layer, n: int, block: int, samples: np.ndarray | None = None, ctx=None):
        self.ctx = _ctx(ctx)
        self.layer, self.n, self.block = tuple(layer), int(n), int(block)
        lay = L.Layer(*layer)
        if samples is None:
            sp, dt = None, L.F32
        else:
            a = np.ascontiguousarray(samples)
            span = 2 * self.n - 1
            if a.shape != (span, span) or a.dtype not in _CPLX:
                raise L.ValidationError("FringeLut: support must be (2N-1) x (2N-1) complex")
            sp, dt = L.ptr(a), _CPLX[a.dtype]
        h = C.c_void_p()
        L.check(self.ctx.lib.wcgh_lut_create(self.ctx.h, C.byref(lay), self.n, self.block, sp, dt,
                                             C.byref(h)))
        self.h = h

    def download(self) -> np.ndarray:
        span = 2 * self.n - 1
        out = np.empty((span, span), np.complex64)
        L.check(self.ctx.lib.wcgh_lut_download(self.h, L.ptr(out)))
        return out

    def apply_blocks(self, plane: DevicePlane, cells, w_re, w_im=None) -> int:
        """plane += sum_i (w_re + i w_im)_i crop(S_B at cell_i); returns ops."""
        cells = np.ascontiguousarray(cells, np.uint32)
        wr = np.ascontiguousarray(w_re, np.float32)
        wi = None if w_im is None else np.ascontiguousarray(w_im, np.float32)
        ops = C.c_uint64(0)
        L.check(self.ctx.lib.wcgh_lut_apply_blocks(self.h, L.ptr(cells), L.ptr(wr), L.ptr(wi),
                                                   len(cells), plane.h, C.byref(ops)))
        return int(ops.value)

    def refine(self, plane: DevicePlane, h, v, d, saliency_finer, threshold: float):
        h, v, d = (np.ascontiguousarray(a, np.float64) for a in (h, v, d))
        sal = np.ascontiguousarray(saliency_finer, np.float64)
        m = h.shape[0]
        if v.shape != h.shape or d.shape != h.shape:
            raise L.ValidationError("expand_residual: detail subbands differ in size")
        if sal.shape != (2 * m, 2 * m):
            raise L.ValidationError("refine: saliency level does not match the residual resolution")
        mask = np.empty((2 * m, 2 * m), np.uint8)
        ops = C.c_uint64(0)
        L.check(self.ctx.lib.wcgh_lut_refine(self.h, L.ptr(h), L.ptr(v), L.ptr(d), m, L.ptr(sal),
                                             float(threshold), plane.h, L.ptr(mask), C.byref(ops)))
        return mask, int(ops.value)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.wcgh_lut_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def write_cgh1(path, plane: np.ndarray, layer) -> None:
    """save_hologram (image_io.cpp:220-242): CGH1 header + f32 (re, im) payload."""
    plane = np.ascontiguousarray(plane, np.complex64)
    n = plane.shape[0]
    if plane.ndim != 2 or plane.shape[1] != n:
        raise L.ValidationError("save_hologram: field size does not match scene plane_size")
    lay = L.Layer(*layer)
    L.check(L.load().wcgh_write_cgh1(str(path).encode(), L.ptr(plane), n, C.byref(lay)))


def read_cgh1(path):
    """load_hologram (image_io.cpp:244-278) -> (plane complex64, (wavelength, pitch, z))."""
    lib = L.load()
    n = C.c_int(0)
    lay = L.Layer()
    L.check(lib.wcgh_read_cgh1(str(path).encode(), None, 0, C.byref(n), C.byref(lay)))
    plane = np.empty((n.value, n.value), np.complex64)
    L.check(lib.wcgh_read_cgh1(str(path).encode(), L.ptr(plane), plane.size, C.byref(n), C.byref(lay)))
    return plane, (lay.wavelength, lay.pitch, lay.z)


# ---- reconstruction and metrics (angular_spectrum.cpp, fft.cpp, metrics.cpp) ----

def _complex_in(field: np.ndarray):
    field = np.ascontiguousarray(field)
    if field.dtype == np.complex64:
        return field, L.F32
    if field.dtype == np.complex128:
        return field, L.F64
    return np.ascontiguousarray(field, np.complex128), L.F64


def _square_side(field: np.ndarray, what: str) -> int:
    if field.ndim != 2 or field.shape[0] != field.shape[1]:
        raise L.ValidationError(f"{what}: field must be square")
    return field.shape[0]


def fft_2d(field: np.ndarray, inverse: bool = False, ctx=None) -> np.ndarray:
    """fft_2d (fft.cpp:45-68) on the device: complex128 in and out."""
    f = np.ascontiguousarray(field, np.complex128)
    n = _square_side(f, "fft_2d")
    out = np.empty_like(f)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_fft_2d(c.h, L.ptr(f), n, int(bool(inverse)), L.ptr(out)))
    return out


def propagation_kernel(layer, n: int, z_signed: float, ctx=None) -> np.ndarray:
    """build_kernel (angular_spectrum.cpp:11-33) transfer samples, DC first."""
    out = np.empty((n, n), np.complex128)
    lay = L.Layer(*layer)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_propagation_kernel(c.h, C.byref(lay), n, float(z_signed), L.ptr(out)))
    return out


def propagate(field: np.ndarray, layer, z_signed: float, ctx=None) -> np.ndarray:
    """propagate (angular_spectrum.cpp:35-45): complex64 or complex128 field."""
    f, dt = _complex_in(field)
    n = _square_side(f, "propagate")
    out = np.empty((n, n), np.complex128)
    lay = L.Layer(*layer)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_propagate(c.h, L.ptr(f), dt, n, C.byref(lay), float(z_signed), L.ptr(out)))
    return out


def reconstruct(hologram: np.ndarray, layer, intensity: bool = False, ctx=None) -> np.ndarray:
    """reconstruct (angular_spectrum.cpp:47-61): back-propagate by -z, |.| or |.|^2."""
    f, dt = _complex_in(hologram)
    n = _square_side(f, "reconstruct")
    out = np.empty((n, n))
    lay = L.Layer(*layer)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_reconstruct(c.h, L.ptr(f), dt, n, C.byref(lay), int(bool(intensity)),
                                   L.ptr(out)))
    return out


def ssim(a: np.ndarray, b: np.ndarray, window: int = 8, k1: float = 0.01, k2: float = 0.03,
         dynamic_range: float = 1.0, ctx=None) -> float:
    """ssim (metrics.cpp:49-85): mean box-window SSIM on the device."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape or a.ndim != 2:
        raise L.ValidationError("ssim: image sizes differ")
    h, w = a.shape
    out = C.c_double(0.0)
    c = _ctx(ctx)
    L.check(c.lib.wcgh_ssim(c.h, L.ptr(a), L.ptr(b), w, h, int(window), float(k1), float(k2),
                            float(dynamic_range), C.byref(out)))
    return float(out.value)


def random_phase_field(amplitude: np.ndarray, seed: int) -> np.ndarray:
    """random_phase_field (synthesis.cpp:288-296) through the library's host
    function: polar(amplitude, U[0, 2pi)) from std::mt19937_64(seed) — the
    reference's own engine, so the complex128 result is bit-identical."""
    a = np.ascontiguousarray(amplitude, np.float64)
    if a.ndim != 2:
        raise L.ValidationError("random_phase_field: amplitude must be 2-D")
    out = np.empty(a.shape, np.complex128)
    L.check(L.load().wcgh_random_phase_field(L.ptr(a), a.shape[1], a.shape[0],
                                             int(seed) & 0xFFFFFFFFFFFFFFFF, L.ptr(out)))
    return out


def write_cghl(path, lut: np.ndarray, n: int, block: int, layer) -> None:
    """lut_cache_store (fringe_lut.cpp:95-115): CGHL header + f32 (re, im) payload."""
    lut = np.ascontiguousarray(lut, np.complex64)
    if lut.shape != (2 * n - 1, 2 * n - 1):
        raise L.ValidationError("lut cache: support size does not match the plane size")
    lay = L.Layer(*layer)
    L.check(L.load().wcgh_write_cghl(str(path).encode(), L.ptr(lut), n, int(block), C.byref(lay)))


def read_cghl(path):
    """CGHL file -> (lut complex64 (2N-1)^2, N, block, (wavelength, pitch, z))."""
    lib = L.load()
    n, b = C.c_int(0), C.c_int(0)
    lay = L.Layer()
    L.check(lib.wcgh_read_cghl(str(path).encode(), None, 0, C.byref(n), C.byref(b), C.byref(lay)))
    span = 2 * n.value - 1
    lut = np.empty((span, span), np.complex64)
    L.check(lib.wcgh_read_cghl(str(path).encode(), L.ptr(lut), lut.size, C.byref(n), C.byref(b),
                               C.byref(lay)))
    return lut, n.value, b.value, (lay.wavelength, lay.pitch, lay.z)
