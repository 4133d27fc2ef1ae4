"""Python mirror of the reference's hot-path API (wavecgh 0.1.0), on the GPU.

Same names, argument meaning and error behaviour as the reference's C++
free functions and types (paths under /root/reference/proj):

  field.hpp:17-143       SceneParams, make_scene, OpLevel, OpCounter
  haar.hpp:14-51         DetailBands, HaarPyramid, haar_analyze, haar_synthesize,
                         expand_residual, upsample_replicate
  saliency.hpp:11-30     SaliencyPyramid, quantize_saliency, uniform_saliency
  fringe_lut.hpp:15-62   point_fringe, FringeLut, build_block_lut, LutSet,
                         lut_cache_store, lut_cache_load (CGHL files)
  synthesis.hpp:18-104   RefinementPlan, GateMask, ProgressiveResult, GridCell,
                         apply_block, synthesize_base, refine,
                         synthesize_progressive, synthesize_pointwise_oracle
  fft.hpp, angular_spectrum.hpp, metrics.hpp
                         fft_2d, PropagationKernel, build_kernel, propagate,
                         reconstruct, ssim, StageMetrics, MetricsReport,
                         build_report (the validation step after the path)

Images are numpy arrays indexed [y, x] (RealImage/ComplexField are row-major
with at(x, y)). Every hot-path call runs on the sm_100a kernels through the
C ABI (include/wcgh.h); the few host-side helpers (haar_synthesize,
upsample_replicate, uniform_saliency) are validation utilities that the
reference's tests use, not part of the synthesis path. Planes are computed
in complex64 and returned as complex128 (the reference's ComplexField type).
`workers` is accepted and ignored: results never depend on it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib as L
from . import stages
from .hologram import HologramJob, JobSpec

ValidationError = L.ValidationError
IoError = L.IoError


class StaleCacheError(IoError):
    """errors.hpp:24-27"""


def is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


# ---- field.hpp ------------------------------------------------------------------

class SceneParams:
    """field.hpp:91-108; validation field.cpp:71-80."""

    def __init__(self, wavelength: float, pitch: float, z: float, plane_size: int):
        if not wavelength > 0.0:
            raise ValidationError("scene: wavelength must be positive")
        if not pitch > 0.0:
            raise ValidationError("scene: pitch must be positive")
        if not z > 0.0:
            raise ValidationError("scene: z must be positive")
        if not is_power_of_two(int(plane_size)):
            raise ValidationError(f"scene: plane_size must be a power of two, got {plane_size}")
        self._t = (float(wavelength), float(pitch), float(z), int(plane_size))

    def wavelength(self) -> float:
        return self._t[0]

    def pitch(self) -> float:
        return self._t[1]

    def z(self) -> float:
        return self._t[2]

    def plane_size(self) -> int:
        return self._t[3]

    def wave_number(self) -> float:
        return 2.0 * math.pi / self._t[0]  # field.cpp:82

    def layer(self):
        return self._t[:3]

    def __eq__(self, other) -> bool:
        return isinstance(other, SceneParams) and self._t == other._t

    def __repr__(self):
        return "SceneParams(%r, %r, %r, %r)" % self._t


def make_scene(wavelength: float, pitch: float, z: float, plane_size: int) -> SceneParams:
    return SceneParams(wavelength, pitch, z, plane_size)


class OpLevel(IntEnum):
    """field.hpp:114-120"""
    BASE_LLL = 0
    REFINE_LL = 1
    REFINE_L = 2
    REFINE_FULL = 3
    POINTWISE_ORACLE = 4


ALL_OP_LEVELS = list(OpLevel)
STAGE_OP_LEVELS = [OpLevel.BASE_LLL, OpLevel.REFINE_LL, OpLevel.REFINE_L, OpLevel.REFINE_FULL]
STAGE_NAMES = ["base_LLL", "after_LL", "after_L", "after_full"]


class OpCounter:
    """field.hpp:131-143: per-level tally of LUT block applications."""

    def __init__(self):
        self._c = [0] * len(OpLevel)

    def add(self, level: OpLevel, n: int) -> None:
        self._c[int(level)] += int(n)

    def get(self, level: OpLevel) -> int:
        return self._c[int(level)]

    def total(self) -> int:
        return sum(self._c)


def _square(a: np.ndarray, what: str) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValidationError(f"{what} must be square")
    return a


def _require_finite(a: np.ndarray, what: str) -> None:
    if not np.all(np.isfinite(a)):
        raise ValidationError(f"{what}: non-finite sample")


# ---- haar.hpp -------------------------------------------------------------------

@dataclass
class DetailBands:
    h: np.ndarray
    v: np.ndarray
    d: np.ndarray


@dataclass
class HaarPyramid:
    approx: np.ndarray
    details: list = field(default_factory=list)  # details[0] finest
    original_size: int = 0

    def levels(self) -> int:
        return len(self.details)


def haar_analyze(image: np.ndarray, levels: int) -> HaarPyramid:
    """haar.cpp:52-74, on the GPU (fp64, bit-identical to the reference)."""
    if levels < 1:
        raise ValidationError("haar_analyze: levels must be >= 1")
    image = np.asarray(image)
    if image.ndim != 2 or image.shape[0] != image.shape[1]:
        raise ValidationError("haar_analyze: image must be square")
    n = image.shape[0]
    if n % (1 << levels):
        raise ValidationError(f"haar_analyze: side {n} not divisible by 2^{levels}")
    flat = stages.haar_analyze(np.ascontiguousarray(image, np.float64), levels)
    ma = n >> levels
    p = HaarPyramid(flat[: ma * ma].reshape(ma, ma).copy(), [], n)
    off = ma * ma
    for l in range(levels):
        m = n >> (l + 1)
        mm = m * m
        p.details.append(DetailBands(*(flat[off + k * mm: off + (k + 1) * mm].reshape(m, m).copy()
                                       for k in range(3))))
        off += 3 * mm
    return p


def haar_synthesize(pyramid: HaarPyramid) -> np.ndarray:
    """haar.cpp:76-86 (validation helper), on the device (bit-identical)."""
    if not pyramid.details:
        raise ValidationError("haar_synthesize: empty pyramid")
    cur = np.asarray(pyramid.approx, np.float64)
    if cur.shape[0] != cur.shape[1]:
        raise ValidationError("haar_synthesize: pyramid must be square (haar_analyze's)")
    side = cur.shape[0]
    for b in reversed(pyramid.details):
        if (side, side) != b.h.shape or b.v.shape != b.h.shape or b.d.shape != b.h.shape:
            raise ValidationError("haar_synthesize: subband sizes inconsistent")
        side *= 2
    flat = np.concatenate([cur.ravel()] + [np.concatenate([np.ravel(b.h), np.ravel(b.v), np.ravel(b.d)])
                                           for b in pyramid.details])
    return stages.haar_synthesize(flat, side, len(pyramid.details))


def expand_residual(h: np.ndarray, v: np.ndarray, d: np.ndarray) -> np.ndarray:
    """haar.cpp:88-96, on the GPU."""
    h, v, d = (np.asarray(a, np.float64) for a in (h, v, d))
    if not (h.shape == v.shape == d.shape):
        raise ValidationError("expand_residual: detail subbands differ in size")
    return stages.expand_residual(h, v, d)


def upsample_replicate(coarse: np.ndarray, factor: int) -> np.ndarray:
    """haar.cpp:98-109, on the device."""
    if factor < 2 or not is_power_of_two(factor):
        raise ValidationError("upsample_replicate: factor must be a power of two >= 2")
    return stages.upsample_replicate(coarse, factor)


# ---- saliency.hpp ---------------------------------------------------------------

class SaliencyPyramid:
    """saliency.hpp:11-26"""

    def __init__(self, full, half, quarter, eighth):
        self._maps = {1: full, 2: half, 4: quarter, 8: eighth}

    def by_factor(self, factor: int) -> np.ndarray:
        if factor not in self._maps:
            raise ValidationError("SaliencyPyramid: factor must be 1, 2, 4, or 8")
        return self._maps[factor]

    def full_size(self) -> int:
        return self._maps[1].shape[0]


def quantize_saliency(full: np.ndarray) -> SaliencyPyramid:
    """saliency.cpp:41-61, on the GPU (bit-identical block maxima)."""
    full = np.asarray(full)
    if full.ndim != 2 or full.shape[0] != full.shape[1]:
        raise ValidationError("quantize_saliency: map must be square")
    n = full.shape[0]
    if n % 8:
        raise ValidationError(f"quantize_saliency: side must be divisible by 8, got {n}")
    sp = stages.quantize_saliency(np.ascontiguousarray(full, np.float64))
    h2, q2 = n * n // 4, n * n // 16
    return SaliencyPyramid(np.asarray(full, np.float64), sp[:h2].reshape(n // 2, n // 2),
                           sp[h2:h2 + q2].reshape(n // 4, n // 4),
                           sp[h2 + q2:].reshape(n // 8, n // 8))


def uniform_saliency(n: int) -> np.ndarray:
    return np.ones((n, n))


# ---- fringe_lut.hpp -------------------------------------------------------------

LUT_BLOCK_SIZES = (1, 2, 4, 8)


def point_fringe(scene: SceneParams, dx: int, dy: int) -> complex:
    """fringe_lut.cpp:27-32 in fp64 on the device (sin/cos within 2 ulp)."""
    return stages.point_fringe(scene.layer(), dx, dy)


class FringeLut:
    """fringe_lut.hpp:45-62: (2N-1)^2 support of a B x B block (complex64,
    the CGHL payload precision)."""

    def __init__(self, scene: SceneParams, block_size: int, support: np.ndarray, _owned=False):
        if block_size not in LUT_BLOCK_SIZES:
            raise ValidationError(f"FringeLut: unsupported block size {block_size}")
        span = 2 * scene.plane_size() - 1
        if support.shape != (span, span):
            raise ValidationError("FringeLut: support must be (2N-1) x (2N-1)")
        # the reference's FringeLut owns its samples (value semantics,
        # fringe_lut.cpp:34-51): keep a private read-only copy, so the device
        # copy made once by device() can never go stale
        sup = support if _owned else np.array(support, copy=True)
        sup.setflags(write=False)
        self._scene, self._b, self._support = scene, block_size, sup
        self._dev = None

    def device(self) -> "stages.DeviceLut":
        """These samples on the device (uploaded on first use): what every
        apply_block / refine / synthesize_* call superposes, as the
        reference's apply_block_unchecked reads lut.support()
        (synthesis.cpp:18-42)."""
        if self._dev is None:
            self._dev = stages.DeviceLut(self._scene.layer(), self._scene.plane_size(), self._b,
                                         self._support)
        return self._dev

    def scene(self) -> SceneParams:
        return self._scene

    def block_size(self) -> int:
        return self._b

    def support(self) -> np.ndarray:
        return self._support

    def at_offset(self, dx: int, dy: int) -> complex:
        n = self._scene.plane_size()
        if dx <= -n or dx >= n or dy <= -n or dy >= n:
            raise ValidationError("FringeLut: offset outside support")
        return complex(self._support[dy + n - 1, dx + n - 1])


def build_block_lut(scene: SceneParams, block_size: int, workers: int = 1) -> FringeLut:
    """fringe_lut.cpp:53-93, on the GPU (fp64 sums, complex64 store)."""
    if block_size not in LUT_BLOCK_SIZES:
        raise ValidationError(f"build_block_lut: unsupported block size {block_size}")
    if block_size > scene.plane_size():
        raise ValidationError("build_block_lut: block size exceeds plane size")
    sup = stages.build_block_lut(scene.layer(), scene.plane_size(), block_size)
    return FringeLut(scene, block_size, sup, _owned=True)


def lut_cache_store(lut: FringeLut, path) -> None:
    """fringe_lut.cpp:95-115: CGHL header + f32 (re, im) payload."""
    stages.write_cghl(path, lut.support(), lut.scene().plane_size(), lut.block_size(),
                      lut.scene().layer())


def lut_cache_load(path, expected_scene: SceneParams, expected_block_size: int) -> FringeLut:
    """fringe_lut.cpp:117-166: IoError for unreadable / malformed files,
    StaleCacheError when the block size or scene does not match."""
    support, n, block, layer = stages.read_cghl(path)
    if block != expected_block_size:
        raise StaleCacheError(f"lut cache: block size {block} != expected {expected_block_size}")
    if n != expected_scene.plane_size() or tuple(layer) != tuple(expected_scene.layer()):
        raise StaleCacheError(f"lut cache: scene parameters in {path} do not match the requested scene")
    return FringeLut(expected_scene, expected_block_size, support, _owned=True)


class LutSet:
    """fringe_lut.hpp:135-145"""

    def __init__(self):
        self._luts: list[FringeLut] = []

    @staticmethod
    def build(scene: SceneParams, workers: int = 1) -> "LutSet":
        s = LutSet()
        for b in LUT_BLOCK_SIZES:
            s.put(build_block_lut(scene, b, workers))
        return s

    def put(self, lut: FringeLut) -> None:
        if self._luts and not (self._luts[0].scene() == lut.scene()):
            raise ValidationError("LutSet: mixed scene parameters")
        for i, e in enumerate(self._luts):
            if e.block_size() == lut.block_size():
                self._luts[i] = lut
                return
        self._luts.append(lut)

    def has(self, block_size: int) -> bool:
        return any(l.block_size() == block_size for l in self._luts)

    def of(self, block_size: int) -> FringeLut:
        for l in self._luts:
            if l.block_size() == block_size:
                return l
        raise ValidationError(f"LutSet: no LUT for block size {block_size}")


# ---- synthesis.hpp --------------------------------------------------------------

@dataclass
class RefinementPlan:
    """synthesis.hpp:18-29; validate: synthesis.cpp:127-131."""
    t_ll: float = 0.5
    t_l: float = 0.7
    t_full: float = 0.9
    enable_ll: bool = True
    enable_l: bool = True
    enable_full: bool = True
    BASE_THRESHOLD = 0.0

    def validate(self) -> None:
        if not (0.0 <= self.t_ll <= self.t_l <= self.t_full <= 1.0):
            raise ValidationError("thresholds: need 0 <= t_ll <= t_l <= t_full <= 1")


@dataclass
class GateMask:
    """synthesis.hpp:32-39"""
    width: int = 0
    height: int = 0
    on: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint8))

    def at(self, x: int, y: int) -> bool:
        return bool(self.on[y, x])

    def count(self) -> int:
        return int(np.count_nonzero(self.on))


@dataclass
class GridCell:
    x: int = 0
    y: int = 0


@dataclass
class ProgressiveResult:
    """synthesis.hpp:43-54"""
    base_lll: np.ndarray = None
    after_ll: np.ndarray = None
    after_l: np.ndarray = None
    after_full: np.ndarray = None
    mask_ll: GateMask = None
    mask_l: GateMask = None
    mask_full: GateMask = None
    ops: OpCounter = field(default_factory=OpCounter)

    def stage(self, index: int) -> np.ndarray:
        if index not in (0, 1, 2, 3):
            raise ValidationError("ProgressiveResult: stage index out of range")
        return [self.base_lll, self.after_ll, self.after_l, self.after_full][index]


DevicePlane = stages.DevicePlane  # a device-resident ComplexField

_scratch: dict = {}


def _scratch_plane(n: int) -> "stages.DevicePlane":
    """Per-size device plane for calls on host (numpy) planes: the
    contribution is formed on the device, then added on the host."""
    p = _scratch.get(n)
    if p is None:
        p = _scratch[n] = stages.DevicePlane(n)
    return p.zero()


def _plane_matches(plane, lut: FringeLut, where: str) -> int:
    n = lut.scene().plane_size()
    shape = (plane.n, plane.n) if isinstance(plane, stages.DevicePlane) else plane.shape
    if shape != (n, n):
        raise ValidationError(f"{where}: plane size does not match the LUT scene")
    return n


def _add_contribution(plane: np.ndarray, contrib: np.ndarray) -> None:
    plane += contrib.astype(plane.dtype, copy=False)


def apply_block(plane, lut: FringeLut, cell: GridCell, weight: complex,
                counter: OpCounter, level: OpLevel) -> None:
    """synthesis.cpp:149-160: plane += weight * crop(S_B at cell * B), in place,
    with the caller's LUT samples. `plane` is a numpy ComplexField (the
    contribution is added on the host) or a DevicePlane (stays on the device)."""
    n = _plane_matches(plane, lut, "apply_block")
    b = lut.block_size()
    cells = n // b
    if cell.x < 0 or cell.y < 0 or cell.x >= cells or cell.y >= cells:
        raise ValidationError(f"apply_block: cell ({cell.x},{cell.y}) out of range")
    w = complex(weight)
    idx = [cell.y * cells + cell.x]
    target = plane if isinstance(plane, stages.DevicePlane) else _scratch_plane(n)
    lut.device().apply_blocks(target, idx, [w.real], [w.imag] if w.imag != 0.0 else None)
    if target is not plane:
        _add_contribution(plane, target.download(np.complex128))
    counter.add(level, 1)


def synthesize_base(pyramid: HaarPyramid, saliency: SaliencyPyramid, luts: LutSet,
                    counter: OpCounter, workers: int = 1) -> np.ndarray:
    """synthesis.cpp:162-169 / 77-88: the caller's B = 8 LUT on every
    approximation cell."""
    if saliency.full_size() != pyramid.original_size:
        raise ValidationError("synthesize_base: saliency and pyramid sizes differ")
    block = pyramid.original_size // pyramid.approx.shape[0]
    lut = luts.of(block)
    n = lut.scene().plane_size()
    m = pyramid.approx.shape[0]
    if m * block != n:
        raise ValidationError("synthesize_base: approximation grid does not tile the plane")
    plane = _scratch_plane(n)
    ops = lut.device().apply_blocks(plane, np.arange(m * m), pyramid.approx.ravel())
    counter.add(OpLevel.BASE_LLL, ops)
    return plane.download(np.complex128)


def refine(plane, detail_h, detail_v, detail_d, saliency_finer, lut: FringeLut,
           threshold: float, counter: OpCounter, level: OpLevel, mask: GateMask | None = None,
           workers: int = 1) -> None:
    """synthesis.cpp:171-178 + 90-123: residual, strict '>' gate, the caller's
    block LUT; numpy plane (host add) or DevicePlane (on the device)."""
    n = _plane_matches(plane, lut, "refine")
    h, v, d = (np.asarray(a, np.float64) for a in (detail_h, detail_v, detail_d))
    if not (h.shape == v.shape == d.shape):
        raise ValidationError("expand_residual: detail subbands differ in size")
    m = h.shape[0]
    sal = np.asarray(saliency_finer, np.float64)
    if sal.shape != (2 * m, 2 * m):
        raise ValidationError("refine: saliency level does not match the residual resolution")
    if 2 * m * lut.block_size() != n:
        raise ValidationError("refine: LUT block size does not match the residual level")
    target = plane if isinstance(plane, stages.DevicePlane) else _scratch_plane(n)
    on, ops = lut.device().refine(target, h, v, d, sal, threshold)
    if target is not plane:
        _add_contribution(plane, target.download(np.complex128))
    counter.add(level, ops)
    if mask is not None:
        mask.width = mask.height = 2 * m
        mask.on = on


def _job(n_obj: int, scene: SceneParams, plan: RefinementPlan, method: str,
         obj_dtype: str = "f64") -> HologramJob:
    return HologramJob(JobSpec(object_size=n_obj, plane_size=scene.plane_size(),
                               layers=[scene.layer()], t_ll=plan.t_ll, t_l=plan.t_l,
                               t_full=plan.t_full, enable_ll=plan.enable_ll,
                               enable_l=plan.enable_l, enable_full=plan.enable_full,
                               method=method, obj_dtype=obj_dtype, sal_dtype="f64"))


def random_phase_field(amplitude: np.ndarray, seed: int) -> np.ndarray:
    """synthesis.cpp:288-296: polar(amplitude, U[0, 2pi)) from mt19937_64(seed),
    drawn on the host by the library with the reference's engine (bit-identical)."""
    return stages.random_phase_field(amplitude, seed)


def synthesize_progressive(object_: np.ndarray, saliency: np.ndarray, scene: SceneParams,
                           plan: RefinementPlan, luts: LutSet, workers: int = 1,
                           random_phase_seed: int | None = None,
                           method: str = "lut") -> ProgressiveResult:
    """synthesis.cpp:180-253. method "lut" (the reference's algorithm), "direct"
    or "fft": the same four stage snapshots from each."""
    plan.validate()
    n = scene.plane_size()
    if n < 8:
        raise ValidationError("synthesize_progressive: plane_size must be >= 8")
    obj = np.asarray(object_, np.float64)
    sal = np.asarray(saliency, np.float64)
    if obj.shape != (n, n):
        raise ValidationError("synthesize_progressive: object size does not match the scene")
    if sal.shape != obj.shape:
        raise ValidationError("synthesize_progressive: saliency size does not match the object")
    _require_finite(obj, "object")
    for b in LUT_BLOCK_SIZES:
        if not luts.has(b):
            raise ValidationError(f"synthesize_progressive: missing LUT for block size {b}")
    if not (luts.of(1).scene() == scene):
        raise ValidationError("synthesize_progressive: LUTs built for a different scene")
    # random initial phase (synthesis.cpp:205-214): a complex object, analysed
    # and synthesised part by part on the device (WCGH_C128 job)
    src = obj if random_phase_seed is None else random_phase_field(obj, random_phase_seed)
    job = _job(n, scene, plan, method, "f64" if random_phase_seed is None else "c128")
    try:
        if method == "lut":  # the caller's LutSet (synthesis.cpp:230-250 reads luts.of(B))
            for b in LUT_BLOCK_SIZES:
                job.use_lut(0, luts.of(b).device())
        job(np.ascontiguousarray(src), np.ascontiguousarray(sal))
        st = job.stats()
        snaps = job.download_stages()
    finally:
        job.close()
    an = stages.analyze(obj, sal, t=(plan.t_ll, plan.t_l, plan.t_full),
                        en=(int(plan.enable_ll), int(plan.enable_l), int(plan.enable_full)),
                        want_points=False, want_cells=False)
    q2, h2 = n * n // 16, n * n // 4
    masks = an["masks"]
    r = ProgressiveResult()
    r.mask_ll = GateMask(n // 4, n // 4, masks[:q2].reshape(n // 4, n // 4))
    r.mask_l = GateMask(n // 2, n // 2, masks[q2:q2 + h2].reshape(n // 2, n // 2))
    r.mask_full = GateMask(n, n, masks[q2 + h2:].reshape(n, n))
    for lev, v in zip(OpLevel, st["ops"]):
        r.ops.add(lev, v)
    r.base_lll, r.after_ll, r.after_l, r.after_full = (s.astype(np.complex128) for s in snaps)
    return r


def synthesize_pointwise_oracle(object_: np.ndarray, scene: SceneParams, counter: OpCounter,
                                unit_lut: FringeLut, workers: int = 1,
                                random_phase_seed: int | None = None) -> np.ndarray:
    """synthesis.cpp:255-286: the 1x1 LUT applied at every object pixel."""
    n = scene.plane_size()
    obj = np.asarray(object_, np.float64)
    if obj.shape != (n, n):
        raise ValidationError("pointwise oracle: object size does not match the scene")
    if unit_lut.block_size() != 1:
        raise ValidationError("pointwise oracle: needs the 1x1 LUT")
    if not (unit_lut.scene() == scene):
        raise ValidationError("pointwise oracle: LUT built for a different scene")
    _require_finite(obj, "object")
    plane = _scratch_plane(n)
    cells = np.arange(n * n)
    if random_phase_seed is None:
        ops = unit_lut.device().apply_blocks(plane, cells, obj.ravel())
    else:
        # complex amplitudes (synthesis.cpp:269-284): plane += (re + i im) S_1;
        # one operator per cell
        rotated = random_phase_field(obj, random_phase_seed)
        ops = unit_lut.device().apply_blocks(plane, cells, rotated.real.ravel(),
                                             rotated.imag.ravel())
    counter.add(OpLevel.POINTWISE_ORACLE, ops)
    return plane.download(np.complex128)


# ---- fft.hpp / angular_spectrum.hpp / metrics.hpp (validation, on the device) ----

STAGE_NAMES = ["base_LLL", "after_LL", "after_L", "after_full"]  # synthesis.hpp:56-57


def _field(field_: np.ndarray, what: str) -> np.ndarray:
    f = np.asarray(field_)
    if f.ndim != 2:
        raise ValidationError(f"{what}: field must be 2-D")
    return f


def fft_2d(field_: np.ndarray, inverse: bool) -> np.ndarray:
    """fft.cpp:45-68: 2-D DFT (inverse scaled by 1/n^2); square power-of-two side."""
    f = _field(field_, "fft_2d")
    if f.shape[0] != f.shape[1]:
        raise ValidationError("fft_2d: field must be square")
    if not is_power_of_two(f.shape[0]):
        raise ValidationError("fft_2d: side must be a power of two")
    return stages.fft_2d(f, inverse)


@dataclass
class PropagationKernel:
    """angular_spectrum.hpp:11-15"""
    scene: SceneParams
    z_signed: float
    transfer: np.ndarray


def build_kernel(scene: SceneParams, z_signed: float) -> PropagationKernel:
    """angular_spectrum.cpp:11-33"""
    if z_signed == 0.0:
        raise ValidationError("build_kernel: |z| must be positive")
    t = stages.propagation_kernel(scene.layer(), scene.plane_size(), z_signed)
    return PropagationKernel(scene, float(z_signed), t)


def propagate(field_: np.ndarray, kernel: PropagationKernel) -> np.ndarray:
    """angular_spectrum.cpp:35-45: IDFT(DFT(field) * transfer). The device
    evaluates the transfer function of (kernel.scene, kernel.z_signed) on the
    fly, i.e. kernel.transfer as build_kernel made it."""
    f = _field(field_, "propagate")
    if f.shape != kernel.transfer.shape:
        raise ValidationError("propagate: field size does not match kernel")
    return stages.propagate(f, kernel.scene.layer(), kernel.z_signed)


def reconstruct(hologram: np.ndarray, scene: SceneParams, intensity: bool = False) -> np.ndarray:
    """angular_spectrum.cpp:47-61"""
    h = _field(hologram, "reconstruct")
    n = scene.plane_size()
    if h.shape != (n, n):
        raise ValidationError("reconstruct: hologram size does not match scene")
    return stages.reconstruct(h, scene.layer(), intensity)


def ssim(a: np.ndarray, b: np.ndarray, window: int, k1: float, k2: float,
         dynamic_range: float) -> float:
    """metrics.cpp:49-85"""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValidationError("ssim: image sizes differ")
    if window <= 0 or window > min(a.shape):
        raise ValidationError("ssim: window must fit inside the images")
    if not dynamic_range > 0.0:
        raise ValidationError("ssim: dynamic range must be positive")
    return stages.ssim(a, b, window, k1, k2, dynamic_range)


@dataclass
class StageMetrics:
    """metrics.hpp:17-22"""
    name: str = ""
    ssim: float = 0.0
    ops: int = 0
    ops_cumulative: int = 0


@dataclass
class MetricsReport:
    """metrics.hpp:26-37"""
    stages: list = field(default_factory=list)
    pointwise_ops: int = 0
    window: int = 8
    k1: float = 0.01
    k2: float = 0.03
    dynamic_range: float = 1.0
    intensity: bool = False


def build_report(result: ProgressiveResult, oracle_recon: np.ndarray, scene: SceneParams,
                 intensity: bool = False) -> MetricsReport:
    """metrics.cpp:87-112: per-stage SSIM of the reconstructions against the
    oracle reconstruction, dynamic range = the oracle's value range."""
    report = MetricsReport(intensity=intensity)
    report.pointwise_ops = scene.plane_size() * scene.plane_size()
    lo, hi = float(np.min(oracle_recon)), float(np.max(oracle_recon))
    report.dynamic_range = hi - lo if hi - lo > 0.0 else 1.0
    cumulative = 0
    for s in range(4):
        recon = reconstruct(result.stage(s), scene, intensity)
        m = StageMetrics(name=STAGE_NAMES[s])
        m.ssim = ssim(recon, oracle_recon, report.window, report.k1, report.k2,
                      report.dynamic_range)
        m.ops = result.ops.get(STAGE_OP_LEVELS[s])
        cumulative += m.ops
        m.ops_cumulative = cumulative
        report.stages.append(m)
    return report
