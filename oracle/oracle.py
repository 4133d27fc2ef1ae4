"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.

Python access to
  * liboracle.so — this repo's plain-C fp64 restatement of the reference hot
    path (oracle.c; each function cites the reference file:line), and
  * _ref/libwavecgh_ref.so — the UNMODIFIED reference sources compiled here
    (Makefile) behind an extern "C" shim (ref_shim.cpp), when present.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libwavecgh_ref.so"

_orc = None
_ref = None

D = C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_oracle() -> Path:
    src = HERE / "oracle.c"
    if not ORC_LIB.exists() or ORC_LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "liboracle.so"], check=True, capture_output=True)
    return ORC_LIB


def build_ref() -> Path | None:
    if not Path("/root/reference/proj").exists():
        return REF_LIB if REF_LIB.exists() else None
    if not REF_LIB.exists() or REF_LIB.stat().st_mtime < (HERE / "ref_shim.cpp").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "ref"], check=True, capture_output=True)
    return REF_LIB


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        lib = C.CDLL(str(build_oracle()))
        V = C.c_void_p
        lib.orc_haar_analyze.argtypes = [V, C.c_int, C.c_int, V]
        lib.orc_expand_residual.argtypes = [V, V, V, C.c_int, V]
        lib.orc_upsample_replicate.argtypes = [V, C.c_int, C.c_int, V]
        lib.orc_quantize_saliency.argtypes = [V, C.c_int, V]
        lib.orc_analysis.argtypes = [V, V, C.c_int, V, V, V, V, V, V, V]
        lib.orc_compact.argtypes = [V, C.c_int, C.c_int, V, V, V]
        lib.orc_compact.restype = C.c_int64
        lib.orc_point_fringe.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, V]
        lib.orc_direct_pixels.argtypes = [V, V, V, V, C.c_int64, V, V, V, V, V, C.c_int64, V]
        lib.orc_build_block_lut.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, V]
        lib.orc_apply_block.argtypes = [V, C.c_int, V, C.c_int, C.c_int, C.c_double, C.c_double]
        lib.orc_synthesize_progressive.argtypes = [V, V, C.c_int, V, V, V, V, V, V, V]
        lib.orc_ssim.argtypes = [V, V, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        lib.orc_ssim.restype = C.c_double
        _orc = lib
    return _orc


def ref() -> C.CDLL | None:
    """The reference itself (None when it was never built here)."""
    global _ref
    if _ref is None:
        path = build_ref()
        if path is None or not Path(path).exists():
            return None
        lib = C.CDLL(str(path))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_lutset_build.restype = C.c_void_p
        lib.ref_lutset_build.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int]
        lib.ref_lutset_free.argtypes = [C.c_void_p]
        lib.ref_time_refine.argtypes = [C.c_void_p] + [C.c_void_p] * 3 + [C.c_int, C.c_void_p,
                                        C.c_double, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_time_progressive.argtypes = [C.c_void_p] * 5 + [C.c_int] + [C.c_void_p] * 3
        for name in ["ref_point_fringe", "ref_build_block_lut", "ref_apply_block",
                     "ref_synthesize_progressive", "ref_synthesize_pointwise_oracle",
                     "ref_pointwise_hologram_reference", "ref_reconstruct", "ref_ssim"]:
            getattr(lib, name).argtypes = None
        _ref = lib
    return _ref


def _ref_check(rc: int):
    if rc != 0:
        msg = ref().ref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


# ---- fp64 restatement (liboracle) -----------------------------------------

def pyr_len(n: int, levels: int = 3) -> int:
    t, s = 0, n
    for _ in range(levels):
        s //= 2
        t += 3 * s * s
    return t + s * s


def split_pyramid(flat: np.ndarray, n: int, levels: int = 3):
    """flat -> (approx, [(h, v, d) finest first])"""
    ma = n >> levels
    approx = flat[: ma * ma].reshape(ma, ma)
    off = ma * ma
    det = []
    for l in range(levels):
        m = n >> (l + 1)
        h = flat[off: off + m * m].reshape(m, m)
        v = flat[off + m * m: off + 2 * m * m].reshape(m, m)
        d = flat[off + 2 * m * m: off + 3 * m * m].reshape(m, m)
        det.append((h, v, d))
        off += 3 * m * m
    return approx, det


def haar_analyze(img: np.ndarray, levels: int = 3) -> np.ndarray:
    img = np.ascontiguousarray(img, np.float64)
    n = img.shape[0]
    out = np.empty(pyr_len(n, levels))
    if orc().orc_haar_analyze(_p(img), n, levels, _p(out)):
        raise ValueError("haar_analyze: bad dimensions")
    return out


def expand_residual(h, v, d) -> np.ndarray:
    h, v, d = (np.ascontiguousarray(a, np.float64) for a in (h, v, d))
    m = h.shape[0]
    out = np.empty((2 * m, 2 * m))
    orc().orc_expand_residual(_p(h), _p(v), _p(d), m, _p(out))
    return out


def quantize_saliency(sal: np.ndarray) -> np.ndarray:
    sal = np.ascontiguousarray(sal, np.float64)
    n = sal.shape[0]
    out = np.empty(n * n // 4 + n * n // 16 + n * n // 64)
    if orc().orc_quantize_saliency(_p(sal), n, _p(out)):
        raise ValueError("quantize_saliency: invalid map")
    return out


def analysis(obj: np.ndarray, sal: np.ndarray, t=(0.5, 0.7, 0.9), en=(1, 1, 1)) -> dict:
    obj = np.ascontiguousarray(obj, np.float64)
    sal = np.ascontiguousarray(sal, np.float64)
    n = obj.shape[0]
    n2 = n * n
    pyr = np.empty(pyr_len(n))
    sp = np.empty(n2 // 4 + n2 // 16 + n2 // 64)
    masks = np.empty(n2 // 16 + n2 // 4 + n2, np.uint8)
    a_eff = np.empty((n, n))
    ops = np.zeros(5, np.uint64)
    th = np.array(t, np.float64)
    ens = np.array(en, np.int32)
    if orc().orc_analysis(_p(obj), _p(sal), n, _p(th), _p(ens), _p(pyr), _p(sp), _p(masks),
                          _p(a_eff), _p(ops)):
        raise ValueError("analysis: validation error")
    return {"pyramid": pyr, "sal_pyr": sp, "masks": masks, "a_eff": a_eff, "ops": ops}


def compact(a_eff: np.ndarray, off: int = 0, layer: int = 0):
    a = np.ascontiguousarray(a_eff, np.float64)
    n = a.shape[0]
    cnt = orc().orc_compact(_p(a), n, off, None, None, None)
    xs = np.empty(cnt, np.int32)
    ys = np.empty(cnt, np.int32)
    amps = np.empty(cnt)
    orc().orc_compact(_p(a), n, off, _p(xs), _p(ys), _p(amps))
    return xs, ys, amps, np.full(cnt, layer, np.int32)


def direct_pixels(xs, ys, amps, layer, layers, px, py) -> np.ndarray:
    """Direct Eq.(1) fp64 at pixels (px[i], py[i]); layers = [(wl, pitch, z)]."""
    xs = np.ascontiguousarray(xs, np.int32)
    ys = np.ascontiguousarray(ys, np.int32)
    amps = np.ascontiguousarray(amps, np.float64)
    layer = np.ascontiguousarray(layer, np.int32)
    wl = np.array([l[0] for l in layers], np.float64)
    pt = np.array([l[1] for l in layers], np.float64)
    zz = np.array([l[2] for l in layers], np.float64)
    px = np.ascontiguousarray(px, np.int32)
    py = np.ascontiguousarray(py, np.int32)
    out = np.empty(len(px), np.complex128)
    orc().orc_direct_pixels(_p(xs), _p(ys), _p(amps), _p(layer), len(xs), _p(wl), _p(pt), _p(zz),
                            _p(px), _p(py), len(px), _p(out))
    return out


def build_block_lut(wl, pitch, z, n, block) -> np.ndarray:
    span = 2 * n - 1
    out = np.empty((span, span), np.complex128)
    if orc().orc_build_block_lut(wl, pitch, z, n, block, _p(out)):
        raise ValueError("build_block_lut: unsupported block size")
    return out


def synthesize_progressive(obj, sal, wl, pitch, z, t=(0.5, 0.7, 0.9), en=(1, 1, 1), luts=None):
    """LUT method in fp64 (synthesis.cpp:180-253), object == plane size."""
    obj = np.ascontiguousarray(obj, np.float64)
    sal = np.ascontiguousarray(sal, np.float64)
    n = obj.shape[0]
    if luts is None:
        luts = [build_block_lut(wl, pitch, z, n, b) for b in (1, 2, 4, 8)]
    ptrs = (C.c_void_p * 4)(*[l.ctypes.data for l in luts])
    planes = np.empty((4, n, n), np.complex128)
    masks = np.empty(n * n // 16 + n * n // 4 + n * n, np.uint8)
    ops = np.zeros(5, np.uint64)
    th = np.array(t, np.float64)
    ens = np.array(en, np.int32)
    if orc().orc_synthesize_progressive(_p(obj), _p(sal), n, _p(th), _p(ens), ptrs, _p(planes),
                                        None, _p(masks), _p(ops)):
        raise ValueError("synthesize_progressive: validation error")
    return planes, masks, ops


def ssim(a, b, window=8, k1=0.01, k2=0.03, dynamic_range=1.0) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    h, w = a.shape
    return float(orc().orc_ssim(_p(a), _p(b), w, h, window, k1, k2, dynamic_range))


def reconstruct(holo: np.ndarray, wl: float, pitch: float, z: float, intensity=False) -> np.ndarray:
    """Angular-spectrum back-propagation by -z (angular_spectrum.cpp:11-61)
    with numpy FFTs (the reference's radix-2 FFT differs only by rounding)."""
    n = holo.shape[0]
    df = 1.0 / (n * pitch)
    m = np.fft.fftfreq(n) * n
    fx = (m * df)[None, :]
    fy = (m * df)[:, None]
    s = 1.0 / (wl * wl) - fx * fx - fy * fy
    transfer = np.where(s >= 0.0, np.exp(1j * 2 * np.pi * (-z) * np.sqrt(np.maximum(s, 0.0))), 0.0)
    field = np.fft.ifft2(np.fft.fft2(np.asarray(holo, np.complex128)) * transfer)
    return np.abs(field) ** 2 if intensity else np.abs(field)


def max_rel_error(actual, reference) -> float:
    """tests/support/oracles.cpp:129-137"""
    a = np.asarray(actual, np.complex128)
    r = np.asarray(reference, np.complex128)
    mr = np.abs(r).max()
    md = np.abs(a - r).max()
    return float(md / mr) if mr > 0 else float(md)


def rel_l2(actual, reference) -> float:
    a = np.asarray(actual, np.complex128)
    r = np.asarray(reference, np.complex128)
    return float(np.linalg.norm(a - r) / np.linalg.norm(r))


def scene_points(objects: np.ndarray, saliency01: np.ndarray, plane_size: int,
                 t=(0.5, 0.7, 0.9), en=(1, 1, 1)):
    """Oracle point list of a layered scene: per layer A_eff (fp64) compacted
    in row-major order with the centring offset; concatenated layer-major."""
    L, n, _ = objects.shape
    off = (plane_size - n) // 2
    xs, ys, amps, lay, ops = [], [], [], [], np.zeros(5, np.uint64)
    for l in range(L):
        an = analysis(objects[l], saliency01[l], t, en)
        x, y, a, ll = compact(an["a_eff"], off, l)
        xs.append(x), ys.append(y), amps.append(a), lay.append(ll)
        ops += an["ops"]
    return (np.concatenate(xs), np.concatenate(ys), np.concatenate(amps), np.concatenate(lay),
            ops)


# ---- the reference itself (_ref) ------------------------------------------

def ref_available() -> bool:
    return ref() is not None


def ref_haar_analyze(img, levels=3):
    img = np.ascontiguousarray(img, np.float64)
    n = img.shape[0]
    out = np.empty(pyr_len(n, levels))
    _ref_check(ref().ref_haar_analyze(_p(img), C.c_int(n), C.c_int(levels), _p(out)))
    return out


def ref_quantize_saliency(sal):
    sal = np.ascontiguousarray(sal, np.float64)
    n = sal.shape[0]
    out = np.empty(n * n // 4 + n * n // 16 + n * n // 64)
    _ref_check(ref().ref_quantize_saliency(_p(sal), C.c_int(n), _p(out)))
    return out


def ref_expand_residual(h, v, d):
    h, v, d = (np.ascontiguousarray(a, np.float64) for a in (h, v, d))
    m = h.shape[0]
    out = np.empty((2 * m, 2 * m))
    _ref_check(ref().ref_expand_residual(_p(h), _p(v), _p(d), C.c_int(m), _p(out)))
    return out


def ref_point_fringe(wl, pitch, z, n, dx, dy):
    out = np.empty(2)
    _ref_check(ref().ref_point_fringe(C.c_double(wl), C.c_double(pitch), C.c_double(z), C.c_int(n),
                                      C.c_int(dx), C.c_int(dy), _p(out)))
    return complex(out[0], out[1])


def ref_build_block_lut(wl, pitch, z, n, block, workers=0):
    span = 2 * n - 1
    out = np.empty((span, span), np.complex128)
    _ref_check(ref().ref_build_block_lut(C.c_double(wl), C.c_double(pitch), C.c_double(z),
                                         C.c_int(n), C.c_int(block), C.c_int(workers), _p(out)))
    return out


def ref_apply_block_lut(plane, support, wl, pitch, z, block, cx, cy, w):
    """apply_block (synthesis.cpp:149-160) of the reference with the CALLER's
    LUT samples (FringeLut(scene, block, support)); plane complex128, returned
    updated, plus the op count."""
    p = np.ascontiguousarray(plane, np.complex128).copy()
    sup = np.ascontiguousarray(support, np.complex128)
    n = p.shape[0]
    ops = C.c_uint64()
    w = complex(w)
    _ref_check(ref().ref_apply_block_lut(C.c_double(wl), C.c_double(pitch), C.c_double(z), C.c_int(n),
                                         C.c_int(block), _p(sup), C.c_int(cx), C.c_int(cy),
                                         C.c_double(w.real), C.c_double(w.imag), _p(p), C.byref(ops)))
    return p, int(ops.value)


def ref_synthesize_progressive_luts(obj, sal, wl, pitch, z, supports, t=(0.5, 0.7, 0.9),
                                    en=(1, 1, 1)):
    """synthesize_progressive with a caller LutSet; supports = {1: S1, 2: S2,
    4: S4, 8: S8}, (2n-1)^2 complex128 each. Returns (planes[4], ops[5])."""
    obj = np.ascontiguousarray(obj, np.float64)
    sal = np.ascontiguousarray(sal, np.float64)
    n = obj.shape[0]
    sups = [np.ascontiguousarray(supports[b], np.complex128) for b in (1, 2, 4, 8)]
    arr = (C.c_void_p * 4)(*[a.ctypes.data for a in sups])
    planes = np.empty((4, n, n), np.complex128)
    ops = np.zeros(5, np.uint64)
    th = np.array(t, np.float64)
    ens = np.array(en, np.int32)
    _ref_check(ref().ref_synthesize_progressive_luts(
        _p(obj), _p(sal), C.c_int(n), C.c_double(wl), C.c_double(pitch), C.c_double(z), _p(th),
        _p(ens), arr, _p(planes), _p(ops)))
    return planes, ops


def ref_synthesize_progressive(obj, sal, wl, pitch, z, t=(0.5, 0.7, 0.9), en=(1, 1, 1),
                               workers=0, seed=None):
    obj = np.ascontiguousarray(obj, np.float64)
    sal = np.ascontiguousarray(sal, np.float64)
    n = obj.shape[0]
    planes = np.empty((4, n, n), np.complex128)
    masks = np.empty(n * n // 16 + n * n // 4 + n * n, np.uint8)
    ops = np.zeros(5, np.uint64)
    th = np.array(t, np.float64)
    ens = np.array(en, np.int32)
    _ref_check(ref().ref_synthesize_progressive(
        _p(obj), _p(sal), C.c_int(n), C.c_double(wl), C.c_double(pitch), C.c_double(z), _p(th),
        _p(ens), C.c_int(workers), C.c_int(seed is not None), C.c_uint64(seed or 0), _p(planes),
        _p(masks), _p(ops)))
    return planes, masks, ops


def ref_pointwise_oracle(obj, wl, pitch, z, workers=0, seed=None):
    obj = np.ascontiguousarray(obj, np.float64)
    n = obj.shape[0]
    out = np.empty((n, n), np.complex128)
    ops = C.c_uint64()
    _ref_check(ref().ref_synthesize_pointwise_oracle(_p(obj), C.c_int(n), C.c_double(wl),
                                                     C.c_double(pitch), C.c_double(z),
                                                     C.c_int(workers), C.c_int(seed is not None),
                                                     C.c_uint64(seed or 0), _p(out), C.byref(ops)))
    return out, int(ops.value)


def ref_pointwise_hologram_reference(amp, wl, pitch, z):
    """amp real (float64) or complex (complex128)."""
    amp = np.asarray(amp)
    n = amp.shape[0]
    out = np.empty((n, n), np.complex128)
    re = np.ascontiguousarray(amp.real, np.float64)
    im = np.ascontiguousarray(amp.imag, np.float64) if np.iscomplexobj(amp) else None
    _ref_check(ref().ref_pointwise_hologram_reference(_p(re), _p(im) if im is not None else None,
                                                      C.c_int(n), C.c_double(wl),
                                                      C.c_double(pitch), C.c_double(z), _p(out)))
    return out


def ref_random_phase_field(amp, seed):
    """random_phase_field (synthesis.cpp:288-296) of the reference itself."""
    amp = np.ascontiguousarray(amp, np.float64)
    n = amp.shape[0]
    out = np.empty((n, n), np.complex128)
    _ref_check(ref().ref_random_phase_field(_p(amp), C.c_int(n), C.c_uint64(seed), _p(out)))
    return out


def ref_random_image(w, h, seed):
    out = np.empty((h, w))
    _ref_check(ref().ref_random_image(C.c_int(w), C.c_int(h), C.c_uint64(seed), _p(out)))
    return out


def ref_lut_cache_store(path, wl, pitch, z, n, block):
    _ref_check(ref().ref_lut_cache_store(str(path).encode(), C.c_double(wl), C.c_double(pitch),
                                         C.c_double(z), C.c_int(n), C.c_int(block)))


def ref_reconstruct(holo, wl, pitch, z, intensity=False):
    holo = np.ascontiguousarray(holo, np.complex128)
    n = holo.shape[0]
    out = np.empty((n, n))
    _ref_check(ref().ref_reconstruct(_p(holo), C.c_int(n), C.c_double(wl), C.c_double(pitch),
                                     C.c_double(z), C.c_int(int(intensity)), _p(out)))
    return out


def ref_ssim(a, b, window=8, k1=0.01, k2=0.03, dynamic_range=1.0):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    out = C.c_double()
    _ref_check(ref().ref_ssim(_p(a), _p(b), C.c_int(a.shape[0]), C.c_int(window), C.c_double(k1),
                              C.c_double(k2), C.c_double(dynamic_range), C.byref(out)))
    return out.value


def ref_default_workers() -> int:
    return int(ref().ref_default_worker_count())


# ---- full-plane fp64 oracle by FFT (for the 4096^2 configs) -------------------

def fft_hologram(a_eff_layers, layers, plane_size: int, rows: tuple[int, int] | None = None):
    """fp64 H = sum_layers A_eff (*) F on a 2Nh circular grid (no wrap reaches
    the output window since 2Nh >= Nh + No - 1), F the exact point fringe
    (fringe_lut.cpp:27-32). Mathematically the direct sum of
    tests/support/oracles.cpp:12-36; pinned against it and against the
    reference's goldens in tests/test_oracle_pins.py. Multi-threaded scipy FFT."""
    import scipy.fft as sf

    a = np.asarray(a_eff_layers, np.float64)
    if a.ndim == 2:
        a = a[None]
    nl, no, _ = a.shape
    n = plane_size
    L = 2 * n
    off = (n - no) // 2
    c = np.arange(L)
    d = np.where(c < n, c, c - L).astype(np.float64)
    acc = None
    for l in range(nl):
        wl, pitch, z = layers[l]
        k = 2.0 * np.pi / wl
        px = (d * pitch)[None, :]
        py = (d * pitch)[:, None]
        r = np.sqrt(px * px + py * py + z * z)
        f = np.exp(1j * k * r) / r
        f[n, :] = 0.0
        f[:, n] = 0.0
        g = np.zeros((L, L), np.complex128)
        g[off:off + no, off:off + no] = a[l]
        spec = sf.fft2(g, workers=-1) * sf.fft2(f, workers=-1)
        acc = spec if acc is None else acc + spec
        del f, g
    h = sf.ifft2(acc, workers=-1)
    r0, r1 = (0, n) if rows is None else rows
    return np.ascontiguousarray(h[r0:r1, :n])


def scene_a_eff(objects: np.ndarray, saliency01: np.ndarray, t=(0.5, 0.7, 0.9), en=(1, 1, 1)):
    """Per-layer fp64 A_eff of a layered scene (orc_analysis)."""
    return np.stack([analysis(objects[l], saliency01[l], t, en)["a_eff"]
                     for l in range(objects.shape[0])])
