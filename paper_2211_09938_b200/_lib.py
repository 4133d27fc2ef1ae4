"""ctypes binding of libwcgh.so (include/wcgh.h).

The product path: every call goes to the sm_100a kernels. There is no CPU
fallback — if the library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libwcgh.so"
# WCGH_CHECKED=1 loads the checked build (same sources, -DWCGH_CHECKED: device
# bounds checks + poisoned scratch; test use only, built by build(checked=True))
if os.environ.get("WCGH_CHECKED") == "1":
    LIB_PATH = LIB_PATH.with_name("libwcgh_checked.so")

WCGH_OK, WCGH_EVALIDATION, WCGH_ERUNTIME = 0, 1, 2
U8, F32, F64, C128 = 0, 1, 2, 3
METHOD_DIRECT, METHOD_LUT, METHOD_FFT = 0, 1, 2
PHASE_FIXED, PHASE_FP64 = 0, 1
OP_LEVELS = 5


class Layer(C.Structure):
    _fields_ = [("wavelength", C.c_double), ("pitch", C.c_double), ("z", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("t_ll", C.c_double), ("t_l", C.c_double), ("t_full", C.c_double),
                ("enable_ll", C.c_int), ("enable_l", C.c_int), ("enable_full", C.c_int)]


class Point(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("a", C.c_float), ("layer", C.c_int32)]


POINT_DTYPE = np.dtype([("x", np.int32), ("y", np.int32), ("a", np.float32), ("layer", np.int32)])


class Desc(C.Structure):
    _fields_ = [("object_size", C.c_int), ("plane_size", C.c_int), ("n_layers", C.c_int),
                ("layers", C.POINTER(Layer)), ("plan", Plan), ("method", C.c_int),
                ("phase_mode", C.c_int), ("row0", C.c_int), ("rows", C.c_int),
                ("obj_dtype", C.c_int), ("obj_scale", C.c_double), ("sal_dtype", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("ops", C.c_uint64 * OP_LEVELS), ("n_points", C.c_int64), ("updates", C.c_double),
                ("ms_analysis", C.c_float), ("ms_synthesis", C.c_float), ("ms_reduce", C.c_float),
                ("ms_total", C.c_float), ("synth_launches", C.c_int), ("total_launches", C.c_int)]


class Analysis(C.Structure):
    _fields_ = [("pyramid", C.POINTER(C.c_double)), ("sal_pyr", C.POINTER(C.c_double)),
                ("masks", C.POINTER(C.c_uint8)), ("a_eff", C.POINTER(C.c_float)),
                ("cells", C.POINTER(C.c_uint32)), ("cell_counts", C.c_int64 * 3),
                ("points", C.POINTER(Point)), ("n_points", C.c_int64),
                ("ops", C.c_uint64 * OP_LEVELS)]


# (name, restype, argtypes) for every symbol include/wcgh.h declares.
_VP = C.c_void_p
_SIGS = [
    ("wcgh_abi_version", C.c_int, []),
    ("wcgh_create", C.c_int, [C.c_int, C.POINTER(_VP)]),
    ("wcgh_destroy", None, [_VP]),
    ("wcgh_last_error", C.c_char_p, [_VP]),
    ("wcgh_set_stream", C.c_int, [_VP, _VP]),
    ("wcgh_device_info", C.c_int, [_VP, C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    ("wcgh_haar_analyze", C.c_int, [_VP, _VP, C.c_int, C.c_double, C.c_int, C.c_int, _VP]),
    ("wcgh_expand_residual", C.c_int, [_VP, _VP, _VP, _VP, C.c_int, _VP]),
    ("wcgh_quantize_saliency", C.c_int, [_VP, _VP, C.c_int, C.c_int, _VP]),
    ("wcgh_analyze", C.c_int, [_VP, _VP, C.c_int, C.c_double, _VP, C.c_int, C.c_int,
                               C.POINTER(Plan), C.c_int, C.c_int, C.POINTER(Analysis)]),
    ("wcgh_synth_points", C.c_int, [_VP, _VP, C.c_int64, C.POINTER(Layer), C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_int, _VP]),
    ("wcgh_build_block_lut", C.c_int, [_VP, C.POINTER(Layer), C.c_int, C.c_int, _VP]),
    ("wcgh_apply_blocks", C.c_int, [_VP, C.POINTER(Layer), C.c_int, C.c_int, _VP, _VP,
                                    C.c_int64, _VP, C.POINTER(C.c_uint64)]),
    ("wcgh_refine", C.c_int, [_VP, C.POINTER(Layer), C.c_int, _VP, _VP, _VP, C.c_int, _VP,
                              C.c_double, _VP, _VP, C.POINTER(C.c_uint64)]),
    ("wcgh_job_create", C.c_int, [_VP, C.POINTER(Desc), C.POINTER(_VP)]),
    ("wcgh_job_destroy", None, [_VP]),
    ("wcgh_job_upload", C.c_int, [_VP, _VP, _VP]),
    ("wcgh_job_upload_dev", C.c_int, [_VP, _VP, _VP]),
    ("wcgh_job_run", C.c_int, [_VP]),
    ("wcgh_job_analyze", C.c_int, [_VP]),
    ("wcgh_job_download", C.c_int, [_VP, _VP]),
    ("wcgh_job_set_peer_planes", C.c_int, [_VP, C.POINTER(_VP), C.c_int]),
    ("wcgh_ipc_alloc_plane", C.c_int, [C.c_int, C.c_int, C.POINTER(_VP), C.c_char_p]),
    ("wcgh_ipc_open_plane", C.c_int, [C.c_int, C.c_char_p, C.POINTER(_VP)]),
    ("wcgh_ipc_close_plane", C.c_int, [_VP]),
    ("wcgh_ipc_free_plane", C.c_int, [_VP]),
    ("wcgh_job_download_a_eff", C.c_int, [_VP, _VP]),
    ("wcgh_job_download_points", C.c_int, [_VP, _VP, C.c_int64, C.POINTER(C.c_int64)]),
    ("wcgh_job_download_a_eff_im", C.c_int, [_VP, _VP]),
    ("wcgh_job_download_points_im", C.c_int, [_VP, _VP, C.c_int64]),
    ("wcgh_random_phase_field", C.c_int, [_VP, C.c_int, C.c_int, C.c_uint64, _VP]),
    ("wcgh_job_download_stages", C.c_int, [_VP, _VP]),
    ("wcgh_job_plane_dev", _VP, [_VP]),
    ("wcgh_job_stats", C.c_int, [_VP, C.POINTER(Stats)]),
    ("wcgh_job_direct_form", C.c_int, [_VP, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("wcgh_write_cgh1", C.c_int, [C.c_char_p, _VP, C.c_int, C.POINTER(Layer)]),
    ("wcgh_read_cgh1", C.c_int, [C.c_char_p, _VP, C.c_int64, C.POINTER(C.c_int), C.POINTER(Layer)]),
    ("wcgh_job_write_cgh1", C.c_int, [_VP, C.c_char_p, C.c_int]),
    ("wcgh_fft_2d", C.c_int, [_VP, _VP, C.c_int, C.c_int, _VP]),
    ("wcgh_propagation_kernel", C.c_int, [_VP, C.POINTER(Layer), C.c_int, C.c_double, _VP]),
    ("wcgh_propagate", C.c_int, [_VP, _VP, C.c_int, C.c_int, C.POINTER(Layer), C.c_double, _VP]),
    ("wcgh_reconstruct", C.c_int, [_VP, _VP, C.c_int, C.c_int, C.POINTER(Layer), C.c_int, _VP]),
    ("wcgh_job_reconstruct", C.c_int, [_VP, C.POINTER(Layer), C.c_int, _VP]),
    ("wcgh_ssim", C.c_int, [_VP, _VP, _VP, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                            C.c_double, C.POINTER(C.c_double)]),
    ("wcgh_write_cghl", C.c_int, [C.c_char_p, _VP, C.c_int, C.c_int, C.POINTER(Layer)]),
    ("wcgh_read_cghl", C.c_int, [C.c_char_p, _VP, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(Layer)]),
    ("wcgh_job_load_lut", C.c_int, [_VP, C.c_int, C.c_int, _VP]),
    ("wcgh_job_use_lut", C.c_int, [_VP, C.c_int, _VP]),
    ("wcgh_haar_synthesize", C.c_int, [_VP, _VP, C.c_int, C.c_int, _VP]),
    ("wcgh_upsample_replicate", C.c_int, [_VP, _VP, C.c_int, C.c_int, C.c_int, _VP]),
    ("wcgh_point_fringe", C.c_int, [_VP, C.POINTER(Layer), C.c_int, C.c_int, _VP]),
    ("wcgh_lut_create", C.c_int, [_VP, C.POINTER(Layer), C.c_int, C.c_int, _VP, C.c_int,
                                  C.POINTER(_VP)]),
    ("wcgh_lut_destroy", None, [_VP]),
    ("wcgh_lut_download", C.c_int, [_VP, _VP]),
    ("wcgh_plane_create", C.c_int, [_VP, C.c_int, C.POINTER(_VP)]),
    ("wcgh_plane_destroy", None, [_VP]),
    ("wcgh_plane_zero", C.c_int, [_VP]),
    ("wcgh_plane_upload", C.c_int, [_VP, _VP, C.c_int]),
    ("wcgh_plane_download", C.c_int, [_VP, _VP, C.c_int]),
    ("wcgh_plane_dev", _VP, [_VP]),
    ("wcgh_lut_apply_blocks", C.c_int, [_VP, _VP, _VP, _VP, C.c_int64, _VP, C.POINTER(C.c_uint64)]),
    ("wcgh_lut_refine", C.c_int, [_VP, _VP, _VP, _VP, C.c_int, _VP, C.c_double, _VP, _VP,
                                  C.POINTER(C.c_uint64)]),
    ("wcgh_synthesize", C.c_int, [_VP, C.POINTER(Desc), _VP, _VP, _VP, C.POINTER(Stats)]),
    ("wcgh_synthesize_multi", C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(Desc), _VP, _VP, _VP,
                                        C.POINTER(Stats)]),
]
EXPORTED = [s[0] for s in _SIGS]

_lib = None


def load() -> C.CDLL:
    """Loads libwcgh.so (building it first if only the sources exist)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        from . import build as _build
        _build.build(checked=LIB_PATH.name == "libwcgh_checked.so")
    lib = C.CDLL(str(LIB_PATH))
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class ValidationError(ValueError):
    """The reference's ValidationError (errors.hpp:10-13)."""


class IoError(RuntimeError):
    """The reference's IoError class (errors.hpp:17-20): CUDA / runtime failures."""


def check(rc: int) -> None:
    if rc == WCGH_OK:
        return
    msg = load().wcgh_last_error(None).decode()
    if rc == WCGH_EVALIDATION:
        raise ValidationError(msg)
    raise IoError(msg)


def ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


class Context:
    """One context per GPU (one process per GPU)."""

    def __init__(self, device: int | None = None):
        lib = load()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        h = C.c_void_p()
        check(lib.wcgh_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self.lib = lib

    def close(self):
        if getattr(self, "h", None):
            self.lib.wcgh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        check(self.lib.wcgh_set_stream(self.h, C.c_void_p(stream_handle or 0)))

    def device_info(self):
        n = C.c_int()
        name = C.create_string_buffer(256)
        check(self.lib.wcgh_device_info(self.h, C.byref(n), name, 256))
        return n.value, name.value.decode()


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx
