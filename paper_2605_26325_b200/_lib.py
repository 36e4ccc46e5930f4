"""ctypes binding of libdare_b200.so (the C ABI declared in include/dare_b200.h).

The product path has no CPU fallback: if the shared library is missing or a
call fails, a DareError/RuntimeError is raised.  ctypes releases the GIL for
the duration of every foreign call, so concurrent reslices from Python
threads run concurrently on the device (each thread gets its own stream).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import InvalidArgumentError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdare_b200.so")
if os.environ.get("DARE_CHECKED") == "1":  # bounds-asserting build (build.py --checked), for test runs
    LIB_PATH = os.path.join(_HERE, "libdare_b200_checked.so")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_sz = ctypes.c_size_t
c_vp = ctypes.c_void_p
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_f64 = ctypes.POINTER(ctypes.c_double)
P_f32 = ctypes.POINTER(ctypes.c_float)
P_u8 = ctypes.POINTER(ctypes.c_uint8)

DARE_OK = 0
DARE_ERR_INVALID = -1
DARE_ERR_CUDA = -2
DARE_ERR_NOMEM = -3
DARE_ERR_LIMIT = -4


class ResliceCfg(ctypes.Structure):
    _fields_ = [
        ("radius", c_f64), ("cos_normal", c_f64), ("cos_inplane", c_f64),
        ("k_normal", c_f64), ("k_inplane", c_f64), ("k_dist", c_f64),
        ("unassigned", c_i32), ("schedule", c_i32), ("exact", c_i32), ("_pad", c_i32),
    ]


class VolumeInfo(ctypes.Structure):
    _fields_ = [
        ("device", c_i32), ("_pad", c_i32),
        ("origin", c_f64 * 3), ("voxel_size", c_f64), ("dims", c_i64 * 3),
        ("n_samples", c_i64), ("n_orientations", c_i64), ("rejected_out_of_bounds", c_i64),
        ("d_cell_offsets", c_vp), ("d_records", c_vp), ("d_orientations", c_vp),
        ("d_bins", c_vp), ("d_perm", c_vp),
        ("device_bytes", c_sz),
    ]


class ScalarInfo(ctypes.Structure):
    _fields_ = [
        ("device", c_i32), ("_pad", c_i32),
        ("origin", c_f64 * 3), ("voxel_size", c_f64), ("dims", c_i64 * 3),
        ("d_values", c_vp), ("d_flags", c_vp), ("d_counts", c_vp),
    ]


WRITE_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, c_sz)

# name -> argtypes (restype is always c_int except dare_last_error)
_SIGNATURES = {
    "dare_version": [],
    "dare_get_device_count": [P_i32],
    "dare_set_device": [c_i32],
    "dare_synchronize": [],
    "dare_host_alloc": [c_sz, ctypes.POINTER(c_vp)],
    "dare_host_free": [c_vp],
    "dare_device_alloc": [c_sz, ctypes.POINTER(c_vp)],
    "dare_device_free": [c_vp],
    "dare_memcpy": [c_vp, c_vp, c_sz, c_vp],
    "dare_stream_sync": [c_vp],
    "dare_last_device_ms": [P_f64],
    "dare_init": [c_i32],
    "dare_trim": [c_sz],
    "dare_reconstruct": [c_vp, c_i64, c_i32, c_i32, c_i32, P_i32, c_i64, P_f64, P_f32, c_f64,
                         c_f64, P_u8, P_f64, c_f64, P_i64, ctypes.POINTER(c_vp), P_i64],
    "dare_volume_seal": [P_f64, c_f64, P_i64, c_i64, P_f32, P_f32, P_u8, ctypes.POINTER(c_vp)],
    "dare_volume_upload": [P_f64, c_f64, P_i64, P_i64, P_i64, c_i64, P_f32, P_f32, P_u8,
                           ctypes.POINTER(c_vp)],
    "dare_volume_download": [c_vp, P_i64, P_i64, P_f32, P_f32, P_u8],
    "dare_volume_get_info": [c_vp, ctypes.POINTER(VolumeInfo)],
    "dare_volume_save_stream": [c_vp, WRITE_FN, c_vp, c_sz],
    "dare_volume_destroy": [c_vp],
    "dare_frame_poses": [c_i64, P_f64, P_f64, P_f64, P_f64, c_i32, c_i32, c_f64, c_f64, P_f64, P_f64, P_f64,
                         P_f32, P_f64, P_f64, ctypes.POINTER(c_i32), ctypes.POINTER(c_i64),
                         ctypes.POINTER(c_f64)],
    "dare_interpolate_poses": [c_i64, P_f64, P_i64, P_f64, P_f64, P_f64, P_f64, P_f64],
    "dare_reslice": [c_vp, c_i32, P_f64, c_i32, c_i32, ctypes.POINTER(ResliceCfg), P_u8, P_u8],
    "dare_reslice_packed": [c_vp, c_i32, P_f64, c_i32, c_i32, ctypes.POINTER(ResliceCfg), P_u8, P_u8],
    "dare_reslice_bruteforce": [c_vp, c_i32, P_f64, c_i32, c_i32, ctypes.POINTER(ResliceCfg), P_u8,
                                P_u8],
    "dare_poses_coherent": [P_f64, c_i32, c_i32, c_i32, c_f64],
    "dare_reslice_device": [c_vp, c_i32, c_vp, c_i32, c_i32, ctypes.POINTER(ResliceCfg), c_vp,
                            c_vp, c_vp],
    "dare_compound": [c_vp, c_i64, c_i32, c_i32, c_i32, P_i32, c_i64, P_f64, c_f64, c_f64, P_u8,
                      P_f64, c_f64, P_i64, ctypes.POINTER(c_vp)],
    "dare_volume_merge": [P_f64, c_f64, P_i64, c_i32, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                          ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), P_i64, P_i64, P_i64, ctypes.POINTER(c_vp)],
    "dare_compound_accumulate": [c_vp, c_i64, c_i32, c_i32, c_i32, P_i32, c_i64, P_f64, c_f64, c_f64,
                                 P_u8, P_f64, c_f64, P_i64, c_vp, c_vp, c_vp],
    "dare_scalar_from_sums": [P_f64, c_f64, P_i64, c_vp, c_vp, ctypes.POINTER(c_vp)],
    "dare_scalar_upload": [P_f64, c_f64, P_i64, P_f32, P_u8, P_i64, ctypes.POINTER(c_vp)],
    "dare_scalar_download": [c_vp, P_f32, P_u8, P_i64],
    "dare_scalar_get_info": [c_vp, ctypes.POINTER(ScalarInfo)],
    "dare_scalar_destroy": [c_vp],
    "dare_fill_holes": [c_vp, c_i32, ctypes.POINTER(c_vp), P_i32],
    "dare_reslice_trilinear": [c_vp, c_i32, P_f64, c_i32, c_i32, P_u8, P_u8, P_f64],
    "dare_reslice_trilinear_device": [c_vp, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp],
    "dare_similarity": [c_i32, c_i32, c_i32, c_i32, c_vp, P_u8, c_vp, P_u8, c_i32, c_f64, c_f64, P_f64, P_f64,
                        P_i64, P_i32],
    "dare_similarity_device": [c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_f64, c_f64, c_vp,
                               c_vp, c_vp, c_vp, c_vp],
    "dare_exp_device": [c_vp, c_vp, c_i64, c_vp],
    "dare_reslice_last_fallback": [P_i64],
    "dare_fastmath_check": [P_f64, P_f64, P_i32],
    "dare_cell_thresholds": [P_f64, c_f64, P_i64, c_i32, P_f64, P_i64],
}

EXPORTED = ["dare_last_error", *_SIGNATURES]

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


class DareRuntimeError(RuntimeError):
    """A libdare_b200 call failed (CUDA error, allocation failure, ...)."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def load() -> ctypes.CDLL:
    """Loads the CUDA library; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2605_26325_b200.build` "
                "(the CUDA extension is required; there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        lib.dare_last_error.restype = ctypes.c_char_p
        lib.dare_last_error.argtypes = []
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib = lib
    return _lib


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != DARE_OK:
        msg = lib.dare_last_error().decode(errors="replace")
        if rc == DARE_ERR_INVALID:
            raise InvalidArgumentError(f"{name}: {msg}")
        raise DareRuntimeError(name, rc, msg)


def ptr(arr: np.ndarray | None, ctype):
    """Pointer to a C-contiguous numpy array (or NULL)."""
    if arr is None:
        return ctypes.cast(None, ctypes.POINTER(ctype))
    assert arr.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


def vptr(arr: np.ndarray | None) -> ctypes.c_void_p:
    if arr is None:
        return ctypes.c_void_p(None)
    assert arr.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return ctypes.c_void_p(arr.ctypes.data)


def device_count() -> int:
    n = ctypes.c_int32(0)
    call("dare_get_device_count", ctypes.byref(n))
    return int(n.value)


def set_device(dev: int) -> None:
    call("dare_set_device", int(dev))


def init(dev: int = 0) -> None:
    """dare_init: device, stream and the one-time fast-math check up front."""
    call("dare_init", int(dev))


def trim(keep_bytes: int = 0) -> None:
    """dare_trim: release unused pooled device memory (volumes / build scratch)."""
    call("dare_trim", int(keep_bytes))
