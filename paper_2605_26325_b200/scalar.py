"""Direction-blind comparison arm on the device (drop-in for pkg/src/dare/baseline.py).

compound -> fill_holes -> reslice_trilinear, with the reference signatures,
validation and return types; the work runs in csrc/scalar.cu.  A ScalarVolume
holds a device handle; values / flags / counts are downloaded lazily.
"""
from __future__ import annotations

import ctypes
import struct
import threading
import time
import weakref

import numpy as np

from . import _lib
from .errors import InvalidArgumentError, VolumeFormatError
from .reslice import ResliceImage, plane_params
from .sweep import grid_for, plan_frames, validate_margin

SCALAR_MAGIC = b"DARS"
SCALAR_VERSION = 1
VOXEL_EMPTY = 0
VOXEL_OBSERVED = 1
VOXEL_FILLED = 2
_HEADER = struct.Struct("<4sI3dd3IQ")
_REC = np.dtype([("value", "<f4"), ("flag", "u1")])


def _destroy(raw: int) -> None:
    try:
        _lib.load().dare_scalar_destroy(ctypes.c_void_p(raw))
    except Exception:
        pass


class ScalarVolume:
    """Mean-compounded voxel grid (baseline.py:32-61), device-resident."""

    def __init__(self, origin, voxel_size, dims, values=None, flags=None, counts=None, *, _raw=None):
        self.origin = np.asarray(origin, dtype=float).reshape(3).copy()
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(d) for d in dims)
        self._lock = threading.Lock()
        self._raw = None
        self._host = None
        if _raw is not None:
            self._raw = ctypes.c_void_p(_raw)
            self._fin = weakref.finalize(self, _destroy, _raw)
            info = _lib.ScalarInfo()
            _lib.call("dare_scalar_get_info", self._raw, ctypes.byref(info))
            self._has_counts = bool(info.d_counts)
        else:
            if values is None or flags is None:
                raise InvalidArgumentError("values and flags required without a device handle")
            self._set_host(values, flags, counts)

    def _set_host(self, values, flags, counts):
        v = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        f = np.ascontiguousarray(flags, dtype=np.uint8).reshape(-1)
        c = None if counts is None else np.ascontiguousarray(counts, dtype=np.int64).reshape(-1)
        for a in (v, f, c):
            if a is not None:
                a.flags.writeable = False
        self._host = (v, f, c)
        self._has_counts = c is not None

    def _host_arrays(self):
        if self._host is None:
            with self._lock:
                if self._host is None:
                    n = self.cell_count
                    v = np.empty(n, np.float32)
                    f = np.empty(n, np.uint8)
                    c = np.empty(n, np.int64) if self._has_counts else None
                    _lib.call("dare_scalar_download", self._raw, _lib.ptr(v, ctypes.c_float),
                              _lib.ptr(f, ctypes.c_uint8), _lib.ptr(c, ctypes.c_int64))
                    self._set_host(v, f, c)
        return self._host

    def device_handle(self) -> ctypes.c_void_p:
        if self._raw is None:
            with self._lock:
                if self._raw is None:
                    v, f, c = self._host
                    raw = ctypes.c_void_p()
                    o = np.ascontiguousarray(self.origin, dtype=np.float64)
                    d = np.ascontiguousarray(self.dims, dtype=np.int64)
                    _lib.call("dare_scalar_upload", _lib.ptr(o, ctypes.c_double), self.voxel_size,
                              _lib.ptr(d, ctypes.c_int64), _lib.ptr(v, ctypes.c_float),
                              _lib.ptr(f, ctypes.c_uint8), _lib.ptr(c, ctypes.c_int64), ctypes.byref(raw))
                    self._raw = raw
                    self._fin = weakref.finalize(self, _destroy, raw.value)
        return self._raw

    @property
    def values(self) -> np.ndarray:
        return self._host_arrays()[0]

    @property
    def flags(self) -> np.ndarray:
        return self._host_arrays()[1]

    @property
    def counts(self):
        return self._host_arrays()[2]

    @property
    def cell_count(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    @property
    def observed_count(self) -> int:
        return int(np.count_nonzero(self.flags == VOXEL_OBSERVED))

    def grid_view(self, arr: np.ndarray) -> np.ndarray:
        return arr.reshape(self.dims)


_foreign: "weakref.WeakKeyDictionary[object, ScalarVolume]" = weakref.WeakKeyDictionary()


def as_device_scalar(volume) -> ScalarVolume:
    if isinstance(volume, ScalarVolume):
        return volume
    def convert():
        return ScalarVolume(volume.origin, volume.voxel_size, volume.dims, volume.values, volume.flags,
                            getattr(volume, "counts", None))

    try:
        cached = _foreign.get(volume)
    except TypeError:  # not weak-referenceable: no caching
        return convert()
    if cached is None:
        cached = convert()
        _foreign[volume] = cached
    return cached


def compound(sweep, voxel_size: float = 0.125, margin: float = 1.0) -> ScalarVolume:
    """Per-voxel mean of all pixel intensities (baseline.py:64-97)."""
    validate_margin(margin)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, voxel_size, margin)
    from .reconstruct import frames_arg

    images, frames_ptr, on_device = frames_arg(sweep)
    mask = None
    if sweep.mask is not None:
        mask = np.ascontiguousarray(np.asarray(sweep.mask, dtype=bool).reshape(-1).astype(np.uint8))
    axes = plan.axes()
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    raw = ctypes.c_void_p()
    _lib.call("dare_compound", frames_ptr, int(images.shape[0]), plan.height, plan.width, on_device,
              _lib.ptr(plan.image_index, ctypes.c_int32), plan.n_frames, _lib.ptr(axes, ctypes.c_double),
              plan.pixel_pitch[0], plan.pixel_pitch[1], _lib.ptr(mask, ctypes.c_uint8),
              _lib.ptr(o, ctypes.c_double), voxel, _lib.ptr(d, ctypes.c_int64), ctypes.byref(raw))
    return ScalarVolume(origin, voxel, dims, _raw=raw.value)


def fill_holes(volume, max_passes: int = 3) -> ScalarVolume:
    """Jacobi hole filling over 26-neighbourhoods (baseline.py:100-127)."""
    src = as_device_scalar(volume)
    raw = ctypes.c_void_p()
    runs = ctypes.c_int32(0)
    _lib.call("dare_fill_holes", src.device_handle(), int(max_passes), ctypes.byref(raw), ctypes.byref(runs))
    out = ScalarVolume(src.origin, src.voxel_size, src.dims, _raw=raw.value)
    out.passes_run = int(runs.value)
    return out


def _trilinear(volume, planes, want_values: bool):
    planes = list(planes)
    params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
    w, h = planes[0].width, planes[0].height
    if any(p.width != w or p.height != h for p in planes):
        raise InvalidArgumentError("all planes of a batch must share width and height")
    t0 = time.perf_counter()
    handle = as_device_scalar(volume).device_handle()
    pixels = np.empty((len(planes), h, w), np.uint8)
    cov = np.empty((len(planes), h, w), np.uint8)
    vals = np.empty((len(planes), h, w), np.float64) if want_values else None
    _lib.call("dare_reslice_trilinear", handle, len(planes), _lib.ptr(params, ctypes.c_double), w, h,
              _lib.ptr(pixels, ctypes.c_uint8), _lib.ptr(cov, ctypes.c_uint8), _lib.ptr(vals, ctypes.c_double))
    ms = (time.perf_counter() - t0) * 1000.0
    return pixels, cov.view(np.bool_), vals, ms


def reslice_trilinear(volume, plane) -> ResliceImage:
    """Direction-blind trilinear reslice (baseline.py:130-155)."""
    pixels, cov, _, ms = _trilinear(volume, [plane], False)
    return ResliceImage(pixels=pixels[0], coverage=cov[0], timing_ms=ms)


def reslice_trilinear_batch(volume, planes):
    pixels, cov, _, ms = _trilinear(volume, planes, False)
    return pixels, cov, ms


def trilinear_at_points(volume, points) -> tuple[np.ndarray, np.ndarray]:
    """Pre-rounding trilinear values at world points (baseline.py:158-182):
    each point is a 1x1 plane with identity axes."""
    from .geometry import Pose, Quaternion
    from .reslice import ReslicePlane

    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if len(pts) == 0:
        return np.zeros(0), np.zeros(0, dtype=bool)
    planes = [ReslicePlane(Pose(Quaternion.identity(), p), 1, 1, (1.0, 1.0)) for p in pts]
    _, cov, vals, _ = _trilinear(volume, planes, True)
    return vals.reshape(-1), cov.reshape(-1)


def save_scalar_volume(volume, path) -> None:
    """.scalarvol writer (baseline.py:185-199), byte-identical."""
    n = int(np.prod(volume.dims))
    observed = int(np.count_nonzero(np.asarray(volume.flags) == VOXEL_OBSERVED))
    header = _HEADER.pack(SCALAR_MAGIC, SCALAR_VERSION, *[float(c) for c in volume.origin],
                          float(volume.voxel_size), *volume.dims, observed)
    rec = np.zeros(n, dtype=_REC)
    rec["value"] = volume.values
    rec["flag"] = volume.flags
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(rec.tobytes())


def load_scalar_volume(path) -> ScalarVolume:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER.size:
        raise VolumeFormatError(f"{path}: truncated header")
    magic, version, ox, oy, oz, voxel, nx, ny, nz, _ = _HEADER.unpack_from(raw, 0)
    if magic != SCALAR_MAGIC:
        raise VolumeFormatError(f"{path}: bad magic {magic!r}, expected {SCALAR_MAGIC!r}")
    if version != SCALAR_VERSION:
        raise VolumeFormatError(f"{path}: unsupported format version {version}")
    n = nx * ny * nz
    expected = _HEADER.size + n * _REC.itemsize
    if len(raw) != expected:
        raise VolumeFormatError(f"{path}: size {len(raw)} != expected {expected}")
    rec = np.frombuffer(raw, dtype=_REC, count=n, offset=_HEADER.size)
    return ScalarVolume((ox, oy, oz), voxel, (nx, ny, nz), np.ascontiguousarray(rec["value"]),
                        np.ascontiguousarray(rec["flag"]))
