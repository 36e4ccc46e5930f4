"""Direction-aware reslicing on the device (drop-in for pkg/src/dare/reslice.py).

`reslice(volume, plane, cfg)` keeps the reference signature, validation,
defaults and return type (reslice.py:168-187); the per-pixel work runs in the
sm_100a kernel (csrc/reslice.cu) through the C ABI.  `reslice_batch` is the
B200-native entry point: many poses of one raster size in one launch.
`timing_ms` covers host->device parameter copy, kernels and the
device->host copy of pixels + coverage ("query to final image").
"""
from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import geometry as geo
from .errors import InvalidArgumentError
from .geometry import FrameAxes, Pose
from .volume import as_device_volume

DEFAULT_INTERP_RADIUS_MM = 0.125
DEFAULT_NORMAL_THRESHOLD_DEG = 25.0
DEFAULT_INPLANE_THRESHOLD_DEG = 15.0
DEFAULT_K_NORMAL = 10.0
DEFAULT_K_INPLANE = 5.0
DEFAULT_K_DIST = 2.0


@dataclass(frozen=True)
class ReslicePlane:
    """Virtual image plane: pose of pixel (0,0) plus raster (reslice.py:45-60)."""

    pose: Pose
    width: int
    height: int
    pixel_pitch: tuple[float, float]

    def world_point(self, u: float, v: float) -> np.ndarray:
        px, py = self.pixel_pitch
        return self.pose.apply((u * px, v * py, 0.0))


@dataclass(frozen=True)
class ResliceConfig:
    """Radius, angular gates and weighting exponents (reslice.py:63-100)."""

    interp_radius: float = DEFAULT_INTERP_RADIUS_MM
    normal_threshold_deg: float = DEFAULT_NORMAL_THRESHOLD_DEG
    inplane_threshold_deg: float = DEFAULT_INPLANE_THRESHOLD_DEG
    k_normal: float = DEFAULT_K_NORMAL
    k_inplane: float = DEFAULT_K_INPLANE
    k_dist: float = DEFAULT_K_DIST
    unassigned_value: int = 0

    def __post_init__(self):
        if self.interp_radius <= 0:
            raise InvalidArgumentError("interp_radius must be > 0")
        for name in ("normal_threshold_deg", "inplane_threshold_deg"):
            if not (0.0 < getattr(self, name) < 90.0):
                raise InvalidArgumentError(f"{name} must lie in (0, 90) degrees")
        for name in ("k_normal", "k_inplane", "k_dist"):
            if getattr(self, name) < 0:
                raise InvalidArgumentError(f"{name} must be >= 0")
        if not (0 <= self.unassigned_value <= 255):
            raise InvalidArgumentError("unassigned_value must be a gray level 0..255")

    @property
    def cos_normal_threshold(self) -> float:
        return math.cos(math.radians(self.normal_threshold_deg))

    @property
    def cos_inplane_threshold(self) -> float:
        return math.cos(math.radians(self.inplane_threshold_deg))


@dataclass
class ResliceImage:
    pixels: np.ndarray    # (H, W) u8
    coverage: np.ndarray  # (H, W) bool
    timing_ms: float


def directional_dots(sample_axes: FrameAxes, plane_axes: FrameAxes) -> tuple[float, float]:
    """(signed normal dot, |in-plane x dot|) -- reslice.py:109-114."""
    return (float(np.dot(sample_axes.normal, plane_axes.normal)),
            float(abs(np.dot(sample_axes.x_axis, plane_axes.x_axis))))


def accept(dots: tuple[float, float], cfg) -> bool:
    d_normal, d_inplane = dots
    return d_normal >= cfg.cos_normal_threshold and d_inplane >= cfg.cos_inplane_threshold


def sample_weight(dots: tuple[float, float], dist: float, cfg) -> float:
    """Scalar twin of the kernel weight (reslice.py:127-132)."""
    d_normal, d_inplane = dots
    orient = math.exp(cfg.k_normal * (d_normal - 1.0) + cfg.k_inplane * (d_inplane - 1.0))
    return orient * math.exp(-cfg.k_dist * dist / cfg.interp_radius)


def plane_params(plane) -> tuple[float, ...]:
    """14 f64 kernel scalars from a plane (reslice.py:135-148)."""
    if plane.width <= 0 or plane.height <= 0:
        raise InvalidArgumentError("reslice plane must have at least one pixel")
    q = plane.pose.rotation
    if abs(math.sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z) - 1.0) > 1e-3:
        raise InvalidArgumentError("plane rotation must be unit norm")
    r = geo.rotation_matrix(q)
    t = plane.pose.translation
    return (float(t[0]), float(t[1]), float(t[2]),
            float(r[0, 0]), float(r[0, 1]), float(r[0, 2]),
            float(r[1, 0]), float(r[1, 1]), float(r[1, 2]),
            float(r[2, 0]), float(r[2, 1]), float(r[2, 2]),
            float(plane.pixel_pitch[0]), float(plane.pixel_pitch[1]))


def kernel_cfg(cfg, schedule: int = 0, exact: bool = False) -> _lib.ResliceCfg:
    """Kernel scalars; schedule 0 = auto, 1 = pixel-major, 2 = pose-major;
    exact=True forces FP64 reference arithmetic for every pixel (the default
    certified path gives the same pixels, see csrc/reslice.cu)."""
    return _lib.ResliceCfg(float(cfg.interp_radius), float(cfg.cos_normal_threshold),
                           float(cfg.cos_inplane_threshold), float(cfg.k_normal),
                           float(cfg.k_inplane), float(cfg.k_dist), int(cfg.unassigned_value), int(schedule),
                           1 if exact else 0, 0)


def _run(fn: str, volume, planes, cfg):
    cfg = cfg or ResliceConfig()
    planes = list(planes)
    if not planes:
        raise InvalidArgumentError("at least one plane required")
    params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
    w, h = planes[0].width, planes[0].height
    if any(p.width != w or p.height != h for p in planes):
        raise InvalidArgumentError("all planes of a batch must share width and height")
    kc = kernel_cfg(cfg)
    t0 = time.perf_counter()
    vol = as_device_volume(volume).device_handle()
    pixels = np.empty((len(planes), h, w), dtype=np.uint8)
    cov = np.empty((len(planes), h, w), dtype=np.uint8)
    _lib.call(fn, vol.raw, len(planes), _lib.ptr(params, ctypes.c_double), w, h, ctypes.byref(kc),
              _lib.ptr(pixels, ctypes.c_uint8), _lib.ptr(cov, ctypes.c_uint8))
    timing_ms = (time.perf_counter() - t0) * 1000.0
    return pixels, cov.view(np.bool_), timing_ms


def reslice(volume, plane, cfg=None) -> ResliceImage:
    """Grid-accelerated directional reslice (reslice.py:168-187) on the GPU."""
    pixels, cov, ms = _run("dare_reslice", volume, [plane], cfg)
    return ResliceImage(pixels=pixels[0], coverage=cov[0], timing_ms=ms)


def reslice_bruteforce(volume, plane, cfg=None) -> ResliceImage:
    """Contract twin (reslice.py:190-205): every sample for every pixel, on the GPU."""
    pixels, cov, ms = _run("dare_reslice_bruteforce", volume, [plane], cfg)
    return ResliceImage(pixels=pixels[0], coverage=cov[0], timing_ms=ms)


def reslice_batch(volume, planes, cfg=None) -> tuple[np.ndarray, np.ndarray, float]:
    """Many planes (same raster) in one launch -> (pixels (P,H,W), coverage (P,H,W), ms)."""
    return _run("dare_reslice", volume, planes, cfg)
