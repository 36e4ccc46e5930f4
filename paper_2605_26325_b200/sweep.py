"""Sweep recordings and the host-side frame plan fed to the device.

Restates pkg/src/dare/reconstruct.py:30-163 (TrackedFrame, SweepRecording,
interpolate_pose, synchronize, frame_world_positions) and volume.py:57-73
(compute_bounds).  The per-frame pose pipeline is vectorised over frames
(the reference spends 0.4 ms/frame here in Python loops)
while keeping every floating-point expression identical to the scalar
reference; only frames that need slerp (timestamps strictly between two pose
samples) take the scalar path, because slerp's math.acos/sin and BLAS dot are
not elementwise numpy.
"""
from __future__ import annotations

import ctypes
import itertools
import math
import operator
from dataclasses import dataclass, field

import numpy as np

from . import geometry as geo
from .errors import InvalidArgumentError, SynchronizationError
from .geometry import Pose, Quaternion


@dataclass
class TrackedFrame:
    """One image with its synchronized image-plane pose (reconstruct.py:30-52)."""

    pixels: np.ndarray
    pixel_pitch: tuple[float, float]
    timestamp: float
    pose: Pose

    def __post_init__(self):
        self.pixels = np.asarray(self.pixels, dtype=np.uint8)
        if self.pixels.ndim != 2:
            raise InvalidArgumentError("frame pixels must be 2D")
        if self.pixel_pitch[0] <= 0 or self.pixel_pitch[1] <= 0:
            raise InvalidArgumentError("pixel pitch must be positive on both axes")

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


@dataclass
class SweepRecording:
    """Timestamped images + timestamped tracker poses (reconstruct.py:64-99)."""

    images: np.ndarray
    image_timestamps: np.ndarray
    pose_timestamps: np.ndarray
    poses: list
    pixel_pitch: tuple[float, float]
    calibration: Pose = field(default_factory=Pose.identity)
    mask: np.ndarray | None = None

    def __post_init__(self):
        self.images = np.asarray(self.images, dtype=np.uint8)
        self.image_timestamps = np.asarray(self.image_timestamps, dtype=float)
        self.pose_timestamps = np.asarray(self.pose_timestamps, dtype=float)
        if self.images.ndim != 3 or self.images.shape[0] == 0:
            raise InvalidArgumentError("recording needs at least one frame")
        if len(self.image_timestamps) != self.images.shape[0]:
            raise InvalidArgumentError("one timestamp per frame required")
        if len(self.poses) != len(self.pose_timestamps):
            raise InvalidArgumentError("one timestamp per pose sample required")
        if not (np.all(np.isfinite(self.image_timestamps)) and np.all(np.isfinite(self.pose_timestamps))):
            raise InvalidArgumentError("timestamps must be finite")
        if np.any(np.diff(self.image_timestamps) < 0) or np.any(np.diff(self.pose_timestamps) < 0):
            raise InvalidArgumentError("timestamps must be monotone non-decreasing")
        if abs(self.calibration.rotation.norm() - 1.0) > 1e-3:
            raise InvalidArgumentError("calibration rotation must be unit norm")

    @property
    def frame_count(self) -> int:
        return int(self.images.shape[0])


def interpolate_pose(t: float, timestamps: np.ndarray, poses: list) -> Pose:
    """Pose at time t (reconstruct.py:102-116)."""
    i = int(np.searchsorted(timestamps, t, side="right")) - 1
    if i < 0 or t > timestamps[-1]:
        raise InvalidArgumentError(f"time {t} outside pose stream range")
    if i == len(poses) - 1 or timestamps[i] == t:
        return poses[i]
    t0, t1 = timestamps[i], timestamps[i + 1]
    alpha = 0.0 if t1 == t0 else (t - t0) / (t1 - t0)
    p0, p1 = poses[i], poses[i + 1]
    return Pose(geo.slerp(p0.rotation, p1.rotation, alpha),
                (1.0 - alpha) * p0.translation + alpha * p1.translation)


@dataclass
class FramePlan:
    """Everything the device needs per synchronized frame, in frame order."""

    image_index: np.ndarray  # (n,) int32: which image each synchronized frame uses
    rotations: np.ndarray    # (n, 4) f64 image-plane quaternions (w,x,y,z), not canonicalised
    translations: np.ndarray  # (n, 3) f64
    dropped: int
    pixel_pitch: tuple[float, float]
    height: int
    width: int
    # from dare_frame_poses (csrc/plan.cu), same bits as the numpy restatements
    # below; None when the plan was built from arrays directly
    _axes: np.ndarray | None = field(default=None, repr=False)
    _quats32: np.ndarray | None = field(default=None, repr=False)
    _corner_box: tuple | None = field(default=None, repr=False)  # (lo, hi) before the margin
    _corner_error: str | None = field(default=None, repr=False)

    @property
    def n_frames(self) -> int:
        return int(len(self.image_index))

    def axes(self) -> np.ndarray:
        """(n, 9): R[:,0], R[:,1], t per frame (reconstruct.py:155-162)."""
        if self._axes is not None:
            return self._axes
        r = geo.rotation_matrices(self.rotations)
        return np.ascontiguousarray(np.concatenate([r[:, :, 0], r[:, :, 1], self.translations], axis=1))

    def canonical_quats_f32(self) -> np.ndarray:
        """(n, 4) f32 canonical frame quaternions (reconstruct.py:192-195)."""
        if self._quats32 is not None:
            return self._quats32
        q = self.rotations
        w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
        flip = (w < 0.0) | ((w == 0.0) & ((x < 0.0) | ((x == 0.0) & ((y < 0.0) | ((y == 0.0) & (z < 0.0))))))
        return np.ascontiguousarray(np.where(flip[:, None], -q, q).astype(np.float32))

    def bounds(self, margin: float):
        """compute_bounds (volume.py:57-73) over the four image corners."""
        from .volume import BoundingBox

        if self.n_frames == 0:
            raise InvalidArgumentError("compute_bounds requires at least one frame")
        if self._corner_box is not None:
            if self._corner_error is not None:
                raise InvalidArgumentError(self._corner_error)
            return BoundingBox(*self._corner_box).expanded(margin)
        # numpy restatement: the same sequential np.minimum / np.maximum
        px, py = self.pixel_pitch
        umax = (self.width - 1) * px
        vmax = (self.height - 1) * py
        corners = np.array([(0.0, 0.0, 0.0), (umax, 0.0, 0.0), (0.0, vmax, 0.0), (umax, vmax, 0.0)])
        c = (geo.rotate_grid(self.rotations, corners) + self.translations[:, None, :]).reshape(-1, 3)
        lo, hi = np.full(3, np.inf), np.full(3, -np.inf)
        for row in c:
            lo = np.minimum(lo, row)
            hi = np.maximum(hi, row)
        return BoundingBox(lo, hi).expanded(margin)


_wxyz = operator.attrgetter("w", "x", "y", "z")
_rotation = operator.attrgetter("rotation")


def _quat_array(poses) -> np.ndarray:
    return np.fromiter(itertools.chain.from_iterable(map(_wxyz, map(_rotation, poses))), dtype=float,
                       count=4 * len(poses)).reshape(-1, 4)


def _translation_array(poses) -> np.ndarray:
    if not poses:
        return np.zeros((0, 3))
    return np.concatenate([p.translation for p in poses]).astype(float, copy=False).reshape(-1, 3)


def plan_frames(sweep) -> FramePlan:
    """synchronize() (reconstruct.py:119-149) as arrays: drop images outside the
    pose stream, interpolate the marker pose, compose the calibration."""
    t_img = np.asarray(sweep.image_timestamps, dtype=float)
    ts = np.asarray(sweep.pose_timestamps, dtype=float)
    poses = list(sweep.poses)
    n_img, height, width = (int(d) for d in sweep.images.shape)  # numpy or CUDA tensor
    inside = ~((t_img < ts[0]) | (t_img > ts[-1]))
    kept = np.nonzero(inside)[0]
    dropped = int(n_img - len(kept))
    if len(kept) == 0:
        raise SynchronizationError(
            "no image falls inside the pose stream time range "
            f"(images {t_img[0]:.3f}..{t_img[-1]:.3f}s, poses {ts[0]:.3f}..{ts[-1]:.3f}s)"
        )
    px, py = sweep.pixel_pitch
    if px <= 0 or py <= 0:
        raise InvalidArgumentError("pixel pitch must be positive on both axes")

    t = t_img[kept]
    idx = np.searchsorted(ts, t, side="right") - 1
    exact = (idx == len(poses) - 1) | (ts[idx] == t)
    mq = np.empty((len(kept), 4))
    mt = np.empty((len(kept), 3))
    all_q = _quat_array(poses)
    all_t = _translation_array(poses)
    mq[exact] = all_q[idx[exact]]
    mt[exact] = all_t[idx[exact]]
    interp = np.nonzero(~exact)[0]
    if len(interp):  # slerp + lerp in one host call (csrc/plan.cu: dare_interpolate_poses)
        from . import _lib

        ti = np.ascontiguousarray(t[interp], dtype=np.float64)
        ii = np.ascontiguousarray(idx[interp], dtype=np.int64)
        oq = np.empty((len(interp), 4))
        ot = np.empty((len(interp), 3))
        P = ctypes.c_double
        tsc = np.ascontiguousarray(ts, dtype=np.float64)
        _lib.call("dare_interpolate_poses", len(interp), _lib.ptr(ti, P), _lib.ptr(ii, ctypes.c_int64),
                  _lib.ptr(tsc, P), _lib.ptr(all_q, P), _lib.ptr(all_t, P), _lib.ptr(oq, P), _lib.ptr(ot, P))
        mq[interp] = oq
        mt[interp] = ot

    return _compose_plan(kept, mq, mt, sweep.calibration, dropped, (float(px), float(py)), int(height), int(width))


def _compose_plan(kept, mq, mt, cal, dropped, pitch, height, width) -> FramePlan:
    """Marker pose o calibration, axes, canonical f32 quaternions and image
    corners for every frame in one host call (csrc/plan.cu: dare_frame_poses)."""
    from . import _lib

    n = len(kept)
    mq = np.ascontiguousarray(mq, dtype=np.float64)
    mt = np.ascontiguousarray(mt, dtype=np.float64)
    cq = cal.rotation
    cal_q = np.array([cq.w, cq.x, cq.y, cq.z], dtype=np.float64)
    cal_t = np.ascontiguousarray(np.asarray(cal.translation, dtype=float).reshape(3))
    rot = np.empty((n, 4))
    trans = np.empty((n, 3))
    axes = np.empty((n, 9))
    q32 = np.empty((n, 4), dtype=np.float32)
    lo, hi = np.empty(3), np.empty(3)
    status, bad, bad_norm = ctypes.c_int32(0), ctypes.c_int64(-1), ctypes.c_double(0.0)
    P = ctypes.c_double
    _lib.call("dare_frame_poses", n, _lib.ptr(mq, P), _lib.ptr(mt, P), _lib.ptr(cal_q, P), _lib.ptr(cal_t, P),
              int(width), int(height), pitch[0], pitch[1], _lib.ptr(rot, P), _lib.ptr(trans, P),
              _lib.ptr(axes, P), _lib.ptr(q32, ctypes.c_float), _lib.ptr(lo, P), _lib.ptr(hi, P), ctypes.byref(status),
              ctypes.byref(bad), ctypes.byref(bad_norm))
    norm_msg = "quaternion norm {:.6f} deviates from 1 by more than " + str(geo.UNIT_NORM_TOL)
    if status.value == 1:
        raise InvalidArgumentError("cannot normalize zero quaternion")
    if status.value == 2:
        raise InvalidArgumentError(norm_msg.format(bad_norm.value))
    corner_error = norm_msg.format(bad_norm.value) if status.value == 3 else None
    return FramePlan(kept.astype(np.int32), rot, trans, dropped, pitch, height, width,
                     _axes=axes, _quats32=q32, _corner_box=(lo, hi), _corner_error=corner_error)


def _compose_plan_numpy(kept, mq, mt, cal, dropped, pitch, height, width) -> FramePlan:
    """The same composition restated in numpy (cross-check for tests)."""
    px, py = pitch
    cq = cal.rotation
    w, x, y, z = mq[:, 0], mq[:, 1], mq[:, 2], mq[:, 3]
    prod = np.stack([
        w * cq.w - x * cq.x - y * cq.y - z * cq.z,
        w * cq.x + x * cq.w + y * cq.z - z * cq.y,
        w * cq.y - x * cq.z + y * cq.w + z * cq.x,
        w * cq.z + x * cq.y - y * cq.x + z * cq.w,
    ], axis=1)
    n = np.sqrt(prod[:, 0] * prod[:, 0] + prod[:, 1] * prod[:, 1]
                + prod[:, 2] * prod[:, 2] + prod[:, 3] * prod[:, 3])
    if np.any(n == 0.0):
        raise InvalidArgumentError("cannot normalize zero quaternion")
    rot = prod / n[:, None]
    trans = geo.rotate_many(mq, np.asarray(cal.translation, dtype=float)) + mt
    return FramePlan(kept.astype(np.int32), np.ascontiguousarray(rot), np.ascontiguousarray(trans),
                     dropped, (float(px), float(py)), int(height), int(width))


def synchronize(recording) -> tuple[list[TrackedFrame], int]:
    """Host API twin of reconstruct.py:119-149 (list of TrackedFrame objects)."""
    plan = plan_frames(recording)
    frames = []
    for j, k in enumerate(plan.image_index):
        q = Quaternion(*(float(c) for c in plan.rotations[j]))
        frames.append(TrackedFrame(np.asarray(recording.images)[k], recording.pixel_pitch,
                                   float(recording.image_timestamps[k]), Pose(q, plan.translations[j])))
    return frames, plan.dropped


def pixel_to_world(frame: TrackedFrame, u: float, v: float) -> np.ndarray:
    if not (0 <= u < frame.width) or not (0 <= v < frame.height):
        raise InvalidArgumentError(f"pixel ({u}, {v}) outside {frame.width}x{frame.height} image")
    px, py = frame.pixel_pitch
    return frame.pose.apply((u * px, v * py, 0.0))


def frame_world_positions(frame) -> np.ndarray:
    """(H, W, 3) f64 world positions (reconstruct.py:152-163); host helper."""
    px, py = frame.pixel_pitch
    r = geo.rotation_matrix(frame.pose.rotation)
    u = np.arange(frame.pixels.shape[1], dtype=np.float64) * px
    v = np.arange(frame.pixels.shape[0], dtype=np.float64) * py
    return u[None, :, None] * r[:, 0] + v[:, None, None] * r[:, 1] + frame.pose.translation


def validate_margin(margin: float) -> None:
    if margin < 0:
        raise InvalidArgumentError("margin must be >= 0")


def grid_for(plan: FramePlan, voxel_size: float, margin: float):
    """Bounds + VolumeBuilder sizing (reconstruct.py:181-184, volume.py:197-206)."""
    bounds = plan.bounds(margin)
    if margin == 0.0 and np.all(bounds.extent == 0.0):
        raise InvalidArgumentError("degenerate bounds: zero extent on all axes and no margin")
    if voxel_size <= 0:
        raise InvalidArgumentError("voxel_size must be > 0")
    dims = tuple(int(np.floor(e / voxel_size)) + 1 for e in bounds.extent)
    return bounds.min.copy(), float(voxel_size), dims


__all__ = [
    "TrackedFrame", "SweepRecording", "FramePlan", "interpolate_pose", "plan_frames",
    "synchronize", "pixel_to_world", "frame_world_positions", "grid_for", "validate_margin",
]
