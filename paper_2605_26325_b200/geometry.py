"""Host-side rigid-pose arithmetic feeding the kernels (f64, bit-exact).

Restates pkg/src/dare/geometry.py:1-180.  Every value the device consumes
(frame axes, plane rotation matrices, canonical frame quaternions) is derived
here, so each expression keeps the reference's operation order and uses the
same primitives (Python float ops, math.sqrt/acos/sin, np.cross,
np.linalg.norm).  All functions are duck-typed: they accept this module's
Quaternion/Pose or the reference's (anything with .w/.x/.y/.z and
.rotation/.translation).

Vectorised helpers (`*_many`) evaluate the same per-element expressions over
arrays of frames; numpy's elementwise +,-,*,/ and sqrt are IEEE-exact, so they
reproduce the scalar path bit for bit (geometry.py:99-107 uses np.cross on
single vectors, which is the same elementwise formula).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidArgumentError

UNIT_NORM_TOL = 1e-3  # geometry.py:20


def _quat_norm(w: float, x: float, y: float, z: float) -> float:
    return math.sqrt(w * w + x * x + y * y + z * z)


@dataclass(frozen=True)
class Quaternion:
    """Scalar-first Hamilton quaternion (geometry.py:22-96)."""

    w: float
    x: float
    y: float
    z: float

    @staticmethod
    def identity() -> "Quaternion":
        return Quaternion(1.0, 0.0, 0.0, 0.0)

    @staticmethod
    def from_axis_angle(axis, angle_rad: float) -> "Quaternion":
        a = np.asarray(axis, dtype=float)
        n = np.linalg.norm(a)
        if n == 0.0:
            raise InvalidArgumentError("rotation axis must be nonzero")
        a = a / n
        s = math.sin(0.5 * angle_rad)
        return Quaternion(math.cos(0.5 * angle_rad), a[0] * s, a[1] * s, a[2] * s)

    def norm(self) -> float:
        return _quat_norm(self.w, self.x, self.y, self.z)

    def normalized(self) -> "Quaternion":
        return Quaternion(*normalize(self))

    def canonical(self) -> "Quaternion":
        return Quaternion(*canonical(self))

    def conjugate(self) -> "Quaternion":
        return Quaternion(self.w, -self.x, -self.y, -self.z)

    def multiply(self, other) -> "Quaternion":
        return Quaternion(*qmul(self, other))

    def rotation_matrix(self) -> np.ndarray:
        return rotation_matrix(self)

    def as_array(self) -> np.ndarray:
        return np.array([self.w, self.x, self.y, self.z])

    def angle_to(self, other) -> float:
        d = abs(self.w * other.w + self.x * other.x + self.y * other.y + self.z * other.z)
        return 2.0 * math.acos(min(1.0, d))


def normalize(q) -> tuple[float, float, float, float]:
    n = _quat_norm(q.w, q.x, q.y, q.z)
    if n == 0.0:
        raise InvalidArgumentError("cannot normalize zero quaternion")
    return (q.w / n, q.x / n, q.y / n, q.z / n)


def canonical(q) -> tuple[float, float, float, float]:
    """Sign flip so that w >= 0 (ties broken on x, y, z) -- geometry.py:56-64."""
    w, x, y, z = q.w, q.x, q.y, q.z
    flip = w < 0.0 or (w == 0.0 and (x < 0.0 or (x == 0.0 and (y < 0.0 or (y == 0.0 and z < 0.0)))))
    return (-w, -x, -y, -z) if flip else (w, x, y, z)


def qmul(a, b) -> tuple[float, float, float, float]:
    """Hamilton product a*b, component expressions as geometry.py:69-77."""
    return (
        a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
        a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
        a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
        a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w,
    )


def rotation_matrix(q) -> np.ndarray:
    """R(q) without renormalisation (geometry.py:79-88)."""
    w, x, y, z = q.w, q.x, q.y, q.z
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def rotate(q, v) -> np.ndarray:
    """R(q) v via v + w t + u x t, t = 2 u x v (geometry.py:99-107)."""
    if abs(_quat_norm(q.w, q.x, q.y, q.z) - 1.0) > UNIT_NORM_TOL:
        raise InvalidArgumentError(
            f"quaternion norm {_quat_norm(q.w, q.x, q.y, q.z):.6f} deviates from 1 by more than {UNIT_NORM_TOL}"
        )
    v = np.asarray(v, dtype=float)
    u = np.array([q.x, q.y, q.z])
    t = 2.0 * np.cross(u, v)
    return v + q.w * t + np.cross(u, t)


def rotate_many(quats: np.ndarray, vecs: np.ndarray) -> np.ndarray:
    """rotate() for arrays: quats (n,4) w,x,y,z; vecs (n,3) or (3,)."""
    norms = np.sqrt(quats[:, 0] * quats[:, 0] + quats[:, 1] * quats[:, 1]
                    + quats[:, 2] * quats[:, 2] + quats[:, 3] * quats[:, 3])
    bad = np.abs(norms - 1.0) > UNIT_NORM_TOL
    if np.any(bad):
        raise InvalidArgumentError(
            f"quaternion norm {float(norms[bad][0]):.6f} deviates from 1 by more than {UNIT_NORM_TOL}"
        )
    # np.cross restated per component with numpy's own order (a1*b2 - a2*b1,
    # a2*b0 - a0*b2, a0*b1 - a1*b0; separately rounded): identical bits,
    # without np.cross's per-call axis shuffling
    w, u0, u1, u2 = quats[:, 0], quats[:, 1], quats[:, 2], quats[:, 3]
    v = np.broadcast_to(np.asarray(vecs, dtype=float), (len(quats), 3))
    v0, v1, v2 = v[:, 0], v[:, 1], v[:, 2]
    t0, t1, t2 = 2.0 * (u1 * v2 - u2 * v1), 2.0 * (u2 * v0 - u0 * v2), 2.0 * (u0 * v1 - u1 * v0)
    out = np.empty((len(quats), 3))
    out[:, 0] = (v0 + w * t0) + (u1 * t2 - u2 * t1)
    out[:, 1] = (v1 + w * t1) + (u2 * t0 - u0 * t2)
    out[:, 2] = (v2 + w * t2) + (u0 * t1 - u1 * t0)
    return out


def rotate_grid(quats: np.ndarray, vecs: np.ndarray) -> np.ndarray:
    """rotate() of k vectors by each of n quaternions -> (n, k, 3); the same
    separately rounded expressions as rotate_many, broadcast (n,1) x (1,k)."""
    norms = np.sqrt(quats[:, 0] * quats[:, 0] + quats[:, 1] * quats[:, 1]
                    + quats[:, 2] * quats[:, 2] + quats[:, 3] * quats[:, 3])
    bad = np.abs(norms - 1.0) > UNIT_NORM_TOL
    if np.any(bad):
        raise InvalidArgumentError(
            f"quaternion norm {float(norms[bad][0]):.6f} deviates from 1 by more than {UNIT_NORM_TOL}"
        )
    w, u0, u1, u2 = (quats[:, i:i + 1] for i in range(4))
    v = np.asarray(vecs, dtype=float)
    v0, v1, v2 = v[None, :, 0], v[None, :, 1], v[None, :, 2]
    t0, t1, t2 = 2.0 * (u1 * v2 - u2 * v1), 2.0 * (u2 * v0 - u0 * v2), 2.0 * (u0 * v1 - u1 * v0)
    out = np.empty((len(quats), len(v), 3))
    out[:, :, 0] = (v0 + w * t0) + (u1 * t2 - u2 * t1)
    out[:, :, 1] = (v1 + w * t1) + (u2 * t0 - u0 * t2)
    out[:, :, 2] = (v2 + w * t2) + (u0 * t1 - u1 * t0)
    return out


def rotation_matrices(quats: np.ndarray) -> np.ndarray:
    """rotation_matrix() for quats (n,4) -> (n,3,3)."""
    w, x, y, z = (quats[:, i] for i in range(4))
    out = np.empty((len(quats), 3, 3))
    out[:, 0, 0] = 1 - 2 * (y * y + z * z)
    out[:, 0, 1] = 2 * (x * y - w * z)
    out[:, 0, 2] = 2 * (x * z + w * y)
    out[:, 1, 0] = 2 * (x * y + w * z)
    out[:, 1, 1] = 1 - 2 * (x * x + z * z)
    out[:, 1, 2] = 2 * (y * z - w * x)
    out[:, 2, 0] = 2 * (x * z - w * y)
    out[:, 2, 1] = 2 * (y * z + w * x)
    out[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return out


@dataclass(frozen=True)
class Pose:
    """Rigid transform local -> world: rotate, then translate (geometry.py:110-137)."""

    rotation: Quaternion
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        object.__setattr__(self, "translation", np.asarray(self.translation, dtype=float).reshape(3))

    @staticmethod
    def identity() -> "Pose":
        return Pose(Quaternion.identity(), np.zeros(3))

    def apply(self, point) -> np.ndarray:
        return rotate(self.rotation, point) + self.translation

    def compose(self, other) -> "Pose":
        return compose(self, other)

    def inverse(self) -> "Pose":
        inv = self.rotation.conjugate()
        return Pose(inv, -rotate(inv, self.translation))


def compose(a, b) -> Pose:
    """a o b (apply b first) -- geometry.py:128-133."""
    rot = Quaternion(*normalize(Quaternion(*qmul(a.rotation, b.rotation))))
    return Pose(rot, rotate(a.rotation, b.translation) + a.translation)


@dataclass(frozen=True)
class FrameAxes:
    x_axis: np.ndarray
    y_axis: np.ndarray
    normal: np.ndarray


def frame_axes(p) -> FrameAxes:
    r = rotation_matrix(p.rotation)
    return FrameAxes(x_axis=r[:, 0].copy(), y_axis=r[:, 1].copy(), normal=r[:, 2].copy())


def slerp(q0, q1, t: float) -> Quaternion:
    """Shortest-arc slerp with the nlerp branch above dot 0.9995 (geometry.py:159-180)."""
    a = np.array([q0.w, q0.x, q0.y, q0.z])
    b = np.array([q1.w, q1.x, q1.y, q1.z])
    dot = float(np.dot(a, b))
    if dot < 0.0:
        b = -b
        dot = -dot
    if dot > 0.9995:
        out = a + t * (b - a)
        return Quaternion(*(out / np.linalg.norm(out)))
    theta = math.acos(min(1.0, dot))
    s = math.sin(theta)
    out = (math.sin((1.0 - t) * theta) / s) * a + (math.sin(t * theta) / s) * b
    return Quaternion(*(out / np.linalg.norm(out)))
