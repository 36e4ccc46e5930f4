"""Synthetic workloads of BASELINE.json's configs.

Geometry follows the reference harness: cfg1/cfg2 are SweepPlan.linear
(phantom.py:202-216) from identity to (0, 0, L), L = (W-1)*pitch; cfg3 merges
four 2000-frame sweeps (normals +z, -z, +x, +y) over one cube the way
phantom.merge_recordings does (timestamps continue after a 0.5 s gap); frames
at 30 Hz with the pose stream equal to the frame timestamps, identity
calibration, no mask.  Reslice planes: cfg1/cfg2 rng = default_rng(0),
rotation about x by U(-10, 10) deg, translation (0, 0, L*(0.1 + 0.8 U));
cfg4 is a 10k-pose haptic-style trajectory on the cfg3 volume (random-walk
centre with N(0, 0.05 mm) steps reflected inside the cube, base orientation
cycling A -> B -> C -> D every 2500 poses plus a bounded +-20 deg tilt random
walk with 0.2 deg steps).  Image content is a synthetic phantom (background 24,
spherical inclusions, speckle) rendered on the GPU with torch -- the reference's
CPU renderer takes ~2 min for cfg2 and ~16 min for cfg3; content does not
change the work the hot path does (every pixel is scattered, every visited
sample is evaluated).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CONFIGS = {
    # frames, H=W, pitch, voxel, plane raster, poses per step, sweeps
    "cfg1": dict(frames=200, size=128, pitch=0.25, voxel=0.25, plane=128, batch=64, sweeps=1),
    "cfg2": dict(frames=1000, size=512, pitch=0.125, voxel=0.25, plane=256, batch=64, sweeps=1),
    "cfg3": dict(frames=8000, size=512, pitch=0.125, voxel=0.125, plane=512, batch=16, sweeps=4),
    "cfg4": dict(frames=8000, size=512, pitch=0.125, voxel=0.125, plane=512, batch=100, sweeps=4),
}


@dataclass
class Workload:
    name: str
    n_frames: int
    size: int
    pitch: float
    voxel: float
    plane: int
    batch: int
    sweeps: int

    @property
    def length(self) -> float:
        return (self.size - 1) * self.pitch


def workload(name: str) -> Workload:
    c = CONFIGS[name]
    return Workload(name, c["frames"], c["size"], c["pitch"], c["voxel"], c["plane"], c["batch"], c["sweeps"])


def _q(axis, deg):
    from paper_2605_26325_b200.geometry import Quaternion

    if deg == 0.0:
        return Quaternion(1.0, 0.0, 0.0, 0.0)
    return Quaternion.from_axis_angle(axis, math.radians(deg))


def sweep_poses(wl: Workload):
    """Frame poses and timestamps.  cfg1/cfg2: SweepPlan.linear(identity,
    Pose(I, (0,0,L)), n) -- slerp(I, I, t) = I exactly, translation (1-t)*0 + t*L.
    cfg3/cfg4: four sweeps (A) identity at (0,0,s), (B) 180 deg about x at
    (0,L,s), (C) +90 deg about y at (s,0,L), (D) -90 deg about x at (0,s,L),
    s = linspace(0, L, n/4), merged in that order."""
    from paper_2605_26325_b200.geometry import Pose

    L = wl.length
    if wl.sweeps == 1:
        n = wl.n_frames
        start, end = np.zeros(3), np.array([0.0, 0.0, L])
        poses = [Pose(_q((1, 0, 0), 0.0), (1.0 - k / (n - 1)) * start + (k / (n - 1)) * end) for k in range(n)]
        return poses, np.arange(n, dtype=float) / 30.0
    m = wl.n_frames // 4
    s = np.linspace(0.0, L, m)
    specs = [(_q((1, 0, 0), 0.0), lambda x: (0.0, 0.0, x)), (_q((1, 0, 0), 180.0), lambda x: (0.0, L, x)),
             (_q((0, 1, 0), 90.0), lambda x: (x, 0.0, L)), (_q((1, 0, 0), -90.0), lambda x: (0.0, x, L))]
    poses, ts, offset = [], [], 0.0
    for q, where in specs:
        t = offset + np.arange(m, dtype=float) / 30.0
        poses.extend(Pose(q, where(float(x))) for x in s)
        ts.append(t)
        offset = float(t[-1]) + 0.5
    return poses, np.concatenate(ts)


def render_frames_torch(wl: Workload, device="cuda", seed=7):
    """(n, H, W) u8 frames on the device: background 24, three spheres, speckle,
    sampled at each frame's world pixel positions."""
    import torch

    from paper_2605_26325_b200.geometry import rotation_matrix

    poses, _ = sweep_poses(wl)
    n, sz, p = wl.n_frames, wl.size, wl.pitch
    L = wl.length
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    uu = torch.arange(sz, device=device, dtype=torch.float32) * p
    U = uu[None, :].expand(sz, sz)
    V = uu[:, None].expand(sz, sz)
    centers = [(0.3 * L, 0.4 * L, 0.35 * L, 0.12 * L, 200.0), (0.65 * L, 0.55 * L, 0.6 * L, 0.15 * L, 140.0),
               (0.5 * L, 0.3 * L, 0.8 * L, 0.08 * L, 255.0)]
    R = torch.tensor(np.array([rotation_matrix(q.rotation) for q in poses]), dtype=torch.float32, device=device)
    T = torch.tensor(np.array([q.translation for q in poses]), dtype=torch.float32, device=device)
    frames = torch.empty((n, sz, sz), dtype=torch.uint8, device=device)
    chunk = 64
    for k0 in range(0, n, chunk):
        k1 = min(n, k0 + chunk)
        r, t = R[k0:k1], T[k0:k1]
        xyz = [t[:, a, None, None] + U[None] * r[:, a, 0, None, None] + V[None] * r[:, a, 1, None, None]
               for a in range(3)]
        val = torch.full((k1 - k0, sz, sz), 24.0, device=device)
        for cx, cy, cz, rad, level in centers:
            inside = (xyz[0] - cx) ** 2 + (xyz[1] - cy) ** 2 + (xyz[2] - cz) ** 2 <= rad * rad
            val = torch.where(inside, torch.full_like(val, level), val)
        val = val + 5.0 * torch.randn(val.shape, generator=g, device=device)
        frames[k0:k1] = val.clamp(0, 255).round().to(torch.uint8)
    return frames


def render_frames_numpy(wl: Workload, seed=7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, (wl.n_frames, wl.size, wl.size), dtype=np.uint8)


def reslice_planes(wl: Workload, count: int, seed: int = 0):
    """cfg1/cfg2 planes (Appendix B): rotation about x by U(-10,10) deg, z = L*(0.1+0.8U);
    cfg3/cfg4: the trajectory below."""
    from paper_2605_26325_b200.geometry import Pose, Quaternion
    from paper_2605_26325_b200.reslice import ReslicePlane

    if wl.sweeps > 1:
        return trajectory_planes(wl, count, seed)
    rng = np.random.default_rng(seed)
    L = wl.length
    pitch = L / (wl.plane - 1)
    planes = []
    for _ in range(count):
        ang = math.radians(float(rng.uniform(-10.0, 10.0)))
        z = L * (0.1 + 0.8 * float(rng.uniform()))
        planes.append(ReslicePlane(Pose(Quaternion.from_axis_angle((1, 0, 0), ang), (0.0, 0.0, z)),
                                   wl.plane, wl.plane, (pitch, pitch)))
    return planes


def trajectory_planes(wl: Workload, count: int, seed: int = 0, period: int = 2500):
    """cfg4: smooth haptic-style trajectory of 512x512 planes (pitch = frame pitch)."""
    from paper_2605_26325_b200.geometry import Pose, Quaternion, qmul, rotation_matrix
    from paper_2605_26325_b200.reslice import ReslicePlane

    rng = np.random.default_rng(seed)
    L = wl.length
    bases = [_q((1, 0, 0), 0.0), _q((1, 0, 0), 180.0), _q((0, 1, 0), 90.0), _q((1, 0, 0), -90.0)]
    p = np.full(3, 0.5 * L)
    tilt = np.zeros(2)
    planes = []
    half = np.array([wl.plane * wl.pitch / 2, wl.plane * wl.pitch / 2, 0.0])
    for k in range(count):
        p = p + rng.normal(0.0, 0.05, 3)
        p = np.where(p < 0, -p, p)
        p = np.where(p > L, 2 * L - p, p)
        tilt = np.clip(tilt + rng.normal(0.0, 0.2, 2), -20.0, 20.0)
        base = bases[(k // period) % 4]
        q = Quaternion(*qmul(Quaternion(*qmul(base, _q((1, 0, 0), float(tilt[0])))), _q((0, 1, 0), float(tilt[1]))))
        origin = p - rotation_matrix(q) @ half
        planes.append(ReslicePlane(Pose(q, origin), wl.plane, wl.plane, (wl.pitch, wl.pitch)))
    return planes
