"""Synthetic workloads of BASELINE.json's configs.

Geometry follows the reference harness exactly: SweepPlan.linear
(phantom.py:202-216) from identity to (0, 0, L), L = (W-1)*pitch, frames at
30 Hz with the pose stream equal to the frame timestamps (simulate_sweep,
phantom.py:219-249), identity calibration, no mask; reslice planes with
rng = default_rng(0), rotation about x by U(-10, 10) deg and translation
(0, 0, L*(0.1 + 0.8 U)).  Image content is a synthetic phantom (background 24,
spherical inclusions, speckle) rendered on the GPU with torch -- the
reference's CPU renderer (phantom.render_intensities) takes ~2 min for cfg2
and its RNG stream cannot be reproduced on the device; content does not
change the work the hot path does (every pixel is scattered, every visited
sample is evaluated).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CONFIGS = {
    # name: frames, H=W, pitch, voxel, plane raster, poses per step
    "cfg1": dict(frames=200, size=128, pitch=0.25, voxel=0.25, plane=128, batch=64),
    "cfg2": dict(frames=1000, size=512, pitch=0.125, voxel=0.25, plane=256, batch=64),
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

    @property
    def length(self) -> float:
        return (self.size - 1) * self.pitch


def workload(name: str) -> Workload:
    c = CONFIGS[name]
    return Workload(name, c["frames"], c["size"], c["pitch"], c["voxel"], c["plane"], c["batch"])


def sweep_poses(wl: Workload):
    """SweepPlan.linear(identity, Pose(I, (0,0,L)), n): slerp(I, I, t) = I exactly,
    translation (1-t)*0 + t*L."""
    from paper_2605_26325_b200.geometry import Pose, Quaternion

    n = wl.n_frames
    start = np.zeros(3)
    end = np.array([0.0, 0.0, wl.length])
    poses = []
    for k in range(n):
        t = k / (n - 1)
        poses.append(Pose(Quaternion(1.0, 0.0, 0.0, 0.0), (1.0 - t) * start + t * end))
    ts = np.arange(n, dtype=float) / 30.0
    return poses, ts


def render_frames_torch(wl: Workload, device="cuda", seed=7):
    """(n, H, W) u8 frames on the device: background 24, three spheres, speckle."""
    import torch

    n, s, p = wl.n_frames, wl.size, wl.pitch
    L = wl.length
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.arange(s, device=device, dtype=torch.float32) * p
    x = u[None, :].expand(s, s)
    y = u[:, None].expand(s, s)
    centers = [(0.3 * L, 0.4 * L, 0.35 * L, 0.12 * L, 200.0), (0.65 * L, 0.55 * L, 0.6 * L, 0.15 * L, 140.0),
               (0.5 * L, 0.3 * L, 0.8 * L, 0.08 * L, 255.0)]
    frames = torch.empty((n, s, s), dtype=torch.uint8, device=device)
    chunk = 64
    for k0 in range(0, n, chunk):
        k1 = min(n, k0 + chunk)
        z = (torch.arange(k0, k1, device=device, dtype=torch.float32) / (n - 1) * L)[:, None, None]
        val = torch.full((k1 - k0, s, s), 24.0, device=device)
        for cx, cy, cz, r, level in centers:
            inside = (x - cx) ** 2 + (y - cy) ** 2 + (z - cz) ** 2 <= r * r
            val = torch.where(inside, torch.full_like(val, level), val)
        val = val + 5.0 * torch.randn(val.shape, generator=g, device=device)
        frames[k0:k1] = val.clamp(0, 255).round().to(torch.uint8)
    return frames


def render_frames_numpy(wl: Workload, seed=7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, (wl.n_frames, wl.size, wl.size), dtype=np.uint8)


def reslice_planes(wl: Workload, count: int, seed: int = 0):
    """Appendix B planes: rotation about x by U(-10,10) deg, z = L*(0.1+0.8U)."""
    from paper_2605_26325_b200.geometry import Pose, Quaternion
    from paper_2605_26325_b200.reslice import ReslicePlane

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
