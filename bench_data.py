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
walk with 0.2 deg steps).  Image content is the reference's benchmark phantom
(phantom.py:402-467 default_benchmark_scene: vessels, sphere, two-sided slab,
speckle seed 7 amplitude 5), render_intensities (phantom.py:113-152) restated
in torch f64 on the GPU with numpy's own per-frame speckle streams -- the
reference's CPU renderer takes ~2 min for cfg2 and ~16 min for cfg3.
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


# ---------------------------------------------------------------- phantom content
# The reference's benchmark scene (phantom.py:402-467 default_benchmark_scene,
# seed 7, speckle 5): background 24, specular exponent 4, two vessel tubes, a
# sphere and a tilted two-sided reflector slab (scene_from_dict, phantom.py:308-348).
_W96, _P96 = 96, 0.25
_CX = 0.5 * (_W96 - 1) * _P96
_DEPTH = (_W96 - 1) * _P96
_SWEEP_LEN = 28.0
SCENE = dict(
    background=24.0, specular=4.0, speckle=5.0, seed=7,
    inclusions=[
        ("tube", dict(point=(_CX, 0.45 * _DEPTH, 0.0), direction=(0.0, 0.0, 1.0), radius=4.2, intensity=195.0,
                      back=None, wall=0.9)),
        ("tube", dict(point=(_CX - 6.5, 0.72 * _DEPTH, 0.0), direction=(0.2, 0.0, 1.0), radius=2.4,
                      intensity=165.0, back=None, wall=0.8)),
        ("sphere", dict(center=(_CX + 6.0, 0.3 * _DEPTH, 0.45 * _SWEEP_LEN), radius=3.4, intensity=225.0,
                        back=None, wall=0.9)),
        ("slab", dict(point=(_CX, 0.9 * _DEPTH, 0.0), normal=(0.0, -1.0, 0.15), intensity=90.0, back=190.0,
                      wall=0.8)),
    ],
)


def frame_keys(wl: Workload) -> np.ndarray:
    """phantom.simulate_sweep seeds speckle with frame_key = index within its
    sweep (phantom.py:226-231); merge_recordings concatenates sweeps."""
    per = wl.n_frames // wl.sweeps
    return np.concatenate([np.arange(per) for _ in range(wl.sweeps)])


def speckle(key: int, shape, scene=SCENE) -> np.ndarray:
    """The reference's per-frame speckle stream (phantom.py:149-151)."""
    rng = np.random.default_rng((scene["seed"], int(key)))
    return rng.normal(0.0, scene["speckle"], shape)


def _norm3(x, y, z, torch):
    return torch.sqrt((x * x + y * y) + z * z)


def render_phantom(poses, width: int, height: int, pitch, keys, device="cuda", scene=SCENE, noise=True,
                   threads: int = 0):
    """(n, H, W) u8 frames: phantom.render_intensities (phantom.py:113-152) for
    `poses` restated with torch in f64 on `device` (same expressions and
    evaluation order; the speckle is numpy's own per-frame generator, drawn on
    host threads).  Equal to the reference's frames except where an f64
    rounding difference (pow / dot order) moves a value across a rint tie
    (tests/test_bench_phantom.py measures it)."""
    import concurrent.futures
    import os

    import torch

    from paper_2605_26325_b200.geometry import rotation_matrix

    n = len(poses)
    px, py = pitch
    f64 = dict(dtype=torch.float64, device=device)
    u = torch.arange(width, **f64) * px
    v = torch.arange(height, **f64) * py
    out = torch.empty((n, height, width), dtype=torch.uint8, device=device)
    prims = []
    for kind, a in scene["inclusions"]:
        if kind == "tube":
            d = np.asarray(a["direction"], dtype=float)
            d = d / np.linalg.norm(d)
            prims.append((kind, np.asarray(a["point"], float), d, a))
        elif kind == "sphere":
            prims.append((kind, np.asarray(a["center"], float), None, a))
        else:
            nn = np.asarray(a["normal"], dtype=float)
            nn = nn / np.linalg.norm(nn)
            prims.append((kind, np.asarray(a["point"], float), nn, a))
    pool = concurrent.futures.ThreadPoolExecutor(threads or min(32, os.cpu_count() or 1)) if noise else None
    chunk = 32
    try:
        pending = None
        if noise:
            pending = [pool.submit(speckle, int(keys[i]), (height, width), scene) for i in range(min(chunk, n))]
        for k0 in range(0, n, chunk):
            k1 = min(n, k0 + chunk)
            nxt = None
            if noise and k1 < n:
                nxt = [pool.submit(speckle, int(keys[i]), (height, width), scene)
                       for i in range(k1, min(n, k1 + chunk))]
            R = torch.tensor(np.array([rotation_matrix(p.rotation) for p in poses[k0:k1]]), **f64)
            T = torch.tensor(np.array([p.translation for p in poses[k0:k1]], dtype=float), **f64)
            xa, ya = R[:, :, 0], R[:, :, 1]  # frame_axes: x = R[:,0], y = R[:,1] (= beam)
            # pts = (u * x_axis + v * y_axis) + t, per component
            P = [(u[None, None, :] * xa[:, c, None, None] + v[None, :, None] * ya[:, c, None, None])
                 + T[:, c, None, None] for c in range(3)]
            img = torch.full((k1 - k0, height, width), float(scene["background"]), **f64)
            for kind, anchor, d, a in prims:
                rel = [P[c] - float(anchor[c]) for c in range(3)]
                if kind == "sphere":
                    dist = _norm3(*rel, torch)
                    safe = torch.clamp(dist, min=1e-9)
                    nrm = [rel[c] / safe for c in range(3)]
                    shell = torch.abs(dist - a["radius"]) <= 0.5 * a["wall"]
                elif kind == "tube":
                    axial = (rel[0] * d[0] + rel[1] * d[1]) + rel[2] * d[2]
                    radial = [rel[c] - axial * d[c] for c in range(3)]
                    dist = _norm3(*radial, torch)
                    safe = torch.clamp(dist, min=1e-9)
                    nrm = [radial[c] / safe for c in range(3)]
                    shell = torch.abs(dist - a["radius"]) <= 0.5 * a["wall"]
                else:
                    off = (rel[0] * d[0] + rel[1] * d[1]) + rel[2] * d[2]
                    shell = torch.abs(off) <= 0.5 * a["wall"]
                    nrm = [torch.full_like(off, float(d[c])) for c in range(3)]
                cos_t = (nrm[0] * ya[:, 0, None, None] + nrm[1] * ya[:, 1, None, None]) + nrm[2] * ya[:, 2, None, None]
                back = a["intensity"] if a["back"] is None else a["back"]
                wall = torch.where(cos_t < 0.0, torch.full_like(cos_t, a["intensity"]), torch.full_like(cos_t, back))
                c2 = cos_t * cos_t
                img = img + (shell.to(torch.float64) * wall) * (c2 * c2 if scene["specular"] == 4.0
                                                               else torch.abs(cos_t) ** scene["specular"])
            if noise:
                img = img + torch.from_numpy(np.stack([f.result() for f in pending])).to(device)
            out[k0:k1] = torch.clamp(torch.round(img), 0, 255).to(torch.uint8)
            pending = nxt
    finally:
        if pool is not None:
            pool.shutdown(wait=True)
    return out


def render_frames_torch(wl: Workload, device="cuda"):
    """(n, H, W) u8 frames of the workload's sweep(s): the reference's benchmark
    phantom (default_benchmark_scene, seed 7, speckle 5) rendered at every frame pose."""
    poses, _ = sweep_poses(wl)
    return render_phantom(poses, wl.size, wl.size, (wl.pitch, wl.pitch), frame_keys(wl), device=device)


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
