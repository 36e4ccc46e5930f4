"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Python front-end of liboracle.so (dare_oracle.c): a restatement of the
reference's hot path (arxiv/paper_2605_26325, pkg/src/dare/) used to check the
CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs may import this module; the product package never does.

The host pose pipeline here is a deliberately independent, scalar,
frame-by-frame restatement (reconstruct.py:102-149 synchronize /
interpolate_pose, geometry.py:69-133 quaternion product / rotate / compose,
volume.py:57-73 compute_bounds, volume.py:197-206 grid sizing), so that the
product's vectorised version is checked against it rather than against
itself.  Everything is pinned to outputs of the real reference by
tests/test_oracle_golden.py (fixtures: tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None

_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_p = ctypes.c_void_p


def build() -> str:
    src = os.path.join(HERE, "dare_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB_PATH)
        sig = {
            "oracle_frame_cells": [_i32, _i32, _f64, _f64, _p, _p, _p, _p, _f64, _p, _p, _p],
            "oracle_seal": [_i64, _p, _i64, _p, _p, _p],
            "oracle_reslice_grid": [_p, _p, _i32, _i32, _p, _p, _f64, _p, _p, _p, _p, _p, _p, _p, _i32],
            "oracle_reslice_bruteforce": [_p, _p, _i32, _i32, _p, _i64, _p, _p, _p, _p, _i32],
            "oracle_trilinear": [_p, _p, _p, _i32, _i32, _p, _p, _f64, _p, _p, _p],
            "oracle_compound_frame": [_i32, _i32, _f64, _f64, _p, _p, _p, _p, _f64, _p, _p, _p, _p, _p],
            "oracle_compound_finalize": [_i64, _p, _p, _p, _p],
            "oracle_fill_holes": [_p, _p, _p, _i32],
            "oracle_exp": [_i64, _p, _p],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int32 if name == "oracle_fill_holes" else None
        _lib = lib
    return _lib


def _a(x):
    return None if x is None else x.ctypes.data


# ---------------------------------------------------------------- host poses

def _qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return (aw * bw - ax * bx - ay * by - az * bz,
            aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx,
            aw * bz + ax * by - ay * bx + az * bw)


def _qnorm(q):
    return math.sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3])


def _rot(q, v):
    u = np.array([q[1], q[2], q[3]])
    v = np.asarray(v, dtype=float)
    t = 2.0 * np.cross(u, v)
    return v + q[0] * t + np.cross(u, t)


def _rmat(q):
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def _slerp(q0, q1, t):
    a, b = np.array(q0, dtype=float), np.array(q1, dtype=float)
    dot = float(np.dot(a, b))
    if dot < 0.0:
        b, dot = -b, -dot
    if dot > 0.9995:
        out = a + t * (b - a)
        out = out / np.linalg.norm(out)
        return tuple(out)
    th = math.acos(min(1.0, dot))
    s = math.sin(th)
    out = (math.sin((1.0 - t) * th) / s) * a + (math.sin(t * th) / s) * b
    return tuple(out / np.linalg.norm(out))


def _quat_of(p):
    r = p.rotation
    return (r.w, r.x, r.y, r.z)


@dataclass
class OracleFrame:
    image: int
    quat: tuple  # normalized image-plane rotation (w, x, y, z)
    trans: np.ndarray


def frame_poses(sweep) -> list[OracleFrame]:
    ts = np.asarray(sweep.pose_timestamps, dtype=float)
    cal_q, cal_t = _quat_of(sweep.calibration), np.asarray(sweep.calibration.translation, float)
    out = []
    for k, t in enumerate(np.asarray(sweep.image_timestamps, dtype=float)):
        t = float(t)
        if t < ts[0] or t > ts[-1]:
            continue
        i = int(np.searchsorted(ts, t, side="right")) - 1
        if i == len(sweep.poses) - 1 or ts[i] == t:
            mq, mt = _quat_of(sweep.poses[i]), np.asarray(sweep.poses[i].translation, float)
        else:
            t0, t1 = ts[i], ts[i + 1]
            al = 0.0 if t1 == t0 else (t - t0) / (t1 - t0)
            p0, p1 = sweep.poses[i], sweep.poses[i + 1]
            mq = _slerp(_quat_of(p0), _quat_of(p1), al)
            mt = (1.0 - al) * np.asarray(p0.translation, float) + al * np.asarray(p1.translation, float)
        prod = _qmul(mq, cal_q)
        n = _qnorm(prod)
        q = (prod[0] / n, prod[1] / n, prod[2] / n, prod[3] / n)
        out.append(OracleFrame(k, q, _rot(mq, cal_t) + mt))
    if not out:
        raise ValueError("no image falls inside the pose stream time range")
    return out


def grid(frames, width, height, pitch, voxel, margin):
    px, py = pitch
    lo, hi = np.full(3, np.inf), np.full(3, -np.inf)
    umax, vmax = (width - 1) * px, (height - 1) * py
    for f in frames:
        for u, v in ((0.0, 0.0), (umax, 0.0), (0.0, vmax), (umax, vmax)):
            c = _rot(f.quat, (u, v, 0.0)) + f.trans
            lo, hi = np.minimum(lo, c), np.maximum(hi, c)
    lo, hi = lo - margin, hi + margin
    if margin == 0.0 and np.all(hi - lo == 0.0):
        raise ValueError("degenerate bounds")
    dims = tuple(int(np.floor(e / voxel)) + 1 for e in (hi - lo))
    return lo.copy(), float(voxel), dims


def _canon32(q):
    w, x, y, z = q
    if w < 0.0 or (w == 0.0 and (x < 0.0 or (x == 0.0 and (y < 0.0 or (y == 0.0 and z < 0.0))))):
        q = (-w, -x, -y, -z)
    return np.array(q, dtype=np.float32)


# ---------------------------------------------------------------- volumes

@dataclass
class OracleVolume:
    origin: np.ndarray
    voxel_size: float
    dims: tuple
    cell_starts: np.ndarray
    cell_counts: np.ndarray
    positions: np.ndarray
    orientations: np.ndarray
    intensities: np.ndarray
    rejected_out_of_bounds: int = 0


def frame_cells(frame: OracleFrame, width, height, pitch, origin, voxel, dims):
    lib = load()
    r = _rmat(frame.quat)
    c0, c1 = np.ascontiguousarray(r[:, 0]), np.ascontiguousarray(r[:, 1])
    t = np.ascontiguousarray(frame.trans, dtype=np.float64)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    lin = np.empty(width * height, np.int64)
    pos = np.empty((width * height, 3), np.float32)
    lib.oracle_frame_cells(height, width, pitch[0], pitch[1], _a(c0), _a(c1), _a(t), _a(o), voxel,
                           _a(d), _a(lin), _a(pos))
    return lin, pos


def seal(origin, voxel, dims, lin, pos, quat, inten) -> OracleVolume:
    lib = load()
    nc = int(np.prod(dims))
    n = len(lin)
    counts, starts, order = np.empty(nc, np.int64), np.empty(nc, np.int64), np.empty(n, np.int64)
    lin = np.ascontiguousarray(lin, dtype=np.int64)
    lib.oracle_seal(n, _a(lin), nc, _a(counts), _a(starts), _a(order))
    return OracleVolume(np.asarray(origin, float), float(voxel), tuple(dims), starts, counts,
                        np.ascontiguousarray(pos[order]), np.ascontiguousarray(quat[order]),
                        np.ascontiguousarray(inten[order]))


def reconstruct(sweep, voxel_size=0.125, margin=1.0) -> OracleVolume:
    """reconstruct_volume (reconstruct.py:166-199)."""
    images = np.asarray(sweep.images, dtype=np.uint8)
    _, h, w = images.shape
    frames = frame_poses(sweep)
    origin, voxel, dims = grid(frames, w, h, sweep.pixel_pitch, voxel_size, margin)
    mask = None if sweep.mask is None else np.asarray(sweep.mask, bool).reshape(-1)
    lins, poss, quats, ints, rejected = [], [], [], [], 0
    for f in frames:
        lin, pos = frame_cells(f, w, h, sweep.pixel_pitch, origin, voxel, dims)
        inten = images[f.image].reshape(-1)
        if mask is not None:
            lin, pos, inten = lin[mask], pos[mask], inten[mask]
        ok = lin >= 0
        rejected += int(np.count_nonzero(~ok))
        lins.append(lin[ok])
        poss.append(pos[ok])
        ints.append(inten[ok])
        quats.append(np.broadcast_to(_canon32(f.quat), (int(ok.sum()), 4)))
    vol = seal(origin, voxel, dims, np.concatenate(lins), np.concatenate(poss), np.concatenate(quats),
               np.concatenate(ints))
    vol.rejected_out_of_bounds = rejected
    return vol


def reconstruct_subset(sweep, frames: list[OracleFrame], origin, voxel, dims) -> OracleVolume:
    """Slab oracle: reconstruct only `frames` (a subset of
    frame_poses(sweep), in order) into the FULL grid.  Every cell whose
    contributing frames are all in the subset is identical to the full
    reconstruction, so a reslice that only visits such cells is exact."""
    images = sweep.images
    _, h, w = images.shape
    lins, poss, quats, ints = [], [], [], []
    for f in frames:
        lin, pos = frame_cells(f, w, h, sweep.pixel_pitch, origin, voxel, dims)
        inten = np.asarray(images[f.image]).reshape(-1)
        ok = lin >= 0
        lins.append(lin[ok])
        poss.append(pos[ok])
        ints.append(inten[ok])
        quats.append(np.broadcast_to(_canon32(f.quat), (int(ok.sum()), 4)))
    return seal(origin, voxel, dims, np.concatenate(lins), np.concatenate(poss), np.concatenate(quats),
                np.concatenate(ints))


def cell_records(sweep, origin, voxel, dims, cells):
    """Slab oracle: the exact sample list of each cell in
    `cells`, in the reference's insertion order (synchronized frame order, then
    row-major pixels; volume.py:240-256), streamed frame by frame through the
    same frame_cells restatement -- no full volume is built.  Returns
    {cell: (positions f32 (k,3), quaternions f32 (k,4), intensities u8 (k))}."""
    images = sweep.images
    _, h, w = images.shape
    nc = int(np.prod(dims))
    lut = np.zeros(nc, dtype=bool)
    cells = np.asarray(cells, dtype=np.int64)
    lut[cells] = True
    parts = {int(c): ([], [], []) for c in cells}
    for f in frame_poses(sweep):
        lin, pos = frame_cells(f, w, h, sweep.pixel_pitch, origin, voxel, dims)
        ok = lin >= 0
        hit = np.zeros_like(ok)
        hit[ok] = lut[lin[ok]]
        if not hit.any():
            continue
        img = np.asarray(images[f.image]).reshape(-1)
        q = _canon32(f.quat)
        for i in np.nonzero(hit)[0]:  # row-major pixel order
            p = parts[int(lin[i])]
            p[0].append(pos[i])
            p[1].append(q)
            p[2].append(img[i])
    out = {}
    for c, (ps, qs, its) in parts.items():
        out[c] = (np.array(ps, np.float32).reshape(-1, 3), np.array(qs, np.float32).reshape(-1, 4),
                  np.array(its, np.uint8))
    return out


def seal_samples(origin, voxel, dims, positions, orientations, intensities) -> OracleVolume:
    """VolumeBuilder.insert_batch + seal (volume.py:223-269) for arbitrary samples."""
    pos = np.ascontiguousarray(positions, dtype=np.float32).reshape(-1, 3)
    quat = np.ascontiguousarray(orientations, dtype=np.float32).reshape(-1, 4)
    inten = np.ascontiguousarray(intensities, dtype=np.uint8).reshape(-1)
    idx = np.floor((pos.astype(np.float64) - np.asarray(origin, float)) / voxel).astype(np.int64)
    ok = np.all((idx >= 0) & (idx < np.asarray(dims)), axis=1)
    idx = idx[ok]
    lin = (idx[:, 0] * dims[1] + idx[:, 1]) * dims[2] + idx[:, 2]
    vol = seal(origin, voxel, dims, lin, pos[ok], quat[ok], inten[ok])
    vol.rejected_out_of_bounds = int(np.count_nonzero(~ok))
    return vol


# ---------------------------------------------------------------- reslice

def plane_params(plane) -> np.ndarray:
    q = _quat_of(plane.pose)
    r = _rmat(q)
    t = np.asarray(plane.pose.translation, float)
    return np.array([t[0], t[1], t[2], r[0, 0], r[0, 1], r[0, 2], r[1, 0], r[1, 1], r[1, 2],
                     r[2, 0], r[2, 1], r[2, 2], plane.pixel_pitch[0], plane.pixel_pitch[1]], dtype=np.float64)


def cfg_array(cfg) -> np.ndarray:
    return np.array([cfg.interp_radius, math.cos(math.radians(cfg.normal_threshold_deg)),
                     math.cos(math.radians(cfg.inplane_threshold_deg)), cfg.k_normal, cfg.k_inplane,
                     cfg.k_dist], dtype=np.float64)


def reslice(vol, params, cfg, width, height, unassigned=0, brute=False):
    """reslice_rows_grid / reslice_rows_bruteforce for one plane -> (pixels, coverage)."""
    lib = load()
    out = np.empty((height, width), np.uint8)
    cov = np.empty((height, width), np.uint8)
    p = np.ascontiguousarray(params, dtype=np.float64)
    c = np.ascontiguousarray(cfg, dtype=np.float64)
    pos = np.ascontiguousarray(vol.positions, dtype=np.float32)
    quat = np.ascontiguousarray(vol.orientations, dtype=np.float32)
    inten = np.ascontiguousarray(vol.intensities, dtype=np.uint8)
    if brute:
        lib.oracle_reslice_bruteforce(_a(out), _a(cov), height, width, _a(p), len(inten), _a(pos),
                                      _a(quat), _a(inten), _a(c), int(unassigned))
    else:
        o = np.ascontiguousarray(vol.origin, dtype=np.float64)
        d = np.ascontiguousarray(vol.dims, dtype=np.int64)
        st = np.ascontiguousarray(vol.cell_starts, dtype=np.int64)
        ct = np.ascontiguousarray(vol.cell_counts, dtype=np.int64)
        lib.oracle_reslice_grid(_a(out), _a(cov), height, width, _a(p), _a(o), float(vol.voxel_size),
                                _a(d), _a(st), _a(ct), _a(pos), _a(quat), _a(inten), _a(c), int(unassigned))
    return out, cov.astype(bool)


# ---------------------------------------------------------------- scalar arm

def compound(sweep, voxel_size=0.125, margin=1.0):
    """compound (baseline.py:64-97) -> (origin, voxel, dims, values, flags, counts)."""
    lib = load()
    images = np.asarray(sweep.images, dtype=np.uint8)
    _, h, w = images.shape
    frames = frame_poses(sweep)
    origin, voxel, dims = grid(frames, w, h, sweep.pixel_pitch, voxel_size, margin)
    nc = int(np.prod(dims))
    sums, counts = np.zeros(nc, np.int64), np.zeros(nc, np.int64)
    mask = None if sweep.mask is None else np.ascontiguousarray(np.asarray(sweep.mask, bool).reshape(-1).astype(np.uint8))
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    for f in frames:
        r = _rmat(f.quat)
        c0, c1 = np.ascontiguousarray(r[:, 0]), np.ascontiguousarray(r[:, 1])
        t = np.ascontiguousarray(f.trans, dtype=np.float64)
        px = np.ascontiguousarray(images[f.image])
        lib.oracle_compound_frame(h, w, sweep.pixel_pitch[0], sweep.pixel_pitch[1], _a(c0), _a(c1), _a(t),
                                  _a(o), voxel, _a(d), _a(px), _a(mask), _a(sums), _a(counts))
    values, flags = np.empty(nc, np.float32), np.empty(nc, np.uint8)
    lib.oracle_compound_finalize(nc, _a(sums), _a(counts), _a(values), _a(flags))
    return origin, voxel, dims, values, flags, counts


def fill_holes(values, flags, dims, max_passes=3):
    """fill_holes (baseline.py:100-127) -> (values f32, flags u8)."""
    lib = load()
    v = np.ascontiguousarray(values, dtype=np.float32).astype(np.float64)
    f = np.ascontiguousarray(flags, dtype=np.uint8).copy()
    d = np.ascontiguousarray(dims, dtype=np.int64)
    lib.oracle_fill_holes(_a(v), _a(f), _a(d), int(max_passes))
    return v.astype(np.float32), f


def trilinear(origin, voxel, dims, values, flags, params, width, height):
    """reslice_trilinear (baseline.py:130-155) -> (pixels, coverage, values f64)."""
    lib = load()
    out, cov = np.empty((height, width), np.uint8), np.empty((height, width), np.uint8)
    val = np.empty((height, width), np.float64)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    p = np.ascontiguousarray(params, dtype=np.float64)
    v = np.ascontiguousarray(values, dtype=np.float32)
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    lib.oracle_trilinear(_a(out), _a(cov), _a(val), height, width, _a(p), _a(o), float(voxel), _a(d),
                         _a(v), _a(f))
    return out, cov.astype(bool), val


def exp(x: np.ndarray) -> np.ndarray:
    lib = load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib.oracle_exp(len(x), _a(x), _a(y))
    return y


# ---------------------------------------------------------------- evaluation

def similarity(a, b, a_mask=None, b_mask=None, window=7, c1=(0.01 * 255.0) ** 2, c2=(0.03 * 255.0) ** 2):
    """evaluation.py:41-84 (ncc, ssim) for one 2-D pair -> (ncc, ssim, valid,
    status) with dare_similarity's status bits (1 < 2 valid, 2 zero variance,
    4 no complete window, 8 image smaller than the window).

    Restated in the summation order the CUDA path uses, which equals the
    reference's wherever the reference's order is fixed: window moments as row
    sums (left to right) added top to bottom -- exact for integer-valued
    images, so each window value is the reference's bit for bit; means and the
    final window mean via np.sum (numpy pairwise, = the reference's np.mean);
    the NCC dot products via np.sum of the products (the reference's np.dot is
    BLAS, whose order is host-dependent: the tests compare that to rounding)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mask = np.ones(a.shape, dtype=bool)
    for m in (a_mask, b_mask):
        if m is not None:
            mask &= np.asarray(m, dtype=bool)
    status = 0
    va, vb = a[mask], b[mask]
    n = va.size
    nc = 0.0
    if n < 2:
        status |= 1
    else:
        da = va - np.sum(va) / n
        db = vb - np.sum(vb) / n
        den = math.sqrt(float(np.sum(da * da)) * float(np.sum(db * db)))
        if den == 0.0:
            status |= 2
        else:
            nc = float(np.sum(da * db)) / den
    H, W = a.shape
    ss = 0.0
    if H < window or W < window:
        status |= 8
    else:
        HH, WW = H - window + 1, W - window + 1
        mf = mask.astype(np.float64)
        rows = [np.zeros((H, WW)) for _ in range(6)]
        for dx in range(window):
            sl = np.s_[:, dx:dx + WW]
            p, q = a[sl], b[sl]
            for k, v in enumerate((p, q, p * p, q * q, p * q, mf[sl])):
                rows[k] = rows[k] + v
        s = [np.zeros((HH, WW)) for _ in range(6)]
        for dy in range(window):
            for k in range(6):
                s[k] = s[k] + rows[k][dy:dy + HH]
        nn = float(window * window)
        norm = nn / (nn - 1.0)
        mu_a, mu_b = s[0] / nn, s[1] / nn
        var_a = norm * (s[2] / nn - mu_a * mu_a)
        var_b = norm * (s[3] / nn - mu_b * mu_b)
        cov = norm * (s[4] / nn - mu_a * mu_b)
        val = ((2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2)) / ((mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2))
        complete = s[5] == nn
        if not complete.any():
            status |= 4
        else:
            sel = val[complete]
            ss = float(np.sum(sel)) / sel.size
    return nc, ss, n, status
