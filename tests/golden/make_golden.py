"""Generate tests/golden/golden.npz from the REAL reference implementation.

Run in the build container (where /root/reference exists):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Imports the reference package `dare` from /root/reference/pkg/src (read-only;
numba's cache is redirected) and records inputs + outputs of its hot-path
functions on small seeded cases:
  rec_*   reconstruct_volume (reconstruct.py:166-199), incl. calibration,
          slerp-interpolated poses, masks, margin 0 with out-of-bounds pixels
  seal_*  VolumeBuilder.insert_batch + seal on conftest.random_volume-style data
  rs_*    reslice + reslice_bruteforce (acceptance-criterion-1 style random cases,
          plus planes through a reconstructed sweep)
  cmp_*   compound; fill_*: fill_holes (multi-pass, random grids); tri_*: reslice_trilinear
  exp_*   math.exp (glibc) on random arguments in the weight range
The file travels with the repo; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from dare.baseline import compound, fill_holes, reslice_trilinear, ScalarVolume
    from dare.geometry import Pose, Quaternion
    from dare.reconstruct import SweepRecording, reconstruct_volume
    from dare.reslice import ReslicePlane, ResliceConfig, reslice, reslice_bruteforce
    from dare.volume import BoundingBox, VolumeBuilder

    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(20240809)

    def qdeg(axis, deg):
        return Quaternion.from_axis_angle(axis, math.radians(deg))

    def rand_q():
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        return Quaternion(*q)

    def put_sweep(key, rec, voxel, margin):
        g[f"{key}.images"] = rec.images
        g[f"{key}.image_ts"] = rec.image_timestamps
        g[f"{key}.pose_ts"] = rec.pose_timestamps
        g[f"{key}.pose_q"] = np.array([[p.rotation.w, p.rotation.x, p.rotation.y, p.rotation.z] for p in rec.poses])
        g[f"{key}.pose_t"] = np.array([p.translation for p in rec.poses])
        g[f"{key}.pitch"] = np.array(rec.pixel_pitch, dtype=float)
        c = rec.calibration
        g[f"{key}.cal_q"] = np.array([c.rotation.w, c.rotation.x, c.rotation.y, c.rotation.z])
        g[f"{key}.cal_t"] = np.asarray(c.translation, dtype=float)
        if rec.mask is not None:
            g[f"{key}.mask"] = np.asarray(rec.mask, dtype=bool)
        g[f"{key}.voxel"] = np.float64(voxel)
        g[f"{key}.margin"] = np.float64(margin)

    def put_volume(key, v):
        g[f"{key}.origin"] = np.asarray(v.origin, float)
        g[f"{key}.dims"] = np.asarray(v.dims, np.int64)
        g[f"{key}.starts"] = v.cell_starts
        g[f"{key}.counts"] = v.cell_counts
        g[f"{key}.positions"] = v.positions
        g[f"{key}.orientations"] = v.orientations
        g[f"{key}.intensities"] = v.intensities
        g[f"{key}.rejected"] = np.int64(getattr(v, "rejected_out_of_bounds", 0))

    # ---- reconstruction -------------------------------------------------
    sweeps = {}
    # (a) tilted sweep, calibration, pose stream at half the frame period -> slerp
    n, h, w = 12, 20, 24
    img = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
    its = np.arange(n) / 30.0
    pts = np.arange(2 * n + 1) / 60.0 - 1.0 / 120.0
    poses = [Pose(qdeg((1, 0.2, 0), 3.0 * k), (0.05 * k, 0.0, 0.2 * k)) for k in range(len(pts))]
    cal = Pose(qdeg((0, 0, 1), 7.0), (0.5, -0.25, 0.1))
    sweeps["rec_tilt"] = (SweepRecording(img, its, pts, poses, (0.1, 0.12), cal), 0.125, 1.0)
    # (b) mask + rotations about z, exact timestamps
    n, h, w = 5, 6, 7
    img = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
    ts = np.arange(n) / 30.0
    poses = [Pose(qdeg((0, 0, 1), 5 * k), (0.1 * k, 0, 0.2 * k)) for k in range(n)]
    mask = rng.random((h, w)) > 0.3
    sweeps["rec_mask"] = (SweepRecording(img, ts, ts, poses, (0.1, 0.1), Pose(qdeg((1, 0, 0), 2), (0.5, 0, 0)),
                                         mask), 0.25, 1.0)
    # (c) parallel sweep (test_reconstruct.py:132-152)
    n, h, w = 50, 8, 9
    img = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
    ts = np.arange(n) / 10.0
    poses = [Pose(Quaternion.identity(), (0, 0, 0.3 * k)) for k in range(n)]
    sweeps["rec_parallel"] = (SweepRecording(img, ts, ts, poses, (0.25, 0.25)), 0.25, 1.0)
    # (d) margin 0 with arbitrary rotations (f32 rounding can leave the grid)
    n, h, w = 16, 17, 19
    img = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
    ts = np.arange(n) * 0.05
    poses = [Pose(rand_q(), rng.uniform(-3, 3, 3)) for _ in range(n)]
    sweeps["rec_margin0"] = (SweepRecording(img, ts, ts, poses, (0.13, 0.07)), 0.1, 0.0)
    # (e) images outside the pose stream are dropped; negative-w poses canonicalised
    n, h, w = 8, 9, 10
    img = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
    its = np.arange(n) * 0.1
    pts = np.array([0.15, 0.32, 0.41, 0.58])
    poses = [Pose(Quaternion(-q.w, -q.x, -q.y, -q.z), rng.uniform(-1, 1, 3)) for q in (rand_q() for _ in range(4))]
    sweeps["rec_drop"] = (SweepRecording(img, its, pts, poses, (0.2, 0.2)), 0.2, 0.5)
    import hashlib
    import tempfile

    from dare.volume import save_volume

    for key, (rec, voxel, margin) in sweeps.items():
        v = reconstruct_volume(rec, voxel_size=voxel, margin=margin)
        put_sweep(key, rec, voxel, margin)
        put_volume(key + ".out", v)
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "v.darevol")
            save_volume(v, path)
            raw = open(path, "rb").read()
        g[f"{key}.darevol_sha256"] = np.array(hashlib.sha256(raw).hexdigest())
        g[f"{key}.darevol_size"] = np.int64(len(raw))
        print(key, v.dims, v.sample_count, "rejected", v.rejected_out_of_bounds)

    # ---- seal of arbitrary samples (conftest.random_volume) --------------
    seal_vols = {}
    for i, (ns, ext, vox) in enumerate([(0, 10.0, 0.5), (1, 10.0, 0.5), (3000, 10.0, 0.5), (10000, 10.0, 0.25),
                                        (5000, 10.0, 1.0), (2000, 4.0, 2.5)]):
        key = f"seal_{i}"
        b = VolumeBuilder(BoundingBox((0, 0, 0), (ext, ext, ext)), vox)
        pos = rng.uniform(0, ext, size=(ns, 3))
        if ns > 10:
            pos[:5] = rng.uniform(ext, ext + 2.0, size=(5, 3))  # out of bounds
        quats = rng.normal(size=(ns, 4))
        quats /= np.linalg.norm(quats, axis=1, keepdims=True)
        quats[quats[:, 0] < 0] *= -1.0
        inten = rng.integers(0, 256, ns)
        b.insert_batch(pos, quats, inten)
        v = b.seal()
        v.rejected_out_of_bounds = b.rejected_out_of_bounds
        g[f"{key}.bounds"] = np.array([0, 0, 0, ext, ext, ext], float)
        g[f"{key}.voxel"] = np.float64(vox)
        g[f"{key}.in_pos"] = pos
        g[f"{key}.in_quat"] = quats
        g[f"{key}.in_inten"] = inten
        put_volume(key + ".out", v)
        seal_vols[key] = v

    # ---- reslice --------------------------------------------------------
    def put_case(key, vol_key, plane, cfg, fast, brute):
        q = plane.pose.rotation
        g[f"{key}.vol"] = np.array(vol_key)
        g[f"{key}.plane_q"] = np.array([q.w, q.x, q.y, q.z])
        g[f"{key}.plane_t"] = np.asarray(plane.pose.translation, float)
        g[f"{key}.plane_wh"] = np.array([plane.width, plane.height], np.int64)
        g[f"{key}.plane_pitch"] = np.array(plane.pixel_pitch, float)
        g[f"{key}.cfg"] = np.array([cfg.interp_radius, cfg.normal_threshold_deg, cfg.inplane_threshold_deg,
                                    cfg.k_normal, cfg.k_inplane, cfg.k_dist, cfg.unassigned_value], float)
        g[f"{key}.pixels"] = fast.pixels
        g[f"{key}.coverage"] = fast.coverage
        if brute is not None:
            g[f"{key}.brute_pixels"] = brute.pixels
            g[f"{key}.brute_coverage"] = brute.coverage

    case = 0
    for vol_key in ("seal_2", "seal_3", "seal_4", "seal_5"):
        vol = seal_vols[vol_key]
        for _ in range(6):
            plane = ReslicePlane(Pose(rand_q(), rng.uniform(-1, 11, 3)), int(rng.integers(4, 25)),
                                 int(rng.integers(4, 25)), (float(rng.uniform(0.1, 0.6)),) * 2)
            cfg = ResliceConfig(interp_radius=float(rng.uniform(0.15, 1.5)),
                                normal_threshold_deg=float(rng.uniform(5, 85)),
                                inplane_threshold_deg=float(rng.uniform(5, 85)),
                                k_normal=float(rng.uniform(0, 20)), k_inplane=float(rng.uniform(0, 10)),
                                k_dist=float(rng.choice([0.0, 1.0, 2.0, 4.0])),
                                unassigned_value=int(rng.integers(0, 256)))
            put_case(f"rs_{case}", vol_key, plane, cfg, reslice(vol, plane, cfg), reslice_bruteforce(vol, plane, cfg))
            case += 1
    # planes through a reconstructed sweep (power-of-two radius -> reciprocal path)
    rec, voxel, margin = sweeps["rec_tilt"]
    v = reconstruct_volume(rec, voxel_size=voxel, margin=margin)
    for k in range(6):
        q = qdeg((1, 0, 0), float(rng.uniform(-10, 10)))
        plane = ReslicePlane(Pose(q, (0.2, 0.1, 0.2 * (k + 2))), 26, 22, (0.1, 0.1))
        for cfg in (ResliceConfig(interp_radius=0.125), ResliceConfig(interp_radius=0.25, k_dist=0.0),
                    ResliceConfig(interp_radius=0.3, normal_threshold_deg=30.0)):
            put_case(f"rs_{case}", "rec_tilt.out", plane, cfg, reslice(v, plane, cfg), None)
            case += 1
    g["rs.count"] = np.int64(case)

    # ---- scalar arm -----------------------------------------------------
    for key in ("rec_tilt", "rec_mask", "rec_parallel", "rec_margin0"):
        rec, voxel, margin = sweeps[key]
        s = compound(rec, voxel_size=voxel, margin=margin)
        g[f"cmp_{key}.values"] = s.values
        g[f"cmp_{key}.flags"] = s.flags
        g[f"cmp_{key}.counts"] = s.counts
        g[f"cmp_{key}.origin"] = s.origin
        g[f"cmp_{key}.dims"] = np.asarray(s.dims, np.int64)
    for i, (shape, p_obs, passes) in enumerate([((7, 1, 1), None, 3), ((9, 8, 7), 0.15, 3), ((12, 5, 9), 0.05, 5),
                                                ((6, 6, 6), 0.5, 1), ((5, 5, 5), 1.0, 3), ((10, 3, 4), 0.02, 0)]):
        if p_obs is None:
            vals = np.zeros(shape)
            flags = np.zeros(shape, np.uint8)
            for x, val in ((0, 0.0), (1, 0.0), (5, 90.0), (6, 90.0)):
                vals[x] = val
                flags[x] = 1
        else:
            vals = rng.uniform(0, 255, shape)
            flags = (rng.random(shape) < p_obs).astype(np.uint8)
            vals[flags == 0] = 0.0
        sv = ScalarVolume((0.5, -1.0, 2.0), 0.5, shape, vals.astype(np.float32).reshape(-1), flags.reshape(-1))
        out = fill_holes(sv, max_passes=passes)
        g[f"fill_{i}.in_values"] = sv.values
        g[f"fill_{i}.in_flags"] = sv.flags
        g[f"fill_{i}.dims"] = np.asarray(shape, np.int64)
        g[f"fill_{i}.passes"] = np.int64(passes)
        g[f"fill_{i}.values"] = out.values
        g[f"fill_{i}.flags"] = out.flags
        # trilinear through the filled grid
        for j in range(3):
            plane = ReslicePlane(Pose(rand_q(), rng.uniform(-1.0, 4.0, 3)), int(rng.integers(3, 17)),
                                 int(rng.integers(3, 17)), (float(rng.uniform(0.05, 0.4)),) * 2)
            r = reslice_trilinear(out, plane)
            key = f"tri_{i}_{j}"
            q = plane.pose.rotation
            g[f"{key}.plane_q"] = np.array([q.w, q.x, q.y, q.z])
            g[f"{key}.plane_t"] = np.asarray(plane.pose.translation, float)
            g[f"{key}.plane_wh"] = np.array([plane.width, plane.height], np.int64)
            g[f"{key}.plane_pitch"] = np.array(plane.pixel_pitch, float)
            g[f"{key}.pixels"] = r.pixels
            g[f"{key}.coverage"] = r.coverage
    g["fill.count"] = np.int64(6)

    # ---- glibc exp --------------------------------------------------------
    x = np.concatenate([-rng.uniform(0, 60, 20000), -rng.uniform(0, 1e-3, 2000),
                        rng.uniform(-800, 800, 2000), np.array([0.0, -0.0, -745.2, -708.5, 709.7, -1e-300])])
    g["exp.x"] = x
    g["exp.y"] = np.array([math.exp(v) if v < 709.78 else float("inf") for v in x])

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
