"""Generate tests/golden/scale.npz: outputs of the REAL reference at BASELINE scale.

Run in the build container (where /root/reference exists; cfg2 needs ~35 GB of
RAM and ~6 min):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_scale.py [cfg1 cfg1t cfg2]

Inputs are reproducible on the GPU box without the reference: frames are
numpy `default_rng(seed).integers(0, 256, (n, H, W), uint8)` (their SHA-256 is
stored so the test can prove it regenerated the same bytes), and the frame
poses / reslice planes are stored as arrays.  Outputs are stored as SHA-256
hashes (the arrays themselves are GBs at cfg2):

  <cfg>.darevol_sha256   save_volume(reconstruct_volume(...)) bytes (volume.py:272-297)
  <cfg>.rs_pix / rs_cov  per-pose SHA-256 of reslice() pixels / coverage (reslice.py:168-187)
  <cfg>.cmp_*            compound() values / flags / counts (baseline.py:64-97)
  <cfg>.fill_*           fill_holes(compound(sparse sweep), 3) (baseline.py:100-127)
  <cfg>.tri_pix/tri_cov  reslice_trilinear() on the filled sparse grid (baseline.py:130-155)

Configs (SURVEY.md Appendix B geometry):
  cfg1   200 frames 128x128, pitch 0.25, linear sweep 0 -> (0,0,31.75), voxel 0.25,
         margin 0 -> 128^3; 64 planes 128x128 (rng 0: rot x U(-10,10) deg,
         z = L(0.1 + 0.8U)); sparse = every 4th frame
  cfg1t  cfg1's frames on a TRACKED sweep: pose stream at 47 Hz (tracker rate !=
         frame rate -> slerp-interpolated frame poses, reconstruct.py:102-149)
         with a wobbling tilt and a non-identity calibration; margin 0.5
  cfg2   1000 frames 512x512, pitch 0.125, linear sweep 0 -> (0,0,63.875), voxel
         0.25, margin 0 -> 256^3; 24 planes 256x256; sparse = every 8th frame
"""
from __future__ import annotations

import gc
import hashlib
import math
import os
import sys
import tempfile
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale.npz")

SPECS = {
    "cfg1": dict(frames=200, size=128, pitch=0.25, voxel=0.25, margin=0.0, planes=64, plane=128, sparse=4,
                 seed=101, tracked=False),
    "cfg1t": dict(frames=200, size=128, pitch=0.25, voxel=0.25, margin=0.5, planes=16, plane=128, sparse=4,
                  seed=101, tracked=True),
    "cfg2": dict(frames=1000, size=512, pitch=0.125, voxel=0.25, margin=0.0, planes=24, plane=256, sparse=8,
                 seed=202, tracked=False),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def frames_for(spec) -> np.ndarray:
    """The test-side generator (tests/scale_io.py) must produce the same bytes."""
    rng = np.random.default_rng(spec["seed"])
    return rng.integers(0, 256, (spec["frames"], spec["size"], spec["size"]), dtype=np.uint8)


def main(names) -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from dare.baseline import compound, fill_holes, reslice_trilinear
    from dare.geometry import Pose, Quaternion
    from dare.phantom import SweepPlan
    from dare.reconstruct import SweepRecording, reconstruct_volume
    from dare.reslice import ReslicePlane, ResliceConfig, reslice
    from dare.volume import save_volume

    g: dict[str, np.ndarray] = {}
    if os.path.exists(OUT):
        old = np.load(OUT, allow_pickle=False)
        g.update({k: old[k] for k in old.files})
    for name in names:
        spec = SPECS[name]
        t_start = time.time()
        for k in [k for k in g if k.startswith(name + ".")]:
            del g[k]
        n, sz, pitch = spec["frames"], spec["size"], spec["pitch"]
        L = (sz - 1) * pitch
        images = frames_for(spec)
        g[f"{name}.frames_sha256"] = np.array(sha(images))
        g[f"{name}.spec"] = np.array([n, sz, pitch, spec["voxel"], spec["margin"], spec["plane"], spec["sparse"],
                                      spec["seed"]], dtype=np.float64)
        if not spec["tracked"]:
            plan = SweepPlan.linear(Pose.identity(), Pose(Quaternion.identity(), (0.0, 0.0, L)), n,
                                    width=sz, height=sz, pixel_pitch=(pitch, pitch))
            poses = list(plan.poses)
            its = np.arange(n, dtype=float) / plan.frame_rate
            pts = its.copy()
            cal = Pose.identity()
        else:
            # tracker at 47 Hz covering the frames (30 Hz), tilt wobble +-4 deg, calibration
            its = np.arange(n, dtype=float) / 30.0
            m = int(math.ceil(its[-1] * 47.0)) + 2
            pts = np.arange(m, dtype=float) / 47.0 - 0.01
            poses = []
            for k, t in enumerate(pts):
                tilt = 4.0 * math.sin(0.7 * t) + 1.5 * math.sin(2.3 * t + 0.4)
                q = Quaternion.from_axis_angle((1.0, 0.15, 0.0), math.radians(tilt))
                poses.append(Pose(q, (0.3 * math.sin(0.5 * t), 0.2 * math.cos(0.9 * t), L * t / its[-1])))
            cal = Pose(Quaternion.from_axis_angle((0.0, 0.0, 1.0), math.radians(3.0)), (0.25, -0.125, 0.5))
        rec = SweepRecording(images, its, pts, poses, (pitch, pitch), cal)
        g[f"{name}.image_ts"] = its
        g[f"{name}.pose_ts"] = np.asarray(pts, dtype=float)
        g[f"{name}.pose_q"] = np.array([[p.rotation.w, p.rotation.x, p.rotation.y, p.rotation.z] for p in poses])
        g[f"{name}.pose_t"] = np.array([p.translation for p in poses], dtype=float)
        g[f"{name}.cal_q"] = np.array([cal.rotation.w, cal.rotation.x, cal.rotation.y, cal.rotation.z])
        g[f"{name}.cal_t"] = np.asarray(cal.translation, dtype=float)

        t0 = time.time()
        vol = reconstruct_volume(rec, voxel_size=spec["voxel"], margin=spec["margin"])
        t_rec = time.time() - t0
        g[f"{name}.origin"] = np.asarray(vol.origin, dtype=float)
        g[f"{name}.dims"] = np.asarray(vol.dims, dtype=np.int64)
        g[f"{name}.n_samples"] = np.int64(vol.sample_count)
        g[f"{name}.rejected"] = np.int64(vol.rejected_out_of_bounds)
        g[f"{name}.counts_sha256"] = np.array(sha(vol.cell_counts.astype(np.int64)))
        with tempfile.TemporaryDirectory(dir="/tmp") as tmp:
            path = os.path.join(tmp, "v.darevol")
            save_volume(vol, path)
            h = hashlib.sha256()
            with open(path, "rb") as fh:
                for chunk in iter(lambda: fh.read(64 << 20), b""):
                    h.update(chunk)
            g[f"{name}.darevol_sha256"] = np.array(h.hexdigest())
            g[f"{name}.darevol_size"] = np.int64(os.path.getsize(path))
        print(name, "reconstruct", f"{t_rec:.1f}s", vol.dims, vol.sample_count, "rejected",
              vol.rejected_out_of_bounds, flush=True)

        # reslice planes (Appendix B; bench_data.reslice_planes draws in the same order)
        rng = np.random.default_rng(0)
        ppitch = L / (spec["plane"] - 1)
        pq, pt = [], []
        rs_pix, rs_cov = [], []
        cfg = ResliceConfig(interp_radius=spec["voxel"])
        planes = []
        for _ in range(spec["planes"]):
            ang = math.radians(float(rng.uniform(-10.0, 10.0)))
            z = L * (0.1 + 0.8 * float(rng.uniform()))
            q = Quaternion.from_axis_angle((1, 0, 0), ang)
            planes.append(ReslicePlane(Pose(q, (0.0, 0.0, z)), spec["plane"], spec["plane"], (ppitch, ppitch)))
            pq.append([q.w, q.x, q.y, q.z])
            pt.append([0.0, 0.0, z])
        t0 = time.time()
        for p in planes:
            img = reslice(vol, p, cfg)
            rs_pix.append(sha(img.pixels))
            rs_cov.append(sha(img.coverage))
        print(name, "reslice", f"{(time.time() - t0) / len(planes) * 1e3:.1f} ms/pose", flush=True)
        g[f"{name}.plane_q"] = np.array(pq)
        g[f"{name}.plane_t"] = np.array(pt)
        g[f"{name}.plane_pitch"] = np.float64(ppitch)
        g[f"{name}.rs_pix"] = np.array(rs_pix)
        g[f"{name}.rs_cov"] = np.array(rs_cov)
        del vol
        gc.collect()

        # scalar arm: compound of the full sweep, fill + trilinear on the sparse sweep
        t0 = time.time()
        s = compound(rec, voxel_size=spec["voxel"], margin=spec["margin"])
        g[f"{name}.cmp_values"] = np.array(sha(s.values))
        g[f"{name}.cmp_flags"] = np.array(sha(s.flags))
        g[f"{name}.cmp_counts"] = np.array(sha(s.counts.astype(np.int64)))
        g[f"{name}.cmp_observed"] = np.int64(int(np.count_nonzero(s.flags)))
        del s
        gc.collect()
        k = spec["sparse"]
        keep = np.arange(0, n, k)
        if spec["tracked"]:
            sparse = SweepRecording(images[keep], its[keep], pts, poses, (pitch, pitch), cal)
        else:
            sparse = SweepRecording(images[keep], its[keep], pts[keep], [poses[i] for i in keep], (pitch, pitch),
                                    cal)
        ss = compound(sparse, voxel_size=spec["voxel"], margin=spec["margin"])
        filled = fill_holes(ss, max_passes=3)
        g[f"{name}.sparse_observed"] = np.int64(int(np.count_nonzero(ss.flags)))
        g[f"{name}.fill_values"] = np.array(sha(filled.values))
        g[f"{name}.fill_flags"] = np.array(sha(filled.flags))
        g[f"{name}.fill_filled"] = np.int64(int(np.count_nonzero(filled.flags == 2)))
        tri_pix, tri_cov = [], []
        for p in planes:
            img = reslice_trilinear(filled, p)
            tri_pix.append(sha(img.pixels))
            tri_cov.append(sha(img.coverage))
        g[f"{name}.tri_pix"] = np.array(tri_pix)
        g[f"{name}.tri_cov"] = np.array(tri_cov)
        print(name, "scalar arm", f"{time.time() - t0:.1f}s", "filled", int(g[f"{name}.fill_filled"]),
              "total", f"{time.time() - t_start:.1f}s", flush=True)
        del ss, filled, rec, images
        gc.collect()
        np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main(sys.argv[1:] or list(SPECS))
