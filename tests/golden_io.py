"""Access to tests/golden/golden.npz (outputs of the real reference, see
tests/golden/make_golden.py) as objects of this package."""
from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig
from paper_2605_26325_b200.sweep import SweepRecording

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")

REC_KEYS = ("rec_tilt", "rec_mask", "rec_parallel", "rec_margin0", "rec_drop")
SEAL_KEYS = tuple(f"seal_{i}" for i in range(6))


class Golden:
    def __init__(self):
        self.z = np.load(PATH, allow_pickle=False)

    def __getitem__(self, k):
        return self.z[k]

    def has(self, k) -> bool:
        return k in self.z.files

    def sweep(self, key):
        g = self.z
        poses = [Pose(Quaternion(*q), t) for q, t in zip(g[f"{key}.pose_q"], g[f"{key}.pose_t"])]
        cal = Pose(Quaternion(*g[f"{key}.cal_q"]), g[f"{key}.cal_t"])
        mask = g[f"{key}.mask"] if self.has(f"{key}.mask") else None
        rec = SweepRecording(g[f"{key}.images"], g[f"{key}.image_ts"], g[f"{key}.pose_ts"], poses,
                             tuple(float(x) for x in g[f"{key}.pitch"]), cal, mask)
        return rec, float(g[f"{key}.voxel"]), float(g[f"{key}.margin"])

    def volume(self, key):
        """Reference-layout arrays of a stored volume (key = 'rec_tilt.out', 'seal_3.out', ...)."""
        g = self.z
        return SimpleNamespace(
            origin=g[f"{key}.origin"], voxel_size=None, dims=tuple(int(d) for d in g[f"{key}.dims"]),
            cell_starts=g[f"{key}.starts"], cell_counts=g[f"{key}.counts"], positions=g[f"{key}.positions"],
            orientations=g[f"{key}.orientations"], intensities=g[f"{key}.intensities"],
            rejected_out_of_bounds=int(g[f"{key}.rejected"]))

    def volume_voxel(self, vol_key) -> float:
        base = vol_key.split(".")[0]
        return float(self.z[f"{base}.voxel"])

    def full_volume(self, vol_key):
        v = self.volume(vol_key)
        v.voxel_size = self.volume_voxel(vol_key)
        return v

    def reslice_cases(self):
        for i in range(int(self.z["rs.count"])):
            yield i, self.reslice_case(i)

    def reslice_case(self, i):
        g, k = self.z, f"rs_{i}"
        c = g[f"{k}.cfg"]
        cfg = ResliceConfig(float(c[0]), float(c[1]), float(c[2]), float(c[3]), float(c[4]), float(c[5]),
                            int(c[6]))
        w, h = (int(x) for x in g[f"{k}.plane_wh"])
        plane = ReslicePlane(Pose(Quaternion(*g[f"{k}.plane_q"]), g[f"{k}.plane_t"]), w, h,
                             tuple(float(x) for x in g[f"{k}.plane_pitch"]))
        brute = (g[f"{k}.brute_pixels"], g[f"{k}.brute_coverage"]) if self.has(f"{k}.brute_pixels") else None
        vol_key = str(g[f"{k}.vol"])
        if not vol_key.endswith(".out"):
            vol_key += ".out"
        return SimpleNamespace(vol_key=vol_key, plane=plane, cfg=cfg, pixels=g[f"{k}.pixels"],
                               coverage=g[f"{k}.coverage"], brute=brute)

    def trilinear_plane(self, key):
        g = self.z
        w, h = (int(x) for x in g[f"{key}.plane_wh"])
        return ReslicePlane(Pose(Quaternion(*g[f"{key}.plane_q"]), g[f"{key}.plane_t"]), w, h,
                            tuple(float(x) for x in g[f"{key}.plane_pitch"]))
