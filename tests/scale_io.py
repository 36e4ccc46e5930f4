"""Access to tests/golden/scale.npz (SHA-256 hashes of the REAL reference's
outputs at BASELINE scale, tests/golden/make_golden_scale.py): rebuilds the
same inputs as this package's objects, and hashes outputs the same way."""
from __future__ import annotations

import hashlib
import os

import numpy as np

from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig
from paper_2605_26325_b200.sweep import SweepRecording

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale.npz")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class HashSink:
    """Writable binary file object that only hashes (streamed .darevol bytes)."""

    def __init__(self):
        self.h = hashlib.sha256()
        self.size = 0

    def write(self, b) -> int:
        self.h.update(b)
        n = memoryview(b).nbytes
        self.size += n
        return n

    def hexdigest(self) -> str:
        return self.h.hexdigest()


class Scale:
    def __init__(self):
        self.z = np.load(PATH, allow_pickle=False)

    def has(self, name) -> bool:
        return f"{name}.darevol_sha256" in self.z.files

    def __getitem__(self, k):
        return self.z[k]

    def spec(self, name):
        s = self.z[f"{name}.spec"]
        return dict(frames=int(s[0]), size=int(s[1]), pitch=float(s[2]), voxel=float(s[3]), margin=float(s[4]),
                    plane=int(s[5]), sparse=int(s[6]), seed=int(s[7]))

    def frames(self, name) -> np.ndarray:
        sp = self.spec(name)
        rng = np.random.default_rng(sp["seed"])
        return rng.integers(0, 256, (sp["frames"], sp["size"], sp["size"]), dtype=np.uint8)

    def sweep(self, name, images=None, every: int = 1):
        z, sp = self.z, self.spec(name)
        images = self.frames(name) if images is None else images
        poses = [Pose(Quaternion(*q), t) for q, t in zip(z[f"{name}.pose_q"], z[f"{name}.pose_t"])]
        its, pts = z[f"{name}.image_ts"], z[f"{name}.pose_ts"]
        cal = Pose(Quaternion(*z[f"{name}.cal_q"]), z[f"{name}.cal_t"])
        keep = np.arange(0, sp["frames"], every)
        if every > 1:
            images = images[keep] if not hasattr(images, "is_cuda") else images[::every].contiguous()
            its = its[keep]
            tracked = len(pts) != sp["frames"] or not np.array_equal(pts, z[f"{name}.image_ts"])
            if not tracked:
                pts = pts[keep]
                poses = [poses[i] for i in keep]
        return SweepRecording(images, its, pts, poses, (sp["pitch"], sp["pitch"]), cal)

    def planes(self, name):
        z, sp = self.z, self.spec(name)
        pitch = float(z[f"{name}.plane_pitch"])
        return [ReslicePlane(Pose(Quaternion(*q), t), sp["plane"], sp["plane"], (pitch, pitch))
                for q, t in zip(z[f"{name}.plane_q"], z[f"{name}.plane_t"])]

    def cfg(self, name) -> ResliceConfig:
        return ResliceConfig(interp_radius=self.spec(name)["voxel"])
