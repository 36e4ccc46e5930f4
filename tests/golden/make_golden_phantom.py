"""Generate tests/golden/phantom.npz: frames of the REAL reference's benchmark
phantom (phantom.py:402-467 default_benchmark_scene, seed 7, speckle 5;
render_intensities phantom.py:113-152) at the bench's sweep poses, so the
bench's GPU restatement (bench_data.render_phantom) can be checked on CPU.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_phantom.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "phantom.npz")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    import bench_data
    from dare.geometry import Pose, Quaternion
    from dare.phantom import default_benchmark_scene, render_intensities, scene_from_dict

    scene, _ = scene_from_dict(default_benchmark_scene(seed=7, speckle=5.0))
    g = {}
    cases = [("cfg1", [0, 57, 123, 199]), ("cfg2", [0, 250, 999]), ("cfg3", [10, 2500, 4321, 7999])]
    for cfg, idx in cases:
        wl = bench_data.workload(cfg)
        poses, _ = bench_data.sweep_poses(wl)
        keys = bench_data.frame_keys(wl)
        imgs, q, t, k = [], [], [], []
        for i in idx:
            p = poses[i]
            r = p.rotation
            rp = Pose(Quaternion(r.w, r.x, r.y, r.z), np.asarray(p.translation, float))
            imgs.append(render_intensities(scene, rp, wl.size, wl.size, (wl.pitch, wl.pitch), frame_key=int(keys[i])))
            q.append([r.w, r.x, r.y, r.z])
            t.append(p.translation)
            k.append(int(keys[i]))
        g[f"{cfg}.frames"] = np.stack(imgs)
        g[f"{cfg}.q"] = np.array(q)
        g[f"{cfg}.t"] = np.array(t, dtype=float)
        g[f"{cfg}.keys"] = np.array(k, np.int64)
        g[f"{cfg}.index"] = np.array(idx, np.int64)
        print(cfg, g[f"{cfg}.frames"].shape, [int(im.max()) for im in imgs])
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
