"""CPU: the bench's frame content (bench_data.render_phantom: the reference's
benchmark phantom restated in torch f64 with numpy's speckle streams) against
frames rendered by the REAL reference at the bench's own sweep poses
(tests/golden/phantom.npz, tests/golden/make_golden_phantom.py): bit-identical."""
import os

import numpy as np
import pytest

import bench_data
from paper_2605_26325_b200.geometry import Pose, Quaternion

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "phantom.npz")


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_phantom_frames_match_reference(cfg):
    z = np.load(PATH)
    wl = bench_data.workload(cfg)
    poses = [Pose(Quaternion(*q), t) for q, t in zip(z[f"{cfg}.q"], z[f"{cfg}.t"])]
    # the bench's poses / frame keys at those indices are the ones the reference rendered
    bp, _ = bench_data.sweep_poses(wl)
    keys = bench_data.frame_keys(wl)
    for i, p in zip(z[f"{cfg}.index"], poses):
        np.testing.assert_array_equal(bp[i].translation, p.translation)
        assert keys[i] == z[f"{cfg}.keys"][list(z[f"{cfg}.index"]).index(i)]
    got = bench_data.render_phantom(poses, wl.size, wl.size, (wl.pitch, wl.pitch), z[f"{cfg}.keys"],
                                    device="cpu").numpy()
    ref = z[f"{cfg}.frames"]
    assert np.array_equal(got, ref), np.count_nonzero(got != ref)


@pytest.mark.gpu
def test_phantom_frames_on_gpu_match_reference():
    z = np.load(PATH)
    for cfg in ("cfg2", "cfg3"):
        wl = bench_data.workload(cfg)
        poses = [Pose(Quaternion(*q), t) for q, t in zip(z[f"{cfg}.q"], z[f"{cfg}.t"])]
        got = bench_data.render_phantom(poses, wl.size, wl.size, (wl.pitch, wl.pitch), z[f"{cfg}.keys"],
                                        device="cuda").cpu().numpy()
        assert np.array_equal(got, z[f"{cfg}.frames"]), (cfg, np.count_nonzero(got != z[f"{cfg}.frames"]))
