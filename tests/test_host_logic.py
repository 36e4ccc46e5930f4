"""CPU-only checks of the host side of the drop-in: the vectorised pose
pipeline, grid sizing, plane parameters, validation errors, file formats and
the C ABI surface.  No CUDA calls."""
import ctypes
import hashlib
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2605_26325_b200 as dare_b200
from golden_io import REC_KEYS
from oracle import oracle
from paper_2605_26325_b200 import _lib
from paper_2605_26325_b200.errors import InvalidArgumentError, SynchronizationError, VolumeFormatError
from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig, plane_params
from paper_2605_26325_b200.sweep import SweepRecording, grid_for, plan_frames

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("key", REC_KEYS)
def test_frame_plan_matches_scalar_oracle_and_reference_grid(golden, key):
    rec, voxel, margin = golden.sweep(key)
    plan = plan_frames(rec)
    frames = oracle.frame_poses(rec)
    assert list(plan.image_index) == [f.image for f in frames]
    for j, f in enumerate(frames):
        np.testing.assert_array_equal(plan.rotations[j], np.array(f.quat))
        np.testing.assert_array_equal(plan.translations[j], f.trans)
        r = oracle._rmat(f.quat)
        np.testing.assert_array_equal(plan.axes()[j], np.concatenate([r[:, 0], r[:, 1], f.trans]))
        np.testing.assert_array_equal(plan.canonical_quats_f32()[j], oracle._canon32(f.quat))
    origin, vox, dims = grid_for(plan, voxel, margin)
    np.testing.assert_array_equal(origin, golden[f"{key}.out.origin"])
    assert tuple(dims) == tuple(golden[f"{key}.out.dims"])


def test_plane_params_match_oracle(rng):
    for _ in range(50):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        plane = ReslicePlane(Pose(Quaternion(*q), rng.uniform(-5, 5, 3)), 8, 9, (0.3, 0.2))
        np.testing.assert_array_equal(np.array(plane_params(plane)), oracle.plane_params(plane))


def test_reslice_config_validation():
    with pytest.raises(InvalidArgumentError):
        ResliceConfig(interp_radius=0)
    with pytest.raises(InvalidArgumentError):
        ResliceConfig(normal_threshold_deg=90.0)
    with pytest.raises(InvalidArgumentError):
        ResliceConfig(k_dist=-1.0)
    with pytest.raises(InvalidArgumentError):
        ResliceConfig(unassigned_value=256)
    assert ResliceConfig().cos_normal_threshold == math.cos(math.radians(25.0))


def test_plane_validation_errors_before_any_device_call():
    with pytest.raises(InvalidArgumentError):
        plane_params(ReslicePlane(Pose.identity(), 0, 4, (0.1, 0.1)))
    with pytest.raises(InvalidArgumentError):
        plane_params(ReslicePlane(Pose(Quaternion(2.0, 0, 0, 0)), 4, 4, (0.1, 0.1)))


def _rec(n=2, ts_img=None, ts_pose=None):
    images = np.full((n, 1, 1), 9, np.uint8)
    ts_img = np.arange(n, dtype=float) if ts_img is None else ts_img
    ts_pose = ts_img if ts_pose is None else ts_pose
    return SweepRecording(images, ts_img, ts_pose, [Pose.identity()] * len(ts_pose), (0.1, 0.1))


def test_reconstruct_preconditions_raise_reference_errors():
    with pytest.raises(InvalidArgumentError, match="margin"):
        dare_b200.reconstruct_volume(_rec(), margin=-1.0)
    with pytest.raises(InvalidArgumentError, match="degenerate"):
        dare_b200.reconstruct_volume(_rec(1), margin=0.0)
    with pytest.raises(SynchronizationError, match="time range"):
        dare_b200.reconstruct_volume(_rec(2, np.array([0.0, 0.1]), np.array([5.0, 6.0])))
    with pytest.raises(InvalidArgumentError, match="voxel_size"):
        dare_b200.reconstruct_volume(_rec(), voxel_size=0.0)


def test_darevol_bytes_identical_to_reference(golden, tmp_path):
    for key in REC_KEYS:
        v = golden.full_volume(key + ".out")
        vol = dare_b200.DirectionalVolume(v.origin, float(golden[f"{key}.voxel"]), v.dims, v.cell_starts,
                                          v.cell_counts, v.positions, v.orientations, v.intensities)
        path = tmp_path / f"{key}.darevol"
        dare_b200.save_volume(vol, path)
        raw = path.read_bytes()
        assert len(raw) == int(golden[f"{key}.darevol_size"])
        assert hashlib.sha256(raw).hexdigest() == str(golden[f"{key}.darevol_sha256"])
        back = dare_b200.load_volume(path)
        np.testing.assert_array_equal(back.positions, v.positions)
        np.testing.assert_array_equal(back.cell_counts, v.cell_counts)


def test_volume_format_errors(tmp_path):
    p = tmp_path / "bad.darevol"
    p.write_bytes(b"XXXX" + bytes(60))
    with pytest.raises(VolumeFormatError):
        dare_b200.load_volume(p)
    with pytest.raises(VolumeFormatError):
        dare_b200.load_scalar_volume(p)


def test_scalarvol_round_trip_host(tmp_path, rng):
    values = rng.uniform(0, 255, 4 * 5 * 6).astype(np.float32)
    flags = rng.choice([0, 1, 2], 4 * 5 * 6).astype(np.uint8)
    v = dare_b200.ScalarVolume((1, 2, 3), 0.125, (4, 5, 6), values, flags)
    path = tmp_path / "x.scalarvol"
    dare_b200.save_scalar_volume(v, path)
    w = dare_b200.load_scalar_volume(path)
    np.testing.assert_array_equal(w.values, values)
    np.testing.assert_array_equal(w.flags, flags)
    assert w.dims == (4, 5, 6)


def _header_functions():
    text = open(os.path.join(ROOT, "include", "dare_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(dare_\w+)\(", text, flags=re.M)))


def test_c_abi_exports_every_declared_symbol():
    """The library loads (no CUDA call is made) and exports each header symbol."""
    lib = _lib.load()
    declared = _header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)


def test_library_exports_only_c_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    dare_syms = {line.split()[-1] for line in out.splitlines() if " T dare_" in line}
    assert dare_syms == set(_header_functions())


def test_device_code_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_frame_pose_pipeline_c_equals_numpy():
    """dare_frame_poses (csrc/plan.cu) gives the numpy restatement's bits:
    rotations, translations, axes, canonical f32 quaternions, bounds; and the
    reference's errors."""
    from paper_2605_26325_b200 import sweep as S

    rng = np.random.default_rng(11)
    n = 300
    mq = rng.normal(size=(n, 4))
    mq /= np.linalg.norm(mq, axis=1, keepdims=True)
    mq[::7] *= -1.0
    mq[5] = (0.0, -0.6, 0.8, 0.0)  # w == 0: tie-broken sign
    mt = rng.uniform(-50, 50, (n, 3))
    cal = Pose(Quaternion.from_axis_angle((0.3, -1.0, 0.2), 0.7), (1.5, -2.25, 0.125))
    kept = np.arange(n)
    a = S._compose_plan(kept, mq, mt, cal, 0, (0.137, 0.211), 47, 63)
    b = S._compose_plan_numpy(kept, mq, mt, cal, 0, (0.137, 0.211), 47, 63)
    np.testing.assert_array_equal(a.rotations, b.rotations)
    np.testing.assert_array_equal(a.translations, b.translations)
    np.testing.assert_array_equal(a.axes(), b.axes())
    np.testing.assert_array_equal(a.canonical_quats_f32(), b.canonical_quats_f32())
    ba, bb = a.bounds(0.5), b.bounds(0.5)
    np.testing.assert_array_equal(ba.min, bb.min)
    np.testing.assert_array_equal(ba.max, bb.max)
    bad = mq.copy()
    bad[3] = 0.0
    with pytest.raises(InvalidArgumentError, match="cannot normalize zero quaternion"):
        S._compose_plan(kept, bad, mt, cal, 0, (0.1, 0.1), 4, 4)
    bad = mq.copy()
    bad[9] *= 1.01
    with pytest.raises(InvalidArgumentError, match="quaternion norm 1.010000 deviates from 1 by more than 0.001"):
        S._compose_plan(kept, bad, mt, cal, 0, (0.1, 0.1), 4, 4)
    with pytest.raises(InvalidArgumentError, match="quaternion norm 1.010000 deviates"):
        S._compose_plan_numpy(kept, bad, mt, cal, 0, (0.1, 0.1), 4, 4)


def test_interpolated_poses_c_equal_reference_formula():
    """dare_interpolate_poses (csrc/plan.cu) == interpolate_pose's numpy/math
    formula (reconstruct.py:102-116, slerp geometry.py:159-180) bit for bit:
    random streams incl. near-parallel (nlerp branch) and antipodal neighbours,
    repeated timestamps; 8000 interpolated frames in well under a second."""
    import time

    from paper_2605_26325_b200 import sweep as S

    rng = np.random.default_rng(17)
    m = 900
    ts = np.cumsum(rng.uniform(0.0, 0.03, m))
    ts[100:103] = ts[100]  # t1 == t0 brackets
    q = rng.normal(size=(m, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[1::3] = q[0::3][: len(q[1::3])] + rng.normal(scale=1e-3, size=(len(q[1::3]), 4))  # nearly parallel
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[2::5] *= -1.0  # antipodal sign flips
    poses = [Pose(Quaternion(*qq), rng.uniform(-5, 5, 3)) for qq in q]
    t_img = np.sort(np.concatenate([rng.uniform(ts[0], ts[-1], 7950), ts[:50]]))  # incl. exact timestamps
    images = np.zeros((len(t_img), 2, 2), np.uint8)
    rec = SweepRecording(images, t_img, ts, poses, (0.1, 0.1))
    t0 = time.perf_counter()
    plan = plan_frames(rec)
    dt = time.perf_counter() - t0
    assert dt < 1.0, dt
    for j in range(0, len(t_img), 7):
        ref = S.interpolate_pose(float(t_img[j]), ts, poses).compose(Pose.identity())
        np.testing.assert_array_equal(plan.rotations[j], [ref.rotation.w, ref.rotation.x, ref.rotation.y,
                                                          ref.rotation.z])
        np.testing.assert_array_equal(plan.translations[j], ref.translation)


def test_numpy_dot4_is_the_fma_chain():
    """The restatement's premise: numpy's dot of two 4-vectors (slerp, norm) is
    a0 b0 then fma(a_i, b_i, s) on this host (checked exactly with fractions)."""
    from fractions import Fraction as F

    rng = np.random.default_rng(3)
    for _ in range(2000):
        a, b = rng.normal(size=4), rng.normal(size=4)
        s = a[0] * b[0]
        for i in (1, 2, 3):
            s = float(F(a[i]) * F(b[i]) + F(s))
        assert s == float(np.dot(a, b))
