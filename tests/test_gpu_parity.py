"""Parity of the CUDA path (through the C ABI) with the reference golden
outputs and with the CPU oracle.  Bit-exact for indices, counts, positions,
orientations, intensities, pixels and coverage (no tolerance is needed: the
device restates the reference's f64 operation order and glibc's exp)."""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2605_26325_b200 as db
from golden_io import REC_KEYS, SEAL_KEYS
from oracle import oracle
from paper_2605_26325_b200 import _lib
from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig

pytestmark = pytest.mark.gpu

FILL_ORIGIN = (0.5, -1.0, 2.0)
FILL_VOXEL = 0.5
VOL_FIELDS = ("cell_starts", "cell_counts", "positions", "orientations", "intensities")


def assert_volume_equal(v, ref):
    np.testing.assert_array_equal(v.origin, ref.origin)
    assert tuple(v.dims) == tuple(ref.dims)
    for name in VOL_FIELDS:
        np.testing.assert_array_equal(getattr(v, name), getattr(ref, name), err_msg=name)
    assert v.rejected_out_of_bounds == ref.rejected_out_of_bounds


def test_device_present():
    assert _lib.device_count() >= 1


def test_exp_device_bit_exact(golden, rng):
    import torch

    x = np.concatenate([golden["exp.x"], -rng.uniform(0, 60, 2_000_000), rng.uniform(-1100, 1100, 100_000)])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    _lib.call("dare_exp_device", _lib.c_vp(xd.data_ptr()), _lib.c_vp(yd.data_ptr()), len(x), _lib.c_vp(0))
    _lib.call("dare_stream_sync", _lib.c_vp(0))
    y = yd.cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint64), oracle.exp(x).view(np.uint64))


@pytest.mark.parametrize("key", REC_KEYS)
def test_reconstruct_matches_reference(golden, key):
    rec, voxel, margin = golden.sweep(key)
    v = db.reconstruct_volume(rec, voxel_size=voxel, margin=margin)
    assert_volume_equal(v, golden.volume(key + ".out"))


def _random_sweep(rng, n, h, w, pitch, spread):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    poses = [Pose(Quaternion(*qq), rng.uniform(-spread, spread, 3)) for qq in q]
    ts = np.arange(n) * 0.03
    return db.SweepRecording(rng.integers(0, 256, (n, h, w), dtype=np.uint8), ts, ts, poses, pitch)


@pytest.mark.parametrize("env,value", [("DARE_COUNT_LEGACY", "1"), ("DARE_NARROW_KEYS", "1"),
                                       ("DARE_KEY_GROUPS", "3"), ("DARE_KEY_GROUPS", "7"), ("DARE_KEY_MODE", "0"),
                                       ("DARE_COMPOUND_TABLES", "1"), ("DARE_COMPOUND_V1", "1"),
                                       ("DARE_SEAL_BULK", "1"), ("DARE_FILL_U8", "0"), ("DARE_FILL_BUCKETS", "1"),
                                       ("DARE_FILL_BUCKETS", "0")])
@pytest.mark.parametrize("key", REC_KEYS)
def test_reconstruct_alternative_passes_match_reference(golden, key, env, value, monkeypatch):
    """The kept alternative passes (the FP64-chain count / compound kernels used
    when a threshold table cannot be built, 32-bit sort keys, and frame-grouped
    keys with the regroup pass -- the default for sweeps over ~1000 frames)
    give the same bytes as the default path."""
    monkeypatch.setenv(env, value)
    if env == "DARE_COMPOUND_TABLES":
        monkeypatch.setenv("DARE_COMPOUND_PACKED", "1" if key in ("rec_tilt", "rec_margin0") else "0")
    rec, voxel, margin = golden.sweep(key)
    v = db.reconstruct_volume(rec, voxel_size=voxel, margin=margin)
    assert_volume_equal(v, golden.volume(key + ".out"))
    if key != "rec_drop" and env != "DARE_KEY_GROUPS":
        s = db.compound(rec, voxel_size=voxel, margin=margin)
        np.testing.assert_array_equal(s.values, golden[f"cmp_{key}.values"])
        np.testing.assert_array_equal(s.counts, golden[f"cmp_{key}.counts"])


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("groups", ["0", "2", "3", "5"])
def test_reconstruct_frame_grouped_keys_match_oracle(groups, mode, monkeypatch):
    """Multi-direction sweep of 330 frames (three sub-sweeps at different probe
    orientations over one region, like cfg3) with per-frame-group counters:
    mode 2 (default for long sweeps) places single-run (group, cell) keys
    without atomics, mode 1 keeps group-major key CSRs and regroups them
    (DARE_KEY_GROUPS; 0 = the default choice, one group at this length)."""
    monkeypatch.setenv("DARE_KEY_MODE", mode)
    if groups != "0":
        monkeypatch.setenv("DARE_KEY_GROUPS", groups)
    rng = np.random.default_rng(44)
    poses = []
    for k in range(330):
        base = [Quaternion.identity(), Quaternion.from_axis_angle((0, 1, 0), 1.2),
                Quaternion.from_axis_angle((1, 0, 0), -1.0)][k // 110]
        s_ = (k % 110) * 0.02
        poses.append(Pose(base, [(0.0, 0.0, s_), (s_, 0.0, 2.0), (0.0, s_, 2.0)][k // 110]))
    ts = np.arange(330) / 30.0
    rec = db.SweepRecording(rng.integers(0, 256, (330, 21, 23), dtype=np.uint8), ts, ts, poses, (0.1, 0.1))
    v = db.reconstruct_volume(rec, voxel_size=0.1, margin=0.2)
    assert_volume_equal(v, oracle.reconstruct(rec, 0.1, 0.2))


@pytest.mark.parametrize("seed,voxel,margin", [(1, 0.25, 0.0), (2, 0.1, 0.5), (3, 0.37, 1.0)])
def test_reconstruct_random_sweeps_match_oracle(seed, voxel, margin):
    rng = np.random.default_rng(seed)
    rec = _random_sweep(rng, 40, 33, 47, (0.11, 0.09), 2.0)
    v = db.reconstruct_volume(rec, voxel_size=voxel, margin=margin)
    assert_volume_equal(v, oracle.reconstruct(rec, voxel, margin))


@pytest.mark.parametrize("buckets", ["0", "1"])
def test_reconstruct_host_frames_many_upload_groups(buckets, monkeypatch):
    """A linear sweep long enough for several 64-frame chunks: host frames upload in groups and
    the fill runs one launch per group; frames on the device take one fill launch.  Both equal
    the oracle (insertion order across chunk and group boundaries), with the per-cell and the
    bucketed fill (bucket cursors carried across the group launches)."""
    import torch

    monkeypatch.setenv("DARE_FILL_BUCKETS", buckets)

    rng = np.random.default_rng(17)
    n, h, w = 300, 12, 14
    poses = [Pose(Quaternion.from_axis_angle((1, 0.2, 0), 0.002 * k), (0.0, 0.0, 0.021 * k)) for k in range(n)]
    ts = np.arange(n) * 0.03
    rec = db.SweepRecording(rng.integers(0, 256, (n, h, w), dtype=np.uint8), ts, ts, poses, (0.1, 0.1))
    ref = oracle.reconstruct(rec, 0.2, 0.3)
    assert_volume_equal(db.reconstruct_volume(rec, voxel_size=0.2, margin=0.3), ref)
    frames_d = torch.from_numpy(np.asarray(rec.images)).cuda()
    dev = db.SweepRecording(np.asarray(rec.images), ts, ts, poses, (0.1, 0.1))
    v = db.reconstruct_volume(dev, voxel_size=0.2, margin=0.3, frames_device_ptr=frames_d.data_ptr())
    assert_volume_equal(v, ref)


@pytest.mark.parametrize("n", [8, 80])
def test_reconstruct_dense_cells_use_large_run_path(n):
    # many frames at one pose: > 32 samples per cell -> segmented-sort path;
    # n = 8 keeps every cell <= 255 samples (u8 fill cursors), n = 80 does not
    rng = np.random.default_rng(5)
    ts = np.arange(n) * 0.1
    rec = db.SweepRecording(rng.integers(0, 256, (n, 6, 5), dtype=np.uint8), ts, ts, [Pose.identity()] * n,
                            (0.05, 0.05))
    v = db.reconstruct_volume(rec, voxel_size=0.5, margin=0.25)
    assert v.cell_counts.max() > 32 and (v.cell_counts.max() <= 255) == (n == 8)
    assert_volume_equal(v, oracle.reconstruct(rec, 0.5, 0.25))


@pytest.mark.parametrize("key", SEAL_KEYS)
def test_volume_builder_seal_matches_reference(golden, key):
    b = golden[f"{key}.bounds"]
    builder = db.VolumeBuilder(db.BoundingBox(b[:3], b[3:]), float(golden[f"{key}.voxel"]))
    builder.insert_batch(golden[f"{key}.in_pos"], golden[f"{key}.in_quat"], golden[f"{key}.in_inten"])
    v = builder.seal()
    v.rejected_out_of_bounds = builder.rejected_out_of_bounds
    assert_volume_equal(v, golden.volume(key + ".out"))


def test_reslice_matches_reference_goldens(golden):
    vols = {}
    for i, c in golden.reslice_cases():
        if c.vol_key not in vols:
            vols[c.vol_key] = golden.full_volume(c.vol_key)  # foreign (reference-layout) volume
        vol = vols[c.vol_key]
        out = db.reslice(vol, c.plane, c.cfg)
        np.testing.assert_array_equal(out.pixels, c.pixels, err_msg=f"rs_{i}")
        np.testing.assert_array_equal(out.coverage, c.coverage, err_msg=f"rs_{i}")
        if c.brute is not None:
            b = db.reslice_bruteforce(vol, c.plane, c.cfg)
            np.testing.assert_array_equal(b.pixels, c.brute[0])
            np.testing.assert_array_equal(b.coverage, c.brute[1])


def _random_volume(rng, n, extent=10.0, voxel=0.5):
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (extent,) * 3), voxel)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1.0
    b.insert_batch(rng.uniform(0, extent, (n, 3)), q, rng.integers(0, 256, n))
    return b.seal()


def test_acceptance_criterion_1_against_oracle(rng):
    """>= 100 randomized (volume, plane, config) cases, bit-exact vs the CPU oracle
    (grid and brute force), as test_acceptance.py:92-123 does for the reference."""
    for case in range(100):
        vol = _random_volume(rng, int(rng.integers(0, 10_001)), 10.0, float(rng.choice([0.25, 0.5, 1.0])))
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        plane = ReslicePlane(Pose(Quaternion(*q), rng.uniform(-1, 11, 3)), int(rng.integers(4, 25)),
                             int(rng.integers(4, 25)), (float(rng.uniform(0.1, 0.6)),) * 2)
        cfg = ResliceConfig(interp_radius=float(rng.uniform(0.15, 1.5)),
                            normal_threshold_deg=float(rng.uniform(5, 85)),
                            inplane_threshold_deg=float(rng.uniform(5, 85)), k_normal=float(rng.uniform(0, 20)),
                            k_inplane=float(rng.uniform(0, 10)), k_dist=float(rng.choice([0.0, 1.0, 2.0, 4.0])),
                            unassigned_value=int(rng.integers(0, 256)))
        fast = db.reslice(vol, plane, cfg)
        ref = oracle.reslice(vol, oracle.plane_params(plane), oracle.cfg_array(cfg), plane.width, plane.height,
                             cfg.unassigned_value)
        np.testing.assert_array_equal(fast.pixels, ref[0], err_msg=f"case {case}")
        np.testing.assert_array_equal(fast.coverage, ref[1], err_msg=f"case {case}")
        brute = db.reslice_bruteforce(vol, plane, cfg)
        np.testing.assert_array_equal(brute.pixels, fast.pixels)
        np.testing.assert_array_equal(brute.coverage, fast.coverage)


def test_reslice_batch_equals_single_calls(rng):
    vol = _random_volume(rng, 20000, 10.0, 0.25)
    planes = []
    for _ in range(9):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        planes.append(ReslicePlane(Pose(Quaternion(*q), rng.uniform(2, 8, 3)), 40, 33, (0.2, 0.2)))
    cfg = ResliceConfig(interp_radius=0.25)
    px, cov, _ = db.reslice_batch(vol, planes, cfg)
    for k, p in enumerate(planes):
        one = db.reslice(vol, p, cfg)
        np.testing.assert_array_equal(px[k], one.pixels)
        np.testing.assert_array_equal(cov[k], one.coverage)


def test_pose_major_schedule_identical(rng):
    """The pose-major schedule (lanes = one pixel of 32 consecutive poses) gives
    the same bits as the pixel-major one, on a coherent trajectory and on a
    random batch (forced)."""
    import ctypes

    from paper_2605_26325_b200 import _lib
    from paper_2605_26325_b200.reslice import kernel_cfg, plane_params

    vol = _random_volume(rng, 30000, 10.0, 0.25)
    q0 = Quaternion.from_axis_angle((1, 0.2, 0), 0.3)
    traj = [ReslicePlane(Pose(Quaternion.from_axis_angle((1, 0.2, 0), 0.3 + 0.002 * k), (2.0 + 0.01 * k, 2.0, 5.0)),
                         23, 19, (0.2, 0.2)) for k in range(70)]
    rand = []
    for _ in range(40):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        rand.append(ReslicePlane(Pose(Quaternion(*q), rng.uniform(2, 8, 3)), 23, 19, (0.2, 0.2)))
    cfg = ResliceConfig(interp_radius=0.25, normal_threshold_deg=60, inplane_threshold_deg=60)
    handle = vol.device_handle().raw
    for planes in (traj, rand):
        params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
        outs = []
        for sched in (1, 2):
            px = np.empty((len(planes), 19, 23), np.uint8)
            cv = np.empty((len(planes), 19, 23), np.uint8)
            kc = kernel_cfg(cfg, sched)
            _lib.call("dare_reslice", handle, len(planes), _lib.ptr(params, ctypes.c_double), 23, 19,
                      ctypes.byref(kc), _lib.ptr(px, ctypes.c_uint8), _lib.ptr(cv, ctypes.c_uint8))
            outs.append((px, cv))
        np.testing.assert_array_equal(outs[0][0], outs[1][0])
        np.testing.assert_array_equal(outs[0][1], outs[1][1])
        assert outs[0][1].any()
    p_traj = np.ascontiguousarray([plane_params(p) for p in traj], dtype=np.float64)
    assert _lib.load().dare_poses_coherent(_lib.ptr(p_traj, ctypes.c_double), len(traj), 23, 19, 0.25) == 1
    assert q0 is not None


def test_concurrent_reslices_identical(rng):
    vol = _random_volume(rng, 4000)
    plane = ReslicePlane(Pose(Quaternion.identity(), (2.0, 2.0, 5.0)), 24, 20, (0.3, 0.3))
    cfg = ResliceConfig(interp_radius=0.6, normal_threshold_deg=80, inplane_threshold_deg=80)
    ref = db.reslice(vol, plane, cfg)
    with ThreadPoolExecutor(max_workers=6) as pool:
        results = list(pool.map(lambda _: db.reslice(vol, plane, cfg), range(24)))
    for r in results:
        np.testing.assert_array_equal(r.pixels, ref.pixels)
        np.testing.assert_array_equal(r.coverage, ref.coverage)


def test_reference_behaviour_cases():
    # empty volume -> all unassigned (test_reslice.py:164-169)
    vol = _random_volume(np.random.default_rng(0), 0)
    out = db.reslice(vol, ReslicePlane(Pose.identity(), 5, 4, (0.3, 0.3)), ResliceConfig(unassigned_value=7))
    assert not out.coverage.any() and (out.pixels == 7).all()
    # single sample (test_reslice.py:171-179)
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (4, 4, 1)), 0.25)
    b.insert_sample(db.DirectionalSample(177, Quaternion.identity(), (2.0, 2.0, 0.5)))
    vol = b.seal()
    plane = ReslicePlane(Pose(Quaternion.identity(), (2.0, 2.0, 0.5)), 1, 1, (0.25, 0.25))
    for fn in (db.reslice, db.reslice_bruteforce):
        o = fn(vol, plane, ResliceConfig(interp_radius=0.25))
        assert o.coverage[0, 0] and o.pixels[0, 0] == 177
    # cube, not ball (test_reslice.py:247-257)
    r = 0.25
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (4, 4, 2)), r)
    b.insert_sample(db.DirectionalSample(99, Quaternion.identity(), np.array([2.0 + r, 2.0 + r, 0.5 + r]) - 1e-6))
    o = db.reslice(b.seal(), ReslicePlane(Pose(Quaternion.identity(), (2.0, 2.0, 0.5)), 1, 1, (r, r)),
                   ResliceConfig(interp_radius=r))
    assert o.coverage[0, 0]
    # 25 degree gate rejects a 30 degree tilt, 40 accepts (test_reslice.py:232-240)
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (4, 4, 1)), 0.25)
    b.insert_sample(db.DirectionalSample(200, Quaternion.from_axis_angle((1, 0, 0), math.radians(30)),
                                         (2.0, 2.0, 0.5)))
    vol = b.seal()
    assert not db.reslice(vol, plane, ResliceConfig(interp_radius=0.25)).coverage[0, 0]
    assert db.reslice(vol, plane, ResliceConfig(interp_radius=0.25, normal_threshold_deg=40)).coverage[0, 0]


def test_single_frame_round_trip_within_one_gray(rng):
    """Acceptance criterion 2 (test_acceptance.py:126-139)."""
    img = rng.integers(0, 256, (48, 64), dtype=np.uint8)
    rec = db.SweepRecording(img[None], [0.0], [0.0], [Pose.identity()], (0.2, 0.2))
    vol = db.reconstruct_volume(rec, voxel_size=0.125, margin=0.5)
    out = db.reslice(vol, ReslicePlane(Pose.identity(), 64, 48, (0.2, 0.2)), ResliceConfig())
    assert out.coverage.all()
    assert np.abs(out.pixels.astype(int) - img.astype(int)).max() <= 1


@pytest.mark.parametrize("key", ("rec_tilt", "rec_mask", "rec_parallel", "rec_margin0"))
def test_compound_matches_reference(golden, key):
    rec, voxel, margin = golden.sweep(key)
    s = db.compound(rec, voxel_size=voxel, margin=margin)
    np.testing.assert_array_equal(s.origin, golden[f"cmp_{key}.origin"])
    np.testing.assert_array_equal(s.values, golden[f"cmp_{key}.values"])
    np.testing.assert_array_equal(s.flags, golden[f"cmp_{key}.flags"])
    np.testing.assert_array_equal(s.counts, golden[f"cmp_{key}.counts"])


@pytest.mark.parametrize("i", range(6))
def test_fill_holes_and_trilinear_match_reference(golden, i):
    dims = tuple(int(d) for d in golden[f"fill_{i}.dims"])
    sv = db.ScalarVolume(FILL_ORIGIN, FILL_VOXEL, dims, golden[f"fill_{i}.in_values"], golden[f"fill_{i}.in_flags"])
    out = db.fill_holes(sv, max_passes=int(golden[f"fill_{i}.passes"]))
    np.testing.assert_array_equal(out.values, golden[f"fill_{i}.values"])
    np.testing.assert_array_equal(out.flags, golden[f"fill_{i}.flags"])
    for j in range(3):
        key = f"tri_{i}_{j}"
        r = db.reslice_trilinear(out, golden.trilinear_plane(key))
        np.testing.assert_array_equal(r.pixels, golden[f"{key}.pixels"])
        np.testing.assert_array_equal(r.coverage, golden[f"{key}.coverage"])


def test_scalar_arm_random_sweep_matches_oracle():
    rng = np.random.default_rng(11)
    rec = _random_sweep(rng, 30, 21, 25, (0.1, 0.1), 1.5)
    s = db.compound(rec, voxel_size=0.2, margin=0.3)
    origin, voxel, dims, values, flags, counts = oracle.compound(rec, 0.2, 0.3)
    np.testing.assert_array_equal(s.values, values)
    np.testing.assert_array_equal(s.counts, counts)
    f = db.fill_holes(s, 3)
    fv, ff = oracle.fill_holes(values, flags, dims, 3)
    np.testing.assert_array_equal(f.values, fv)
    np.testing.assert_array_equal(f.flags, ff)
    for k in range(5):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        plane = ReslicePlane(Pose(Quaternion(*q), rng.uniform(-1, 1, 3)), 31, 29, (0.07, 0.07))
        r = db.reslice_trilinear(f, plane)
        px, cov, _ = oracle.trilinear(origin, voxel, dims, fv, ff, oracle.plane_params(plane), 31, 29)
        np.testing.assert_array_equal(r.pixels, px)
        np.testing.assert_array_equal(r.coverage, cov)


def test_trilinear_at_points_values():
    vals = np.zeros((2, 1, 1), np.float32)
    vals[1, 0, 0] = 200.0
    sv = db.ScalarVolume((0, 0, 0), 1.0, (2, 1, 1), vals.reshape(-1), np.ones(2, np.uint8))
    v, c = db.trilinear_at_points(sv, [(1.0, 0.5, 0.5)])
    assert c[0] and v[0] == 100.0


def test_darevol_from_device_volume_identical(golden, tmp_path):
    import hashlib

    rec, voxel, margin = golden.sweep("rec_tilt")
    v = db.reconstruct_volume(rec, voxel_size=voxel, margin=margin)
    path = tmp_path / "v.darevol"
    db.save_volume(v, path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == str(golden["rec_tilt.darevol_sha256"])


# ---------------------------------------------------------------- certified path

def _fallback_pixels():
    import ctypes

    n = ctypes.c_int64()
    _lib.call("dare_reslice_last_fallback", ctypes.byref(n))
    return n.value


def _reslice_raw(vol, planes, cfg, exact, schedule=0):
    import ctypes

    from paper_2605_26325_b200.reslice import kernel_cfg, plane_params

    w, h = planes[0].width, planes[0].height
    params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
    px = np.empty((len(planes), h, w), np.uint8)
    cv = np.empty((len(planes), h, w), np.uint8)
    kc = kernel_cfg(cfg, schedule, exact)
    _lib.call("dare_reslice", vol.device_handle().raw, len(planes), _lib.ptr(params, ctypes.c_double), w, h,
              ctypes.byref(kc), _lib.ptr(px, ctypes.c_uint8), _lib.ptr(cv, ctypes.c_uint8))
    return px, cv, _fallback_pixels()


def test_fastmath_constants_hold_exhaustively():
    """Every f32 input of ex2.approx / sqrt.approx in the ranges the certified
    bound uses is within the assumed 2^-21 relative error on this device."""
    import ctypes

    e1, e2, ok = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
    _lib.call("dare_fastmath_check", ctypes.byref(e1), ctypes.byref(e2), ctypes.byref(ok))
    print(f"ex2.approx max rel err {e1.value:.3e}, sqrt.approx max rel err {e2.value:.3e}")
    assert ok.value == 1
    assert 0 < e1.value <= 2.0 ** -21 and 0 < e2.value <= 2.0 ** -21


def test_certified_path_equals_exact_path(rng):
    """Default (certified f32 + exact fallback) and exact=1 (FP64 everywhere)
    give identical pixels over random volumes, planes and configs, both
    schedules."""
    for case in range(30):
        vol = _random_volume(rng, int(rng.integers(2000, 40_001)), 10.0, float(rng.choice([0.25, 0.5])))
        planes = []
        for _ in range(int(rng.integers(1, 40))):
            q = rng.normal(size=4)
            q /= np.linalg.norm(q)
            planes.append(ReslicePlane(Pose(Quaternion(*q), rng.uniform(1, 9, 3)), 21, 17,
                                       (float(rng.uniform(0.1, 0.4)),) * 2))
        cfg = ResliceConfig(interp_radius=float(rng.uniform(0.15, 1.0)),
                            normal_threshold_deg=float(rng.uniform(5, 89)),
                            inplane_threshold_deg=float(rng.uniform(5, 89)), k_normal=float(rng.uniform(0, 20)),
                            k_inplane=float(rng.uniform(0, 10)), k_dist=float(rng.choice([0.0, 0.5, 2.0, 4.0])),
                            unassigned_value=int(rng.integers(0, 256)))
        ex = _reslice_raw(vol, planes, cfg, True)
        assert ex[2] == 0
        for sched in (1, 2):
            fa = _reslice_raw(vol, planes, cfg, False, sched)
            np.testing.assert_array_equal(fa[0], ex[0], err_msg=f"case {case} sched {sched}")
            np.testing.assert_array_equal(fa[1], ex[1], err_msg=f"case {case} sched {sched}")


def _lattice_volume(rng, n=24, spacing=0.125, checker=False):
    """Samples on an exact f32 lattice, one orientation, random intensities:
    equal weights (k_dist = 0) or symmetric distances make half-integer
    weighted means common -- the cases the certified bound cannot decide.
    checker=True: intensity 10 + (x index mod 2), so any cube spanning an even
    number of x lattice lines has a mean of exactly 10.5."""
    g = np.arange(n, dtype=np.float64) * spacing + spacing / 2
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    q = np.tile([1.0, 0.0, 0.0, 0.0], (len(pos), 1))
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (n * spacing,) * 3), 0.25)
    if checker:
        inten = 10 + (np.arange(len(pos)) // (n * n)) % 2
    else:
        inten = rng.integers(0, 256, len(pos))
    b.insert_batch(pos, q, inten)
    return b.seal()


@pytest.mark.parametrize("k_dist", [0.0, 2.0])
def test_half_integer_ties_take_the_exact_fallback(rng, k_dist):
    vol = _lattice_volume(rng)
    planes = [ReslicePlane(Pose(Quaternion.identity(), (0.0, 0.0, 0.0625 + 0.125 * k)), 24, 24, (0.125, 0.125))
              for k in range(8)]
    cfg = ResliceConfig(interp_radius=0.125, k_dist=k_dist)
    fa = _reslice_raw(vol, planes, cfg, False)
    ex = _reslice_raw(vol, planes, cfg, True)
    assert fa[2] > 0, "lattice ties should reach the exact fallback"
    np.testing.assert_array_equal(fa[0], ex[0])
    np.testing.assert_array_equal(fa[1], ex[1])
    for k, p in enumerate(planes[:3]):
        ref = oracle.reslice(vol, oracle.plane_params(p), oracle.cfg_array(cfg), p.width, p.height,
                             cfg.unassigned_value)
        np.testing.assert_array_equal(fa[0][k], ref[0], err_msg=f"plane {k}")
        np.testing.assert_array_equal(fa[1][k].astype(bool), ref[1], err_msg=f"plane {k}")


def test_z_binned_layout_round_trips_every_run_length():
    """Cells of 1..40 samples inserted in descending z (so z-quarter binning
    permutes every binned cell): the device layout regroups cells of <= 32
    samples by quarter, and download / reslice still see insertion order."""
    import torch

    from paper_2605_26325_b200.parallel import _CudaArray

    pos, inten = [], []
    for c in range(40):
        for j in range(c + 1):
            pos.append((c + 0.5, 0.5, 0.99 - j * 0.98 / (c + 1)))
            inten.append((7 * j + c) % 256)
    pos = np.array(pos)
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (40, 1, 1)), 1.0)
    b.insert_batch(pos, np.tile([1.0, 0, 0, 0], (len(pos), 1)), np.array(inten))
    v = b.seal()
    np.testing.assert_array_equal(np.asarray(v.positions), pos.astype(np.float32))
    np.testing.assert_array_equal(np.asarray(v.intensities), np.array(inten, np.uint8))
    info = v.device_info()
    counts = np.asarray(v.cell_counts)
    bins = torch.as_tensor(_CudaArray(info.d_bins, (len(counts),), "<u4"), device="cuda").cpu().numpy()
    perm = torch.as_tensor(_CudaArray(info.d_perm, (int(info.n_samples),), "|i1"), device="cuda").cpu().numpy()
    for c in np.nonzero(counts)[0]:
        binned = bool(bins[c] >> 24)
        assert binned == (counts[c] <= 32), c
        if binned and counts[c] > 1:
            assert (perm[v.cell_starts[c]:v.cell_starts[c] + counts[c]] != 0).any()
    # reslice through the binned layout == oracle on the reference layout
    plane = ReslicePlane(Pose(Quaternion.identity(), (0.3, 0.5, 0.4)), 40, 1, (1.0, 1.0))
    cfg = ResliceConfig(interp_radius=0.6, k_dist=2.0)
    got = db.reslice(v, plane, cfg)
    ref = oracle.reslice(v, oracle.plane_params(plane), oracle.cfg_array(cfg), 40, 1, 0)
    np.testing.assert_array_equal(got.pixels, ref[0])
    np.testing.assert_array_equal(got.coverage, ref[1])


def test_certified_path_guard_rails(rng):
    """Extreme weighting configs: exponents beyond the accurate ex2 range make
    the certified path stand down for the launch (exact FP64 everywhere), tiny
    radii / huge k_dist put many pixels near the coverage threshold; both must
    still match the FP64 path and the oracle bit for bit."""
    vol = _random_volume(rng, 20000, 10.0, 0.5)
    planes = []
    for _ in range(6):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        planes.append(ReslicePlane(Pose(Quaternion(*q), rng.uniform(2, 8, 3)), 19, 17, (0.3, 0.3)))
    cfgs = [ResliceConfig(interp_radius=0.4, k_normal=1000.0, k_inplane=1000.0, k_dist=50.0,
                          normal_threshold_deg=89.0, inplane_threshold_deg=89.0),   # M > 99: exact path
            ResliceConfig(interp_radius=0.4, k_dist=16.0, normal_threshold_deg=85.0,
                          inplane_threshold_deg=85.0, k_normal=0.0, k_inplane=0.0),  # weights down to e^-27.7
            ResliceConfig(interp_radius=0.05, k_dist=0.0)]
    for cfg in cfgs:
        fa = _reslice_raw(vol, planes, cfg, False)
        ex = _reslice_raw(vol, planes, cfg, True)
        np.testing.assert_array_equal(fa[0], ex[0])
        np.testing.assert_array_equal(fa[1], ex[1])
        ref = oracle.reslice(vol, oracle.plane_params(planes[0]), oracle.cfg_array(cfg), 19, 17,
                             cfg.unassigned_value)
        np.testing.assert_array_equal(fa[0][0], ref[0])
        np.testing.assert_array_equal(fa[1][0].astype(bool), ref[1])


@pytest.mark.parametrize("radius", [0.6, 1.1])
def test_fallback_wide_neighbourhoods(rng, radius):
    """Ties on a dense lattice with radii spanning 5 (25 columns, > 256
    survivors per pixel: the flattened fallback overflows its shared-memory
    capacity) and 9-10 cells per axis (> 32 columns): the fallback's general
    warp walk must still reproduce the FP64 path bit for bit; single poses
    (split-pixel certified kernel) and batches."""
    vol = _lattice_volume(rng, checker=True)
    planes = [ReslicePlane(Pose(Quaternion.identity(), (0.3, 0.2, 0.0625 + 0.25 * k)), 12, 10, (0.125, 0.125))
              for k in range(6)]
    cfg = ResliceConfig(interp_radius=radius, k_dist=0.0)
    ex = _reslice_raw(vol, planes, cfg, True)
    fa = _reslice_raw(vol, planes, cfg, False)
    assert fa[2] > 0
    np.testing.assert_array_equal(fa[0], ex[0])
    np.testing.assert_array_equal(fa[1], ex[1])
    one = _reslice_raw(vol, planes[:1], cfg, False)
    np.testing.assert_array_equal(one[0][0], ex[0][0])
    np.testing.assert_array_equal(one[1][0], ex[1][0])


@pytest.mark.parametrize("parts", ["1", "2", "4"])
def test_split_pixel_variants_identical(rng, parts, monkeypatch):
    """Small batches split a pixel's column phases over 1, 2 or 4 threads (host
    cost model; DARE_SPLIT forces one): same bits as the oracle for each."""
    vol = _random_volume(rng, 30000, 10.0, 0.25)
    cfg = ResliceConfig(interp_radius=0.25, normal_threshold_deg=70, inplane_threshold_deg=70)
    planes = []
    for _ in range(3):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        planes.append(ReslicePlane(Pose(Quaternion(*q), rng.uniform(2, 8, 3)), 37, 29, (0.2, 0.2)))
    monkeypatch.setenv("DARE_SPLIT", parts)
    for P in (1, 3):
        px, cov, _ = db.reslice_batch(vol, planes[:P], cfg)
        for k in range(P):
            ref = oracle.reslice(vol, oracle.plane_params(planes[k]), oracle.cfg_array(cfg), 37, 29)
            np.testing.assert_array_equal(px[k], ref[0])
            np.testing.assert_array_equal(cov[k], ref[1])


def _few_orient_volume(rng, n, k, extent=10.0, voxel=0.5):
    """Samples sharing k distinct orientations (sweeps at fixed probe
    orientations; k > 1024 takes the global-gate form of the index walk)."""
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (extent,) * 3), voxel)
    qs = rng.normal(size=(k, 4))
    qs /= np.linalg.norm(qs, axis=1, keepdims=True)
    qs[qs[:, 0] < 0] *= -1.0
    pos = rng.uniform(0, extent, (n, 3))
    b.insert_batch(pos, qs[rng.integers(0, k, n)], rng.integers(0, 256, n))
    return b.seal(), qs


@pytest.mark.parametrize("k", [2, 3, 6, 17, 200, 2000])
def test_direction_cluster_index_identical(rng, k, monkeypatch):
    """The certified path over the direction-cluster index (split.cu: only the
    clusters a pose accepts are walked) equals the exact FP64 path, the
    certified path on the canonical layout (DARE_ORIENT_SPLIT=0, a second copy
    of the volume) and the oracle, for planes aligned with the volume's
    orientations and random ones, narrow and wide gates, 1..40 poses per call."""
    for case in range(6):
        n = int(rng.integers(5000, 40_001))
        seed = int(rng.integers(1 << 30))
        vol, qs = _few_orient_volume(np.random.default_rng(seed), n, k)
        monkeypatch.setenv("DARE_ORIENT_SPLIT", "0")
        canon, _ = _few_orient_volume(np.random.default_rng(seed), n, k)
        _reslice_raw(canon, [ReslicePlane(Pose(Quaternion(1.0, 0.0, 0.0, 0.0), (5.0, 5.0, 5.0)), 4, 4,
                                          (0.2, 0.2))], ResliceConfig(interp_radius=0.5), False)  # index decided
        monkeypatch.delenv("DARE_ORIENT_SPLIT")
        planes = []
        for j in range(int(rng.choice([1, 2, 8, 40]))):
            q = qs[j % k] + (rng.normal(scale=0.05, size=4) if j % 3 else rng.normal(size=4))
            q /= np.linalg.norm(q)
            planes.append(ReslicePlane(Pose(Quaternion(*q), rng.uniform(1, 9, 3)), 23, 19,
                                       (float(rng.uniform(0.1, 0.4)),) * 2))
        wide = bool(case % 2)
        cfg = ResliceConfig(interp_radius=float(rng.uniform(0.25, 1.0)),
                            normal_threshold_deg=float(rng.uniform(60, 89) if wide else rng.uniform(10, 40)),
                            inplane_threshold_deg=float(rng.uniform(60, 89) if wide else rng.uniform(10, 40)),
                            k_normal=float(rng.uniform(0, 20)), k_inplane=float(rng.uniform(0, 10)),
                            k_dist=float(rng.choice([0.0, 2.0])), unassigned_value=int(rng.integers(0, 256)))
        ex = _reslice_raw(vol, planes, cfg, True)
        fa = _reslice_raw(vol, planes, cfg, False, 1)
        ca = _reslice_raw(canon, planes, cfg, False, 1)
        for got, what in ((fa, "split"), (ca, "canonical")):
            np.testing.assert_array_equal(got[0], ex[0], err_msg=f"k {k} case {case} {what}")
            np.testing.assert_array_equal(got[1], ex[1], err_msg=f"k {k} case {case} {what}")
        p = planes[0]
        ref = oracle.reslice(vol, oracle.plane_params(p), oracle.cfg_array(cfg), p.width, p.height,
                             cfg.unassigned_value)
        np.testing.assert_array_equal(fa[0][0], ref[0])
        np.testing.assert_array_equal(fa[1][0], ref[1])


@pytest.mark.parametrize("n", [8, 1000])
def test_bucketed_fill_forced_and_oversized_buckets(n, monkeypatch):
    """DARE_FILL_BUCKETS=1: the bucketed fill on a dense stack (n = 8: every
    bucket fits the placement stage) and with a bucket over its capacity
    (n = 1000: 30k samples in one cell -> the per-cell fill), both equal to the
    oracle."""
    monkeypatch.setenv("DARE_FILL_BUCKETS", "1")
    rng = np.random.default_rng(7)
    ts = np.arange(n) * 0.1
    rec = db.SweepRecording(rng.integers(0, 256, (n, 6, 5), dtype=np.uint8), ts, ts, [Pose.identity()] * n,
                            (0.05, 0.05))
    v = db.reconstruct_volume(rec, voxel_size=0.5, margin=0.25)
    assert (v.cell_counts.max() > 24 * 1024) == (n == 1000)
    assert_volume_equal(v, oracle.reconstruct(rec, 0.5, 0.25))
