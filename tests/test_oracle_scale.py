"""CPU: the oracle (oracle/, test infrastructure) reproduces the REAL
reference's outputs at BASELINE configs[0] scale (tests/golden/scale.npz:
cfg1 = 200 x 128^2 -> 128^3, and cfg1t, the same frames on a tracked,
slerp-interpolated sweep with calibration) -- the .darevol bytes, reslices,
compound, fill_holes and trilinear hashes -- and this repo's workload
generator reproduces the reference's sweep geometry (SweepPlan.linear)."""
import numpy as np
import pytest

import bench_data
import paper_2605_26325_b200 as db
from oracle import oracle
from scale_io import HashSink, Scale, sha

SCALE = Scale()


@pytest.mark.parametrize("name", ["cfg1", "cfg1t"])
def test_oracle_matches_reference_at_cfg1_scale(name):
    sp = SCALE.spec(name)
    frames = SCALE.frames(name)
    assert sha(frames) == str(SCALE[f"{name}.frames_sha256"])
    sweep = SCALE.sweep(name, frames)
    vol = oracle.reconstruct(sweep, sp["voxel"], sp["margin"])
    assert tuple(vol.dims) == tuple(int(d) for d in SCALE[f"{name}.dims"])
    assert vol.rejected_out_of_bounds == int(SCALE[f"{name}.rejected"])
    sink = HashSink()
    db.save_volume(vol, sink)  # host-array path of the writer (oracle volume)
    assert sink.hexdigest() == str(SCALE[f"{name}.darevol_sha256"])
    cfg = SCALE.cfg(name)
    planes = SCALE.planes(name)
    for k in range(0, len(planes), 4):  # every 4th pose (the GPU test does all)
        p = planes[k]
        px, cov = oracle.reslice(vol, oracle.plane_params(p), oracle.cfg_array(cfg), p.width, p.height)
        assert sha(px) == str(SCALE[f"{name}.rs_pix"][k]), k
        assert sha(cov) == str(SCALE[f"{name}.rs_cov"][k]), k
    o, vx, dims, values, flags, counts = oracle.compound(sweep, sp["voxel"], sp["margin"])
    assert sha(values) == str(SCALE[f"{name}.cmp_values"])
    assert sha(flags) == str(SCALE[f"{name}.cmp_flags"])
    assert sha(counts) == str(SCALE[f"{name}.cmp_counts"])
    o, vx, dims, values, flags, _ = oracle.compound(SCALE.sweep(name, frames, every=sp["sparse"]), sp["voxel"],
                                                    sp["margin"])
    fv, ff = oracle.fill_holes(values, flags, dims, 3)
    assert sha(fv) == str(SCALE[f"{name}.fill_values"])
    assert sha(ff) == str(SCALE[f"{name}.fill_flags"])
    for k in range(0, len(planes), 8):
        p = planes[k]
        tp, tc, _ = oracle.trilinear(o, vx, dims, fv, ff, oracle.plane_params(p), p.width, p.height)
        assert sha(tp) == str(SCALE[f"{name}.tri_pix"][k]), k
        assert sha(tc) == str(SCALE[f"{name}.tri_cov"][k]), k


@pytest.mark.parametrize("name,cfg", [("cfg1", "cfg1"), ("cfg2", "cfg2")])
def test_bench_geometry_is_the_reference_sweep(name, cfg):
    """bench_data's sweep poses / planes == the reference's SweepPlan.linear and
    Appendix B planes stored with the hashes (so bench and parity tests run the
    same geometry)."""
    if not SCALE.has(name):
        pytest.skip(f"{name} not in scale.npz")
    wl = bench_data.workload(cfg)
    poses, ts = bench_data.sweep_poses(wl)
    q = np.array([[p.rotation.w, p.rotation.x, p.rotation.y, p.rotation.z] for p in poses])
    t = np.array([p.translation for p in poses])
    np.testing.assert_array_equal(q, SCALE[f"{name}.pose_q"])
    np.testing.assert_array_equal(t, SCALE[f"{name}.pose_t"])
    np.testing.assert_array_equal(ts, SCALE[f"{name}.image_ts"])
    planes = bench_data.reslice_planes(wl, len(SCALE[f"{name}.plane_q"]))
    for p, pq, pt in zip(planes, SCALE[f"{name}.plane_q"], SCALE[f"{name}.plane_t"]):
        r = p.pose.rotation
        np.testing.assert_array_equal([r.w, r.x, r.y, r.z], pq)
        np.testing.assert_array_equal(p.pose.translation, pt)
        assert p.pixel_pitch[0] == float(SCALE[f"{name}.plane_pitch"])


def test_oracle_cell_records_equal_its_full_reconstruction():
    """The streamed sampled-cell restatement used at cfg2/cfg3 scale
    (oracle.cell_records) equals the full oracle volume's runs at cfg1 (itself
    pinned to the reference's .darevol above)."""
    frames = SCALE.frames("cfg1")
    sweep = SCALE.sweep("cfg1", frames)
    vol = oracle.reconstruct(sweep, 0.25, 0.0)
    rng = np.random.default_rng(1)
    cells = np.sort(rng.choice(int(np.prod(vol.dims)), 3000, replace=False))
    ref = oracle.cell_records(sweep, vol.origin, vol.voxel_size, vol.dims, cells)
    for c in cells:
        a, b = vol.cell_starts[c], vol.cell_counts[c]
        p, q, i = ref[int(c)]
        assert np.array_equal(p, vol.positions[a:a + b]) and np.array_equal(q, vol.orientations[a:a + b])
        assert np.array_equal(i, vol.intensities[a:a + b])
