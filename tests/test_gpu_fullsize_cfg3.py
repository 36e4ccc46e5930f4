"""Full-size cfg3 (BASELINE configs[2]: 8000 frames of 512x512 in four sweeps ->
512^3 grid, 2.1 G samples) through size-independent properties, plus bit-exact
slab-oracle parity of reslices at that size: 64x64 patches of
512x512 planes, and a cfg4-style trajectory batch against single-pose calls."""
import numpy as np
import pytest

import bench_data
import paper_2605_26325_b200 as db

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg3():
    import torch

    wl = bench_data.workload("cfg3")
    frames = bench_data.render_frames_torch(wl)
    poses, ts = bench_data.sweep_poses(wl)
    from types import SimpleNamespace

    sweep = SimpleNamespace(images=frames, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                            pixel_pitch=(wl.pitch, wl.pitch), calibration=db.Pose.identity(), mask=None)
    vol = db.reconstruct_volume(sweep, voxel_size=wl.voxel, margin=0.0)
    torch.cuda.synchronize()
    yield wl, sweep, vol
    del vol
    torch.cuda.empty_cache()


def test_cfg3_csr_invariants(cfg3):
    import torch

    from paper_2605_26325_b200.parallel import _CudaArray

    wl, sweep, vol = cfg3
    info = vol.device_info()
    n_px = wl.n_frames * wl.size * wl.size
    assert int(info.n_samples) + vol.rejected_out_of_bounds == n_px
    assert int(info.n_samples) > 0.99 * n_px
    dims = tuple(int(d) for d in info.dims)
    nc = int(np.prod(dims))
    off = torch.as_tensor(_CudaArray(info.d_cell_offsets, (nc + 1,), "<i4"), device="cuda").long() & 0xFFFFFFFF
    rec = torch.as_tensor(_CudaArray(info.d_records, (int(info.n_samples), 4), "<i4"), device="cuda")
    counts = off[1:] - off[:-1]
    assert int(counts.min()) >= 0 and int(off[-1]) == int(info.n_samples)
    # intensity multiset: input pixels (in-bounds ones) == stored records, chunked
    hist_in = torch.zeros(256, dtype=torch.long, device="cuda")
    for f0 in range(0, wl.n_frames, 500):
        hist_in += torch.bincount(sweep.images[f0:f0 + 500].reshape(-1).long(), minlength=256)
    hist_out = torch.zeros(256, dtype=torch.long, device="cuda")
    for s0 in range(0, rec.shape[0], 1 << 28):
        hist_out += torch.bincount((rec[s0:s0 + (1 << 28), 3] & 0xFF).long(), minlength=256)
    assert bool((hist_in >= hist_out).all())
    assert int((hist_in - hist_out).sum()) == vol.rejected_out_of_bounds
    # sampled cells: every record of the cell lies in it (floor((f64(p32) - o) / voxel))
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    cells = torch.randint(0, nc, (200_000,), device="cuda", generator=g)
    starts, n = off[cells], counts[cells]
    cell = torch.repeat_interleave(cells, n)
    idx_in = torch.repeat_interleave(starts, n) + (torch.arange(int(n.sum()), device="cuda")
                                                   - torch.repeat_interleave(torch.cumsum(n, 0) - n, n))
    pos = rec[idx_in, :3].view(torch.float32).double()
    o = torch.tensor(info.origin, dtype=torch.float64, device="cuda")
    ijk = torch.floor((pos - o) / info.voxel_size).long()
    lin = (ijk[:, 0] * dims[1] + ijk[:, 1]) * dims[2] + ijk[:, 2]
    assert bool((lin == cell).all())
    assert int(info.n_orientations) == 4  # one canonical f32 quaternion per sweep


def test_cfg3_reslice_patches_match_slab_oracle(cfg3):
    import bench

    wl, sweep, vol = cfg3
    host = bench.host_sweep(wl, sweep.images.cpu().numpy())
    cfg = db.ResliceConfig(interp_radius=wl.voxel)
    planes = [bench.patch_plane(p, 64) for p in bench_data.reslice_planes(wl, 2, seed=11)]
    slab = bench.OracleSlab(wl, host)
    px, cov, _ = db.reslice_batch(vol, planes, cfg)
    for k, plane in enumerate(planes):
        _, rp, rc, nf = slab.reslice(plane, cfg)
        assert 0 < nf < wl.n_frames
        np.testing.assert_array_equal(px[k], rp)
        np.testing.assert_array_equal(cov[k], rc)
        assert rc.mean() > 0.5


def test_cfg4_trajectory_batch_equals_single_calls(cfg3):
    wl, _, vol = cfg3
    cfg = db.ResliceConfig(interp_radius=wl.voxel)
    traj = bench_data.trajectory_planes(bench_data.workload("cfg4"), 40, seed=2)
    px, cov, _ = db.reslice_batch(vol, traj, cfg)  # coherent batch: the auto schedule's choice
    for k in (0, 17, 39):
        one = db.reslice(vol, traj[k], cfg)
        np.testing.assert_array_equal(px[k], one.pixels)
        np.testing.assert_array_equal(cov[k], one.coverage)
    assert cov.mean() > 0.5


def test_cfg3_sampled_cells_records_match_slab_oracle(cfg3):
    """SURVEY §8c (1) at BASELINE configs[2] scale (2.1 G samples, four sweeps):
    100k random cells' exact insertion-order sample lists streamed from the
    8000 frames by the oracle, against the device volume read through perm."""
    import bench
    from cells_io import assert_cells_equal, device_cell_records
    from oracle import oracle

    wl, sweep, vol = cfg3
    host = bench.host_sweep(wl, sweep.images.cpu().numpy())
    rng = np.random.default_rng(31)
    cells = np.sort(rng.choice(int(np.prod(vol.dims)), 100_000, replace=False))
    ref = oracle.cell_records(host, vol.origin, vol.voxel_size, vol.dims, cells)
    n = assert_cells_equal(device_cell_records(vol, cells), ref)
    assert n > 1_000_000


def test_cfg4_trajectory_patches_match_slab_oracle(cfg3):
    """cfg4 (haptic trajectory on the cfg3 volume): 64x64 centre patches of
    trajectory planes from different base orientations against the slab
    oracle, bit-exact."""
    import bench

    wl, sweep, vol = cfg3
    host = bench.host_sweep(wl, sweep.images.cpu().numpy())
    cfg = db.ResliceConfig(interp_radius=wl.voxel)
    traj = bench_data.trajectory_planes(bench_data.workload("cfg4"), 7501, seed=4)
    planes = [bench.patch_plane(traj[k], 64) for k in (300, 7500)]  # bases A and D
    slab = bench.OracleSlab(wl, host)
    px, cov, _ = db.reslice_batch(vol, planes, cfg)
    for k, plane in enumerate(planes):
        _, rp, rc, nf = slab.reslice(plane, cfg)
        np.testing.assert_array_equal(px[k], rp)
        np.testing.assert_array_equal(cov[k], rc)
