"""Full-size (BASELINE configs[1] = cfg2: 1000 x 512x512 -> 256^3, 262M samples)
checks through size-independent properties, plus bit-exact slab-oracle parity
of full 256x256 reslices (only the frames that can reach the
plane's cells are reconstructed on the CPU, into the full grid)."""
import numpy as np
import pytest

import bench_data
import paper_2605_26325_b200 as db
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2():
    import torch

    wl = bench_data.workload("cfg2")
    frames = bench_data.render_frames_torch(wl)
    poses, ts = bench_data.sweep_poses(wl)
    from types import SimpleNamespace

    sweep = SimpleNamespace(images=frames, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                            pixel_pitch=(wl.pitch, wl.pitch), calibration=db.Pose.identity(), mask=None)
    vol = db.reconstruct_volume(sweep, voxel_size=wl.voxel, margin=0.0)
    torch.cuda.synchronize()
    return wl, sweep, vol


def _device_arrays(vol):
    import torch

    from paper_2605_26325_b200.parallel import _CudaArray

    info = vol.device_info()
    nc = int(np.prod(info.dims))
    off = torch.as_tensor(_CudaArray(info.d_cell_offsets, (nc + 1,), "<i4"), device="cuda").long() & 0xFFFFFFFF
    rec = torch.as_tensor(_CudaArray(info.d_records, (int(info.n_samples), 4), "<i4"), device="cuda")
    return info, off, rec


def test_cfg2_csr_invariants(cfg2):
    import torch

    wl, sweep, vol = cfg2
    info, off, rec = _device_arrays(vol)
    n_px = wl.n_frames * wl.size * wl.size
    assert vol.dims == (256, 256, 256)
    assert int(info.n_samples) + vol.rejected_out_of_bounds == n_px
    counts = off[1:] - off[:-1]
    assert int(counts.min()) >= 0 and int(off[-1]) == int(info.n_samples)
    # every record lies in its cell: floor((f64(p32) - origin) / voxel) == cell of its slot
    cell = torch.repeat_interleave(torch.arange(len(counts), device="cuda"), counts)
    pos = rec[:, :3].view(torch.float32).double()
    o = torch.tensor(info.origin, dtype=torch.float64, device="cuda")
    idx = torch.floor((pos - o) / info.voxel_size).long()
    lin = (idx[:, 0] * 256 + idx[:, 1]) * 256 + idx[:, 2]
    assert bool((lin == cell).all())
    # intensity multiset == input pixels (nothing lost or duplicated)
    hist_in = torch.bincount(sweep.images.reshape(-1).long(), minlength=256)
    hist_out = torch.bincount((rec[:, 3] & 0xFF).long(), minlength=256)
    assert bool((hist_in == hist_out).all())


def test_cfg2_reslice_matches_slab_oracle(cfg2):
    import bench

    wl, sweep, vol = cfg2
    host = bench.host_sweep(wl, sweep.images.cpu().numpy())
    planes = bench_data.reslice_planes(wl, 2, seed=5)
    cfg = db.ResliceConfig(interp_radius=wl.voxel)
    slab = bench.OracleSlab(wl, host)
    px, cov, _ = db.reslice_batch(vol, planes, cfg)
    for k, plane in enumerate(planes):
        _, rp, rc, nf = slab.reslice(plane, cfg)
        assert nf < wl.n_frames
        np.testing.assert_array_equal(px[k], rp)
        np.testing.assert_array_equal(cov[k], rc)
        assert rc.mean() > 0.5


def test_cfg2_compound_matches_oracle_on_slab(cfg2):
    """compound over the full sweep vs the oracle's per-frame integer sums."""
    import torch

    wl, sweep, vol = cfg2
    s = db.compound(sweep, voxel_size=wl.voxel, margin=0.0)
    counts = torch.from_numpy(np.asarray(s.counts))
    assert int(counts.sum()) == wl.n_frames * wl.size * wl.size
    # a few frames' worth of cells checked exactly against the oracle
    host = sweep.images[:3].cpu().numpy()
    from types import SimpleNamespace

    frames = oracle.frame_poses(SimpleNamespace(images=host, image_timestamps=sweep.image_timestamps[:3],
                                                pose_timestamps=sweep.pose_timestamps, poses=sweep.poses,
                                                calibration=sweep.calibration))
    lin, _ = oracle.frame_cells(frames[0], wl.size, wl.size, sweep.pixel_pitch, s.origin, wl.voxel, s.dims)
    assert (lin >= 0).all()
    assert (np.asarray(s.flags)[lin] == 1).all()


def test_cfg2_sampled_cells_records_match_slab_oracle(cfg2):
    """SURVEY §8c (1) at BASELINE configs[1] scale: for 100k random cells the
    exact sample list in the reference's insertion order (positions' bits,
    canonical f32 quaternions, intensities) streamed from the frames by the
    oracle, against the device volume read through perm."""
    import bench
    from cells_io import assert_cells_equal, device_cell_records

    wl, sweep, vol = cfg2
    host = bench.host_sweep(wl, sweep.images.cpu().numpy())
    rng = np.random.default_rng(21)
    cells = np.sort(rng.choice(int(np.prod(vol.dims)), 100_000, replace=False))
    ref = oracle.cell_records(host, vol.origin, vol.voxel_size, vol.dims, cells)
    n = assert_cells_equal(device_cell_records(vol, cells), ref)
    assert n > 1_000_000


def test_cfg2_certified_equals_exact_on_1024_poses(cfg2):
    """The certified f32 path against the FP64-everywhere path on 1024 cfg2
    poses (256^2): identical pixels and coverage (stress of the
    error bound at the headline config)."""
    import ctypes

    from paper_2605_26325_b200 import _lib
    from paper_2605_26325_b200.reslice import kernel_cfg, plane_params

    wl, sweep, vol = cfg2
    planes = bench_data.reslice_planes(wl, 1024, seed=77)
    cfg = db.ResliceConfig(interp_radius=wl.voxel)
    params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
    h = w = wl.plane
    out = {}
    fb = {}
    for exact in (0, 1):
        px = np.empty((len(planes), h, w), np.uint8)
        cov = np.empty((len(planes), h, w), np.uint8)
        kc = kernel_cfg(cfg, 0, exact=bool(exact))
        _lib.call("dare_reslice", vol.device_handle().raw, len(planes), _lib.ptr(params, ctypes.c_double), w, h,
                  ctypes.byref(kc), _lib.ptr(px, ctypes.c_uint8), _lib.ptr(cov, ctypes.c_uint8))
        n = ctypes.c_int64()
        _lib.call("dare_reslice_last_fallback", ctypes.byref(n))
        out[exact], fb[exact] = (px, cov), n.value
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    assert fb[1] == 0 and 0 < fb[0] < 0.01 * len(planes) * h * w
