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
