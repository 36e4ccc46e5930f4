"""The CUDA halves of the sharded paths, with R ranks emulated on one GPU:
R partial volumes (consecutive frame blocks into the full grid) merged by
dare_volume_merge must equal the single-GPU reconstruction bit-for-bit; R
partial compound accumulators summed must equal compound()."""
import numpy as np
import pytest

import paper_2605_26325_b200 as db
from oracle import oracle
from paper_2605_26325_b200 import parallel
from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.sweep import grid_for, plan_frames

pytestmark = pytest.mark.gpu


def _sweep(seed, n=60, h=37, w=41):
    rng = np.random.default_rng(seed)
    poses = [Pose(Quaternion.from_axis_angle((1, 0.3, 0), 0.02 * k), (0.01 * k, 0.0, 0.06 * k)) for k in range(n)]
    ts = np.arange(n) / 30.0
    return db.SweepRecording(rng.integers(0, 256, (n, h, w), dtype=np.uint8), ts, ts, poses, (0.1, 0.1))


def _raw(vol):
    import torch

    info = vol.device_info()
    nc, n, no = int(np.prod(info.dims)), int(info.n_samples), int(info.n_orientations)
    t = lambda p, shape, ts: torch.as_tensor(parallel._CudaArray(p, shape, ts), device="cuda").cpu().numpy()  # noqa
    return {"offsets": t(info.d_cell_offsets, (nc + 1,), "<i4"), "records": t(info.d_records, (n, 4), "<i4"),
            "perm": t(info.d_perm, (n,), "|i1"), "bins": t(info.d_bins, (nc,), "<i4"),
            "orient": t(info.d_orientations, (no, 4), "<f4"), "n_orient": np.array(no)}


@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
def test_merge_of_frame_blocks_equals_single_build(ranks):
    sweep = _sweep(ranks)
    full = db.reconstruct_volume(sweep, voxel_size=0.2, margin=0.3)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, 0.2, 0.3)
    parts = [parallel.CudaOps.reconstruct_subset(sweep, plan, s, e, origin, voxel, dims)
             for s, e in parallel.blocks(plan.n_frames, ranks)]
    merged = parallel.CudaOps.merge([parallel.CudaOps.part_of(p) for p in parts], origin, voxel, dims)
    for name in ("cell_starts", "cell_counts", "positions", "orientations", "intensities"):
        np.testing.assert_array_equal(getattr(merged, name), getattr(full, name), err_msg=name)
    assert sum(p.rejected_out_of_bounds for p in parts) == full.rejected_out_of_bounds
    # the device records themselves are identical in insertion order (read through
    # perm), including the orientation ids: the merge deduplicates the parts'
    # orientation tables, so merged replicas keep the single-orientation fast path
    a, b = _raw(full), _raw(merged)
    for name in ("offsets", "orient", "n_orient"):
        np.testing.assert_array_equal(a[name], b[name], err_msg=name)
    j = np.arange(len(a["perm"]))
    np.testing.assert_array_equal(a["records"][j + a["perm"]], b["records"][j + b["perm"]])


def test_merged_volume_reslices_identically():
    sweep = _sweep(9)
    full = db.reconstruct_volume(sweep, voxel_size=0.125, margin=0.0)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, 0.125, 0.0)
    parts = [parallel.CudaOps.reconstruct_subset(sweep, plan, s, e, origin, voxel, dims)
             for s, e in parallel.blocks(plan.n_frames, 4)]
    merged = parallel.CudaOps.merge([parallel.CudaOps.part_of(p) for p in parts], origin, voxel, dims)
    planes = [db.ReslicePlane(Pose(Quaternion.from_axis_angle((1, 0, 0), 0.05 * k), (0.3, 0.2, 0.5 + 0.4 * k)),
                              30, 26, (0.11, 0.11)) for k in range(6)]
    cfg = db.ResliceConfig(interp_radius=0.125)
    a, ca, _ = db.reslice_batch(full, planes, cfg)
    b, cb, _ = db.reslice_batch(merged, planes, cfg)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ca, cb)
    assert ca.any()


@pytest.mark.parametrize("ranks", [2, 5])
def test_compound_partials_sum_to_compound(ranks):
    import torch

    sweep = _sweep(20 + ranks)
    ref = db.compound(sweep, voxel_size=0.2, margin=0.3)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, 0.2, 0.3)
    acc = sum(parallel.CudaOps.compound_partial(sweep, plan, s, e, origin, voxel, dims)
              for s, e in parallel.blocks(plan.n_frames, ranks))
    out = parallel.CudaOps.scalar_from_sums(acc.contiguous(), origin, voxel, dims)
    np.testing.assert_array_equal(out.values, ref.values)
    np.testing.assert_array_equal(out.flags, ref.flags)
    np.testing.assert_array_equal(out.counts, ref.counts)
    _, _, _, v, f, c = oracle.compound(sweep, 0.2, 0.3)
    np.testing.assert_array_equal(out.values, v)
    assert torch.is_tensor(acc)
