import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import paper_2605_26325_b200 as db
from paper_2605_26325_b200 import parallel
from paper_2605_26325_b200.sweep import grid_for, plan_frames
from oracle import oracle
from test_gpu_parallel import _sweep
for ranks in (2, 8):
    sweep = _sweep(ranks)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, 0.2, 0.3)
    full = db.reconstruct_volume(sweep, voxel_size=0.2, margin=0.3)
    of = oracle.reconstruct(sweep, 0.2, 0.3)
    print("full vs oracle", np.array_equal(np.asarray(full.positions), np.asarray(of.positions)),
          np.array_equal(np.asarray(full.cell_counts), np.asarray(of.cell_counts)), flush=True)
    fr = oracle.frame_poses(sweep)
    for k, (s, e) in enumerate(parallel.blocks(plan.n_frames, ranks)):
        p = parallel.CudaOps.reconstruct_subset(sweep, plan, s, e, origin, voxel, dims)
        ref = oracle.reconstruct_subset(sweep, fr[s:e], origin, voxel, dims)
        dl, rp = np.asarray(p.positions), np.asarray(ref.positions)
        cc, rc = np.asarray(p.cell_counts), np.asarray(ref.cell_counts)
        bad = np.nonzero(np.any(dl != rp, axis=1))[0] if dl.shape == rp.shape else []
        print(f"ranks {ranks} part {k} n={len(dl)} counts_eq {np.array_equal(cc, rc)} pos mismatches {len(bad)}", flush=True)
        if len(bad):
            i = bad[0]
            starts = np.asarray(p.cell_starts)
            c = np.searchsorted(starts, i, side='right') - 1
            print("  first bad idx", i, "cell", c, "count", cc[c], "start", starts[c])
            print("  gpu", dl[starts[c]:starts[c]+cc[c]].tolist())
            print("  ref", rp[starts[c]:starts[c]+cc[c]].tolist())
            break
