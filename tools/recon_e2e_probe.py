import sys, time, torch
sys.path.insert(0, '.')
import bench, bench_data
import paper_2605_26325_b200 as db
wl = bench_data.workload('cfg2')
frames_d = bench_data.render_frames_torch(wl); torch.cuda.synchronize()
pinned = frames_d.cpu().pin_memory()
sw = bench.host_sweep(wl, pinned.numpy())
for i in range(4):
    t0 = time.perf_counter(); v = db.reconstruct_volume(sw, voxel_size=wl.voxel, margin=0.0); t1 = time.perf_counter()
    print(f"e2e {1e3*(t1-t0):.2f} ms", file=sys.stderr)
    del v
t0 = time.perf_counter(); x = pinned.cuda(); torch.cuda.synchronize(); print(f"plain H2D {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr)
# frames already in HBM (bench `recon.ms` path)
swd = bench.host_sweep(wl, frames_d)  # images as a CUDA tensor
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v = db.reconstruct_volume(swd, voxel_size=wl.voxel, margin=0.0); torch.cuda.synchronize()
    print(f"device-frames {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr)
    del v
# host-side planning alone (synchronize + bounds + per-frame axes/quaternions)
from paper_2605_26325_b200 import sweep as _sw
for i in range(3):
    t0 = time.perf_counter(); plan = _sw.plan_frames(swd); g = _sw.grid_for(plan, wl.voxel, 0.0)
    plan.axes(); plan.canonical_quats_f32()
    print(f"host plan {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr)
