"""Probe: per-call device span of compound() at cfg2 (DARE_PROFILE phases on stderr)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, bench_data
import paper_2605_26325_b200 as db
from types import SimpleNamespace
from paper_2605_26325_b200.geometry import Pose
wl = bench_data.workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
frames = bench_data.render_frames_torch(wl)
poses, ts = bench_data.sweep_poses(wl)
sw = SimpleNamespace(images=frames, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                     pixel_pitch=(wl.pitch, wl.pitch), calibration=Pose.identity(), mask=None)
for i in range(6):
    t0 = time.perf_counter()
    s = db.compound(sw, voxel_size=wl.voxel, margin=0.0)
    w = (time.perf_counter() - t0) * 1e3
    print(f"call {i}: wall {w:.3f} ms, device span {bench.last_device_ms():.3f} ms", flush=True)
    del s
