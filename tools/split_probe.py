"""Device time of small pixel-major batches (P = 1, 2, 4 poses of 256x256 on the
cfg2 volume) for each threads-per-pixel split (DARE_SPLIT override)."""
import ctypes
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for sp in ("1", "2", "4", ""):
        env = dict(os.environ, DARE_SPLIT=sp) if sp else dict(os.environ)
        env.pop("DARE_SPLIT", None) if not sp else None
        print(f"split={sp or 'auto'}:", subprocess.run([sys.executable, __file__, "run"], env=env,
                                                       capture_output=True, text=True).stdout.strip())
    sys.exit(0)

import numpy as np
import torch

sys.path.insert(0, ".")
import bench_data  # noqa: E402
import paper_2605_26325_b200 as db  # noqa: E402
from paper_2605_26325_b200 import _lib  # noqa: E402
from paper_2605_26325_b200.reslice import ResliceConfig, kernel_cfg, plane_params  # noqa: E402
from types import SimpleNamespace  # noqa: E402

wl = bench_data.workload("cfg2")
frames = bench_data.render_frames_torch(wl)
poses, ts = bench_data.sweep_poses(wl)
sw = SimpleNamespace(images=frames, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                     pixel_pitch=(wl.pitch, wl.pitch), calibration=db.Pose.identity(), mask=None)
vol = db.reconstruct_volume(sw, voxel_size=wl.voxel, margin=0.0)
cfg = ResliceConfig(interp_radius=wl.voxel)
kc = kernel_cfg(cfg)
h = vol.device_handle().raw
planes = bench_data.reslice_planes(wl, 400, seed=3)
prm_d = torch.from_numpy(np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)).cuda()
out = torch.empty((2, 4, 256, 256), dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
res = []
for P in (1, 2, 4):
    t = []
    with torch.cuda.stream(st):
        for k in range(0, 400 - P, P):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.call("dare_reslice_device", h, P, ctypes.c_void_p(prm_d[k].data_ptr()), 256, 256, ctypes.byref(kc),
                      ctypes.c_void_p(out[0].data_ptr()), ctypes.c_void_p(out[1].data_ptr()),
                      ctypes.c_void_p(st.cuda_stream))
            e1.record(st)
            st.synchronize()
            t.append(e0.elapsed_time(e1))
    res.append(f"P={P}: {np.percentile(t[10:], 50) * 1000:.1f} us")
print("  ".join(res))
