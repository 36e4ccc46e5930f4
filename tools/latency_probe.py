"""Single-pose reslice latency breakdown on the cfg2 volume: Python API, raw C-ABI
host call, and device time of the launch sequence (CUDA events)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench_data  # noqa: E402
import paper_2605_26325_b200 as db  # noqa: E402
from paper_2605_26325_b200 import _lib  # noqa: E402
from paper_2605_26325_b200.reslice import ResliceConfig, kernel_cfg, plane_params  # noqa: E402

wl = bench_data.workload("cfg2")
frames = bench_data.render_frames_torch(wl)
torch.cuda.synchronize()
poses, ts = bench_data.sweep_poses(wl)
from types import SimpleNamespace  # noqa: E402
sw = SimpleNamespace(images=frames, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                     pixel_pitch=(wl.pitch, wl.pitch), calibration=db.Pose.identity(), mask=None)
vol = db.reconstruct_volume(sw, voxel_size=wl.voxel, margin=0.0)
cfg = ResliceConfig(interp_radius=wl.voxel)
planes = bench_data.reslice_planes(wl, 200, seed=3)
for p in planes[:20]:
    db.reslice(vol, p, cfg)
t_py = []
for p in planes:
    t0 = time.perf_counter()
    db.reslice(vol, p, cfg)
    t_py.append((time.perf_counter() - t0) * 1e3)
kc = kernel_cfg(cfg)
h = vol.device_handle().raw
px = torch.empty((256, 256), dtype=torch.uint8).pin_memory().numpy()
cv = torch.empty((256, 256), dtype=torch.uint8).pin_memory().numpy()
prm = [np.ascontiguousarray(plane_params(p), dtype=np.float64) for p in planes]
t_c = []
for q in prm:
    t0 = time.perf_counter()
    _lib.call("dare_reslice", h, 1, _lib.ptr(q, ctypes.c_double), 256, 256, ctypes.byref(kc),
              _lib.ptr(px, ctypes.c_uint8), _lib.ptr(cv, ctypes.c_uint8))
    t_c.append((time.perf_counter() - t0) * 1e3)
prm_d = torch.from_numpy(np.stack(prm)).cuda()
out = torch.empty((2, 256, 256), dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
t_d = []
with torch.cuda.stream(st):
    for k in range(len(prm)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.call("dare_reslice_device", h, 1, ctypes.c_void_p(prm_d[k].data_ptr()), 256, 256, ctypes.byref(kc),
                  ctypes.c_void_p(out[0].data_ptr()), ctypes.c_void_p(out[1].data_ptr()), ctypes.c_void_p(st.cuda_stream))
        e1.record(st)
        st.synchronize()
        t_d.append(e0.elapsed_time(e1))
print(f"p50 ms: python reslice() {np.percentile(t_py, 50):.4f}  C-ABI dare_reslice {np.percentile(t_c, 50):.4f}  "
      f"device (events around dare_reslice_device) {np.percentile(t_d, 50):.4f}")
