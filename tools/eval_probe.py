"""Times dare_similarity on a cfg2-like batch (128 pairs of 256x256 u8 with
coverage masks) on device tensors; used with ncu to size its two kernels."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2605_26325_b200 import evaluation as ev  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rng = np.random.default_rng(0)
t = np.clip(np.cumsum(rng.integers(-9, 10, (P, 256, 256)), axis=2) + 128, 0, 255).astype(np.uint8)
c = np.clip(t.astype(int) + rng.integers(-20, 21, t.shape), 0, 255).astype(np.uint8)
yy, xx = np.mgrid[0:256, 0:256]
cov = np.broadcast_to((yy - 128) ** 2 + (xx - 128) ** 2 < 110 ** 2, t.shape)
a, b, m = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (c, t, cov))
ev.similarity_batch(a, b, m, None)
best = None
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ev.similarity_batch(a, b, m, None)
    e1.record()
    e1.synchronize()
    best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
print(f"pairs={P} best_ms={best:.3f} pairs_per_s={P / best * 1e3:.0f} ssim0={r.ssim[0]!r} ncc0={r.ncc[0]!r}")

# breakdown: the raw C-ABI call on prepared device buffers vs the Python wrapper
from paper_2605_26325_b200 import _lib  # noqa: E402

mu8 = m.to(torch.uint8).contiguous()
out = [torch.empty(P, dtype=dt, device="cuda") for dt in (torch.float64, torch.float64, torch.int64, torch.int32)]
stream = torch.cuda.current_stream().cuda_stream
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("dare_similarity_device", P, 256, 256, 0, a.data_ptr(), mu8.data_ptr(), b.data_ptr(), None, 7,
              ev.SSIM_C1, ev.SSIM_C2, *(o.data_ptr() for o in out), stream)
    e1.record()
    e1.synchronize()
    t1 = time.perf_counter()
    print(f"raw call: events {e0.elapsed_time(e1):.3f} ms, wall {1e3 * (t1 - t0):.3f} ms")
