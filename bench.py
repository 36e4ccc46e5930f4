#!/usr/bin/env python
"""Benchmark of the DARE hot paths on B200 (BASELINE.json metric:
"reslices/sec and p50 reslice latency; recon input Mpix/sec; % HBM roofline").

Workload (N=1): BASELINE.json configs[1], cfg2 -- 1000 frames 512x512 -> 256^3
directional grid, reslices at 256x256 (SURVEY Appendix B geometry, synthetic
content).  A step = one batch of B=64 reslice poses through the device path.

  value      reslices/s over all ranks, inputs (volume, pose params) resident
             in HBM, CUDA events on the launching stream, max over ranks
  e2e        reslices/s through the C ABI host-buffer call (dare_reslice):
             per step H2D of 64 x 14 f64 pose params and D2H of pixels+coverage
  latency    p50/p95 of single-pose reslice() through the public API
  recon      reconstruct_volume input Mpix/s (frames in HBM, and e2e from pinned host)
  roofline   dominant kernel (reslice_fast_k) algorithmic bytes (SURVEY §8d
             reference-layout formula) / measured step time vs MEASURED_PEAKS hbm_gbs
  cpu_baseline  CPU oracle (oracle/, C + OpenMP) on a bounded sample (slab oracle)

`--impl reference` times the reference's CPU algorithm (the oracle port; the
reference is pure Python/numba and is not installed on the GPU box) on the same
config, rank 0 only.  Multi-GPU (torchrun): every rank builds its replica of
the volume and reslices its own poses (pose-sharded, no data-path collective;
scaling "weak").
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bench_data  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="cfg2", choices=sorted(bench_data.CONFIGS))
    p.add_argument("--batch", type=int, default=0, help="poses per step (default: config's)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-scalar", action="store_true", help="skip the direction-blind arm timings")
    p.add_argument("--schedule", type=int, default=0, choices=[0, 1, 2],
                   help="reslice schedule: 0 auto (as dare_reslice decides), 1 pixel-major, 2 pose-major")
    p.add_argument("--exact", action="store_true",
                   help="FP64 reference arithmetic for every pixel (default: certified f32 + exact fallback)")
    return p.parse_args()


# ----------------------------------------------------------------------------- helpers

class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    polled every 2 ms from a thread (a cfg2 timed region is ~40 ms), with
    nvidia-smi -lms 50 as the fallback when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, int]] = []
        self.nvml = None
        self._stop = threading.Event()
        self._thread = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _poll(self):
        p = self.nvml
        while not self._stop.is_set():
            try:
                sm = float(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
                reasons = int(p.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                self.samples.append((sm, self.smax, reasons))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.nvml is not None:
            self._stop.set()
            self._thread.join(timeout=2)
            p = self.nvml
            bits = {"hw_slowdown": p.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": p.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": p.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": p.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted({n for _, _, r in self.samples for n, b in bits.items() if r & b})
            sm = [x for x, _, _ in self.samples]
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax, "reasons": reasons,
                    "samples": len(sm), "source": "nvml, 2 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(self.NAMES, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi, 50 ms"}


class DevArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def cells_visited(torch, dims, origin, voxel, p14, W, H, radius):
    dev = "cuda"
    u = torch.arange(W, device=dev, dtype=torch.float64)
    v = torch.arange(H, device=dev, dtype=torch.float64)
    du = (u * p14[12])[None, :]
    dv = (v * p14[13])[:, None]
    inv_v = 1.0 / voxel
    lo, hi = [], []
    for a, (ci, cj) in enumerate(((3, 4), (6, 7), (9, 10))):
        w = (p14[a] + du * p14[ci]) + dv * p14[cj]
        l = torch.floor(((w - radius) - origin[a]) * inv_v - 1e-9).clamp(min=0)
        h = torch.floor(((w + radius) - origin[a]) * inv_v + 1e-9).clamp(max=dims[a] - 1)
        lo.append(l.reshape(-1).long())
        hi.append(h.reshape(-1).long())
    span = [int((hi[a] - lo[a]).max().item()) + 1 for a in range(3)]
    cells = []
    for ox in range(max(span[0], 0)):
        for oy in range(max(span[1], 0)):
            for oz in range(max(span[2], 0)):
                cx, cy, cz = lo[0] + ox, lo[1] + oy, lo[2] + oz
                ok = (cx <= hi[0]) & (cy <= hi[1]) & (cz <= hi[2])
                lin = (cx * dims[1] + cy) * dims[2] + cz
                cells.append(lin[ok])
    if not cells:
        return torch.empty(0, dtype=torch.long, device=dev)
    return torch.unique(torch.cat(cells))


def _pow2(x: float) -> bool:
    m, _ = math.frexp(x)
    return x > 0 and m == 0.5


def ncu_traffic(kernel: str, batch: int, config: str):
    """DRAM bytes (read+write) per launch of `kernel` from the committed ncu capture
    (profiles/round1_traffic.json, cfg2 with 64 poses per launch), or None."""
    path = os.path.join(ROOT, "profiles", "round2_traffic.json")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "profiles", "round1_traffic.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        if config != "cfg2" or batch != 64:
            return None, "ncu capture is for cfg2 / 64 poses per launch"
        table = data["dram_bytes_per_launch"]
        # (captures before the parts-per-pixel template argument printed it as the bool 0)
        alt = kernel[:-2] + "0>" if kernel.endswith(", 1>") else kernel
        key = kernel if kernel in table else alt
        return float(table[key]), f"profiles/{os.path.basename(path)} (" + data["source"] + ")"
    except Exception as e:  # noqa: BLE001
        return None, f"no ncu capture ({type(e).__name__})"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def host_cores() -> dict:
    n = os.cpu_count() or 1
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = n
    return {"cpu_count": n, "affinity": avail, "model": cpu_model()}


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` (N > 1, devices checked by main) without a torchrun
    environment: relaunch this script under torch.distributed.run with N ranks
    on 127.0.0.1 (NCCL_DEBUG=INFO, so every rank's communicator is logged)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def last_device_ms() -> float:
    """Device span (CUDA events on the library's stream) of this thread's last
    reconstruct / compound / fill_holes C-ABI call."""
    from paper_2605_26325_b200 import _lib

    ms = ctypes.c_double(-1.0)
    _lib.call("dare_last_device_ms", ctypes.byref(ms))
    return float(ms.value)


def recon_traffic(config: str):
    """ncu DRAM bytes (read + write) of one reconstruction's kernels, from the
    committed capture (profiles/round2_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "round2_traffic.json")) as fh:
            data = json.load(fh)
        rec = data.get("recon", {}).get(config)
        return (float(rec["dram_bytes"]), "profiles/round2_traffic.json (" + data["source"] + ")") if rec else \
            (None, f"no ncu capture of the {config} reconstruction")
    except Exception as e:  # noqa: BLE001
        return None, f"no ncu capture ({type(e).__name__})"


def make_rank_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- CPU oracle legs

def patch_plane(plane, size: int):
    """A size x size sub-plane at the centre of `plane` (same orientation and pitch):
    the same per-pixel work, used to bound CPU samples of 512x512 planes."""
    from paper_2605_26325_b200.geometry import Pose, rotation_matrix
    from paper_2605_26325_b200.reslice import ReslicePlane

    if size >= plane.width and size >= plane.height:
        return plane
    u0, v0 = (plane.width - size) // 2, (plane.height - size) // 2
    r = rotation_matrix(plane.pose.rotation)
    t = plane.pose.translation + r @ np.array([u0 * plane.pixel_pitch[0], v0 * plane.pixel_pitch[1], 0.0])
    return ReslicePlane(Pose(plane.pose.rotation, t), size, size, plane.pixel_pitch)


class OracleSlab:
    """Bounded CPU-oracle sample of a reslice (SURVEY §8c slab oracle): only the
    frames whose image rectangle comes within one voxel of the plane's pixel
    cubes are reconstructed, into the FULL grid -- every cell the plane visits
    is then complete, so the oracle reslice is exact for that plane."""

    def __init__(self, wl, sweep):
        from oracle import oracle

        self.o = oracle
        self.sweep = sweep
        self.frames = oracle.frame_poses(sweep)
        self.grid = oracle.grid(self.frames, wl.size, wl.size, sweep.pixel_pitch, wl.voxel, 0.0)
        umax, vmax = (wl.size - 1) * wl.pitch, (wl.size - 1) * wl.pitch
        lo, hi = [], []
        for f in self.frames:
            c = np.array([oracle._rot(f.quat, (uu, vv, 0.0)) + f.trans
                          for uu, vv in ((0.0, 0.0), (umax, 0.0), (0.0, vmax), (umax, vmax))])
            lo.append(c.min(axis=0))
            hi.append(c.max(axis=0))
        self.flo, self.fhi = np.array(lo), np.array(hi)

    def volume_for(self, plane, radius):
        p = self.o.plane_params(plane)
        t, c0, c1 = p[0:3], p[[3, 6, 9]], p[[4, 7, 10]]
        pts = np.array([t + a * c0 + b * c1 for a in (0.0, (plane.width - 1) * p[12])
                        for b in (0.0, (plane.height - 1) * p[13])])
        pad = radius + 2 * self.grid[1]
        rlo, rhi = pts.min(axis=0) - pad, pts.max(axis=0) + pad
        keep = np.all((self.fhi >= rlo) & (self.flo <= rhi), axis=1)
        sub = [f for f, k in zip(self.frames, keep) if k]
        origin, voxel, dims = self.grid
        return self.o.reconstruct_subset(self.sweep, sub, origin, voxel, dims), len(sub)

    def reslice(self, plane, cfg):
        vol, nf = self.volume_for(plane, cfg.interp_radius)
        p = self.o.plane_params(plane)
        t0 = time.perf_counter()
        px, cov = self.o.reslice(vol, p, self.o.cfg_array(cfg), plane.width, plane.height, cfg.unassigned_value)
        return (time.perf_counter() - t0) * 1000.0, px, cov, nf


def oracle_baseline(wl, sweep, plane, cfg, gpu_px=None, gpu_cov=None, reps: int = 3):
    """CPU oracle (C; reslice rows in parallel with OpenMP over the host cores
    like the reference's thread pool, reconstruction single-threaded like the
    reference's numpy loop) on a bounded sample of the workload: the slab of
    frames that can reach `plane` is reconstructed into the full
    grid (timed: recon Mpix/s), then the full plane is resliced once untimed
    (warm-up) and `reps` times timed (reslices/s).  Bit-exact parity of the
    oracle pixels with the GPU's is reported."""
    slab = OracleSlab(wl, sweep)
    t0 = time.perf_counter()
    vol, nf = slab.volume_for(plane, cfg.interp_radius)
    t_rec = time.perf_counter() - t0
    p = slab.o.plane_params(plane)
    c = slab.o.cfg_array(cfg)
    slab.o.reslice(vol, p, c, plane.width, plane.height, cfg.unassigned_value)  # warm-up
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        px, cov = slab.o.reslice(vol, p, c, plane.width, plane.height, cfg.unassigned_value)
        times.append(time.perf_counter() - t0)
    hc = host_cores()
    parity = None if gpu_px is None else bool(np.array_equal(px, gpu_px) and np.array_equal(cov, gpu_cov))
    ms = 1000.0 * statistics.median(times)
    reslice = {"value": 1000.0 / ms, "unit": "reslices/s", "cores": hc["affinity"], "kind": "port",
               "cpu": hc["model"], "ms_per_reslice": ms,
               "sample": f"{reps} timed full {plane.width}x{plane.height} reslices (median; 1 untimed warm-up) on a "
                         f"slab-oracle volume ({nf} frames that reach the plane, full grid); C + OpenMP over "
                         f"{hc['affinity']} host threads",
               "parity_with_gpu": parity}
    npx = nf * wl.size * wl.size
    recon = {"value": npx / 1e6 / t_rec, "unit": "Mpix/s", "cores": 1, "kind": "port", "cpu": hc["model"],
             "sample": f"oracle reconstruct of {nf} frames ({npx} pixels) into the full grid (frame_cells + "
                       f"stable seal, single-threaded C), {t_rec:.2f} s"}
    return reslice, recon


def _best_ms(fn, reps=3):
    best, out = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ms = (time.perf_counter() - t0) * 1000.0
        best = ms if best is None else min(best, ms)
    return best, out


def scalar_arm_bench(db, wl, dev_sweep, frames_d, planes, peak, torch):
    """Config 5 (direction-blind comparison arm) on the same sweep: compound of
    the full sweep, fill_holes + trilinear on a sparse variant (every 8th frame,
    SURVEY §8d) so that gap filling does real work.  Per call: the wall time of
    the public function (frames in HBM) and its device span (CUDA events on the
    library stream, dare_last_device_ms); best of 4 after a warm-up call (the
    first call of a size also grows the device pool).  Algorithmic bytes per
    SURVEY §8d."""
    from types import SimpleNamespace

    def timed(fn, reps=4):
        out = fn()  # warm-up
        walls, devs = [], []
        for _ in range(reps):
            del out
            t0 = time.perf_counter()
            out = fn()
            walls.append((time.perf_counter() - t0) * 1000.0)
            devs.append(last_device_ms())
        return min(walls), min(devs), out

    n_in = wl.n_frames * wl.size * wl.size
    ms_c, dev_c, sv = timed(lambda: db.compound(dev_sweep, voxel_size=wl.voxel, margin=0.0))
    ncells = int(np.prod(sv.dims))
    sparse = SimpleNamespace(images=frames_d[::8].contiguous(), image_timestamps=dev_sweep.image_timestamps[::8],
                             pose_timestamps=dev_sweep.pose_timestamps[::8], poses=dev_sweep.poses[::8],
                             pixel_pitch=dev_sweep.pixel_pitch, calibration=dev_sweep.calibration, mask=None)
    sv_sparse = db.compound(sparse, voxel_size=wl.voxel, margin=0.0)
    ms_f, dev_f, filled = timed(lambda: db.fill_holes(sv_sparse, 3))
    passes = filled.passes_run
    nc_sparse = int(np.prod(sv_sparse.dims))
    db.reslice_trilinear_batch(filled, planes)
    walls = []
    for _ in range(4):
        t0 = time.perf_counter()
        db.reslice_trilinear_batch(filled, planes)
        walls.append((time.perf_counter() - t0) * 1000.0)
    ms_t = min(walls)
    hw = planes[0].width * planes[0].height
    comp_bytes = n_in + ncells * 5
    fill_bytes = passes * nc_sparse * 10
    gbs = lambda b, ms: b / (ms / 1000.0) / 1e9  # noqa: E731
    return {
        "compound": {"ms": ms_c, "device_ms": dev_c, "input_Mpix_per_s": n_in / 1e6 / (ms_c / 1000.0),
                     "device_input_Mpix_per_s": n_in / 1e6 / (dev_c / 1000.0),
                     "algorithmic_GBps": gbs(comp_bytes, dev_c), "frac": gbs(comp_bytes, dev_c) / peak,
                     "note": "ms = wall time of compound() (host plan + C-ABI call); device_ms = its device span "
                             "(zeroing + compound_tab_k + finalize); frac uses device_ms"},
        "fill_holes": {"ms": ms_f, "device_ms": dev_f, "passes_run": passes, "cells": nc_sparse,
                       "algorithmic_GBps": gbs(fill_bytes, dev_f) if passes else None,
                       "sweep": f"every 8th frame ({len(sparse.poses)} frames)"},
        "trilinear": {"ms_per_batch": ms_t, "poses": len(planes), "reslices_per_s": len(planes) / (ms_t / 1000.0),
                      "note": "host-buffer C-ABI call incl. pose upload and image download"},
        "timing": "best of 4 calls after a warm-up call (each synchronises)",
    }, filled


def evaluation_bench(db, vol, filled, planes, cfg, torch):
    """The reference CLI benchmark's evaluation loop (cli.py:253-287, SURVEY
    8f row 4) on this step's planes: directional reslices and trilinear
    baseline reslices compared with the noise-free phantom rendered at each
    plane (phantom.ground_truth_reslice), the 2P (NCC, SSIM) metrics in one
    dare_similarity launch on device tensors; medians and paired Wilcoxon p
    from run_comparison.  CPU: the oracle's numpy restatement per pair."""
    from paper_2605_26325_b200 import evaluation as ev
    from paper_2605_26325_b200.reslice import ResliceImage

    from oracle import oracle

    W, H = planes[0].width, planes[0].height
    truth = bench_data.render_phantom([p.pose for p in planes], W, H, planes[0].pixel_pitch, None, noise=False)
    dp, dc, _ = db.reslice_batch(vol, planes, cfg)
    bp, bc, _ = db.reslice_trilinear_batch(filled, planes)
    a = torch.from_numpy(np.concatenate([dp, bp])).cuda()
    am = torch.from_numpy(np.concatenate([dc, bc])).cuda()
    t2 = torch.cat([truth, truth])
    ev.similarity_batch(a, t2, am, None)  # warm-up
    best_dev = best_wall = None
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        r = ev.similarity_batch(a, t2, am, None)  # returns after the results' D2H
        e1.record()
        e1.synchronize()
        wall = (time.perf_counter() - t0) * 1000.0
        dev = e0.elapsed_time(e1)
        best_dev = dev if best_dev is None else min(best_dev, dev)
        best_wall = wall if best_wall is None else min(best_wall, wall)
    th = truth.cpu().numpy()
    ones = np.ones((H, W), bool)
    T = [ResliceImage(pixels=th[k], coverage=ones, timing_ms=0.0) for k in range(len(planes))]
    A = [ResliceImage(pixels=dp[k], coverage=dc[k], timing_ms=0.0) for k in range(len(planes))]
    B = [ResliceImage(pixels=bp[k], coverage=bc[k], timing_ms=0.0) for k in range(len(planes))]
    rep = ev.run_comparison(A, B, T)
    t0 = time.perf_counter()
    ncpu = 2
    for k in range(ncpu):
        o = oracle.similarity(dp[k], th[k], dc[k], None)
    cpu_ms = (time.perf_counter() - t0) * 1000.0 / ncpu
    parity = bool(o[0] == r.ncc[ncpu - 1] and o[1] == r.ssim[ncpu - 1])
    n = 2 * len(planes)
    s = rep.summary
    return {"pairs": n, "raster": f"{W}x{H}", "device_ms": best_dev, "wall_ms": best_wall,
            "pairs_per_s": n / (best_dev / 1000.0),
            "cpu_baseline": {"ms_per_pair": cpu_ms, "kind": "port", "cores": 1,
                             "sample": f"{ncpu} pairs through oracle.similarity (numpy)",
                             "parity_with_gpu": parity},
            "median": {m: {k: s[m][k]["median"] for k in ("dare", "baseline")} for m in ("ncc", "ssim")},
            "wilcoxon_p": {m: s[m]["wilcoxon_p"] for m in ("ncc", "ssim")},
            "excluded_pairs": len(s["excluded_pairs"]),
            "note": "truth = noise-free phantom at each plane (bench_data.render_phantom, noise=False); "
                    "device_ms = CUDA events around similarity_batch on device tensors (best of 4)"}


def service_bench(vol, planes, cfg, clients: int = 8):
    """Requests (pose7, raster, raw8) from `clients` threads through
    service.ResliceBatcher: wire-ready responses (pixels + device-packed
    coverage), coalesced across clients into batched launches."""
    import threading

    from paper_2605_26325_b200 import service as svc

    reqs = []
    for i, p in enumerate(planes):
        r = p.pose.rotation
        reqs.append(svc.ResliceRequest(i, (*(float(c) for c in p.pose.translation), r.w, r.x, r.y, r.z),
                                       p.width, p.height, tuple(p.pixel_pitch)))
    with svc.ResliceBatcher(vol, cfg, max_batch=64) as b:
        for f in [b.submit(r) for r in reqs[:16]]:
            f.result()  # warm-up
        b.launches = b.requests = 0
        lat = []

        def client(chunk):
            for r in chunk:  # each client waits for its answer before the next request
                lat.append(b.submit(r).result().latency_ms)

        threads = [threading.Thread(target=client, args=(reqs[j::clients],)) for j in range(clients)]
        t0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        wall = time.perf_counter() - t0
        return {"requests_per_s": len(reqs) / wall, "clients": clients, "requests": len(reqs),
                "launches": b.launches, "p50_latency_ms": float(np.percentile(lat, 50)),
                "note": "service.ResliceBatcher: validation, batched dare_reslice_packed, raw8 payload + "
                        "packed coverage per response; each client sends its next request after the answer"}


def host_sweep(wl, frames_np):
    from types import SimpleNamespace

    from paper_2605_26325_b200.geometry import Pose

    poses, ts = bench_data.sweep_poses(wl)
    return SimpleNamespace(images=frames_np, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                           pixel_pitch=(wl.pitch, wl.pitch), calibration=Pose.identity(), mask=None)


def bench_frames(wl):
    """The workload's frames (the reference's benchmark phantom, bench_data):
    rendered on the GPU when one is visible (setup only), else on the CPU."""
    import torch

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    return bench_data.render_frames_torch(wl, device=dev).cpu().numpy()


def run_reference(args):
    """Reference arm: the reference's CPU algorithm (the oracle port, C + OpenMP;
    the reference itself is pure Python/numba and is not on the GPU box) on this
    box's host cores, same config, frames and planes as the B200 arm.  Single-
    sweep configs: the full volume is reconstructed once (timed: recon Mpix/s,
    single-threaded like the reference's numpy loop), then every step reslices
    one full plane (rows in parallel over all host threads, like the reference's
    pool).  Multi-sweep configs (cfg3/cfg4 need ~300 GB on the host): slab
    volumes of 64x64 centre patches, time scaled by pixel count."""
    ws, rank, _ = make_rank_info()
    if rank != 0:
        return
    from oracle import oracle

    from paper_2605_26325_b200.reslice import ResliceConfig

    wl = bench_data.workload(args.config)
    sweep = host_sweep(wl, bench_frames(wl))
    cfg = ResliceConfig(interp_radius=wl.voxel)
    planes = bench_data.reslice_planes(wl, args.warmup + args.steps)
    cfga = oracle.cfg_array(cfg)
    hc = host_cores()
    recon = None
    if wl.sweeps == 1:
        t0 = time.perf_counter()
        vol = oracle.reconstruct(sweep, wl.voxel, 0.0)
        t_rec = time.perf_counter() - t0
        npx = wl.n_frames * wl.size * wl.size
        recon = {"value": npx / 1e6 / t_rec, "unit": "Mpix/s", "ms": 1000.0 * t_rec, "cores": 1,
                 "sample": f"full reconstruct_volume of the workload ({npx} pixels -> dims {tuple(vol.dims)})"}
        jobs = [(p, vol, 1.0) for p in planes]
        what = (f"full {wl.plane}x{wl.plane} planes on the full {tuple(vol.dims)} oracle volume (built once, "
                f"timed separately as recon)")
    else:
        patch = 64
        slab = OracleSlab(wl, sweep)
        distinct = [patch_plane(p, patch) for p in planes[args.warmup: args.warmup + 2]]
        vols = [slab.volume_for(p, cfg.interp_radius)[0] for p in distinct]
        scale = (wl.plane * wl.plane) / (patch * patch)
        jobs = [(distinct[i % 2], vols[i % 2], scale) for i in range(args.warmup + args.steps)]
        what = (f"{patch}x{patch} centre patches of {wl.plane}x{wl.plane} planes (cycling over 2 poses, time "
                f"scaled by pixel count) on slab-oracle volumes (frames that reach the patch, full grid)")
    for i in range(args.warmup):
        p, v, _ = jobs[i]
        oracle.reslice(v, oracle.plane_params(p), cfga, p.width, p.height, cfg.unassigned_value)
    times = []
    for i in range(args.warmup, args.warmup + args.steps):
        p, v, sc = jobs[i]
        pp = oracle.plane_params(p)
        t0 = time.perf_counter()
        oracle.reslice(v, pp, cfga, p.width, p.height, cfg.unassigned_value)
        times.append((time.perf_counter() - t0) * 1000.0 * sc)
    ms = statistics.mean(times)
    value = 1000.0 / ms
    out = {
        "impl": "reference", "metric": "reslices/sec", "value": value, "unit": "reslices/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference's benchmark phantom at the workload's sweep poses, as the B200 arm)",
        "p50_reslice_ms": statistics.median(times),
        "config": {"workload": f"{args.config}: {wl.n_frames} frames {wl.size}x{wl.size} -> "
                               f"{wl.voxel} mm grid, 1 pose/step at {wl.plane}x{wl.plane}",
                   "parallelism": f"host threads (OpenMP, {hc['affinity']})"},
        "cpu_baseline": {"value": value, "unit": "reslices/s", "cores": hc["affinity"], "kind": "port",
                         "cpu": hc["model"], "sample": f"{args.steps} reslices: {what}; C + OpenMP"},
        "recon": recon,
        "e2e": {"value": value, "unit": "reslices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ----------------------------------------------------------------------------- B200 arm

def run_b200(args):
    import torch

    import paper_2605_26325_b200 as db
    from paper_2605_26325_b200 import _lib
    from paper_2605_26325_b200.reslice import ResliceConfig, kernel_cfg, plane_params

    ws, rank, local = make_rank_info()
    if torch.cuda.device_count() <= local:
        sys.stderr.write(f"bench.py: rank {rank} needs CUDA device {local} but only "
                         f"{torch.cuda.device_count()} are visible; refusing to run\n")
        sys.exit(2)
    torch.cuda.set_device(local)
    _lib.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        import datetime

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        # failure detection: the NCCL watchdog aborts a collective stuck for 10 min
        # (a dead or hung rank) instead of hanging the job
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "3")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(minutes=10))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    wl = bench_data.workload(args.config)
    B = args.batch or wl.batch
    cfg = ResliceConfig(interp_radius=wl.voxel)

    # ---- reconstruction (every rank builds its replica) ----
    frames_d = bench_data.render_frames_torch(wl)
    torch.cuda.synchronize()
    poses, ts = bench_data.sweep_poses(wl)
    from types import SimpleNamespace

    from paper_2605_26325_b200.geometry import Pose

    dev_sweep = SimpleNamespace(images=frames_d, image_timestamps=ts, pose_timestamps=ts.copy(), poses=poses,
                                pixel_pitch=(wl.pitch, wl.pitch), calibration=Pose.identity(), mask=None)
    npix = wl.n_frames * wl.size * wl.size
    db.reconstruct_volume(dev_sweep, voxel_size=wl.voxel, margin=0.0)  # warm-up (allocator pools, modules)
    recon_ms, recon_span = [], []
    vol = None
    for _ in range(3):
        del vol
        barrier()
        t0 = time.perf_counter()
        vol = db.reconstruct_volume(dev_sweep, voxel_size=wl.voxel, margin=0.0)
        recon_ms.append((time.perf_counter() - t0) * 1000.0)
        recon_span.append(last_device_ms())
    best = int(np.argmin(recon_ms))
    recon_dev_ms = max_over_ranks(recon_ms[best])
    recon_span_ms = max_over_ranks(recon_span[best])
    frames_pinned = frames_d.cpu().pin_memory()
    frames_np = frames_pinned.numpy()
    host_sw = host_sweep(wl, frames_np)
    e2e_ms = []
    for _ in range(2):  # the first call also grows the device pool for a 2nd live volume
        barrier()
        t0 = time.perf_counter()
        vol_e2e = db.reconstruct_volume(host_sw, voxel_size=wl.voxel, margin=0.0)
        e2e_ms.append((time.perf_counter() - t0) * 1000.0)
        del vol_e2e
    recon_e2e_ms = max_over_ranks(min(e2e_ms))
    sharded_ms = sharded_err = None
    if ws > 1:  # frame-sharded build: all-gather of partial CSRs + merge on every rank
        from paper_2605_26325_b200 import parallel

        try:  # a secondary leg: its failure is reported, not allowed to void the reslice line
            for it in range(2):
                barrier()
                t0 = time.perf_counter()
                rep = parallel.reconstruct_volume_sharded(dev_sweep, voxel_size=wl.voxel, margin=0.0)
                torch.cuda.synchronize()
                sharded_ms = max_over_ranks((time.perf_counter() - t0) * 1000.0)
                del rep
        except Exception as e:  # noqa: BLE001
            sharded_ms, sharded_err = None, f"{type(e).__name__}: {e}"[:300]
    info = vol.device_info()

    # ---- reslice poses ----
    planes = bench_data.reslice_planes(wl, (args.warmup + args.steps) * B, seed=rank)
    params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
    params_d = torch.from_numpy(params).cuda()
    H = W = wl.plane
    out_d = torch.empty((2, B, H, W), dtype=torch.uint8, device="cuda")
    # schedule for the device-pointer path: pose-major when the batch is a
    # coherent trajectory (what dare_reslice decides by itself on host params)
    p0 = params[args.warmup * B:(args.warmup + 1) * B]
    coherent = _lib.load().dare_poses_coherent(p0.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), B, W, H,
                                               float(wl.voxel))
    schedule = args.schedule or (2 if coherent and args.exact else 1)  # same rule as dare_reslice's auto
    kc = kernel_cfg(cfg, schedule, exact=args.exact)
    # a real (non-default) stream: the kernels and the timing events share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    handle = vol.device_handle().raw

    def launch(step):
        pp = params_d[step * B:(step + 1) * B]
        _lib.call("dare_reslice_device", handle, B, ctypes.c_void_p(pp.data_ptr()), W, H, ctypes.byref(kc),
                  ctypes.c_void_p(out_d[0].data_ptr()), ctypes.c_void_p(out_d[1].data_ptr()), sptr)

    for s in range(args.warmup):
        launch(s)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in range(args.steps):
        launch(args.warmup + s)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    dev_ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_per_step = dev_ms / args.steps
    value = ws * B * args.steps / (dev_ms / 1000.0)

    # ---- e2e through the C ABI with host buffers ----
    params_pin = torch.from_numpy(params).pin_memory().numpy()
    px_pin = torch.empty((B, H, W), dtype=torch.uint8).pin_memory().numpy()
    cov_pin = torch.empty((B, H, W), dtype=torch.uint8).pin_memory().numpy()

    def host_call(step):
        pp = params_pin[step * B:(step + 1) * B]
        _lib.call("dare_reslice", handle, B, pp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), W, H,
                  ctypes.byref(kc), px_pin.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                  cov_pin.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))

    for s in range(min(args.warmup, 3)):
        host_call(s)
    barrier()
    t0 = time.perf_counter()
    for s in range(args.steps):
        host_call(args.warmup + s)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = ws * B * args.steps / e2e_s
    # the same calls from two host threads (the API is re-entrant, one CUDA stream per
    # thread): one call's copies overlap the other's kernels -- reported beside `e2e`
    import threading

    bufs = [(torch.empty((B, H, W), dtype=torch.uint8).pin_memory().numpy(),
             torch.empty((B, H, W), dtype=torch.uint8).pin_memory().numpy()) for _ in range(2)]

    def worker(tid, steps):
        px_t, cov_t = bufs[tid]
        for s in steps:
            pp = params_pin[s * B:(s + 1) * B]
            _lib.call("dare_reslice", handle, B, pp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), W, H,
                      ctypes.byref(kc), px_t.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                      cov_t.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))

    for tid in range(2):  # warm the second thread's stream, arena and staging
        worker(tid, [tid])
    barrier()
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(tid, range(args.warmup + tid, args.warmup + args.steps, 2)))
           for tid in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    e2e2_value = ws * B * args.steps / max_over_ranks(time.perf_counter() - t0)
    fb = ctypes.c_int64()
    _lib.call("dare_reslice_last_fallback", ctypes.byref(fb))
    certified = {"path": "exact" if args.exact else "certified f32 + exact fallback",
                 "fallback_pixels_last_step": int(fb.value), "fallback_fraction": fb.value / (B * H * W)}

    # ---- p50 single-pose latency through the public API ----
    lat = []
    for p in planes[:10]:
        db.reslice(vol, p, cfg)
    for p in planes[: max(100, args.steps)]:
        lat.append(db.reslice(vol, p, cfg).timing_ms)
    p50, p95 = float(np.percentile(lat, 50)), float(np.percentile(lat, 95))

    # ---- service request path: concurrent clients through ResliceBatcher ----
    service = None
    if rank == 0:
        service = service_bench(vol, planes[: 8 * 32], cfg)

    # ---- roofline of reslice_k ----
    offsets = torch.as_tensor(DevArray(info.d_cell_offsets, (int(np.prod(info.dims)) + 1,), "<i4"), device="cuda")
    counts = (offsets[1:].long() - offsets[:-1].long())
    dims = tuple(int(d) for d in info.dims)
    origin = tuple(float(o) for o in info.origin)
    ref_bytes = own_bytes = 0.0
    visits = 0
    step0 = args.warmup
    for k in range(B):
        p14 = params[step0 * B + k]
        cells = cells_visited(torch, dims, origin, float(info.voxel_size), p14, W, H, cfg.interp_radius)
        c = counts[cells]
        ref_bytes += 12 * len(cells) + 29 * float(c.sum().item()) + H * W * (1 + 1 / 8)
        own_bytes += 4 * len(cells) + 16 * float(c.sum().item()) + H * W * 2
    peak, peak_kind = hbm_peak()
    if args.exact:
        main_kernel = f"reslice_k<{1 if (cfg.k_dist != 0 and _pow2(cfg.interp_radius)) else (2 if cfg.k_dist == 0 else 0)}>"
    else:
        n_or = int(info.n_orientations)
        split = 2 <= n_or <= 1024 and schedule == 1 and os.environ.get("DARE_ORIENT_SPLIT") != "0"
        # register / direction-cluster index (split.cu) / smem / global gate
        gmode = 2 if n_or == 1 else (3 if split else (1 if schedule == 1 and n_or <= 1024 else 0))
        main_kernel = f"reslice_fast_k<{2 if cfg.k_dist == 0 else 0}, {gmode}, 1>"  # 1 part per pixel
    traffic, traffic_src = ncu_traffic(main_kernel, B, args.config)
    # launches per step: prep_k (gate table + launch order; gate_k alone when not sorted), main
    # kernel, [fallback kernel on the certified path]
    launches_per_step = (1 if (schedule == 1 and B >= 4) or int(info.n_orientations) > 0 else 0) + 1 + \
        (0 if args.exact else 1)
    achieved = ref_bytes / (ms_per_step / 1000.0) / 1e9

    # ---- direction-blind arm (config 5): compound -> fill_holes -> trilinear ----
    scalar_arm = evaluation = None
    if rank == 0 and not args.no_scalar:
        step_planes = planes[step0 * B:(step0 + 1) * B]
        scalar_arm, filled = scalar_arm_bench(db, wl, dev_sweep, frames_d, step_planes, peak, torch)
        evaluation = evaluation_bench(db, vol, filled, step_planes, cfg, torch)
        del filled

    # ---- CPU baseline (rank 0, bounded sample) ----
    cpu = recon_cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        plane0 = full0 = planes[step0 * B]
        if wl.sweeps > 1:
            # cfg3/cfg4: every cross sweep's frame reaches a full 512^2 plane (host RAM), so the
            # oracle times the 64x64 centre patch and the rate is scaled by pixel count
            plane0 = patch_plane(full0, 64)
        gp, gc, _ = db.reslice_batch(vol, [plane0], cfg)
        cpu, recon_cpu = oracle_baseline(wl, host_sw, plane0, cfg, gp[0], gc[0])
        if plane0 is not full0:
            scale = plane0.width * plane0.height / (full0.width * full0.height)
            cpu.update(value=cpu["value"] * scale, ms_per_reslice=cpu["ms_per_reslice"] / scale,
                       sample=cpu["sample"] + f"; EXTRAPOLATED to a full {full0.width}x{full0.height} plane by "
                                              f"pixel count (x{scale:.5f}); parity is on the patch")
    ncells_total = int(np.prod(dims))
    recon_alg = npix * 1 + 29 * int(info.n_samples) + 12 * ncells_total
    r_traffic, r_traffic_src = recon_traffic(args.config)
    recon_roof = {
        "bound": "hbm", "algorithmic_bytes": recon_alg,
        "formula": "N_in*1 + N_samples*29 + ncells*12 (SURVEY 8d, reference layout)",
        "achieved_device": recon_alg / (recon_span_ms / 1000.0) / 1e9,
        "frac_device": recon_alg / (recon_span_ms / 1000.0) / 1e9 / peak,
        "achieved_wall": recon_alg / (recon_dev_ms / 1000.0) / 1e9,
        "frac_wall": recon_alg / (recon_dev_ms / 1000.0) / 1e9 / peak,
        "peak": peak, "unit": "GB/s", "traffic": r_traffic, "traffic_source": r_traffic_src,
        "note": "device = CUDA-event span of the dare_reconstruct call on its stream (first kernel to seal); "
                "wall = the Python reconstruct_volume call incl. host pose pipeline and syncs"}

    if rank == 0:
        out = {
            "metric": "reslices/sec", "value": value, "unit": "reslices/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if args.exact else "f32 weights + f64 sums (certified, exact u8 output)",
            "data": "synthetic (the reference's benchmark phantom rendered at the workload's sweep poses)",
            "config": {"workload": f"{args.config}: {wl.n_frames} frames {wl.size}x{wl.size} -> dims {dims} "
                                   f"({info.n_samples} samples), {B} poses/step at {W}x{H}, r={cfg.interp_radius}",
                       "poses_per_step": B, "parallelism": f"pose-sharded x{ws} (replicated volume)",
                       "schedule": "pose-major" if schedule == 2 else "pixel-major",
                       "l2": "inputs larger than L2 (volume records "
                             f"{info.n_samples * 16 / 1e9:.1f} GB; each step's poses touch "
                             f"{own_bytes / 1e9:.2f} GB)"},
            "p50_reslice_ms": p50, "p95_reslice_ms": p95,
            "recon": {"metric": "recon input Mpix/s", "value": ws * npix / 1e6 / (recon_dev_ms / 1000.0),
                      "ms": recon_dev_ms, "device_ms": recon_span_ms,
                      "device_value": ws * npix / 1e6 / (recon_span_ms / 1000.0),
                      "e2e_value": ws * npix / 1e6 / (recon_e2e_ms / 1000.0),
                      "e2e_ms": recon_e2e_ms, "input_pixels": npix, "samples": int(info.n_samples),
                      "frame_sharded_ms": sharded_ms, "frame_sharded_error": sharded_err,
                      "roofline": recon_roof, "cpu_baseline": recon_cpu,
                      "note": "value/ms = wall time of reconstruct_volume with frames in HBM (host pose pipeline + "
                              "C-ABI call incl. syncs); e2e = the same from pinned host frames (PCIe upload inside)"},
            "e2e_2threads": {"value": e2e2_value, "unit": "reslices/s",
                             "note": "the e2e calls issued from two host threads (re-entrant API)"},
            "e2e": {"value": e2e_value, "unit": "reslices/s", "h2d_bytes_per_step": B * 14 * 8,
                    "d2h_bytes_per_step": 2 * B * H * W},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": main_kernel,
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_step_ref_layout": ref_bytes,
                         "compulsory_bytes_per_step_own_layout": own_bytes},
            "gpu_launches": launches_per_step * args.steps,
            "certified": certified,
            "clocks": clk,
            "cpu_baseline": cpu,
            "scalar_arm": scalar_arm, "service": service, "evaluation": evaluation,
        }
        print(json.dumps(out))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse_args()
    ws_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        run_reference(args)
        return
    if ws_env is None:
        import torch

        n_dev = torch.cuda.device_count()
        if n_dev < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {n_dev} CUDA device(s) are visible; "
                             f"refusing to run {args.gpus} ranks on fewer GPUs\n")
            sys.exit(2)
        if args.gpus > 1:
            sys.exit(spawn_ranks(args))
    if ws_env is not None and int(ws_env) != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}\n")
        sys.exit(2)
    run_b200(args)


if __name__ == "__main__":
    main()
