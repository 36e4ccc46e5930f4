"""Freehand-sweep reconstruction on the device (drop-in for reconstruct.py:166-199).

Host: synchronize + calibration + bounds + grid sizing, vectorised over frames
(sweep.plan_frames / grid_for, bit-exact with the reference's scalar code).
Device (one C-ABI call, csrc/reconstruct.cu): pixel -> world -> cell for every
pixel of every frame, warp-aggregated histogram, scan, slot fill, per-cell
insertion-order sort and 16 B record materialisation -- the reference's
per-frame insert_batch loop plus seal().
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import InvalidArgumentError
from .sweep import FramePlan, SweepRecording, grid_for, plan_frames, validate_margin
from .volume import DirectionalVolume, _Handle


def frames_arg(sweep, frames_device_ptr: int | None = None):
    """(images, pointer, on_device) for the image stack: a CUDA tensor or an
    explicit device pointer is used in place, anything else is a host array."""
    images = sweep.images
    if frames_device_ptr is None and getattr(images, "is_cuda", False):
        if images.dtype.itemsize != 1 or not images.is_contiguous():
            raise InvalidArgumentError("device images must be a contiguous uint8 tensor")
        import torch

        # the library reads the frames on its own (non-blocking) stream: finish
        # whatever torch work produced them first
        torch.cuda.current_stream(images.device).synchronize()
        frames_device_ptr = images.data_ptr()
    if frames_device_ptr is not None:
        return images, ctypes.c_void_p(int(frames_device_ptr)), 1
    images = np.ascontiguousarray(np.asarray(images), dtype=np.uint8)
    return images, _lib.vptr(images), 0


def frames_block(sweep, plan: FramePlan, start: int, end: int, frames_device_ptr: int | None = None):
    """(n_images, pointer, on_device, frame_image, keepalive) for synchronized
    frames [start, end): only the contiguous image range the block references
    is passed (a frame-sharded rank uploads / reads its own images, not the
    whole stack), frame_image rebased to it.  `keepalive` owns the memory the
    pointer refers to (hold it until the call returns)."""
    images, base_ptr, on_device = frames_arg(sweep, frames_device_ptr)
    idx = np.ascontiguousarray(plan.image_index[start:end], dtype=np.int32)
    if len(idx) == 0:
        return 0, base_ptr, on_device, idx, images
    i0, i1 = int(idx.min()), int(idx.max()) + 1
    hw = int(plan.height) * int(plan.width)
    ptr = ctypes.c_void_p((base_ptr.value or 0) + i0 * hw)
    return i1 - i0, ptr, on_device, np.ascontiguousarray(idx - i0, dtype=np.int32), images


def _mask(sweep):
    if sweep.mask is None:
        return None
    return np.ascontiguousarray(np.asarray(sweep.mask, dtype=bool).reshape(-1).astype(np.uint8))


def reconstruct_subset(sweep, plan: FramePlan, start: int, end: int, origin, voxel: float, dims,
                       frames_device_ptr: int | None = None) -> DirectionalVolume:
    """Synchronized frames [start, end) into the given grid (the full grid for
    frame-sharded multi-GPU builds; start=0, end=n for a whole sweep)."""
    n_img, frames_ptr, on_device, idx, _keep = frames_block(sweep, plan, start, end, frames_device_ptr)
    axes = np.ascontiguousarray(plan.axes()[start:end])
    quats = np.ascontiguousarray(plan.canonical_quats_f32()[start:end])
    mask = _mask(sweep)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    raw = ctypes.c_void_p()
    rejected = ctypes.c_int64(0)
    _lib.call("dare_reconstruct", frames_ptr, n_img, int(plan.height), int(plan.width),
              on_device, _lib.ptr(idx, ctypes.c_int32), int(end - start),
              _lib.ptr(axes, ctypes.c_double), _lib.ptr(quats, ctypes.c_float),
              plan.pixel_pitch[0], plan.pixel_pitch[1], _lib.ptr(mask, ctypes.c_uint8),
              _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64), ctypes.byref(raw),
              ctypes.byref(rejected))
    vol = DirectionalVolume(origin, voxel, dims, _handle=_Handle(raw.value))
    vol.rejected_out_of_bounds = int(rejected.value)
    return vol


def reconstruct_volume(sweep: SweepRecording, voxel_size: float = 0.125, margin: float = 1.0,
                       *, frames_device_ptr: int | None = None) -> DirectionalVolume:
    """Scatter every unmasked pixel of every synchronized frame into its cell.

    frames_device_ptr: optional device pointer to the (n, H, W) u8 image
    stack already resident in HBM (skips the host->device copy).  A CUDA
    tensor passed as `sweep.images` is used in place the same way.
    """
    validate_margin(margin)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, voxel_size, margin)
    return reconstruct_subset(sweep, plan, 0, plan.n_frames, origin, voxel, dims, frames_device_ptr)
