"""Multi-GPU paths: one process per GPU, torch.distributed for the plumbing.

SURVEY §8e:
  * frame-sharded reconstruction -- rank r builds the contiguous block r of
    synchronized frames into the FULL grid on its GPU (only the images that
    block references are uploaded); the partial CSRs (offsets, storage-order
    records, perm, orientation table) are exchanged unpadded (one broadcast
    per rank, NCCL over NVLink) and merged on every rank by dare_volume_merge,
    which reads records through perm and deduplicates orientation tables in
    rank order, into a replica bit-identical to a single-GPU build (integer
    counts, deterministic placement: rank order = frame order);
  * pose-sharded batched reslicing -- every rank reslices its contiguous block
    of poses on its replica, no collective on the data path (results are
    gathered only if the caller asks for them);
  * frame-sharded compounding -- per-rank u64 sums/counts, one all-reduce SUM
    (exact integers), then the normalise pass;
  * pose-sharded trilinear reslicing -- the scalar grid (f32 values + u8
    flags, 5 B/cell) is broadcast from one rank, then every rank reslices its
    pose block; no collective on the data path.

The collective logic is device-agnostic (it runs with NCCL on CUDA tensors
and with gloo on CPU tensors); the per-rank compute is delegated to an `ops`
object -- `CudaOps` here (libdare_b200), a CPU-oracle implementation in the
gloo tests -- so the sharding/merge logic is tested on CPU with world_size 2.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .reslice import ResliceConfig, kernel_cfg, plane_params
from .sweep import grid_for, plan_frames, validate_margin


def _dist():
    import torch.distributed as dist

    return dist


def world(group=None) -> tuple[int, int]:
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _device(group=None) -> str:
    return "cuda" if _dist().get_backend(group) == "nccl" else "cpu"


def blocks(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [start, end) blocks; block r precedes block r+1."""
    base, extra = divmod(n, parts)
    out, s = [], 0
    for r in range(parts):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


@dataclass
class Part:
    """One rank's partial volume as flat tensors (device or host)."""

    offsets: object  # (ncells+1,) int32 (u32 bit pattern)
    records: object  # (n, 4) int32 (16 B records), storage order
    orient: object   # (n_orient, 4) float32
    n_samples: int
    n_orient: int
    rejected: int
    perm: object = None  # (n,) int8: insertion -> storage offset (None: records in insertion order)


def _bcast(t, src, group):
    if t.numel():
        _dist().broadcast(t, src=src, group=group)
    return t


def all_gather_parts(local: Part, group=None) -> list[Part]:
    """Every rank's Part on every rank, without padding: sizes are exchanged
    first (one small all-gather), then each rank's arrays are broadcast from
    it into exactly-sized buffers (the local part is used in place)."""
    import torch

    dist = _dist()
    rank, size = world(group)
    if size == 1:
        return [local]
    dev = local.offsets.device
    has_perm = local.perm is not None
    meta = torch.tensor([local.n_samples, local.n_orient, local.rejected, int(has_perm)], dtype=torch.int64,
                        device=dev)
    metas = [torch.empty_like(meta) for _ in range(size)]
    dist.all_gather(metas, meta, group=group)
    metas = [m.cpu().tolist() for m in metas]
    nc1 = int(local.offsets.shape[0])
    parts = []
    for r in range(size):
        n, no, rej, hp = metas[r]
        if r == rank:
            p = local
        else:
            p = Part(torch.empty(nc1, dtype=torch.int32, device=dev),
                     torch.empty((n, 4), dtype=torch.int32, device=dev),
                     torch.empty((no, 4), dtype=torch.float32, device=dev), n, no, rej,
                     torch.empty(n, dtype=torch.int8, device=dev) if hp else None)
        _bcast(p.offsets, r, group)
        _bcast(p.records, r, group)
        if hp:
            _bcast(p.perm, r, group)
        _bcast(p.orient, r, group)
        parts.append(p)
    return parts


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


class CudaOps:
    """Per-rank compute through libdare_b200 (the product path)."""

    @staticmethod
    def reconstruct_subset(sweep, plan, start, end, origin, voxel, dims):
        from .reconstruct import reconstruct_subset

        return reconstruct_subset(sweep, plan, start, end, origin, voxel, dims)

    @staticmethod
    def part_of(volume) -> Part:
        """Zero-copy views of a device volume's arrays (storage order + perm)."""
        import torch

        info = volume.device_info()
        nc = int(np.prod(info.dims))
        n, no = int(info.n_samples), int(info.n_orientations)
        offs = torch.as_tensor(_CudaArray(info.d_cell_offsets, (nc + 1,), "<i4"), device="cuda")
        if n:
            recs = torch.as_tensor(_CudaArray(info.d_records, (n, 4), "<i4"), device="cuda")
            perm = torch.as_tensor(_CudaArray(info.d_perm, (n,), "|i1"), device="cuda")
        else:
            recs = torch.zeros((0, 4), dtype=torch.int32, device="cuda")
            perm = torch.zeros(0, dtype=torch.int8, device="cuda")
        oris = torch.as_tensor(_CudaArray(info.d_orientations, (no, 4), "<f4"), device="cuda") if no else \
            torch.zeros((0, 4), dtype=torch.float32, device="cuda")
        part = Part(offs, recs, oris, n, no, int(info.rejected_out_of_bounds), perm)
        part._owner = volume  # the views stay valid while the Part lives
        return part

    @staticmethod
    def merge(parts: list[Part], origin, voxel, dims):
        import torch

        from .volume import DirectionalVolume, _Handle

        # parts may come from NCCL on torch's stream; the merge runs on the
        # library's per-thread stream
        torch.cuda.current_stream().synchronize()
        k = len(parts)
        offs = (ctypes.c_void_p * k)(*[p.offsets.data_ptr() for p in parts])
        recs = (ctypes.c_void_p * k)(*[p.records.data_ptr() if p.n_samples else 0 for p in parts])
        perms = (ctypes.c_void_p * k)(*[p.perm.data_ptr() if (p.perm is not None and p.n_samples) else 0
                                        for p in parts])
        oris = (ctypes.c_void_p * k)(*[p.orient.data_ptr() if p.n_orient else 0 for p in parts])
        ns = np.array([p.n_samples for p in parts], dtype=np.int64)
        no = np.array([p.n_orient for p in parts], dtype=np.int64)
        rj = np.array([p.rejected for p in parts], dtype=np.int64)
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        raw = ctypes.c_void_p()
        _lib.call("dare_volume_merge", _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64), k,
                  offs, recs, perms, oris, _lib.ptr(ns, ctypes.c_int64), _lib.ptr(no, ctypes.c_int64),
                  _lib.ptr(rj, ctypes.c_int64), ctypes.byref(raw))
        return DirectionalVolume(origin, voxel, dims, _handle=_Handle(raw.value))

    @staticmethod
    def reslice_block(volume, planes, cfg):
        from .reslice import reslice_batch

        px, cov, _ = reslice_batch(volume, planes, cfg)
        return px, cov

    @staticmethod
    def trilinear_block(volume, planes):
        from .scalar import reslice_trilinear_batch

        px, cov, _ = reslice_trilinear_batch(volume, planes)
        return px, cov

    @staticmethod
    def scalar_tensors(volume):
        """(values f32, flags u8) device views of a scalar volume."""
        import torch

        from .scalar import as_device_scalar

        sv = as_device_scalar(volume)
        info = _lib.ScalarInfo()
        _lib.call("dare_scalar_get_info", sv.device_handle(), ctypes.byref(info))
        nc = int(np.prod(sv.dims))
        v = torch.as_tensor(_CudaArray(info.d_values, (nc,), "<f4"), device="cuda")
        f = torch.as_tensor(_CudaArray(info.d_flags, (nc,), "|u1"), device="cuda")
        return v, f

    @staticmethod
    def scalar_from_tensors(origin, voxel, dims, values, flags):
        import torch

        from .scalar import ScalarVolume

        torch.cuda.current_stream().synchronize()  # received on torch's stream
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        raw = ctypes.c_void_p()
        _lib.call("dare_scalar_upload", _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64),
                  ctypes.cast(values.data_ptr(), ctypes.POINTER(ctypes.c_float)),
                  ctypes.cast(flags.data_ptr(), ctypes.POINTER(ctypes.c_uint8)),
                  ctypes.cast(None, ctypes.POINTER(ctypes.c_int64)), ctypes.byref(raw))
        return ScalarVolume(origin, voxel, dims, _raw=raw.value)

    @staticmethod
    def compound_partial(sweep, plan, start, end, origin, voxel, dims, stream=0):
        """u64 sums/counts of frames [start, end) (torch (2, ncells) int64 on the
        current device).  With a non-zero `stream` (cudaStream_t as int, the torch
        current stream) nothing synchronises.  Only the images the block
        references are uploaded."""
        import torch

        from .reconstruct import frames_block

        nc = int(np.prod(dims))
        acc = torch.zeros((2, nc), dtype=torch.int64, device="cuda")
        if not stream:  # the library's own stream does not order after torch's zero fill
            torch.cuda.current_stream().synchronize()
        n_img, frames_ptr, on_device, idx, _keep = frames_block(sweep, plan, start, end)
        axes = np.ascontiguousarray(plan.axes()[start:end])
        mask = _mask_arg(sweep)
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        _lib.call("dare_compound_accumulate", frames_ptr, n_img, plan.height, plan.width, on_device,
                  _lib.ptr(idx, ctypes.c_int32), int(end - start), _lib.ptr(axes, ctypes.c_double),
                  plan.pixel_pitch[0], plan.pixel_pitch[1], _lib.ptr(mask, ctypes.c_uint8),
                  _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64),
                  ctypes.c_void_p(acc[0].data_ptr()), ctypes.c_void_p(acc[1].data_ptr()), ctypes.c_void_p(stream))
        return acc

    @staticmethod
    def scalar_from_sums(acc, origin, voxel, dims):
        import torch

        from .scalar import ScalarVolume

        torch.cuda.current_stream().synchronize()  # acc may come from an all-reduce on torch's stream

        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        raw = ctypes.c_void_p()
        _lib.call("dare_scalar_from_sums", _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64),
                  ctypes.c_void_p(acc[0].data_ptr()), ctypes.c_void_p(acc[1].data_ptr()), ctypes.byref(raw))
        return ScalarVolume(origin, voxel, dims, _raw=raw.value)


def _mask_arg(sweep):
    if sweep.mask is None:
        return None
    return np.ascontiguousarray(np.asarray(sweep.mask, dtype=bool).reshape(-1).astype(np.uint8))


def reconstruct_volume_sharded(sweep, voxel_size: float = 0.125, margin: float = 1.0, group=None, ops=CudaOps):
    """Frame-sharded reconstruct_volume: returns the full volume on every rank."""
    validate_margin(margin)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, voxel_size, margin)
    rank, size = world(group)
    start, end = blocks(plan.n_frames, size)[rank]
    local = ops.reconstruct_subset(sweep, plan, start, end, origin, voxel, dims)
    parts = all_gather_parts(ops.part_of(local), group)
    merged = ops.merge(parts, origin, voxel, dims)
    merged.rejected_out_of_bounds = sum(p.rejected for p in parts)
    return merged


def _gather_images(px, cov, n_planes, h, w, group):
    """All ranks' pose-block results, in pose order, on every rank."""
    import torch

    dist = _dist()
    rank, size = world(group)
    dev = _device(group)
    bl = blocks(n_planes, size)
    outs = []
    for r, (s, e) in enumerate(bl):
        buf = torch.empty((2, e - s, h, w), dtype=torch.uint8, device=dev)
        if r == rank:
            buf[0] = torch.from_numpy(np.ascontiguousarray(px)).to(dev)
            buf[1] = torch.from_numpy(np.ascontiguousarray(cov).view(np.uint8)).to(dev)
        if size > 1 and e > s:
            dist.broadcast(buf, src=r, group=group)
        outs.append(buf.cpu().numpy())
    return (np.concatenate([o[0] for o in outs]), np.concatenate([o[1] for o in outs]).view(bool))


def reslice_sharded(volume, planes, cfg: ResliceConfig | None = None, group=None, gather: bool = True,
                    ops=CudaOps):
    """Pose-sharded batched reslice.  Rank r reslices planes[block r] on its
    replica; with gather=True every rank returns all (P, H, W) results."""
    cfg = cfg or ResliceConfig()
    planes = list(planes)
    rank, size = world(group)
    start, end = blocks(len(planes), size)[rank]
    mine = planes[start:end]
    h, w = planes[0].height, planes[0].width
    if mine:
        px, cov = ops.reslice_block(volume, mine, cfg)
    else:
        px = np.zeros((0, h, w), np.uint8)
        cov = np.zeros((0, h, w), bool)
    if not gather or size == 1:
        return px, cov, (start, end)
    px, cov = _gather_images(px, cov, len(planes), h, w, group)
    return px, cov, (0, len(planes))


def broadcast_scalar(volume, src: int = 0, group=None, ops=CudaOps):
    """The scalar grid of rank `src` (f32 values + u8 flags: 5 B/cell) on every
    rank; `volume` is ignored on the other ranks."""
    import torch

    dist = _dist()
    rank, size = world(group)
    if size == 1:
        return volume
    dev = _device(group)
    if rank == src:
        meta = torch.tensor([*volume.origin, volume.voxel_size, *volume.dims], dtype=torch.float64, device=dev)
    else:
        meta = torch.empty(7, dtype=torch.float64, device=dev)
    dist.broadcast(meta, src=src, group=group)
    m = meta.cpu().numpy()
    origin, voxel, dims = tuple(float(x) for x in m[:3]), float(m[3]), tuple(int(x) for x in m[4:7])
    nc = int(np.prod(dims))
    if rank == src:
        values, flags = ops.scalar_tensors(volume)
    else:
        values = torch.empty(nc, dtype=torch.float32, device=dev)
        flags = torch.empty(nc, dtype=torch.uint8, device=dev)
    dist.broadcast(values, src=src, group=group)
    dist.broadcast(flags, src=src, group=group)
    if rank == src:
        return volume
    return ops.scalar_from_tensors(origin, voxel, dims, values, flags)


def reslice_trilinear_sharded(volume, planes, group=None, gather: bool = True, src: int = 0, ops=CudaOps):
    """Pose-sharded reslice_trilinear (baseline.py:130-155): the scalar grid of
    rank `src` is broadcast once (§8e), then rank r reslices planes[block r];
    with gather=True every rank returns all (P, H, W) results."""
    planes = list(planes)
    rank, size = world(group)
    grid = broadcast_scalar(volume, src, group, ops) if size > 1 else volume
    start, end = blocks(len(planes), size)[rank]
    mine = planes[start:end]
    h, w = planes[0].height, planes[0].width
    if mine:
        px, cov = ops.trilinear_block(grid, mine)
    else:
        px = np.zeros((0, h, w), np.uint8)
        cov = np.zeros((0, h, w), bool)
    if not gather or size == 1:
        return px, cov, (start, end)
    px, cov = _gather_images(px, cov, len(planes), h, w, group)
    return px, cov, (0, len(planes))


def compound_sharded(sweep, voxel_size: float = 0.125, margin: float = 1.0, group=None, ops=CudaOps):
    """Frame-sharded compound: per-rank integer sums/counts, all-reduce SUM."""
    validate_margin(margin)
    plan = plan_frames(sweep)
    origin, voxel, dims = grid_for(plan, voxel_size, margin)
    rank, size = world(group)
    start, end = blocks(plan.n_frames, size)[rank]
    acc = ops.compound_partial(sweep, plan, start, end, origin, voxel, dims)
    if size > 1:
        dist = _dist()
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return ops.scalar_from_sums(acc, origin, voxel, dims)


__all__ = ["blocks", "Part", "all_gather_parts", "CudaOps", "reconstruct_volume_sharded", "reslice_sharded",
           "broadcast_scalar", "reslice_trilinear_sharded", "compound_sharded", "world", "kernel_cfg",
           "plane_params"]
