"""Multi-GPU paths: one process per GPU, torch.distributed for the plumbing.

SURVEY §8e:
  * frame-sharded reconstruction -- rank r builds the contiguous block r of
    synchronized frames into the FULL grid on its GPU; the partial CSRs are
    all-gathered (NCCL over NVLink) and merged on every rank by
    dare_volume_merge into a replica bit-identical to a single-GPU build
    (integer counts, deterministic placement: rank order = frame order);
  * pose-sharded batched reslicing -- every rank reslices its contiguous block
    of poses on its replica, no collective on the data path (results are
    all-gathered only if the caller asks for them);
  * frame-sharded compounding -- per-rank u64 sums/counts, one all-reduce SUM
    (exact integers), then the normalise pass.

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
    records: object  # (n, 4) int32 (16 B records)
    orient: object   # (n_orient, 4) float32
    n_samples: int
    n_orient: int
    rejected: int


def all_gather_parts(local: Part, group=None) -> list[Part]:
    """All-gather every rank's Part (sizes first, then padded payloads)."""
    import torch

    dist = _dist()
    rank, size = world(group)
    if size == 1:
        return [local]
    dev = local.offsets.device
    meta = torch.tensor([local.n_samples, local.n_orient, local.rejected], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(size)]
    dist.all_gather(metas, meta, group=group)
    metas = [m.cpu().tolist() for m in metas]
    max_n = max(1, max(m[0] for m in metas))
    max_o = max(1, max(m[1] for m in metas))

    def gather_padded(t, rows):
        padded = torch.zeros((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        padded[: t.shape[0]] = t
        out = [torch.empty_like(padded) for _ in range(size)]
        dist.all_gather(out, padded.contiguous(), group=group)
        return out

    offs = [torch.empty_like(local.offsets) for _ in range(size)]
    dist.all_gather(offs, local.offsets.contiguous(), group=group)
    recs = gather_padded(local.records, max_n)
    oris = gather_padded(local.orient, max_o)
    return [Part(offs[r], recs[r][: metas[r][0]], oris[r][: metas[r][1]], metas[r][0], metas[r][1], metas[r][2])
            for r in range(size)]


class CudaOps:
    """Per-rank compute through libdare_b200 (the product path)."""

    @staticmethod
    def reconstruct_subset(sweep, plan, start, end, origin, voxel, dims):
        from .reconstruct import reconstruct_subset

        return reconstruct_subset(sweep, plan, start, end, origin, voxel, dims)

    @staticmethod
    def part_of(volume) -> Part:
        import torch

        info = volume.device_info()
        nc = int(np.prod(info.dims))
        n, no = int(info.n_samples), int(info.n_orientations)
        offs = torch.as_tensor(_CudaArray(info.d_cell_offsets, (nc + 1,), "<i4"), device="cuda")
        if n:  # records in insertion order: storage index = J + perm[J]
            store = torch.as_tensor(_CudaArray(info.d_records, (n, 4), "<i4"), device="cuda")
            perm = torch.as_tensor(_CudaArray(info.d_perm, (n,), "|i1"), device="cuda")
            recs = store[torch.arange(n, device="cuda") + perm.long()]
        else:
            recs = torch.zeros((0, 4), dtype=torch.int32, device="cuda")
        oris = torch.as_tensor(_CudaArray(info.d_orientations, (no, 4), "<f4"), device="cuda") if no else \
            torch.zeros((0, 4), dtype=torch.float32, device="cuda")
        torch.cuda.current_stream().synchronize()  # the library reads these on its own stream
        return Part(offs, recs, oris, n, no, int(info.rejected_out_of_bounds))

    @staticmethod
    def merge(parts: list[Part], origin, voxel, dims):
        import torch

        from .volume import DirectionalVolume, _Handle

        # parts may come from torch kernels / NCCL on torch's stream; the merge
        # runs on the library's per-thread stream
        torch.cuda.current_stream().synchronize()
        k = len(parts)
        offs = (ctypes.c_void_p * k)(*[p.offsets.data_ptr() for p in parts])
        recs = (ctypes.c_void_p * k)(*[p.records.data_ptr() if p.n_samples else 0 for p in parts])
        oris = (ctypes.c_void_p * k)(*[p.orient.data_ptr() if p.n_orient else 0 for p in parts])
        ns = np.array([p.n_samples for p in parts], dtype=np.int64)
        no = np.array([p.n_orient for p in parts], dtype=np.int64)
        rj = np.array([p.rejected for p in parts], dtype=np.int64)
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        raw = ctypes.c_void_p()
        _lib.call("dare_volume_merge", _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64), k,
                  offs, recs, oris, _lib.ptr(ns, ctypes.c_int64), _lib.ptr(no, ctypes.c_int64),
                  _lib.ptr(rj, ctypes.c_int64), ctypes.byref(raw))
        vol = DirectionalVolume(origin, voxel, dims, _handle=_Handle(raw.value))
        return vol

    @staticmethod
    def reslice_block(volume, planes, cfg):
        from .reslice import reslice_batch

        px, cov, _ = reslice_batch(volume, planes, cfg)
        return px, cov

    @staticmethod
    def compound_partial(sweep, plan, start, end, origin, voxel, dims, stream=0):
        """u64 sums/counts of frames [start, end) (torch (2, ncells) int64 on the
        current device).  With a non-zero `stream` (cudaStream_t as int, the torch
        current stream) nothing synchronises."""
        import torch

        from .reconstruct import frames_arg

        nc = int(np.prod(dims))
        acc = torch.zeros((2, nc), dtype=torch.int64, device="cuda")
        if not stream:  # the library's own stream does not order after torch's zero fill
            torch.cuda.current_stream().synchronize()
        images, frames_ptr, on_device = frames_arg(sweep)
        idx = np.ascontiguousarray(plan.image_index[start:end])
        axes = np.ascontiguousarray(plan.axes()[start:end])
        mask = _mask_arg(sweep)
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        _lib.call("dare_compound_accumulate", frames_ptr, int(images.shape[0]), plan.height, plan.width, on_device,
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


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


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


def reslice_sharded(volume, planes, cfg: ResliceConfig | None = None, group=None, gather: bool = True,
                    ops=CudaOps):
    """Pose-sharded batched reslice.  Rank r reslices planes[block r] on its
    replica; with gather=True every rank returns all (P, H, W) results."""
    import torch

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
    dist = _dist()
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    per = max(e - s for s, e in blocks(len(planes), size))
    buf = torch.zeros((2, per, h, w), dtype=torch.uint8, device=dev)
    buf[0, : len(mine)] = torch.from_numpy(np.ascontiguousarray(px)).to(dev)
    buf[1, : len(mine)] = torch.from_numpy(np.ascontiguousarray(cov).view(np.uint8)).to(dev)
    outs = [torch.empty_like(buf) for _ in range(size)]
    dist.all_gather(outs, buf, group=group)
    all_px, all_cov = [], []
    for r, (s, e) in enumerate(blocks(len(planes), size)):
        all_px.append(outs[r][0, : e - s].cpu().numpy())
        all_cov.append(outs[r][1, : e - s].cpu().numpy().view(bool))
    return np.concatenate(all_px), np.concatenate(all_cov), (0, len(planes))


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
           "compound_sharded", "world", "kernel_cfg", "plane_params"]
