"""Multi-process (world_size 2, gloo on CPU) tests of the sharded paths in
paper_2605_26325_b200.parallel.  The collective logic (frame blocks, size
exchange, unpadded per-rank broadcasts, rank-ordered merge through perm,
orientation-table dedup, integer all-reduce, scalar-grid broadcast and
pose-sharded trilinear) is the product code; only the per-rank compute is
replaced by the CPU oracle (OracleOps below), which mirrors the CUDA kernels.
The result must equal the single-process oracle bit-for-bit."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2605_26325_b200 import parallel
from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig
from paper_2605_26325_b200.sweep import SweepRecording


def _sweep(seed=3, n=13, h=11, w=12):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4)) * [8, 1, 1, 1]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    poses = [Pose(Quaternion(*qq), (0.05 * k, 0.02 * k, 0.15 * k)) for k, qq in enumerate(q)]
    ts = np.arange(n) * 0.04
    return SweepRecording(rng.integers(0, 256, (n, h, w), dtype=np.uint8), ts, ts, poses, (0.1, 0.1))


def _pack(vol):
    """Oracle volume -> parallel.Part on CPU (records as the device packs them)."""
    q = np.ascontiguousarray(vol.orientations)
    keys = q.view(np.dtype((np.void, 16))).reshape(-1)
    uniq, first, inverse = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first)  # ids in first-appearance order, like the device dedup
    rank_of = np.empty_like(order)
    rank_of[order] = np.arange(len(order))
    oid = rank_of[inverse.reshape(-1)].astype(np.uint32)
    table = q[first[order]] if len(q) else np.zeros((0, 4), np.float32)
    rec = np.zeros((len(vol.intensities), 4), np.uint32)
    rec[:, :3] = np.ascontiguousarray(vol.positions).view(np.uint32)
    rec[:, 3] = (oid << 8) | vol.intensities.astype(np.uint32)
    off = np.concatenate([vol.cell_starts, [vol.cell_starts[-1] + vol.cell_counts[-1]]]).astype(np.uint32)
    return parallel.Part(torch.from_numpy(off.view(np.int32).copy()), torch.from_numpy(rec.view(np.int32).copy()),
                         torch.from_numpy(np.ascontiguousarray(table, np.float32)), len(rec), len(table),
                         vol.rejected_out_of_bounds)


class OracleOps:
    @staticmethod
    def reconstruct_subset(sweep, plan, start, end, origin, voxel, dims):
        frames = oracle.frame_poses(sweep)[start:end]
        vol = oracle.reconstruct_subset(sweep, frames, origin, voxel, dims)
        # out-of-bounds count of the subset (reconstruct_subset drops them silently)
        rej = 0
        for f in frames:
            lin, _ = oracle.frame_cells(f, plan.width, plan.height, sweep.pixel_pitch, origin, voxel, dims)
            rej += int(np.count_nonzero(lin < 0))
        vol.rejected_out_of_bounds = rej
        return vol

    part_of = staticmethod(_pack)

    @staticmethod
    def merge(parts, origin, voxel, dims):
        """Rank-ordered run concatenation, records read through perm, orientation
        tables deduplicated in rank order (first occurrence) -- merge.cu's rules."""
        nc = int(np.prod(dims))
        offs = [p.offsets.numpy().view(np.uint32).astype(np.int64) for p in parts]
        recs = []
        for p in parts:
            rec = p.records.numpy().view(np.uint32)
            if p.perm is not None and len(rec):
                j = np.arange(len(rec))
                rec = rec[j + p.perm.numpy().astype(np.int64)]
            recs.append(rec)
        cat = np.concatenate([p.orient.numpy() for p in parts]) if sum(p.n_orient for p in parts) else \
            np.zeros((0, 4), np.float32)
        keys = [bytes(q.tobytes()) for q in cat]
        first, remap_all = {}, []
        for k in keys:
            remap_all.append(first.setdefault(k, len(first)))
        table = np.array([np.frombuffer(k, np.float32) for k in first]) if first else np.zeros((0, 4), np.float32)
        base = np.cumsum([0] + [p.n_orient for p in parts])
        counts = sum(o[1:] - o[:-1] for o in offs)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
        out = np.zeros((int(counts.sum()), 4), np.uint32)
        for c in range(nc):
            dst = starts[c]
            for r, (o, rec) in enumerate(zip(offs, recs)):
                run = rec[o[c]:o[c + 1]].copy()
                local = run[:, 3] >> 8
                run[:, 3] = (np.asarray(remap_all, np.uint32)[base[r] + local] << 8) | (run[:, 3] & 0xFF)
                out[dst:dst + len(run)] = run
                dst += len(run)
        vol = oracle.OracleVolume(np.asarray(origin, float), voxel, tuple(dims), starts, counts,
                                  out[:, :3].copy().view(np.float32), table[out[:, 3] >> 8],
                                  (out[:, 3] & 0xFF).astype(np.uint8))
        vol.n_orient = len(table)
        return vol

    @staticmethod
    def reslice_block(volume, planes, cfg):
        res = [oracle.reslice(volume, oracle.plane_params(p), oracle.cfg_array(cfg), p.width, p.height,
                              cfg.unassigned_value) for p in planes]
        return np.stack([r[0] for r in res]), np.stack([r[1] for r in res])

    @staticmethod
    def compound_partial(sweep, plan, start, end, origin, voxel, dims):
        lib = oracle.load()
        nc = int(np.prod(dims))
        sums, counts = np.zeros(nc, np.int64), np.zeros(nc, np.int64)
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int64)
        for f in oracle.frame_poses(sweep)[start:end]:
            r = oracle._rmat(f.quat)
            c0, c1 = np.ascontiguousarray(r[:, 0]), np.ascontiguousarray(r[:, 1])
            t = np.ascontiguousarray(f.trans, dtype=np.float64)
            px = np.ascontiguousarray(np.asarray(sweep.images)[f.image])
            lib.oracle_compound_frame(plan.height, plan.width, sweep.pixel_pitch[0], sweep.pixel_pitch[1],
                                      c0.ctypes.data, c1.ctypes.data, t.ctypes.data, o.ctypes.data, voxel,
                                      d.ctypes.data, px.ctypes.data, None, sums.ctypes.data, counts.ctypes.data)
        return torch.from_numpy(np.stack([sums, counts]))

    @staticmethod
    def scalar_from_sums(acc, origin, voxel, dims):
        sums, counts = acc[0].numpy(), acc[1].numpy()
        nc = len(sums)
        values, flags = np.empty(nc, np.float32), np.empty(nc, np.uint8)
        oracle.load().oracle_compound_finalize(nc, sums.ctypes.data, counts.ctypes.data, values.ctypes.data,
                                               flags.ctypes.data)
        return SimpleNamespace(origin=tuple(float(x) for x in origin), voxel_size=float(voxel), dims=tuple(dims),
                               values=values, flags=flags, counts=counts)

    @staticmethod
    def scalar_tensors(volume):
        return torch.from_numpy(np.ascontiguousarray(volume.values)), torch.from_numpy(
            np.ascontiguousarray(volume.flags))

    @staticmethod
    def scalar_from_tensors(origin, voxel, dims, values, flags):
        return SimpleNamespace(origin=origin, voxel_size=voxel, dims=dims, values=values.numpy(),
                               flags=flags.numpy(), counts=None)

    @staticmethod
    def trilinear_block(volume, planes):
        res = [oracle.trilinear(volume.origin, volume.voxel_size, volume.dims, volume.values, volume.flags,
                                oracle.plane_params(p), p.width, p.height) for p in planes]
        return np.stack([r[0] for r in res]), np.stack([r[1] for r in res])


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sweep = _sweep()
        full = oracle.reconstruct(sweep, 0.125, 0.0)
        vol = parallel.reconstruct_volume_sharded(sweep, 0.125, 0.0, ops=OracleOps)
        for name in ("cell_starts", "cell_counts", "positions", "orientations", "intensities"):
            np.testing.assert_array_equal(getattr(vol, name), getattr(full, name), err_msg=name)
        assert vol.rejected_out_of_bounds == full.rejected_out_of_bounds
        planes = [ReslicePlane(Pose(Quaternion.from_axis_angle((1, 0, 0), 0.1 * k), (0.2, 0.1, 0.3 + 0.2 * k)),
                               9, 7, (0.11, 0.11)) for k in range(5)]
        cfg = ResliceConfig(interp_radius=0.125, normal_threshold_deg=70, inplane_threshold_deg=70)
        px, cov, _ = parallel.reslice_sharded(full, planes, cfg, ops=OracleOps)
        for k, p in enumerate(planes):
            rp, rc = oracle.reslice(full, oracle.plane_params(p), oracle.cfg_array(cfg), p.width, p.height)
            np.testing.assert_array_equal(px[k], rp)
            np.testing.assert_array_equal(cov[k], rc)
        sv = parallel.compound_sharded(sweep, 0.125, 0.0, ops=OracleOps)
        o, vx, dims, rv, rf, rc = oracle.compound(sweep, 0.125, 0.0)
        np.testing.assert_array_equal(sv.values, rv)
        np.testing.assert_array_equal(sv.flags, rf)
        np.testing.assert_array_equal(sv.counts, rc)
        # pose-sharded trilinear: rank 0's filled grid is broadcast, each rank
        # reslices its pose block, results gathered in pose order
        fv, ff = oracle.fill_holes(rv, rf, dims, 3)
        grid = SimpleNamespace(origin=o, voxel_size=vx, dims=tuple(dims), values=fv, flags=ff) if rank == 0 \
            else None
        tpx, tcov, _ = parallel.reslice_trilinear_sharded(grid, planes, ops=OracleOps)
        for k, p in enumerate(planes):
            rp, rc2, _ = oracle.trilinear(o, vx, dims, fv, ff, oracle.plane_params(p), p.width, p.height)
            np.testing.assert_array_equal(tpx[k], rp)
            np.testing.assert_array_equal(tcov[k], rc2)
        assert tcov.any()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback

        q.put((rank, traceback.format_exc()))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_blocks_are_contiguous_and_balanced():
    for n in range(0, 40):
        for parts in range(1, 9):
            b = parallel.blocks(n, parts)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(parts - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
def test_sharded_paths_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    for r in range(2):
        assert results[r] == "ok", results[r]
