"""Insertion-order records of sampled cells, read from a device volume
(offsets / storage-order records / perm / orientation table via torch) --
for the slab-oracle record comparisons."""
import numpy as np


def device_cell_records(vol, cells):
    import torch

    from paper_2605_26325_b200.parallel import _CudaArray

    info = vol.device_info()
    nc = int(np.prod(info.dims))
    n, no = int(info.n_samples), int(info.n_orientations)
    off = torch.as_tensor(_CudaArray(info.d_cell_offsets, (nc + 1,), "<i4"), device="cuda").long() & 0xFFFFFFFF
    rec = torch.as_tensor(_CudaArray(info.d_records, (n, 4), "<i4"), device="cuda")
    perm = torch.as_tensor(_CudaArray(info.d_perm, (n,), "|i1"), device="cuda").long()
    ori = torch.as_tensor(_CudaArray(info.d_orientations, (no, 4), "<f4"), device="cuda")
    c = torch.as_tensor(np.asarray(cells, dtype=np.int64), device="cuda")
    starts, cnt = off[c], off[c + 1] - off[c]
    total = int(cnt.sum())
    first = torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt)
    canon = torch.repeat_interleave(starts, cnt) + (torch.arange(total, device="cuda") - first)
    r = rec[canon + perm[canon]]  # insertion order through perm
    pos = r[:, :3].contiguous().view(torch.float32).cpu().numpy()
    word = r[:, 3].cpu().numpy().astype(np.uint32)
    quat = ori[torch.as_tensor((word >> 8).astype(np.int64), device="cuda")].cpu().numpy()
    inten = (word & 0xFF).astype(np.uint8)
    bounds = np.concatenate([[0], np.cumsum(cnt.cpu().numpy())])
    return {int(cc): (pos[bounds[i]:bounds[i + 1]], quat[bounds[i]:bounds[i + 1]], inten[bounds[i]:bounds[i + 1]])
            for i, cc in enumerate(np.asarray(cells))}


def assert_cells_equal(dev, ref):
    assert dev.keys() == ref.keys()
    n = 0
    for c in ref:
        for a, b, name in zip(dev[c], ref[c], ("positions", "orientations", "intensities")):
            assert a.shape == b.shape, (c, name, a.shape, b.shape)
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (c, name)
        n += len(ref[c][2])
    return n
