import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_26325_b200 as db
from paper_2605_26325_b200.parallel import _CudaArray
rng = np.random.default_rng(0)
# 40 cells along x (dims 40,1,1), cell c gets c+1 samples with z descending
pos, q, inten = [], [], []
for c in range(40):
    for j in range(c + 1):
        pos.append((c + 0.5, 0.5, 0.99 - j * 0.98 / (c + 1)))
        q.append((1, 0, 0, 0)); inten.append(j % 256)
b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (40, 1, 1)), 1.0)
pos = np.array(pos); b.insert_batch(pos, np.array(q, float), np.array(inten))
v = b.seal()
dl = np.asarray(v.positions)
print("dims", v.dims, "roundtrip", np.array_equal(dl, pos.astype(np.float32)))
info = v.device_info()
n = int(info.n_samples)
perm = torch.as_tensor(_CudaArray(info.d_perm, (n,), "|i1"), device="cuda").cpu().numpy()
bins = torch.as_tensor(_CudaArray(info.d_bins, (40,), "<u4"), device="cuda").cpu().numpy()
starts = np.asarray(v.cell_starts); counts = np.asarray(v.cell_counts)
bins = torch.as_tensor(_CudaArray(info.d_bins, (len(counts),), "<u4"), device="cuda").cpu().numpy()
store = torch.as_tensor(_CudaArray(info.d_records, (n, 4), "<i4"), device="cuda").cpu().numpy()
for c in np.nonzero(counts)[0]:
    s, k = starts[c], counts[c]
    ok = np.array_equal(dl[s:s+k], pos[s:s+k].astype(np.float32))
    if not ok or k in (1, 16, 17, 20):
        print(c, k, hex(bins[c]), "ok" if ok else "BAD", perm[s:s+k].tolist())
        if not ok:
            print("   stored z", store[s:s+k, 2].view(np.float32).round(3).tolist())
