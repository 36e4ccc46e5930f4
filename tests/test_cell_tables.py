"""CPU: the exact threshold tables behind the count / compound passes
(csrc/cells.cu, dare_cell_thresholds) reproduce the reference's per-axis cell
index floor((f64(f32(P)) - origin) / voxel) (volume.py:209, baseline.py:87)
and, on the fine z table, the z-quarter bin -- for P drawn densely around
every boundary (+-64 ulps) and uniformly, on power-of-two and general voxels."""
import ctypes

import numpy as np
import pytest

from paper_2605_26325_b200 import _lib


def tables(origin, voxel, dims, zfine):
    o = np.ascontiguousarray(origin, np.float64)
    d = np.ascontiguousarray(dims, np.int64)
    out = np.empty(int(d[0] + d[1] + 4 * d[2] + 3), np.float64)
    n = np.zeros(3, np.int64)
    _lib.call("dare_cell_thresholds", _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64),
              int(zfine), _lib.ptr(out, ctypes.c_double), _lib.ptr(n, ctypes.c_int64))
    assert (n >= 0).all()
    res, k = [], 0
    for a in range(3):
        res.append(out[k:k + n[a] + 1])
        k += n[a] + 1
    return res


def ref_index(P, o, voxel):
    d = P.astype(np.float32).astype(np.float64) - o
    m, _ = np.frexp(voxel)
    q = d * (1.0 / voxel) if m == 0.5 else d / voxel
    return np.floor(q)


def probes(T, rng):
    fin = T[np.isfinite(T)]
    pts = [rng.uniform(fin.min() - 1.0, fin.max() + 1.0, 20000)]
    for t in fin[:: max(1, len(fin) // 64)]:
        pts.append(t + np.arange(-64, 65) * np.spacing(t))  # +-64 ulps around the boundary
        pts.append(np.array([t, np.nextafter(t, -np.inf), np.nextafter(t, np.inf)]))
    return np.concatenate(pts)


@pytest.mark.parametrize("origin,voxel,dims", [
    ((0.0, 0.0, 0.0), 0.25, (128, 128, 128)),
    ((-3.141592653589793, 1.0000000000000002, 7.3), 0.125, (40, 33, 45)),
    ((0.1, -0.2, 0.30000000000000004), 0.1, (37, 29, 51)),
    ((-12.5, 3.75, -0.0625), 0.3, (17, 64, 23)),
])
def test_threshold_tables_reproduce_reference_cells_and_bins(origin, voxel, dims):
    rng = np.random.default_rng(1)
    plain = tables(origin, voxel, dims, 0)
    fine = tables(origin, voxel, dims, 1)
    for a in range(3):
        T = plain[a]
        P = probes(T, rng)
        want = ref_index(P, origin[a], voxel)
        inb = (want >= 0) & (want < dims[a])
        got = np.searchsorted(T, P, side="right") - 1  # largest k with T[k] <= P
        got_in = (got >= 0) & (got < dims[a])
        np.testing.assert_array_equal(got_in, inb)
        np.testing.assert_array_equal(got[inb], want[inb].astype(np.int64))
    # fine z: cell and quarter bin (zb = f32(oz + (iz + b/4) v), volume.cuh)
    F = fine[2]
    P = probes(F, rng)
    m = np.searchsorted(F, P, side="right") - 1
    iz = ref_index(P, origin[2], voxel)
    ok = (iz >= 0) & (iz < dims[2])
    np.testing.assert_array_equal((m >= 0) & (m < 4 * dims[2]), ok)
    z32 = P[ok].astype(np.float32)
    izk = iz[ok]
    zb = [((origin[2] + (izk + 0.25 * b) * voxel)).astype(np.float32) for b in (1, 2, 3)]
    bin_ref = sum((z32 >= zb[b]).astype(np.int64) for b in range(3))
    np.testing.assert_array_equal(m[ok] >> 2, izk.astype(np.int64))
    np.testing.assert_array_equal(m[ok] & 3, bin_ref)
