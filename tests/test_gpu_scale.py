"""Parity with the REAL reference at BASELINE scale (tests/golden/scale.npz,
made by tests/golden/make_golden_scale.py from /root/reference's own
reconstruct_volume / save_volume / reslice / compound / fill_holes /
reslice_trilinear).  The GPU path rebuilds the same inputs and must reproduce
every hash bit-for-bit:

  cfg1   (BASELINE configs[0]) 200 x 128^2 -> 128^3: .darevol bytes, 64 reslices,
         compound, fill_holes (every 4th frame), 64 trilinear reslices
  cfg1t  the same frames on a tracked sweep (47 Hz pose stream -> slerp,
         calibration, margin 0.5)
  cfg2   (BASELINE configs[1]) 1000 x 512^2 -> 256^3 (262M samples): .darevol
         bytes (7.6 GB, streamed from HBM through a hashing sink), 24 reslices,
         compound, fill_holes (every 8th frame), 24 trilinear reslices
"""
import numpy as np
import pytest

import paper_2605_26325_b200 as db
from scale_io import HashSink, Scale, sha

pytestmark = pytest.mark.gpu

SCALE = Scale()
NAMES = [n for n in ("cfg1", "cfg1t", "cfg2") if SCALE.has(n)]


@pytest.fixture(scope="module", params=NAMES)
def built(request):
    name = request.param
    frames = SCALE.frames(name)
    assert sha(frames) == str(SCALE[f"{name}.frames_sha256"]), "frame generator drifted"
    sp = SCALE.spec(name)
    sweep = SCALE.sweep(name, frames)
    vol = db.reconstruct_volume(sweep, voxel_size=sp["voxel"], margin=sp["margin"])
    yield name, sp, sweep, vol
    del vol


def test_scale_reconstruct_darevol_bytes(built):
    name, sp, sweep, vol = built
    assert vol.dims == tuple(int(d) for d in SCALE[f"{name}.dims"])
    np.testing.assert_array_equal(vol.origin, SCALE[f"{name}.origin"])
    assert vol.sample_count == int(SCALE[f"{name}.n_samples"])
    assert vol.rejected_out_of_bounds == int(SCALE[f"{name}.rejected"])
    sink = HashSink()
    db.save_volume(vol, sink)  # streamed from HBM (host views never materialised)
    assert vol._host is None
    assert sink.size == int(SCALE[f"{name}.darevol_size"])
    assert sink.hexdigest() == str(SCALE[f"{name}.darevol_sha256"])


def test_scale_reslice_hashes(built):
    name, sp, sweep, vol = built
    planes = SCALE.planes(name)
    px, cov, _ = db.reslice_batch(vol, planes, SCALE.cfg(name))
    got_p = [sha(px[k]) for k in range(len(planes))]
    got_c = [sha(cov[k]) for k in range(len(planes))]
    bad = [k for k in range(len(planes))
           if got_p[k] != str(SCALE[f"{name}.rs_pix"][k]) or got_c[k] != str(SCALE[f"{name}.rs_cov"][k])]
    assert not bad, f"{len(bad)} of {len(planes)} poses differ from the reference: {bad[:8]}"
    # the single-pose public entry point agrees as well
    img = db.reslice(vol, planes[0], SCALE.cfg(name))
    assert sha(img.pixels) == str(SCALE[f"{name}.rs_pix"][0])
    assert sha(img.coverage) == str(SCALE[f"{name}.rs_cov"][0])


def test_scale_reslice_exact_mode_hashes(built):
    """The FP64-everywhere path (cfg.exact) gives the same reference bytes."""
    name, sp, sweep, vol = built
    from paper_2605_26325_b200 import _lib
    from paper_2605_26325_b200.reslice import kernel_cfg, plane_params
    import ctypes

    planes = SCALE.planes(name)[:8]
    params = np.ascontiguousarray([plane_params(p) for p in planes], dtype=np.float64)
    h = w = sp["plane"]
    px = np.empty((len(planes), h, w), np.uint8)
    cov = np.empty((len(planes), h, w), np.uint8)
    kc = kernel_cfg(SCALE.cfg(name), 0, exact=True)
    _lib.call("dare_reslice", vol.device_handle().raw, len(planes), _lib.ptr(params, ctypes.c_double), w, h,
              ctypes.byref(kc), _lib.ptr(px, ctypes.c_uint8), _lib.ptr(cov, ctypes.c_uint8))
    for k in range(len(planes)):
        assert sha(px[k]) == str(SCALE[f"{name}.rs_pix"][k])
        assert sha(cov[k].astype(bool)) == str(SCALE[f"{name}.rs_cov"][k])


@pytest.mark.parametrize("name", NAMES)
def test_scale_scalar_arm_hashes(name):
    sp = SCALE.spec(name)
    frames = SCALE.frames(name)
    s = db.compound(SCALE.sweep(name, frames), voxel_size=sp["voxel"], margin=sp["margin"])
    assert sha(s.values) == str(SCALE[f"{name}.cmp_values"])
    assert sha(s.flags) == str(SCALE[f"{name}.cmp_flags"])
    assert sha(np.asarray(s.counts, dtype=np.int64)) == str(SCALE[f"{name}.cmp_counts"])
    del s
    sparse = db.compound(SCALE.sweep(name, frames, every=sp["sparse"]), voxel_size=sp["voxel"],
                         margin=sp["margin"])
    assert int(np.count_nonzero(sparse.flags)) == int(SCALE[f"{name}.sparse_observed"])
    filled = db.fill_holes(sparse, 3)
    assert int(np.count_nonzero(np.asarray(filled.flags) == 2)) == int(SCALE[f"{name}.fill_filled"])
    assert sha(filled.values) == str(SCALE[f"{name}.fill_values"])
    assert sha(filled.flags) == str(SCALE[f"{name}.fill_flags"])
    planes = SCALE.planes(name)
    px, cov = db.reslice_trilinear_batch(filled, planes)[:2]
    bad = [k for k in range(len(planes)) if sha(px[k]) != str(SCALE[f"{name}.tri_pix"][k])
           or sha(np.asarray(cov[k], dtype=bool)) != str(SCALE[f"{name}.tri_cov"][k])]
    assert not bad, f"trilinear poses differ from the reference: {bad[:8]}"
