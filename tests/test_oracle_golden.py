"""Pins the CPU oracle (oracle/) to outputs of the real reference
(tests/golden/golden.npz, produced by tests/golden/make_golden.py from
/root/reference).  CPU only."""
import numpy as np
import pytest

from golden_io import REC_KEYS, SEAL_KEYS
from oracle import oracle

FILL_ORIGIN = (0.5, -1.0, 2.0)
FILL_VOXEL = 0.5


@pytest.mark.parametrize("key", REC_KEYS)
def test_oracle_reconstruct_matches_reference(golden, key):
    rec, voxel, margin = golden.sweep(key)
    v = oracle.reconstruct(rec, voxel, margin)
    ref = golden.volume(key + ".out")
    np.testing.assert_array_equal(v.origin, ref.origin)
    assert v.dims == ref.dims
    for name in ("cell_starts", "cell_counts", "positions", "orientations", "intensities"):
        np.testing.assert_array_equal(getattr(v, name), getattr(ref, name), err_msg=name)
    assert v.rejected_out_of_bounds == ref.rejected_out_of_bounds


@pytest.mark.parametrize("key", SEAL_KEYS)
def test_oracle_seal_matches_reference(golden, key):
    b = golden[f"{key}.bounds"]
    v = oracle.seal_samples(b[:3], float(golden[f"{key}.voxel"]),
                            tuple(int(np.floor(e / float(golden[f"{key}.voxel"]))) + 1 for e in b[3:] - b[:3]),
                            golden[f"{key}.in_pos"], golden[f"{key}.in_quat"], golden[f"{key}.in_inten"])
    ref = golden.volume(key + ".out")
    for name in ("cell_starts", "cell_counts", "positions", "orientations", "intensities"):
        np.testing.assert_array_equal(getattr(v, name), getattr(ref, name), err_msg=name)
    assert v.rejected_out_of_bounds == ref.rejected_out_of_bounds


def test_oracle_reslice_matches_reference(golden):
    n = 0
    for i, c in golden.reslice_cases():
        vol = golden.full_volume(c.vol_key)
        p = oracle.plane_params(c.plane)
        cfg = oracle.cfg_array(c.cfg)
        px, cov = oracle.reslice(vol, p, cfg, c.plane.width, c.plane.height, c.cfg.unassigned_value)
        np.testing.assert_array_equal(px, c.pixels, err_msg=f"rs_{i}")
        np.testing.assert_array_equal(cov, c.coverage, err_msg=f"rs_{i}")
        if c.brute is not None:
            bp, bc = oracle.reslice(vol, p, cfg, c.plane.width, c.plane.height, c.cfg.unassigned_value,
                                    brute=True)
            np.testing.assert_array_equal(bp, c.brute[0])
            np.testing.assert_array_equal(bc, c.brute[1])
        n += 1
    assert n >= 40


@pytest.mark.parametrize("key", ("rec_tilt", "rec_mask", "rec_parallel", "rec_margin0"))
def test_oracle_compound_matches_reference(golden, key):
    rec, voxel, margin = golden.sweep(key)
    origin, _, dims, values, flags, counts = oracle.compound(rec, voxel, margin)
    np.testing.assert_array_equal(origin, golden[f"cmp_{key}.origin"])
    assert tuple(dims) == tuple(golden[f"cmp_{key}.dims"])
    np.testing.assert_array_equal(values, golden[f"cmp_{key}.values"])
    np.testing.assert_array_equal(flags, golden[f"cmp_{key}.flags"])
    np.testing.assert_array_equal(counts, golden[f"cmp_{key}.counts"])


@pytest.mark.parametrize("i", range(6))
def test_oracle_fill_and_trilinear_match_reference(golden, i):
    dims = tuple(int(d) for d in golden[f"fill_{i}.dims"])
    values, flags = oracle.fill_holes(golden[f"fill_{i}.in_values"], golden[f"fill_{i}.in_flags"], dims,
                                      int(golden[f"fill_{i}.passes"]))
    np.testing.assert_array_equal(values, golden[f"fill_{i}.values"])
    np.testing.assert_array_equal(flags, golden[f"fill_{i}.flags"])
    for j in range(3):
        key = f"tri_{i}_{j}"
        plane = golden.trilinear_plane(key)
        px, cov, _ = oracle.trilinear(FILL_ORIGIN, FILL_VOXEL, dims, values, flags, oracle.plane_params(plane),
                                      plane.width, plane.height)
        np.testing.assert_array_equal(px, golden[f"{key}.pixels"])
        np.testing.assert_array_equal(cov, golden[f"{key}.coverage"])


def test_oracle_exp_is_libm(golden):
    y = oracle.exp(golden["exp.x"])
    np.testing.assert_array_equal(y.view(np.uint64), golden["exp.y"].view(np.uint64))
