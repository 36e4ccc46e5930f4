"""GPU: the evaluation metrics (csrc/similarity.cu through dare_similarity)
against the REAL reference (tests/golden/eval.npz: SSIM bit-identical, NCC
within 1e-12) and against the oracle bit for bit (same summation order:
window sums, numpy's pairwise tree for the means and the NCC products)."""
import math

import numpy as np
import pytest

from eval_io import EvalGolden
from oracle import oracle
from paper_2605_26325_b200 import evaluation as ev
from paper_2605_26325_b200.errors import InvalidArgumentError, UndefinedMetricError
from test_oracle_eval import _errors, assert_report_close

pytestmark = pytest.mark.gpu
G = EvalGolden()


@pytest.mark.parametrize("case", list(G.cases()), ids=lambda c: f"c{c['i']}")
def test_metrics_match_reference_and_oracle(case):
    a, b, am, bm, win, kw = case["a"], case["b"], case["am"], case["bm"], case["window"], case["kw"]
    onc, oss, on, ost = oracle.similarity(a, b, am, bm, win, **kw)
    if case["ncc_err"]:
        with pytest.raises(UndefinedMetricError, match=case["ncc_err"]):
            ev.ncc(a, b, am, bm)
    else:
        v = ev.ncc(a, b, am, bm)
        assert abs(v - case["ncc"]) <= 1e-12
        assert v == onc
    if case["ssim_err"]:
        with pytest.raises(UndefinedMetricError, match=case["ssim_err"]):
            ev.ssim(a, b, am, bm, window=win, **kw)
    else:
        assert ev.ssim(a, b, am, bm, window=win, **kw) == case["ssim"]  # bit-identical
    r = ev.similarity_batch(a, b, am, bm, win, **kw)
    assert int(r.status[0]) == ost and int(r.valid[0]) == on


def _check_batch_vs_oracle(a, b, am, bm, win=7):
    r = ev.similarity_batch(a, b, am, bm, win)
    for p in range(len(a)):
        nc, ss, n, st = oracle.similarity(a[p], b[p], None if am is None else am[p], None if bm is None else bm[p],
                                          win)
        assert (int(r.status[p]), int(r.valid[p])) == (st, n), p
        if not st & 3:
            assert r.ncc[p] == nc, p
        if not st & 12:
            assert r.ssim[p] == ss, p


def test_pairwise_tree_many_sizes(rng):
    """NCC over n valid values for n across the pairwise tree's shapes
    (< 8, <= 128, splits, remainders), f64 data so every order matters."""
    sizes = sorted(set([2, 3, 7, 8, 9, 15, 16, 17, 127, 128, 129, 135, 136, 255, 256, 257, 1000, 1023, 1024, 1031,
                        4095, 4096, 4097, 65543] + list(rng.integers(2, 20000, 30))))
    for n in sizes:
        a = rng.normal(100, 50, (1, 1, n)) * np.exp(rng.uniform(-3, 3, (1, 1, n)))
        b = a + rng.normal(0, 20, a.shape)
        _check_batch_vs_oracle(a, b, None, None)


def test_masked_f64_and_windows(rng):
    for win in (3, 5, 7, 9, 15, 31, 33, 41):
        h, w = int(rng.integers(win, 90)), int(rng.integers(win, 130))
        a = rng.uniform(0, 255, (3, h, w))
        b = np.clip(a + rng.normal(0, 15, a.shape), 0, 255)
        am = rng.random(a.shape) < 0.995
        _check_batch_vs_oracle(a, b, am, None, win)


def test_u8_windows(rng):
    """The u8 window kernel (integer running sums) for compile-time 7 and runtime windows."""
    for win in (3, 5, 7, 9, 15, 33, 63):
        h, w = int(rng.integers(win, win + 90)), int(rng.integers(win, win + 140))
        a = rng.integers(0, 256, (2, h, w)).astype(np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-25, 26, a.shape), 0, 255).astype(np.uint8)
        am = rng.random(a.shape) < 0.998
        bm = rng.random(a.shape) < 0.999
        _check_batch_vs_oracle(a, b, am, bm, win)


def test_u8_batch_full_size(rng):
    """64 reslice-sized (256x256) u8 pairs with coverage masks in one launch,
    plus a 512x512 pair."""
    t = np.clip(np.cumsum(rng.integers(-9, 10, (64, 256, 256)), axis=2) + 128, 0, 255).astype(np.uint8)
    c = np.clip(t.astype(int) + rng.integers(-20, 21, t.shape), 0, 255).astype(np.uint8)
    yy, xx = np.mgrid[0:256, 0:256]
    cov = np.stack([(yy - 128) ** 2 + (xx - 100 - k) ** 2 < (60 + k) ** 2 for k in range(64)])
    r = ev.similarity_batch(c, t, cov, None)
    for p in (0, 17, 63):
        nc, ss, n, st = oracle.similarity(c[p], t[p], cov[p], None)
        assert (r.ncc[p], r.ssim[p], r.valid[p], r.status[p]) == (nc, ss, n, st)
    big = rng.integers(0, 256, (1, 512, 512)).astype(np.uint8)
    big2 = np.clip(big.astype(int) + rng.integers(-50, 51, big.shape), 0, 255).astype(np.uint8)
    _check_batch_vs_oracle(big, big2, rng.random(big.shape) < 0.999, None)


def test_chunked_launches(rng):
    """More 1024^2 pairs than one scratch chunk holds."""
    a = rng.integers(0, 256, (45, 1024, 1024), dtype=np.uint8)
    b = np.clip(a.astype(np.int16) + rng.integers(-30, 31, a.shape, dtype=np.int16), 0, 255).astype(np.uint8)
    r = ev.similarity_batch(a, b)
    for p in (0, 41, 44):
        nc, ss, n, st = oracle.similarity(a[p], b[p])
        assert (r.ncc[p], r.ssim[p], r.valid[p], r.status[p]) == (nc, ss, n, st), p


def test_device_tensors_equal_host_path(rng):
    import torch

    a = rng.integers(0, 256, (5, 70, 90)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    m = rng.random(a.shape) < 0.9
    h = ev.similarity_batch(a, b, m, None)
    d = ev.similarity_batch(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), torch.from_numpy(m).cuda(), None)
    for f in ("ncc", "ssim", "valid", "status"):
        np.testing.assert_array_equal(getattr(h, f), getattr(d, f))


def test_run_comparison_matches_reference_report():
    A, B, T, ref = G.comparison()
    rep = ev.run_comparison(A, B, T).to_json_dict()
    assert_report_close(rep, ref)


def test_compare_images_contract(rng):
    from paper_2605_26325_b200.reslice import ResliceImage

    t = ResliceImage(pixels=rng.integers(0, 256, (16, 16)).astype(np.uint8), coverage=np.ones((16, 16), bool),
                     timing_ms=0.0)
    empty = ResliceImage(pixels=t.pixels, coverage=np.zeros((16, 16), bool), timing_ms=0.0)
    with pytest.raises(UndefinedMetricError, match="coverage masks do not intersect"):
        ev.compare_images(empty, t)
    r = ev.compare_images(t, t)
    assert abs(r.ncc - 1.0) <= 1e-12 and abs(r.ssim - 1.0) <= 1e-12 and r.valid_pixel_count == 256
    with pytest.raises(InvalidArgumentError):
        ev.ssim(np.zeros((16, 16)), np.zeros((16, 16)), window=6)
    with pytest.raises(InvalidArgumentError):
        ev.ncc(np.zeros((4, 4)), np.zeros((4, 5)))


def test_evaluate_planes_equals_composition(rng):
    """The batched CLI evaluation loop == reslice + trilinear + run_comparison
    done one call at a time."""
    import paper_2605_26325_b200 as db
    from paper_2605_26325_b200.geometry import Pose, Quaternion
    from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig, ResliceImage

    n = 40000
    pos = rng.uniform(0, 8, (n, 3)).astype(np.float32)
    quat = np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1))
    inten = rng.integers(0, 256, n).astype(np.uint8)
    vol = db.VolumeBuilder(db.BoundingBox((0.0, 0.0, 0.0), (7.5, 7.5, 7.5)), 0.5)
    vol.insert_batch(pos, quat, inten)
    vol = vol.seal()
    from paper_2605_26325_b200.scalar import ScalarVolume, VOXEL_OBSERVED

    vals = rng.uniform(0, 255, 16 ** 3).astype(np.float32)
    flags = np.full(16 ** 3, VOXEL_OBSERVED, np.uint8)
    sc = ScalarVolume((0.0, 0.0, 0.0), 0.5, (16, 16, 16), vals, flags, np.ones(16 ** 3, np.int64))
    planes = [ReslicePlane(Pose(Quaternion(1.0, 0.0, 0.0, 0.0), (0.5, 0.5, 1.0 + 0.25 * k)), 24, 20, (0.3, 0.3))
              for k in range(12)]
    truths = [ResliceImage(pixels=rng.integers(0, 256, (20, 24)).astype(np.uint8),
                           coverage=np.ones((20, 24), bool), timing_ms=0.0) for _ in planes]
    cfg = ResliceConfig(interp_radius=0.5)
    rep = ev.evaluate_planes(vol, sc, planes, truths, cfg)
    a = [db.reslice(vol, p, cfg) for p in planes]
    b = [db.reslice_trilinear(sc, p) for p in planes]
    ref = ev.run_comparison(a, b, truths)
    assert rep.to_json_dict()["pairs"] == ref.to_json_dict()["pairs"]
    assert rep.summary == ref.summary
