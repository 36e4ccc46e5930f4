"""CPU: the evaluation oracle (oracle.similarity) and the host statistics of
paper_2605_26325_b200.evaluation against the REAL reference's outputs
(tests/golden/eval.npz).  SSIM: bit-identical (integer-valued window sums are
exact, the window mean is numpy's pairwise order); NCC: within 1e-13 (the
reference's dot products are BLAS, host-order dependent)."""
import math

import numpy as np
import pytest

from eval_io import EvalGolden
from oracle import oracle
from paper_2605_26325_b200 import evaluation as ev
from paper_2605_26325_b200.errors import InvalidArgumentError

G = EvalGolden()
NCC_TOL = 1e-13

MSG = {1: "ncc needs at least 2 mutually valid pixels", 2: "ncc undefined for zero-variance input",
       4: "no complete ssim window inside the mask intersection", 8: "image smaller than the ssim window"}


def _errors(status):
    ncc_err = next((MSG[b] for b in (1, 2) if status & b), "")
    ssim_err = next((MSG[b] for b in (8, 4) if status & b), "")
    return ncc_err, ssim_err


@pytest.mark.parametrize("case", list(G.cases()), ids=lambda c: f"c{c['i']}")
def test_oracle_similarity_matches_reference(case):
    nc, ss, n, st = oracle.similarity(case["a"], case["b"], case["am"], case["bm"], case["window"], **case["kw"])
    ne, se = _errors(st)
    assert ne == case["ncc_err"] and se == case["ssim_err"]
    if not ne:
        assert abs(nc - case["ncc"]) <= NCC_TOL
    if not se:
        assert ss == case["ssim"]  # bit-identical


@pytest.mark.parametrize("k", range(5))
def test_wilcoxon_matches_reference_bit_for_bit(k):
    d, p = list(G.wilcoxon())[k]
    assert ev.wilcoxon_signed_rank(d) == p


def test_wilcoxon_contract():
    assert ev.wilcoxon_signed_rank([1, 2, 3, 4, 5, 6]) == 0.03125
    assert ev.wilcoxon_signed_rank([3, -3, 5, -5, 7, -7]) == 1.0
    with pytest.raises(InvalidArgumentError):
        ev.wilcoxon_signed_rank([1, 2, 0, 0, 3])


def test_run_comparison_statistics_match_reference(monkeypatch):
    """run_comparison's host logic (exclusions, medians / IQR, Wilcoxon) with
    the per-pair metrics supplied by the oracle (the GPU test runs the same
    comparison through dare_similarity)."""
    A, B, T, ref = G.comparison()

    def oracle_batch(cands, truths):
        out = []
        for c, t in zip(cands, truths):
            inter = int(np.count_nonzero(c.coverage & t.coverage))
            nc, ss, n, st = oracle.similarity(c.pixels, t.pixels, c.coverage, t.coverage)
            ne, se = _errors(st)
            if inter == 0:
                out.append(ev.UndefinedMetricError("coverage masks do not intersect"))
            elif ne or se:
                out.append(ev.UndefinedMetricError(ne or se))
            else:
                out.append(ev.SimilarityResult(nc, ss, n))
        return out

    monkeypatch.setattr(ev, "compare_images_batch", oracle_batch)
    rep = ev.run_comparison(A, B, T).to_json_dict()
    assert_report_close(rep, ref)


def assert_report_close(rep, ref):
    assert rep["methods"] == ref["methods"]
    assert [p["id"] for p in rep["pairs"]] == [p["id"] for p in ref["pairs"]]
    assert rep["summary"]["excluded_pairs"] == ref["summary"]["excluded_pairs"]
    assert rep["summary"]["pair_count"] == ref["summary"]["pair_count"]
    for p, q in zip(rep["pairs"], ref["pairs"]):
        for m in ref["methods"]:
            assert p[m]["valid"] == q[m]["valid"]
            assert p[m]["ssim"] == q[m]["ssim"]
            assert abs(p[m]["ncc"] - q[m]["ncc"]) <= NCC_TOL
    for metric in ("ncc", "ssim"):
        e, r = rep["summary"][metric], ref["summary"][metric]
        for m in ref["methods"]:
            for k, v in r[m].items():
                assert e[m][k] == v if metric == "ssim" else math.isclose(e[m][k], v, abs_tol=NCC_TOL)
        assert math.isclose(e["wilcoxon_p"], r["wilcoxon_p"], rel_tol=1e-9)
        assert e.get("wilcoxon_note") == r.get("wilcoxon_note")


def test_report_files(tmp_path, monkeypatch):
    A, B, T, _ = G.comparison()
    monkeypatch.setattr(ev, "compare_images_batch",
                        lambda c, t: [ev.SimilarityResult(0.5 + 0.01 * k, 0.25, 100) for k in range(len(c))])
    rep = ev.run_comparison(A[:6], B[:6], T[:6], latencies={"dare": [1.0, 2.0]})
    paths = ev.write_report(rep, tmp_path / "out")
    lines = open(paths["csv"]).read().splitlines()
    assert lines[0] == "id,method,ncc,ssim,latency_ms" and len(lines) == 13
    txt = open(paths["txt"]).read()
    assert txt.startswith("paired comparison: dare vs baseline (6 pairs)") and "latency[dare]" in txt


def test_run_comparison_contract(monkeypatch):
    """Exclusions on either side, pair ids zipped with the images (the
    reference's zip semantics), every pair undefined -> InvalidArgumentError,
    timing statistics from latencies."""
    from paper_2605_26325_b200.reslice import ResliceImage

    img = ResliceImage(pixels=np.zeros((8, 8), np.uint8), coverage=np.ones((8, 8), bool), timing_ms=0.0)
    n = 7

    def fake(cands, truths):
        out = []
        for k in range(len(cands)):
            side, pair = divmod(k, n)
            if (pair == 2 and side == 0) or (pair == 5 and side == 1):
                out.append(ev.UndefinedMetricError(f"undefined {side} {pair}"))
            else:
                out.append(ev.SimilarityResult(0.5 + 0.01 * pair * (1 - side), 0.4 + 0.02 * pair * (1 - side), 64))
        return out

    monkeypatch.setattr(ev, "compare_images_batch", fake)
    rep = ev.run_comparison([img] * n, [img] * n, [img] * n, latencies={"dare": [1.0, 3.0], "baseline": []})
    assert rep.pair_ids == ["pair0000", "pair0001", "pair0003", "pair0004", "pair0006"]
    assert [e["reason"] for e in rep.summary["excluded_pairs"]] == ["undefined 0 2", "undefined 1 5"]
    assert rep.timing == {"dare": ev.latency_stats([1.0, 3.0])}
    rep2 = ev.run_comparison([img] * n, [img] * n, [img] * n, pair_ids=["a", "b", "c"])
    assert rep2.pair_ids == ["a", "b"] and rep2.summary["pair_count"] == 2  # 'c' is pair 2: excluded
    monkeypatch.setattr(ev, "compare_images_batch", lambda c, t: [ev.UndefinedMetricError("x")] * len(c))
    with pytest.raises(InvalidArgumentError, match="every pair had undefined metrics"):
        ev.run_comparison([img] * 3, [img] * 3, [img] * 3)
    with pytest.raises(InvalidArgumentError, match="equal-length non-empty"):
        ev.run_comparison([], [], [])
