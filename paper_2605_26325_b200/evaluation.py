"""Evaluation harness on the GPU.

Drop-in for the reference's `dare.evaluation` (pkg/src/dare/evaluation.py):
masked NCC / SSIM (41-84), compare_images (150-160), run_comparison
(193-263), the paired Wilcoxon test (87-140), latency statistics, timing and
report files (266-355).  The image metrics of a whole comparison -- every
(method, pair) against its ground truth -- are computed in one batched launch
(csrc/similarity.cu, `dare_similarity`): SSIM is bit-identical to the
reference for integer-valued images (the u8 reslices), NCC agrees to rounding
(its dot products are BLAS in the reference).  The statistics over the
per-pair metrics stay on the host (tens of numbers).

B200 extensions: `similarity_batch` (numpy or CUDA torch tensors, [P,H,W]),
`compare_images_batch`, and `evaluate_planes` -- the evaluation loop of the
reference CLI benchmark (cli.py:221-287) with directional reslices, trilinear
baseline reslices and the metrics batched on the device.
"""
from __future__ import annotations

import csv
import ctypes
import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InvalidArgumentError, UndefinedMetricError

SSIM_DEFAULT_WINDOW = 7
SSIM_C1 = (0.01 * 255.0) ** 2
SSIM_C2 = (0.03 * 255.0) ** 2

# status bits of dare_similarity
_NCC_FEW, _NCC_FLAT, _SSIM_NO_WINDOW, _SSIM_SMALL = 1, 2, 4, 8
_MSG = {
    _NCC_FEW: "ncc needs at least 2 mutually valid pixels",
    _NCC_FLAT: "ncc undefined for zero-variance input",
    _SSIM_NO_WINDOW: "no complete ssim window inside the mask intersection",
    _SSIM_SMALL: "image smaller than the ssim window",
}


@dataclass(frozen=True)
class SimilarityResult:
    ncc: float
    ssim: float
    valid_pixel_count: int


@dataclass
class SimilarityBatch:
    """Per-pair outputs of one dare_similarity launch."""
    ncc: np.ndarray      # f64 [P]
    ssim: np.ndarray     # f64 [P]
    valid: np.ndarray    # i64 [P] mask-intersection pixel counts
    status: np.ndarray   # i32 [P] status bits (see include/dare_b200.h)

    def ncc_error(self, i: int) -> str | None:
        s = int(self.status[i])
        for bit in (_NCC_FEW, _NCC_FLAT):
            if s & bit:
                return _MSG[bit]
        return None

    def ssim_error(self, i: int) -> str | None:
        s = int(self.status[i])
        for bit in (_SSIM_SMALL, _SSIM_NO_WINDOW):
            if s & bit:
                return _MSG[bit]
        return None


def _is_torch(x) -> bool:
    return hasattr(x, "data_ptr") and hasattr(x, "is_cuda")


def _check_window(window: int) -> None:
    if window % 2 == 0 or window < 3:
        raise InvalidArgumentError("ssim window must be odd and >= 3")


def similarity_batch(a, b, a_mask=None, b_mask=None, window: int = SSIM_DEFAULT_WINDOW,
                     c1: float = SSIM_C1, c2: float = SSIM_C2) -> SimilarityBatch:
    """NCC + SSIM + valid count for every pair (a[p], b[p]) in one launch.

    a, b: [P, H, W] or [H, W] arrays (numpy: uint8 stays u8, anything else is
    taken as f64 like the reference's np.asarray(..., float64); or CUDA torch
    tensors of dtype uint8/float64, evaluated in place on the current stream).
    Masks: same shape, bool/u8, or None (all valid)."""
    _check_window(window)
    if _is_torch(a) or _is_torch(b):
        return _similarity_torch(a, b, a_mask, b_mask, window, c1, c2)
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise InvalidArgumentError(f"image shapes differ: {a.shape} vs {b.shape}")
    if a.ndim == 2:
        a, b = a[None], b[None]
    if a.ndim != 3:
        raise InvalidArgumentError("images must be [P, H, W] or [H, W]")
    u8 = a.dtype == np.uint8 and b.dtype == np.uint8
    dt = np.uint8 if u8 else np.float64
    a = np.ascontiguousarray(a, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    masks = []
    for m in (a_mask, b_mask):
        if m is None:
            masks.append(None)
            continue
        m = np.asarray(m)
        m = np.broadcast_to(m.reshape(m.shape if m.ndim == 3 else (1, *m.shape)), a.shape)
        masks.append(np.ascontiguousarray(m.astype(bool).view(np.uint8)))
    P, H, W = a.shape
    out = SimilarityBatch(np.zeros(P), np.zeros(P), np.zeros(P, np.int64), np.zeros(P, np.int32))
    if P:
        _lib.call("dare_similarity", P, H, W, 0 if u8 else 1, _lib.vptr(a), _lib.ptr(masks[0], ctypes.c_uint8),
                  _lib.vptr(b), _lib.ptr(masks[1], ctypes.c_uint8), int(window), float(c1), float(c2),
                  _lib.ptr(out.ncc, ctypes.c_double), _lib.ptr(out.ssim, ctypes.c_double),
                  _lib.ptr(out.valid, ctypes.c_int64), _lib.ptr(out.status, ctypes.c_int32))
    return out


def _similarity_torch(a, b, a_mask, b_mask, window, c1, c2) -> SimilarityBatch:
    import torch

    if tuple(a.shape) != tuple(b.shape):
        raise InvalidArgumentError(f"image shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    if a.dim() == 2:
        a, b = a[None], b[None]
        a_mask = None if a_mask is None else a_mask[None]
        b_mask = None if b_mask is None else b_mask[None]
    if not (a.is_cuda and b.is_cuda) or a.dim() != 3:
        raise InvalidArgumentError("device similarity needs CUDA tensors [P, H, W]")
    u8 = a.dtype == torch.uint8 and b.dtype == torch.uint8
    dt = torch.uint8 if u8 else torch.float64
    a = a.to(dt).contiguous()
    b = b.to(dt).contiguous()
    ms = [None if m is None else m.to(torch.uint8).expand(a.shape).contiguous() for m in (a_mask, b_mask)]
    P, H, W = a.shape
    dev = a.device
    nc = torch.empty(P, dtype=torch.float64, device=dev)
    ss = torch.empty(P, dtype=torch.float64, device=dev)
    va = torch.empty(P, dtype=torch.int64, device=dev)
    st = torch.empty(P, dtype=torch.int32, device=dev)
    if P:
        _lib.set_device(dev.index or 0)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.call("dare_similarity_device", P, H, W, 0 if u8 else 1, a.data_ptr(),
                  None if ms[0] is None else ms[0].data_ptr(), b.data_ptr(),
                  None if ms[1] is None else ms[1].data_ptr(), int(window), float(c1), float(c2),
                  nc.data_ptr(), ss.data_ptr(), va.data_ptr(), st.data_ptr(), stream)
    return SimilarityBatch(nc.cpu().numpy(), ss.cpu().numpy(), va.cpu().numpy(), st.cpu().numpy())


def _pair_masks(a, a_mask, b_mask):
    # the reference intersects broadcast masks into an all-true mask of a's shape
    return [None if m is None else np.broadcast_to(np.asarray(m, dtype=bool), np.shape(a)) for m in (a_mask, b_mask)]


def ncc(a, b, a_mask=None, b_mask=None) -> float:
    """Zero-mean normalized cross-correlation over the mask intersection
    (evaluation.py:41-53), on the GPU."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise InvalidArgumentError(f"image shapes differ: {a.shape} vs {b.shape}")
    if a.size < 2:
        raise UndefinedMetricError(_MSG[_NCC_FEW])
    am, bm = _pair_masks(a, a_mask, b_mask)
    # NCC depends on the C-order sequence of valid pixels only
    flat = a.shape if a.ndim == 2 else (1, a.size)
    r = similarity_batch(a.reshape(flat), b.reshape(flat), None if am is None else am.reshape(flat),
                         None if bm is None else bm.reshape(flat))
    err = r.ncc_error(0)
    if err:
        raise UndefinedMetricError(err)
    return float(r.ncc[0])


def ssim(a, b, a_mask=None, b_mask=None, window: int = SSIM_DEFAULT_WINDOW,
         c1: float = SSIM_C1, c2: float = SSIM_C2) -> float:
    """Mean local SSIM over the complete windows of the mask intersection
    (evaluation.py:60-84), on the GPU."""
    _check_window(window)
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise InvalidArgumentError(f"image shapes differ: {a.shape} vs {b.shape}")
    if a.ndim != 2:
        raise InvalidArgumentError("ssim needs 2-D images")
    if a.shape[0] < window or a.shape[1] < window:
        raise UndefinedMetricError(_MSG[_SSIM_SMALL])
    am, bm = _pair_masks(a, a_mask, b_mask)
    r = similarity_batch(a, b, am, bm, window, c1, c2)
    err = r.ssim_error(0)
    if err:
        raise UndefinedMetricError(err)
    return float(r.ssim[0])


def compare_images_batch(candidates, truths) -> list:
    """compare_images (evaluation.py:150-160) for every (candidate, truth)
    pair, pairs of one raster size sharing a launch.  Each entry is a
    SimilarityResult or the UndefinedMetricError compare_images would raise."""
    if len(candidates) != len(truths):
        raise InvalidArgumentError("candidate and truth lists differ in length")
    out: list = [None] * len(candidates)
    groups: dict[tuple, list[int]] = {}
    for i, (c, t) in enumerate(zip(candidates, truths)):
        if np.shape(c.pixels) != np.shape(t.pixels):
            raise InvalidArgumentError(f"image shapes differ: {np.shape(c.pixels)} vs {np.shape(t.pixels)}")
        groups.setdefault(np.shape(c.pixels), []).append(i)
    for shape, idx in groups.items():
        if len(shape) != 2:
            raise InvalidArgumentError("ResliceImage pixels must be 2-D")
        stack = lambda imgs, attr, dt: np.stack([np.asarray(getattr(imgs[i], attr), dtype=dt) for i in idx])
        r = similarity_batch(stack(candidates, "pixels", np.uint8), stack(truths, "pixels", np.uint8),
                             stack(candidates, "coverage", bool), stack(truths, "coverage", bool))
        for k, i in enumerate(idx):
            if r.valid[k] == 0:
                out[i] = UndefinedMetricError("coverage masks do not intersect")
            elif (err := r.ncc_error(k) or r.ssim_error(k)) is not None:
                out[i] = UndefinedMetricError(err)
            else:
                out[i] = SimilarityResult(ncc=float(r.ncc[k]), ssim=float(r.ssim[k]),
                                          valid_pixel_count=int(r.valid[k]))
    return out


def compare_images(candidate, truth) -> SimilarityResult:
    """Both metrics over the intersection of the two coverage masks."""
    r = compare_images_batch([candidate], [truth])[0]
    if isinstance(r, Exception):
        raise r
    return r


# ---- paired statistics (host: a few numbers per pair) -----------------------

def _midranks(values: np.ndarray) -> np.ndarray:
    """Average 1-based ranks with ties sharing the mean rank (evaluation.py:113-122)."""
    order = np.argsort(values, kind="stable")
    sv = values[order]
    ranks = np.empty(len(values), dtype=float)
    starts = np.flatnonzero(np.r_[True, sv[1:] != sv[:-1]])
    ends = np.r_[starts[1:], len(sv)] - 1
    for i, j in zip(starts, ends):
        ranks[order[i:j + 1]] = 0.5 * (i + j) + 1.0
    return ranks


def _exact_p(ranks: np.ndarray, w_plus: float) -> float:
    """Exact two-sided tail over all 2^n sign patterns (evaluation.py:125-140):
    subset-sum counts over doubled (integral) midranks."""
    doubled = [int(r) for r in np.rint(2.0 * ranks).astype(np.int64)]
    total = sum(doubled)
    ways = [1] + [0] * total
    for r in doubled:
        for s in range(total, r - 1, -1):
            ways[s] += ways[s - r]
    w2 = int(round(2.0 * w_plus))
    le = sum(ways[: w2 + 1])
    ge = sum(ways[w2:])
    return min(1.0, 2.0 * min(le, ge) / (1 << len(doubled)))


def wilcoxon_signed_rank(diffs) -> float:
    """Two-sided p for paired differences, zeros dropped: exact for n <= 25,
    normal approximation with tie correction above (evaluation.py:87-110)."""
    d = np.asarray(diffs, dtype=float)
    d = d[d != 0.0]
    n = d.size
    if n < 5:
        raise InvalidArgumentError(f"wilcoxon needs >= 5 nonzero differences, got {n}")
    ranks = _midranks(np.abs(d))
    w_plus = float(ranks[d > 0].sum())
    if n <= 25:
        return _exact_p(ranks, w_plus)
    _, ties = np.unique(np.abs(d), return_counts=True)
    var = n * (n + 1) * (2 * n + 1) / 24.0 - float(((ties**3 - ties) / 48.0).sum())
    z = (w_plus - n * (n + 1) / 4.0) / math.sqrt(var)
    return min(1.0, 2.0 * 0.5 * math.erfc(abs(z) / math.sqrt(2.0)))


def _median_iqr(values) -> dict:
    v = np.asarray(values, dtype=float)
    return {"median": float(np.median(v)), "iqr_low": float(np.percentile(v, 25)),
            "iqr_high": float(np.percentile(v, 75))}


def latency_stats(samples_ms) -> dict:
    v = np.asarray(samples_ms, dtype=float)
    return {"count": int(v.size), "median_ms": float(np.median(v)), "p95_ms": float(np.percentile(v, 95)),
            "mean_ms": float(v.mean())}


@dataclass
class ComparisonReport:
    pair_ids: list[str]
    method_a: str
    method_b: str
    results_a: list[SimilarityResult]
    results_b: list[SimilarityResult]
    summary: dict = field(default_factory=dict)
    timing: dict = field(default_factory=dict)

    def to_json_dict(self) -> dict:
        pairs = []
        for pid, ra, rb in zip(self.pair_ids, self.results_a, self.results_b):
            entry = {"id": pid}
            for name, r in ((self.method_a, ra), (self.method_b, rb)):
                entry[name] = {"ncc": r.ncc, "ssim": r.ssim, "valid": r.valid_pixel_count}
            pairs.append(entry)
        return {"methods": [self.method_a, self.method_b], "pairs": pairs, "summary": self.summary,
                "timing": self.timing}


def _metric_summary(method_a, method_b, va, vb) -> dict:
    entry = {method_a: _median_iqr(va), method_b: _median_iqr(vb)}
    diffs = np.asarray(va) - np.asarray(vb)
    if not np.any(diffs != 0.0):
        entry.update(wilcoxon_p=1.0, wilcoxon_note="no difference")
        return entry
    try:
        entry["wilcoxon_p"] = wilcoxon_signed_rank(diffs)
    except InvalidArgumentError:
        entry.update(wilcoxon_p=None, wilcoxon_note="too few nonzero paired differences")
    return entry


def run_comparison(images_a, images_b, ground_truths, pair_ids=None, method_a: str = "dare",
                   method_b: str = "baseline", latencies=None) -> ComparisonReport:
    """Paired evaluation of two methods against shared ground truths
    (evaluation.py:193-263): per-pair NCC/SSIM for all 2P comparisons in one
    batched launch, medians with IQR and the paired Wilcoxon p per metric;
    pairs with an undefined metric on either side are excluded from both."""
    if not images_a or not (len(images_a) == len(images_b) == len(ground_truths)):
        raise InvalidArgumentError("paired comparison needs equal-length non-empty image sets")
    ids = list(pair_ids) if pair_ids is not None else [f"pair{k:04d}" for k in range(len(images_a))]
    n = min(len(ids), len(images_a))  # the reference zips ids with the images
    images_a, images_b, ground_truths = images_a[:n], images_b[:n], ground_truths[:n]
    results = compare_images_batch(list(images_a) + list(images_b), list(ground_truths) * 2)
    kept, ra, rb, excluded = [], [], [], []
    for k in range(n):
        bad = next((r for r in (results[k], results[n + k]) if isinstance(r, Exception)), None)
        if bad is not None:
            excluded.append({"id": ids[k], "reason": str(bad)})
            continue
        kept.append(ids[k])
        ra.append(results[k])
        rb.append(results[n + k])
    if not kept:
        raise InvalidArgumentError("every pair had undefined metrics")
    summary: dict = {"pair_count": len(kept), "excluded_pairs": excluded}
    for metric in ("ncc", "ssim"):
        summary[metric] = _metric_summary(method_a, method_b, [getattr(r, metric) for r in ra],
                                          [getattr(r, metric) for r in rb])
    report = ComparisonReport(kept, method_a, method_b, ra, rb, summary)
    if latencies:
        report.timing = {k: latency_stats(v) for k, v in latencies.items() if len(v) > 0}
    return report


def time_reslice(volume, planes, cfg=None, repetitions: int = 1, warmup: int = 2) -> dict:
    """Wall-clock latency per reslice (query to host image), warm-up calls
    excluded (evaluation.py:266-281)."""
    from .reslice import ResliceConfig, reslice

    if len(planes) < 10:
        raise InvalidArgumentError("latency measurement needs at least 10 planes")
    cfg = cfg or ResliceConfig()
    for plane in planes[:warmup]:
        reslice(volume, plane, cfg)
    samples = []
    for _ in range(repetitions):
        for plane in planes:
            t0 = time.perf_counter()
            reslice(volume, plane, cfg)
            samples.append((time.perf_counter() - t0) * 1e3)
    return latency_stats(samples)


# ---- report files (evaluation.py:287-355) -----------------------------------

def format_summary(report: ComparisonReport) -> str:
    out = [f"paired comparison: {report.method_a} vs {report.method_b} ({len(report.pair_ids)} pairs)"]
    excluded = report.summary.get("excluded_pairs", [])
    if excluded:
        out.append(f"excluded {len(excluded)} pair(s) with undefined metrics")
    out.append("")
    for metric in ("ncc", "ssim"):
        entry = report.summary.get(metric)
        if entry is None:
            continue
        out.append(metric.upper())
        for m in (report.method_a, report.method_b):
            s = entry[m]
            out.append(f"  {m:<10} median {s['median']:+.4f} (IQR {s['iqr_low']:+.4f} .. {s['iqr_high']:+.4f})")
        p, note = entry["wilcoxon_p"], entry.get("wilcoxon_note")
        out.append("  wilcoxon two-sided p = " + ("n/a" if p is None else f"{p:.3e}") + (f" ({note})" if note else ""))
        out.append("")
    for name, s in report.timing.items():
        out.append(f"latency[{name}]: median {s['median_ms']:.2f} ms, p95 {s['p95_ms']:.2f} ms over {s['count']} reslices")
    return "\n".join(out) + "\n"


def write_report(report: ComparisonReport, out_dir, latency_by_pair=None) -> dict:
    """report.json, pairs.csv (id, method, ncc, ssim, latency_ms) and summary.txt."""
    os.makedirs(out_dir, exist_ok=True)
    paths = {k: os.path.join(out_dir, f) for k, f in
             (("json", "report.json"), ("csv", "pairs.csv"), ("txt", "summary.txt"))}
    with open(paths["json"], "w", encoding="utf-8") as fh:
        json.dump(report.to_json_dict(), fh, indent=2, sort_keys=True)
        fh.write("\n")
    with open(paths["csv"], "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["id", "method", "ncc", "ssim", "latency_ms"])
        for pid, ra, rb in zip(report.pair_ids, report.results_a, report.results_b):
            for m, r in ((report.method_a, ra), (report.method_b, rb)):
                lat = (latency_by_pair or {}).get(pid)
                w.writerow([pid, m, f"{r.ncc:.9f}", f"{r.ssim:.9f}",
                            "" if lat is None else f"{lat.get(m, float('nan')):.3f}"])
    with open(paths["txt"], "w", encoding="utf-8") as fh:
        fh.write(format_summary(report))
    return paths


# ---- the CLI benchmark's evaluation loop, batched ---------------------------

def evaluate_planes(volume, scalar, planes, truths, cfg=None, pair_ids=None) -> ComparisonReport:
    """cli.py:253-287 for one raster size: directional reslices of `volume`
    (one reslice_batch launch), trilinear reslices of the filled `scalar`
    volume (one launch), both compared with the ground-truth images `truths`
    (ResliceImages, e.g. the phantom rendered at each plane) in one
    similarity launch, then run_comparison's statistics."""
    from .reslice import ResliceImage, reslice_batch
    from .scalar import reslice_trilinear_batch

    dp, dc, dms = reslice_batch(volume, planes, cfg)
    bp, bc, bms = reslice_trilinear_batch(scalar, planes)
    per_a = dms / max(len(planes), 1)
    per_b = bms / max(len(planes), 1)
    a = [ResliceImage(pixels=dp[k], coverage=dc[k], timing_ms=per_a) for k in range(len(planes))]
    b = [ResliceImage(pixels=bp[k], coverage=bc[k], timing_ms=per_b) for k in range(len(planes))]
    return run_comparison(a, b, truths, pair_ids)
