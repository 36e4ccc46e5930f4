"""Generate tests/golden/eval.npz: outputs of the REAL reference's evaluation
module (pkg/src/dare/evaluation.py: ncc, ssim, compare_images, run_comparison,
wilcoxon_signed_rank) on seeded image pairs, for the evaluation harness's
oracle (oracle.similarity) and GPU path (csrc/similarity.cu).

    python tests/golden/make_golden_eval.py

Cases (inputs stored in the file): u8 pairs with and without coverage masks at
several sizes (incl. 256x256 reslice-like images), f64 images, custom windows
and constants, and the undefined cases (too few valid pixels, zero variance,
no complete window, image smaller than the window).  Metric values are stored
as f64; a missing value is NaN with the reference's error message.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "eval.npz")


def blob_mask(rng, h, w, k=3):
    yy, xx = np.mgrid[0:h, 0:w]
    m = np.zeros((h, w), bool)
    for _ in range(k):
        cy, cx, r = rng.uniform(0, h), rng.uniform(0, w), rng.uniform(0.2, 0.6) * min(h, w)
        m |= (yy - cy) ** 2 + (xx - cx) ** 2 < r * r
    return m


def cases(rng):
    out = []
    for h, w in ((16, 16), (33, 47), (64, 64), (96, 80), (256, 256)):
        t = rng.integers(0, 256, (h, w)).astype(np.uint8)
        # smooth-ish truth so SSIM is informative
        t = np.clip(np.cumsum(rng.integers(-9, 10, (h, w)), axis=1) + 128, 0, 255).astype(np.uint8)
        c = np.clip(t.astype(int) + rng.integers(-25, 26, t.shape), 0, 255).astype(np.uint8)
        out.append(dict(a=c, b=t, am=None, bm=None, window=7))
        out.append(dict(a=c, b=t, am=blob_mask(rng, h, w), bm=None, window=7))
        out.append(dict(a=c, b=t, am=blob_mask(rng, h, w), bm=rng.random((h, w)) < 0.97, window=7))
    a = rng.integers(0, 256, (40, 40)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-40, 41, a.shape), 0, 255).astype(np.uint8)
    out.append(dict(a=a, b=b, am=None, bm=None, window=3))
    out.append(dict(a=a, b=b, am=blob_mask(rng, 40, 40), bm=None, window=9))
    out.append(dict(a=a, b=b, am=None, bm=None, window=11, c1=1.0, c2=3.0))
    out.append(dict(a=a, b=255 - a, am=None, bm=None, window=7))
    fa = rng.uniform(0, 255, (20, 24))
    fb = np.clip(fa + rng.normal(0, 12, fa.shape), 0, 255)
    out.append(dict(a=fa, b=fb, am=None, bm=None, window=7))
    out.append(dict(a=fa, b=1.7 * fa + 11.0, am=blob_mask(rng, 20, 24), bm=None, window=7))
    # undefined cases
    z = np.zeros((16, 16), np.uint8)
    m1 = np.zeros((16, 16), bool)
    m1[3, 4] = True
    out.append(dict(a=a[:16, :16], b=b[:16, :16], am=m1, bm=None, window=7))  # < 2 valid
    out.append(dict(a=np.full((12, 12), 9, np.uint8), b=a[:12, :12], am=None, bm=None, window=7))  # flat
    m3 = np.zeros((16, 16), bool)
    m3[:3, :3] = True
    out.append(dict(a=a[:16, :16], b=b[:16, :16], am=m3, bm=None, window=7))  # no complete window
    out.append(dict(a=a[:5, :30], b=b[:5, :30], am=None, bm=None, window=7))  # smaller than window
    out.append(dict(a=z, b=z, am=None, bm=None, window=7))  # flat, ssim defined
    return out


def main() -> None:
    sys.path.insert(0, REF)
    from dare.errors import UndefinedMetricError
    from dare.evaluation import ncc, run_comparison, ssim, wilcoxon_signed_rank
    from dare.reslice import ResliceImage

    rng = np.random.default_rng(20260)
    g = {}
    cs = cases(rng)
    g["n_cases"] = np.int64(len(cs))
    for i, c in enumerate(cs):
        kw = {k: c[k] for k in ("c1", "c2") if k in c}
        g[f"c{i}.a"], g[f"c{i}.b"] = c["a"], c["b"]
        for k in ("am", "bm"):
            if c[k] is not None:
                g[f"c{i}.{k}"] = c[k]
        g[f"c{i}.window"] = np.int64(c["window"])
        g[f"c{i}.c1c2"] = np.array([kw.get("c1", np.nan), kw.get("c2", np.nan)])
        for name, fn in (("ncc", lambda: ncc(c["a"], c["b"], c["am"], c["bm"])),
                         ("ssim", lambda: ssim(c["a"], c["b"], c["am"], c["bm"], window=c["window"], **kw))):
            try:
                g[f"c{i}.{name}"] = np.float64(fn())
                g[f"c{i}.{name}_err"] = np.str_("")
            except UndefinedMetricError as e:
                g[f"c{i}.{name}"] = np.float64(np.nan)
                g[f"c{i}.{name}_err"] = np.str_(str(e))
    # run_comparison: 24 pairs of 48x64 reslice-like images, some excluded
    truths, A, B = [], [], []
    for k in range(24):
        t = np.clip(np.cumsum(rng.integers(-9, 10, (48, 64)), axis=1) + 128, 0, 255).astype(np.uint8)
        cov_t = np.ones(t.shape, bool)
        ca = blob_mask(rng, 48, 64, 4) if k % 5 else np.zeros(t.shape, bool)  # every 5th: no overlap
        a = np.clip(t.astype(int) + rng.integers(-6, 7, t.shape), 0, 255).astype(np.uint8)
        b = np.clip(t.astype(int) + rng.integers(-30, 31, t.shape), 0, 255).astype(np.uint8)
        truths.append(ResliceImage(pixels=t, coverage=cov_t, timing_ms=0.0))
        A.append(ResliceImage(pixels=a, coverage=ca, timing_ms=1.0))
        B.append(ResliceImage(pixels=b, coverage=np.ones(t.shape, bool), timing_ms=2.0))
        g[f"rc{k}.t"], g[f"rc{k}.a"], g[f"rc{k}.b"], g[f"rc{k}.ca"] = t, a, b, ca
    rep = run_comparison(A, B, truths)
    g["rc.report"] = np.str_(json.dumps(rep.to_json_dict(), sort_keys=True))
    # wilcoxon: exact (ties, n <= 25) and normal approximation (n > 25, ties)
    w = {}
    for k, d in enumerate([rng.integers(-5, 6, 12), rng.normal(0, 1, 20), rng.integers(-9, 10, 60),
                           rng.normal(0.3, 1, 200), [1, 2, 3, 4, 5, 6, 0, 0]]):
        d = np.asarray(d, float)
        g[f"w{k}.d"] = d
        w[k] = wilcoxon_signed_rank(d)
        g[f"w{k}.p"] = np.float64(w[k])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(cs)} cases, {len(A)} comparison pairs")


if __name__ == "__main__":
    main()
