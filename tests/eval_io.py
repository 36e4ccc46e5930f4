"""Loader for tests/golden/eval.npz (outputs of the real reference's
evaluation module; tests/golden/make_golden_eval.py)."""
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "eval.npz")


class EvalGolden:
    def __init__(self):
        self.g = np.load(PATH)

    def cases(self):
        g = self.g
        for i in range(int(g["n_cases"])):
            c1, c2 = g[f"c{i}.c1c2"]
            yield dict(
                i=i, a=g[f"c{i}.a"], b=g[f"c{i}.b"],
                am=g[f"c{i}.am"] if f"c{i}.am" in g else None,
                bm=g[f"c{i}.bm"] if f"c{i}.bm" in g else None,
                window=int(g[f"c{i}.window"]),
                kw={} if np.isnan(c1) else dict(c1=float(c1), c2=float(c2)),
                ncc=float(g[f"c{i}.ncc"]), ncc_err=str(g[f"c{i}.ncc_err"]),
                ssim=float(g[f"c{i}.ssim"]), ssim_err=str(g[f"c{i}.ssim_err"]),
            )

    def comparison(self):
        """(images_a, images_b, truths, reference report dict)."""
        import json

        from paper_2605_26325_b200.reslice import ResliceImage

        g = self.g
        A, B, T = [], [], []
        k = 0
        while f"rc{k}.t" in g:
            t = g[f"rc{k}.t"]
            T.append(ResliceImage(pixels=t, coverage=np.ones(t.shape, bool), timing_ms=0.0))
            A.append(ResliceImage(pixels=g[f"rc{k}.a"], coverage=g[f"rc{k}.ca"], timing_ms=1.0))
            B.append(ResliceImage(pixels=g[f"rc{k}.b"], coverage=np.ones(t.shape, bool), timing_ms=2.0))
            k += 1
        return A, B, T, json.loads(str(g["rc.report"]))

    def wilcoxon(self):
        g = self.g
        k = 0
        while f"w{k}.d" in g:
            yield g[f"w{k}.d"], float(g[f"w{k}.p"])
            k += 1
