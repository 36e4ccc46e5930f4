"""pytest plugin: run the REFERENCE's own hot-path test files against this
repo's B200 drop-in (SURVEY.md §4.4 conformance run).

Loaded with `-p dare_dropin` (tools/conformance.sh): before any test module
is imported it replaces, in the reference package `dare` (installed under
baseline/_ref, git-ignored), the hot-path entry points with this repo's
CUDA-backed ones -- in the defining modules and in every module that imported
them by value (cli.py:17-18, service.py:28,31, evaluation.py:21,
the package __init__):

  reconstruct_volume (reconstruct.py:166-199)   -> paper_2605_26325_b200.reconstruct_volume
  reslice            (reslice.py:168-187)       -> paper_2605_26325_b200.reslice
  compound / fill_holes / reslice_trilinear (baseline.py:64-155)
                                                -> paper_2605_26325_b200.scalar.*
  ncc / ssim / compare_images / run_comparison / wilcoxon_signed_rank /
  latency_stats / time_reslice / write_report / format_summary
  (evaluation.py:41-355)                        -> paper_2605_26325_b200.evaluation.*

The service module's isinstance test of the volume kind (service.py:32,202)
is widened to accept the drop-in's DirectionalVolume.
reslice_bruteforce stays the reference's numba kernel, so the reference's
oracle-equivalence tests (test_reslice.py:152-179, acceptance criterion 1)
compare the GPU path against the reference's own brute force.  Test files are
the reference's, unmodified; scikit-image (absent from the image) is stubbed
for import only, and the tests that call it (SSIM vs skimage) are deselected
by the runner.
"""
from __future__ import annotations

import os
import sys
import types

PATCHED: dict[str, list[str]] = {}


def _stub_skimage():
    if "skimage" in sys.modules:
        return
    try:
        import skimage  # noqa: F401
        return
    except ImportError:
        pass
    sk = types.ModuleType("skimage")
    metrics = types.ModuleType("skimage.metrics")

    def structural_similarity(*_a, **_k):
        raise RuntimeError("scikit-image is not installed in this image (stub)")

    metrics.structural_similarity = structural_similarity
    sk.metrics = metrics
    sys.modules["skimage"] = sk
    sys.modules["skimage.metrics"] = metrics


def pytest_configure(config):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    _stub_skimage()
    import dare
    import dare.baseline
    import dare.cli
    import dare.evaluation
    import dare.reconstruct
    import dare.reslice
    import dare.service
    import dare.volume

    import paper_2605_26325_b200 as b200
    from paper_2605_26325_b200 import _lib, evaluation, scalar

    if not os.environ.get("DARE_DROPIN_DRYRUN"):  # (collection check without a GPU)
        _lib.init(0)
    repl = {
        "reconstruct_volume": b200.reconstruct_volume,
        "reslice": b200.reslice,
        "compound": scalar.compound,
        "fill_holes": scalar.fill_holes,
        "reslice_trilinear": scalar.reslice_trilinear,
    }
    for name in ("ncc", "ssim", "compare_images", "run_comparison", "wilcoxon_signed_rank", "latency_stats",
                 "time_reslice", "write_report", "format_summary"):
        repl[name] = getattr(evaluation, name)
    for mod in (dare, dare.reconstruct, dare.reslice, dare.baseline, dare.cli, dare.service, dare.evaluation):
        for name, fn in repl.items():
            if hasattr(mod, name):
                setattr(mod, name, fn)
                PATCHED.setdefault(mod.__name__, []).append(name)
    # service.py:32 imported DirectionalVolume by value and tests the volume kind
    # with isinstance (service.py:202): accept the drop-in's volumes as well
    import abc

    from paper_2605_26325_b200.volume import DirectionalVolume as B200Volume

    class AnyDirectionalVolume(abc.ABC):
        pass

    AnyDirectionalVolume.register(dare.volume.DirectionalVolume)
    AnyDirectionalVolume.register(B200Volume)
    dare.service.DirectionalVolume = AnyDirectionalVolume
    PATCHED.setdefault("dare.service", []).append("DirectionalVolume (isinstance accepts the drop-in's)")
    config.addinivalue_line("markers", "dropin: conformance run against the B200 drop-in")


def pytest_report_header(config):
    lines = ["B200 drop-in patched into the reference package `dare`:"]
    for mod, names in sorted(PATCHED.items()):
        lines.append(f"  {mod}: {', '.join(names)}")
    return lines
