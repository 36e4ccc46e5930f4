"""CPU: bench.py harness contract -- `--gpus N` spawns N ranks itself when no
torchrun environment is set, and refuses loudly (exit 2, message on stderr)
when fewer than N CUDA devices are visible; a WORLD_SIZE that disagrees with
--gpus is an error too."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=300)


def test_gpus_more_than_visible_fails_loudly():
    import torch

    n = torch.cuda.device_count()
    r = _run(["--gpus", str(n + 1), "--steps", "1", "--warmup", "3"])
    assert r.returncode == 2
    assert "refusing to run" in r.stderr and f"--gpus {n + 1}" in r.stderr


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--steps", "1"], {"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=3" in r.stderr


@pytest.mark.parametrize("rank", ["1"])
def test_reference_arm_non_zero_rank_exits_quietly(rank):
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1"],
             {"WORLD_SIZE": "2", "RANK": rank, "LOCAL_RANK": rank})
    assert r.returncode == 0 and r.stdout.strip() == ""
