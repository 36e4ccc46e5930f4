"""The drop-in boundary used from plain C (tests/c_abi/abi_parity.c): the
header compiles as strict C11, the program links against libdare_b200.so and
the oracle library only (no Python, no torch in the process), and on a GPU it
seals + reslices bit-exactly against the oracle linked into the same binary."""
import os
import subprocess

import pytest

from oracle import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_26325_b200")
ORC = os.path.join(ROOT, "oracle")


def _build(tmp_path):
    oracle.load()  # builds liboracle.so if missing
    exe = str(tmp_path / "abi_parity")
    cmd = ["gcc", "-std=c11", "-D_DEFAULT_SOURCE", "-O2", "-Wall", "-Wextra", "-Werror", "-I",
           os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c_abi", "abi_parity.c"),
           "-L", PKG, "-ldare_b200", "-L", ORC, "-loracle", "-lm", f"-Wl,-rpath,{PKG}:{ORC}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_builds_against_header(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run(["ldd", exe], capture_output=True, text=True)
    assert "libdare_b200.so" in r.stdout and "libtorch" not in r.stdout and "libpython" not in r.stdout


@pytest.mark.gpu
def test_c_program_seal_and_reslice_bit_exact(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c-abi ok" in r.stdout
