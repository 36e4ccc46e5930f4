"""The device `exp` (csrc/dare_exp.h) is a restatement of glibc 2.39's
FMA-variant exp.  Compile the same header for the host and compare it
bit-for-bit with the system libm (what numba's math.exp calls) and with the
reference's recorded values.  CPU only."""
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HARNESS = r"""
#include <stdio.h>
#include <stdlib.h>
#include "dare_exp.h"
int main(int argc, char** argv) {
  long n = atol(argv[1]);
  double* x = (double*)malloc(sizeof(double) * n);
  if (fread(x, sizeof(double), n, stdin) != (size_t)n) return 2;
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    double a = exp(x[i]), b = dare_exp(x[i]);
    if (dare_d2bits(a) != dare_d2bits(b) && !(a != a && b != b)) ++bad;
    fwrite(&b, sizeof(double), 1, stdout);
  }
  fprintf(stderr, "%ld\n", bad);
  return 0;
}
"""


def _run(tmp_path, x):
    src = tmp_path / "h.c"
    src.write_text(HARNESS)
    exe = tmp_path / "h"
    gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([gcc, "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_2605_26325_b200", "csrc"),
                    str(src), "-o", str(exe), "-lm"], check=True)
    p = subprocess.run([str(exe), str(len(x))], input=np.ascontiguousarray(x, np.float64).tobytes(),
                       capture_output=True, check=True)
    return np.frombuffer(p.stdout, dtype=np.float64), int(p.stderr.decode().strip())


def test_exp_port_bit_exact_vs_libm(tmp_path, rng):
    x = np.concatenate([
        -rng.uniform(0, 60, 1_000_000),          # weight arguments
        -rng.uniform(0, 1e-6, 50_000),
        rng.uniform(-1100, 1100, 200_000),        # over/underflow paths
        rng.standard_normal(200_000).view(np.uint64).astype(np.uint64).view(np.float64),
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 709.78, -745.13, -708.4, 1e-320]),
    ])
    _, bad = _run(tmp_path, x)
    assert bad == 0


def test_exp_port_matches_reference_values(tmp_path, golden):
    y, _ = _run(tmp_path, golden["exp.x"])
    np.testing.assert_array_equal(y.view(np.uint64), golden["exp.y"].view(np.uint64))
