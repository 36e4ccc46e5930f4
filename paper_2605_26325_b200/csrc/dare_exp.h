// Bit-exact restatement of the glibc 2.39 double-precision `exp` (FMA ifunc
// variant, the one x86-64 hosts with FMA/AVX2 dispatch to), usable on host
// and device.
//
// Why: the reference weight `w = math.exp(a)` (pkg/src/dare/_kernels.py:65)
// is numba's math.exp, i.e. the system libm.  CUDA's libdevice exp differs
// from glibc in the last ulp for a small fraction of arguments, which can flip
// a rounded gray level at an exact .5 tie.  Porting glibc's algorithm with the
// same fused/unfused operation pattern (read off the `__exp_fma` disassembly:
// kd = fma(x, InvLn2N, Shift); r = fma(kd, NegLn2hiN, x); r = fma(kd,
// NegLn2loN, r); tmp = fma(r2*r2, fma(r,C5,C4), fma(fma(r,C3,C2), r2, r+tail));
// result = fma(scale, tmp, scale)) makes every weight bit-identical.
// tests/test_exp_port.py pins this against the host libm.
//
// Provenance and licence: the algorithm, the polynomial coefficients and the
// 2^(k/128) table follow glibc's sysdeps/ieee754/dbl-64/e_exp.c and
// e_exp_data.c (glibc 2.39; code contributed by Arm Ltd, "Copyright (C)
// 2018-2024 Free Software Foundation, Inc."), distributed under the GNU
// Lesser General Public License v2.1 or later.  The table here is not copied
// from those sources: tools/gen_exp_table.py regenerates it from the defining
// identity (exp_table.h); the constants are the published ones.  Users
// redistributing this file take the LGPL-2.1+ terms of that algorithm into
// account.
#pragma once
#include <stdint.h>
#include <string.h>
#include "exp_table.h"

#if defined(__CUDACC__)
#define DARE_HD __device__ __forceinline__
#define DARE_FMA(a, b, c) __fma_rn((a), (b), (c))
#define DARE_MUL(a, b) __dmul_rn((a), (b))
#define DARE_ADD(a, b) __dadd_rn((a), (b))
#define DARE_SUB(a, b) __dsub_rn((a), (b))
#else
#include <math.h>
#define DARE_HD static inline
#define DARE_FMA(a, b, c) fma((a), (b), (c))
#define DARE_MUL(a, b) ((a) * (b))
#define DARE_ADD(a, b) ((a) + (b))
#define DARE_SUB(a, b) ((a) - (b))
#endif

#if defined(__CUDACC__)
__device__ const uint64_t dare_exp_tab_dev[256] = DARE_EXP_TABLE_INIT;
#else
static const uint64_t dare_exp_tab_host[256] = DARE_EXP_TABLE_INIT;
#endif

DARE_HD double dare_bits2d(uint64_t u) {
#if defined(__CUDACC__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}

DARE_HD uint64_t dare_d2bits(double d) {
#if defined(__CUDACC__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

DARE_HD uint64_t dare_exp_tab(int i) {
#if defined(__CUDACC__)
  return __ldg((const unsigned long long*)&dare_exp_tab_dev[i]);
#else
  return dare_exp_tab_host[i];
#endif
}

// Slow path for |x| in [512, 1024): the scale's exponent may over/underflow.
DARE_HD double dare_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    double scale = dare_bits2d(sbits);
    return DARE_MUL(DARE_FMA(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;
  double scale = dare_bits2d(sbits);
  double st = DARE_MUL(scale, tmp);  // unfused in glibc's slow path
  double y = DARE_ADD(scale, st);
  if (y < 1.0) {
    double hi = DARE_ADD(y, 1.0);
    double lo = DARE_ADD(DARE_SUB(scale, y), st);
    double t = DARE_ADD(DARE_ADD(DARE_SUB(1.0, hi), y), lo);
    y = DARE_SUB(DARE_ADD(t, hi), 1.0);
    if (y == 0.0) return 0.0;
  }
  return DARE_MUL(y, 0x1p-1022);
}

DARE_HD double dare_exp(double x) {
  const double kInvLn2N = 0x1.71547652b82fep7;
  const double kShift = 0x1.8p52;
  const double kNegLn2hiN = -0x1.62e42fefa0000p-8;
  const double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double kC2 = 0x1.ffffffffffdbdp-2;
  const double kC3 = 0x1.555555555543cp-3;
  const double kC4 = 0x1.55555cf172b91p-5;
  const double kC5 = 0x1.1111167a4d017p-7;

  uint64_t ix = dare_d2bits(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  int special = 0;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return DARE_ADD(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                       // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return DARE_ADD(1.0, x);
      return (ix >> 63) ? 0.0 : dare_bits2d(0x7ff0000000000000ull);
    }
    special = 1;
  }
  double kd = DARE_FMA(x, kInvLn2N, kShift);
  uint64_t ki = dare_d2bits(kd);
  kd = DARE_SUB(kd, kShift);
  double r = DARE_FMA(kd, kNegLn2hiN, x);
  r = DARE_FMA(kd, kNegLn2loN, r);
  int idx = 2 * (int)(ki & 127u);
  uint64_t top = ki << 45;
  double tail = dare_bits2d(dare_exp_tab(idx));
  uint64_t sbits = dare_exp_tab(idx + 1) + top;
  double p23 = DARE_FMA(r, kC3, kC2);
  double rt = DARE_ADD(r, tail);
  double r2 = DARE_MUL(r, r);
  double p45 = DARE_FMA(r, kC5, kC4);
  double acc = DARE_FMA(p23, r2, rt);
  double r4 = DARE_MUL(r2, r2);
  double tmp = DARE_FMA(r4, p45, acc);
  if (special) return dare_exp_special(tmp, sbits, ki);
  double scale = dare_bits2d(sbits);
  return DARE_FMA(scale, tmp, scale);
}
