/*
 * dare_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot-path arithmetic
 * (arxiv/paper_2605_26325, package `dare`, pkg/src/dare/), used as the parity
 * checker for the CUDA path and as the CPU baseline arm of bench.py.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library; the product path never does.
 *
 * Numerics follow the reference exactly: f64 throughout, every operation
 * separately rounded (built with -ffp-contract=off; numba does not contract
 * either), glibc `exp`/`floor`/`sqrt` from the system libm (numba's math.exp
 * resolves to the same libm).  Evaluation order mirrors the Python source
 * expression by expression.  Pinned against the reference's own outputs by
 * tests/test_oracle_golden.py (fixtures from tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define COVERAGE_MIN_WEIGHT 1e-12 /* _kernels.py:20 */
#define CELL_RANGE_GUARD 1e-9     /* _kernels.py:26 */

/* floor(x) clamped into [lo-1, hi+1] before the int conversion, so absurd
 * coordinates cannot overflow; only emptiness of the range matters there. */
static int64_t clamp_floor(double x, int64_t n) {
  double f = floor(x);
  if (!(f > -1.0)) return -1; /* also NaN */
  if (f > (double)n) return n;
  return (int64_t)f;
}

/*
 * Pixel -> world -> owning cell for one frame.
 * reconstruct.py:152-163 (frame_world_positions): P = (u*px)*R[:,0] + (v*py)*R[:,1] + t
 * reconstruct.py:188-196 + volume.py:223-238 (insert_batch/_voxel_indices):
 *   p32 = f32(P); idx = floor((f64(p32) - origin) / voxel); keep iff 0<=idx<dims.
 * c0 = R[:,0], c1 = R[:,1].  lin[k] = linear cell or -1 when out of bounds.
 */
void oracle_frame_cells(int32_t H, int32_t W, double px, double py,
                        const double* c0, const double* c1, const double* t,
                        const double* origin, double voxel, const int64_t* dims,
                        int64_t* lin, float* pos) {
  for (int32_t v = 0; v < H; ++v) {
    double V = (double)v * py;
    for (int32_t u = 0; u < W; ++u) {
      double U = (double)u * px;
      int64_t k = (int64_t)v * W + u;
      int ok = 1;
      int64_t idx[3];
      for (int a = 0; a < 3; ++a) {
        double P = (U * c0[a] + V * c1[a]) + t[a];
        float p32 = (float)P;
        pos[3 * k + a] = p32;
        double f = floor(((double)p32 - origin[a]) / voxel);
        if (!(f >= 0.0 && f < (double)dims[a])) ok = 0;
        else idx[a] = (int64_t)f;
      }
      lin[k] = ok ? (idx[0] * dims[1] + idx[1]) * dims[2] + idx[2] : -1;
    }
  }
}

/*
 * volume.py:240-269 (seal): stable sort by linear cell, counts, exclusive
 * cumsum.  `lin` holds the kept samples in insertion order.  Outputs
 * counts/starts (ncells) and `order` (n) = source index of each stored slot.
 */
void oracle_seal(int64_t n, const int64_t* lin, int64_t ncells,
                 int64_t* counts, int64_t* starts, int64_t* order) {
  memset(counts, 0, sizeof(int64_t) * ncells);
  for (int64_t i = 0; i < n; ++i) counts[lin[i]]++;
  int64_t run = 0;
  for (int64_t c = 0; c < ncells; ++c) {
    starts[c] = run;
    run += counts[c];
  }
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (ncells ? ncells : 1));
  memcpy(cursor, starts, sizeof(int64_t) * ncells);
  for (int64_t i = 0; i < n; ++i) order[cursor[lin[i]]++] = i;
  free(cursor);
}

/* _kernels.py:29-68 (_accumulate_run). */
static inline void accumulate_run(int64_t i0, int64_t i1, double wx, double wy, double wz,
                                  double radius, double xrx, double xry, double xrz,
                                  double nrx, double nry, double nrz, const float* positions,
                                  const float* orientations, const uint8_t* intensities,
                                  double cos_nt, double cos_it, double kn, double ki, double kd,
                                  double* wsum, double* iwsum) {
  for (int64_t i = i0; i < i1; ++i) {
    double dx = (double)positions[3 * i + 0] - wx;
    if (dx < -radius || dx > radius) continue;
    double dy = (double)positions[3 * i + 1] - wy;
    if (dy < -radius || dy > radius) continue;
    double dz = (double)positions[3 * i + 2] - wz;
    if (dz < -radius || dz > radius) continue;
    double qw = orientations[4 * i + 0], qx = orientations[4 * i + 1];
    double qy = orientations[4 * i + 2], qz = orientations[4 * i + 3];
    double nsx = 2.0 * (qx * qz + qw * qy);
    double nsy = 2.0 * (qy * qz - qw * qx);
    double nsz = 1.0 - 2.0 * (qx * qx + qy * qy);
    double dn = (nsx * nrx + nsy * nry) + nsz * nrz;
    if (dn < cos_nt) continue;
    double xsx = 1.0 - 2.0 * (qy * qy + qz * qz);
    double xsy = 2.0 * (qx * qy + qw * qz);
    double xsz = 2.0 * (qx * qz - qw * qy);
    double di = fabs((xsx * xrx + xsy * xry) + xsz * xrz);
    if (di < cos_it) continue;
    double dist = sqrt((dx * dx + dy * dy) + dz * dz);
    double w = exp((kn * (dn - 1.0) + ki * (di - 1.0)) - (kd * dist) / radius);
    *wsum += w;
    *iwsum += w * (double)intensities[i];
  }
}

/* _kernels.py:71-81 (_finalize_pixel). */
static inline void finalize_pixel(double wsum, double iwsum, int32_t unassigned,
                                  uint8_t* out, uint8_t* cov) {
  if (wsum >= COVERAGE_MIN_WEIGHT) {
    double val = iwsum / wsum;
    double f = floor(val + 0.5);
    int64_t iv = (f < 0.0) ? 0 : (f > 255.0 ? 255 : (int64_t)f);
    *out = (uint8_t)iv;
    *cov = 1;
  } else {
    *out = (uint8_t)unassigned;
    *cov = 0;
  }
}

/* params: tx,ty,tz, r00,r01,r02, r10,r11,r12, r20,r21,r22, pitch_x, pitch_y
 * (reslice.py:135-148 _plane_params).  cfg: radius, cos_nt, cos_it, kn, ki, kd. */

/* _kernels.py:84-139 (reslice_rows_grid), rows [0, H), parallel over rows
 * (reslice.py:151-165 splits rows across a pool; results are chunking-free). */
void oracle_reslice_grid(uint8_t* out, uint8_t* cov, int32_t H, int32_t W, const double* p,
                         const double* origin, double voxel, const int64_t* dims,
                         const int64_t* cell_starts, const int64_t* cell_counts,
                         const float* positions, const float* orientations,
                         const uint8_t* intensities, const double* cfg, int32_t unassigned) {
  const double tx = p[0], ty = p[1], tz = p[2];
  const double r00 = p[3], r01 = p[4], r02 = p[5], r10 = p[6], r11 = p[7], r12 = p[8];
  const double r20 = p[9], r21 = p[10], r22 = p[11], pitch_x = p[12], pitch_y = p[13];
  const double radius = cfg[0], cos_nt = cfg[1], cos_it = cfg[2];
  const double kn = cfg[3], ki = cfg[4], kd = cfg[5];
  const double ox = origin[0], oy = origin[1], oz = origin[2];
  const int64_t nx = dims[0], ny = dims[1], nz = dims[2];
  const double inv_v = 1.0 / voxel;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t v = 0; v < H; ++v) {
    for (int32_t u = 0; u < W; ++u) {
      double du = (double)u * pitch_x, dv = (double)v * pitch_y;
      double wx = (tx + du * r00) + dv * r01;
      double wy = (ty + du * r10) + dv * r11;
      double wz = (tz + du * r20) + dv * r21;
      int64_t lox = clamp_floor(((wx - radius) - ox) * inv_v - CELL_RANGE_GUARD, nx);
      int64_t hix = clamp_floor(((wx + radius) - ox) * inv_v + CELL_RANGE_GUARD, nx);
      int64_t loy = clamp_floor(((wy - radius) - oy) * inv_v - CELL_RANGE_GUARD, ny);
      int64_t hiy = clamp_floor(((wy + radius) - oy) * inv_v + CELL_RANGE_GUARD, ny);
      int64_t loz = clamp_floor(((wz - radius) - oz) * inv_v - CELL_RANGE_GUARD, nz);
      int64_t hiz = clamp_floor(((wz + radius) - oz) * inv_v + CELL_RANGE_GUARD, nz);
      if (lox < 0) lox = 0;
      if (loy < 0) loy = 0;
      if (loz < 0) loz = 0;
      if (hix >= nx) hix = nx - 1;
      if (hiy >= ny) hiy = ny - 1;
      if (hiz >= nz) hiz = nz - 1;
      double wsum = 0.0, iwsum = 0.0;
      for (int64_t cx = lox; cx <= hix; ++cx)
        for (int64_t cy = loy; cy <= hiy; ++cy) {
          int64_t base = (cx * ny + cy) * nz;
          for (int64_t cz = loz; cz <= hiz; ++cz) {
            int64_t lin = base + cz;
            int64_t start = cell_starts[lin], count = cell_counts[lin];
            if (count > 0)
              accumulate_run(start, start + count, wx, wy, wz, radius, r00, r10, r20, r02, r12,
                             r22, positions, orientations, intensities, cos_nt, cos_it, kn, ki,
                             kd, &wsum, &iwsum);
          }
        }
      int64_t k = (int64_t)v * W + u;
      finalize_pixel(wsum, iwsum, unassigned, out + k, cov + k);
    }
  }
}

/* _kernels.py:142-167 (reslice_rows_bruteforce): every sample for every pixel. */
void oracle_reslice_bruteforce(uint8_t* out, uint8_t* cov, int32_t H, int32_t W, const double* p,
                               int64_t n, const float* positions, const float* orientations,
                               const uint8_t* intensities, const double* cfg, int32_t unassigned) {
  const double tx = p[0], ty = p[1], tz = p[2];
  const double r00 = p[3], r01 = p[4], r02 = p[5], r10 = p[6], r11 = p[7], r12 = p[8];
  const double r20 = p[9], r21 = p[10], r22 = p[11], pitch_x = p[12], pitch_y = p[13];
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t v = 0; v < H; ++v)
    for (int32_t u = 0; u < W; ++u) {
      double du = (double)u * pitch_x, dv = (double)v * pitch_y;
      double wx = (tx + du * r00) + dv * r01;
      double wy = (ty + du * r10) + dv * r11;
      double wz = (tz + du * r20) + dv * r21;
      double wsum = 0.0, iwsum = 0.0;
      accumulate_run(0, n, wx, wy, wz, cfg[0], r00, r10, r20, r02, r12, r22, positions,
                     orientations, intensities, cfg[1], cfg[2], cfg[3], cfg[4], cfg[5], &wsum,
                     &iwsum);
      int64_t k = (int64_t)v * W + u;
      finalize_pixel(wsum, iwsum, unassigned, out + k, cov + k);
    }
}

/* _kernels.py:170-229 (trilinear_rows) + baseline.py:151-153 rounding.
 * values f32 (promoted exactly to f64, as baseline.py:148 does), flags u8 (occupied = flag != 0). */
void oracle_trilinear(uint8_t* out, uint8_t* cov, double* out_val, int32_t H, int32_t W,
                      const double* p, const double* origin, double voxel, const int64_t* dims,
                      const float* values, const uint8_t* flags) {
  const double tx = p[0], ty = p[1], tz = p[2];
  const double r00 = p[3], r01 = p[4], r10 = p[6], r11 = p[7], r20 = p[9], r21 = p[10];
  const double pitch_x = p[12], pitch_y = p[13];
  const int64_t nx = dims[0], ny = dims[1], nz = dims[2];
  const double inv_v = 1.0 / voxel;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t v = 0; v < H; ++v)
    for (int32_t u = 0; u < W; ++u) {
      double du = (double)u * pitch_x, dv = (double)v * pitch_y;
      double wx = (tx + du * r00) + dv * r01;
      double wy = (ty + du * r10) + dv * r11;
      double wz = (tz + du * r20) + dv * r21;
      double g[3] = {(wx - origin[0]) * inv_v - 0.5, (wy - origin[1]) * inv_v - 0.5,
                     (wz - origin[2]) * inv_v - 0.5};
      int64_t i[3];
      double f[3];
      for (int a = 0; a < 3; ++a) {
        double fl = floor(g[a]);
        /* far-away points: every corner index is out of range either way */
        double flc = fl < -2.0 ? -2.0 : (fl > (double)dims[a] + 1.0 ? (double)dims[a] + 1.0 : fl);
        i[a] = (int64_t)flc;
        f[a] = g[a] - fl;
      }
      double wsum = 0.0, vsum = 0.0;
      for (int cx = 0; cx < 2; ++cx) {
        int64_t jx = i[0] + cx;
        if (jx < 0 || jx >= nx) continue;
        double wxc = cx == 1 ? f[0] : 1.0 - f[0];
        for (int cy = 0; cy < 2; ++cy) {
          int64_t jy = i[1] + cy;
          if (jy < 0 || jy >= ny) continue;
          double wyc = cy == 1 ? f[1] : 1.0 - f[1];
          for (int cz = 0; cz < 2; ++cz) {
            int64_t jz = i[2] + cz;
            if (jz < 0 || jz >= nz) continue;
            int64_t lin = (jx * ny + jy) * nz + jz;
            if (flags[lin] != 0) {
              double wc = (wxc * wyc) * (cz == 1 ? f[2] : 1.0 - f[2]);
              wsum += wc;
              vsum += wc * (double)values[lin];
            }
          }
        }
      }
      int64_t k = (int64_t)v * W + u;
      if (wsum >= COVERAGE_MIN_WEIGHT) {
        double val = vsum / wsum;
        double r = floor(val + 0.5);
        if (r < 0.0) r = 0.0;
        if (r > 255.0) r = 255.0;
        if (out_val) out_val[k] = val;
        out[k] = (uint8_t)r;
        cov[k] = 1;
      } else {
        if (out_val) out_val[k] = 0.0;
        out[k] = 0;
        cov[k] = 0;
      }
    }
}

/* baseline.py:82-92: one frame's contribution to the integer sums/counts
 * (same cell mapping as oracle_frame_cells; out-of-bounds dropped silently). */
void oracle_compound_frame(int32_t H, int32_t W, double px, double py, const double* c0,
                           const double* c1, const double* t, const double* origin, double voxel,
                           const int64_t* dims, const uint8_t* pixels, const uint8_t* mask,
                           int64_t* sums, int64_t* counts) {
  int64_t n = (int64_t)H * W;
  int64_t* lin = (int64_t*)malloc(sizeof(int64_t) * n);
  float* pos = (float*)malloc(sizeof(float) * 3 * n);
  oracle_frame_cells(H, W, px, py, c0, c1, t, origin, voxel, dims, lin, pos);
  for (int64_t k = 0; k < n; ++k) {
    if (mask && !mask[k]) continue;
    if (lin[k] < 0) continue;
    sums[lin[k]] += pixels[k];
    counts[lin[k]] += 1;
  }
  free(lin);
  free(pos);
}

/* baseline.py:93-96: values = f32(f64(sum) / f64(count)) where observed. */
void oracle_compound_finalize(int64_t ncells, const int64_t* sums, const int64_t* counts,
                              float* values, uint8_t* flags) {
  for (int64_t c = 0; c < ncells; ++c) {
    if (counts[c] > 0) {
      values[c] = (float)((double)sums[c] / (double)counts[c]);
      flags[c] = 1;
    } else {
      values[c] = 0.0f;
      flags[c] = 0;
    }
  }
}

/*
 * baseline.py:100-127 (fill_holes): Jacobi passes over the 26-neighbourhood.
 * The neighbour sum runs over offsets in C order (x outermost, z innermost,
 * centre skipped), the order scipy.ndimage.convolve visits a symmetric 3x3x3
 * footprint; unknown / out-of-grid neighbours contribute 0.  `v` is the f64
 * working grid (in/out), flags in/out.  Returns the number of passes that
 * filled at least one voxel.
 */
int32_t oracle_fill_holes(double* v, uint8_t* flags, const int64_t* dims, int32_t max_passes) {
  const int64_t nx = dims[0], ny = dims[1], nz = dims[2], n = nx * ny * nz;
  uint8_t* known = (uint8_t*)malloc(n ? n : 1);
  double* newv = (double*)malloc(sizeof(double) * (n ? n : 1));
  uint8_t* fill = (uint8_t*)malloc(n ? n : 1);
  int32_t passes = 0;
  for (int32_t pass = 0; pass < max_passes; ++pass) {
    int64_t nknown = 0;
    for (int64_t c = 0; c < n; ++c) {
      known[c] = flags[c] != 0;
      nknown += known[c];
    }
    if (nknown == n) break;
    int64_t nfill = 0;
#pragma omp parallel for reduction(+ : nfill) schedule(static)
    for (int64_t x = 0; x < nx; ++x)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t z = 0; z < nz; ++z) {
          int64_t c = (x * ny + y) * nz + z;
          fill[c] = 0;
          if (known[c]) continue;
          double s = 0.0, cnt = 0.0;
          for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
              for (int dz = -1; dz <= 1; ++dz) {
                if (dx == 0 && dy == 0 && dz == 0) continue;
                int64_t X = x + dx, Y = y + dy, Z = z + dz;
                double val = 0.0, k = 0.0;
                if (X >= 0 && X < nx && Y >= 0 && Y < ny && Z >= 0 && Z < nz) {
                  int64_t q = (X * ny + Y) * nz + Z;
                  if (known[q]) {
                    val = v[q];
                    k = 1.0;
                  }
                }
                s += val;
                cnt += k;
              }
          if (cnt > 0.0) {
            newv[c] = s / cnt;
            fill[c] = 1;
            nfill++;
          }
        }
    if (nfill == 0) break;
    for (int64_t c = 0; c < n; ++c)
      if (fill[c]) {
        v[c] = newv[c];
        flags[c] = 2;
      }
    passes++;
  }
  free(known);
  free(newv);
  free(fill);
  return passes;
}

/* host libm exp, exposed so tests can pin the device port against it */
void oracle_exp(int64_t n, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = exp(x[i]);
}
