/*
 * C-only client of the drop-in boundary (include/dare_b200.h): no Python, no
 * torch.  Seals a random sample set on the device (dare_volume_seal, the
 * VolumeBuilder.seal seam, volume.py:240-269), downloads it (reference layout)
 * and reslices random planes (dare_reslice, the reslice_rows_grid seam,
 * _kernels.py:84-139), checking everything bit-for-bit against the CPU oracle
 * (oracle/dare_oracle.c, test infrastructure) linked into the same program.
 *
 *   gcc -O2 -I include tests/c_abi/abi_parity.c -L paper_2605_26325_b200 -ldare_b200 \
 *       -L oracle -loracle -lm -Wl,-rpath,$PWD/paper_2605_26325_b200:$PWD/oracle -o abi_parity
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dare_b200.h"

/* oracle entry points (oracle/dare_oracle.c) */
void oracle_seal(int64_t n, const int64_t* lin, int64_t ncells, int64_t* counts, int64_t* starts, int64_t* order);
void oracle_reslice_grid(uint8_t* out, uint8_t* cov, int32_t H, int32_t W, const double* p, const double* origin,
                         double voxel, const int64_t* dims, const int64_t* cell_starts, const int64_t* cell_counts,
                         const float* positions, const float* orientations, const uint8_t* intensities,
                         const double* cfg, int32_t unassigned);

static uint64_t rs = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* xorshift64*, uniform [0,1) */
  rs ^= rs >> 12;
  rs ^= rs << 25;
  rs ^= rs >> 27;
  return (double)((rs * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

#define CHECK(call)                                                             \
  do {                                                                          \
    int rc_ = (call);                                                           \
    if (rc_ != DARE_OK) {                                                       \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, dare_last_error());   \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main(void) {
  const int64_t n = 60000, dims[3] = {24, 20, 28};
  const double origin[3] = {-0.5, 0.25, 1.0}, voxel = 0.25;
  const int64_t ncells = dims[0] * dims[1] * dims[2];
  float* pos = malloc(sizeof(float) * 3 * n);
  float* quat = malloc(sizeof(float) * 4 * n);
  uint8_t* inten = malloc(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) pos[3 * i + a] = (float)(origin[a] + urand() * dims[a] * voxel);
    /* a few orientations (frames), canonical w >= 0 */
    const double ang = 0.3 * (double)(i % 7), c = cos(0.5 * ang), s = sin(0.5 * ang);
    quat[4 * i + 0] = (float)c;
    quat[4 * i + 1] = (float)s;
    quat[4 * i + 2] = 0.0f;
    quat[4 * i + 3] = 0.0f;
    inten[i] = (uint8_t)(urand() * 256.0);
  }
  CHECK(dare_set_device(0));
  CHECK(dare_init(0));
  dare_volume_t vol = NULL;
  CHECK(dare_volume_seal(origin, voxel, dims, n, pos, quat, inten, &vol));
  dare_volume_info info;
  CHECK(dare_volume_get_info(vol, &info));

  /* oracle: voxel index (volume.py:209), stable seal */
  int64_t* lin = malloc(sizeof(int64_t) * n);
  int64_t kept = 0;
  int64_t* src = malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t idx[3];
    int ok = 1;
    for (int a = 0; a < 3; ++a) {
      const double f = floor(((double)pos[3 * i + a] - origin[a]) / voxel);
      ok = ok && f >= 0.0 && f < (double)dims[a];
      idx[a] = ok ? (int64_t)f : 0;
    }
    if (ok) {
      lin[kept] = (idx[0] * dims[1] + idx[1]) * dims[2] + idx[2];
      src[kept++] = i;
    }
  }
  int64_t *counts = malloc(sizeof(int64_t) * ncells), *starts = malloc(sizeof(int64_t) * ncells);
  int64_t* order = malloc(sizeof(int64_t) * kept);
  oracle_seal(kept, lin, ncells, counts, starts, order);
  float *rpos = malloc(sizeof(float) * 3 * kept), *rquat = malloc(sizeof(float) * 4 * kept);
  uint8_t* rint = malloc(kept);
  for (int64_t j = 0; j < kept; ++j) {
    const int64_t i = src[order[j]];
    memcpy(rpos + 3 * j, pos + 3 * i, 12);
    memcpy(rquat + 4 * j, quat + 4 * i, 16);
    rint[j] = inten[i];
  }
  if (info.n_samples != kept) {
    fprintf(stderr, "sample count %lld vs oracle %lld\n", (long long)info.n_samples, (long long)kept);
    return 1;
  }
  int64_t *dstarts = malloc(sizeof(int64_t) * ncells), *dcounts = malloc(sizeof(int64_t) * ncells);
  float *dpos = malloc(sizeof(float) * 3 * kept), *dquat = malloc(sizeof(float) * 4 * kept);
  uint8_t* dint = malloc(kept);
  CHECK(dare_volume_download(vol, dstarts, dcounts, dpos, dquat, dint));
  if (memcmp(dstarts, starts, sizeof(int64_t) * ncells) || memcmp(dcounts, counts, sizeof(int64_t) * ncells) ||
      memcmp(dpos, rpos, 12 * kept) || memcmp(dquat, rquat, 16 * kept) || memcmp(dint, rint, kept)) {
    fprintf(stderr, "sealed volume differs from the oracle\n");
    return 1;
  }

  /* reslices: planes oriented like one of the sample frames (rotation about x,
     perturbed by a few degrees about a random axis) so the direction gate passes */
  const int W = 48, H = 40, P = 6;
  double* params = malloc(sizeof(double) * 14 * P);
  for (int p = 0; p < P; ++p) {
    const double ang = 0.3 * (double)(p % 7);
    double q[4] = {cos(0.5 * ang), sin(0.5 * ang), 0.0, 0.0};
    double e[3] = {urand() - 0.5, urand() - 0.5, urand() - 0.5};
    const double ne = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]), de = 0.08 * urand();
    const double dq[4] = {cos(0.5 * de), sin(0.5 * de) * e[0] / ne, sin(0.5 * de) * e[1] / ne,
                          sin(0.5 * de) * e[2] / ne};
    const double r0 = dq[0] * q[0] - dq[1] * q[1] - dq[2] * q[2] - dq[3] * q[3];
    const double r1 = dq[0] * q[1] + dq[1] * q[0] + dq[2] * q[3] - dq[3] * q[2];
    const double r2 = dq[0] * q[2] - dq[1] * q[3] + dq[2] * q[0] + dq[3] * q[1];
    const double r3 = dq[0] * q[3] + dq[1] * q[2] - dq[2] * q[1] + dq[3] * q[0];
    const double w = r0, x = r1, y = r2, z = r3;
    double* pp = params + 14 * p;
    pp[0] = origin[0] + 1.0 + 2.0 * urand();
    pp[1] = origin[1] + 1.0 + 1.0 * urand();
    pp[2] = origin[2] + 1.0 + 2.0 * urand();
    pp[3] = 1 - 2 * (y * y + z * z); pp[4] = 2 * (x * y - w * z); pp[5] = 2 * (x * z + w * y);
    pp[6] = 2 * (x * y + w * z); pp[7] = 1 - 2 * (x * x + z * z); pp[8] = 2 * (y * z - w * x);
    pp[9] = 2 * (x * z - w * y); pp[10] = 2 * (y * z + w * x); pp[11] = 1 - 2 * (x * x + y * y);
    pp[12] = 0.05; pp[13] = 0.04;
  }
  dare_reslice_cfg cfg = {voxel, cos(25.0 * M_PI / 180.0), cos(15.0 * M_PI / 180.0), 10.0, 5.0, 2.0, 7, 0, 0, 0};
  const double ocfg[6] = {cfg.radius, cfg.cos_normal, cfg.cos_inplane, cfg.k_normal, cfg.k_inplane, cfg.k_dist};
  uint8_t *px = malloc((size_t)P * W * H), *cv = malloc((size_t)P * W * H);
  uint8_t *opx = malloc((size_t)W * H), *ocv = malloc((size_t)W * H);
  for (int exact = 0; exact <= 1; ++exact) {
    cfg.exact = exact;
    CHECK(dare_reslice(vol, P, params, W, H, &cfg, px, cv));
    int covered = 0;
    for (int p = 0; p < P; ++p) {
      oracle_reslice_grid(opx, ocv, H, W, params + 14 * p, origin, voxel, dims, starts, counts, rpos, rquat, rint,
                          ocfg, cfg.unassigned);
      if (memcmp(opx, px + (size_t)p * W * H, (size_t)W * H) || memcmp(ocv, cv + (size_t)p * W * H, (size_t)W * H)) {
        fprintf(stderr, "reslice pose %d (exact=%d) differs from the oracle\n", p, exact);
        return 1;
      }
      for (int k = 0; k < W * H; ++k) covered += ocv[k];
    }
    if (covered < P * W * H / 4) {
      fprintf(stderr, "only %d covered pixels: degenerate test\n", covered);
      return 1;
    }
  }
  CHECK(dare_volume_destroy(vol));
  CHECK(dare_trim(0));
  printf("c-abi ok: sealed %lld samples, %d reslices x 2 modes bit-exact vs the oracle\n", (long long)kept, P);
  return 0;
}
