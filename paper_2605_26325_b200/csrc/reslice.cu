// Direction-aware reslicing (batched poses per launch).
//
// Reference: reslice.py:168-187 (reslice) -> _kernels.reslice_rows_grid
// (_kernels.py:84-139) -> _accumulate_run (29-68) -> _finalize_pixel (71-81).
//
// Per pixel the reference walks the clamped cell range x -> y -> z ascending
// and, per cell, its run in storage order, accumulating wsum / iwsum in FP64.
// That order is kept exactly (thread per pixel, same walk), so every pixel is
// bit-identical.  What changes is where the work goes:
//   * orientation gates and the orientation exponent
//       A = k_n (d_n - 1) + k_i (d_i - 1)                  (_kernels.py:47-65)
//     depend only on (pose, sample quaternion); they are evaluated once per
//     (pose, distinct orientation) by gate_k, bit-identically, and the walk
//     reads one double per visit instead of redoing 30 FP64 ops;
//   * because rejection is a pure filter, the gate is tested before the cube
//     (same survivors, same order);
//   * for fixed (cx, cy) the cells loz..hiz are adjacent in the CSR, so their
//     runs form ONE contiguous sample range [off[base+loz], off[base+hiz+1]);
//   * (k_d * dist) / r uses an exact reciprocal multiply when r is a power of
//     two, and is skipped entirely when k_d == 0 (the term is exactly +0.0);
//   * exp is the bit-exact glibc port (dare_exp.h).
#include <math_constants.h>

#include "dare_exp.h"
#include <cub/device/device_radix_sort.cuh>

#include "volume.cuh"

namespace dare {

constexpr double kCoverageMinWeight = 1e-12;  // _kernels.py:20
constexpr double kCellRangeGuard = 1e-9;      // _kernels.py:26

struct ResliceArgs {
  const uint32_t* offsets;
  const uint4* records;
  const double* params;  // P x 14
  const double* gate;    // P x n_orient (A, or +inf when rejected)
  int64_t n_orient;
  double origin[3];
  double voxel;
  int64_t dims[3];
  double radius, inv_radius, kd;
  int dist_mode;  // 0: divide, 1: exact reciprocal, 2: k_d == 0
  int unassigned;
  int W, H, P;
  int tiles_x;
  int brute;           // 1: scan every sample (reslice_rows_bruteforce)
  const int* order;    // launch slot -> pose (spatially sorted batch), or null
  int pose_major;      // lanes = one pixel of 32 consecutive poses (coherent batches)
  uint32_t n_samples;
};

// gate table: one thread per (orientation, pose)
__global__ void gate_k(const float4* __restrict__ orient, int64_t n_orient,
                       const double* __restrict__ params, int P, dare_reslice_cfg cfg,
                       double* gate) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int p = blockIdx.y;
  if (o >= n_orient || p >= P) return;
  const double* pp = params + (size_t)p * 14;
  const double xrx = pp[3], xry = pp[6], xrz = pp[9];   // R[:,0]
  const double nrx = pp[5], nry = pp[8], nrz = pp[11];  // R[:,2]
  float4 q4 = orient[o];
  double qw = q4.x, qx = q4.y, qy = q4.z, qz = q4.w;
  double nsx = 2.0 * (qx * qz + qw * qy);
  double nsy = 2.0 * (qy * qz - qw * qx);
  double nsz = 1.0 - 2.0 * (qx * qx + qy * qy);
  double dn = (nsx * nrx + nsy * nry) + nsz * nrz;
  double A = CUDART_INF;
  if (!(dn < cfg.cos_normal)) {
    double xsx = 1.0 - 2.0 * (qy * qy + qz * qz);
    double xsy = 2.0 * (qx * qy + qw * qz);
    double xsz = 2.0 * (qx * qz - qw * qy);
    double di = fabs((xsx * xrx + xsy * xry) + xsz * xrz);
    if (!(di < cfg.cos_inplane)) A = cfg.k_normal * (dn - 1.0) + cfg.k_inplane * (di - 1.0);
  }
  gate[(size_t)p * n_orient + o] = A;
}

__device__ __forceinline__ void cell_range(double w, double r, double o, double inv_v, int64_t n,
                                           int64_t& lo, int64_t& hi) {
  double l = floor(((w - r) - o) * inv_v - kCellRangeGuard);
  double h = floor(((w + r) - o) * inv_v + kCellRangeGuard);
  if (!(l <= h)) {  // empty or NaN
    lo = 1;
    hi = 0;
    return;
  }
  lo = l < 0.0 ? 0 : (l > (double)n ? n : (int64_t)l);
  hi = h >= (double)n ? n - 1 : (h < -1.0 ? -1 : (int64_t)h);
}

// Exact f32 form of the reference's closed cube test on one axis:
// keep  <=>  -r <= fl64(f64(p) - w) <= r.  fl64(p - w) is monotone in p, so the
// kept f32 values form an interval [lo, hi]; find its ends by stepping ulps
// from the rounded guesses (<= 2 steps in practice).
__device__ __forceinline__ float keep_hi(double w, double r) {
  float p = __double2float_rn(w + r);
  for (int i = 0; i < 4 && !((double)p - w <= r); ++i) p = nextafterf(p, -CUDART_INF_F);
  for (int i = 0; i < 4; ++i) {
    float q = nextafterf(p, CUDART_INF_F);
    if ((double)q - w <= r) p = q;
    else break;
  }
  return p;
}

__device__ __forceinline__ float keep_lo(double w, double r) {
  float p = __double2float_rn(w - r);
  for (int i = 0; i < 4 && !((double)p - w >= -r); ++i) p = nextafterf(p, CUDART_INF_F);
  for (int i = 0; i < 4; ++i) {
    float q = nextafterf(p, -CUDART_INF_F);
    if ((double)q - w >= -r) p = q;
    else break;
  }
  return p;
}

constexpr int kGateSmem = 512;  // orientation table entries staged in shared memory
constexpr int kSmemBytes = (int)(sizeof(double) * kGateSmem);

// 256 threads = one 16x16 pixel tile; each warp covers 8x4 pixels; thread per
// pixel, walking its cell columns in the reference order.  Per-visit work is
// an exact f32 interval test (keep_lo/keep_hi) plus, when this pose rejects
// any orientation, the gate lookup; survivors get the FP64 weight.  To keep
// the FP64 path converged, the warp advances in rounds: every lane scans
// forward to its next survivor (cheap, divergent), then all lanes that found
// one evaluate it together.
//
// Measured alternatives (profiles/round1_reslice_variants.md): warp-
// cooperative run scans with per-pixel survivor rows (coalesced, DRAM at the
// compulsory 59 MB/pose) and per-lane survivor queues both lost to this
// version on instruction count or on L1 capacity.
template <int kDistMode>
__global__ void __launch_bounds__(256, 4) reslice_k(ResliceArgs a, uint8_t* __restrict__ out,
                                                 uint8_t* __restrict__ cov) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_gate = reinterpret_cast<double*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int pose, u, v;
  bool active;
  const double* gate;
  bool gate_filter = true;  // some orientation rejected for this pose -> test it per visit
  if (a.pose_major) {
    // pose-coherent batches (trajectories): lanes = the same pixel in 32
    // consecutive poses, whose visit streams nearly coincide (broadcast loads);
    // warps of a block = a 4x2 pixel patch.
    pose = blockIdx.y * 32 + lane;
    const int tiles_x4 = (a.W + 3) >> 2;
    u = (blockIdx.x % tiles_x4) * 4 + (warp & 3);
    v = (blockIdx.x / tiles_x4) * 2 + (warp >> 2);
    active = pose < a.P && u < a.W && v < a.H;
    if (pose >= a.P) pose = a.P - 1;  // inactive lanes read a valid pose
    gate = a.gate + (size_t)pose * a.n_orient;
  } else {
    pose = a.order ? a.order[blockIdx.y] : (int)blockIdx.y;
    const double* __restrict__ gate_g = a.gate + (size_t)pose * a.n_orient;
    const bool gate_in_smem = a.n_orient <= kGateSmem;
    if (gate_in_smem) {
      bool rej = false;
      for (int i = threadIdx.x; i < a.n_orient; i += blockDim.x) {
        const double g = gate_g[i];
        s_gate[i] = g;
        rej |= g == CUDART_INF;
      }
      gate_filter = __syncthreads_or(rej);
    }
    gate = gate_in_smem ? s_gate : gate_g;
    const int tile = blockIdx.x;
    u = (tile % a.tiles_x) * 16 + (warp & 1) * 8 + (lane & 7);
    v = (tile / a.tiles_x) * 16 + (warp >> 1) * 4 + (lane >> 3);
    active = u < a.W && v < a.H;
  }

  const double* pp = a.params + (size_t)pose * 14;
  const double du = (double)u * pp[12], dv = (double)v * pp[13];
  const double wx = (pp[0] + du * pp[3]) + dv * pp[4];
  const double wy = (pp[1] + du * pp[6]) + dv * pp[7];
  const double wz = (pp[2] + du * pp[9]) + dv * pp[10];
  const double r = a.radius;
  const double inv_v = 1.0 / a.voxel;
  int64_t lox, hix, loy, hiy, loz, hiz;
  cell_range(wx, r, a.origin[0], inv_v, a.dims[0], lox, hix);
  cell_range(wy, r, a.origin[1], inv_v, a.dims[1], loy, hiy);
  cell_range(wz, r, a.origin[2], inv_v, a.dims[2], loz, hiz);
  const float xlo = keep_lo(wx, r), xhi = keep_hi(wx, r);
  const float ylo = keep_lo(wy, r), yhi = keep_hi(wy, r);
  const float zlo = keep_lo(wz, r), zhi = keep_hi(wz, r);

  // run cursor over the (cx, cy) columns; each column's cells loz..hiz are one
  // contiguous sample range [off[base+loz], off[base+hiz+1])
  int64_t cx = lox, cy = loy;
  uint32_t s = 0, e = 0;
  auto open_run = [&]() -> bool {
    if (a.brute) {
      if (cx > lox) return false;
      s = 0;
      e = a.n_samples;
      cx = lox + 1;
      return s < e;
    }
    while (cx <= hix) {
      const int64_t base = (cx * a.dims[1] + cy) * a.dims[2];
      s = __ldg(a.offsets + base + loz);
      e = __ldg(a.offsets + base + hiz + 1);
      if (++cy > hiy) {
        cy = loy;
        ++cx;
      }
      if (s < e) return true;
    }
    return false;
  };
  bool live = active && (a.brute ? true : (lox <= hix && loy <= hiy && loz <= hiz)) && open_run();
  auto keep = [&](const uint4& c) -> bool {
    const float x = __uint_as_float(c.x), y = __uint_as_float(c.y), z = __uint_as_float(c.z);
    return x >= xlo && x <= xhi && y >= ylo && y <= yhi && z >= zlo && z <= zhi &&
           (!gate_filter || gate[c.w >> 8] != CUDART_INF);
  };

  // Each lane holds a batch of up to 4 consecutive records of its current run
  // (4 independent loads in flight) and a bit mask of the batch's survivors.
  // Rounds: lanes with an exhausted batch refill (cheap, divergent); then
  // every lane with a pending survivor evaluates it (converged FP64 path).
  uint4 r0 = make_uint4(0, 0, 0, 0), r1 = r0, r2 = r0, r3 = r0;
  unsigned mask = 0;
  double wsum = 0.0, iwsum = 0.0;
  while (true) {
    while (live && mask == 0) {
      const uint32_t n = min(4u, e - s);
      const uint4* __restrict__ q = a.records + s;
      r0 = __ldg(q);
      if (n > 1) r1 = __ldg(q + 1);
      if (n > 2) r2 = __ldg(q + 2);
      if (n > 3) r3 = __ldg(q + 3);
      s += n;
      mask = (keep(r0) ? 1u : 0u) | ((n > 1 && keep(r1)) ? 2u : 0u) | ((n > 2 && keep(r2)) ? 4u : 0u) |
             ((n > 3 && keep(r3)) ? 8u : 0u);
      if (s == e) live = open_run();
    }
    if (!__any_sync(0xffffffffu, mask != 0)) break;
    if (mask) {
      const unsigned kk = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint4 cur = kk == 0 ? r0 : (kk == 1 ? r1 : (kk == 2 ? r2 : r3));
      const double dx = (double)__uint_as_float(cur.x) - wx;
      const double dy = (double)__uint_as_float(cur.y) - wy;
      const double dz = (double)__uint_as_float(cur.z) - wz;
      double arg = gate[cur.w >> 8];
      if (kDistMode != 2) {
        const double dist = sqrt((dx * dx + dy * dy) + dz * dz);
        const double kdd = a.kd * dist;
        arg = arg - (kDistMode == 1 ? kdd * a.inv_radius : kdd / r);
      }
      const double w = dare_exp(arg);
      wsum += w;
      iwsum += w * (double)(cur.w & 0xffu);
    }
  }
  if (!active) return;
  const size_t k = ((size_t)pose * a.H + v) * a.W + u;
  if (wsum >= kCoverageMinWeight) {
    double f = floor(iwsum / wsum + 0.5);
    f = f < 0.0 ? 0.0 : (f > 255.0 ? 255.0 : f);
    out[k] = (uint8_t)f;
    cov[k] = 1;
  } else {
    out[k] = (uint8_t)a.unassigned;
    cov[k] = 0;
  }
}

// Batch scheduling: blocks are dispatched pose-major, so ~2 poses are in flight
// at a time.  Launching the batch in spatial order (plane centre, coarse z
// then y then x) makes consecutive poses share cells in L2.  Pure
// scheduling: every pose's pixels are computed exactly as before.
__global__ void pose_key_k(const double* __restrict__ params, int P, int W, int H, double ox,
                           double oy, double oz, double cell, unsigned long long* keys, int* idx) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double* pp = params + (size_t)p * 14;
  const double hu = 0.5 * (W - 1) * pp[12], hv = 0.5 * (H - 1) * pp[13];
  const double c[3] = {pp[0] + hu * pp[3] + hv * pp[4], pp[1] + hu * pp[6] + hv * pp[7],
                       pp[2] + hu * pp[9] + hv * pp[10]};
  const double o[3] = {ox, oy, oz};
  unsigned long long q[3];
  for (int k = 0; k < 3; ++k) {
    double f = floor((c[k] - o[k]) / cell);
    f = f < 0.0 ? 0.0 : (f > 1048575.0 ? 1048575.0 : (f != f ? 0.0 : f));
    q[k] = (unsigned long long)f;
  }
  keys[p] = (q[2] << 40) | (q[1] << 20) | q[0];
  idx[p] = p;
}

__global__ void exp_k(const double* x, double* y, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = dare_exp(x[i]);
}

static void launch_reslice(dare_volume_t vol, int32_t P, const double* d_params, int32_t W,
                           int32_t H, const dare_reslice_cfg* cfg, uint8_t* d_pixels,
                           uint8_t* d_cov, cudaStream_t s, int brute = 0, bool coherent = false) {
  DARE_REQUIRE(vol != nullptr && cfg != nullptr, "null argument");
  DARE_REQUIRE(W > 0 && H > 0, "reslice plane must have at least one pixel");
  DARE_REQUIRE(P >= 0 && P <= 65535, "n_poses must be in [0, 65535] per launch");
  DARE_REQUIRE(cfg->radius > 0, "interp_radius must be > 0");
  if (P == 0) return;
  ResliceArgs a;
  a.offsets = vol->d_offsets;
  a.records = vol->d_records;
  a.params = d_params;
  a.n_orient = std::max<int64_t>(vol->n_orient, 1);
  for (int i = 0; i < 3; ++i) {
    a.origin[i] = vol->origin[i];
    a.dims[i] = vol->dims[i];
  }
  a.voxel = vol->voxel;
  a.radius = cfg->radius;
  a.kd = cfg->k_dist;
  a.inv_radius = 1.0 / cfg->radius;
  a.dist_mode = cfg->k_dist == 0.0 ? 2 : (exact_reciprocal(cfg->radius) ? 1 : 0);
  a.unassigned = cfg->unassigned;
  a.W = W;
  a.H = H;
  a.P = P;
  a.tiles_x = (int)ceil_div(W, 16);
  a.brute = brute;
  a.n_samples = (uint32_t)vol->n_samples;
  const int tiles_y = (int)ceil_div(H, 16);
  PhaseTimer pt(s, "reslice");
  Scratch<double> gate((size_t)P * a.n_orient, s);
  a.gate = gate.ptr;
  if (vol->n_orient > 0) {
    gate_k<<<dim3(ceil_div(vol->n_orient, 256), P), 256, 0, s>>>(vol->d_orient, vol->n_orient,
                                                                 d_params, P, *cfg, gate.ptr);
    DARE_CUDA(cudaGetLastError());
  }
  pt.mark("gate");
  a.order = nullptr;
  a.pose_major = (cfg->schedule == 2 || (cfg->schedule == 0 && coherent)) && !brute ? 1 : 0;
  Scratch<int> order(P >= 4 ? P : 0, s);
  if (P >= 4 && !brute && !a.pose_major) {
    Scratch<unsigned long long> keys(2 * (size_t)P, s);
    Scratch<int> idx(P, s);
    pose_key_k<<<ceil_div(P, 128), 128, 0, s>>>(d_params, P, W, H, a.origin[0], a.origin[1],
                                                 a.origin[2], 8.0 * a.voxel, keys.ptr, idx.ptr);
    size_t bytes = 0;
    DARE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.ptr, keys.ptr + P, idx.ptr,
                                              order.ptr, P, 0, 60, s));
    Scratch<uint8_t> tmp(bytes, s);
    DARE_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, bytes, keys.ptr, keys.ptr + P, idx.ptr,
                                              order.ptr, P, 0, 60, s));
    a.order = order.ptr;
  }
  pt.mark("order");
  const dim3 grid = a.pose_major ? dim3(ceil_div(W, 4) * ceil_div(H, 2), ceil_div(P, 32))
                                  : dim3(a.tiles_x * tiles_y, P);
  static bool attr_done = false;  // benign race: idempotent attribute set
  if (!attr_done) {
    DARE_CUDA(cudaFuncSetAttribute(reslice_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    DARE_CUDA(cudaFuncSetAttribute(reslice_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    DARE_CUDA(cudaFuncSetAttribute(reslice_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    attr_done = true;
  }
  if (a.dist_mode == 0)
    reslice_k<0><<<grid, 256, kSmemBytes, s>>>(a, d_pixels, d_cov);
  else if (a.dist_mode == 1)
    reslice_k<1><<<grid, 256, kSmemBytes, s>>>(a, d_pixels, d_cov);
  else
    reslice_k<2><<<grid, 256, kSmemBytes, s>>>(a, d_pixels, d_cov);
  pt.mark("reslice_k");
  DARE_CUDA(cudaGetLastError());
}

}  // namespace dare

using namespace dare;

extern "C" int dare_reslice_device(dare_volume_t vol, int32_t n_poses, const double* d_params,
                                   int32_t width, int32_t height, const dare_reslice_cfg* cfg,
                                   uint8_t* d_pixels, uint8_t* d_coverage, void* stream) {
  return guard([&] {
    cudaStream_t s = stream ? (cudaStream_t)stream : thread_stream();
    launch_reslice(vol, n_poses, d_params, width, height, cfg, d_pixels, d_coverage, s);
  });
}

// Coherence test for the pose-major schedule (host params).
static bool poses_coherent(const double* p, int32_t P, int32_t W, int32_t H, double voxel) {
  if (P < 32) return false;
  int close = 0;
  double prev[3] = {0, 0, 0};
  for (int32_t i = 0; i < P; ++i) {
    const double* q = p + (size_t)i * 14;
    const double hu = 0.5 * (W - 1) * q[12], hv = 0.5 * (H - 1) * q[13];
    const double c[3] = {q[0] + hu * q[3] + hv * q[4], q[1] + hu * q[6] + hv * q[7],
                         q[2] + hu * q[9] + hv * q[10]};
    if (i > 0) {
      const double* o = q - 14;
      double dr = 0.0;
      for (int k = 3; k < 12; ++k) dr = fmax(dr, fabs(q[k] - o[k]));
      const double dc = fmax(fabs(c[0] - prev[0]), fmax(fabs(c[1] - prev[1]), fabs(c[2] - prev[2])));
      close += (dc <= voxel && dr <= 0.05) ? 1 : 0;
    }
    for (int k = 0; k < 3; ++k) prev[k] = c[k];
  }
  return close >= (int)(0.9 * (P - 1));
}

// host-buffer wrapper: params H2D, launches (<= 65535 poses each), outputs D2H
static void reslice_host(dare_volume_t vol, int32_t n_poses, const double* params, int32_t width,
                         int32_t height, const dare_reslice_cfg* cfg, uint8_t* pixels,
                         uint8_t* coverage, int brute) {
  DARE_REQUIRE(n_poses >= 0, "negative pose count");
  DARE_REQUIRE(width > 0 && height > 0, "reslice plane must have at least one pixel");
  if (n_poses == 0) return;
  cudaStream_t s = thread_stream();
  const size_t npix = (size_t)n_poses * width * height;
  Scratch<double> d_params((size_t)n_poses * 14, s);
  Scratch<uint8_t> d_out(2 * npix, s);
  DARE_CUDA(cudaMemcpyAsync(d_params.ptr, params, sizeof(double) * 14 * n_poses,
                            cudaMemcpyHostToDevice, s));
  for (int32_t p0 = 0; p0 < n_poses; p0 += 65535) {
    int32_t np = std::min<int32_t>(65535, n_poses - p0);
    size_t off = (size_t)p0 * width * height;
    launch_reslice(vol, np, d_params.ptr + (size_t)p0 * 14, width, height, cfg, d_out.ptr + off,
                   d_out.ptr + npix + off, s, brute,
                   poses_coherent(params + (size_t)p0 * 14, np, width, height, vol->voxel));
  }
  DARE_CUDA(cudaMemcpyAsync(pixels, d_out.ptr, npix, cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaMemcpyAsync(coverage, d_out.ptr + npix, npix, cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaStreamSynchronize(s));
}

extern "C" int dare_reslice(dare_volume_t vol, int32_t n_poses, const double* params,
                            int32_t width, int32_t height, const dare_reslice_cfg* cfg,
                            uint8_t* pixels, uint8_t* coverage) {
  return guard([&] { reslice_host(vol, n_poses, params, width, height, cfg, pixels, coverage, 0); });
}

extern "C" int dare_reslice_bruteforce(dare_volume_t vol, int32_t n_poses, const double* params,
                                       int32_t width, int32_t height, const dare_reslice_cfg* cfg,
                                       uint8_t* pixels, uint8_t* coverage) {
  return guard([&] { reslice_host(vol, n_poses, params, width, height, cfg, pixels, coverage, 1); });
}

extern "C" int dare_poses_coherent(const double* params, int32_t n_poses, int32_t width,
                                   int32_t height, double voxel_size) {
  return poses_coherent(params, n_poses, width, height, voxel_size) ? 1 : 0;
}

extern "C" int dare_exp_device(const double* d_x, double* d_y, int64_t n, void* stream) {
  return guard([&] {
    cudaStream_t s = stream ? (cudaStream_t)stream : thread_stream();
    if (n > 0) exp_k<<<ceil_div(n, 256), 256, 0, s>>>(d_x, d_y, n);
    DARE_CUDA(cudaGetLastError());
  });
}
