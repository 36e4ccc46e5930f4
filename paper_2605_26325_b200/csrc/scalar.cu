// Direction-blind (PLUS-style) comparison arm: compound -> fill_holes ->
// reslice_trilinear.  Reference: baseline.py:64-155, _kernels.py:170-229.
//
//  compound  : same pixel -> cell map as reconstruction; u64 sum / u64 count
//              atomics, warp-aggregated over equal cells (integer sums are
//              order-free, so atomics are exact -- baseline.py:67 relies on it);
//              then values = f32(f64(sum) / f64(count)) (baseline.py:93-96).
//  fill_holes: Jacobi passes in f64 (baseline.py:108: values are promoted to
//              f64 and filled values are NOT re-rounded between passes).  Only
//              voxels filled by this call need f64 storage (flag >= 3); every
//              other value is read from the f32 input, whose promotion is
//              exact.  Neighbour sums run in C order over the 26 offsets (the
//              order scipy's convolve visits the footprint), unknown and
//              out-of-grid neighbours add 0.  In-place with pass tags: a voxel
//              filled in pass p carries flag 3+p and is "unknown" to readers in
//              pass p (Jacobi), "known" afterwards; finalize maps tags -> 2.
//  trilinear : thread per pixel, 8 corners in (cx, cy, cz) order, f32 values
//              read directly (the reference's per-call f64 copy of the whole
//              grid, baseline.py:142-149, is pure overhead: f32->f64 is exact).
#include <cmath>
#include <memory>
#include <vector>

#include "cells.cuh"
#include "volume.cuh"

namespace dare {

struct ScalarFrameView {
  const uint8_t* frames;
  const int32_t* image;
  const double* axes;
  const uint8_t* mask;
  int64_t n_frames;
  int32_t H, W;
  double px, py;
};

// Thread = one pixel (u, v) over a chunk of kCFrames consecutive frames; warp
// = an 8(u) x 4(v) patch, block = 16 x 16 pixels.  Each thread keeps a running
// (cell, sum, count) and only flushes when its pixel moves to another cell --
// consecutive frames of a sweep land in the same cell for several frames --
// and a flush is warp-aggregated over lanes flushing the same cell (image
// neighbours).  Integer sums make the result independent of the order
// (baseline.py:67), so the atomics are exact.
constexpr int kCFrames = 64;

// Warp-converged flush: lanes with need=false get a unique non-cell key, so
// MATCH / REDUX run once on the full warp (no divergent collective loops).
__device__ __forceinline__ void compound_flush(bool need, int64_t lin, unsigned sum, unsigned cnt,
                                               unsigned long long* sums, unsigned long long* counts) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned long long key = need ? (unsigned long long)lin : (0x8000000000000000ull | lane);
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const unsigned total = __reduce_add_sync(peers, sum);
  const unsigned n = __reduce_add_sync(peers, cnt);
  if (need && lane == (unsigned)(__ffs(peers) - 1)) {
    atomicAdd(&sums[lin], (unsigned long long)total);
    atomicAdd(&counts[lin], (unsigned long long)n);
  }
}

template <bool kInv>
__global__ void __launch_bounds__(256) compound_k(ScalarFrameView fv, VoxelMap m,
                                                  unsigned long long* sums,
                                                  unsigned long long* counts) {
  __shared__ double s_axes[kCFrames * 9];
  __shared__ long long s_img[kCFrames];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t W = (uint32_t)fv.W, H = (uint32_t)fv.H;
  const uint32_t tiles_u = (W + 15) / 16;
  const uint32_t u = (blockIdx.x % tiles_u) * 16 + (warp & 1) * 8 + (lane & 7);
  const uint32_t v = (blockIdx.x / tiles_u) * 16 + (warp >> 1) * 4 + (lane >> 3);
  const uint32_t p = v * W + u;
  const bool in_frame = u < W && v < H && (!fv.mask || fv.mask[p] != 0);
  const long long hw = (long long)H * W;
  const int64_t f0 = (int64_t)blockIdx.y * kCFrames;
  const int nf = (int)min((int64_t)kCFrames, fv.n_frames - f0);
  for (int i = threadIdx.x; i < nf * 9; i += blockDim.x) s_axes[i] = fv.axes[f0 * 9 + i];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) s_img[i] = (long long)fv.image[f0 + i] * hw;
  __syncthreads();
  const double U = (double)u * fv.px, V = (double)v * fv.py;
  int64_t cur = -1;
  unsigned sum = 0, cnt = 0;
  for (int j = 0; j < nf; ++j) {  // block-uniform trip count
    // the cell is computed for every lane (no divergent branch) and masked
    const int64_t cell = frame_cell<kInv>(s_axes + j * 9, U, V, m);
    const int64_t lin = in_frame ? cell : -1;
    const unsigned inten = in_frame ? (unsigned)fv.frames[s_img[j] + p] : 0u;
    const bool change = lin != cur;
    const bool need = change && cur >= 0;
    if (__any_sync(0xffffffffu, need)) compound_flush(need, cur, sum, cnt, sums, counts);
    if (change) {
      cur = lin;
      sum = 0;
      cnt = 0;
    }
    sum += inten;
    cnt += 1;
  }
  if (__any_sync(0xffffffffu, cur >= 0)) compound_flush(cur >= 0, cur, sum, cnt, sums, counts);
}

// compound_k on the exact threshold tables (cells.cuh; same integer sums):
// per frame two compares per axis against the current cell's interval, the
// f64 in-plane product reused across frames with identical axis columns,
// 32-bit cells and a 32-bit MATCH for the warp-aggregated flush.
// kPacked: one 64-bit atomic per flush into count << 40 | sum (the host
// enables it only when no cell can collect 2^24 observations, so the sum,
// <= 255 * count, stays below 2^40); split into sums / counts afterwards.
template <bool kPacked>
__device__ __forceinline__ void compound_flush32(bool need, int32_t lin, unsigned sum, unsigned cnt,
                                                 unsigned long long* sums, unsigned long long* counts) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned key = need ? (unsigned)lin : (0x80000000u | lane);
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const unsigned total = __reduce_add_sync(peers, sum);
  const unsigned n = __reduce_add_sync(peers, cnt);
  if (need && lane == (unsigned)(__ffs(peers) - 1)) {
    if (kPacked) {
      atomicAdd(&sums[lin], ((unsigned long long)n << 40) | (unsigned long long)total);
    } else {
      atomicAdd(&sums[lin], (unsigned long long)total);
      atomicAdd(&counts[lin], (unsigned long long)n);
    }
  }
}

// packed -> the caller's (accumulating) sums / counts
__global__ void compound_unpack_k(int64_t n, const unsigned long long* __restrict__ packed,
                                  unsigned long long* sums, unsigned long long* counts) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const unsigned long long v = packed[c];
  if (v == 0) return;
  sums[c] += v & ((1ull << 40) - 1);
  counts[c] += v >> 40;
}

template <bool kPacked>
__global__ void __launch_bounds__(256) compound_tab_k(ScalarFrameView fv, CellTables ct, VoxelMap m,
                                                      unsigned long long* sums, unsigned long long* counts) {
  __shared__ double s_axes[kCFrames * 9];
  __shared__ long long s_img[kCFrames];
  __shared__ int s_same[kCFrames];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t W = (uint32_t)fv.W, H = (uint32_t)fv.H;
  const uint32_t tiles_u = (W + 15) / 16;
  const uint32_t u = (blockIdx.x % tiles_u) * 16 + (warp & 1) * 8 + (lane & 7);
  const uint32_t v = (blockIdx.x / tiles_u) * 16 + (warp >> 1) * 4 + (lane >> 3);
  const uint32_t p = v * W + u;
  const bool in_frame = u < W && v < H && (!fv.mask || fv.mask[p] != 0);
  const long long hw = (long long)H * W;
  const int64_t f0 = (int64_t)blockIdx.y * kCFrames;
  const int nf = (int)min((int64_t)kCFrames, fv.n_frames - f0);
  for (int i = threadIdx.x; i < nf * 9; i += blockDim.x) s_axes[i] = fv.axes[f0 * 9 + i];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) s_img[i] = (long long)fv.image[f0 + i] * hw;
  __syncthreads();
  for (int j = threadIdx.x; j < nf; j += blockDim.x) {
    bool same = j > 0;
    for (int c = 0; c < 6 && same; ++c)
      same = __double_as_longlong(s_axes[j * 9 + c]) == __double_as_longlong(s_axes[(j - 1) * 9 + c]);
    s_same[j] = same;
  }
  __syncthreads();
  const double U = (double)u * fv.px, V = (double)v * fv.py;
  const uint32_t ny = (uint32_t)m.dims[1], nz = (uint32_t)m.dims[2];
  AxisCell ax[3];
  double S[3];
  for (int a = 0; a < 3; ++a) {
    ax[a].g = -2;
    ax[a].lo = ax[a].hi = 0.0;
    S[a] = 0.0;
  }
  int32_t cur = -1;
  unsigned sum = 0, cnt = 0;
  for (int j = 0; j < nf; ++j) {  // block-uniform trip count
    const double* fa = s_axes + j * 9;
    double P[3];
    if (s_same[j]) {
#pragma unroll
      for (int a = 0; a < 3; ++a) P[a] = S[a] + fa[6 + a];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        S[a] = U * fa[a] + V * fa[3 + a];
        P[a] = S[a] + fa[6 + a];
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {  // relocate only the axes whose interval the point left
      if (!axis_same(P[a], ax[a])) {
        if (ax[a].g == -2) ax[a].g = axis_guess(P[a], m.origin[a], m.inv_voxel, ct.n[a], 0);
        axis_locate(P[a], ct.t[a], ct.n[a], ax[a]);
      }
    }
    const bool ok = in_frame && ax[0].g >= 0 && ax[0].g < ct.n[0] && ax[1].g >= 0 && ax[1].g < ct.n[1] &&
                    ax[2].g >= 0 && ax[2].g < ct.n[2];
    const int32_t lin = ok ? (int32_t)(((uint32_t)ax[0].g * ny + (uint32_t)ax[1].g) * nz + (uint32_t)ax[2].g) : -1;
    DARE_CHECK(lin < 0 || (int64_t)lin < m.dims[0] * m.dims[1] * m.dims[2]);
    const unsigned inten = in_frame ? (unsigned)fv.frames[s_img[j] + p] : 0u;
    const bool change = lin != cur;
    const bool need = change && cur >= 0;
    if (__any_sync(0xffffffffu, need)) compound_flush32<kPacked>(need, cur, sum, cnt, sums, counts);
    if (change) {
      cur = lin;
      sum = 0;
      cnt = 0;
    }
    sum += inten;
    cnt += 1;
  }
  if (__any_sync(0xffffffffu, cur >= 0)) compound_flush32<kPacked>(cur >= 0, cur, sum, cnt, sums, counts);
}

// compound_k with the in-plane product U*R[a,0] + V*R[a,1] reused across
// consecutive frames whose axis columns are bit-identical (the same f64 value
// the reference computes, so P = that + t[a] is bit-identical), 32-bit cell
// indices (frame_cell32's quotient bounds test and truncating conversion) and
// a 32-bit MATCH for the flush.
template <bool kInv>
__global__ void __launch_bounds__(256) compound2_k(ScalarFrameView fv, VoxelMap m, unsigned long long* sums,
                                                   unsigned long long* counts) {
  __shared__ double s_axes[kCFrames * 9];
  __shared__ long long s_img[kCFrames];
  __shared__ int s_same[kCFrames];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t W = (uint32_t)fv.W, H = (uint32_t)fv.H;
  const uint32_t tiles_u = (W + 15) / 16;
  const uint32_t u = (blockIdx.x % tiles_u) * 16 + (warp & 1) * 8 + (lane & 7);
  const uint32_t v = (blockIdx.x / tiles_u) * 16 + (warp >> 1) * 4 + (lane >> 3);
  const uint32_t p = v * W + u;
  const bool in_frame = u < W && v < H && (!fv.mask || fv.mask[p] != 0);
  const long long hw = (long long)H * W;
  const int64_t f0 = (int64_t)blockIdx.y * kCFrames;
  const int nf = (int)min((int64_t)kCFrames, fv.n_frames - f0);
  for (int i = threadIdx.x; i < nf * 9; i += blockDim.x) s_axes[i] = fv.axes[f0 * 9 + i];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) s_img[i] = (long long)fv.image[f0 + i] * hw;
  __syncthreads();
  for (int j = threadIdx.x; j < nf; j += blockDim.x) {
    bool same = j > 0;
    for (int c = 0; c < 6 && same; ++c)
      same = __double_as_longlong(s_axes[j * 9 + c]) == __double_as_longlong(s_axes[(j - 1) * 9 + c]);
    s_same[j] = same;
  }
  __syncthreads();
  const double U = (double)u * fv.px, V = (double)v * fv.py;
  const uint32_t ny = (uint32_t)m.dims[1], nz = (uint32_t)m.dims[2];
  double S[3] = {0.0, 0.0, 0.0};
  int32_t cur = -1;
  unsigned sum = 0, cnt = 0;
  for (int j = 0; j < nf; ++j) {  // block-uniform trip count and branches
    const double* fa = s_axes + j * 9;
    if (!s_same[j]) {
#pragma unroll
      for (int a = 0; a < 3; ++a) S[a] = U * fa[a] + V * fa[3 + a];
    }
    bool ok = true;
    uint32_t idx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double d = (double)__double2float_rn(S[a] + fa[6 + a]) - m.origin[a];
      // 0 <= floor(q) < n  <=>  0 <= q < n (n integral; NaN fails both)
      const double q = kInv ? d * m.inv_voxel : d / m.voxel;
      ok = ok && (q >= 0.0) && (q < (double)m.dims[a]);
      idx[a] = ok ? __double2uint_rz(q) : 0u;
    }
    const int32_t lin = (ok && in_frame) ? (int32_t)((idx[0] * ny + idx[1]) * nz + idx[2]) : -1;
    const unsigned inten = in_frame ? (unsigned)fv.frames[s_img[j] + p] : 0u;
    const bool change = lin != cur;
    const bool need = change && cur >= 0;
    if (__any_sync(0xffffffffu, need)) compound_flush32<false>(need, cur, sum, cnt, sums, counts);
    if (change) {
      cur = lin;
      sum = 0;
      cnt = 0;
    }
    sum += inten;
    cnt += 1;
  }
  if (__any_sync(0xffffffffu, cur >= 0)) compound_flush32<false>(cur >= 0, cur, sum, cnt, sums, counts);
}

__global__ void compound_finalize_k(int64_t n, const unsigned long long* __restrict__ sums,
                                    const unsigned long long* __restrict__ counts, float* values,
                                    uint8_t* flags) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  unsigned long long k = counts[c];
  if (k > 0) {
    values[c] = __double2float_rn((double)(long long)sums[c] / (double)(long long)k);
    flags[c] = 1;
  } else {
    values[c] = 0.0f;
    flags[c] = 0;
  }
}

// known in pass p: observed (1), filled earlier (2 or a tag from pass < p)
__device__ __forceinline__ bool known_in_pass(uint8_t f, int tag) { return f != 0 && f != tag; }

// One Jacobi pass, tiled: a block owns a 4(x) x 8(y) x 32(z) brick (thread =
// one (y, z) line of 4 x-cells, z fastest -> coalesced), stages the brick plus
// a one-cell halo as (known ? value : 0, known) in shared memory, and every
// empty cell sums its 26 neighbours in C order from there.  In place: a cell
// filled in this pass carries `tag` and reads as unknown to every reader of
// this pass, whether it sees the old or the new flag (Jacobi semantics).
constexpr int kFX = 4, kFY = 8, kFZ = 32;
constexpr int kHX = kFX + 2, kHY = kFY + 2, kHZ = kFZ + 2;

__global__ void __launch_bounds__(256) fill_pass_k(int64_t nx, int64_t ny, int64_t nz,
                                                   const float* __restrict__ vin, double* v,
                                                   uint8_t* flags, int tag,
                                                   unsigned long long* filled, unsigned long long* left,
                                                   const unsigned long long* prev_filled,
                                                   const unsigned long long* prev_left) {
  // previous pass changed nothing (no fillable voxel) or left no empty voxel
  // (all known): the reference breaks out of its loop in both cases
  if (prev_filled && (*prev_filled == 0 || *prev_left == 0)) return;
  __shared__ double s_val[kHX * kHY * kHZ];
  __shared__ uint8_t s_known[kHX * kHY * kHZ];
  const int64_t bz = (nz + kFZ - 1) / kFZ, by = (ny + kFY - 1) / kFY;
  const int64_t b = blockIdx.x;
  const int64_t z0 = (b % bz) * kFZ, y0 = ((b / bz) % by) * kFY, x0 = (b / (bz * by)) * kFX;
  const int tz = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t y = y0 + ty, z = z0 + tz;
  bool empty_here = false;
  for (int i = 0; i < kFX; ++i) {
    const int64_t x = x0 + i;
    if (x < nx && y < ny && z < nz) empty_here |= flags[(x * ny + y) * nz + z] == 0;
  }
  if (!__syncthreads_or(empty_here)) return;  // nothing to fill in this brick
  for (int e = threadIdx.x; e < kHX * kHY * kHZ; e += blockDim.x) {
    const int hz = e % kHZ, hy = (e / kHZ) % kHY, hx = e / (kHZ * kHY);
    const int64_t X = x0 + hx - 1, Y = y0 + hy - 1, Z = z0 + hz - 1;
    double val = 0.0;
    uint8_t kn = 0;
    if (X >= 0 && X < nx && Y >= 0 && Y < ny && Z >= 0 && Z < nz) {
      const int64_t q = (X * ny + Y) * nz + Z;
      const uint8_t f = ((volatile uint8_t*)flags)[q];
      if (known_in_pass(f, tag)) {  // filled in an earlier pass: f64 work value; else the f32 input
        val = f >= 3 ? ((volatile double*)v)[q] : (double)vin[q];
        kn = 1;
      }
    }
    s_val[e] = val;
    s_known[e] = kn;
  }
  __syncthreads();
  bool did = false, still_empty = false;
  for (int i = 0; i < kFX; ++i) {
    const int64_t x = x0 + i;
    if (x >= nx || y >= ny || z >= nz) continue;
    const int64_t c = (x * ny + y) * nz + z;
    if (flags[c] != 0) continue;
    // the value sum stays FP64 in scipy's C order; the known count is a sum
    // of <= 26 ones, exact in integers (identical to the FP64 convolution)
    double s = 0.0;
    int known_n = 0;
#pragma unroll
    for (int dx = 0; dx < 3; ++dx)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dz = 0; dz < 3; ++dz) {
          if (dx == 1 && dy == 1 && dz == 1) continue;
          const int e = ((i + dx) * kHY + (ty + dy)) * kHZ + (tz + dz);
          s += s_val[e];
          known_n += s_known[e];
        }
    const double cnt = (double)known_n;
    if (cnt > 0.0) {
      v[c] = s / cnt;
      flags[c] = (uint8_t)tag;
      did = true;
    } else {
      still_empty = true;
    }
  }
  if (__syncthreads_or(did) && threadIdx.x == 0) atomicAdd(filled, 1ull);
  if (__syncthreads_or(still_empty) && threadIdx.x == 0) atomicAdd(left, 1ull);
}

// 4 voxels per thread (u8 flags as one 32-bit word, values as float4)
__global__ void fill_finalize_k(int64_t n, const float* __restrict__ vin, const double* __restrict__ v,
                                const uint8_t* flags_in, float* values, uint8_t* flags) {
  const int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c0 >= n) return;
  if (c0 + 4 <= n) {
    const uchar4 f = *reinterpret_cast<const uchar4*>(flags_in + c0);
    float4 x = *reinterpret_cast<const float4*>(vin + c0);  // f32(f64(x)) == x unless refilled
    if (f.x >= 3) x.x = __double2float_rn(v[c0]);
    if (f.y >= 3) x.y = __double2float_rn(v[c0 + 1]);
    if (f.z >= 3) x.z = __double2float_rn(v[c0 + 2]);
    if (f.w >= 3) x.w = __double2float_rn(v[c0 + 3]);
    *reinterpret_cast<float4*>(values + c0) = x;
    *reinterpret_cast<uchar4*>(flags + c0) =
        make_uchar4(f.x >= 3 ? 2 : f.x, f.y >= 3 ? 2 : f.y, f.z >= 3 ? 2 : f.z, f.w >= 3 ? 2 : f.w);
    return;
  }
  for (int64_t c = c0; c < n; ++c) {
    const uint8_t f = flags_in[c];
    values[c] = f >= 3 ? __double2float_rn(v[c]) : vin[c];
    flags[c] = f >= 3 ? 2 : f;
  }
}

struct TrilinearArgs {
  const float* values;
  const uint8_t* flags;
  const double* params;
  double origin[3];
  double voxel;
  int64_t dims[3];
  int W, H, tiles_x;
};

__global__ void __launch_bounds__(256) trilinear_k(TrilinearArgs a, uint8_t* out, uint8_t* cov,
                                                   double* out_val) {
  const int pose = blockIdx.y;
  const int tile = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = (tile % a.tiles_x) * 16 + (warp & 1) * 8 + (lane & 7);
  const int v = (tile / a.tiles_x) * 16 + (warp >> 1) * 4 + (lane >> 3);
  if (u >= a.W || v >= a.H) return;
  const double* pp = a.params + (size_t)pose * 14;
  const double du = (double)u * pp[12], dv = (double)v * pp[13];
  const double w[3] = {(pp[0] + du * pp[3]) + dv * pp[4], (pp[1] + du * pp[6]) + dv * pp[7],
                       (pp[2] + du * pp[9]) + dv * pp[10]};
  const double inv_v = 1.0 / a.voxel;
  int64_t i[3];
  double fr[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double g = (w[k] - a.origin[k]) * inv_v - 0.5;
    const double fl = floor(g);
    const double lim = (double)a.dims[k] + 1.0;
    i[k] = (int64_t)(fl < -2.0 ? -2.0 : (fl > lim ? lim : fl));
    fr[k] = g - fl;
  }
  // all 8 corners' loads first (independent), then the reference's
  // (cx, cy, cz) accumulation order (_kernels.py:205-221)
  uint8_t fl8[8];
  float val8[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int64_t jx = i[0] + (c >> 2), jy = i[1] + ((c >> 1) & 1), jz = i[2] + (c & 1);
    const bool in = jx >= 0 && jx < a.dims[0] && jy >= 0 && jy < a.dims[1] && jz >= 0 && jz < a.dims[2];
    const int64_t lin = in ? (jx * a.dims[1] + jy) * a.dims[2] + jz : 0;
    fl8[c] = in ? __ldg(a.flags + lin) : (uint8_t)0;
    val8[c] = in ? __ldg(a.values + lin) : 0.0f;
  }
  double wsum = 0.0, vsum = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (fl8[c] != 0) {
      const double wxc = (c >> 2) ? fr[0] : 1.0 - fr[0];
      const double wyc = ((c >> 1) & 1) ? fr[1] : 1.0 - fr[1];
      const double wc = (wxc * wyc) * ((c & 1) ? fr[2] : 1.0 - fr[2]);
      wsum += wc;
      vsum += wc * (double)val8[c];
    }
  }
  const size_t k = ((size_t)pose * a.H + v) * a.W + u;
  if (wsum >= 1e-12) {
    const double val = vsum / wsum;
    double r = floor(val + 0.5);
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
    out[k] = (uint8_t)r;
    cov[k] = 1;
    if (out_val) out_val[k] = val;
  } else {
    out[k] = 0;
    cov[k] = 0;
    if (out_val) out_val[k] = 0.0;
  }
}

static std::unique_ptr<dare_scalar_s> new_scalar(const double* origin, double voxel,
                                                  const int64_t* dims, bool with_counts) {
  DARE_REQUIRE(voxel > 0, "voxel_size must be > 0");
  DARE_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
  auto sv = std::make_unique<dare_scalar_s>();
  DARE_CUDA(cudaGetDevice(&sv->device));
  for (int a = 0; a < 3; ++a) {
    sv->origin[a] = origin[a];
    sv->dims[a] = dims[a];
  }
  sv->voxel = voxel;
  sv->ncells = dims[0] * dims[1] * dims[2];
  dev_alloc(&sv->d_values, sizeof(float) * sv->ncells);
  dev_alloc(&sv->d_flags, sv->ncells);
  if (with_counts) dev_alloc(&sv->d_counts, sizeof(int64_t) * sv->ncells);
  return sv;
}

static void launch_trilinear(dare_scalar_t vol, int32_t P, const double* d_params, int32_t W,
                             int32_t H, uint8_t* d_pixels, uint8_t* d_cov, double* d_values,
                             cudaStream_t s) {
  DARE_REQUIRE(vol != nullptr, "null volume");
  DARE_REQUIRE(W > 0 && H > 0, "reslice plane must have at least one pixel");
  DARE_REQUIRE(P >= 0 && P <= 65535, "n_poses must be in [0, 65535] per launch");
  if (P == 0) return;
  TrilinearArgs a;
  a.values = vol->d_values;
  a.flags = vol->d_flags;
  a.params = d_params;
  for (int k = 0; k < 3; ++k) {
    a.origin[k] = vol->origin[k];
    a.dims[k] = vol->dims[k];
  }
  a.voxel = vol->voxel;
  a.W = W;
  a.H = H;
  a.tiles_x = (int)ceil_div(W, 16);
  trilinear_k<<<dim3(a.tiles_x * ceil_div(H, 16), P), 256, 0, s>>>(a, d_pixels, d_cov, d_values);
  DARE_CUDA(cudaGetLastError());
}

}  // namespace dare

using namespace dare;

// Accumulates integer intensity sums / observation counts of the given frames
// into caller-owned device arrays (ncells u64 each).  Frame-sharded multi-GPU
// compounding all-reduces these (exact integers) before finalising.
extern "C" int dare_compound_accumulate(const uint8_t* frames, int64_t n_images, int32_t height,
                                        int32_t width, int32_t frames_on_device,
                                        const int32_t* frame_image, int64_t n_frames,
                                        const double* frame_axes, double pitch_x, double pitch_y,
                                        const uint8_t* mask, const double* origin,
                                        double voxel_size, const int64_t* dims, uint64_t* d_sums,
                                        uint64_t* d_counts, void* stream) {
  return guard([&] {
    DARE_REQUIRE(d_sums != nullptr && d_counts != nullptr, "null accumulator");
    DARE_REQUIRE(voxel_size > 0, "voxel_size must be > 0");
    cudaStream_t s = stream ? (cudaStream_t)stream : thread_stream();
    FrameSet fs(frames, n_images, height, width, frames_on_device, frame_image, n_frames,
                frame_axes, pitch_x, pitch_y, mask, s);
    VoxelMap m = make_voxel_map(origin, voxel_size, dims);
    fs.start_upload();
    fs.wait_frames(s, 0, n_frames);  // host frames: every image uploaded before compound_k reads them
    ScalarFrameView fv{fs.d_frames, fs.d_image, fs.d_axes, fs.d_mask, fs.n_frames,
                       fs.H,        fs.W,       fs.px,     fs.py};
    const int64_t hw = (int64_t)height * width;
    if (n_frames > 0) {
      (void)hw;
      PhaseTimer pt(s, "compound_accumulate");
      DARE_LIMIT(ceil_div(n_frames, kCFrames) <= 65535, "too many frames for one compound launch");
      dim3 grid(ceil_div(width, 16) * ceil_div(height, 16), ceil_div(n_frames, kCFrames));
      Scratch<double> tab_store;
      CellTables ct;
      // The threshold-table variant (compound_tab_k) measured slower than the
      // FP64-chain kernel here (cfg2: 1.56 vs 1.09 ms; the per-crossing table
      // walk's dependent loads sit on the flush path), unlike the count pass:
      // opt-in with DARE_COMPOUND_TABLES=1.
      const char* tabs = getenv("DARE_COMPOUND_TABLES");
      const int64_t ncells = m.dims[0] * m.dims[1] * m.dims[2];
      if ((tabs && tabs[0] == '1') && ncells < (int64_t)INT32_MAX &&
          build_cell_tables(m, false, s, tab_store, ct)) {
        // packed 64-bit flushes when lanes rarely share a cell (under 2 pixels per
        // cell and frame: every flush is its own atomic pair) and no cell can
        // reach 2^24 observations (a cell spans <= floor(sqrt3 v / p) + 2
        // pixels per image axis, per frame)
        const double per_frame = (std::floor(1.7320508075688772 * voxel_size / pitch_x) + 2.0) *
                                 (std::floor(1.7320508075688772 * voxel_size / pitch_y) + 2.0);
        const char* penv = getenv("DARE_COMPOUND_PACKED");  // development override (0 / 1)
        const bool packed = penv ? penv[0] == '1'
                                 : (voxel_size / pitch_x) * (voxel_size / pitch_y) < 2.0 &&
                                       (double)n_frames * per_frame < 16777216.0;
        if (packed && (double)n_frames * per_frame < 16777216.0) {
          Scratch<unsigned long long> pk(ncells, s);
          DARE_CUDA(cudaMemsetAsync(pk.ptr, 0, sizeof(unsigned long long) * ncells, s));
          compound_tab_k<true><<<grid, 256, 0, s>>>(fv, ct, m, pk.ptr, nullptr);
          compound_unpack_k<<<ceil_div(ncells, 256), 256, 0, s>>>(ncells, pk.ptr, (unsigned long long*)d_sums,
                                                                  (unsigned long long*)d_counts);
        } else {
          compound_tab_k<false><<<grid, 256, 0, s>>>(fv, ct, m, (unsigned long long*)d_sums,
                                                     (unsigned long long*)d_counts);
        }
      } else if (ncells < (int64_t)INT32_MAX && !(getenv("DARE_COMPOUND_V1") && getenv("DARE_COMPOUND_V1")[0] == '1'))
        (m.exact_inv ? compound2_k<true> : compound2_k<false>)<<<grid, 256, 0, s>>>(
            fv, m, (unsigned long long*)d_sums, (unsigned long long*)d_counts);
      else
        (m.exact_inv ? compound_k<true> : compound_k<false>)<<<grid, 256, 0, s>>>(
            fv, m, (unsigned long long*)d_sums, (unsigned long long*)d_counts);
      pt.mark("compound_k");
      DARE_CUDA(cudaGetLastError());
    }
    if (!frames_on_device || !stream) DARE_CUDA(cudaStreamSynchronize(s));
  });
}

// values = f32(f64(sum) / f64(count)), flags 0/1, counts kept (baseline.py:93-96).
extern "C" int dare_scalar_from_sums(const double* origin, double voxel_size, const int64_t* dims,
                                     const uint64_t* d_sums, const uint64_t* d_counts,
                                     dare_scalar_t* out) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr, "out handle pointer is null");
    cudaStream_t s = thread_stream();
    auto sv = new_scalar(origin, voxel_size, dims, true);
    DARE_CUDA(cudaMemcpyAsync(sv->d_counts, d_counts, sizeof(int64_t) * sv->ncells,
                              cudaMemcpyDeviceToDevice, s));
    compound_finalize_k<<<ceil_div(sv->ncells, 256), 256, 0, s>>>(
        sv->ncells, (const unsigned long long*)d_sums, (const unsigned long long*)d_counts,
        sv->d_values, sv->d_flags);
    DARE_CUDA(cudaGetLastError());
    DARE_CUDA(cudaStreamSynchronize(s));
    *out = sv.release();
  });
}

extern "C" int dare_compound(const uint8_t* frames, int64_t n_images, int32_t height,
                             int32_t width, int32_t frames_on_device, const int32_t* frame_image,
                             int64_t n_frames, const double* frame_axes, double pitch_x,
                             double pitch_y, const uint8_t* mask, const double* origin,
                             double voxel_size, const int64_t* dims, dare_scalar_t* out) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr, "out handle pointer is null");
    DARE_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
    cudaStream_t s = thread_stream();
    const int64_t ncells = dims[0] * dims[1] * dims[2];
    DeviceClock clock(s);
    PhaseTimer pt(s, "compound");
    Scratch<unsigned long long> acc(2 * ncells, s);
    DARE_CUDA(cudaMemsetAsync(acc.ptr, 0, sizeof(unsigned long long) * 2 * ncells, s));
    pt.mark("alloc+memset");
    int rc = dare_compound_accumulate(frames, n_images, height, width, frames_on_device,
                                      frame_image, n_frames, frame_axes, pitch_x, pitch_y, mask,
                                      origin, voxel_size, dims, (uint64_t*)acc.ptr,
                                      (uint64_t*)(acc.ptr + ncells), (void*)s);
    if (rc != DARE_OK) throw Error{rc, dare_last_error()};
    pt.mark("accumulate");
    rc = dare_scalar_from_sums(origin, voxel_size, dims, (const uint64_t*)acc.ptr,
                               (const uint64_t*)(acc.ptr + ncells), out);
    if (rc != DARE_OK) throw Error{rc, dare_last_error()};
    pt.mark("finalize");
    clock.stop();
  });
}

extern "C" int dare_scalar_upload(const double* origin, double voxel_size, const int64_t* dims,
                                  const float* values, const uint8_t* flags,
                                  const int64_t* counts, dare_scalar_t* out) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr, "out handle pointer is null");
    auto sv = new_scalar(origin, voxel_size, dims, counts != nullptr);
    cudaStream_t s = thread_stream();
    DARE_CUDA(cudaMemcpyAsync(sv->d_values, values, sizeof(float) * sv->ncells,
                              cudaMemcpyDefault, s));
    DARE_CUDA(cudaMemcpyAsync(sv->d_flags, flags, sv->ncells, cudaMemcpyDefault, s));
    if (counts)
      DARE_CUDA(cudaMemcpyAsync(sv->d_counts, counts, sizeof(int64_t) * sv->ncells,
                                cudaMemcpyDefault, s));
    DARE_CUDA(cudaStreamSynchronize(s));
    *out = sv.release();
  });
}

extern "C" int dare_scalar_download(dare_scalar_t vol, float* values, uint8_t* flags,
                                    int64_t* counts) {
  return guard([&] {
    DARE_REQUIRE(vol != nullptr, "null volume");
    cudaStream_t s = thread_stream();
    if (values)
      DARE_CUDA(cudaMemcpyAsync(values, vol->d_values, sizeof(float) * vol->ncells,
                                cudaMemcpyDeviceToHost, s));
    if (flags) DARE_CUDA(cudaMemcpyAsync(flags, vol->d_flags, vol->ncells, cudaMemcpyDeviceToHost, s));
    if (counts && vol->d_counts)
      DARE_CUDA(cudaMemcpyAsync(counts, vol->d_counts, sizeof(int64_t) * vol->ncells,
                                cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int dare_scalar_get_info(dare_scalar_t vol, dare_scalar_info* info) {
  return guard([&] {
    DARE_REQUIRE(vol != nullptr && info != nullptr, "null argument");
    info->device = vol->device;
    for (int a = 0; a < 3; ++a) {
      info->origin[a] = vol->origin[a];
      info->dims[a] = vol->dims[a];
    }
    info->voxel_size = vol->voxel;
    info->d_values = vol->d_values;
    info->d_flags = vol->d_flags;
    info->d_counts = vol->d_counts;
  });
}

extern "C" int dare_scalar_destroy(dare_scalar_t vol) {
  return guard([&] { delete vol; });
}

extern "C" int dare_fill_holes(dare_scalar_t in, int32_t max_passes, dare_scalar_t* out,
                               int32_t* passes_run) {
  return guard([&] {
    DARE_REQUIRE(in != nullptr && out != nullptr, "null argument");
    DARE_REQUIRE(max_passes >= 0 && max_passes <= 250, "max_passes must be in [0, 250]");
    cudaStream_t s = thread_stream();
    DeviceClock clock(s);
    PhaseTimer pt(s, "fill_holes");
    auto sv = new_scalar(in->origin, in->voxel, in->dims, in->d_counts != nullptr);
    pt.mark("alloc_out");
    const int64_t n = in->ncells;
    Scratch<double> work(n, s);
    Scratch<uint8_t> flags(n, s);
    Scratch<unsigned long long> filled(2 * std::max(max_passes, 1), s);  // per pass: filled, left
    DARE_CUDA(cudaMemsetAsync(filled.ptr, 0, sizeof(unsigned long long) * 2 * std::max(max_passes, 1), s));
    DARE_CUDA(cudaMemcpyAsync(flags.ptr, in->d_flags, n, cudaMemcpyDeviceToDevice, s));
    pt.mark("scratch");
    for (int p = 0; p < max_passes; ++p) {
      const unsigned fill_blocks = ceil_div(in->dims[0], kFX) * ceil_div(in->dims[1], kFY) *
                                   ceil_div(in->dims[2], kFZ);
      fill_pass_k<<<fill_blocks, 256, 0, s>>>(in->dims[0], in->dims[1], in->dims[2], in->d_values,
                                                    work.ptr, flags.ptr, 3 + p, filled.ptr + 2 * p,
                                                    filled.ptr + 2 * p + 1,
                                                    p ? filled.ptr + 2 * p - 2 : nullptr,
                                                    p ? filled.ptr + 2 * p - 1 : nullptr);
      DARE_CUDA(cudaGetLastError());
    }
    pt.mark("passes");
    fill_finalize_k<<<ceil_div(ceil_div(n, 4), 256), 256, 0, s>>>(n, in->d_values, work.ptr, flags.ptr,
                                                                  sv->d_values, sv->d_flags);
    DARE_CUDA(cudaGetLastError());
    pt.mark("finalize");
    if (in->d_counts)
      DARE_CUDA(cudaMemcpyAsync(sv->d_counts, in->d_counts, sizeof(int64_t) * n,
                                cudaMemcpyDeviceToDevice, s));
    pt.mark("counts");
    std::vector<unsigned long long> h(2 * std::max(max_passes, 1));
    DARE_CUDA(cudaMemcpyAsync(h.data(), filled.ptr, sizeof(unsigned long long) * h.size(),
                              cudaMemcpyDeviceToHost, s));
    clock.stop();
    int32_t runs = 0;
    for (int p = 0; p < max_passes; ++p) runs += h[2 * p] > 0;
    if (passes_run) *passes_run = runs;
    *out = sv.release();
  });
}

extern "C" int dare_reslice_trilinear_device(dare_scalar_t vol, int32_t n_poses,
                                             const double* d_params, int32_t width,
                                             int32_t height, uint8_t* d_pixels,
                                             uint8_t* d_coverage, double* d_values,
                                             void* stream) {
  return guard([&] {
    cudaStream_t s = stream ? (cudaStream_t)stream : thread_stream();
    launch_trilinear(vol, n_poses, d_params, width, height, d_pixels, d_coverage, d_values, s);
  });
}

extern "C" int dare_reslice_trilinear(dare_scalar_t vol, int32_t n_poses, const double* params,
                                      int32_t width, int32_t height, uint8_t* pixels,
                                      uint8_t* coverage, double* values) {
  return guard([&] {
    DARE_REQUIRE(n_poses >= 0, "negative pose count");
    if (n_poses == 0) return;
    cudaStream_t s = thread_stream();
    const size_t npix = (size_t)n_poses * width * height;
    Scratch<double> d_params((size_t)n_poses * 14, s);
    Scratch<uint8_t> d_out(2 * npix, s);
    Scratch<double> d_val(values ? npix : 0, s);
    DARE_CUDA(cudaMemcpyAsync(d_params.ptr, params, sizeof(double) * 14 * n_poses,
                              cudaMemcpyHostToDevice, s));
    for (int32_t p0 = 0; p0 < n_poses; p0 += 65535) {
      int32_t np = std::min<int32_t>(65535, n_poses - p0);
      size_t off = (size_t)p0 * width * height;
      launch_trilinear(vol, np, d_params.ptr + (size_t)p0 * 14, width, height, d_out.ptr + off,
                       d_out.ptr + npix + off, values ? d_val.ptr + off : nullptr, s);
    }
    DARE_CUDA(cudaMemcpyAsync(pixels, d_out.ptr, npix, cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaMemcpyAsync(coverage, d_out.ptr + npix, npix, cudaMemcpyDeviceToHost, s));
    if (values)
      DARE_CUDA(cudaMemcpyAsync(values, d_val.ptr, sizeof(double) * npix, cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaStreamSynchronize(s));
  });
}
