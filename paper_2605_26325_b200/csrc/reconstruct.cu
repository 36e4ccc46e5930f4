// Directional reconstruction: pixel -> cell scatter and the sealed CSR build.
//
// Reference: reconstruct.py:166-199 (reconstruct_volume), 152-163
// (frame_world_positions), volume.py:208-238 (insert_batch/_voxel_indices),
// volume.py:240-269 (seal: stable argsort by linear cell + bincount + cumsum).
//
// Device pipeline (all FP64 chains bit-identical to numpy; -fmad=false):
//   1. count : per pixel -> cell; runs of consecutive frames in one cell are
//              aggregated per thread, flushes warp-aggregated (__match_any_sync
//              groups equal cells, one atomic per group); out-of-bounds pixels
//              counted (volume.py:230-233).
//   2. scan  : exclusive prefix of counts -> cell offsets (CUB).
//   3. fill  : same runs -> slots = offset + atomic cursor; stores the 64-bit
//              key (insertion index << 10 | z bin << 8 | intensity); the
//              insertion index orders like synchronized frame * H*W + row-major
//              pixel (bit-packed (frame, v, u) when the widths fit 32 bits).
//   4. seal  : per cell, sort its (tiny) key run ascending = insertion order --
//              this is what makes the atomic fill identical to numpy's stable
//              argsort -- and materialise the 16 B records.  A warp seals 32
//              consecutive cells: their keys are staged in shared memory with
//              coalesced loads, each lane sorts its cell, and the records are
//              written back coalesced.  Runs longer than 32 go through CUB's
//              segmented sort and are (re)written afterwards.
// All pixel/cell index math is 32-bit (dims < 2^31 cells, < 2^32 pixels) with
// a multiply-high divider, which keeps the per-pixel instruction count low.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <memory>
#include <vector>

#include "cells.cuh"
#include "volume.cuh"

namespace dare {

// n / d for every 32-bit n (round-up multiply-high with the "add" fix-up).
struct FastDiv {
  uint32_t d = 1, mul = 0, shift = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (d <= 1) return;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    mul = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    shift = l;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d == 1) return n;
    const uint32_t t = __umulhi(n, mul);
    return (t + ((n - t) >> 1)) >> (shift - 1);
  }
};

struct FrameView {
  const uint8_t* frames;
  const int32_t* image;
  const double* axes;
  const uint8_t* mask;
  uint32_t n_frames;
  uint32_t H, W, hw;
  double px, py;
  const uint32_t* oid;  // orientation id per synchronized frame
  FastDiv div_w, div_hw;
  // insertion index encoding in the keys: packed (f << fshift | v << ushift | u)
  // when the bit widths fit 32 bits -- same order as f * hw + v * W + u, decoded
  // with shifts in the seal -- else linear (f * hw + p, decoded with FastDiv)
  uint32_t packed, ushift, fshift, fstride;
  // frame groups of the count / fill passes (see build_csr): chunk k of 64
  // frames belongs to group k / chunks_per_group, whose per-cell counters and
  // key offsets live at + group * ncells
  uint32_t chunks_per_group, ncells;
  // direct slots (group mode 2): 64-bit counters (samples | runs << 32) per
  // (group, cell); a (group, cell) with a single run gets its slot from the
  // per-group prefix table without an atomic
  uint32_t direct;
  // fill cursors packed 4 per word (u8; one key CSR, every cell <= 255 samples):
  // a quarter of the cursor footprint, so the cursor atomics stay in L2
  uint32_t byte_cursors;
  // bucketed fill (64-bit keys): slots per bucket of kBucketCells cells, the
  // key tagged with its cell within the bucket; bucket_place_k then places the
  // bucket's keys in their cells through shared memory (see build_csr)
  uint32_t bucketed;
  const uint32_t* pre;  // (group, cell) -> samples of the cell in earlier groups | single-run << 31
  __device__ __forceinline__ size_t group_base(uint32_t chunk) const {
    return (size_t)(chunk / chunks_per_group) * ncells;
  }
  __device__ __forceinline__ uint32_t pixel_key(uint32_t u, uint32_t v) const {
    return packed ? (v << ushift) | u : v * W + u;
  }
  __device__ __forceinline__ void decode(uint32_t pid, uint32_t& f, uint32_t& u, uint32_t& v) const {
    if (packed) {
      f = pid >> fshift;
      v = (pid >> ushift) & ((1u << (fshift - ushift)) - 1u);
      u = pid & ((1u << ushift) - 1u);
    } else {
      f = div_hw.div(pid);
      const uint32_t p = pid - f * hw;
      v = div_w.div(p);
      u = p - v * W;
    }
  }
};

static inline bool ncells_total_fits(int64_t ncells, int64_t groups) {
  return ncells * groups < (int64_t)UINT32_MAX - 1;
}

static inline uint32_t ceil_log2(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// One run of k samples of cell `cell` into the count histogram of its frame
// group (counts already offset to the group in the 32-bit layout; the direct
// mode's 64-bit counters also count runs).
__device__ __forceinline__ void count_run(uint32_t* counts, size_t gb64, bool direct, uint32_t cell, uint32_t k) {
  if (direct)
    atomicAdd(reinterpret_cast<unsigned long long*>(counts) + gb64 + cell, (1ull << 32) | (unsigned long long)k);
  else
    atomicAdd(counts + cell, k);
}

// Warp-aggregated histogram (kFill=false) or slot assignment (kFill=true):
// lanes holding the same cell form one __match_any_sync group; the lowest lane
// does one atomic for the whole group and lanes take consecutive slots.
template <bool kFill>
__device__ __forceinline__ void warp_scatter(bool kept, int32_t lin, unsigned long long key,
                                             uint32_t* counts,
                                             const uint32_t* __restrict__ offsets,
                                             unsigned long long* keys) {
  const unsigned active = __ballot_sync(0xffffffffu, kept);
  if (!kept) return;
  const unsigned peers = __match_any_sync(active, (unsigned)lin);
  const unsigned leader = __ffs(peers) - 1;
  const unsigned n = __popc(peers);
  if (!kFill) {
    if (lane_id() == leader) atomicAdd(&counts[lin], n);
  } else {
    unsigned base = 0;
    if (lane_id() == leader) base = atomicAdd(&counts[lin], n);
    base = __shfl_sync(peers, base, leader);
    const unsigned rank = __popc(peers & ((1u << lane_id()) - 1u));
    keys[offsets[lin] + base + rank] = key;
  }
}

// Frames.  Thread = one pixel (u, v) over a chunk of kRunFrames consecutive
// synchronized frames; warp = an 8(u) x 4(v) patch, block = 16 x 16 pixels.
// Consecutive frames of a sweep put a pixel into the same cell for several
// frames, so each thread keeps a run (cell, first frame, length <= kMaxRun)
// and only emits it when the cell changes.
//   count pass (frame_count_k): the FP64 pixel -> world -> f32 -> cell chain,
//     one u32 reduction per run into the cell histogram, and the run itself
//     stored as an 8 B record (cell | first frame, length, z-quarter bins of
//     its samples) in a lane-interleaved per-thread list;
//   fill pass (frame_fill_k): no FP64 -- each thread replays its run list;
//     lanes emitting runs of the same cell (image neighbours) are grouped with
//     MATCH, one returning atomic per group, slots = cell offset + cursor +
//     rank; the 64-bit key (insertion index, z bin, intensity read from the
//     frame) is written for every sample.  Slot order inside a cell is
//     irrelevant: the seal sorts every run by insertion key.
constexpr int kRunFrames = 64;
constexpr int kMaxRun = 8;  // bins of a run's samples fit 16 bits

// Sort keys: insertion index << kKeyShift | z bin << 8 | low byte (intensity for
// frames).  The z bin (z quarter of the cell, volume.cuh) rides in bits 8-9 so
// the seal need not recompute z; it sits below the index, so key order is
// insertion order.
constexpr int kKeyShift = 10;
// bucketed fill: 1024 cells per bucket, the cell within the bucket in key bits
// 42.. (insertion index << kKeyShift | bin << 8 | byte uses bits 0..41)
constexpr int kBucketShift = 10, kBucketCells = 1 << kBucketShift, kBucketTag = 42;
constexpr int kPlaceCap = 24 * 1024;  // keys of one bucket staged in shared memory (192 KB)


template <bool kInv>
__device__ __forceinline__ int32_t frame_cell32(const double* fa, double U, double V, const VoxelMap& m,
                                                float& z32, uint32_t& iz) {
  bool ok = true;
  uint32_t idx[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float p32 = __double2float_rn((U * fa[a] + V * fa[3 + a]) + fa[6 + a]);
    if (a == 2) z32 = p32;
    const double d = (double)p32 - m.origin[a];
    // 0 <= floor(q) < n  <=>  0 <= q < n (n integral; NaN fails both): no separate floor
    const double q = kInv ? d * m.inv_voxel : d / m.voxel;
    ok = ok && (q >= 0.0) && (q < (double)m.dims[a]);
    idx[a] = ok ? __double2uint_rz(q) : 0u;
  }
  iz = idx[2];
  return ok ? (int32_t)((idx[0] * (uint32_t)m.dims[1] + idx[1]) * (uint32_t)m.dims[2] + idx[2]) : -1;
}

// thread -> pixel of a 16 x 16 tile (warp = 8 x 4), shared by both passes
__device__ __forceinline__ void tile_pixel(const FrameView& fv, uint32_t& u, uint32_t& v) {
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t tiles_u = (fv.W + 15) / 16;
  u = (blockIdx.x % tiles_u) * 16 + (warp & 1) * 8 + (lane & 7);
  v = (blockIdx.x / tiles_u) * 16 + (warp >> 1) * 4 + (lane >> 3);
}

// Run record: x = cell, y = first frame in the chunk (6 bits) | length << 6 |
// z bins (2 bits per sample) << 10.  Lane-interleaved: run r of thread t of
// block b at runs[(b * kRunFrames + r) * 256 + t].
template <bool kInv>
__global__ void __launch_bounds__(256, 5) frame_count_k(FrameView fv, VoxelMap m, uint32_t* counts,
                                                      uint2* __restrict__ runs, uint8_t* __restrict__ nruns,
                                                      unsigned long long* rejected) {
  __shared__ double s_axes[kRunFrames * 9];
  uint32_t u, v;
  tile_pixel(fv, u, v);
  const uint32_t lane = lane_id();
  const uint32_t p = v * fv.W + u;
  const bool in_frame = u < fv.W && v < fv.H && (!fv.mask || fv.mask[p] != 0);
  const uint32_t f0 = blockIdx.y * kRunFrames;
  const int nf = (int)min((uint32_t)kRunFrames, fv.n_frames - f0);
  for (int i = threadIdx.x; i < nf * 9; i += blockDim.x) s_axes[i] = fv.axes[(size_t)f0 * 9 + i];
  __syncthreads();
  const size_t blk = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  uint2* my = runs + blk * kRunFrames * 256 + threadIdx.x;
  const size_t gb64 = fv.group_base(blockIdx.y);  // (direct mode: 64-bit counters)
  if (!fv.direct) counts += gb64;
  const double U = (double)u * fv.px, V = (double)v * fv.py;
  int32_t cur = -1;
  uint32_t run_j = 0, k = 0, bb = 0, nr = 0, n_oob = 0;
  float zb1 = 0.f, zb2 = 0.f, zb3 = 0.f;  // z-quarter bounds of the run's cell
  for (int j = 0; j < nf; ++j) {  // block-uniform trip count
    float z = 0.f;
    uint32_t iz = 0;
    // computed for every lane (no divergent branch), then masked
    const int32_t cell = frame_cell32<kInv>(s_axes + j * 9, U, V, m, z, iz);
    const int32_t lin = in_frame ? cell : -1;
    n_oob += (in_frame && cell < 0) ? 1u : 0u;
    const bool restart = lin != cur || k == (uint32_t)kMaxRun;
    if (restart && cur >= 0) {
      count_run(counts, gb64, fv.direct, (uint32_t)cur, k);
      my[(size_t)nr * 256] = make_uint2((uint32_t)cur, run_j | (k << 6) | (bb << 10));
      ++nr;
    }
    if (restart) {
      cur = lin;
      run_j = (uint32_t)j;
      k = 0;
      bb = 0;
      if (lin >= 0) {
        zb1 = zbin_bound(m.origin[2], m.voxel, iz, 1);
        zb2 = zbin_bound(m.origin[2], m.voxel, iz, 2);
        zb3 = zbin_bound(m.origin[2], m.voxel, iz, 3);
      }
    }
    if (lin >= 0) bb |= (uint32_t)((z >= zb1) + (z >= zb2) + (z >= zb3)) << (2 * k);
    ++k;
  }
  if (cur >= 0) {
    count_run(counts, gb64, fv.direct, (uint32_t)cur, k);
    my[(size_t)nr * 256] = make_uint2((uint32_t)cur, run_j | (k << 6) | (bb << 10));
    ++nr;
  }
  nruns[blk * 256 + threadIdx.x] = (uint8_t)nr;  // <= kRunFrames
  const unsigned oob = __reduce_add_sync(0xffffffffu, n_oob);  // one atomic per warp
  if (lane == 0 && oob) atomicAdd(rejected, (unsigned long long)oob);
}

// Count pass on the exact threshold tables (cells.cuh): per frame the pixel's
// world point P (the reference's FP64 chain, reconstruct.py:156-162) is
// compared with the [lo, hi) interval of its current cell per axis (z on the
// fine cell/quarter table, so the z bin comes with it); only a crossing walks
// the tables.  No f32 rounding, division or float->int conversion per frame.
// Consecutive frames with bit-identical axis columns R[:,0], R[:,1] (sweeps
// at a fixed probe orientation) reuse U*R[a,0] + V*R[a,1]: the same f64 value
// the reference computes, so P = that + t[a] is bit-identical.  Output (run
// records, histogram, out-of-bounds tally) is exactly frame_count_k's.
template <bool kBins>
__global__ void __launch_bounds__(256, 5) frame_count_tab_k(FrameView fv, CellTables ct, VoxelMap m,
                                                           uint32_t* counts, uint2* __restrict__ runs,
                                                           uint8_t* __restrict__ nruns,
                                                           unsigned long long* rejected) {
  __shared__ double s_axes[kRunFrames * 9];
  __shared__ uint32_t s_same[kRunFrames / 32];  // bit j: frame j reuses frame j-1's in-plane axes
  static_assert(kRunFrames == 64 && kRunFrames <= 256, "two ballot words from the first two warps");
  uint32_t u, v;
  tile_pixel(fv, u, v);
  const uint32_t lane = lane_id();
  const uint32_t p = v * fv.W + u;
  const bool in_frame = u < fv.W && v < fv.H && (!fv.mask || fv.mask[p] != 0);
  const uint32_t f0 = blockIdx.y * kRunFrames;
  const int nf = (int)min((uint32_t)kRunFrames, fv.n_frames - f0);
  for (int i = threadIdx.x; i < nf * 9; i += blockDim.x) s_axes[i] = fv.axes[(size_t)f0 * 9 + i];
  __syncthreads();
  if (threadIdx.x < kRunFrames) {  // warps 0 and 1: one ballot word each
    const int j = threadIdx.x;
    bool same = j > 0 && j < nf;
    for (int c = 0; c < 6 && same; ++c)
      same = __double_as_longlong(s_axes[j * 9 + c]) == __double_as_longlong(s_axes[(j - 1) * 9 + c]);
    const uint32_t word = __ballot_sync(0xffffffffu, same);
    if (lane == 0) s_same[j >> 5] = word;
  }
  __syncthreads();
  const unsigned long long same_bits = (unsigned long long)s_same[0] | ((unsigned long long)s_same[1] << 32);
  const size_t blk = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  uint2* my = runs + blk * kRunFrames * 256 + threadIdx.x;
  const size_t gb64 = fv.group_base(blockIdx.y);  // (direct mode: 64-bit counters)
  if (!fv.direct) counts += gb64;
  const double U = (double)u * fv.px, V = (double)v * fv.py;
  const uint32_t ny = (uint32_t)m.dims[1], nz = (uint32_t)m.dims[2];
  AxisCell ax[2];
  AxisCellZ az;
  double S[3];
  for (int a = 0; a < 2; ++a) {
    ax[a].g = -2;  // unknown: the first frame locates from a guess
    ax[a].lo = ax[a].hi = 0.0;
  }
  az.g = -2;
  az.lo = az.hi = az.q1 = az.q2 = az.q3 = 0.0;
  for (int a = 0; a < 3; ++a) S[a] = 0.0;
  const int nzc = ct.n[2] >> 2;  // cells along z (the fine table has 4 per cell)
  // the current frame's cell (-1 out of bounds), recomputed only on a crossing
  int32_t tracked = -1;
  int32_t cur = -1;
  uint32_t run_j = 0, k = 0, bb = 0, nr = 0, n_in = 0;
  for (int j = 0; j < nf; ++j) {  // block-uniform trip count and branches
    const double* fa = s_axes + j * 9;
    double P[3];
    if ((same_bits >> j) & 1ull) {
#pragma unroll
      for (int a = 0; a < 3; ++a) P[a] = S[a] + fa[6 + a];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        S[a] = U * fa[a] + V * fa[3 + a];
        P[a] = S[a] + fa[6 + a];
      }
    }
    const bool sx = axis_same(P[0], ax[0]), sy = axis_same(P[1], ax[1]);
    const bool sz = az.lo <= P[2] && P[2] < az.hi;
    if (!(sx & sy & sz)) {  // a crossing: relocate only the axes the point left
      if (!sx) {
        if (ax[0].g == -2) ax[0].g = axis_guess(P[0], m.origin[0], m.inv_voxel, ct.n[0], 0);
        axis_locate(P[0], ct.t[0], ct.n[0], ax[0]);
      }
      if (!sy) {
        if (ax[1].g == -2) ax[1].g = axis_guess(P[1], m.origin[1], m.inv_voxel, ct.n[1], 0);
        axis_locate(P[1], ct.t[1], ct.n[1], ax[1]);
      }
      if (!sz) {
        if (az.g == -2) az.g = axis_guess(P[2], m.origin[2], m.inv_voxel, nzc, 0);
        axis_locate_z(P[2], ct.t[2], nzc, az);
      }
      const bool ok = (unsigned)ax[0].g < (unsigned)ct.n[0] && (unsigned)ax[1].g < (unsigned)ct.n[1] &&
                      (unsigned)az.g < (unsigned)nzc;
      tracked = ok ? (int32_t)(((uint32_t)ax[0].g * ny + (uint32_t)ax[1].g) * nz + (uint32_t)az.g) : -1;
    }
    const int32_t lin = in_frame ? tracked : -1;
    const bool restart = lin != cur || k == (uint32_t)kMaxRun;
    if (restart && cur >= 0) {
      DARE_CHECK(nr < (uint32_t)kRunFrames && (uint32_t)cur < fv.ncells);
      count_run(counts, gb64, fv.direct, (uint32_t)cur, k);
      my[(size_t)nr * 256] = make_uint2((uint32_t)cur, run_j | (k << 6) | (bb << 10));
      ++nr;
      n_in += k;
    }
    if (restart) {
      cur = lin;
      run_j = (uint32_t)j;
      k = 0;
      bb = 0;
    }
    if constexpr (kBins) bb |= az.bin(P[2]) << (2 * k);  // (garbage for out-of-bounds runs: never stored)
    ++k;
  }
  if (cur >= 0) {
    count_run(counts, gb64, fv.direct, (uint32_t)cur, k);
    my[(size_t)nr * 256] = make_uint2((uint32_t)cur, run_j | (k << 6) | (bb << 10));
    ++nr;
    n_in += k;
  }
  // out-of-bounds samples = the frames of in-frame pixels not in a kept run
  const uint32_t n_oob = in_frame ? (uint32_t)nf - n_in : 0u;
  nruns[blk * 256 + threadIdx.x] = (uint8_t)nr;  // <= kRunFrames
  const unsigned oob = __reduce_add_sync(0xffffffffu, n_oob);  // one atomic per warp
  if (lane == 0 && oob) atomicAdd(rejected, (unsigned long long)oob);
}

// Fill pass over the chunks [chunk_begin, chunk_begin + gridDim.y): replays
// each thread's runs (see frame_count_k); no pixel geometry is recomputed.
// Key = u64: insertion index << kKeyShift | z bin << 8 | intensity.  Key = u32
// (when the packed (frame, v, u) index and the 2-bit z bin fit 32 bits):
// insertion index << 2 | z bin -- half the key traffic; the seal then reads
// the intensity from the frame.
template <class Key>
__global__ void __launch_bounds__(256) frame_fill_k(FrameView fv, uint32_t chunk_begin,
                                                    const uint2* __restrict__ runs,
                                                    const uint8_t* __restrict__ nruns, uint32_t* counts,
                                                    const uint32_t* __restrict__ offsets,
                                                    Key* keys) {
  constexpr bool kWide = sizeof(Key) == 8;
  __shared__ uint32_t s_img[kRunFrames];
  uint32_t u, v;
  tile_pixel(fv, u, v);
  const unsigned lane = lane_id(), lt = (1u << lane) - 1u;
  const uint32_t p = v * fv.W + u, pk = fv.pixel_key(u, v);
  const uint32_t chunk = chunk_begin + blockIdx.y, f0 = chunk * kRunFrames;
  const int nf = (int)min((uint32_t)kRunFrames, fv.n_frames - f0);
  for (int i = threadIdx.x; i < nf; i += blockDim.x) s_img[i] = (uint32_t)fv.image[f0 + i];
  __syncthreads();
  const size_t blk = (size_t)chunk * gridDim.x + blockIdx.x;
  const uint2* my = runs + blk * kRunFrames * 256 + threadIdx.x;
  const uint32_t nr = nruns[blk * 256 + threadIdx.x];
  const size_t gb = fv.group_base(chunk);
  counts += gb;  // 32-bit cursors per (group, cell) in both group modes
  if (!fv.direct) offsets += gb;  // group-major key CSR (mode 1); mode 2 writes cell-major
  const uint32_t max_nr = __reduce_max_sync(0xffffffffu, nr);
  uint2 next = nr > 0 ? my[0] : make_uint2(0u, 0u);
  for (uint32_t r = 0; r < max_nr; ++r) {
    const bool need = r < nr;
    const uint2 run = next;
    if (r + 1 < nr) next = my[(size_t)(r + 1) * 256];  // one run ahead
    const uint32_t lin = run.x, run_j = run.y & 63u, k = (run.y >> 6) & 15u, bb = run.y >> 10;
    // intensities first: their latency overlaps the grouping and the atomic
    uint32_t inten[kMaxRun];
#pragma unroll
    for (int t = 0; t < kMaxRun; ++t)
      inten[t] = (kWide && need && (uint32_t)t < k) ? fv.frames[(size_t)s_img[run_j + t] * fv.hw + p] : 0u;
    uint32_t pre_w = 0;
    if (fv.direct && need) pre_w = fv.pre[gb + lin];
    const bool solo = (pre_w >> 31) != 0;  // the only run of its (group, cell): slot known, no atomic
    // bucketed: slots per bucket (absolute cursors), grouping by bucket
    const bool bk = kWide && fv.bucketed;
    const uint32_t gkey = bk ? lin >> kBucketShift : lin;
    const uint32_t cell_off = (need && !bk) ? offsets[lin] + (pre_w & 0x7fffffffu) : 0u;  // early: overlaps the atomic
    // lanes not emitting (or solo) get a key no cell has, so MATCH runs on the full warp
    const unsigned peers = __match_any_sync(0xffffffffu, (need && !solo) ? gkey : (0x80000000u | lane));
    // Groups whose runs cover the same frames (the common case: image
    // neighbours crossing a cell together) take their slots frame-major --
    // (frame, pixel) = insertion order -- so the seal's sort finds them presorted.
    const unsigned leader = __ffs(peers) - 1;
    const uint32_t fk = (run_j << 4) | k;
    const uint32_t leader_fk = __shfl_sync(0xffffffffu, fk, leader);  // all lanes (full mask)
    const unsigned diff = __ballot_sync(0xffffffffu, need && leader_fk != fk);
    const bool uniform = (diff & peers) == 0u;
    unsigned total = __popc(peers) * k, prefix = 0;
    if (diff != 0u) {  // some group mixes run shapes: slots by a bit-sliced prefix of the lengths
      total = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {  // k <= kMaxRun < 16
        const unsigned mb = __ballot_sync(0xffffffffu, need && ((k >> b) & 1u)) & peers;
        total += (unsigned)__popc(mb) << b;
        prefix += (unsigned)__popc(mb & lt) << b;
      }
    }
    unsigned base = 0;
    if (need && !solo && lane == leader) {
      if (bk) {
        base = atomicAdd(&counts[gkey], total);
      } else if (fv.byte_cursors) {
        const uint32_t sh = 8u * (lin & 3u);
        base = (atomicAdd(&counts[lin >> 2], total << sh) >> sh) & 0xffu;
      } else {
        base = atomicAdd(&counts[lin], total);
      }
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (need) {
      const unsigned n = __popc(peers), rank = __popc(peers & lt);
      const uint32_t stride = uniform ? n : 1u;
      DARE_CHECK(fv.direct || bk || base + total <= offsets[lin + 1] - cell_off);
      DARE_CHECK(!bk || base + total <= offsets[min((gkey + 1) << kBucketShift, fv.ncells)]);
      Key* dst = keys + cell_off + base + (uniform ? rank : prefix);
      if constexpr (kWide) {
        const unsigned long long key0 = (((unsigned long long)((f0 + run_j) * fv.fstride + pk)) << kKeyShift) |
                                        (bk ? (unsigned long long)(lin & (kBucketCells - 1)) << kBucketTag : 0ull);
        const unsigned long long kstep = (unsigned long long)fv.fstride << kKeyShift;
#pragma unroll
        for (int t = 0; t < kMaxRun; ++t) {
          if ((uint32_t)t < k) {
            *dst = key0 + (unsigned long long)t * kstep + (((bb >> (2 * t)) & 3u) << 8) + inten[t];
            dst += stride;
          }
        }
      } else {
        const uint32_t key0 = ((f0 + run_j) * fv.fstride + pk) << 2;
#pragma unroll
        for (int t = 0; t < kMaxRun; ++t) {
          if ((uint32_t)t < k) {
            *dst = key0 + ((uint32_t)t * fv.fstride << 2) + ((bb >> (2 * t)) & 3u);
            dst += stride;
          }
        }
      }
    }
  }
}

// Arbitrary samples (VolumeBuilder.seal, volume.py:240-269): key = sample index
// << kKeyShift (no z bin: the seal computes it from the positions).
template <bool kFill>
__global__ void __launch_bounds__(256) sample_scatter_k(const float* __restrict__ pos, int64_t n,
                                                        VoxelMap m, uint32_t* counts,
                                                        const uint32_t* __restrict__ offsets,
                                                        unsigned long long* keys,
                                                        unsigned long long* rejected) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  int32_t lin = -1;
  if (valid) {
    bool ok = true;
    uint32_t idx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double f = floor(voxel_coord(m, a, pos[3 * i + a]));
      ok = ok && (f >= 0.0) && (f < (double)m.dims[a]);
      idx[a] = ok ? (uint32_t)f : 0u;
    }
    if (ok) lin = (int32_t)((idx[0] * (uint32_t)m.dims[1] + idx[1]) * (uint32_t)m.dims[2] + idx[2]);
  }
  const bool kept = lin >= 0;
  if (!kFill) {
    const int oob = __syncthreads_count(valid && !kept);
    if (threadIdx.x == 0 && oob) atomicAdd(rejected, (unsigned long long)oob);
  }
  warp_scatter<kFill>(kept, lin, (unsigned long long)i << kKeyShift, counts, offsets, keys);
}

// Seal-side frame table (96 B per frame, 32 B aligned): the axis pairs
// (R[a][0], R[a][1]) and t in two 256-bit loads, t[2] + orientation id in one
// 128-bit load -- 3 loads per record instead of 10 (the seal is bound by L1
// wavefronts on these lookups).
struct __align__(32) SealAxes {
  double r0x, r0y, r1x, r1y;  // load A
  double r2x, r2y, t0, t1;    // load B
  double t2;                  // load C: t2 | oid | image
  uint32_t oid, image;
  double pad2[2];
};
static_assert(sizeof(SealAxes) == 96, "SealAxes layout");

__global__ void seal_axes_k(const double* __restrict__ axes, const uint32_t* __restrict__ oid,
                            const int32_t* __restrict__ image, uint32_t n, SealAxes* out) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const double* fa = axes + (size_t)f * 9;
  SealAxes x;
  x.r0x = fa[0];
  x.r0y = fa[3];
  x.r1x = fa[1];
  x.r1y = fa[4];
  x.r2x = fa[2];
  x.r2y = fa[5];
  x.t0 = fa[6];
  x.t1 = fa[7];
  x.t2 = fa[8];
  x.oid = oid[f];
  x.image = (uint32_t)image[f];
  x.pad2[0] = x.pad2[1] = 0.0;
  out[f] = x;
}

__device__ __forceinline__ void ld256_f64(const void* p, double& a, double& b, double& c, double& d) {
  uint32_t w[8];
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
      : "l"(p));
  a = __hiloint2double((int)w[1], (int)w[0]);
  b = __hiloint2double((int)w[3], (int)w[2]);
  c = __hiloint2double((int)w[5], (int)w[4]);
  d = __hiloint2double((int)w[7], (int)w[6]);
}

struct FrameRecords {
  using Key = unsigned long long;
  static constexpr bool kKeyBins = true;  // z bins computed by the fill pass
  __device__ static uint32_t key_pid(Key k) { return (uint32_t)(k >> kKeyShift); }
  __device__ static uint32_t key_bin(Key k) { return (uint32_t)(k >> 8) & 3u; }
  __device__ static uint32_t key_byte(Key k) { return (uint32_t)(k & 0xffu); }
  FrameView fv;
  const SealAxes* sa;
  __device__ __forceinline__ uint4 operator()(uint32_t pid, uint32_t inten) const {
    uint32_t f, u, v;
    fv.decode(pid, f, u, v);
    const SealAxes* x = sa + f;
    double r0x, r0y, r1x, r1y, r2x, r2y, t0, t1;
    ld256_f64(&x->r0x, r0x, r0y, r1x, r1y);
    ld256_f64(&x->r2x, r2x, r2y, t0, t1);
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(&x->t2));
    const double t2 = __hiloint2double((int)c.y, (int)c.x);
    const double U = (double)u * fv.px, V = (double)v * fv.py;
    // reconstruct.py:156-162: ((U*R[a,0]) + (V*R[a,1])) + t[a]
    const float p0 = __double2float_rn((U * r0x + V * r0y) + t0);
    const float p1 = __double2float_rn((U * r1x + V * r1y) + t1);
    const float p2 = __double2float_rn((U * r2x + V * r2y) + t2);
    return make_uint4(__float_as_uint(p0), __float_as_uint(p1), __float_as_uint(p2),
                      (c.z << 8) | inten);
  }
  // z only (the binning key), same arithmetic as operator()
  __device__ __forceinline__ float z_of(uint32_t pid) const {
    uint32_t f, u, v;
    fv.decode(pid, f, u, v);
    const SealAxes& x = sa[f];
    const double U = (double)u * fv.px, V = (double)v * fv.py;
    return __double2float_rn((U * x.r2x + V * x.r2y) + x.t2);
  }
};

// 32-bit keys (insertion index only): the intensity is read from the frame
// (the seal visits cells z-chunk-major, so the frames of the concurrently
// sealed cells are a small L2-resident band) and z is binned from the
// recomputed position.
struct FrameRecords32 {
  using Key = uint32_t;
  static constexpr bool kKeyBins = true;  // key = insertion index << 2 | z bin
  __device__ static uint32_t key_pid(Key k) { return k >> 2; }
  __device__ static uint32_t key_bin(Key k) { return k & 3u; }
  __device__ static uint32_t key_byte(Key) { return 0u; }
  FrameView fv;
  const SealAxes* sa;
  __device__ __forceinline__ uint4 operator()(uint32_t pid, uint32_t) const {
    uint32_t f, u, v;
    fv.decode(pid, f, u, v);
    const SealAxes* x = sa + f;
    double r0x, r0y, r1x, r1y, r2x, r2y, t0, t1;
    ld256_f64(&x->r0x, r0x, r0y, r1x, r1y);
    ld256_f64(&x->r2x, r2x, r2y, t0, t1);
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(&x->t2));
    const uint32_t inten = __ldg(fv.frames + (size_t)c.w * fv.hw + v * fv.W + u);
    const double t2 = __hiloint2double((int)c.y, (int)c.x);
    const double U = (double)u * fv.px, V = (double)v * fv.py;
    // reconstruct.py:156-162: ((U*R[a,0]) + (V*R[a,1])) + t[a]
    const float p0 = __double2float_rn((U * r0x + V * r0y) + t0);
    const float p1 = __double2float_rn((U * r1x + V * r1y) + t1);
    const float p2 = __double2float_rn((U * r2x + V * r2y) + t2);
    return make_uint4(__float_as_uint(p0), __float_as_uint(p1), __float_as_uint(p2), (c.z << 8) | inten);
  }
  __device__ __forceinline__ float z_of(uint32_t pid) const {
    uint32_t f, u, v;
    fv.decode(pid, f, u, v);
    const SealAxes& x = sa[f];
    const double U = (double)u * fv.px, V = (double)v * fv.py;
    return __double2float_rn((U * x.r2x + V * x.r2y) + x.t2);
  }
};

struct SampleRecords {
  using Key = unsigned long long;
  static constexpr bool kKeyBins = false;
  __device__ static uint32_t key_pid(Key k) { return (uint32_t)(k >> kKeyShift); }
  __device__ static uint32_t key_bin(Key) { return 0u; }
  __device__ static uint32_t key_byte(Key k) { return (uint32_t)(k & 0xffu); }
  const float* pos;
  const uint32_t* word;  // (oid << 8) | intensity
  __device__ __forceinline__ uint4 operator()(uint32_t pid, uint32_t) const {
    const size_t i = (size_t)pid;
    return make_uint4(__float_as_uint(pos[3 * i]), __float_as_uint(pos[3 * i + 1]),
                      __float_as_uint(pos[3 * i + 2]), word[i]);
  }
  __device__ __forceinline__ float z_of(uint32_t pid) const { return pos[3 * (size_t)pid + 2]; }
};

constexpr int kSmallRun = 32;  // longest per-cell run sorted in shared memory by one lane
constexpr int kSealWarps = 4;  // warps per seal block
// Stage slot of the j-th key of the warp's cell `col`: rows of 32 with an XOR
// swizzle.  Lane-per-cell loops (fixed j) touch a permutation of a row; the
// key-per-lane passes (consecutive keys: runs of j within a cell, then the
// next cell) hit distinct banks within a cell (2j mod 32 over <= 16 j) and
// between neighbouring cells (col ^ 2j keeps col's parity).
__device__ __forceinline__ uint32_t stage_at(uint32_t j, uint32_t col) { return j * 32u + (col ^ ((2u * j) & 31u)); }

// kRun = the longest run the stage holds (16 or 32): the host picks 16 when no
// cell has more samples (half the shared memory: 10 instead of 7 blocks/SM)
template <int kRun>
struct SealSmem {
  uint32_t st[kRun * 32];  // st[stage_at(k, lane)] = k-th insertion index of cell c0+lane
  uint16_t sx[kRun * 32];  // its low key byte | z bin << 8, later | destination << 8
  uint16_t pos_of[kRun * 32];  // key position -> (index in its cell) << 5 | lane of its cell
  float zb[3][32];             // z-quarter boundaries of each lane's cell (SampleRecords)
};

// z-quarter binning of the sealed runs (layout in volume.cuh)
struct BinOut {
  double oz, voxel;
  int64_t nz;
  uint32_t* bins;
  int8_t* perm;
};

// Warp seals cells [c0, c0+32).  Keys are loaded coalesced into a transposed,
// padded stage (cell = column), each lane insertion-sorts its column (runs are
// ~16 keys; the padded pitch makes the lanes' row accesses bank-conflict
// free) -- that is the reference's insertion order.  The cell is then stored
// grouped by z quarter (volume.cuh): z bins computed coalesced, a lane per
// cell turns them into stable destinations + the bins word, and the records
// are written back coalesced with perm.  Runs longer than kSmallRun are listed
// for the CUB segmented-sort path; they, and the small runs of a warp that
// has one, stay in insertion order (bins 0, perm 0).
// Bulk prefetch of a warp's key segment (kBulk): one elected lane issues a
// cp.async.bulk (TMA engine, SASS UBLKCP) of the whole 16 B-aligned segment
// into shared memory, completing on a per-warp mbarrier, while the warp lays
// out its cells; the staging pass then reads the keys from shared memory --
// every key load is in flight at once instead of four per lane per round.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <class Rec, int kRun, bool kBulk>
__global__ void __launch_bounds__(kSealWarps * 32, kRun <= 16 ? (kBulk ? 6 : 10) : 1) seal_k(Rec rec,
                                                          const uint32_t* __restrict__ offsets,
                                                          const typename Rec::Key* __restrict__ keys,
                                                          uint32_t ncells, uint4* records,
                                                          uint32_t* big_cells, uint32_t* n_big,
                                                          BinOut bo) {
  using Key = typename Rec::Key;
  constexpr int kRaw = kBulk ? kRun * 32 * (int)sizeof(Key) + 16 : 16;
  __shared__ SealSmem<kRun> smem[kSealWarps];
  __shared__ __align__(16) unsigned char kraw[kSealWarps][kRaw];
  __shared__ __align__(8) unsigned long long kbar[kSealWarps];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  SealSmem<kRun>& sm = smem[warp];
  // warp -> 32 consecutive cells of one column, z-chunk-major across warps:
  // concurrently resident warps cover the same z range of many columns, so a
  // z sweep's records come from the same few frames (L1-resident axes)
  const uint32_t nz = (uint32_t)bo.nz, zchunks = (nz + 31u) / 32u, ncols = ncells / nz;
  const uint32_t g = blockIdx.x * kSealWarps + warp;
  const uint32_t zc = g / ncols, col = g - zc * ncols;
  if (zc >= zchunks) return;
  const uint32_t c0 = col * nz + zc * 32u;
  const uint32_t c = c0 + lane;
  const uint32_t c_end = min(c0 + 32u, col * nz + nz);
  const uint32_t s0 = offsets[c0], s1 = offsets[c_end];
  uint32_t cs = 0, cn = 0;
  if (c < c_end) {
    cs = offsets[c];
    cn = offsets[c + 1] - cs;
  }
  const bool big = cn > kRun;
  if (big) big_cells[atomicAdd(n_big, 1u)] = c;
  const uint32_t len = s1 - s0;
  const bool staged = !__any_sync(0xffffffffu, big);  // then len <= 32 * 32
  DARE_CHECK(!staged || len <= (uint32_t)kRun * 32u);
  uint32_t kshift = 0;  // keys of the segment start at kbuf[kshift] (16 B alignment of the copy)
  if (kBulk && staged && len > 0) {
    const uint32_t mb = smem_u32(&kbar[warp]);
    const uintptr_t a = (uintptr_t)(keys + s0), a0 = a & ~(uintptr_t)15;
    kshift = (uint32_t)((a - a0) / sizeof(Key));
    const uint32_t bytes = (uint32_t)(((a - a0) + (uintptr_t)len * sizeof(Key) + 15) & ~(uintptr_t)15);
    DARE_CHECK(bytes <= (uint32_t)kRaw);
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(kraw[warp])),
          "l"(a0), "r"(bytes), "r"(mb)
          : "memory");
    }
    __syncwarp();
  }
  if (staged) {
    for (uint32_t k = 0; k < cn; ++k) sm.pos_of[cs - s0 + k] = (uint16_t)((k << 5) | lane);
    if constexpr (!Rec::kKeyBins) {
      const int64_t iz = (int64_t)c % bo.nz;
#pragma unroll
      for (int q = 0; q < 3; ++q) sm.zb[q][lane] = zbin_bound(bo.oz, bo.voxel, iz, q + 1);
    }
    __syncwarp();
    if (kBulk && len > 0) {  // the segment has landed in shared memory
      const uint32_t mb = smem_u32(&kbar[warp]);
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(mb)
            : "memory");
    }
    const Key* kbuf = reinterpret_cast<const Key*>(kraw[warp]) + kshift;
    // keys staged as u32 index + u16 (byte | z bin << 8): smaller stage, more
    // warps.  Four loads in flight per lane (from shared memory after the bulk
    // prefetch); global keys are read once (streaming, L1 kept for the
    // frame-axes lookups of the record pass)
    for (uint32_t i0 = 0; i0 < len; i0 += 128) {
      Key kk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t i = i0 + 32u * q + lane;
        kk[q] = i < len ? (kBulk ? kbuf[i] : __ldcs(keys + s0 + i)) : (Key)0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t i = i0 + 32u * q + lane;
        if (i < len) {
          const uint32_t pw = sm.pos_of[i], col = pw & 31u;
          const uint32_t at = stage_at(pw >> 5, col);
          const uint32_t pid = Rec::key_pid(kk[q]);
          uint32_t bin;
          if constexpr (Rec::kKeyBins) {
            bin = Rec::key_bin(kk[q]);
          } else {
            const float z = rec.z_of(pid);
            bin = (z >= sm.zb[0][col]) + (z >= sm.zb[1][col]) + (z >= sm.zb[2][col]);
          }
          sm.st[at] = pid;
          sm.sx[at] = (uint16_t)(Rec::key_byte(kk[q]) | (bin << 8));
        }
      }
    }
    __syncwarp();
    // by insertion index (unique); byte and bin move along.  `top` = the
    // largest key so far: presorted runs (frame-major fill) cost one load each
    uint32_t top = cn ? sm.st[lane] : 0u;
    for (uint32_t i = 1; i < cn; ++i) {
      const uint32_t x = sm.st[stage_at(i, lane)];
      if (x > top) {
        top = x;
        continue;
      }
      const uint16_t xs = sm.sx[stage_at(i, lane)];
      uint32_t j = i;
      uint32_t y = top;  // st[j - 1] for j = i
      do {
        sm.st[stage_at(j, lane)] = y;
        sm.sx[stage_at(j, lane)] = sm.sx[stage_at(j - 1, lane)];
        --j;
      } while (j > 0 && (y = sm.st[stage_at(j - 1, lane)]) > x);
      sm.st[stage_at(j, lane)] = x;
      sm.sx[stage_at(j, lane)] = xs;
    }
    if (c < c_end) {  // lane = cell: stable destinations by bin, bins word
      // per-bin counters packed as bytes (runs <= 32): registers, not local memory
      uint32_t n = 0;
      for (uint32_t j = 0; j < cn; ++j) n += 1u << (8u * (sm.sx[stage_at(j, lane)] >> 8));
      const uint32_t c1 = n & 0xffu, c2 = c1 + ((n >> 8) & 0xffu), c3 = c2 + ((n >> 16) & 0xffu);
      uint32_t next = (c1 << 8) | (c2 << 16) | (c3 << 24);  // byte b = first slot of bin b
      for (uint32_t j = 0; j < cn; ++j) {
        const uint32_t w = sm.sx[stage_at(j, lane)], sh = 8u * (w >> 8);
        sm.sx[stage_at(j, lane)] = (uint16_t)((w & 0xffu) | (((next >> sh) & 0xffu) << 8));
        next += 1u << sh;
      }
      bo.bins[c] = c1 | (c2 << 8) | (c3 << 16) | (1u << 24);
    }
    __syncwarp();
    for (uint32_t i = lane; i < len; i += 32) {
      const uint32_t pw = sm.pos_of[i], col = pw & 31u, j = pw >> 5;
      const uint32_t w = sm.sx[stage_at(j, col)], dest = w >> 8;
      DARE_CHECK(j < (uint32_t)kRun && dest < (uint32_t)kRun && s0 + i - j + dest < s1);
      records[s0 + i - j + dest] = rec(sm.st[stage_at(j, col)], w & 0xffu);
      bo.perm[s0 + i] = (int8_t)((int)dest - (int)j);
    }
  } else if (cn > 0 && !big) {
    // a big run in this warp's chunk: the small runs are sealed lane by lane
    typename Rec::Key k[kRun];
    for (uint32_t i = 0; i < cn; ++i) {
      const typename Rec::Key x = keys[cs + i];
      uint32_t j = i;
      while (j > 0 && k[j - 1] > x) {
        k[j] = k[j - 1];
        --j;
      }
      k[j] = x;
    }
    for (uint32_t i = 0; i < cn; ++i) {
      records[cs + i] = rec(Rec::key_pid(k[i]), Rec::key_byte(k[i]));
      bo.perm[cs + i] = 0;
    }
  }
  if (!staged && c < c_end) {  // insertion order kept (big runs: sorted by the CUB path)
    bo.bins[c] = 0;
    if (big)
      for (uint32_t i = 0; i < cn; ++i) bo.perm[cs + i] = 0;
  }
}

__global__ void big_bounds_k(const uint32_t* big_cells, uint32_t n_big,
                             const uint32_t* __restrict__ offsets, uint32_t* begins,
                             uint32_t* ends) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_big) return;
  uint32_t c = big_cells[i];
  begins[i] = offsets[c];
  ends[i] = offsets[c + 1];
}

// block per big cell: records from the segment-sorted keys
template <class Rec>
__global__ void big_materialize_k(Rec rec, const uint32_t* begins, const uint32_t* ends,
                                  const typename Rec::Key* __restrict__ sorted, uint4* records) {
  uint32_t b = begins[blockIdx.x], e = ends[blockIdx.x];
  for (uint32_t s = b + threadIdx.x; s < e; s += blockDim.x)
    records[s] = rec(Rec::key_pid(sorted[s]), Rec::key_byte(sorted[s]));
}

// Frame-grouped keys (groups > 1): the count / fill passes keep one CSR of
// keys per group of frames (group-major: koff[g * ncells + c]), so that the
// fill of a group -- a contiguous frame range, typically one sweep direction
// -- writes each cell's keys in one visit, into memory its neighbouring cells'
// keys share; with one CSR for every frame, multi-direction sweeps (cfg3: four
// sweeps) visit each cell's 32 B of keys four times far apart in time and L2
// merges the partial sectors in DRAM (67 GB of traffic for 16.8 GB of keys).
// The regroup pass then lays the keys out cell-major for the seal: warp per 32
// consecutive cells, per group one coalesced segment read, written into the
// cells' final ranges (a contiguous window per warp, fully written at once).
__global__ void group_totals_k(const uint32_t* __restrict__ koff, uint32_t ncells, uint32_t groups,
                               uint32_t* totals) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  uint32_t t = 0;
  for (uint32_t g = 0; g < groups; ++g) {
    const size_t i = (size_t)g * ncells + c;
    t += koff[i + 1] - koff[i];
  }
  totals[c] = t;
}

// Direct mode: per cell, the samples of earlier groups (its runs of group g
// start there, after offsets[c]) with bit 31 set when group g holds exactly
// one run of the cell, and the cell's total.
__global__ void direct_pre_k(const unsigned long long* __restrict__ cnt64, uint32_t ncells, uint32_t groups,
                             uint32_t* pre, uint32_t* totals) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  uint32_t acc = 0;
  for (uint32_t g = 0; g < groups; ++g) {
    const size_t i = (size_t)g * ncells + c;
    const unsigned long long v = cnt64[i];
    pre[i] = acc | ((uint32_t)(v >> 32) == 1u ? 0x80000000u : 0u);
    acc += (uint32_t)v;
  }
  totals[c] = acc;
}

template <class Key>
__global__ void __launch_bounds__(256) regroup_keys_k(const uint32_t* __restrict__ koff,
                                                      const uint32_t* __restrict__ offsets, uint32_t ncells,
                                                      uint32_t groups, const Key* __restrict__ in, Key* out) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
  const uint32_t c0 = warp * 32u;
  if (c0 >= ncells) return;  // warp-uniform
  const uint32_t c = c0 + lane, c_end = min(c0 + 32u, ncells);
  uint32_t dst = c < c_end ? offsets[c] : 0u;  // this lane's cell: next free output slot
  for (uint32_t g = 0; g < groups; ++g) {
    const size_t base = (size_t)g * ncells;
    const uint32_t seg0 = koff[base + c0], seg1 = koff[base + c_end];
    const uint32_t my0 = c < c_end ? koff[base + c] : seg1;
    const uint32_t my1 = c < c_end ? koff[base + c + 1] : seg1;
    for (uint32_t i0 = seg0; i0 < seg1; i0 += 32) {  // warp-uniform trip count
      const uint32_t i = i0 + lane;
      // owner of key i: the last lane whose cell starts at or before i
      int lo = 0, hi = 31;
#pragma unroll
      for (int st = 0; st < 5; ++st) {
        const int mid = (lo + hi + 1) >> 1;
        const uint32_t m0 = __shfl_sync(0xffffffffu, my0, mid);
        if (m0 <= i) lo = mid;
        else hi = mid - 1;
      }
      const uint32_t o_start = __shfl_sync(0xffffffffu, my0, lo);
      const uint32_t o_dst = __shfl_sync(0xffffffffu, dst, lo);
      DARE_CHECK(i >= seg1 || (i >= o_start && o_dst + (i - o_start) < offsets[c_end]));
      if (i < seg1) out[o_dst + (i - o_start)] = __ldcs(in + i);
    }
    dst += my1 - my0;
  }
}

// Bucketed fill, placement: CTA per bucket of kBucketCells cells.  The bucket's
// keys (tagged with their cell within the bucket) occupy exactly the bucket's
// key range; they are placed into their cells through shared memory and the
// range is written back in place, coalesced -- no partially written 32 B
// sectors reach DRAM, unlike a fill that scatters each run straight into its
// cell (cfg3: one lone pixel per cell and sweep).
__global__ void __launch_bounds__(1024) bucket_place_k(const uint32_t* __restrict__ offsets, int64_t ncells,
                                                       unsigned long long* keys) {
  extern __shared__ unsigned long long sreg[];  // kPlaceCap
  __shared__ uint32_t scur[kBucketCells];
  const int64_t c0 = (int64_t)blockIdx.x << kBucketShift;
  const int64_t c1 = min(c0 + (int64_t)kBucketCells, ncells);
  const uint32_t r0 = offsets[c0], n = offsets[c1] - r0;
  DARE_CHECK(n <= (uint32_t)kPlaceCap);
  for (int c = threadIdx.x; c < kBucketCells; c += blockDim.x) scur[c] = c0 + c < c1 ? offsets[c0 + c] - r0 : 0u;
  __syncthreads();
  // four loads in flight per thread, then their placements
  for (uint32_t i0 = threadIdx.x; i0 < n; i0 += 4 * blockDim.x) {
    unsigned long long e[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t i = i0 + q * blockDim.x;
      e[q] = i < n ? __ldcs(keys + r0 + i) : ~0ull;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (e[q] != ~0ull) {
        const uint32_t slot = atomicAdd(&scur[(uint32_t)(e[q] >> kBucketTag)], 1u);
        DARE_CHECK(slot < n);
        sreg[slot] = e[q] & ((1ull << kBucketTag) - 1ull);
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) keys[r0 + i] = sreg[i];
}

// Bucket cursors (the key offset of each bucket's first cell) and the largest bucket.
__global__ void bucket_init_k(const uint32_t* __restrict__ offsets, int64_t ncells, int64_t nb, uint32_t* cursors,
                              uint32_t* max_bucket) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int64_t c0 = b << kBucketShift, c1 = min(c0 + (int64_t)kBucketCells, ncells);
  cursors[b] = offsets[c0];
  atomicMax(max_bucket, offsets[c1] - offsets[c0]);
}

// count -> scan -> fill -> seal, shared by frames and arbitrary samples.
// `scatter(fill, counts, offsets, keys, rejected)` launches the source's pass.
template <class Rec, class Scatter>
void build_csr(dare_volume_s* vol, Rec rec, Scatter scatter, cudaStream_t s, int seal_carveout = -1,
               uint32_t groups = 1, uint32_t* direct_pre = nullptr, bool byte_ok = false,
               bool bucket_ok = false) {
  const int64_t ncells = vol->ncells;
  const int64_t nkc = ncells * (int64_t)groups;  // per-group counters (groups > 1: frame-grouped keys)
  DARE_LIMIT(nkc < (int64_t)UINT32_MAX, "too many cells x frame groups");
  const bool direct = direct_pre != nullptr;  // group mode 2 (64-bit counters, solo runs placed directly)
  PhaseTimer pt(s, "build_csr");
  const int64_t ncount = direct ? 2 * nkc : nkc + 1;
  Scratch<uint32_t> counts(ncount, s);
  Scratch<unsigned long long> rej(1, s);
  DARE_CUDA(cudaMemsetAsync(counts.ptr, 0, sizeof(uint32_t) * ncount, s));
  DARE_CUDA(cudaMemsetAsync(rej.ptr, 0, sizeof(unsigned long long), s));
  dev_alloc(&vol->d_offsets, sizeof(uint32_t) * (ncells + 1));
  Scratch<uint32_t> koff(groups > 1 && !direct ? nkc + 1 : 0, s);
  Scratch<uint32_t> totals(groups > 1 ? ncells + 1 : 0, s);
  pt.mark("alloc+memset");
  using Key = typename Rec::Key;
  scatter(false, counts.ptr, (const uint32_t*)nullptr, (void*)nullptr, rej.ptr, false, false);
  DARE_CUDA(cudaGetLastError());
  pt.mark("count");
  size_t tmp_bytes = 0, max_bytes = 0, tmp2_bytes = 0;
  Scratch<uint32_t> max_d(1, s);
  // per-cell totals: the counters themselves (one group) or their sum over groups
  uint32_t* tot = counts.ptr;
  if (direct) {
    direct_pre_k<<<ceil_div(ncells, 256), 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(counts.ptr),
                                                       (uint32_t)ncells, groups, direct_pre, totals.ptr);
    DARE_CUDA(cudaGetLastError());
    DARE_CUDA(cudaMemsetAsync(totals.ptr + ncells, 0, sizeof(uint32_t), s));
    tot = totals.ptr;
  } else if (groups > 1) {
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2_bytes, counts.ptr, koff.ptr, nkc + 1, s));
    Scratch<uint8_t> tmp(tmp2_bytes, s);
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp2_bytes, counts.ptr, koff.ptr, nkc + 1, s));
    group_totals_k<<<ceil_div(ncells, 256), 256, 0, s>>>(koff.ptr, (uint32_t)ncells, groups, totals.ptr);
    DARE_CUDA(cudaGetLastError());
    DARE_CUDA(cudaMemsetAsync(totals.ptr + ncells, 0, sizeof(uint32_t), s));
    tot = totals.ptr;
  }
  DARE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, tot, vol->d_offsets, ncells + 1, s));
  DARE_CUDA(cub::DeviceReduce::Max(nullptr, max_bytes, tot, max_d.ptr, ncells, s));
  {
    Scratch<uint8_t> tmp(std::max(tmp_bytes, max_bytes), s);
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, tot, vol->d_offsets, ncells + 1, s));
    DARE_CUDA(cub::DeviceReduce::Max(tmp.ptr, max_bytes, tot, max_d.ptr, ncells, s));
  }
  pt.mark("scan");
  uint32_t n_kept = 0, max_run = 0;
  unsigned long long n_rej = 0;
  DARE_CUDA(cudaMemcpyAsync(&max_run, max_d.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaMemcpyAsync(&n_kept, vol->d_offsets + ncells, sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaMemcpyAsync(&n_rej, rej.ptr, sizeof(n_rej), cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaStreamSynchronize(s));
  vol->n_samples = n_kept;
  vol->rejected = (int64_t)n_rej;
  dev_alloc(&vol->d_records, sizeof(uint4) * std::max<uint32_t>(n_kept, 1));
  dev_alloc(&vol->d_perm, std::max<uint32_t>(n_kept, 1));
  dev_alloc(&vol->d_bins, sizeof(uint32_t) * std::max<int64_t>(ncells, 1));
  if (n_kept == 0) {
    DARE_CUDA(cudaMemsetAsync(vol->d_bins, 0, sizeof(uint32_t) * std::max<int64_t>(ncells, 1), s));
    return;
  }
  Scratch<Key> keys(n_kept + 4, s);  // + slack: the seal's 16 B-aligned bulk copies may read past the end
  // one key CSR and no cell over 255 samples: u8 fill cursors, 4 per word
  const char* u8_env = getenv("DARE_FILL_U8");
  bool byte_cursors = byte_ok && groups == 1 && !direct && max_run <= 255 && !(u8_env && u8_env[0] == '0');
  // bucketed fill (frames whose pixels rarely share a cell, e.g. pitch >= voxel:
  // every run is a lone scattered write): if every bucket fits the placement stage
  bool bucketed = bucket_ok && groups == 1 && !direct && sizeof(Key) == 8;
  const int64_t nb = (ncells + kBucketCells - 1) >> kBucketShift;
  if (bucketed) {
    Scratch<uint32_t> maxb(1, s);
    DARE_CUDA(cudaMemsetAsync(maxb.ptr, 0, sizeof(uint32_t), s));
    bucket_init_k<<<ceil_div(nb, 256), 256, 0, s>>>(vol->d_offsets, ncells, nb, counts.ptr, maxb.ptr);
    DARE_CUDA(cudaGetLastError());
    uint32_t h_maxb = 0;
    DARE_CUDA(cudaMemcpyAsync(&h_maxb, maxb.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaStreamSynchronize(s));
    bucketed = h_maxb <= (uint32_t)kPlaceCap;
    byte_cursors = false;
  }
  if (!bucketed)
    DARE_CUDA(cudaMemsetAsync(counts.ptr, 0, byte_cursors ? 4 * ((size_t)ncells / 4 + 1) : sizeof(uint32_t) * nkc, s));
  pt.mark("readback+alloc");
  if (groups > 1 && !direct) {
    Scratch<Key> gkeys(n_kept, s);
    scatter(true, counts.ptr, (const uint32_t*)koff.ptr, (void*)gkeys.ptr, (unsigned long long*)nullptr, false, false);
    DARE_CUDA(cudaGetLastError());
    pt.mark("fill");
    regroup_keys_k<Key><<<ceil_div(ceil_div(ncells, 32) * 32, 256), 256, 0, s>>>(
        koff.ptr, vol->d_offsets, (uint32_t)ncells, groups, gkeys.ptr, keys.ptr);
    DARE_CUDA(cudaGetLastError());
    pt.mark("regroup");
  } else {
    scatter(true, counts.ptr, (const uint32_t*)vol->d_offsets, (void*)keys.ptr, (unsigned long long*)nullptr,
            byte_cursors, bucketed);
    DARE_CUDA(cudaGetLastError());
    pt.mark("fill");
    if (bucketed) {
      static std::once_flag place_attr;
      std::call_once(place_attr, [] {
        DARE_CUDA(cudaFuncSetAttribute(bucket_place_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(unsigned long long) * kPlaceCap)));
      });
      bucket_place_k<<<(unsigned)nb, 1024, sizeof(unsigned long long) * kPlaceCap, s>>>(
          vol->d_offsets, ncells, (unsigned long long*)keys.ptr);
      DARE_CUDA(cudaGetLastError());
      pt.mark("place");
    }
  }
  uint32_t* big_cells = counts.ptr;  // reuse: #big runs <= ncells
  Scratch<uint32_t> n_big_d(1, s);
  DARE_CUDA(cudaMemsetAsync(n_big_d.ptr, 0, sizeof(uint32_t), s));
  {
    // records are recomputed from their frame's axes; when the axes table is
    // large (many frames, scattered across a warp's cells) the seal is bound by
    // L1 misses, so trade shared-memory carve-out (occupancy) for L1
    const char* e = getenv("DARE_SEAL_CARVEOUT");  // development override
    const int carve = e ? atoi(e) : seal_carveout;
    const int c = carve >= 0 ? carve : (int)cudaSharedmemCarveoutDefault;
    DARE_CUDA(cudaFuncSetAttribute(seal_k<Rec, 16, false>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
    DARE_CUDA(cudaFuncSetAttribute(seal_k<Rec, kSmallRun, false>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
    DARE_CUDA(cudaFuncSetAttribute(seal_k<Rec, 16, true>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  }
  // measured at cfg2: seal 1.90 ms with the bulk prefetch vs 1.73 ms without (the
  // extra 16 KB of shared memory per block cuts residency from 10 to 6 blocks;
  // the kernel is bound by L1 throughput, which the prefetch does not relieve) --
  // opt-in with DARE_SEAL_BULK=1
  const char* bulk_env = getenv("DARE_SEAL_BULK");
  const bool bulk = bulk_env && bulk_env[0] == '1';
  // (bulk prefetch with the 16-key stage only: the 32-key stage's buffer would
  // exceed the 48 KB of static shared memory per block)
  (max_run <= 16 ? (bulk ? seal_k<Rec, 16, true> : seal_k<Rec, 16, false>) : seal_k<Rec, kSmallRun, false>)<<<
      ceil_div((ncells / vol->dims[2]) * ceil_div(vol->dims[2], 32), kSealWarps), 32 * kSealWarps, 0, s>>>(
      rec, vol->d_offsets, keys.ptr, (uint32_t)ncells, vol->d_records, big_cells, n_big_d.ptr,
      BinOut{vol->origin[2], vol->voxel, vol->dims[2], vol->d_bins, vol->d_perm});
  DARE_CUDA(cudaGetLastError());
  pt.mark("seal");
  uint32_t n_big = 0;
  DARE_CUDA(cudaMemcpyAsync(&n_big, n_big_d.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaStreamSynchronize(s));
  if (n_big == 0) return;
  DARE_LIMIT(n_kept < (uint32_t)INT32_MAX, "segmented sort limited to 2^31 samples");
  Scratch<uint32_t> begins(n_big, s), ends(n_big, s);
  Scratch<Key> sorted(n_kept, s);
  big_bounds_k<<<ceil_div(n_big, 256), 256, 0, s>>>(big_cells, n_big, vol->d_offsets,
                                                    begins.ptr, ends.ptr);
  size_t sort_bytes = 0;
  DARE_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, sort_bytes, keys.ptr, sorted.ptr,
                                               (int)n_kept, (int)n_big, begins.ptr, ends.ptr, s));
  Scratch<uint8_t> tmp(sort_bytes, s);
  DARE_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.ptr, sort_bytes, keys.ptr, sorted.ptr,
                                               (int)n_kept, (int)n_big, begins.ptr, ends.ptr, s));
  big_materialize_k<<<n_big, 256, 0, s>>>(rec, begins.ptr, ends.ptr, sorted.ptr, vol->d_records);
  DARE_CUDA(cudaGetLastError());
}

static std::unique_ptr<dare_volume_s> new_volume(const double* origin, double voxel,
                                                 const int64_t* dims) {
  DARE_REQUIRE(voxel > 0, "voxel_size must be > 0");
  DARE_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
  auto vol = std::make_unique<dare_volume_s>();
  DARE_CUDA(cudaGetDevice(&vol->device));
  for (int a = 0; a < 3; ++a) {
    vol->origin[a] = origin[a];
    vol->dims[a] = dims[a];
  }
  vol->voxel = voxel;
  vol->ncells = dims[0] * dims[1] * dims[2];
  DARE_LIMIT(vol->ncells < (int64_t)INT32_MAX, "more than 2^31 cells");
  return vol;
}

}  // namespace dare

using namespace dare;

extern "C" int dare_reconstruct(const uint8_t* frames, int64_t n_images, int32_t height,
                                int32_t width, int32_t frames_on_device,
                                const int32_t* frame_image, int64_t n_frames,
                                const double* frame_axes, const float* frame_quats,
                                double pitch_x, double pitch_y, const uint8_t* mask,
                                const double* origin, double voxel_size, const int64_t* dims,
                                dare_volume_t* out, int64_t* rejected_out_of_bounds) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr, "out handle pointer is null");
    const int64_t hw = (int64_t)height * width;
    DARE_LIMIT(n_frames * hw < (int64_t)UINT32_MAX, "more than 2^32-1 input pixels");
    DARE_LIMIT(n_frames < (1 << 24), "more than 2^24 frames (orientation id is 24 bits)");
    auto vol = new_volume(origin, voxel_size, dims);
    cudaStream_t s = thread_stream();
    DeviceClock clock(s);
    FrameSet fs(frames, n_images, height, width, frames_on_device, frame_image, n_frames,
                frame_axes, pitch_x, pitch_y, mask, s);
    VoxelMap m = make_voxel_map(origin, voxel_size, dims);
    // frames sharing a canonical f32 quaternion share an orientation id, so the
    // reslice gate table stays tiny for sweeps with few distinct orientations
    std::vector<uint32_t> word((size_t)std::max<int64_t>(n_frames, 1));
    std::vector<uint8_t> zeros((size_t)std::max<int64_t>(n_frames, 1), 0);
    std::vector<float4> table;
    dedup_orientations(frame_quats, zeros.data(), n_frames, word.data(), table);
    for (auto& w : word) w >>= 8;
    Scratch<uint32_t> d_oid((size_t)std::max<int64_t>(n_frames, 1), s);
    DARE_CUDA(cudaMemcpyAsync(d_oid.ptr, word.data(), sizeof(uint32_t) * word.size(),
                              cudaMemcpyHostToDevice, s));
    FrameView fv{fs.d_frames, fs.d_image, fs.d_axes, fs.d_mask, (uint32_t)n_frames,
                 (uint32_t)height, (uint32_t)width, (uint32_t)hw, pitch_x, pitch_y, d_oid.ptr,
                 FastDiv((uint32_t)width), FastDiv((uint32_t)hw), 0u, 0u, 0u, (uint32_t)hw,
                 0xffffffffu, (uint32_t)vol->ncells, 0u, 0u, 0u, nullptr};
    {
      const uint32_t ub = ceil_log2((uint64_t)width), vb = ceil_log2((uint64_t)height);
      if (ub + vb + ceil_log2((uint64_t)std::max<int64_t>(n_frames, 1)) <= 32 && ub + vb < 32) {
        fv.packed = 1;
        fv.ushift = ub;
        fv.fshift = ub + vb;
        fv.fstride = 1u << (ub + vb);
      }
    }
    vol->n_orient = (int64_t)table.size();
    if (!table.empty()) {
      dev_alloc(&vol->d_orient, sizeof(float4) * table.size());
      DARE_CUDA(cudaMemcpyAsync(vol->d_orient, table.data(), sizeof(float4) * table.size(),
                                cudaMemcpyHostToDevice, s));
    }
    DARE_LIMIT(ceil_div(n_frames, kRunFrames) <= 65535, "too many frames for one launch");
    const unsigned tiles = ceil_div(width, 16) * ceil_div(height, 16);
    const unsigned chunks = ceil_div(std::max<int64_t>(n_frames, 1), kRunFrames);
    // per-thread run lists of the count pass (8 B per run, <= one run per frame)
    Scratch<uint2> runs(n_frames > 0 ? (size_t)tiles * chunks * kRunFrames * 256 : 0, s);
    Scratch<uint8_t> nruns(n_frames > 0 ? (size_t)tiles * chunks * 256 : 0, s);
    // exact per-axis threshold tables (cells.cuh); the plain kernel when the
    // fine z table is not monotone or the development switch asks for it
    Scratch<double> tab_store;
    CellTables ct;
    const char* legacy = getenv("DARE_COUNT_LEGACY");
    const bool tabs_ok = !(legacy && legacy[0] == '1') && build_cell_tables(m, true, s, tab_store, ct);
    // 32-bit keys when the packed (frame, v, u) insertion index fits
    // (measured at cfg2: fill 1.09 -> 0.68 ms but seal 1.77 -> 2.36 ms from the
    // intensity gather, so 64-bit keys stay the default; DARE_NARROW_KEYS=1 selects them)
    const char* narrow_env = getenv("DARE_NARROW_KEYS");
    const bool narrow_keys = fv.packed != 0 && fv.fshift + ceil_log2((uint64_t)std::max<int64_t>(n_frames, 1)) <= 30 &&
                             narrow_env && narrow_env[0] == '1';
    const bool narrow = narrow_keys;
    auto scatter = [&](bool fill, uint32_t* counts, const uint32_t* offsets, void* keys,
                       unsigned long long* rej, bool byte_cursors, bool bucketed) {
      if (n_frames == 0) return;
      fv.byte_cursors = byte_cursors ? 1u : 0u;
      fv.bucketed = bucketed ? 1u : 0u;
      if (!fill) {  // needs no intensities: runs while host frames are still uploading
        if (tabs_ok)
          frame_count_tab_k<true><<<dim3(tiles, chunks), 256, 0, s>>>(fv, ct, m, counts, runs.ptr, nruns.ptr, rej);
        else
          (m.exact_inv ? frame_count_k<true> : frame_count_k<false>)<<<dim3(tiles, chunks), 256, 0, s>>>(
              fv, m, counts, runs.ptr, nruns.ptr, rej);
        return;
      }
      // fill in groups of chunks, each launched once its images are resident
      // (one launch per upload group, so fill overlaps the rest of the transfer)
      const int64_t step = fs.done.empty() ? chunks : std::max<int64_t>(1, ceil_div(fs.per_group, kRunFrames));
      for (int64_t c0 = 0; c0 < (int64_t)chunks; c0 += step) {
        const int64_t c1 = std::min<int64_t>(chunks, c0 + step);
        fs.wait_frames(s, c0 * kRunFrames, std::min<int64_t>(n_frames, c1 * kRunFrames));
        if (narrow)
          frame_fill_k<uint32_t><<<dim3(tiles, (unsigned)(c1 - c0)), 256, 0, s>>>(
              fv, (uint32_t)c0, runs.ptr, nruns.ptr, counts, offsets, (uint32_t*)keys);
        else
          frame_fill_k<unsigned long long><<<dim3(tiles, (unsigned)(c1 - c0)), 256, 0, s>>>(
              fv, (uint32_t)c0, runs.ptr, nruns.ptr, counts, offsets, (unsigned long long*)keys);
      }
    };
    Scratch<SealAxes> sa((size_t)std::max<int64_t>(n_frames, 1), s);
    if (n_frames > 0) {
      seal_axes_k<<<ceil_div(n_frames, 256), 256, 0, s>>>(fs.d_axes, d_oid.ptr, fs.d_image, (uint32_t)n_frames,
                                                          sa.ptr);
      DARE_CUDA(cudaGetLastError());
    }
    // measured: cfg3 (8000 frames, 576 KB of axes) seal 52.3 -> 46.0 ms at 75%
    fs.start_upload();  // after the small uploads above (they would queue behind the frames)
    const int carve = n_frames * (int64_t)sizeof(SealAxes) > (128 << 10) ? 75 : -1;
    // frame groups for the keys (see group_totals_k), a multiple of the 64-frame
    // chunk each.  Measured at cfg3 (8 groups): fill 35 -> 26 ms, but the
    // regroup (11.7 ms), the per-group counters and scans cost more -- the cfg3
    // fill is bound by its ~525M returning atomics (one pixel per cell and
    // sweep, so no lane aggregation), not by the partial sectors alone.  One
    // group by default; DARE_KEY_GROUPS=n selects the grouped layout.
    uint32_t groups = 1;
    Scratch<uint32_t> pre_store;
    {
      // Opt-in (measured at cfg3, profiles/round2_recon_variants.md): mode 2
      // (direct slots) fill 35.5 ms vs 35-38 ms with one group -- the cfg3
      // fill is not bound by its returning atomics either; mode 1 (group-major
      // key CSRs + regroup) removes the partial-sector DRAM merges (fill 26 ms)
      // but its regroup and counters cost more.  DARE_KEY_GROUPS=n selects n
      // groups of frames, DARE_KEY_MODE the layout (2 when groups are requested).
      const char* genv = getenv("DARE_KEY_GROUPS");
      const char* menv = getenv("DARE_KEY_MODE");
      const int mode = menv ? atoi(menv) : 2;
      const int64_t want = genv ? atoi(genv) : 1;
      if (mode != 0 && want > 1 && ncells_total_fits(2 * vol->ncells, want)) {
        const uint32_t cpg = (uint32_t)ceil_div(ceil_div(n_frames, want), kRunFrames);
        fv.chunks_per_group = cpg;
        groups = (uint32_t)ceil_div(ceil_div(n_frames, kRunFrames), cpg);
        if (mode == 2 && groups > 1) {
          pre_store.stream = s;
          DARE_CUDA(cudaMallocAsync((void**)&pre_store.ptr, sizeof(uint32_t) * (size_t)groups * vol->ncells, s));
          fv.direct = 1;
          fv.pre = pre_store.ptr;
        }
      }
    }
    // bucketed fill when image neighbours rarely share a cell (pixel pitch >= ~3/4 voxel:
    // the fill's MATCH finds no lane to aggregate with and every run is a lone
    // scattered write); DARE_FILL_BUCKETS=1 / 0 forces it on / off
    const char* bk_env = getenv("DARE_FILL_BUCKETS");
    const bool bucket_ok = bk_env ? bk_env[0] == '1' : std::min(pitch_x, pitch_y) >= 0.75 * voxel_size;
    if (narrow_keys)
      build_csr(vol.get(), FrameRecords32{fv, sa.ptr}, scatter, s, carve, groups, fv.direct ? pre_store.ptr : nullptr,
                true);
    else
      build_csr(vol.get(), FrameRecords{fv, sa.ptr}, scatter, s, carve, groups, fv.direct ? pre_store.ptr : nullptr,
                true, bucket_ok);
    clock.stop();
    DARE_CUDA(cudaStreamSynchronize(s));
    if (rejected_out_of_bounds) *rejected_out_of_bounds = vol->rejected;
    *out = vol.release();
  });
}

// VolumeBuilder.seal on the device: positions f32[n,3], orientations f32[n,4]
// (deduplicated on the host into the orientation table), intensities u8[n].
// Out-of-bounds samples are dropped and counted (insert_batch semantics).
extern "C" int dare_volume_seal(const double* origin, double voxel_size, const int64_t* dims,
                                int64_t n_samples, const float* positions,
                                const float* orientations, const uint8_t* intensities,
                                dare_volume_t* out) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr, "out handle pointer is null");
    DARE_REQUIRE(n_samples >= 0, "negative sample count");
    DARE_LIMIT(n_samples < (int64_t)UINT32_MAX, "more than 2^32-1 samples");
    auto vol = new_volume(origin, voxel_size, dims);
    std::vector<uint32_t> word((size_t)std::max<int64_t>(n_samples, 1));
    std::vector<float4> table;
    dedup_orientations(orientations, intensities, n_samples, word.data(), table);
    cudaStream_t s = thread_stream();
    vol->n_orient = (int64_t)table.size();
    dev_alloc(&vol->d_orient, sizeof(float4) * std::max<size_t>(table.size(), 1));
    if (!table.empty())
      DARE_CUDA(cudaMemcpyAsync(vol->d_orient, table.data(), sizeof(float4) * table.size(),
                                cudaMemcpyHostToDevice, s));
    Scratch<float> d_pos((size_t)n_samples * 3, s);
    Scratch<uint32_t> d_word((size_t)n_samples, s);
    if (n_samples) {
      DARE_CUDA(cudaMemcpyAsync(d_pos.ptr, positions, sizeof(float) * 3 * n_samples,
                                cudaMemcpyHostToDevice, s));
      DARE_CUDA(cudaMemcpyAsync(d_word.ptr, word.data(), sizeof(uint32_t) * n_samples,
                                cudaMemcpyHostToDevice, s));
    }
    VoxelMap m = make_voxel_map(origin, voxel_size, dims);
    const float* pos = d_pos.ptr;
    auto scatter = [&](bool fill, uint32_t* counts, const uint32_t* offsets, void* keys,
                       unsigned long long* rej, bool, bool) {
      if (n_samples == 0) return;
      if (fill)
        sample_scatter_k<true><<<ceil_div(n_samples, 256), 256, 0, s>>>(
            pos, n_samples, m, counts, offsets, (unsigned long long*)keys, rej);
      else
        sample_scatter_k<false><<<ceil_div(n_samples, 256), 256, 0, s>>>(
            pos, n_samples, m, counts, offsets, (unsigned long long*)keys, rej);
    };
    build_csr(vol.get(), SampleRecords{d_pos.ptr, d_word.ptr}, scatter, s);
    DARE_CUDA(cudaStreamSynchronize(s));
    *out = vol.release();
  });
}
