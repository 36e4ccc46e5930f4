// z-quarter binning of a sealed directional volume (layout in volume.cuh).
//
// Pure storage permutation: every cell keeps exactly its samples; cells of
// <= kMaxBinnedRun samples are regrouped stably by z quarter and the
// insertion order stays recoverable through perm, so every consumer that
// needs the reference order (volume.py:240-269 seal order) still sees it.
#include "volume.cuh"

namespace dare {

// Half-warp per cell (cfg-typical cells hold ~16 samples): lanes load the
// cell's records in insertion order, compute the z bin, rank stably within
// the bin with ballots, then write back in place (all loads precede the
// stores through the __syncwarp).
__global__ void __launch_bounds__(256) bin_cells_k(const uint32_t* __restrict__ off, int64_t ncells,
                                                   int64_t nz, double oz, double voxel,
                                                   uint4* records, uint32_t* bins, int8_t* perm) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  const int64_t n_half = (int64_t)gridDim.x * (blockDim.x >> 4);
  for (int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4; ; c0 += n_half) {
    // warp-uniform loop control: both halves iterate while either has a cell
    const bool have = c0 < ncells;
    if (!__any_sync(0xffffffffu, have)) break;
    uint32_t s = 0, cnt = 0;
    if (have) {
      s = off[c0];
      cnt = off[c0 + 1] - s;
    }
    const bool big = cnt > 16;
    // cells of 17..32 samples: the whole warp takes them one at a time below.
    // Ballots run on the full warp (converged); each half reads its 16 bits.
    const bool small = have && !big;
    const bool mine = small && (uint32_t)hl < cnt;
    uint4 rec = make_uint4(0, 0, 0, 0);
    int bin = 0;
    if (mine) {
      rec = records[s + hl];
      const int64_t iz = c0 % nz;
      const float z = __uint_as_float(rec.z);
      bin = (z >= zbin_bound(oz, voxel, iz, 1)) + (z >= zbin_bound(oz, voxel, iz, 2)) +
            (z >= zbin_bound(oz, voxel, iz, 3));
    }
    unsigned m[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) m[b] = (__ballot_sync(0xffffffffu, mine && bin == b) >> (16 * half)) & 0xffffu;
    {
      const uint32_t c1 = __popc(m[0]), c2 = c1 + __popc(m[1]), c3 = c2 + __popc(m[2]);
      const uint32_t before = bin == 0 ? 0 : (bin == 1 ? c1 : (bin == 2 ? c2 : c3));
      const uint32_t dest = before + __popc(m[bin] & ((1u << hl) - 1u));
      __syncwarp();
      if (mine) {  // sweeps mostly insert a cell's samples in z order: skip unmoved records
        if (dest != (uint32_t)hl) records[s + dest] = rec;
        perm[s + hl] = (int8_t)((int)dest - hl);
      }
      if (small && hl == 0) bins[c0] = c1 | (c2 << 8) | (c3 << 16) | (1u << 24);
    }
    // big cells of this iteration (one leader lane per half), one at a time with the full warp
    unsigned bigmask = __ballot_sync(0xffffffffu, have && big && hl == 0);
    while (bigmask) {
      const int src = __ffs(bigmask) - 1;
      bigmask &= bigmask - 1;
      const int64_t c = __shfl_sync(0xffffffffu, c0, src);
      const uint32_t cs = __shfl_sync(0xffffffffu, s, src), cn = __shfl_sync(0xffffffffu, cnt, src);
      if (cn > (uint32_t)kMaxBinnedRun) {  // stays in insertion order
        for (uint32_t j = lane; j < cn; j += 32) perm[cs + j] = 0;
        if (lane == 0) bins[c] = 0;
        continue;
      }
      uint4 rec = make_uint4(0, 0, 0, 0);
      int bin = 0;
      const bool mine = (uint32_t)lane < cn;
      if (mine) {
        rec = records[cs + lane];
        const int64_t iz = c % nz;
        const float z = __uint_as_float(rec.z);
        bin = (z >= zbin_bound(oz, voxel, iz, 1)) + (z >= zbin_bound(oz, voxel, iz, 2)) +
              (z >= zbin_bound(oz, voxel, iz, 3));
      }
      unsigned m[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) m[b] = __ballot_sync(0xffffffffu, mine && bin == b);
      const uint32_t c1 = __popc(m[0]), c2 = c1 + __popc(m[1]), c3 = c2 + __popc(m[2]);
      const uint32_t before = bin == 0 ? 0 : (bin == 1 ? c1 : (bin == 2 ? c2 : c3));
      const uint32_t dest = before + __popc(m[bin] & ((1u << lane) - 1u));
      __syncwarp();
      if (mine) {
        if (dest != (uint32_t)lane) records[cs + dest] = rec;
        perm[cs + lane] = (int8_t)((int)dest - lane);
      }
      if (lane == 0) bins[c] = c1 | (c2 << 8) | (c3 << 16) | (1u << 24);
      __syncwarp();
    }
  }
}

void bin_volume(dare_volume_s* vol, cudaStream_t s) {
  PhaseTimer pt(s, "bin_volume");
  dev_alloc(&vol->d_bins, sizeof(uint32_t) * std::max<int64_t>(vol->ncells, 1));
  dev_alloc(&vol->d_perm, std::max<int64_t>(vol->n_samples, 1));
  if (vol->ncells > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(vol->ncells, 16), (int64_t)sm_count() * 16);
    bin_cells_k<<<grid, 256, 0, s>>>(vol->d_offsets, vol->ncells, vol->dims[2], vol->origin[2],
                                     vol->voxel, vol->d_records, vol->d_bins, vol->d_perm);
    DARE_CUDA(cudaGetLastError());
  }
  pt.mark("bin_cells_k");
}

}  // namespace dare
