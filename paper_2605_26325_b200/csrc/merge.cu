// Merge of per-rank partial directional volumes (frame-sharded reconstruction,
// SURVEY §8e).  Rank r reconstructed a contiguous block of synchronized frames
// into the FULL grid; ranks are ordered by frame block, so the reference's
// insertion order within a cell is "rank 0's run, then rank 1's, ...".  The
// merged CSR is therefore bit-identical to a single-device reconstruction:
//   count[c]  = sum_r count_r[c]               (integer, exact)
//   offset    = exclusive scan of count
//   records   = per cell, the parts' runs concatenated in rank order, with the
//               orientation id rebased into the concatenated orientation table.
// The parts are device buffers on the calling device (the local volume plus
// buffers received through NCCL, or several local partial volumes when the
// ranks are emulated on one GPU in tests): a part's records in its storage
// order plus its perm (insertion order is read through perm, so no gathered
// copy is ever made) or, with a null perm, already in insertion order.
// Orientation tables are deduplicated in rank order (first occurrence wins,
// = the single-device dedup order over frames), so the merged records,
// orientation table, bins and perm equal a single-device build's exactly;
// the merged volume is z-binned like every other (volume.cuh).
#include <cub/device/device_scan.cuh>

#include <memory>
#include <vector>

#include "volume.cuh"

namespace dare {

struct MergeParts {
  const uint32_t* const* offsets;  // device array of n device pointers
  const uint4* const* records;     // storage order
  const int8_t* const* perm;       // per part: insertion -> storage offset, or null
  const uint32_t* const* remap;    // per part: local orientation id -> merged id
  int n;
};

__global__ void merge_count_k(MergeParts p, int64_t ncells, uint32_t* counts) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  uint32_t n = 0;
  for (int r = 0; r < p.n; ++r) n += p.offsets[r][c + 1] - p.offsets[r][c];
  counts[c] = n;
}

// warp per cell: lanes copy the concatenated runs (coalesced within each run)
__global__ void merge_copy_k(MergeParts p, int64_t ncells, const uint32_t* __restrict__ out_off,
                             uint4* out) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncells) return;
  uint32_t dst = out_off[c];
  for (int r = 0; r < p.n; ++r) {
    const uint32_t s = p.offsets[r][c], e = p.offsets[r][c + 1];
    const int8_t* perm = p.perm[r];
    const uint32_t* remap = p.remap[r];
    for (uint32_t j = s + lane; j < e; j += 32) {
      uint4 rec = p.records[r][perm ? canon_to_store(perm, j) : j];
      rec.w = (__ldg(remap + (rec.w >> 8)) << 8) | (rec.w & 0xffu);
      DARE_CHECK(dst + (j - s) < out_off[c + 1] && (rec.w >> 8) < (1u << 24));
      out[dst + (j - s)] = rec;
    }
    dst += e - s;
  }
}

}  // namespace dare

using namespace dare;

extern "C" int dare_volume_merge(const double* origin, double voxel_size, const int64_t* dims,
                                 int32_t n_parts, const uint32_t* const* d_offsets,
                                 const void* const* d_records, const int8_t* const* d_perm,
                                 const float* const* d_orient, const int64_t* n_samples,
                                 const int64_t* n_orient, const int64_t* rejected, dare_volume_t* out) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr && n_parts >= 1, "need an output handle and at least one part");
    DARE_REQUIRE(voxel_size > 0, "voxel_size must be > 0");
    DARE_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
    const int64_t ncells = dims[0] * dims[1] * dims[2];
    DARE_LIMIT(ncells < (int64_t)INT32_MAX, "more than 2^31 cells");
    int64_t total = 0, total_rej = 0, total_orient = 0;
    for (int r = 0; r < n_parts; ++r) {
      total += n_samples[r];
      total_orient += n_orient[r];
      total_rej += rejected ? rejected[r] : 0;
    }
    DARE_LIMIT(total < (int64_t)UINT32_MAX, "more than 2^32-1 samples");
    DARE_LIMIT(total_orient < (1 << 24), "more than 2^24 orientations");
    cudaStream_t s = thread_stream();
    // orientation tables: rank-ordered first-occurrence dedup on the host
    // (tables are small: at most one entry per frame)
    std::vector<float4> cat((size_t)std::max<int64_t>(total_orient, 1));
    {
      int64_t o = 0;
      for (int r = 0; r < n_parts; ++r) {
        if (n_orient[r] > 0)
          DARE_CUDA(cudaMemcpyAsync(cat.data() + o, d_orient[r], sizeof(float4) * n_orient[r],
                                    cudaMemcpyDeviceToHost, s));
        o += n_orient[r];
      }
      DARE_CUDA(cudaStreamSynchronize(s));
    }
    std::vector<uint32_t> word((size_t)std::max<int64_t>(total_orient, 1));
    std::vector<uint8_t> zeros((size_t)std::max<int64_t>(total_orient, 1), 0);
    std::vector<float4> table;
    dedup_orientations(reinterpret_cast<const float*>(cat.data()), zeros.data(), total_orient, word.data(),
                       table);
    for (auto& w : word) w >>= 8;  // concatenated local id -> merged id

    auto vol = std::make_unique<dare_volume_s>();
    DARE_CUDA(cudaGetDevice(&vol->device));
    for (int a = 0; a < 3; ++a) {
      vol->origin[a] = origin[a];
      vol->dims[a] = dims[a];
    }
    vol->voxel = voxel_size;
    vol->ncells = ncells;
    vol->n_samples = total;
    vol->n_orient = (int64_t)table.size();
    vol->rejected = total_rej;

    Scratch<uint32_t> d_map((size_t)std::max<int64_t>(total_orient, 1), s);
    DARE_CUDA(cudaMemcpyAsync(d_map.ptr, word.data(), sizeof(uint32_t) * word.size(), cudaMemcpyHostToDevice, s));
    std::vector<const uint32_t*> remap(n_parts);
    std::vector<const int8_t*> perms(n_parts);
    {
      int64_t o = 0;
      for (int r = 0; r < n_parts; ++r) {
        remap[r] = d_map.ptr + o;
        perms[r] = d_perm ? d_perm[r] : nullptr;
        o += n_orient[r];
      }
    }
    Scratch<const uint32_t*> d_off_ptrs(n_parts, s);
    Scratch<const uint4*> d_rec_ptrs(n_parts, s);
    Scratch<const int8_t*> d_perm_ptrs(n_parts, s);
    Scratch<const uint32_t*> d_remap_ptrs(n_parts, s);
    DARE_CUDA(cudaMemcpyAsync(d_off_ptrs.ptr, d_offsets, sizeof(void*) * n_parts, cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMemcpyAsync(d_rec_ptrs.ptr, d_records, sizeof(void*) * n_parts, cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMemcpyAsync(d_perm_ptrs.ptr, perms.data(), sizeof(void*) * n_parts, cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMemcpyAsync(d_remap_ptrs.ptr, remap.data(), sizeof(void*) * n_parts, cudaMemcpyHostToDevice,
                              s));
    MergeParts parts{d_off_ptrs.ptr, d_rec_ptrs.ptr, d_perm_ptrs.ptr, d_remap_ptrs.ptr, n_parts};

    dev_alloc(&vol->d_offsets, sizeof(uint32_t) * (ncells + 1));
    dev_alloc(&vol->d_records, sizeof(uint4) * std::max<int64_t>(total, 1));
    dev_alloc(&vol->d_orient, sizeof(float4) * std::max<size_t>(table.size(), 1));
    if (!table.empty())
      DARE_CUDA(cudaMemcpyAsync(vol->d_orient, table.data(), sizeof(float4) * table.size(),
                                cudaMemcpyHostToDevice, s));
    Scratch<uint32_t> counts(ncells + 1, s);
    DARE_CUDA(cudaMemsetAsync(counts.ptr + ncells, 0, sizeof(uint32_t), s));
    merge_count_k<<<ceil_div(ncells, 256), 256, 0, s>>>(parts, ncells, counts.ptr);
    DARE_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts.ptr, vol->d_offsets,
                                            ncells + 1, s));
    {
      Scratch<uint8_t> tmp(tmp_bytes, s);
      DARE_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, counts.ptr, vol->d_offsets,
                                              ncells + 1, s));
    }
    merge_copy_k<<<ceil_div(ncells * 32, 256), 256, 0, s>>>(parts, ncells, vol->d_offsets,
                                                             vol->d_records);
    DARE_CUDA(cudaGetLastError());
    bin_volume(vol.get(), s);
    DARE_CUDA(cudaStreamSynchronize(s));
    *out = vol.release();
  });
}
