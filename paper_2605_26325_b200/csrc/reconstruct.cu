// Directional reconstruction: pixel -> cell scatter and the sealed CSR build.
//
// Reference: reconstruct.py:166-199 (reconstruct_volume), 152-163
// (frame_world_positions), volume.py:208-238 (insert_batch/_voxel_indices),
// volume.py:240-269 (seal: stable argsort by linear cell + bincount + cumsum).
//
// Device pipeline (all FP64 chains bit-identical to numpy; -fmad=false):
//   1. count   : per pixel -> cell; warp-aggregated u32 histogram
//                (__match_any_sync groups equal cells, one atomic per group);
//                out-of-bounds pixels counted (volume.py:230-233).
//   2. scan    : exclusive prefix of counts -> cell offsets (CUB).
//   3. fill    : per pixel -> slot = offset + atomic cursor; stores the pixel's
//                global insertion key (synchronized frame * H*W + pixel).
//   4. seal    : per cell, sort its (tiny) key run ascending = insertion order
//                (this is what makes the atomic fill identical to numpy's
//                stable argsort) and materialise the 16 B records; runs > 32
//                keys go through CUB's segmented sort.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <memory>
#include <vector>

#include "volume.cuh"

namespace dare {

struct FrameView {
  const uint8_t* frames;
  const int32_t* image;
  const double* axes;
  const uint8_t* mask;
  int64_t n_frames;
  int32_t H, W;
  double px, py;
  const uint32_t* oid;  // orientation id per synchronized frame
};

static FrameView view_of(const FrameSet& fs) {
  return FrameView{fs.d_frames, fs.d_image, fs.d_axes, fs.d_mask, fs.n_frames,
                   fs.H,        fs.W,       fs.px,     fs.py,      nullptr};
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Warp-aggregated histogram (kFill=false) or slot assignment (kFill=true):
// lanes holding the same cell form one __match_any_sync group; the lowest lane
// does one atomic for the whole group and lanes take consecutive slots in lane
// order (= insertion order within the warp).
template <bool kFill>
__device__ __forceinline__ void warp_scatter(bool kept, int64_t lin, uint32_t key,
                                             uint32_t* counts,
                                             const uint32_t* __restrict__ offsets,
                                             uint32_t* keys) {
  unsigned active = __ballot_sync(0xffffffffu, kept);
  if (!kept) return;
  unsigned peers = __match_any_sync(active, (unsigned long long)lin);
  unsigned leader = __ffs(peers) - 1;
  unsigned n = __popc(peers);
  if (!kFill) {
    if (lane_id() == leader) atomicAdd(&counts[lin], n);
  } else {
    unsigned base = 0;
    if (lane_id() == leader) base = atomicAdd(&counts[lin], n);
    base = __shfl_sync(peers, base, leader);
    unsigned rank = __popc(peers & ((1u << lane_id()) - 1u));
    keys[offsets[lin] + base + rank] = key;
  }
}

// Frames: grid x over pixel blocks of one frame, y over frames (strided).
template <bool kFill>
__global__ void __launch_bounds__(256) frame_scatter_k(FrameView fv, VoxelMap m,
                                                       uint32_t* counts,
                                                       const uint32_t* __restrict__ offsets,
                                                       uint32_t* keys,
                                                       unsigned long long* rejected) {
  __shared__ double s_axes[9];
  const int64_t hw = (int64_t)fv.H * fv.W;
  for (int64_t f = blockIdx.y; f < fv.n_frames; f += gridDim.y) {
    __syncthreads();
    if (threadIdx.x < 9) s_axes[threadIdx.x] = fv.axes[f * 9 + threadIdx.x];
    __syncthreads();
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool valid = p < hw;
    if (valid && fv.mask) valid = fv.mask[p] != 0;
    int64_t lin = -1;
    if (valid) {
      float p32[3];
      lin = pixel_cell(s_axes, (int)(p % fv.W), (int)(p / fv.W), fv.px, fv.py, m, p32);
    }
    bool kept = lin >= 0;
    if (!kFill) {
      int oob = __syncthreads_count(valid && !kept);
      if (threadIdx.x == 0 && oob) atomicAdd(rejected, (unsigned long long)oob);
    }
    warp_scatter<kFill>(kept, lin, (uint32_t)(f * hw + p), counts, offsets, keys);
  }
}

// Arbitrary samples (VolumeBuilder.seal, volume.py:240-269): key = sample index.
template <bool kFill>
__global__ void __launch_bounds__(256) sample_scatter_k(const float* __restrict__ pos, int64_t n,
                                                        VoxelMap m, uint32_t* counts,
                                                        const uint32_t* __restrict__ offsets,
                                                        uint32_t* keys,
                                                        unsigned long long* rejected) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = i < n;
  int64_t lin = -1;
  if (valid) {
    bool ok = true;
    int64_t idx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double f = floor(voxel_coord(m, a, pos[3 * i + a]));
      ok = ok && (f >= 0.0) && (f < (double)m.dims[a]);
      idx[a] = ok ? (int64_t)f : 0;
    }
    if (ok) lin = (idx[0] * m.dims[1] + idx[1]) * m.dims[2] + idx[2];
  }
  bool kept = lin >= 0;
  if (!kFill) {
    int oob = __syncthreads_count(valid && !kept);
    if (threadIdx.x == 0 && oob) atomicAdd(rejected, (unsigned long long)oob);
  }
  warp_scatter<kFill>(kept, lin, (uint32_t)i, counts, offsets, keys);
}

struct FrameRecords {
  FrameView fv;
  __device__ __forceinline__ uint4 operator()(uint32_t key) const {
    const uint32_t hw = (uint32_t)fv.H * (uint32_t)fv.W;
    uint32_t f = key / hw, p = key - f * hw;
    int u = (int)(p % (uint32_t)fv.W), v = (int)(p / (uint32_t)fv.W);
    const double* fa = fv.axes + (size_t)f * 9;
    double U = (double)u * fv.px, V = (double)v * fv.py;
    float p32[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      p32[a] = __double2float_rn((U * fa[a] + V * fa[3 + a]) + fa[6 + a]);
    uint8_t inten = fv.frames[(size_t)fv.image[f] * hw + p];
    return make_uint4(__float_as_uint(p32[0]), __float_as_uint(p32[1]), __float_as_uint(p32[2]),
                      (fv.oid[f] << 8) | inten);
  }
};

struct SampleRecords {
  const float* pos;
  const uint32_t* word;  // (oid << 8) | intensity
  __device__ __forceinline__ uint4 operator()(uint32_t key) const {
    return make_uint4(__float_as_uint(pos[3 * (size_t)key]), __float_as_uint(pos[3 * (size_t)key + 1]),
                      __float_as_uint(pos[3 * (size_t)key + 2]), word[key]);
  }
};

constexpr int kSmallRun = 32;

// thread per cell: sort the run's keys (= insertion order) and write records
template <class Rec>
__global__ void __launch_bounds__(256) seal_k(Rec rec, const uint32_t* __restrict__ offsets,
                                              const uint32_t* __restrict__ keys, int64_t ncells,
                                              uint4* records, uint32_t* big_cells,
                                              uint32_t* n_big) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  uint32_t s0 = offsets[c], n = offsets[c + 1] - s0;
  if (n == 0) return;
  if (n > kSmallRun) {
    big_cells[atomicAdd(n_big, 1u)] = (uint32_t)c;
    return;
  }
  uint32_t k[kSmallRun];
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t x = keys[s0 + i];
    uint32_t j = i;
    while (j > 0 && k[j - 1] > x) {
      k[j] = k[j - 1];
      --j;
    }
    k[j] = x;
  }
  for (uint32_t i = 0; i < n; ++i) records[s0 + i] = rec(k[i]);
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
                                  const uint32_t* __restrict__ sorted, uint4* records) {
  uint32_t b = begins[blockIdx.x], e = ends[blockIdx.x];
  for (uint32_t s = b + threadIdx.x; s < e; s += blockDim.x) records[s] = rec(sorted[s]);
}

// count -> scan -> fill -> seal, shared by frames and arbitrary samples.
// `scatter(fill, counts, offsets, keys, rejected)` launches the source's pass.
template <class Rec, class Scatter>
void build_csr(dare_volume_s* vol, Rec rec, Scatter scatter, cudaStream_t s) {
  const int64_t ncells = vol->ncells;
  PhaseTimer pt(s, "build_csr");
  Scratch<uint32_t> counts(ncells + 1, s);
  Scratch<unsigned long long> rej(1, s);
  DARE_CUDA(cudaMemsetAsync(counts.ptr, 0, sizeof(uint32_t) * (ncells + 1), s));
  DARE_CUDA(cudaMemsetAsync(rej.ptr, 0, sizeof(unsigned long long), s));
  dev_alloc(&vol->d_offsets, sizeof(uint32_t) * (ncells + 1));
  pt.mark("alloc+memset");
  scatter(false, counts.ptr, (const uint32_t*)nullptr, (uint32_t*)nullptr, rej.ptr);
  DARE_CUDA(cudaGetLastError());
  pt.mark("count");
  size_t tmp_bytes = 0;
  DARE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts.ptr, vol->d_offsets,
                                          ncells + 1, s));
  {
    Scratch<uint8_t> tmp(tmp_bytes, s);
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, counts.ptr, vol->d_offsets,
                                            ncells + 1, s));
  }
  pt.mark("scan");
  uint32_t n_kept = 0;
  unsigned long long n_rej = 0;
  DARE_CUDA(cudaMemcpyAsync(&n_kept, vol->d_offsets + ncells, sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaMemcpyAsync(&n_rej, rej.ptr, sizeof(n_rej), cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaStreamSynchronize(s));
  vol->n_samples = n_kept;
  vol->rejected = (int64_t)n_rej;
  dev_alloc(&vol->d_records, sizeof(uint4) * std::max<uint32_t>(n_kept, 1));
  if (n_kept == 0) return;
  Scratch<uint32_t> keys(n_kept, s);
  DARE_CUDA(cudaMemsetAsync(counts.ptr, 0, sizeof(uint32_t) * ncells, s));
  pt.mark("readback+alloc");
  scatter(true, counts.ptr, (const uint32_t*)vol->d_offsets, keys.ptr,
          (unsigned long long*)nullptr);
  DARE_CUDA(cudaGetLastError());
  pt.mark("fill");
  uint32_t* big_cells = counts.ptr;  // reuse: #big runs <= ncells
  Scratch<uint32_t> n_big_d(1, s);
  DARE_CUDA(cudaMemsetAsync(n_big_d.ptr, 0, sizeof(uint32_t), s));
  seal_k<<<ceil_div(ncells, 256), 256, 0, s>>>(rec, vol->d_offsets, keys.ptr, ncells,
                                                vol->d_records, big_cells, n_big_d.ptr);
  DARE_CUDA(cudaGetLastError());
  pt.mark("seal");
  uint32_t n_big = 0;
  DARE_CUDA(cudaMemcpyAsync(&n_big, n_big_d.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaStreamSynchronize(s));
  if (n_big == 0) return;
  DARE_LIMIT(n_kept < (uint32_t)INT32_MAX, "segmented sort limited to 2^31 samples");
  Scratch<uint32_t> begins(n_big, s), ends(n_big, s), sorted(n_kept, s);
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
    FrameSet fs(frames, n_images, height, width, frames_on_device, frame_image, n_frames,
                frame_axes, pitch_x, pitch_y, mask, s);
    FrameView fv = view_of(fs);
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
    fv.oid = d_oid.ptr;
    vol->n_orient = (int64_t)table.size();
    if (!table.empty()) {
      dev_alloc(&vol->d_orient, sizeof(float4) * table.size());
      DARE_CUDA(cudaMemcpyAsync(vol->d_orient, table.data(), sizeof(float4) * table.size(),
                                cudaMemcpyHostToDevice, s));
    }
    dim3 grid(ceil_div(hw, 256), (unsigned)std::min<int64_t>(std::max<int64_t>(n_frames, 1), 65535));
    auto scatter = [&](bool fill, uint32_t* counts, const uint32_t* offsets, uint32_t* keys,
                       unsigned long long* rej) {
      if (n_frames == 0) return;
      if (fill)
        frame_scatter_k<true><<<grid, 256, 0, s>>>(fv, m, counts, offsets, keys, rej);
      else
        frame_scatter_k<false><<<grid, 256, 0, s>>>(fv, m, counts, offsets, keys, rej);
    };
    build_csr(vol.get(), FrameRecords{fv}, scatter, s);
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
    auto scatter = [&](bool fill, uint32_t* counts, const uint32_t* offsets, uint32_t* keys,
                       unsigned long long* rej) {
      if (n_samples == 0) return;
      if (fill)
        sample_scatter_k<true><<<ceil_div(n_samples, 256), 256, 0, s>>>(pos, n_samples, m, counts,
                                                                        offsets, keys, rej);
      else
        sample_scatter_k<false><<<ceil_div(n_samples, 256), 256, 0, s>>>(pos, n_samples, m, counts,
                                                                         offsets, keys, rej);
    };
    build_csr(vol.get(), SampleRecords{d_pos.ptr, d_word.ptr}, scatter, s);
    DARE_CUDA(cudaStreamSynchronize(s));
    *out = vol.release();
  });
}
