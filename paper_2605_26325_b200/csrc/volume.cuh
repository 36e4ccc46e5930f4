// Device-resident volume layouts.
//
// Directional volume (the reference's DirectionalVolume, volume.py:76-93):
// CSR by linear cell (x-major, (ix*ny+iy)*nz+iz, volume.py:103-106) with the
// per-cell runs in insertion order.  B200 layout, 16 B per sample instead of
// the reference's 29 B:
//   offsets  u32[ncells+1]   exclusive prefix of cell counts
//   records  uint4[n]        {f32 x, f32 y, f32 z, u32 (oid << 8) | intensity}
//   orients  float4[n_oid]   distinct canonical f32 quaternions (w,x,y,z)
//   bins     u32[ncells]      z-quarter bin bounds of the cell (see below)
//   perm     i8[n]            reference (insertion) order -> storage order
// Positions stay bit-identical f32 (the reslice cube test needs them exactly).
//
// z-binning: within every cell of <= 32 samples the run is stored stably
// grouped by z quarter (bin b holds zb(iz, b) <= z < zb(iz, b+1), zb below),
// so a reslice column walk can drop the quarters of its first and last z-cell
// that lie outside the pixel's cube and still read ONE contiguous range.
// bins[c] = b1 | b2 << 8 | b3 << 16 | 1 << 24 with bk = #samples in bins < k
// (bit 24 clear: cell kept in insertion order).  The reference's insertion
// order is recovered through perm: the cell's j-th sample in insertion order,
// canonical index J = off[c] + j, is stored at J + perm[J].  Exact consumers
// (FP64 reslice path, brute force, download, merge) read through perm.
// Quaternions are deduplicated: every sample of a reconstructed frame shares
// the frame's quaternion (reconstruct.py:192-196), so oid = frame slot and the
// per-pose orientation gates are evaluated once per oid, not per sample.
#pragma once
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

struct dare_volume_s {
  int device = 0;
  double origin[3] = {0, 0, 0};
  double voxel = 0;
  int64_t dims[3] = {0, 0, 0};
  int64_t ncells = 0;
  int64_t n_samples = 0;
  int64_t n_orient = 0;
  int64_t rejected = 0;
  uint32_t* d_offsets = nullptr;
  uint4* d_records = nullptr;
  float4* d_orient = nullptr;
  uint32_t* d_bins = nullptr;
  int8_t* d_perm = nullptr;
  // Direction-cluster index for the certified reslice (split.cu, built on
  // first use): the records again, grouped by the cluster of their beam
  // direction (dominant axis of the sample normal and its sign: 6 clusters),
  // one CSR per cluster over the same grid with the same z-quarter binning --
  // a pose walks only the clusters holding an orientation its gate accepts.
  uint32_t* d_soffsets = nullptr;  // n_clusters x ncells + 1 (cluster-major, absolute)
  uint32_t* d_sbins = nullptr;     // n_clusters x ncells
  uint4* d_srecords = nullptr;     // n_samples
  uint8_t* d_ocluster = nullptr;   // n_orient: cluster of each orientation id
  std::atomic<int> split_state{0};  // 0 not tried, 1 built, -1 not applicable
  size_t split_bytes = 0;           // device bytes of the index once built
  int split_single[6] = {-1, -1, -1, -1, -1, -1};  // per cluster: its only orientation id, or -1
  std::mutex split_mu;
  ~dare_volume_s();
};

struct dare_scalar_s {
  int device = 0;
  double origin[3] = {0, 0, 0};
  double voxel = 0;
  int64_t dims[3] = {0, 0, 0};
  int64_t ncells = 0;
  float* d_values = nullptr;
  uint8_t* d_flags = nullptr;
  int64_t* d_counts = nullptr;
  ~dare_scalar_s();
};

namespace dare {

constexpr int kMaxBinnedRun = 32;  // cells with more samples stay in insertion order

// z-bin boundary k (1..3) of cell row iz: f32(origin_z + (iz + k/4) * voxel).
__device__ __forceinline__ float zbin_bound(double oz, double voxel, int64_t iz, int k) {
  return __double2float_rn(oz + ((double)iz + 0.25 * k) * voxel);
}

// Number of samples of a binned cell in bins < b (b = 0..3); bins word w.
__device__ __forceinline__ uint32_t bin_start(uint32_t w, int b) {
  return b == 0 ? 0u : (w >> (8 * (b - 1))) & 0xffu;
}

// Canonical (insertion-order) index -> storage index.
__device__ __forceinline__ uint32_t canon_to_store(const int8_t* __restrict__ perm, uint32_t j) {
  return j + (int32_t)__ldg(perm + j);
}

// Groups every cell of <= kMaxBinnedRun samples by z quarter in place (stable),
// allocates and fills d_bins / d_perm.  Input: records in insertion order.
void bin_volume(dare_volume_s* vol, cudaStream_t s);

VoxelMap make_voxel_map(const double* origin, double voxel, const int64_t* dims);

// Host: maps each sample's f32 quaternion to a dense orientation id; writes
// word[i] = (id << 8) | intensity[i] and appends distinct quaternions to table.
void dedup_orientations(const float* orientations, const uint8_t* intensities, int64_t n,
                        uint32_t* word, std::vector<float4>& table);

// Uploads frames/axes for a reconstruct-style pass; owns the device copies.
struct FrameSet {
  const uint8_t* d_frames = nullptr;  // n_images x H x W
  int32_t* d_image = nullptr;         // n_frames
  double* d_axes = nullptr;           // n_frames x 9
  uint8_t* d_mask = nullptr;          // H x W or null
  int64_t n_frames = 0;
  int32_t H = 0, W = 0;
  double px = 0, py = 0;
  uint8_t* owned_frames = nullptr;
  cudaStream_t stream = nullptr;
  // host frames are uploaded in groups of images on the thread's copy stream;
  // group g (images [g * per_group, ...)) is resident once done[g] completed
  std::vector<cudaEvent_t> done;
  int64_t per_group = 0;
  std::vector<int32_t> h_image;  // frame -> image (host copy, for wait_frames)
  const uint8_t* h_frames = nullptr;
  int64_t n_images = 0;
  FrameSet(const uint8_t* frames, int64_t n_images, int32_t H, int32_t W, int32_t on_device,
           const int32_t* frame_image, int64_t n_frames, const double* axes, double px, double py,
           const uint8_t* mask, cudaStream_t s);
  // start the grouped upload of host frames -- after every small (pageable)
  // upload of the call, which would otherwise queue behind it on the copy engine
  void start_upload();
  // make `s` wait until the images of frames [f_begin, f_end) are on the device
  void wait_frames(cudaStream_t s, int64_t f_begin, int64_t f_end) const;
  ~FrameSet();
};

// Direction-cluster index (split.cu): builds it on first use if applicable;
// true when vol->d_soffsets / d_sbins / d_srecords / d_ocluster are usable.
bool ensure_orient_split(dare_volume_s* vol, cudaStream_t s);

}  // namespace dare
