// Device-resident volume layouts.
//
// Directional volume (the reference's DirectionalVolume, volume.py:76-93):
// CSR by linear cell (x-major, (ix*ny+iy)*nz+iz, volume.py:103-106) with the
// per-cell runs in insertion order.  B200 layout, 16 B per sample instead of
// the reference's 29 B:
//   offsets  u32[ncells+1]   exclusive prefix of cell counts
//   records  uint4[n]        {f32 x, f32 y, f32 z, u32 (oid << 8) | intensity}
//   orients  float4[n_oid]   distinct canonical f32 quaternions (w,x,y,z)
// Positions stay bit-identical f32 (the reslice cube test needs them exactly).
// Quaternions are deduplicated: every sample of a reconstructed frame shares
// the frame's quaternion (reconstruct.py:192-196), so oid = frame slot and the
// per-pose orientation gates are evaluated once per oid, not per sample.
#pragma once
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
  FrameSet(const uint8_t* frames, int64_t n_images, int32_t H, int32_t W, int32_t on_device,
           const int32_t* frame_image, int64_t n_frames, const double* axes, double px, double py,
           const uint8_t* mask, cudaStream_t s);
  ~FrameSet();
};

}  // namespace dare
