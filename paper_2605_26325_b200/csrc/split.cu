// Direction-cluster index of a directional volume (volume.cuh, d_s*), for the
// certified reslice path.
//
// A reslice pose accepts a sample only if its beam direction agrees with the
// plane's (normal within cos_nt, in-plane axis within cos_it: the gate of
// _kernels.py:49-58).  Volumes built from several sweeps in different
// directions (four sweeps, normals +-z, x, y) hold samples a
// pose can never accept in every cell it visits -- three quarters of the
// visits at cfg3.  The index groups each cell's records by the cluster of
// their orientation (dominant axis of the sample normal and its sign), one CSR
// per present cluster over the same grid, each cell's cluster run keeping the
// canonical storage order (so it stays grouped by z quarter, with its own
// bins word).  The certified kernel then walks, per pixel, only the clusters
// holding at least one orientation the pose's gate accepts; within a cluster
// the per-record gate still decides.  Rejected samples contribute nothing to
// the reference's sums, so the certified sums and their bound are unchanged
// (the visit count used by the bound only shrinks).  The exact paths keep
// using the canonical layout.
//
// Built once per volume on the first certified reslice (thread-safe), when the
// volume has 2..kMaxOrient orientations in >= 2 clusters and the device has
// room for the copy (16 B per sample + 8 B per cell and cluster).
// DARE_ORIENT_SPLIT=0 disables it.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "volume.cuh"

namespace dare {
namespace {

constexpr int kMaxClusters = 6;
constexpr int64_t kMaxOrient = 1 << 20;  // (cluster ids: one byte per orientation)

// Per cell and cluster: record count and the cluster run's z-quarter bins word.
__global__ void split_count_k(int64_t ncells, const uint32_t* __restrict__ offsets,
                              const uint4* __restrict__ records, const uint32_t* __restrict__ bins,
                              const uint8_t* __restrict__ ocluster, int nclu, uint32_t* __restrict__ cnt,
                              uint32_t* __restrict__ sbins) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const uint32_t cs = offsets[c], ce = offsets[c + 1], w = bins[c];
  const bool binned = (w >> 24) != 0;
  const uint32_t b1 = w & 0xffu, b2 = (w >> 8) & 0xffu, b3 = (w >> 16) & 0xffu;
  uint32_t n[kMaxClusters] = {0, 0, 0, 0, 0, 0}, q1[kMaxClusters] = {0, 0, 0, 0, 0, 0},
           q2[kMaxClusters] = {0, 0, 0, 0, 0, 0}, q3[kMaxClusters] = {0, 0, 0, 0, 0, 0};
  for (uint32_t j = cs; j < ce; ++j) {
    const uint32_t k = ocluster[__ldg(&records[j].w) >> 8];
    const uint32_t pos = j - cs;
#pragma unroll
    for (int t = 0; t < kMaxClusters; ++t) {
      const uint32_t hit = (uint32_t)t == k;
      n[t] += hit;
      q1[t] += hit & (pos < b1);
      q2[t] += hit & (pos < b2);
      q3[t] += hit & (pos < b3);
    }
  }
#pragma unroll
  for (int t = 0; t < kMaxClusters; ++t) {
    if (t < nclu) {
      cnt[(size_t)t * ncells + c] = n[t];
      sbins[(size_t)t * ncells + c] = binned ? (q1[t] | (q2[t] << 8) | (q3[t] << 16) | (1u << 24)) : 0u;
    }
  }
}

// Stable scatter of each cell's records into its cluster runs.
__global__ void split_scatter_k(int64_t ncells, const uint32_t* __restrict__ offsets,
                                const uint4* __restrict__ records, const uint8_t* __restrict__ ocluster,
                                int nclu, const uint32_t* __restrict__ soffsets, uint4* __restrict__ srecords) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const uint32_t cs = offsets[c], ce = offsets[c + 1];
  if (cs == ce) return;
  uint32_t next[kMaxClusters];
#pragma unroll
  for (int t = 0; t < kMaxClusters; ++t) next[t] = t < nclu ? soffsets[(size_t)t * ncells + c] : 0u;
  for (uint32_t j = cs; j < ce; ++j) {
    const uint4 r = __ldg(&records[j]);
    const uint32_t k = ocluster[r.w >> 8];
    uint32_t dst = 0;
#pragma unroll
    for (int t = 0; t < kMaxClusters; ++t) {
      const bool hit = (uint32_t)t == k;
      dst = hit ? next[t] : dst;
      next[t] += hit;
    }
    srecords[dst] = r;
  }
}

bool split_enabled() {
  const char* e = getenv("DARE_ORIENT_SPLIT");
  return !(e && e[0] == '0');
}

}  // namespace

// Builds the cluster index if applicable; true when vol->d_s* are usable.
bool ensure_orient_split(dare_volume_s* vol, cudaStream_t s) {
  if (vol->split_state != 0) return vol->split_state > 0;  // (benign race: set once under the lock)
  std::lock_guard<std::mutex> lock(vol->split_mu);
  if (vol->split_state != 0) return vol->split_state > 0;
  vol->split_state = -1;
  if (!split_enabled() || vol->n_orient < 2 || vol->n_orient > kMaxOrient || vol->n_samples == 0) return false;
  // clusters of the orientations on the host (f32 quaternions -> sample normal,
  // _kernels.py:49-51; any deterministic grouping is valid)
  std::vector<float4> q((size_t)vol->n_orient);
  DARE_CUDA(cudaMemcpyAsync(q.data(), vol->d_orient, sizeof(float4) * q.size(), cudaMemcpyDeviceToHost, s));
  DARE_CUDA(cudaStreamSynchronize(s));
  std::vector<int> raw(q.size());
  int used[kMaxClusters] = {0, 0, 0, 0, 0, 0};
  for (size_t i = 0; i < q.size(); ++i) {
    const double w = q[i].x, x = q[i].y, y = q[i].z, z = q[i].w;
    const double n[3] = {2.0 * (x * z + w * y), 2.0 * (y * z - w * x), 1.0 - 2.0 * (x * x + y * y)};
    int a = 0;
    for (int k = 1; k < 3; ++k)
      if (std::fabs(n[k]) > std::fabs(n[a])) a = k;
    raw[i] = 2 * a + (n[a] < 0.0 ? 1 : 0);
    used[raw[i]] = 1;
  }
  int remap[kMaxClusters], nclu = 0;
  for (int k = 0; k < kMaxClusters; ++k) remap[k] = used[k] ? nclu++ : -1;
  if (nclu < 2) return false;
  std::vector<uint8_t> clu(q.size());
  int single[kMaxClusters], members[kMaxClusters] = {0, 0, 0, 0, 0, 0};
  for (size_t i = 0; i < q.size(); ++i) {
    clu[i] = (uint8_t)remap[raw[i]];
    if (members[clu[i]]++ == 0) single[clu[i]] = (int)i;
  }
  const int64_t ncells = vol->ncells, nk = (int64_t)nclu * ncells;
  if (nk + 1 >= (int64_t)INT32_MAX) return false;
  size_t free_b = 0, total_b = 0;
  DARE_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t need = sizeof(uint4) * (size_t)vol->n_samples + sizeof(uint32_t) * (size_t)(3 * nk + 2);
  if (free_b < need + (size_t(4) << 30)) return false;  // keep room for the caller
  uint8_t* d_clu = nullptr;
  uint32_t *d_soff = nullptr, *d_sbins = nullptr;
  uint4* d_srec = nullptr;
  try {
    dev_alloc(&d_clu, clu.size());
    dev_alloc(&d_soff, sizeof(uint32_t) * (size_t)(nk + 1));
    dev_alloc(&d_sbins, sizeof(uint32_t) * (size_t)nk);
    dev_alloc(&d_srec, sizeof(uint4) * (size_t)vol->n_samples);
    Scratch<uint32_t> cnt((size_t)nk + 1, s);
    DARE_CUDA(cudaMemcpyAsync(d_clu, clu.data(), clu.size(), cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMemsetAsync(cnt.ptr + nk, 0, sizeof(uint32_t), s));
    split_count_k<<<ceil_div(ncells, 256), 256, 0, s>>>(ncells, vol->d_offsets, vol->d_records, vol->d_bins, d_clu,
                                                        nclu, cnt.ptr, d_sbins);
    DARE_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.ptr, d_soff, (int)(nk + 1), s));
    Scratch<uint8_t> tmp(tmp_bytes, s);
    DARE_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, cnt.ptr, d_soff, (int)(nk + 1), s));
    split_scatter_k<<<ceil_div(ncells, 256), 256, 0, s>>>(ncells, vol->d_offsets, vol->d_records, d_clu, nclu,
                                                          d_soff, d_srec);
    DARE_CUDA(cudaGetLastError());
    DARE_CUDA(cudaStreamSynchronize(s));  // usable from every stream once published
  } catch (const Error&) {  // no room after all: the certified path runs on the canonical layout
    cudaGetLastError();
    cudaStreamSynchronize(s);
    dev_free(d_clu);
    dev_free(d_soff);
    dev_free(d_sbins);
    dev_free(d_srec);
    return false;
  }
  vol->d_ocluster = d_clu;
  vol->d_soffsets = d_soff;
  vol->d_sbins = d_sbins;
  vol->d_srecords = d_srec;
  vol->split_bytes = need + clu.size();
  for (int k = 0; k < kMaxClusters; ++k) vol->split_single[k] = k < nclu && members[k] == 1 ? single[k] : -1;
  vol->split_state = 1;
  return true;
}

}  // namespace dare
