// Volume handles: upload from / download to the reference's host layout
// (volume.py:76-93; .darevol I/O volume.py:272-330 works on these arrays).
#include <cstring>
#include <unordered_map>
#include <vector>

#include <memory>

#include "volume.cuh"

namespace {

struct QuatKey {
  uint64_t a, b;
  bool operator==(const QuatKey& o) const { return a == o.a && b == o.b; }
};
struct QuatHash {
  size_t operator()(const QuatKey& k) const {
    uint64_t h = k.a * 0x9E3779B97F4A7C15ull ^ (k.b + 0x632BE59BD9B4E019ull + (k.a << 6));
    return (size_t)(h ^ (h >> 29));
  }
};

}  // namespace

namespace dare {

void dedup_orientations(const float* orientations, const uint8_t* intensities, int64_t n,
                        uint32_t* word, std::vector<float4>& table) {
  std::unordered_map<QuatKey, uint32_t, QuatHash> ids;
  QuatKey last{~0ull, ~0ull};
  uint32_t last_id = 0;
  for (int64_t i = 0; i < n; ++i) {
    QuatKey k;
    std::memcpy(&k, orientations + 4 * i, 16);
    if (!(k == last)) {
      auto it = ids.find(k);
      if (it == ids.end()) {
        DARE_LIMIT(table.size() < (1u << 24), "more than 2^24 distinct orientations");
        last_id = (uint32_t)table.size();
        float4 q;
        std::memcpy(&q, orientations + 4 * i, 16);
        table.push_back(q);
        ids.emplace(k, last_id);
      } else {
        last_id = it->second;
      }
      last = k;
    }
    word[i] = (last_id << 8) | intensities[i];
  }
}

}  // namespace dare

using namespace dare;

extern "C" int dare_volume_upload(const double* origin, double voxel_size, const int64_t* dims,
                                  const int64_t* cell_starts, const int64_t* cell_counts,
                                  int64_t n_samples, const float* positions,
                                  const float* orientations, const uint8_t* intensities,
                                  dare_volume_t* out) {
  return guard([&] {
    DARE_REQUIRE(out != nullptr, "out handle pointer is null");
    DARE_REQUIRE(voxel_size > 0, "voxel_size must be > 0");
    DARE_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
    DARE_REQUIRE(n_samples >= 0, "negative sample count");
    DARE_LIMIT(n_samples < (int64_t)UINT32_MAX, "more than 2^32-1 samples");
    const int64_t ncells = dims[0] * dims[1] * dims[2];
    DARE_LIMIT(ncells < (int64_t)INT32_MAX, "more than 2^31 cells");

    // CSR offsets; the reference's runs need not be packed (load_volume takes
    // arbitrary offsets), so gather runs into a packed store when they are not.
    std::vector<uint32_t> offsets(ncells + 1);
    bool packed = true;
    int64_t run = 0;
    for (int64_t c = 0; c < ncells; ++c) {
      DARE_REQUIRE(cell_counts[c] >= 0, "negative cell count");
      offsets[c] = (uint32_t)run;
      if (cell_counts[c] > 0) {
        DARE_REQUIRE(cell_starts[c] >= 0 && cell_starts[c] + cell_counts[c] <= n_samples,
                     "cell run outside the sample store");
        if (cell_starts[c] != run) packed = false;
      }
      run += cell_counts[c];
      DARE_LIMIT(run < (int64_t)UINT32_MAX, "more than 2^32-1 referenced samples");
    }
    offsets[ncells] = (uint32_t)run;
    const int64_t n = run;

    std::vector<uint32_t> word((size_t)std::max<int64_t>(n_samples, 1));
    std::vector<float4> table;
    dedup_orientations(orientations, intensities, n_samples, word.data(), table);
    std::vector<uint4> records((size_t)std::max<int64_t>(n, 1));
    auto emit = [&](int64_t dst, int64_t i) {
      uint4 r;
      std::memcpy(&r, positions + 3 * i, 12);
      r.w = word[i];
      records[dst] = r;
    };
    if (packed) {
      for (int64_t i = 0; i < n; ++i) emit(i, i);
    } else {
      for (int64_t c = 0; c < ncells; ++c)
        for (int64_t j = 0; j < cell_counts[c]; ++j) emit(offsets[c] + j, cell_starts[c] + j);
    }

    auto vol = std::make_unique<dare_volume_s>();
    DARE_CUDA(cudaGetDevice(&vol->device));
    for (int a = 0; a < 3; ++a) {
      vol->origin[a] = origin[a];
      vol->dims[a] = dims[a];
    }
    vol->voxel = voxel_size;
    vol->ncells = ncells;
    vol->n_samples = n;
    vol->n_orient = (int64_t)table.size();
    cudaStream_t s = thread_stream();
    dev_alloc(&vol->d_offsets, sizeof(uint32_t) * (ncells + 1));
    dev_alloc(&vol->d_records, sizeof(uint4) * records.size());
    dev_alloc(&vol->d_orient, sizeof(float4) * std::max<size_t>(table.size(), 1));
    DARE_CUDA(cudaMemcpyAsync(vol->d_offsets, offsets.data(), sizeof(uint32_t) * (ncells + 1),
                              cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMemcpyAsync(vol->d_records, records.data(), sizeof(uint4) * records.size(),
                              cudaMemcpyHostToDevice, s));
    if (!table.empty())
      DARE_CUDA(cudaMemcpyAsync(vol->d_orient, table.data(), sizeof(float4) * table.size(),
                                cudaMemcpyHostToDevice, s));
    bin_volume(vol.get(), s);
    DARE_CUDA(cudaStreamSynchronize(s));
    *out = vol.release();
  });
}

extern "C" int dare_volume_download(dare_volume_t vol, int64_t* cell_starts, int64_t* cell_counts,
                                    float* positions, float* orientations,
                                    uint8_t* intensities) {
  return guard([&] {
    DARE_REQUIRE(vol != nullptr, "null volume handle");
    cudaStream_t s = thread_stream();
    std::vector<uint32_t> offsets(vol->ncells + 1);
    std::vector<uint4> records((size_t)vol->n_samples);
    std::vector<float4> table((size_t)vol->n_orient);
    std::vector<int8_t> perm((size_t)vol->n_samples);
    DARE_CUDA(cudaMemcpyAsync(offsets.data(), vol->d_offsets, sizeof(uint32_t) * offsets.size(),
                              cudaMemcpyDeviceToHost, s));
    if (!records.empty()) {
      DARE_CUDA(cudaMemcpyAsync(records.data(), vol->d_records, sizeof(uint4) * records.size(),
                                cudaMemcpyDeviceToHost, s));
      DARE_CUDA(cudaMemcpyAsync(perm.data(), vol->d_perm, perm.size(), cudaMemcpyDeviceToHost, s));
    }
    if (!table.empty())
      DARE_CUDA(cudaMemcpyAsync(table.data(), vol->d_orient, sizeof(float4) * table.size(),
                                cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaStreamSynchronize(s));
    for (int64_t c = 0; c < vol->ncells; ++c) {
      if (cell_starts) cell_starts[c] = offsets[c];
      if (cell_counts) cell_counts[c] = (int64_t)offsets[c + 1] - offsets[c];
    }
    for (int64_t i = 0; i < vol->n_samples; ++i) {  // insertion order through perm
      const uint4& r = records[i + perm[i]];
      if (positions) std::memcpy(positions + 3 * i, &r, 12);
      if (orientations) std::memcpy(orientations + 4 * i, &table[r.w >> 8], 16);
      if (intensities) intensities[i] = (uint8_t)(r.w & 0xffu);
    }
  });
}

// .darevol writer (volume.py:272-297) streamed from the device: the header,
// the cell table (u64 offset, u32 count per cell, packed 12 B) and the samples
// (3 f32 position, 4 f32 quaternion, u8 intensity, 3 zero bytes = 32 B) in the
// reference's insertion order (records read through perm, quaternions from
// the orientation table).  Chunks are produced by a kernel into device
// scratch, copied into one of two pinned buffers and handed to `write` while
// the next chunk is produced and copied (double buffering) -- host memory
// stays at two chunks whatever the volume size.
namespace {

__global__ void export_table_k(const uint32_t* __restrict__ offsets, int64_t c0, int64_t n,
                               uint32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t a = offsets[c0 + i], b = offsets[c0 + i + 1];
  out[3 * i] = a;  // u64 offset (< 2^32), little-endian
  out[3 * i + 1] = 0u;
  out[3 * i + 2] = b - a;
}

__global__ void export_samples_k(const uint4* __restrict__ records, const int8_t* __restrict__ perm,
                                 const float4* __restrict__ orient, int64_t s0, int64_t n,
                                 uint4* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = s0 + i;
  const uint4 r = records[j + perm[j]];
  const float4 q = orient[r.w >> 8];
  out[2 * i] = make_uint4(r.x, r.y, r.z, __float_as_uint(q.x));
  out[2 * i + 1] = make_uint4(__float_as_uint(q.y), __float_as_uint(q.z), __float_as_uint(q.w), r.w & 0xffu);
}

}  // namespace

extern "C" int dare_volume_save_stream(dare_volume_t vol, dare_write_fn write, void* ctx,
                                       size_t chunk_bytes) {
  return guard([&] {
    DARE_REQUIRE(vol != nullptr && write != nullptr, "null argument");
    DARE_LIMIT(vol->dims[0] < (1ll << 32) && vol->dims[1] < (1ll << 32) && vol->dims[2] < (1ll << 32),
               "dims do not fit the .darevol u32 header fields");
    if (chunk_bytes < (1u << 20)) chunk_bytes = 64u << 20;
    chunk_bytes -= chunk_bytes % 96;  // whole table entries (12 B) and samples (32 B)
    cudaStream_t s = thread_stream();
    // header: "<4sI3dd3IQ" (volume.py:23)
    uint8_t hdr[4 + 4 + 32 + 12 + 8];
    std::memcpy(hdr, "DARE", 4);
    const uint32_t version = 1;
    std::memcpy(hdr + 4, &version, 4);
    std::memcpy(hdr + 8, vol->origin, 24);
    std::memcpy(hdr + 32, &vol->voxel, 8);
    for (int a = 0; a < 3; ++a) {
      const uint32_t d = (uint32_t)vol->dims[a];
      std::memcpy(hdr + 40 + 4 * a, &d, 4);
    }
    const uint64_t count = (uint64_t)vol->n_samples;
    std::memcpy(hdr + 52, &count, 8);
    DARE_REQUIRE(write(ctx, hdr, sizeof(hdr)) == 0, "write callback failed (header)");

    const int64_t cells_per = (int64_t)(chunk_bytes / 12);
    const int64_t samples_per = (int64_t)(chunk_bytes / 32);
    Scratch<uint8_t> dbuf[2] = {Scratch<uint8_t>(chunk_bytes, s), Scratch<uint8_t>(chunk_bytes, s)};
    struct Pinned {
      void* p = nullptr;
      ~Pinned() {
        if (p) cudaFreeHost(p);
      }
    } hbuf[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
    struct Events {
      cudaEvent_t* e;
      ~Events() {
        for (int i = 0; i < 2; ++i)
          if (e[i]) cudaEventDestroy(e[i]);
      }
    } ev_guard{ev};
    for (int i = 0; i < 2; ++i) {
      DARE_CUDA(cudaMallocHost(&hbuf[i].p, chunk_bytes));
      DARE_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    // chunk list: table chunks, then sample chunks
    struct Chunk {
      bool table;
      int64_t first, n;
    };
    std::vector<Chunk> chunks;
    for (int64_t c = 0; c < vol->ncells; c += cells_per)
      chunks.push_back({true, c, std::min(cells_per, vol->ncells - c)});
    for (int64_t j = 0; j < vol->n_samples; j += samples_per)
      chunks.push_back({false, j, std::min(samples_per, vol->n_samples - j)});
    auto bytes_of = [](const Chunk& c) { return (size_t)c.n * (c.table ? 12 : 32); };
    auto produce = [&](size_t k) {
      const Chunk& c = chunks[k];
      void* d = dbuf[k & 1].ptr;
      if (c.table)
        export_table_k<<<ceil_div(c.n, 256), 256, 0, s>>>(vol->d_offsets, c.first, c.n, (uint32_t*)d);
      else
        export_samples_k<<<ceil_div(c.n, 256), 256, 0, s>>>(vol->d_records, vol->d_perm, vol->d_orient,
                                                           c.first, c.n, (uint4*)d);
      DARE_CUDA(cudaGetLastError());
      DARE_CUDA(cudaMemcpyAsync(hbuf[k & 1].p, d, bytes_of(c), cudaMemcpyDeviceToHost, s));
      DARE_CUDA(cudaEventRecord(ev[k & 1], s));
    };
    if (!chunks.empty()) produce(0);
    for (size_t k = 0; k < chunks.size(); ++k) {
      if (k + 1 < chunks.size()) produce(k + 1);  // overlaps the host write of chunk k
      DARE_CUDA(cudaEventSynchronize(ev[k & 1]));
      DARE_REQUIRE(write(ctx, hbuf[k & 1].p, bytes_of(chunks[k])) == 0, "write callback failed");
    }
    DARE_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int dare_volume_get_info(dare_volume_t vol, dare_volume_info* info) {
  return guard([&] {
    DARE_REQUIRE(vol != nullptr && info != nullptr, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->device = vol->device;
    for (int a = 0; a < 3; ++a) {
      info->origin[a] = vol->origin[a];
      info->dims[a] = vol->dims[a];
    }
    info->voxel_size = vol->voxel;
    info->n_samples = vol->n_samples;
    info->n_orientations = vol->n_orient;
    info->rejected_out_of_bounds = vol->rejected;
    info->d_cell_offsets = vol->d_offsets;
    info->d_records = vol->d_records;
    info->d_orientations = (const float*)vol->d_orient;
    info->d_bins = vol->d_bins;
    info->d_perm = vol->d_perm;
    info->device_bytes = sizeof(uint32_t) * (2 * vol->ncells + 1) + (sizeof(uint4) + 1) * vol->n_samples +
                         sizeof(float4) * vol->n_orient + (vol->split_state > 0 ? vol->split_bytes : 0);
  });
}

extern "C" int dare_volume_destroy(dare_volume_t vol) {
  return guard([&] { delete vol; });
}
