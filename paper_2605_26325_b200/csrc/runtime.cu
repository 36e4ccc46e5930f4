// Runtime entry points of the C ABI: errors, devices, streams, memory.
#include <map>
#include <mutex>

#include "volume.cuh"

namespace dare {

static thread_local std::string g_last_error;
static thread_local double g_last_device_ms = -1.0;

DeviceClock::DeviceClock(cudaStream_t s) : s_(s) {
  DARE_CUDA(cudaEventCreate(&a_));
  DARE_CUDA(cudaEventCreate(&b_));
  DARE_CUDA(cudaEventRecord(a_, s_));
}

void DeviceClock::stop() {
  DARE_CUDA(cudaEventRecord(b_, s_));
  DARE_CUDA(cudaEventSynchronize(b_));
  float ms = 0.f;
  DARE_CUDA(cudaEventElapsedTime(&ms, a_, b_));
  g_last_device_ms = ms;
}

DeviceClock::~DeviceClock() {
  if (a_) cudaEventDestroy(a_);
  if (b_) cudaEventDestroy(b_);
}

void set_error(const std::string& msg) { g_last_error = msg; }

cudaStream_t thread_stream() {
  // One stream per (thread, device); destroyed with the thread.
  struct Streams {
    std::map<int, cudaStream_t> by_dev;
    ~Streams() {
      for (auto& kv : by_dev) cudaStreamDestroy(kv.second);
    }
  };
  static thread_local Streams streams;
  int dev = 0;
  DARE_CUDA(cudaGetDevice(&dev));
  auto it = streams.by_dev.find(dev);
  if (it != streams.by_dev.end()) return it->second;
  cudaStream_t s;
  DARE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  streams.by_dev[dev] = s;
  static std::mutex mu;
  static std::map<int, bool> pool_done;
  std::lock_guard<std::mutex> lock(mu);
  if (!pool_done[dev]) {
    cudaMemPool_t pool;
    DARE_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    DARE_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    pool_done[dev] = true;
  }
  return s;
}

cudaStream_t thread_copy_stream() {
  // Second per-(thread, device) stream for host<->device copies overlapping compute.
  struct Streams {
    std::map<int, cudaStream_t> by_dev;
    ~Streams() {
      for (auto& kv : by_dev) cudaStreamDestroy(kv.second);
    }
  };
  static thread_local Streams streams;
  int dev = 0;
  DARE_CUDA(cudaGetDevice(&dev));
  auto it = streams.by_dev.find(dev);
  if (it != streams.by_dev.end()) return it->second;
  cudaStream_t s;
  DARE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  streams.by_dev[dev] = s;
  return s;
}

void dev_alloc_bytes(void** p, size_t bytes) {
  cudaStream_t s = thread_stream();
  DARE_CUDA(cudaMallocAsync(p, bytes ? bytes : 1, s));
  DARE_CUDA(cudaStreamSynchronize(s));  // usable from any stream once this returns
}

void* thread_arena(int slot, size_t bytes, cudaStream_t s) {
  struct Block {
    void* p = nullptr;
    size_t cap = 0;
  };
  struct Arena {
    std::map<std::pair<int, int>, Block> blocks;
    ~Arena() {
      for (auto& kv : blocks)
        if (kv.second.p) cudaFree(kv.second.p);
    }
  };
  static thread_local Arena arena;
  int dev = 0;
  DARE_CUDA(cudaGetDevice(&dev));
  Block& b = arena.blocks[{dev, slot}];
  if (b.cap < bytes) {
    const size_t old_cap = b.cap;
    if (b.p) DARE_CUDA(cudaFreeAsync(b.p, s));
    b.p = nullptr;
    b.cap = 0;
    const size_t want = std::max(bytes, old_cap * 2);  // geometric growth
    DARE_CUDA(cudaMallocAsync(&b.p, want, s));
    b.cap = want;
  }
  return b.p;
}

void* thread_pinned(size_t bytes) {
  struct Pinned {
    void* p = nullptr;
    size_t cap = 0;
    ~Pinned() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Pinned b;
  if (b.cap < bytes) {
    const size_t old_cap = b.cap;
    if (b.p) DARE_CUDA(cudaFreeHost(b.p));
    b.p = nullptr;
    b.cap = 0;
    // sized to the request (rounded to 64 KB) the first time -- a service's
    // per-connection threads each own one -- then geometric growth: pinned
    // allocations are slow and cudaFreeHost synchronises
    const size_t want = std::max<size_t>((bytes + 0xffff) & ~(size_t)0xffff, 2 * old_cap);
    DARE_CUDA(cudaMallocHost(&b.p, want));
    b.cap = want;
  }
  return b.p;
}

bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // clear: plain pageable memory on older runtimes
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

void dev_free(void* p) {
  if (!p) return;
  try {
    cudaFreeAsync(p, thread_stream());
  } catch (...) {
  }
}

int sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  DARE_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  DARE_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = n;
  return n;
}

PhaseTimer::PhaseTimer(cudaStream_t s, const char* what) : s_(s), what_(what) {
  const char* env = getenv("DARE_PROFILE");
  on_ = env && env[0] && env[0] != '0';
  if (on_) mark("start");
}

void PhaseTimer::mark(const char* phase) {
  if (!on_ || n_ >= 32) return;
  cudaEventCreate(&marks_[n_].ev);
  cudaEventRecord(marks_[n_].ev, s_);
  marks_[n_].name = phase;
  ++n_;
}

PhaseTimer::~PhaseTimer() {
  if (!on_) return;
  mark("end");
  cudaEventSynchronize(marks_[n_ - 1].ev);
  float total = 0;
  cudaEventElapsedTime(&total, marks_[0].ev, marks_[n_ - 1].ev);
  fprintf(stderr, "[dare-profile] %s total %.3f ms:", what_, total);
  for (int i = 1; i < n_; ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, marks_[i - 1].ev, marks_[i].ev);
    fprintf(stderr, " %s=%.3f", marks_[i].name, ms);
  }
  fprintf(stderr, "\n");
  for (int i = 0; i < n_; ++i) cudaEventDestroy(marks_[i].ev);
}

VoxelMap make_voxel_map(const double* origin, double voxel, const int64_t* dims) {
  VoxelMap m;
  for (int a = 0; a < 3; ++a) {
    m.origin[a] = origin[a];
    m.dims[a] = dims[a];
  }
  m.voxel = voxel;
  m.exact_inv = exact_reciprocal(voxel) ? 1 : 0;
  m.inv_voxel = 1.0 / voxel;
  return m;
}

FrameSet::FrameSet(const uint8_t* frames, int64_t n_images, int32_t H_, int32_t W_,
                   int32_t on_device, const int32_t* frame_image, int64_t n_frames_,
                   const double* axes, double px_, double py_, const uint8_t* mask,
                   cudaStream_t s)
    : n_frames(n_frames_), H(H_), W(W_), px(px_), py(py_), stream(s) {
  DARE_REQUIRE(H > 0 && W > 0, "frame height and width must be positive");
  DARE_REQUIRE(n_frames >= 0 && n_images >= 0, "negative frame count");
  const size_t hw = (size_t)H * W;
  for (int64_t i = 0; i < n_frames; ++i)
    DARE_REQUIRE(frame_image[i] >= 0 && frame_image[i] < n_images, "frame_image index out of range");
  if (on_device) {
    d_frames = frames;
  } else {
    size_t bytes = hw * (size_t)n_images;
    if (bytes) {
      // grouped upload on the copy stream (start_upload): the count pass (which
      // needs no intensities) and the early fill launches overlap the transfer
      DARE_CUDA(cudaMallocAsync((void**)&owned_frames, bytes, s));
      h_frames = frames;
      this->n_images = n_images;
      h_image.assign(frame_image, frame_image + n_frames);
    }
    d_frames = owned_frames;
  }
  if (n_frames) {
    DARE_CUDA(cudaMallocAsync((void**)&d_image, sizeof(int32_t) * n_frames, s));
    DARE_CUDA(cudaMemcpyAsync(d_image, frame_image, sizeof(int32_t) * n_frames,
                              cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMallocAsync((void**)&d_axes, sizeof(double) * 9 * n_frames, s));
    DARE_CUDA(cudaMemcpyAsync(d_axes, axes, sizeof(double) * 9 * n_frames,
                              cudaMemcpyHostToDevice, s));
  }
  if (mask) {
    DARE_CUDA(cudaMallocAsync((void**)&d_mask, hw, s));
    DARE_CUDA(cudaMemcpyAsync(d_mask, mask, hw, cudaMemcpyHostToDevice, s));
  }
}

void FrameSet::start_upload() {
  if (!h_frames || !done.empty()) return;
  const size_t hw = (size_t)H * W;
  cudaEvent_t ready;
  DARE_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  DARE_CUDA(cudaEventRecord(ready, stream));  // allocation visible to the copy stream
  cudaStream_t cs = thread_copy_stream();
  DARE_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  DARE_CUDA(cudaEventDestroy(ready));
  const int64_t groups = std::min<int64_t>(8, n_images);
  per_group = (n_images + groups - 1) / groups;
  for (int64_t g = 0; g * per_group < n_images; ++g) {
    const int64_t i0 = g * per_group, i1 = std::min(n_images, i0 + per_group);
    DARE_CUDA(cudaMemcpyAsync(owned_frames + hw * (size_t)i0, h_frames + hw * (size_t)i0,
                              hw * (size_t)(i1 - i0), cudaMemcpyHostToDevice, cs));
    cudaEvent_t e;
    DARE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    DARE_CUDA(cudaEventRecord(e, cs));
    done.push_back(e);
  }
}

void FrameSet::wait_frames(cudaStream_t s, int64_t f_begin, int64_t f_end) const {
  if (done.empty() || f_begin >= f_end) return;
  int32_t last = 0;
  for (int64_t f = f_begin; f < f_end; ++f) last = std::max(last, h_image[f]);
  DARE_CUDA(cudaStreamWaitEvent(s, done[std::min<size_t>(last / per_group, done.size() - 1)], 0));
}

FrameSet::~FrameSet() {
  // no DMA may still read the caller's host frames when the call returns (a
  // block may reference only some upload groups): wait for the last copy
  if (!done.empty()) cudaEventSynchronize(done.back());
  for (cudaEvent_t e : done) cudaEventDestroy(e);
  if (owned_frames) cudaFreeAsync(owned_frames, stream);
  if (d_image) cudaFreeAsync(d_image, stream);
  if (d_axes) cudaFreeAsync(d_axes, stream);
  if (d_mask) cudaFreeAsync(d_mask, stream);
}

}  // namespace dare

dare_volume_s::~dare_volume_s() {
  using dare::dev_free;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  // work enqueued by *_device calls on caller streams may still read the
  // volume: nothing orders those streams before this free, so wait for the device
  cudaDeviceSynchronize();
  dev_free(d_offsets);
  dev_free(d_records);
  dev_free(d_orient);
  dev_free(d_bins);
  dev_free(d_perm);
  dev_free(d_soffsets);
  dev_free(d_sbins);
  dev_free(d_srecords);
  dev_free(d_ocluster);
  cudaSetDevice(prev);
}

dare_scalar_s::~dare_scalar_s() {
  using dare::dev_free;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  dev_free(d_values);
  dev_free(d_flags);
  dev_free(d_counts);
  cudaSetDevice(prev);
}

using namespace dare;

extern "C" {

const char* dare_last_error(void) { return g_last_error.c_str(); }

int dare_version(void) { return 200; }

int dare_last_device_ms(double* ms) {
  return guard([&] {
    DARE_REQUIRE(ms != nullptr, "null argument");
    *ms = g_last_device_ms;
  });
}

int dare_get_device_count(int32_t* count) {
  return guard([&] {
    int n = 0;
    DARE_CUDA(cudaGetDeviceCount(&n));
    *count = n;
  });
}

int dare_set_device(int32_t device) { return guard([&] { DARE_CUDA(cudaSetDevice(device)); }); }

int dare_synchronize(void) { return guard([&] { DARE_CUDA(cudaDeviceSynchronize()); }); }

int dare_host_alloc(size_t bytes, void** ptr) {
  return guard([&] { DARE_CUDA(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable)); });
}

int dare_host_free(void* ptr) { return guard([&] { DARE_CUDA(cudaFreeHost(ptr)); }); }

int dare_device_alloc(size_t bytes, void** ptr) {
  return guard([&] { DARE_CUDA(cudaMalloc(ptr, bytes)); });
}

int dare_device_free(void* ptr) { return guard([&] { DARE_CUDA(cudaFree(ptr)); }); }

int dare_memcpy(void* dst, const void* src, size_t bytes, void* stream) {
  return guard([&] {
    cudaStream_t s = stream ? (cudaStream_t)stream : thread_stream();
    DARE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    if (!stream) DARE_CUDA(cudaStreamSynchronize(s));
  });
}

int dare_trim(size_t keep_bytes) {
  return guard([&] {
    int dev = 0;
    DARE_CUDA(cudaGetDevice(&dev));
    DARE_CUDA(cudaDeviceSynchronize());  // pending frees of every stream complete
    cudaMemPool_t pool;
    DARE_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    DARE_CUDA(cudaMemPoolTrimTo(pool, keep_bytes));
  });
}

int dare_stream_sync(void* stream) {
  return guard([&] {
    DARE_CUDA(cudaStreamSynchronize(stream ? (cudaStream_t)stream : thread_stream()));
  });
}

}  // extern "C"
