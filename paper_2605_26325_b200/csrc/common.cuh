// Shared runtime plumbing for libdare_b200.so: status/error reporting,
// per-thread streams, stream-ordered scratch, and the exact-arithmetic
// helpers every kernel uses.  The whole library is compiled with -fmad=false
// so no multiply-add is ever contracted (the reference never fuses either).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/dare_b200.h"

namespace dare {

void set_error(const std::string& msg);

struct Error {
  int code;
  std::string msg;
};

#define DARE_CUDA(expr)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      throw ::dare::Error{DARE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                             " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
    }                                                                                    \
  } while (0)

#define DARE_REQUIRE(cond, msg)                                   \
  do {                                                            \
    if (!(cond)) throw ::dare::Error{DARE_ERR_INVALID, (msg)};    \
  } while (0)

#define DARE_LIMIT(cond, msg)                                     \
  do {                                                            \
    if (!(cond)) throw ::dare::Error{DARE_ERR_LIMIT, (msg)};      \
  } while (0)

// Runs `body`, converting exceptions into a status code + thread-local message.
template <class F>
int guard(F&& body) {
  try {
    body();
    return DARE_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return DARE_ERR_NOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return DARE_ERR_INVALID;
  }
}

// One non-blocking stream per (host thread, device): concurrent reslice calls
// from different threads never serialise on a shared stream.
cudaStream_t thread_stream();
cudaStream_t thread_copy_stream();  // companion stream for overlapped host<->device copies

// Stream-ordered device scratch (cudaMallocAsync pool) freed on scope exit.
template <class T>
struct Scratch {
  T* ptr = nullptr;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(size_t n, cudaStream_t s) : stream(s) {
    if (n) DARE_CUDA(cudaMallocAsync((void**)&ptr, n * sizeof(T), s));
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// Grow-only device buffer per (host thread, device, slot), for scratch of work
// enqueued on the thread's own stream: stream order makes reuse across calls
// safe and saves the per-call allocator round trips of small launches.
void* thread_arena(int slot, size_t bytes, cudaStream_t s);

// Grow-only pinned host buffer per host thread: staging for small pageable
// host-buffer calls (latency: async copies, one synchronisation).  Contents
// are only valid until the thread's next call.
void* thread_pinned(size_t bytes);
// true when `p` is page-locked (cudaMallocHost / cudaHostRegister) host memory
bool host_pinned(const void* p);

// Bump carving of one scratch block (256 B aligned pieces).
struct Carve {
  uint8_t* base = nullptr;
  size_t off = 0;
  static size_t up(size_t x) { return (x + 255) & ~(size_t)255; }
  template <class T>
  T* take(size_t n) {
    T* p = reinterpret_cast<T*>(base + off);
    off += up(n * sizeof(T));
    return p;
  }
};

// Development aid: with DARE_PROFILE=1 in the environment, records CUDA events
// at phase boundaries on `stream` and prints per-phase device times to stderr
// when it goes out of scope.  No cost when disabled.
class PhaseTimer {
 public:
  PhaseTimer(cudaStream_t s, const char* what);
  ~PhaseTimer();
  void mark(const char* phase);

 private:
  bool on_ = false;
  cudaStream_t s_ = nullptr;
  const char* what_ = nullptr;
  struct Mark {
    const char* name;
    cudaEvent_t ev;
  };
  Mark marks_[32];
  int n_ = 0;
};

// True when 1/x is exactly representable, so (y / x) == (y * (1/x)) bit-for-bit
// (both are the correctly rounded value of the same real number).
inline bool exact_reciprocal(double x) {
  if (!(x > 0.0) || x > 1e300 || x < 1e-300) return false;
  int e;
  double m = frexp(x, &e);
  return m == 0.5;
}

int sm_count();

// Device span of one C-ABI call: events on the call's stream at entry and
// before its final synchronisation; dare_last_device_ms() reports the span of
// the last timed call on this thread (reconstruct / seal / compound / fill).
class DeviceClock {
 public:
  explicit DeviceClock(cudaStream_t s);
  void stop();  // records the end event, waits for it, publishes the span
  ~DeviceClock();

 private:
  cudaStream_t s_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

// Long-lived device buffers (volumes) come from the device's stream-ordered
// pool with an unlimited release threshold, so rebuilding a volume reuses
// memory instead of paying cudaMalloc/cudaFree of multi-GB buffers.
void dev_alloc_bytes(void** p, size_t bytes);
void dev_free(void* p);
template <class T>
inline void dev_alloc(T** p, size_t bytes) {
  dev_alloc_bytes((void**)p, bytes);
}

}  // namespace dare

// ---- device helpers ------------------------------------------------------

// Checked build (build.py --checked -> libdare_b200_checked.so, loaded with
// DARE_CHECKED=1): device-side bounds / invariant asserts at the hot kernels'
// global and shared-memory accesses; a failure prints the condition and traps
// (the launch fails, the tests report it).  No code in the default build.
#ifdef DARE_CHECKED
#define DARE_CHECK(cond)                                                                  \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("DARE_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define DARE_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// The reference's voxel-index chain `floor((f64(p32) - origin) / voxel)`
// (volume.py:209).  When voxel is a power of two the division is replaced by
// the exact reciprocal multiply (identical result, far cheaper on the FP64 pipe).
struct VoxelMap {
  double origin[3];
  double voxel;
  double inv_voxel;
  int exact_inv;
  int64_t dims[3];
};

__device__ __forceinline__ double voxel_coord(const VoxelMap& m, int a, float p32) {
  double d = (double)p32 - m.origin[a];
  return m.exact_inv ? d * m.inv_voxel : d / m.voxel;
}

// Same map with the pixel's U = u * px and V = v * py precomputed (the
// reference's arange(W) * px and arange(H) * py, reconstruct.py:156-158) and
// the voxel division specialised at compile time (kInv: exact reciprocal).
template <bool kInv>
__device__ __forceinline__ int64_t frame_cell(const double* fa, double U, double V,
                                              const VoxelMap& m) {
  bool ok = true;
  int idx[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double P = (U * fa[a] + V * fa[3 + a]) + fa[6 + a];
    const double d = (double)__double2float_rn(P) - m.origin[a];
    // 0 <= floor(q) < n  <=>  0 <= q < n (n integral; NaN fails both): no separate floor
    const double q = kInv ? d * m.inv_voxel : d / m.voxel;
    ok = ok && (q >= 0.0) && (q < (double)m.dims[a]);
    idx[a] = ok ? (int)__double2uint_rz(q) : 0;
  }
  return ok ? ((int64_t)idx[0] * m.dims[1] + idx[1]) * m.dims[2] + idx[2] : -1;
}

// Pixel (u, v) of a frame with axes fa = {c0[3], c1[3], t[3]} ->
// f32 world position (reconstruct.py:156-162) and linear cell (or -1 if out
// of bounds; volume.py:229-230).
__device__ __forceinline__ int64_t pixel_cell(const double* __restrict__ fa, int u, int v,
                                              double px, double py, const VoxelMap& m,
                                              float* p32) {
  double U = (double)u * px;
  double V = (double)v * py;
  bool ok = true;
  int64_t idx[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double P = (U * fa[a] + V * fa[3 + a]) + fa[6 + a];
    float f32 = __double2float_rn(P);
    p32[a] = f32;
    double f = floor(voxel_coord(m, a, f32));
    ok = ok && (f >= 0.0) && (f < (double)m.dims[a]);
    idx[a] = ok ? (int64_t)f : 0;
  }
  return ok ? (idx[0] * m.dims[1] + idx[1]) * m.dims[2] + idx[2] : -1;
}
