// Host construction of the exact per-axis threshold tables (cells.cuh).
#include <cmath>
#include <cstring>
#include <mutex>

#include "cells.cuh"
#include "volume.cuh"

namespace dare {

namespace {

uint64_t okey(double x) {  // order-preserving map of non-NaN doubles to uint64
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

double from_okey(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
  std::memcpy(&x, &u, 8);
  return x;
}

// The reference's per-axis chain up to the quotient: ((double)(float)P - o) / v
// (volume.py:209), with the device's exact-reciprocal form when 1/v is exact.
double ref_quotient(double P, const VoxelMap& m, int a) {
  const float p32 = (float)P;  // round to nearest even, like __double2float_rn
  const double d = (double)p32 - m.origin[a];
  return m.exact_inv ? d * m.inv_voxel : d / m.voxel;
}

// Smallest double P with pred(P) true (pred monotone false -> true over the
// non-NaN doubles); +inf when it never holds below +inf.  The search brackets
// the answer by doubling a window around `guess` (the true threshold is a few
// ulps from it), then bisects; the full range is the fallback.
template <class Pred>
double threshold(Pred pred, double guess) {
  const uint64_t lo_all = okey(-HUGE_VAL), hi_all = okey(HUGE_VAL);
  uint64_t lo = lo_all, hi = hi_all;  // invariant: pred(lo) false, pred(hi) true
  if (std::isfinite(guess)) {
    const uint64_t g = okey(guess);
    for (uint64_t w = 4; w <= (1ull << 40); w <<= 3) {
      const uint64_t a = g > lo_all + w ? g - w : lo_all, b = g < hi_all - w ? g + w : hi_all;
      if (!pred(from_okey(a)) && pred(from_okey(b))) {
        lo = a;
        hi = b;
        break;
      }
    }
  }
  if (pred(from_okey(lo))) return from_okey(lo);
  if (!pred(from_okey(hi))) return HUGE_VAL;
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (pred(from_okey(mid)))
      hi = mid;
    else
      lo = mid;
  }
  return from_okey(hi);
}

// Smallest double P with (float)P >= ps (ps finite): just above or at the
// midpoint between ps and its f32 predecessor (ties round to the even one).
double float_threshold(float ps) {
  const float pm = std::nextafter(ps, -HUGE_VALF);
  const double mid = 0.5 * ((double)pm + (double)ps);  // exact
  return (float)mid >= ps ? mid : std::nextafter(mid, HUGE_VAL);
}

// T with pred(T) true and pred(prev(T)) false when `cand` is right, else the
// bisection.  pred over doubles is what defines the table.
template <class Pred>
double checked(Pred pred, double cand, double guess) {
  if (std::isfinite(cand) && pred(cand) && !pred(std::nextafter(cand, -HUGE_VAL))) return cand;
  return threshold(pred, guess);
}

}  // namespace

bool build_cell_tables_host(const VoxelMap& m, bool zfine, std::vector<double>& host, size_t off[3],
                            int n_out[3]) {
  host.clear();
  for (int a = 0; a < 3; ++a) {
    const int64_t n = m.dims[a];
    off[a] = host.size();
    std::vector<double> T((size_t)n + 1);
    for (int64_t k = 0; k <= n; ++k) {
      auto pred = [&](double P) { return ref_quotient(P, m, a) >= (double)k; };
      // the smallest f32 p with quotient >= k, by f32 steps from the nearest guess,
      // then the smallest f64 rounding to it
      const double guess = m.origin[a] + (double)k * m.voxel;
      float p = (float)guess;
      for (int i = 0; i < 16 && ref_quotient((double)std::nextafter(p, -HUGE_VALF), m, a) >= (double)k; ++i)
        p = std::nextafter(p, -HUGE_VALF);
      for (int i = 0; i < 16 && !(ref_quotient((double)p, m, a) >= (double)k); ++i) p = std::nextafter(p, HUGE_VALF);
      T[k] = checked(pred, float_threshold(p), guess);
    }
    if (a == 2 && zfine) {
      // fine table: cell boundaries interleaved with the z-quarter bounds
      // zb(iz, b) = f32(oz + (iz + b/4) v) (volume.cuh zbin_bound, same expression)
      std::vector<double> F((size_t)(4 * n + 1));
      for (int64_t iz = 0; iz < n; ++iz) {
        F[4 * iz] = T[iz];
        for (int b = 1; b <= 3; ++b) {
          const float zb = (float)(m.origin[2] + ((double)iz + 0.25 * b) * m.voxel);
          F[4 * iz + b] = checked([&](double P) { return (float)P >= zb; }, float_threshold(zb), (double)zb);
        }
      }
      F[4 * n] = T[n];
      for (size_t i = 1; i < F.size(); ++i)
        if (!(F[i - 1] <= F[i])) return false;
      host.insert(host.end(), F.begin(), F.end());
      n_out[a] = (int)(4 * n);
    } else {
      host.insert(host.end(), T.begin(), T.end());
      n_out[a] = (int)n;
    }
  }
  return true;
}

bool build_cell_tables(const VoxelMap& m, bool zfine, cudaStream_t s, Scratch<double>& storage,
                       CellTables& out) {
  // per-process cache of the tables, on the device as well: rebuilding a
  // volume (or compounding) on the same grid costs no host work and no
  // upload.  Entries are never freed (kernels of other threads may use them);
  // past kMaxEntries grids the tables go into the caller's scratch instead.
  constexpr size_t kMaxEntries = 64;
  struct Entry {
    int device;
    double key[8];
    bool ok;
    int n[3];
    size_t off[3];
    double* d;  // device copy
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  DARE_CUDA(cudaGetDevice(&dev));
  const double key[8] = {m.origin[0], m.origin[1], m.origin[2], m.voxel, (double)m.dims[0], (double)m.dims[1],
                         (double)m.dims[2], zfine ? 1.0 : 0.0};
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
      if (e.device == dev && std::memcmp(e.key, key, sizeof(key)) == 0) {
        if (!e.ok) return false;
        std::memcpy(out.n, e.n, sizeof(e.n));
        for (int a = 0; a < 3; ++a) out.t[a] = e.d + e.off[a];
        out.zfine = zfine ? 1 : 0;
        return true;
      }
  }
  std::vector<double> host;
  Entry e;
  e.device = dev;
  std::memcpy(e.key, key, sizeof(key));
  e.ok = build_cell_tables_host(m, zfine, host, e.off, e.n);
  e.d = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (e.ok && cache.size() < kMaxEntries) {
    DARE_CUDA(cudaMalloc((void**)&e.d, sizeof(double) * host.size()));
    DARE_CUDA(cudaMemcpy(e.d, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice));
    cache.push_back(e);
  } else if (!e.ok && cache.size() < kMaxEntries) {
    cache.push_back(e);
  }
  if (!e.ok) return false;
  std::memcpy(out.n, e.n, sizeof(e.n));
  out.zfine = zfine ? 1 : 0;
  if (e.d) {
    for (int a = 0; a < 3; ++a) out.t[a] = e.d + e.off[a];
    return true;
  }
  // cache full: the caller's stream-ordered scratch
  DARE_CUDA(cudaMallocAsync((void**)&storage.ptr, sizeof(double) * host.size(), s));
  storage.stream = s;
  DARE_CUDA(cudaMemcpyAsync(storage.ptr, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, s));
  for (int a = 0; a < 3; ++a) out.t[a] = storage.ptr + e.off[a];
  return true;
}

}  // namespace dare

using namespace dare;

// Diagnostic (host only, no device): the tables as built for a grid, for the
// CPU tests of their exactness.  out: (nx+1) + (ny+1) + (nz+1 or 4nz+1) doubles.
extern "C" int dare_cell_thresholds(const double* origin, double voxel_size, const int64_t* dims,
                                    int32_t zfine, double* out, int64_t* n_out) {
  return guard([&] {
    DARE_REQUIRE(voxel_size > 0 && dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "bad grid");
    VoxelMap m = make_voxel_map(origin, voxel_size, dims);
    std::vector<double> host;
    size_t off[3];
    int n[3];
    if (!build_cell_tables_host(m, zfine != 0, host, off, n)) {
      for (int a = 0; a < 3; ++a) n_out[a] = -1;
      return;
    }
    std::memcpy(out, host.data(), sizeof(double) * host.size());
    for (int a = 0; a < 3; ++a) n_out[a] = n[a];
  });
}
