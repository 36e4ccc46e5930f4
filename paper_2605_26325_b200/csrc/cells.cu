// Host construction of the exact per-axis threshold tables (cells.cuh).
#include <cmath>
#include <cstring>

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
// non-NaN doubles); +inf when it never holds below +inf.  A narrow bracket
// around `guess` is tried first; the full range otherwise.
template <class Pred>
double threshold(Pred pred, double guess) {
  const uint64_t lo_all = okey(-HUGE_VAL), hi_all = okey(HUGE_VAL);
  uint64_t lo = lo_all, hi = hi_all;  // invariant: pred(lo) false, pred(hi) true
  if (std::isfinite(guess)) {
    const uint64_t g = okey(guess), w = 1ull << 24;
    const uint64_t a = g > lo_all + w ? g - w : lo_all, b = g < hi_all - w ? g + w : hi_all;
    if (!pred(from_okey(a)) && pred(from_okey(b))) {
      lo = a;
      hi = b;
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

}  // namespace

bool build_cell_tables_host(const VoxelMap& m, bool zfine, std::vector<double>& host, size_t off[3],
                            int n_out[3]) {
  host.clear();
  for (int a = 0; a < 3; ++a) {
    const int64_t n = m.dims[a];
    off[a] = host.size();
    std::vector<double> T((size_t)n + 1);
    for (int64_t k = 0; k <= n; ++k)
      T[k] = threshold([&](double P) { return ref_quotient(P, m, a) >= (double)k; },
                       m.origin[a] + (double)k * m.voxel);
    if (a == 2 && zfine) {
      // fine table: cell boundaries interleaved with the z-quarter bounds
      // zb(iz, b) = f32(oz + (iz + b/4) v) (volume.cuh zbin_bound, same expression)
      std::vector<double> F((size_t)(4 * n + 1));
      for (int64_t iz = 0; iz < n; ++iz) {
        F[4 * iz] = T[iz];
        for (int b = 1; b <= 3; ++b) {
          const float zb = (float)(m.origin[2] + ((double)iz + 0.25 * b) * m.voxel);
          F[4 * iz + b] = threshold([&](double P) { return (float)P >= zb; }, (double)zb);
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
  std::vector<double> host;
  size_t off[3];
  if (!build_cell_tables_host(m, zfine, host, off, out.n)) return false;
  out.zfine = zfine ? 1 : 0;
  // storage is an empty Scratch owned by the caller (freed on its scope exit)
  DARE_CUDA(cudaMallocAsync((void**)&storage.ptr, sizeof(double) * host.size(), s));
  storage.stream = s;
  DARE_CUDA(cudaMemcpyAsync(storage.ptr, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, s));
  for (int a = 0; a < 3; ++a) out.t[a] = storage.ptr + off[a];
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
