// Exact pixel -> cell maps through per-axis f64 threshold tables.
//
// The reference maps a world coordinate P (f64, reconstruct.py:156-162) to a
// cell index per axis as floor((f64(f32(P)) - origin) / voxel) (volume.py:209,
// baseline.py:87), in bounds iff 0 <= index < n.  Every step of that chain is
// monotone non-decreasing in P (round-to-nearest f64 -> f32, exact widening,
// correctly rounded subtraction and division / exact-reciprocal multiply,
// floor), so the index is a step function of P: index(P) >= k  <=>  P >= T[k]
// with T[k] = min{P : index(P) >= k}.  The host finds every T[k] (k = 0..n) by
// bisection over the ordered f64 bit patterns, evaluating the reference chain
// itself, so the device never needs the f32 rounding, the division or the
// float->int conversion: a pixel is in cell k of an axis iff T[k] <= P <
// T[k+1], and in bounds iff T[0] <= P < T[n] (NaN fails every comparison).
//
// The reconstruction's z-quarter bins (volume.cuh: bin b of cell iz holds
// f32(P) >= zb(iz, b)) are folded into a fine z table F[4 iz + b] (b = 1..3:
// the smallest P whose f32 reaches zb(iz, b)); when F is non-decreasing (the
// host checks it) the fine index m gives cell m >> 2 and bin m & 3.
//
// Threads track the interval [lo, hi) of their current index per axis: a
// pixel stays in one cell for several consecutive frames of a sweep, so the
// common frame costs two compares per axis and only a crossing walks the
// table (one step per boundary crossed).
#pragma once
#include <math_constants.h>

#include <vector>

#include "common.cuh"

namespace dare {

struct CellTables {
  const double* t[3] = {nullptr, nullptr, nullptr};  // device: x (nx+1), y (ny+1), z (nz+1 or 4nz+1)
  int n[3] = {0, 0, 0};                                // number of intervals per table (nx, ny, nz or 4nz)
  int zfine = 0;                                       // z table is the fine (cell, quarter) table
};

// Host: builds the tables into `storage` (device memory allocated on stream s,
// owned by the caller's Scratch).  Returns false when the fine z table is not
// monotone (the caller then uses its plain path); never for plain tables.
bool build_cell_tables(const VoxelMap& m, bool zfine, cudaStream_t s, Scratch<double>& storage,
                       CellTables& out);
bool build_cell_tables_host(const VoxelMap& m, bool zfine, std::vector<double>& host, size_t off[3],
                            int n_out[3]);

struct AxisCell {
  int g;           // current interval: -1 below T[0], n at/above T[n] (out of bounds)
  double lo, hi;   // T[g], T[g+1] (+-inf outside)
};

// (Re)locates P in table T (n intervals) starting from a.g; exact.
__device__ __forceinline__ void axis_locate(double P, const double* __restrict__ T, int n, AxisCell& a) {
  if (!(P == P)) {  // NaN: out of bounds, and every later fast check fails
    a.g = -1;
    a.lo = a.hi = P;
    return;
  }
  int g = a.g;
  if (g < -1 || g > n) g = -1;
  while (g < n && __ldg(T + g + 1) <= P) ++g;
  while (g >= 0 && P < __ldg(T + g)) --g;
  a.g = g;
  a.lo = g >= 0 ? __ldg(T + g) : -CUDART_INF;
  a.hi = g < n ? __ldg(T + g + 1) : CUDART_INF;
}

__device__ __forceinline__ bool axis_same(double P, const AxisCell& a) { return a.lo <= P && P < a.hi; }

// z on the fine table, tracked at cell granularity: the interval is the cell
// [F[4g], F[4g+4]) and q1..q3 = F[4g+1..3] give the quarter bin by compares.
struct AxisCellZ {
  int g;  // cell index, -1 below, n at/above (out of bounds)
  double lo, hi, q1, q2, q3;
  __device__ __forceinline__ uint32_t bin(double P) const {
    return (uint32_t)(P >= q1) + (uint32_t)(P >= q2) + (uint32_t)(P >= q3);
  }
};

__device__ __forceinline__ void axis_locate_z(double P, const double* __restrict__ F, int n, AxisCellZ& a) {
  if (!(P == P)) {
    a.g = -1;
    a.lo = a.hi = P;
    return;
  }
  int g = a.g;
  if (g < -1 || g > n) g = -1;
  while (g < n && __ldg(F + 4 * (g + 1)) <= P) ++g;
  while (g >= 0 && P < __ldg(F + 4 * g)) --g;
  a.g = g;
  if (g >= 0 && g < n) {
    a.lo = __ldg(F + 4 * g);
    a.q1 = __ldg(F + 4 * g + 1);
    a.q2 = __ldg(F + 4 * g + 2);
    a.q3 = __ldg(F + 4 * g + 3);
    a.hi = __ldg(F + 4 * g + 4);
  } else {
    a.lo = g < 0 ? -CUDART_INF : __ldg(F + 4 * n);
    a.hi = g < 0 ? __ldg(F) : CUDART_INF;
    a.q1 = a.q2 = a.q3 = CUDART_INF;
  }
}

// First guess of the interval of P (any value works; it only shortens the walk).
__device__ __forceinline__ int axis_guess(double P, double origin, double inv_voxel, int n, int fine) {
  const double q = (P - origin) * inv_voxel * (fine ? 4.0 : 1.0);
  return q != q ? -1 : (q < -1.0 ? -1 : (q > (double)n ? n : (int)q));
}

}  // namespace dare
