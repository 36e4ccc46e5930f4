// Image similarity for the evaluation harness: the
// reference's masked NCC and SSIM (evaluation.py:28-84) and compare_images
// (evaluation.py:150-160) for a batch of image pairs of one size.
//
// Exactness.  The reference reduces with numpy: means are np.add.reduce
// (pairwise summation, numpy loops_utils.h.src) divided by the count, SSIM's
// window moments are sums over 7x7 views and the final score is the mean of
// the per-window values of the complete windows in row-major order.
//   * window moments: integer-valued pixels (the u8 reslice images) give
//     exact f64 sums in any order, so per-window values are bit-identical to
//     the reference's elementwise f64 chain (-fmad=false, same association);
//   * the mean over complete windows and the NCC means use numpy's pairwise
//     order exactly (pw_reduce below), so SSIM is bit-identical to the
//     reference for integer-valued images and the NCC means are too;
//   * the NCC dot products are np.dot (BLAS; its summation order depends on
//     the host's OpenBLAS kernel and thread count): here they use the same
//     pairwise order, so NCC agrees to rounding (tests: 1e-12).
//
// Layout: a, b [pairs][H][W] (u8 or f64), optional u8 masks of the same
// shape (null = all valid).  Kernels: ssim_window_k (per-window values,
// separable 7x7 sums through a shared-memory ring), sim_reduce_k (one CTA per
// pair: compaction + pairwise reductions).  HBM-bound: ~3 B/pixel read (u8
// images + masks) + 9 B/window written and re-read; evaluation is off the hot
// path (the reference spends ~0.3 s per 512^2 pair in numpy).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace dare {
namespace {

constexpr int kReduceThreads = 512;
constexpr int kItems = 8;         // compaction: consecutive elements per thread per chunk
constexpr int kLeaf = 128;        // numpy PW_BLOCKSIZE
constexpr int kBand = 64;         // output window rows per ssim_window_k block

// ---- numpy pairwise summation order ---------------------------------------
// pairwise_sum(a, n): n < 8 -> sequential from -0.0; n <= 128 -> eight
// accumulators over the multiple-of-8 prefix, combined ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)), then the tail sequentially; else split at
// n2 = n/2 - (n/2)%8 and add the halves.  The tree is a function of n only;
// nodes are addressed by (depth d, index k) along the bits of k.  A node's
// right child is never smaller than its left, so the deepest leaf lies on the
// right spine.

__host__ __device__ inline int pw_depth(int64_t n) {
  int d = 0;
  while (n > kLeaf) {
    n -= n / 2 - (n / 2) % 8;
    ++d;
  }
  return d;
}

// Walks to node (d, k).  Returns false when an ancestor is already a leaf.
__device__ inline bool pw_node(int64_t n, int d, int64_t k, int64_t& off, int64_t& len) {
  off = 0;
  len = n;
  for (int i = d - 1; i >= 0; --i) {
    if (len <= kLeaf) return false;
    const int64_t n2 = len / 2 - (len / 2) % 8;
    if ((k >> i) & 1) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  return true;
}

// K parallel sums over i in [0, n) of f(i)[0..K) in numpy's pairwise order.
// S: 2^D x K doubles of scratch (D = pw_depth(n)); the result lands in S[0..K).
// Leaves are summed by groups of 8 lanes: lane u keeps numpy's accumulator
// r[u] (elements u, u+8, ... of the leaf, so each step's 8 loads are one
// coalesced 64 B segment), the group combines ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)) with shuffles in exactly that association, and lane 0
// adds the tail.
template <int K, class Fn>
__device__ void pw_reduce(int64_t n, Fn f, double* S) {
  const int D = pw_depth(n);
  const int64_t slots = (int64_t)1 << D;
  const uint32_t lane = threadIdx.x & 31u, u = lane & 7u;
  const unsigned gmask = 0xffu << (lane & ~7u);
  const int64_t groups = blockDim.x >> 3;
  // leaves: slot j represents the leaf containing it if j's bits below the
  // leaf's depth are zero
  for (int64_t j = threadIdx.x >> 3; j < slots; j += groups) {
    int64_t off = 0, len = n;
    int d = 0;
    while (len > kLeaf) {
      const int64_t n2 = len / 2 - (len / 2) % 8;
      if ((j >> (D - 1 - d)) & 1) {
        off += n2;
        len -= n2;
      } else {
        len = n2;
      }
      ++d;
    }
    if (d < D && (j & ((((int64_t)1) << (D - d)) - 1)) != 0) continue;  // group-uniform
    double res[K];
    if (len < 8) {
      if (u == 0) {
#pragma unroll
        for (int c = 0; c < K; ++c) res[c] = -0.0;
        for (int64_t i = 0; i < len; ++i) {
          double v[K];
          f(off + i, v);
#pragma unroll
          for (int c = 0; c < K; ++c) res[c] += v[c];
        }
#pragma unroll
        for (int c = 0; c < K; ++c) S[j * K + c] = res[c];
      }
      continue;
    }
    double r[K];
    f(off + u, r);
    const int64_t body = len - (len % 8);
    for (int64_t i = 8; i < body; i += 8) {
      double v[K];
      f(off + i + u, v);
#pragma unroll
      for (int c = 0; c < K; ++c) r[c] += v[c];
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double x = r[c] + __shfl_down_sync(gmask, r[c], 1, 8);  // u even: r_u + r_{u+1}
      x = x + __shfl_down_sync(gmask, x, 2, 8);               // u % 4 == 0: (..) + (..)
      x = x + __shfl_down_sync(gmask, x, 4, 8);               // u == 0: the full combination
      res[c] = x;
    }
    if (u == 0) {
      for (int64_t i = body; i < len; ++i) {
        double v[K];
        f(off + i, v);
#pragma unroll
        for (int c = 0; c < K; ++c) res[c] += v[c];
      }
#pragma unroll
      for (int c = 0; c < K; ++c) S[j * K + c] = res[c];
    }
  }
  __syncthreads();
  // combine bottom-up: an internal node (d, k) adds its right child's sum
  // (slot (2k+1) << (D-d-1)) into its left child's slot (k << (D-d))
  for (int d = D - 1; d >= 0; --d) {
    for (int64_t k = threadIdx.x; k < ((int64_t)1 << d); k += blockDim.x) {
      int64_t off, len;
      if (!pw_node(n, d, k, off, len) || len <= kLeaf) continue;
      const int64_t L = k << (D - d), R = (2 * k + 1) << (D - d - 1);
#pragma unroll
      for (int c = 0; c < K; ++c) S[L * K + c] = S[L * K + c] + S[R * K + c];
    }
    __syncthreads();
  }
}

// CTA-wide stable compaction of the flagged elements of [0, n) into out
// (order preserved).  Returns the count (all threads).
template <class Flag, class Emit>
__device__ int64_t compact(int64_t n, Flag flag, Emit emit) {
  __shared__ int warp_tot[kReduceThreads / 32];
  __shared__ int64_t base_s;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t chunk = (int64_t)blockDim.x * kItems;
  for (int64_t c0 = 0; c0 < n; c0 += chunk) {
    const int64_t i0 = c0 + (int64_t)threadIdx.x * kItems;
    unsigned bits = 0;
#pragma unroll
    for (int u = 0; u < kItems; ++u)
      if (i0 + u < n && flag(i0 + u)) bits |= 1u << u;
    const int cnt = __popc(bits);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      const int t = warp_tot[w];
      if (w < warp) before += t;
      total += t;
    }
    int64_t pos = base_s + before + incl - cnt;
#pragma unroll
    for (int u = 0; u < kItems; ++u)
      if (bits & (1u << u)) emit(i0 + u, pos++);
    __syncthreads();
    if (threadIdx.x == 0) base_s += total;
    __syncthreads();
  }
  return base_s;
}

template <class T>
__device__ __forceinline__ double ld(const T* p, size_t k) {
  return (double)p[k];
}

__device__ __forceinline__ bool valid_at(const uint8_t* am, const uint8_t* bm, size_t k) {
  return (am == nullptr || am[k] != 0) && (bm == nullptr || bm[k] != 0);
}

// Per-window SSIM value + completeness for output rows [y0, y0+band) of one
// pair; thread = window column.  Each image row's horizontal sums (a, b, a^2,
// b^2, ab, mask) enter a ring of the last `win` rows in shared memory; a
// window sums its rows top to bottom, each row left to right.
template <class T>
__global__ void __launch_bounds__(128) ssim_window_k(const T* __restrict__ a, const uint8_t* __restrict__ am,
                                                     const T* __restrict__ b, const uint8_t* __restrict__ bm,
                                                     int H, int W, int win, double c1, double c2,
                                                     double* __restrict__ V, uint8_t* __restrict__ F) {
  extern __shared__ double sm[];
  const int nt = blockDim.x, tid = threadIdx.x;
  const int HH = H - win + 1, WW = W - win + 1;
  const int64_t pair = blockIdx.z;
  const int x0 = blockIdx.x * nt, x = x0 + tid;
  const int y0 = blockIdx.y * kBand;
  if (y0 >= HH) return;
  const int y1 = min(y0 + kBand, HH);
  const int span = nt + win - 1;
  double* ring = sm;                       // [win][6][nt]
  double* st = sm + (size_t)win * 6 * nt;  // [3][span]
  const size_t base = (size_t)pair * H * W;
  // evaluation.py:73-80: n = window*window, unbiased norm n / (n - 1.0)
  const double n = (double)(win * win);
  const double norm = n / (n - 1.0);
  int slot = 0;  // (r - y0) mod win, kept incrementally
  for (int r = y0; r < y1 + win - 1; ++r, slot = slot + 1 == win ? 0 : slot + 1) {
    __syncthreads();
    for (int i = tid; i < span; i += nt) {
      const int c = x0 + i;
      double va = 0.0, vb = 0.0, vm = 0.0;
      if (c < W) {
        const size_t k = base + (size_t)r * W + c;
        va = ld(a, k);
        vb = ld(b, k);
        vm = valid_at(am, bm, k) ? 1.0 : 0.0;
      }
      st[i] = va;
      st[span + i] = vb;
      st[2 * span + i] = vm;
    }
    __syncthreads();
    double h[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < win; ++j) {
      const double p = st[tid + j], q = st[span + tid + j];
      h[0] += p;
      h[1] += q;
      h[2] += p * p;
      h[3] += q * q;
      h[4] += p * q;
      h[5] += st[2 * span + tid + j];
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) ring[((size_t)slot * 6 + c) * nt + tid] = h[c];
    const int y = r - (win - 1);
    if (y >= y0 && x < WW) {
      double s[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      // rows y .. r in order: row y's slot follows row r's in the ring of win
      for (int j = 0, sl = slot + 1 == win ? 0 : slot + 1; j < win; ++j, sl = sl + 1 == win ? 0 : sl + 1) {
#pragma unroll
        for (int c = 0; c < 6; ++c) s[c] += ring[((size_t)sl * 6 + c) * nt + tid];
      }
      // evaluation.py:74-81, elementwise in the reference's association
      const double mu_a = s[0] / n, mu_b = s[1] / n;
      const double var_a = norm * (s[2] / n - mu_a * mu_a);
      const double var_b = norm * (s[3] / n - mu_b * mu_b);
      const double cov = norm * (s[4] / n - mu_a * mu_b);
      const double num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2);
      const double den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2);
      const size_t o = (size_t)pair * HH * WW + (size_t)y * WW + x;
      V[o] = num / den;
      F[o] = s[5] == n;  // evaluation.py:70 complete windows
    }
  }
}

// u8 images: integer window moments (exact and order-free, so equal to
// ssim_window_k's f64 sums) kept as running column sums -- each image row adds
// its 7-wide row sums, and the row leaving the window subtracts the sums it
// added (an int ring of the last win + 1 rows' sums, 24 KB at win 7, instead
// of the 43 KB f64 ring).  The next image row is fetched into registers while
// the current one is summed; the f64 SSIM expression runs only for complete
// windows (the others are never averaged).
template <int kWin>  // the window at compile time (7, the default), or 0: `win`
__global__ void __launch_bounds__(128) ssim_window_u8_k(const uint8_t* __restrict__ a,
                                                        const uint8_t* __restrict__ am,
                                                        const uint8_t* __restrict__ b,
                                                        const uint8_t* __restrict__ bm, int H, int W, int win_rt,
                                                        double c1, double c2, double* __restrict__ V,
                                                        uint8_t* __restrict__ F) {
  const int win = kWin ? kWin : win_rt;
  extern __shared__ uint8_t sb[];  // [win + 1 rows][3][span]
  const int nt = blockDim.x, tid = threadIdx.x;
  const int HH = H - win + 1, WW = W - win + 1;
  const int64_t pair = blockIdx.z;
  const int x0 = blockIdx.x * nt, x = x0 + tid;
  const int y0 = blockIdx.y * kBand;
  if (y0 >= HH) return;
  const int y1 = min(y0 + kBand, HH);
  const int span = nt + win - 1, R = win + 1;
  int* hring = reinterpret_cast<int*>(sb + (((size_t)R * 3 * span + 15) & ~(size_t)15));  // [R][6][nt]
  const size_t base = (size_t)pair * H * W;
  const double n = (double)(win * win);
  const double norm = n / (n - 1.0);
  int S[6] = {0, 0, 0, 0, 0, 0};
  // a thread stages columns tid and tid + nt of each row (span <= 2 nt);
  // row r + 1 is loaded into registers while row r is summed
  auto fetch = [&](int r, uint32_t (&w)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = tid + h * nt, c = x0 + i;
      w[h] = 0u;
      if (i < span && c < W) {
        const size_t k = base + (size_t)r * W + c;
        w[h] = (uint32_t)a[k] | ((uint32_t)b[k] << 8) | ((valid_at(am, bm, k) ? 1u : 0u) << 16);
      }
    }
  };
  const int r_end = y1 + win - 1;
  uint32_t nxt[2];
  fetch(y0, nxt);
  int slot = 0;  // ring slot of row r: (r - y0) mod R, kept incrementally (no integer division)
  for (int r = y0; r < r_end; ++r, slot = slot + 1 == R ? 0 : slot + 1) {
    const uint32_t cur[2] = {nxt[0], nxt[1]};
    if (r + 1 < r_end) fetch(r + 1, nxt);
    uint8_t* row = sb + (size_t)slot * 3 * span;
    __syncthreads();  // the slot's previous row (r - R) was last read at r - 1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = tid + h * nt;
      if (i < span) {
        row[i] = (uint8_t)cur[h];
        row[span + i] = (uint8_t)(cur[h] >> 8);
        row[2 * span + i] = (uint8_t)(cur[h] >> 16);
      }
    }
    __syncthreads();
    // this row's 7-wide sums enter the window and are kept in the int ring;
    // the sums of the row leaving (r - win) come back from it
    int h[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < (kWin ? kWin : win); ++j) {
      const int p = row[tid + j], q = row[span + tid + j];
      h[0] += p;
      h[1] += q;
      h[2] += p * p;
      h[3] += q * q;
      h[4] += p * q;
      h[5] += row[2 * span + tid + j];
    }
    int* hr = hring + (size_t)slot * 6 * nt + tid;
    const int* ho = hring + (size_t)(slot + 1 == R ? 0 : slot + 1) * 6 * nt + tid;  // row r - win
    const bool leave = r - y0 >= win;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      S[c] += h[c] - (leave ? ho[c * nt] : 0);
      hr[c * nt] = h[c];
    }
    const int y = r - (win - 1);
    if (y >= y0 && x < WW) {
      const size_t o = (size_t)pair * HH * WW + (size_t)y * WW + x;
      const bool complete = S[5] == win * win;
      F[o] = complete;
      if (complete) {  // only complete windows are averaged (evaluation.py:82)
        double s[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) s[c] = (double)S[c];
        const double mu_a = s[0] / n, mu_b = s[1] / n;
        const double var_a = norm * (s[2] / n - mu_a * mu_a);
        const double var_b = norm * (s[3] / n - mu_b * mu_b);
        const double cov = norm * (s[4] / n - mu_a * mu_b);
        const double num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2);
        const double den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2);
        V[o] = num / den;
      }
    }
  }
}

// Per pair two CTAs: blockIdx.y == 0 computes NCC over the mask intersection
// (evaluation.py:41-53) and the valid count, blockIdx.y == 1 the mean of the
// complete windows' SSIM values (evaluation.py:82).  Scratch per pair: A, B
// (masked values), C (complete window values), S (reduction slots, 4 x 2^D).
template <class T>
__global__ void __launch_bounds__(kReduceThreads) sim_reduce_k(
    const T* __restrict__ a, const uint8_t* __restrict__ am, const T* __restrict__ b,
    const uint8_t* __restrict__ bm, int H, int W, int win, int do_ssim, const double* __restrict__ V,
    const uint8_t* __restrict__ F, double* __restrict__ scratch, int64_t scratch_per_pair, int64_t slots,
    double* __restrict__ ncc_out, double* __restrict__ ssim_out, int64_t* __restrict__ valid_out,
    int32_t* __restrict__ status_out) {
  const int64_t pair = blockIdx.x;
  const int64_t HW = (int64_t)H * W;
  const int64_t WN = do_ssim ? (int64_t)(H - win + 1) * (W - win + 1) : 0;
  // masked values compacted in their input type (u8: 1 B each), converted on read
  double* C = scratch + pair * scratch_per_pair;
  double* S = C + WN + (blockIdx.y ? 3 * slots : 0);
  T* A = reinterpret_cast<T*>(C + WN + 4 * slots);
  T* B = A + HW;
  if (blockIdx.y == 0) {
    const size_t base = (size_t)pair * HW;
    const int64_t n = compact(
        HW, [&](int64_t i) { return valid_at(am, bm, base + i); },
        [&](int64_t i, int64_t p) {
          A[p] = a[base + i];
          B[p] = b[base + i];
        });
    int32_t status = 0;
    double ncc = 0.0;
    if (n < 2) {
      status |= 1;  // "ncc needs at least 2 mutually valid pixels"
    } else {
      __syncthreads();
      pw_reduce<2>(n, [&](int64_t i, double* v) { v[0] = (double)A[i]; v[1] = (double)B[i]; }, S);
      const double ma = S[0] / (double)n, mb = S[1] / (double)n;  // va.mean(), vb.mean()
      __syncthreads();
      pw_reduce<3>(
          n,
          [&](int64_t i, double* v) {
            const double da = (double)A[i] - ma, db = (double)B[i] - mb;
            v[0] = da * da;
            v[1] = db * db;
            v[2] = da * db;
          },
          S);
      const double denom = sqrt(S[0] * S[1]);
      if (denom == 0.0)
        status |= 2;  // "ncc undefined for zero-variance input"
      else
        ncc = S[2] / denom;
    }
    if (threadIdx.x == 0) {
      ncc_out[pair] = ncc;
      valid_out[pair] = n;
      atomicOr(status_out + pair, status);
    }
    return;
  }
  int32_t status = 0;
  double ssim = 0.0;
  if (do_ssim) {
    const double* Vp = V + pair * WN;
    const uint8_t* Fp = F + pair * WN;
    const int64_t m = compact(
        WN, [&](int64_t i) { return Fp[i] != 0; }, [&](int64_t i, int64_t p) { C[p] = Vp[i]; });
    if (m == 0) {
      status |= 4;  // "no complete ssim window inside the mask intersection"
    } else {
      __syncthreads();
      pw_reduce<1>(m, [&](int64_t i, double* v) { v[0] = C[i]; }, S);
      ssim = S[0] / (double)m;
    }
  } else {
    status |= 8;  // image smaller than the window: no SSIM
  }
  if (threadIdx.x == 0) {
    ssim_out[pair] = ssim;
    atomicOr(status_out + pair, status);
  }
}

template <class T>
void launch_similarity(int32_t P, int32_t H, int32_t W, const T* a, const uint8_t* am, const T* b,
                       const uint8_t* bm, int32_t win, double c1, double c2, double* ncc, double* ssim,
                       int64_t* valid, int32_t* status, cudaStream_t s) {
  constexpr bool kU8 = sizeof(T) == 1;
  const int64_t HW = (int64_t)H * W;
  const bool do_ssim = H >= win && W >= win;
  const int64_t WN = do_ssim ? (int64_t)(H - win + 1) * (W - win + 1) : 0;
  const int64_t slots = (int64_t)1 << std::max(pw_depth(HW), pw_depth(std::max<int64_t>(WN, 1)));
  // doubles per pair: C (WN) + slots (4 x 2^D) + the compacted a, b values (2 HW of T, 8 B aligned)
  const int64_t per_pair = WN + 4 * slots + (2 * HW * (int64_t)sizeof(T) + 7) / 8;
  // bound the scratch: pairs per launch so that values + flags + reductions
  // stay under ~1 GB
  const int64_t bytes_pair = per_pair * 8 + WN * 9;
  const int32_t chunk = (int32_t)std::max<int64_t>(1, std::min<int64_t>(P, ((int64_t)1 << 30) / bytes_pair));
  Scratch<double> scr((size_t)chunk * per_pair, s);
  Scratch<double> vals((size_t)chunk * WN, s);
  Scratch<uint8_t> flags((size_t)chunk * WN, s);
  // u8 images up to 31-wide windows: integer running sums (ssim_window_u8_k);
  // otherwise the f64 ring kernel (integer-valued inputs give the same sums)
  const bool u8_kernel = kU8 && win <= 31;
  const int nt = u8_kernel || win <= 31 ? 128 : 32;
  const size_t smem = u8_kernel ? (((size_t)(win + 1) * 3 * (nt + win - 1) + 15) & ~(size_t)15) +
                                      (size_t)(win + 1) * 6 * nt * sizeof(int)
                                : ((size_t)win * 6 * nt + 3 * (size_t)(nt + win - 1)) * sizeof(double);
  using WindowFn = void (*)(const T*, const uint8_t*, const T*, const uint8_t*, int, int, int, double, double,
                            double*, uint8_t*);
  auto window_kernel = u8_kernel ? (win == 7 ? (WindowFn)ssim_window_u8_k<7> : (WindowFn)ssim_window_u8_k<0>)
                                 : ssim_window_k<T>;
  if (do_ssim) {
    DARE_LIMIT(smem <= 220 * 1024 && win <= 127, "ssim window too large (at most 127)");
    DARE_CUDA(cudaFuncSetAttribute((const void*)window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  }
  DARE_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * (size_t)P, s));
  for (int32_t p0 = 0; p0 < P; p0 += chunk) {
    const int32_t np = std::min(chunk, P - p0);
    const size_t off = (size_t)p0 * HW;
    const uint8_t* amp = am ? am + off : nullptr;
    const uint8_t* bmp = bm ? bm + off : nullptr;
    for (int32_t q0 = 0; q0 < np; q0 += 65535) {
      const int32_t nq = std::min(65535, np - q0);
      const size_t qo = (size_t)q0 * HW;
      if (do_ssim) {
        dim3 grid(ceil_div(W - win + 1, nt), ceil_div(H - win + 1, kBand), nq);
        window_kernel<<<grid, nt, smem, s>>>(a + off + qo, amp ? amp + qo : nullptr, b + off + qo,
                                             bmp ? bmp + qo : nullptr, H, W, win, c1, c2,
                                             vals.ptr + (size_t)q0 * WN, flags.ptr + (size_t)q0 * WN);
        DARE_CUDA(cudaGetLastError());
      }
    }
    sim_reduce_k<T><<<dim3(np, 2), kReduceThreads, 0, s>>>(a + off, amp, b + off, bmp, H, W, win,
                                                           do_ssim ? 1 : 0, vals.ptr, flags.ptr, scr.ptr,
                                                           per_pair, slots, ncc + p0, ssim + p0, valid + p0,
                                                           status + p0);
    DARE_CUDA(cudaGetLastError());
  }
}

void similarity_device(int32_t P, int32_t H, int32_t W, int32_t elem, const void* a, const uint8_t* am,
                       const void* b, const uint8_t* bm, int32_t win, double c1, double c2, double* ncc,
                       double* ssim, int64_t* valid, int32_t* status, cudaStream_t s) {
  DARE_REQUIRE(P >= 0 && H > 0 && W > 0, "invalid image batch shape");
  DARE_REQUIRE(win >= 3 && win % 2 == 1, "ssim window must be odd and >= 3");
  DARE_REQUIRE(elem == DARE_ELEM_U8 || elem == DARE_ELEM_F64, "element type must be u8 or f64");
  DARE_LIMIT((int64_t)H * W <= ((int64_t)1 << 31), "image too large");
  if (P == 0) return;
  (void)thread_stream();  // first call on this device: keeps the scratch pool (release threshold)
  if (elem == DARE_ELEM_U8)
    launch_similarity<uint8_t>(P, H, W, (const uint8_t*)a, am, (const uint8_t*)b, bm, win, c1, c2, ncc, ssim,
                               valid, status, s);
  else
    launch_similarity<double>(P, H, W, (const double*)a, am, (const double*)b, bm, win, c1, c2, ncc, ssim,
                              valid, status, s);
}

}  // namespace
}  // namespace dare

using namespace dare;

extern "C" int dare_similarity_device(int32_t n_pairs, int32_t height, int32_t width, int32_t elem,
                                      const void* d_a, const uint8_t* d_a_mask, const void* d_b,
                                      const uint8_t* d_b_mask, int32_t window, double c1, double c2,
                                      double* d_ncc, double* d_ssim, int64_t* d_valid, int32_t* d_status,
                                      void* stream) {
  return guard([&] {
    similarity_device(n_pairs, height, width, elem, d_a, d_a_mask, d_b, d_b_mask, window, c1, c2, d_ncc,
                      d_ssim, d_valid, d_status, (cudaStream_t)stream);
  });
}

extern "C" int dare_similarity(int32_t n_pairs, int32_t height, int32_t width, int32_t elem, const void* a,
                               const uint8_t* a_mask, const void* b, const uint8_t* b_mask, int32_t window,
                               double c1, double c2, double* ncc, double* ssim, int64_t* valid,
                               int32_t* status) {
  return guard([&] {
    DARE_REQUIRE(n_pairs >= 0 && height > 0 && width > 0, "invalid image batch shape");
    if (n_pairs == 0) return;
    cudaStream_t s = thread_stream();
    const size_t npix = (size_t)n_pairs * height * width;
    const size_t esz = elem == DARE_ELEM_F64 ? 8 : 1;
    Scratch<uint8_t> d_img(2 * npix * esz, s);
    Scratch<uint8_t> d_mask((a_mask ? npix : 0) + (b_mask ? npix : 0), s);
    Scratch<uint8_t> d_out((size_t)n_pairs * (8 + 8 + 8 + 4), s);
    DARE_CUDA(cudaMemcpyAsync(d_img.ptr, a, npix * esz, cudaMemcpyHostToDevice, s));
    DARE_CUDA(cudaMemcpyAsync(d_img.ptr + npix * esz, b, npix * esz, cudaMemcpyHostToDevice, s));
    uint8_t* dam = nullptr;
    uint8_t* dbm = nullptr;
    if (a_mask) {
      dam = d_mask.ptr;
      DARE_CUDA(cudaMemcpyAsync(dam, a_mask, npix, cudaMemcpyHostToDevice, s));
    }
    if (b_mask) {
      dbm = d_mask.ptr + (a_mask ? npix : 0);
      DARE_CUDA(cudaMemcpyAsync(dbm, b_mask, npix, cudaMemcpyHostToDevice, s));
    }
    double* dn = (double*)d_out.ptr;
    double* ds = dn + n_pairs;
    int64_t* dv = (int64_t*)(ds + n_pairs);
    int32_t* dst = (int32_t*)(dv + n_pairs);
    similarity_device(n_pairs, height, width, elem, d_img.ptr, dam, d_img.ptr + npix * esz, dbm, window, c1, c2,
                      dn, ds, dv, dst, s);
    DARE_CUDA(cudaMemcpyAsync(ncc, dn, 8 * (size_t)n_pairs, cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaMemcpyAsync(ssim, ds, 8 * (size_t)n_pairs, cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaMemcpyAsync(valid, dv, 8 * (size_t)n_pairs, cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaMemcpyAsync(status, dst, 4 * (size_t)n_pairs, cudaMemcpyDeviceToHost, s));
    DARE_CUDA(cudaStreamSynchronize(s));
  });
}
