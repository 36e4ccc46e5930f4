// Host-side pose pipeline of a sweep (no device work): the arithmetic of
// synchronize() after pose interpolation -- marker pose composed with the
// calibration (reconstruct.py:119-149 via Pose.compose, geometry.py:128-133:
// normalised Hamilton product, rotate(q, t_cal) + t) -- the per-frame axes fed
// to the device (rotation_matrix, geometry.py:79-88; reconstruct.py:155-162),
// the canonical f32 quaternions (reconstruct.py:192-195, geometry.py:56-64) and
// the four image corners of compute_bounds (volume.py:57-73).
//
// Every expression is the reference's, evaluated left to right with separately
// rounded IEEE f64 operations (built with -ffp-contract=off, so no FMA), i.e.
// the same bits numpy produces elementwise.  The corner bounds follow
// compute_bounds' sequential lo = np.minimum(lo, corner) (frame order, corner
// order) with np.minimum's semantics -- NaN propagates, a tie returns the
// second operand -- so even the sign of a zero bound is the reference's.
#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace {

constexpr double kUnitNormTol = 1e-3;  // geometry.py:20

// rotate(q, v) = v + w t + u x t, t = 2 u x v (geometry.py:99-107; np.cross
// component order a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0)
inline void rotate(const double* q, const double* v, double* out) {
  const double w = q[0], u0 = q[1], u1 = q[2], u2 = q[3];
  const double t0 = 2.0 * (u1 * v[2] - u2 * v[1]);
  const double t1 = 2.0 * (u2 * v[0] - u0 * v[2]);
  const double t2 = 2.0 * (u0 * v[1] - u1 * v[0]);
  out[0] = (v[0] + w * t0) + (u1 * t2 - u2 * t1);
  out[1] = (v[1] + w * t1) + (u2 * t0 - u0 * t2);
  out[2] = (v[2] + w * t2) + (u0 * t1 - u1 * t0);
}

// np.minimum / np.maximum of two scalars (tie or NaN: as numpy)
inline double np_min(double a, double b) { return a < b ? a : (b < a ? b : (std::isnan(a) ? a : b)); }
inline double np_max(double a, double b) { return a > b ? a : (b > a ? b : (std::isnan(a) ? a : b)); }

inline double norm4(const double* q) {
  return std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
}

}  // namespace

extern "C" int dare_frame_poses(int64_t n, const double* mq, const double* mt, const double* cal_q,
                                const double* cal_t, int32_t width, int32_t height, double px,
                                double py, double* rot, double* trans, double* axes, float* quats32,
                                double* lo, double* hi, int32_t* status, int64_t* bad, double* bad_norm) {
  return dare::guard([&] {
    DARE_REQUIRE(n >= 0, "negative frame count");
    DARE_REQUIRE(status && bad && bad_norm, "null status argument");
    *status = 0;
    *bad = -1;
    *bad_norm = 0.0;
    const double cw = cal_q[0], cx = cal_q[1], cy = cal_q[2], cz = cal_q[3];
    int64_t zero_at = -1, marker_bad = -1, frame_bad = -1;
    double marker_norm = 0.0, frame_norm = 0.0;
    const double umax = (double)(width - 1) * px, vmax = (double)(height - 1) * py;
    const double cv[4][3] = {{0.0, 0.0, 0.0}, {umax, 0.0, 0.0}, {0.0, vmax, 0.0}, {umax, vmax, 0.0}};
    for (int k = 0; k < 3; ++k) {
      lo[k] = INFINITY;
      hi[k] = -INFINITY;
    }
    for (int64_t i = 0; i < n; ++i) {
      const double* m = mq + 4 * i;
      const double w = m[0], x = m[1], y = m[2], z = m[3];
      // qmul(marker, calibration) -- geometry.py:69-77
      const double p0 = w * cw - x * cx - y * cy - z * cz;
      const double p1 = w * cx + x * cw + y * cz - z * cy;
      const double p2 = w * cy - x * cz + y * cw + z * cx;
      const double p3 = w * cz + x * cy - y * cx + z * cw;
      const double nn = std::sqrt(p0 * p0 + p1 * p1 + p2 * p2 + p3 * p3);
      if (nn == 0.0 && zero_at < 0) zero_at = i;
      double* r = rot + 4 * i;
      r[0] = p0 / nn;
      r[1] = p1 / nn;
      r[2] = p2 / nn;
      r[3] = p3 / nn;
      // translation: rotate(marker, t_cal) + t_marker (with rotate's norm check)
      const double mn = norm4(m);
      if (std::fabs(mn - 1.0) > kUnitNormTol && marker_bad < 0) {
        marker_bad = i;
        marker_norm = mn;
      }
      double* t = trans + 3 * i;
      rotate(m, cal_t, t);
      t[0] = t[0] + mt[3 * i];
      t[1] = t[1] + mt[3 * i + 1];
      t[2] = t[2] + mt[3 * i + 2];
      // axes: R[:,0], R[:,1], t (rotation_matrix without renormalisation)
      const double qw = r[0], qx = r[1], qy = r[2], qz = r[3];
      double* a = axes + 9 * i;
      a[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
      a[1] = 2.0 * (qx * qy + qw * qz);
      a[2] = 2.0 * (qx * qz - qw * qy);
      a[3] = 2.0 * (qx * qy - qw * qz);
      a[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
      a[5] = 2.0 * (qy * qz + qw * qx);
      a[6] = t[0];
      a[7] = t[1];
      a[8] = t[2];
      // canonical sign (w >= 0, ties on x, y, z), then f32
      const bool flip = qw < 0.0 || (qw == 0.0 && (qx < 0.0 || (qx == 0.0 && (qy < 0.0 || (qy == 0.0 && qz < 0.0)))));
      float* f = quats32 + 4 * i;
      for (int k = 0; k < 4; ++k) f[k] = (float)(flip ? -r[k] : r[k]);
      // image corners: rotate(frame rotation, corner) + t (compute_bounds)
      const double fn = norm4(r);
      if (std::fabs(fn - 1.0) > kUnitNormTol && frame_bad < 0) {
        frame_bad = i;
        frame_norm = fn;
      }
      for (int c = 0; c < 4; ++c) {
        double o[3];
        rotate(r, cv[c], o);
        for (int k = 0; k < 3; ++k) {
          o[k] = o[k] + t[k];
          lo[k] = np_min(lo[k], o[k]);
          hi[k] = np_max(hi[k], o[k]);
        }
      }
    }
    // the reference raises the first of these it meets (plan order)
    if (zero_at >= 0) {
      *status = 1;
      *bad = zero_at;
    } else if (marker_bad >= 0) {
      *status = 2;
      *bad = marker_bad;
      *bad_norm = marker_norm;
    } else if (frame_bad >= 0) {
      *status = 3;
      *bad = frame_bad;
      *bad_norm = frame_norm;
    }
  });
}

// Pose interpolation of synchronize() (reconstruct.py:102-116 interpolate_pose)
// for the frames whose timestamp falls strictly between two pose samples:
// alpha = (t - t0) / (t1 - t0) (0 when t1 == t0), translation
// (1 - alpha) p0 + alpha p1 elementwise, rotation slerp (geometry.py:159-180).
// numpy's dot of two 4-vectors (slerp's dot and linalg.norm's sum of
// squares) evaluates, with the OpenBLAS tail loop it dispatches to on these
// hosts, s = a0 b0, then s = fma(a_i, b_i, s) for i = 1..3 -- measured equal
// on 200k random vectors, tests/test_host_logic.py -- so that is what is
// restated here; acos / sin are the C library's, the functions Python's math
// module calls.
namespace {

inline double np_dot4(const double* a, const double* b) {
  double s = a[0] * b[0];
  s = std::fma(a[1], b[1], s);
  s = std::fma(a[2], b[2], s);
  s = std::fma(a[3], b[3], s);
  return s;
}

void slerp(const double* q0, const double* q1, double t, double* out) {
  double b[4] = {q1[0], q1[1], q1[2], q1[3]};
  double dot = np_dot4(q0, b);
  if (dot < 0.0) {
    for (int k = 0; k < 4; ++k) b[k] = -b[k];
    dot = -dot;
  }
  double o[4];
  if (dot > 0.9995) {
    for (int k = 0; k < 4; ++k) o[k] = q0[k] + t * (b[k] - q0[k]);
  } else {
    const double theta = std::acos(dot < 1.0 ? dot : 1.0);  // min(1.0, dot)
    const double sin_theta = std::sin(theta);
    const double w0 = std::sin((1.0 - t) * theta) / sin_theta;
    const double w1 = std::sin(t * theta) / sin_theta;
    for (int k = 0; k < 4; ++k) o[k] = w0 * q0[k] + w1 * b[k];
  }
  const double n = std::sqrt(np_dot4(o, o));  // np.linalg.norm
  for (int k = 0; k < 4; ++k) out[k] = o[k] / n;
}

}  // namespace

extern "C" int dare_interpolate_poses(int64_t n, const double* t, const int64_t* idx, const double* ts,
                                      const double* pose_q, const double* pose_t, double* out_q,
                                      double* out_t) {
  return dare::guard([&] {
    DARE_REQUIRE(n >= 0, "negative frame count");
    for (int64_t j = 0; j < n; ++j) {
      const int64_t i = idx[j];
      const double t0 = ts[i], t1 = ts[i + 1];
      const double alpha = t1 == t0 ? 0.0 : (t[j] - t0) / (t1 - t0);
      slerp(pose_q + 4 * i, pose_q + 4 * (i + 1), alpha, out_q + 4 * j);
      for (int k = 0; k < 3; ++k)
        out_t[3 * j + k] = (1.0 - alpha) * pose_t[3 * i + k] + alpha * pose_t[3 * (i + 1) + k];
    }
  });
}
