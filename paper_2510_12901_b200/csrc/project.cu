// simuli_project: per-particle UT projection + ray-based culling (sm_100a).
//
// One thread per particle; 256-thread CTAs.  For each particle: normalise q -> R,
// l_k = s_k R e_k, 7 sigma points, each projected with the pose at its own firing
// time (K fixed-point iterations, A3) by Eq. 3 or the lens model, UT moments,
// outward-rounded 3-sigma box (A11), LiDAR culling by the summed-area-table rectangle count
// (Proc. RayOccupancyCount / ProjectParticles), tile rectangle + count, SH
// features (A17), float32 depth key (A19) and the 80-byte compositing record.
#include <cmath>
#include <cstdio>

#include "abi_util.h"
#include "common.cuh"

namespace simuli {

PoseInterpD make_pose_interp_d(const simuli_pose& a, const simuli_pose& b) {
  PoseInterpD P{};
  double qa[4], qb[4], na = 0, nb = 0;
  for (int i = 0; i < 4; ++i) {
    qa[i] = a.q[i];
    qb[i] = b.q[i];
    na += qa[i] * qa[i];
    nb += qb[i] * qb[i];
  }
  na = std::sqrt(na);
  nb = std::sqrt(nb);
  for (int i = 0; i < 4; ++i) {
    qa[i] /= na;
    qb[i] /= nb;
  }
  bool same = true;
  for (int i = 0; i < 4; ++i) same &= (a.q[i] == b.q[i]);
  for (int i = 0; i < 3; ++i) same &= (a.t[i] == b.t[i]);
  // relative rotation q_rel = conj(qa) * qb on the shortest arc
  const double w1 = qa[0], x1 = -qa[1], y1 = -qa[2], z1 = -qa[3];
  const double w2 = qb[0], x2 = qb[1], y2 = qb[2], z2 = qb[3];
  double r[4] = {w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                 w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2};
  if (r[0] < 0)
    for (double& v : r) v = -v;
  const double vn = std::sqrt(r[1] * r[1] + r[2] * r[2] + r[3] * r[3]);
  for (int i = 0; i < 4; ++i) P.q0[i] = qa[i];
  if (vn > 0) {
    P.half_theta = std::atan2(vn, r[0]);
    for (int i = 0; i < 3; ++i) P.axis[i] = r[1 + i] / vn;
  } else {
    P.half_theta = 0;
    P.axis[0] = 1;
  }
  for (int i = 0; i < 3; ++i) {
    P.t0[i] = a.t[i];
    P.dt[i] = static_cast<double>(b.t[i]) - static_cast<double>(a.t[i]);
  }
  P.same = same ? 1 : 0;
  return P;
}

PoseInterpF make_pose_interp_f(const PoseInterpD& d) {
  PoseInterpF f{};
  for (int i = 0; i < 4; ++i) f.q0[i] = static_cast<float>(d.q0[i]);
  for (int i = 0; i < 3; ++i) {
    f.axis[i] = static_cast<float>(d.axis[i]);
    f.t0[i] = static_cast<float>(d.t0[i]);
    f.dt[i] = static_cast<float>(d.dt[i]);
  }
  f.half_theta = static_cast<float>(d.half_theta);
  f.same = d.same;
  return f;
}

namespace {

struct UTW {
  float spread, wm0, wmi, wc0, wci;
};

struct ProjArgs {
  int64_t n;
  const float *means, *quats, *scales, *opacity, *sh;
  int sh_degree, n_coef;
  const int* actor_id;      // scene graph (A29): -1 static, else object index
  const float* actor_pose;  // [n_actors][7] (q w,x,y,z, t) object -> world at t
  int n_actors;
  PoseInterpF pose;
  int K;
  UTW ut;
  float ks;
  float o_mid[3];
  int write_all;
  // LiDAR
  float az_start, r_min;
  int dir;
  float R0[9], t0w[3], dtw[3], v[3], axis[3], theta;  // start pose, motion, rotation axis / angle
  float beam_div;                                     // theta_div (App. C), 0 = off
  double R0d[9], t0d[3], vd[3], axis_d[3], theta_d;  // the same in double (sigma point 0)
  int small_rot;
  int n_phi, n_theta, rows_per_tile, az_cells, sat_cols, enable_cull;
  float pi_f, two_pi_f, az_tile_scale, az_cell_scale;
  const float *bounds, *row_scale;
  const int* sat;
  const float *beam_sorted, *col_sorted;  // exact culling (A32): ascending beam / column angles
  int n_beams, n_az;
  float col_step;                         // (float)(n_az / 2 pi): search start estimate
  // camera
  int cam_model, width, height, rolling, tile_px, Wt, Ht;
  float fx, fy, cx, cy, k[5], near_m, max_theta, inv_tile;
  // out
  float* record;
  float* view_dir;  // optional [n][3] (backward: the SH direction, A31)
  int* rect;
  float* key;
  int* count;
};

__device__ __forceinline__ int elev_tile(const ProjArgs& A, float w) {
  // number of interior boundaries bounds[1..n_phi-1] <= w (binary search)
  int lo = 1, hi = A.n_phi;  // first index in [1, n_phi) with bound > w
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A.bounds[mid] <= w) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

__device__ __forceinline__ int dense_row_e(const ProjArgs& A, float w, int e) {
  const float u = __fmul_rn(__fsub_rn(w, A.bounds[e]), A.row_scale[e]);
  return e * A.rows_per_tile + clamp_floor(u, A.rows_per_tile);
}

// first index i in [0, n) with a[i] >= x (n if none); a ascending
__device__ __forceinline__ int lower_bound_f(const float* a, int n, float x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// first index i in [0, n) with a[i] > x (n if none); a ascending
__device__ __forceinline__ int upper_bound_f(const float* a, int n, float x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// the same on the (near-uniform) ascending column azimuths: start from the uniform-grid
// estimate and walk (the result is exact; the estimate only saves the log-step search)
__device__ __forceinline__ int col_bound(const ProjArgs& A, float x, bool upper) {
  const float* a = A.col_sorted;
  const float p0 = __ldg(a);
  const int i0 = (int)fminf(fmaxf(floorf((x - p0) * A.col_step), 0.f), (float)A.n_az);
  int i = i0;
  if (upper) {  // first a[i] > x
    while (i > 0 && __ldg(a + i - 1) > x) --i;
    while (i < A.n_az && __ldg(a + i) <= x) ++i;
  } else {      // first a[i] >= x
    while (i > 0 && __ldg(a + i - 1) >= x) --i;
    while (i < A.n_az && __ldg(a + i) < x) ++i;
  }
  return i;
}

// Exact ray-containment culling (reading A32): the render tiles holding a ray inside the
// box.  Rays are beams x columns, so they are the elevation tiles of the beams with
// lo_b <= omega <= hi_b times the azimuth tiles of the columns inside the azimuth interval
// under the render's membership rule (A12: seam-shifted box edges) -- a circular run of the
// ascending column azimuths.  Returns the tile count (0: no ray inside) and the rectangle.
__device__ __forceinline__ int exact_rect(const ProjArgs& A, const float box[4], int rect[4]) {
  const int bl = lower_bound_f(A.beam_sorted, A.n_beams, box[2]);
  const int bh = upper_bound_f(A.beam_sorted, A.n_beams, box[3]) - 1;
  if (bl > bh) return 0;
  const float lo = box[0], hi = box[1];
  const int NA = A.n_az;
  int first, n;  // run of sorted columns: first, length (circular)
  if (__fsub_rn(hi, lo) >= A.two_pi_f || (lo < -A.pi_f && hi > A.pi_f)) {
    first = 0;
    n = NA;
  } else if (lo < -A.pi_f) {  // [lo, hi] covers a prefix, [lo + 2 pi, ...) a suffix
    const int a2 = col_bound(A, hi, true);
    const int s2 = col_bound(A, __fadd_rn(lo, A.two_pi_f), false);
    if (s2 <= a2) { first = 0; n = NA; }
    else { first = s2; n = (NA - s2) + a2; }
  } else if (hi > A.pi_f) {   // [lo, hi] covers a suffix, (..., hi - 2 pi] a prefix
    const int a1 = col_bound(A, lo, false);
    const int s3 = col_bound(A, __fsub_rn(hi, A.two_pi_f), true);
    if (s3 >= a1) { first = 0; n = NA; }
    else { first = a1; n = (NA - a1) + s3; }
  } else {
    first = col_bound(A, lo, false);
    n = col_bound(A, hi, true) - first;
  }
  if (n <= 0) return 0;
  if (first >= NA) first -= NA;  // a run starting past the last column starts at column 0
  int cs, cl;
  if (n >= NA) {
    cs = 0;
    cl = A.n_theta;
  } else {
    const int last = first + n - 1;
    const int cF = az_index(__ldg(A.col_sorted + first), A.pi_f, A.az_tile_scale, A.n_theta);
    const int cL = az_index(__ldg(A.col_sorted + (last < NA ? last : last - NA)), A.pi_f, A.az_tile_scale, A.n_theta);
    if (last < NA) { cs = cF; cl = cL - cF + 1; }
    else if (cL >= cF) { cs = 0; cl = A.n_theta; }
    else { cs = cF; cl = A.n_theta - cF + cL + 1; }
  }
  SIMULI_CHECK(bl >= 0 && bh < A.n_beams && first >= 0 && first < NA, bl, first);
  rect[0] = elev_tile(A, __ldg(A.beam_sorted + bl));
  rect[1] = elev_tile(A, __ldg(A.beam_sorted + bh));
  rect[2] = cs;
  rect[3] = cl;
  SIMULI_CHECK(rect[0] >= 0 && rect[0] <= rect[1] && rect[1] < A.n_phi, rect[0], rect[1]);
  SIMULI_CHECK(cs >= 0 && cs < A.n_theta && cl >= 1 && cl <= A.n_theta, cs, cl);
  return (rect[1] - rect[0] + 1) * cl;
}

__device__ __forceinline__ int sat_rect(const ProjArgs& A, int r0, int r1, int c0, int c1) {
  const int sc = A.sat_cols;
  SIMULI_CHECK(r0 >= 0 && r0 <= r1 && r1 < A.n_phi * A.rows_per_tile, r0, r1);
  SIMULI_CHECK(c0 >= 0 && c0 <= c1 && c1 < A.az_cells && c1 + 1 < sc, c0, c1);
  return __ldg(A.sat + (r1 + 1) * sc + (c1 + 1)) - __ldg(A.sat + r0 * sc + (c1 + 1)) -
         __ldg(A.sat + (r1 + 1) * sc + c0) + __ldg(A.sat + r0 * sc + c0);
}

// ---- LiDAR sensor model (Eq. 3) with the firing-time fixed point (A3, A5).
// A point's sensor-frame position at firing time s is
//   p(s) = R(s)^T (x - t(s)) = E(s)^T (q - s v),   q = R0^T (x - t0), v = R0^T (t1 - t0),
// with R(s) = R0 E(s), E(s) = Exp(s theta k) (k the unit axis of R0^T R1); the start pose
// R0, t0 and v are launch constants, and
//   E(s)^T y = y - sin(a) (k x y) + (1 - cos a)(k (k.y) - y),   a = s theta.
//
// Precision split.  The box edges are the interface values every membership
// decision compares against, so their ABSOLUTE position must match the double oracle to well
// under one float32 ulp: sigma point 0 (the particle mean) is carried in double -- start-frame
// coordinates, the rotation to its firing time, its azimuth and elevation.  The other six
// sigma points are carried as float32 OFFSETS from sigma point 0,
//   p_i = E(ds)^T (p0 + w),  w = E(s0)^T (l_i - ds v),  ds = s_i - s0,
//   p_i - p0 = w + G(ds)(p0 + w),  G(a) y = -sin(a theta)(k x y) + (1 - cos a theta)(k (k.y) - y),
// which never forms the difference of two rounded 100 m positions, and their azimuth /
// elevation offsets are taken from the offsets directly (atan of a cancellation-free ratio).
// Firing times are decisions of float32 accuracy only (an error of 1e-7 in s moves a point by
// < 1e-9 rad), so they stay in float32.

// atan2 in double to ~1e-13 rad (the box edges need ~1e-9; libdevice's full-precision
// atan2 costs ~75 instructions, half of them materialising its 64-bit coefficients): |t| =
// min / max reduced to [0, tan(pi/8)] by atan t = pi/4 + atan((t - 1) / (t + 1)) (formed as
// (min - max) / (min + max): one division), then
// atan t = t + t u P(u), u = t^2, P a degree-7 least-squares Chebyshev fit (max error
// 1.1e-13 on the interval) with its coefficients in constant memory (DFMA operands, no
// immediate moves).  Quadrants and signed zeros as C's atan2 except atan2(+-0, -0) = 0.
__constant__ double c_atan_p[8] = {-0.33333333333168147, 0.19999999929984685, -0.14285707051757754,
                                   0.11110796545187183, -0.09083864602009568, 0.07603707049930997,
                                   -0.06025842127055635, 0.03297683826326521};
__device__ __forceinline__ double atan2_fast(double y, double x) {
  const double ax = fabs(x), ay = fabs(y);
  const double mx = fmax(ax, ay), mn = fmin(ax, ay);
  // t = mn / mx, reduced when t > tan(pi/8) to (t - 1) / (t + 1) = (mn - mx) / (mn + mx):
  // one division either way (the test mn > tan(pi/8) mx is the same comparison)
  const bool big = mn > 0.41421356237309503 * mx;
  const double t = mx > 0.0 ? (big ? mn - mx : mn) / (big ? mn + mx : mx) : 0.0;
  const double u = t * t;
  double p = c_atan_p[7];
#pragma unroll
  for (int i = 6; i >= 0; --i) p = fma(p, u, c_atan_p[i]);
  double r = fma(t * u, p, t);
  if (big) r += 0.78539816339744828;
  if (ay > ax) r = 1.5707963267948966 - r;
  if (x < 0.0) r = 3.1415926535897931 - r;
  return signbit(y) ? -r : r;
}

// sin(a theta), 1 - cos(a theta) in float (Taylor for |a theta| <= 0.5: error < 1e-10)
__device__ __forceinline__ void rot_sc_f(const ProjArgs& A, float s, float* sn, float* omc) {
  const float a = s * A.theta;
  if (fabsf(a) <= 0.5f) {
    const float a2 = a * a;
    *sn = a * (1.f - a2 * (1.f / 6.f) * (1.f - a2 * (1.f / 20.f) * (1.f - a2 * (1.f / 42.f))));
    *omc = 0.5f * a2 * (1.f - a2 * (1.f / 12.f) * (1.f - a2 * (1.f / 30.f) * (1.f - a2 * (1.f / 56.f))));
  } else {
    float sh, ch;
    sincosf(0.5f * a, &sh, &ch);
    *sn = 2.f * sh * ch;
    *omc = 2.f * sh * sh;
  }
}

// y - sn (k x y) + omc (k (k.y) - y), k = rotation axis  (E^T y for (sn, omc) of +a)
template <typename T>
__device__ __forceinline__ void rot_apply(const T k[3], T sn, T omc, const T y[3], T p[3]) {
  const T cx = k[1] * y[2] - k[2] * y[1], cy = k[2] * y[0] - k[0] * y[2], cz = k[0] * y[1] - k[1] * y[0];
  const T kd = k[0] * y[0] + k[1] * y[1] + k[2] * y[2];
  p[0] = y[0] - sn * cx + omc * (k[0] * kd - y[0]);
  p[1] = y[1] - sn * cy + omc * (k[1] * kd - y[1]);
  p[2] = y[2] - sn * cz + omc * (k[2] * kd - y[2]);
}

// atan(t) for |t| <= 0.2 by the odd series to t^11 (truncation < 1e-10); else atan2f
__device__ __forceinline__ float atan_ratio(float num, float den) {
  if (den > 0.f && fabsf(num) <= 0.2f * den) {
    const float t = __fdividef(num, den), t2 = t * t;
    return t * (1.f - t2 * (1.f / 3.f - t2 * (1.f / 5.f - t2 * (1.f / 7.f - t2 * (1.f / 9.f - t2 * (1.f / 11.f))))));
  }
  return atan2f(num, den);
}

__device__ __forceinline__ float wrap01(float s) { return s < 0.f ? s + 1.f : (s >= 1.f ? s - 1.f : s); }

// firing time of a sensor-frame position (A5): wrap(dir (phi - phi_start)) / 2 pi, clamped
__device__ __forceinline__ float fire_time(const ProjArgs& A, float px, float py) {
  const float inv2pi = 0.15915494309189535f;
  float a = (float)A.dir * (atan2f(py, px) - A.az_start);
  a = a - 6.283185307179586f * floorf(a * inv2pi);
  return fminf(fmaxf(a * inv2pi, 0.f), 1.f);
}

// UT moments of the 7 projected sigma points in (azimuth, elevation) (Eq. 3).
// Outputs: *a0, *e0 = azimuth / elevation of sigma point 0 (double); ma, me = UT mean offsets
// from them (azimuth unwrapped about sigma point 0, A21); caa, cab, cbb = UT covariance;
// s0 = firing time of sigma point 0.
// YAW: the sweep's rotation axis is the sensor z axis (A.axis = (0, 0, +-1) exactly, the
// spinning sensor of a ground vehicle turning in the plane): E(s0) and the small rotation
// between firing times act in the xy plane only, and the general Rodrigues forms reduce to
// the planar ones below (same quantities, fewer operations)
template <bool YAW>
__device__ __forceinline__ void lidar_moments(const ProjArgs& A, const float mu[3], const float L[3][3], double* a0,
                                              double* e0, float* ma, float* me, float* caa, float* cab, float* cbb,
                                              float* s0, bool* valid) {
  const double* R0 = A.R0d;
  const double d0 = (double)mu[0] - A.t0d[0], d1 = (double)mu[1] - A.t0d[1], d2 = (double)mu[2] - A.t0d[2];
  const double cd[3] = {R0[0] * d0 + R0[3] * d1 + R0[6] * d2, R0[1] * d0 + R0[4] * d1 + R0[7] * d2,
                        R0[2] * d0 + R0[5] * d1 + R0[8] * d2};
  const float c[3] = {(float)cd[0], (float)cd[1], (float)cd[2]};
  const bool moving = !A.pose.same && A.K >= 1;
  // ---- firing time of sigma point 0 (float32 decisions; K fixed-point steps from s = 0)
  float s_c = 0.f, s_c1 = 0.f;  // s_c1: the first step (start-frame azimuth), for the offsets below
  if (moving) {
    s_c = s_c1 = fire_time(A, c[0], c[1]);
    for (int it = 1; it < A.K; ++it) {
      float sn, omc, p[3];
      rot_sc_f(A, s_c, &sn, &omc);
      const float y[3] = {c[0] - s_c * A.v[0], c[1] - s_c * A.v[1], c[2] - s_c * A.v[2]};
      rot_apply(A.axis, sn, omc, y, p);
      s_c = fire_time(A, p[0], p[1]);
    }
  }
  *s0 = s_c;
  // ---- sigma point 0 in double
  double p0d[3] = {cd[0], cd[1], cd[2]};
  float E[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};  // E(s0)^T, row-major
  if (moving) {
    // sin / 1 - cos of the rotation to s0 in float32: a relative error of ~6e-8 on terms of
    // at most |a| |y| (a = s0 theta <= the sweep's yaw) moves a 100 m point by < 2e-7 m, i.e.
    // < 2e-9 rad -- far below the box-edge tolerance; the rotation itself stays in double
    float fsn, fomc;
    rot_sc_f(A, s_c, &fsn, &fomc);
    const double sn = fsn, omc = fomc;
    const double y[3] = {cd[0] - (double)s_c * A.vd[0], cd[1] - (double)s_c * A.vd[1],
                         cd[2] - (double)s_c * A.vd[2]};
    rot_apply(A.axis_d, sn, omc, y, p0d);
    const float* k = A.axis;
    const float fs = (float)sn, fo = (float)omc;
    // E^T = I - sn [k]x + omc (k k^T - I)
    E[0] = 1.f + fo * (k[0] * k[0] - 1.f); E[1] = fs * k[2] + fo * k[0] * k[1]; E[2] = -fs * k[1] + fo * k[0] * k[2];
    E[3] = -fs * k[2] + fo * k[1] * k[0]; E[4] = 1.f + fo * (k[1] * k[1] - 1.f); E[5] = fs * k[0] + fo * k[1] * k[2];
    E[6] = fs * k[1] + fo * k[2] * k[0]; E[7] = -fs * k[0] + fo * k[2] * k[1]; E[8] = 1.f + fo * (k[2] * k[2] - 1.f);
  }
  const double rho0d = sqrt(p0d[0] * p0d[0] + p0d[1] * p0d[1]);
  *a0 = atan2_fast(p0d[1], p0d[0]);
  *e0 = atan2_fast(p0d[2], rho0d);
  const float p0[3] = {(float)p0d[0], (float)p0d[1], (float)p0d[2]};
  const float rho0 = (float)rho0d, rho02 = (float)(rho0d * rho0d);
  bool ok = rho0d * rho0d + p0d[2] * p0d[2] >= (double)A.r_min * (double)A.r_min;
  const float cxy2 = c[0] * c[0] + c[1] * c[1];
  const bool pax = rho0d > 0.0, pnz = pax || p0d[2] != 0.0;  // sigma point 0 off the sensor axis / origin
  float Sd = 0.f, Se = 0.f, Sdd = 0.f, See = 0.f, Sde = 0.f;
#pragma unroll 1
  // the three columns rotated through registers: a dynamically indexed L[k] in the
  // non-unrolled loop lived in local memory (spills, 175 -> 171 us)
  float La[3] = {L[0][0], L[0][1], L[0][2]}, Lb[3] = {L[1][0], L[1][1], L[1][2]},
        Lc[3] = {L[2][0], L[2][1], L[2][2]};
  for (int k = 0; k < 3; ++k) {
    // l_k in the start frame
    const float lr[3] = {A.R0[0] * La[0] + A.R0[3] * La[1] + A.R0[6] * La[2],
                         A.R0[1] * La[0] + A.R0[4] * La[1] + A.R0[7] * La[2],
                         A.R0[2] * La[0] + A.R0[5] * La[1] + A.R0[8] * La[2]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      La[c] = Lb[c];
      Lb[c] = Lc[c];
    }
#pragma unroll
    for (int sg = 0; sg < 2; ++sg) {
      const float l[3] = {sg ? -lr[0] : lr[0], sg ? -lr[1] : lr[1], sg ? -lr[2] : lr[2]};
      float D[3];  // p_i - p0
      if (!moving) {
        D[0] = l[0]; D[1] = l[1]; D[2] = l[2];
      } else {
        // firing time of sigma point i (float32): start-frame azimuth relative to sigma point 0's
        // (c x q, c . q) with q = c + l, written without the cancellation: (c x l, |c|^2 + c . l);
        // c on the z axis: sigma point 0's azimuth is atan2(0, 0) = 0 (A21), so q's own azimuth
        // (atan_ratio(y, x) is atan2(y, x) for any arguments)
        const float q[3] = {c[0] + l[0], c[1] + l[1], c[2] + l[2]};
        const bool cax = cxy2 > 0.f;
        float s = wrap01(s_c1 + (float)A.dir *
                                    atan_ratio(cax ? c[0] * l[1] - c[1] * l[0] : q[1],
                                               cax ? cxy2 + c[0] * l[0] + c[1] * l[1] : q[0]) *
                                    0.15915494309189535f);
        for (int it = 1; it < A.K; ++it) {
          float sn, omc, p[3];
          rot_sc_f(A, s, &sn, &omc);
          const float y[3] = {q[0] - s * A.v[0], q[1] - s * A.v[1], q[2] - s * A.v[2]};
          rot_apply(A.axis, sn, omc, y, p);
          s = fire_time(A, p[0], p[1]);
        }
        const float ds = s - s_c;
        const float y[3] = {l[0] - ds * A.v[0], l[1] - ds * A.v[1], l[2] - ds * A.v[2]};
        float w[3];
        if (YAW) {  // E = [[c, s, 0], [-s, c, 0], [0, 0, 1]]
          w[0] = E[0] * y[0] + E[1] * y[1];
          w[1] = E[3] * y[0] + E[4] * y[1];
          w[2] = y[2];
        } else {
          w[0] = E[0] * y[0] + E[1] * y[1] + E[2] * y[2];
          w[1] = E[3] * y[0] + E[4] * y[1] + E[5] * y[2];
          w[2] = E[6] * y[0] + E[7] * y[1] + E[8] * y[2];
        }
        // E(ds) - I for the small rotation between the two firing times (|ds theta| is the
        // particle's angular size times the sweep's yaw, ~1e-3): Taylor to a^4 below 1e-2
        // (truncation < 1e-11), the general form otherwise
        float sn, omc;
        const float ad = ds * A.theta;
        if (fabsf(ad) < 1e-2f) {
          const float a2 = ad * ad;
          sn = ad * (1.f - a2 * (1.f / 6.f));
          omc = 0.5f * a2 * (1.f - a2 * (1.f / 12.f));
        } else {
          rot_sc_f(A, ds, &sn, &omc);
        }
        const float z[3] = {p0[0] + w[0], p0[1] + w[1], p0[2] + w[2]};
        if (YAW) {  // k = (0, 0, kz): k x z = kz (-z1, z0, 0), k (k.z) - z = (-z0, -z1, 0)
          const float snk = sn * A.axis[2];
          D[0] = w[0] + snk * z[1] - omc * z[0];
          D[1] = w[1] - snk * z[0] - omc * z[1];
          D[2] = w[2];
        } else {
          const float* kk = A.axis;
          const float cx = kk[1] * z[2] - kk[2] * z[1], cy = kk[2] * z[0] - kk[0] * z[2], cz = kk[0] * z[1] - kk[1] * z[0];
          const float kd = kk[0] * z[0] + kk[1] * z[1] + kk[2] * z[2];
          D[0] = w[0] - sn * cx + omc * (kk[0] * kd - z[0]);
          D[1] = w[1] - sn * cy + omc * (kk[1] * kd - z[1]);
          D[2] = w[2] - sn * cz + omc * (kk[2] * kd - z[2]);
        }
      }
      const float pz = p0[2] + D[2];
      const float xy = p0[0] * D[0] + p0[1] * D[1];
      const float dxy2 = D[0] * D[0] + D[1] * D[1];
      const float rho2 = rho02 + (2.f * xy + dxy2);
      ok = ok && rho2 + pz * pz >= A.r_min * A.r_min;
      // azimuth offset: atan2(p0 x p_i, p0 . p_i) in the xy plane (A21 unwrap about p0); p0 on
      // the z axis has azimuth atan2(0, 0) = 0 (A21), so the offset is p_i's own azimuth
      const float d = atan_ratio(pax ? p0[0] * D[1] - p0[1] * D[0] : D[1], pax ? rho02 + xy : D[0]);
      // elevation offset: atan2(pz_i rho0 - pz0 rho_i, rho_i rho0 + pz_i pz0) with
      // rho_i - rho0 = (2 p0.D + |D|^2) / (rho_i + rho0)
      const float rho = sqrtf(rho2);
      const float drho = __fdividef(2.f * xy + dxy2, rho + rho0);
      // (p0 = 0: elevation atan2(0, 0) = 0, the offset is p_i's own elevation)
      const float e = atan_ratio(pnz ? D[2] * rho0 - p0[2] * drho : D[2], pnz ? rho * rho0 + pz * p0[2] : rho);
      Sd += d;
      Se += e;
      Sdd = fmaf(d, d, Sdd);
      See = fmaf(e, e, See);
      Sde = fmaf(d, e, Sde);
    }
  }
  // sigma point 0 has offset 0; w_m = (wm0, wmi x 6), w_c = (wc0, wci x 6)
  const float m_a = A.ut.wmi * Sd, m_e = A.ut.wmi * Se;
  *ma = m_a;
  *me = m_e;
  *caa = A.ut.wc0 * m_a * m_a + A.ut.wci * (Sdd - 2.f * m_a * Sd + 6.f * m_a * m_a);
  *cbb = A.ut.wc0 * m_e * m_e + A.ut.wci * (See - 2.f * m_e * Se + 6.f * m_e * m_e);
  *cab = A.ut.wc0 * m_a * m_e + A.ut.wci * (Sde - m_a * Se - m_e * Sd + 6.f * m_a * m_e);
  *valid = ok;
}

// lens projection of a camera-frame point; returns 1 valid, 0 invalid, -1 not computable
__device__ __forceinline__ int cam_frame(const ProjArgs& A, float px, float py, float pz, float* u, float* v) {
  if (A.cam_model == SIMULI_CAM_FISHEYE_KB) {
    const float dist = sqrtf(px * px + py * py + pz * pz);
    if (!(dist > 0.f)) return -1;
    const float rho = sqrtf(px * px + py * py);
    const float th = atan2f(rho, pz);
    const float t2 = th * th;
    const float thd = th * (1.f + t2 * (A.k[0] + t2 * (A.k[1] + t2 * (A.k[2] + t2 * A.k[3]))));
    const float sc = rho > 0.f ? thd / rho : 0.f;
    *u = A.fx * sc * px + A.cx;
    *v = A.fy * sc * py + A.cy;
    return (dist >= A.near_m && th <= A.max_theta) ? 1 : 0;
  }
  if (!(pz > 0.f)) return -1;
  const float th = atan2f(sqrtf(px * px + py * py), pz);
  const float xp = px / pz, yp = py / pz;
  const float r2 = xp * xp + yp * yp;
  const float radial = 1.f + r2 * (A.k[0] + r2 * (A.k[1] + r2 * A.k[4]));
  const float xd = xp * radial + 2.f * A.k[2] * xp * yp + A.k[3] * (r2 + 2.f * xp * xp);
  const float yd = yp * radial + A.k[2] * (r2 + 2.f * yp * yp) + 2.f * A.k[3] * xp * yp;
  *u = A.fx * xd + A.cx;
  *v = A.fy * yd + A.cy;
  return (pz >= A.near_m && th <= A.max_theta) ? 1 : 0;
}

// pose0: the pose at s = 0 (pose_at(A.pose, 0), computed once per CTA in shared memory --
// the same values, without a sincos and a quaternion product per sigma point)
__device__ __forceinline__ int camera_point(const ProjArgs& A, const float x[3], float* u, float* v, float* s_out,
                                            const float* pose0) {
  float s = 0.f;
  int valid = 1;
  const int K = A.pose.same ? 0 : A.K;
  const float invH = 1.0f / (float)A.height;
  for (int it = 0; it <= K; ++it) {
    float R[9], t[3];
    if (s == 0.f) {
#pragma unroll
      for (int i = 0; i < 9; ++i) R[i] = pose0[i];
      t[0] = pose0[9]; t[1] = pose0[10]; t[2] = pose0[11];
    } else {
      pose_at(A.pose, s, R, t);
    }
    const float d0 = x[0] - t[0], d1 = x[1] - t[1], d2 = x[2] - t[2];
    const float px = R[0] * d0 + R[3] * d1 + R[6] * d2;
    const float py = R[1] * d0 + R[4] * d1 + R[7] * d2;
    const float pz = R[2] * d0 + R[5] * d1 + R[8] * d2;
    const int st = cam_frame(A, px, py, pz, u, v);
    if (st < 0) return -1;
    if (st == 0) valid = 0;
    if (it < K) s = A.rolling ? fminf(fmaxf(*v * invH, 0.f), 1.f) : 0.f;
  }
  *s_out = s;
  return valid;
}

#ifndef SIMULI_PROJ_MINB
#define SIMULI_PROJ_MINB 4
#endif
#ifndef SIMULI_PROJ_THREADS
#define SIMULI_PROJ_THREADS 256
#endif
constexpr double kPiD = 3.141592653589793;
constexpr int kSmemBounds = 264;

template <int KIND, bool DIV, bool ACT, bool YAW>
__global__ void __launch_bounds__(SIMULI_PROJ_THREADS, SIMULI_PROJ_MINB) k_project(const ProjArgs Ain) {
  pdl_wait();
  pdl_trigger();
  // tiling boundaries / row scales staged in shared memory (binary searches hit smem)
  __shared__ float s_bounds[kSmemBounds], s_rscale[kSmemBounds];
  __shared__ float s_pose0[12];  // camera: the pose at s = 0
  ProjArgs A = Ain;
  if (KIND == SIMULI_SENSOR_CAMERA) {
    if (threadIdx.x == 0) pose_at(Ain.pose, 0.f, s_pose0, s_pose0 + 9);
    __syncthreads();
  }
  if (KIND == SIMULI_SENSOR_LIDAR && Ain.n_phi + 1 <= kSmemBounds) {
    for (int i = threadIdx.x; i <= Ain.n_phi; i += blockDim.x) {
      s_bounds[i] = __ldg(Ain.bounds + i);
      if (i < Ain.n_phi) s_rscale[i] = __ldg(Ain.row_scale + i);
    }
    __syncthreads();
    A.bounds = s_bounds;
    A.row_scale = s_rscale;
  }
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= A.n) return;
#ifndef SIMULI_NO_SH_PREFETCH
  // the degree-3 SH blocks (192 B each) are read only for kept particles, ~2000
  // instructions later; one bulk L2 prefetch of the warp's 32 contiguous blocks now (every
  // particle: culling is not known yet) turns those reads from DRAM misses into L2 hits --
  // they were the kernel's largest stall (long_scoreboard at the first SH FMA: 14 % of its
  // warp samples, r02k_scan)
  if (A.sh_degree == 3 && (threadIdx.x & 31) == 0) {
    const int64_t cnt = A.n - g < 32 ? A.n - g : 32;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.sh + g * 48), "r"((unsigned)(cnt * 192))
                 : "memory");
  }
#endif
  // SoA loads (quaternion as one 16-byte load)
  float mu[3] = {__ldg(A.means + 3 * g), __ldg(A.means + 3 * g + 1), __ldg(A.means + 3 * g + 2)};
  float4 q4 = __ldg(reinterpret_cast<const float4*>(A.quats) + g);
  const float sc[3] = {__ldg(A.scales + 3 * g), __ldg(A.scales + 3 * g + 1), __ldg(A.scales + 3 * g + 2)};
  const float sigma = __ldg(A.opacity + g);
  bool actor_ok = true;
  if (ACT) {
    // scene graph (A29): object particle -> world with its object's pose at t;
    // the mean in double, rounded once; q_w = q_a (x) q in float (normalised below)
    const int a = __ldg(A.actor_id + g);
    if (a >= 0 && a < A.n_actors) {
      const float* ap = A.actor_pose + 7 * (size_t)a;
      const float qa4[4] = {__ldg(ap), __ldg(ap + 1), __ldg(ap + 2), __ldg(ap + 3)};
      const double qn = sqrt((double)qa4[0] * qa4[0] + (double)qa4[1] * qa4[1] + (double)qa4[2] * qa4[2] +
                             (double)qa4[3] * qa4[3]);
      const double w = qa4[0] / qn, x = qa4[1] / qn, y = qa4[2] / qn, z = qa4[3] / qn;
      const double Ra[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                            2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                            2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
      const double m0 = mu[0], m1 = mu[1], m2 = mu[2];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        mu[c] = __double2float_rn(Ra[3 * c] * m0 + Ra[3 * c + 1] * m1 + Ra[3 * c + 2] * m2 + (double)__ldg(ap + 4 + c));
      const float aw = (float)w, ax = (float)x, ay = (float)y, az = (float)z;
      const float4 ql = q4;
      q4.x = aw * ql.x - ax * ql.y - ay * ql.z - az * ql.w;
      q4.y = aw * ql.y + ax * ql.x + ay * ql.w - az * ql.z;
      q4.z = aw * ql.z - ax * ql.w + ay * ql.x + az * ql.y;
      q4.w = aw * ql.w + ax * ql.z - ay * ql.y + az * ql.x;
      actor_ok = qn > 0.0 && isfinite(qn);
    } else {
      actor_ok = a == -1;
    }
  }

  // ---- depth key (A19): exact float32 op sequence
  {
    const float d0 = __fsub_rn(mu[0], A.o_mid[0]), d1 = __fsub_rn(mu[1], A.o_mid[1]),
                d2 = __fsub_rn(mu[2], A.o_mid[2]);
    A.key[g] = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(d0, d0), __fmul_rn(d1, d1)), __fmul_rn(d2, d2)));
  }
  int count = 0;
  int rect[4] = {0, 0, 0, 0};
  float box[4] = {NAN, NAN, NAN, NAN};
  float M[9] = {NAN, NAN, NAN, NAN, NAN, NAN, NAN, NAN, NAN}, f[3] = {0.f, 0.f, 0.f};
  float vdir[3] = {0.f, 0.f, 0.f};
  bool ok = true;

  const float qn2 = q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w;
  ok = actor_ok && qn2 > 0.f && isfinite(qn2);
#pragma unroll
  for (int c = 0; c < 3; ++c) ok = ok && sc[c] > 0.f && isfinite(sc[c]) && isfinite(mu[c]);
  if (ok) {
    const float inv = rsqrtf(qn2);
    const float q[4] = {q4.x * inv, q4.y * inv, q4.z * inv, q4.w * inv};
    float R[9];
    quat_rot(q, R);
    float L[3][3];  // L[k] = spread * s_k * column k of R
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) L[k][c] = A.ut.spread * sc[k] * R[3 * c + k];

    float ma, mb, caa, cab, cbb, s0 = 0.f;
    double a0 = 0.0, e0 = 0.0;
    bool valid = true, computable = true;
    // beam divergence (App. C; A27): Sigma_hat = Sigma + theta^2 (r^2 I - v v^T),
    // v = mu - o, o = sensor position at the mean's firing time; its Cholesky factor is the
    // sigma-point square root and its inverse the canonical transform (Sigma_hat^-1 = M^T M)
    float Mh[9];
    constexpr bool div = KIND == SIMULI_SENSOR_LIDAR && DIV;  // (A.beam_div > 0, a separate instantiation)
    if (div) {
      const float d0 = mu[0] - A.t0w[0], d1 = mu[1] - A.t0w[1], d2 = mu[2] - A.t0w[2];
      const float cs[3] = {A.R0[0] * d0 + A.R0[3] * d1 + A.R0[6] * d2, A.R0[1] * d0 + A.R0[4] * d1 + A.R0[7] * d2,
                           A.R0[2] * d0 + A.R0[5] * d1 + A.R0[8] * d2};
      float sf = 0.f;
      if (!A.pose.same && A.K >= 1) {
        sf = fire_time(A, cs[0], cs[1]);
        for (int it = 1; it < A.K; ++it) {
          float sn, omc, p[3];
          rot_sc_f(A, sf, &sn, &omc);
          const float y[3] = {cs[0] - sf * A.v[0], cs[1] - sf * A.v[1], cs[2] - sf * A.v[2]};
          rot_apply(A.axis, sn, omc, y, p);
          sf = fire_time(A, p[0], p[1]);
        }
      }
      const float v[3] = {mu[0] - (A.t0w[0] + sf * A.dtw[0]), mu[1] - (A.t0w[1] + sf * A.dtw[1]),
                          mu[2] - (A.t0w[2] + sf * A.dtw[2])};
      const float r2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2], t2 = A.beam_div * A.beam_div;
      float Sh[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < 3; ++k) acc += R[3 * i + k] * R[3 * j + k] * (sc[k] * sc[k]);
          Sh[i][j] = acc + t2 * ((i == j ? r2 : 0.f) - v[i] * v[j]);
        }
      const float l00 = sqrtf(Sh[0][0]), l10 = Sh[1][0] / l00, l20 = Sh[2][0] / l00;
      const float q11 = Sh[1][1] - l10 * l10;
      const float l11 = sqrtf(q11), l21 = (Sh[2][1] - l20 * l10) / l11;
      const float q22 = Sh[2][2] - l20 * l20 - l21 * l21;
      const float l22 = sqrtf(q22);
      computable = Sh[0][0] > 0.f && q11 > 0.f && q22 > 0.f && isfinite(l22);
      const float sp = A.ut.spread;
      L[0][0] = sp * l00; L[0][1] = sp * l10; L[0][2] = sp * l20;  // columns of chol(Sigma_hat)
      L[1][0] = 0.f;      L[1][1] = sp * l11; L[1][2] = sp * l21;
      L[2][0] = 0.f;      L[2][1] = 0.f;      L[2][2] = sp * l22;
      const float m00 = 1.0f / l00, m11 = 1.0f / l11, m22 = 1.0f / l22;
      const float m10 = -l10 * m00 * m11, m21 = -l21 * m11 * m22, m20 = -(l20 * m00 + l21 * m10) * m22;
      Mh[0] = m00; Mh[1] = 0.f; Mh[2] = 0.f;
      Mh[3] = m10; Mh[4] = m11; Mh[5] = 0.f;
      Mh[6] = m20; Mh[7] = m21; Mh[8] = m22;
    }
    if (KIND == SIMULI_SENSOR_LIDAR) {
      lidar_moments<YAW>(A, mu, L, &a0, &e0, &ma, &mb, &caa, &cab, &cbb, &s0, &valid);
    } else {
    // ---- 7 sigma points through the sensor model
    float ya[7], yb[7];
#pragma unroll 1
    for (int i = 0; i < 7; ++i) {
      float x[3] = {mu[0], mu[1], mu[2]};
      if (i > 0) {
        const int k = (i - 1) % 3;
        const float sg = i <= 3 ? 1.f : -1.f;
        x[0] += sg * L[k][0];
        x[1] += sg * L[k][1];
        x[2] += sg * L[k][2];
      }
      float s;
      const int st = camera_point(A, x, &ya[i], &yb[i], &s, s_pose0);
      computable = computable && st >= 0;
      valid = valid && st == 1;
      if (i == 0) s0 = s;
    }
    // ---- UT moments
    ma = A.ut.wm0 * ya[0];
    mb = A.ut.wm0 * yb[0];
#pragma unroll
    for (int i = 1; i < 7; ++i) {
      ma += A.ut.wmi * ya[i];
      mb += A.ut.wmi * yb[i];
    }
    caa = 0.f; cab = 0.f; cbb = 0.f;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const float w = i == 0 ? A.ut.wc0 : A.ut.wci;
      const float ea = ya[i] - ma, eb = yb[i] - mb;
      caa += w * ea * ea;
      cab += w * ea * eb;
      cbb += w * eb * eb;
    }
    }
    // UT mean: sigma point 0 (double, LiDAR) + float32 offset; the azimuth wrapped into
    // [-pi, pi) (A11); box edges rounded outward from double (A11)
    double ya_bar = a0 + (double)ma, yb_bar = e0 + (double)mb;
    const float det = caa * cbb - cab * cab;
    const bool boxok = computable && isfinite(ya_bar) && isfinite(yb_bar) && caa > 0.f && cbb > 0.f && det > 0.f &&
                       isfinite(det);
    ok = boxok && valid;
    if (boxok) {
      if (KIND == SIMULI_SENSOR_LIDAR) {
        if (ya_bar >= kPiD) ya_bar -= 2.0 * kPiD;
        else if (ya_bar < -kPiD) ya_bar += 2.0 * kPiD;
      }
      // half-widths: a float32 root (relative error 2^-24 of ~1e-3 rad: ~1e-10 rad) is exact
      // enough; the edges themselves are summed and rounded outward in double
      const double ha = (double)(A.ks * __fsqrt_rn(caa)), hb = (double)(A.ks * __fsqrt_rn(cbb));
      box[0] = __double2float_rd(ya_bar - ha);
      box[1] = __double2float_ru(ya_bar + ha);
      box[2] = __double2float_rd(yb_bar - hb);
      box[3] = __double2float_ru(yb_bar + hb);
    }
    if (ok) {
      // ---- culling + render-tile rectangle
      if (KIND == SIMULI_SENSOR_LIDAR && A.enable_cull == 2) {
        count = exact_rect(A, box, rect);
      } else if (KIND == SIMULI_SENSOR_LIDAR) {
        const float b0 = A.bounds[0], bl = A.bounds[A.n_phi];
        bool keep = !(box[3] < b0 || box[2] > bl);
        const int e0 = elev_tile(A, box[2]), e1 = elev_tile(A, box[3]);
        if (keep && A.enable_cull) {
          const int r0 = dense_row_e(A, box[2], e0), r1 = dense_row_e(A, box[3], e1);
          int cs, cl;
          az_run(box[0], box[1], A.pi_f, A.two_pi_f, A.az_cell_scale, A.az_cells, &cs, &cl);
          const int ce = cs + cl - 1;
          int occ;
          if (ce < A.az_cells) occ = sat_rect(A, r0, r1, cs, ce);
          else occ = sat_rect(A, r0, r1, cs, A.az_cells - 1) + sat_rect(A, r0, r1, 0, ce - A.az_cells);
          keep = occ > 0;
        }
        if (keep) {
          int cs, cl;
          az_run(box[0], box[1], A.pi_f, A.two_pi_f, A.az_tile_scale, A.n_theta, &cs, &cl);
          rect[0] = e0; rect[1] = e1; rect[2] = cs; rect[3] = cl;
          count = (e1 - e0 + 1) * cl;
        }
      } else {
        const bool outside = box[1] < 0.5f || box[0] > (float)A.width - 0.5f || box[3] < 0.5f ||
                             box[2] > (float)A.height - 0.5f;
        if (!outside) {
          const int c0 = clamp_floor(__fmul_rn(box[0], A.inv_tile), A.Wt);
          const int c1 = clamp_floor(__fmul_rn(box[1], A.inv_tile), A.Wt);
          const int r0 = clamp_floor(__fmul_rn(box[2], A.inv_tile), A.Ht);
          const int r1 = clamp_floor(__fmul_rn(box[3], A.inv_tile), A.Ht);
          rect[0] = r0; rect[1] = r1; rect[2] = c0; rect[3] = c1 - c0 + 1;
          count = (r1 - r0 + 1) * (c1 - c0 + 1);
        }
      }
    }
    if (ok && (count > 0 || A.write_all)) {
      // ---- record: canonical transform M = diag(1/s) R^T, SH features (A17)
      if (div) {
#pragma unroll
        for (int i = 0; i < 9; ++i) M[i] = Mh[i];
      } else {
        // R recomputed from the normalised quaternion (not kept live through the UT: registers)
        float Rm[9];
        quat_rot(q, Rm);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float is = 1.0f / sc[k];
#pragma unroll
          for (int c = 0; c < 3; ++c) M[3 * k + c] = Rm[3 * c + k] * is;
        }
      }
      float Rs[9], ts[3];
      if (KIND == SIMULI_SENSOR_LIDAR) {
        ts[0] = A.t0w[0] + s0 * A.dtw[0];
        ts[1] = A.t0w[1] + s0 * A.dtw[1];
        ts[2] = A.t0w[2] + s0 * A.dtw[2];
      } else {
        pose_at(A.pose, s0, Rs, ts);
      }
      float vx = mu[0] - ts[0], vy = mu[1] - ts[1], vz = mu[2] - ts[2];
      vdir[0] = vx; vdir[1] = vy; vdir[2] = vz;  // the view vector, unnormalised (backward, A31)
      const float vn = rsqrtf(vx * vx + vy * vy + vz * vz);
      vx *= vn; vy *= vn; vz *= vn;
      if (isfinite(vn)) {
        // the SH block (192 B, degree 3) is read only for kept particles (A17): 12 float4
        if (A.sh_degree == 3) {
          float bsh[16];
          sh_basis3(vx, vy, vz, bsh);
          sh_dot(A.sh + g * 48, 16, bsh, f);
        } else {
          sh_eval(A.sh + g * A.n_coef * 3, A.sh_degree, vx, vy, vz, f);
        }
      }
    }
  }
  SIMULI_CHECK(count >= 0 && (KIND != SIMULI_SENSOR_LIDAR || count <= A.n_phi * A.n_theta), count, g);
  SIMULI_CHECK(count == 0 || (rect[0] >= 0 && rect[2] >= 0 && rect[3] >= 1), rect[0], rect[2]);
  A.count[g] = count;
  reinterpret_cast<int4*>(A.rect)[g] = make_int4(rect[0], rect[1], rect[2], rect[3]);
  if (count > 0 || A.write_all) {
    float4* rec = reinterpret_cast<float4*>(A.record + g * kRecordFloats);
    rec[0] = make_float4(mu[0], mu[1], mu[2], M[0]);
    rec[1] = make_float4(M[1], M[2], M[3], M[4]);
    rec[2] = make_float4(M[5], M[6], M[7], M[8]);
    rec[3] = make_float4(sigma, f[0], f[1], f[2]);
    rec[4] = ok ? make_float4(box[0], box[1], box[2], box[3]) : make_float4(NAN, NAN, NAN, NAN);
    if (A.view_dir) {
      A.view_dir[3 * g] = vdir[0];
      A.view_dir[3 * g + 1] = vdir[1];
      A.view_dir[3 * g + 2] = vdir[2];
    }
  }
}

}  // namespace

bool ut_weights(float alpha, float beta, float kappa, float* spread, float* wm0, float* wmi, float* wc0, float* wci) {
  const double n = 3.0, a = alpha, b = beta, k = kappa;
  const double lambda = a * a * (n + k) - n;
  if (!(n + lambda > 0.0)) return false;
  *spread = static_cast<float>(std::sqrt(n + lambda));
  *wm0 = static_cast<float>(lambda / (n + lambda));
  *wc0 = static_cast<float>(lambda / (n + lambda) + (1.0 - a * a + b));
  *wmi = *wci = static_cast<float>(1.0 / (2.0 * (n + lambda)));
  return true;
}

// o_mid = t0 + 0.5 (t1 - t0) with float32 ops (host, no FMA): bit-identical definition (A19)
static void depth_origin(const simuli_pose& a, const simuli_pose& b, float out[3]) {
  for (int c = 0; c < 3; ++c) {
    volatile float h = b.t[c] - a.t[c];
    volatile float hm = 0.5f * h;
    volatile float om = a.t[c] + hm;
    out[c] = om;
  }
}

template <int KIND, bool DIV, bool ACT, bool YAW = false>
void launch_project(const ProjArgs& A, unsigned blocks, int threads, cudaStream_t st) {
  launch_pdl(k_project<KIND, DIV, ACT, YAW>, blocks, threads, 0, st, A);
}

}  // namespace simuli

extern "C" int32_t simuli_project(const simuli_gaussians* G, const simuli_project_params* P, simuli_projected* out,
                                  void* stream) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(G && P && out, "simuli_project: NULL argument");
  SIMULI_REQUIRE(G->n >= 0, "simuli_project: n < 0");
  if (G->sh_degree < 0 || G->sh_degree > 3) {
    set_error("simuli_project: sh_degree %d not in 0..3", G->sh_degree);
    return SIMULI_ERR_UNSUPPORTED;
  }
  if (G->n == 0) return SIMULI_OK;
  SIMULI_REQUIRE(G->means && G->quats && G->scales && G->opacity && G->sh, "simuli_project: NULL Gaussian array");
  SIMULI_REQUIRE(out->record && out->tile_rect && out->depth_key && out->tile_count, "simuli_project: NULL output");
  SIMULI_REQUIRE(G->sh_degree != 3 || reinterpret_cast<uintptr_t>(G->sh) % 16 == 0,
                 "simuli_project: sh must be 16-byte aligned for degree 3 (read as float4)");
  SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(G->quats) % 16 == 0 && reinterpret_cast<uintptr_t>(out->record) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(out->tile_rect) % 16 == 0,
                 "simuli_project: quats / record / tile_rect must be 16-byte aligned");
  SIMULI_REQUIRE(P->rs_iterations >= 0 && P->rs_iterations <= 16, "rs_iterations must be in [0, 16]");
  SIMULI_REQUIRE(P->extent_sigma > 0.f, "extent_sigma must be > 0");
  ProjArgs A{};
  A.n = G->n;
  A.means = G->means; A.quats = G->quats; A.scales = G->scales; A.opacity = G->opacity; A.sh = G->sh;
  A.sh_degree = G->sh_degree;
  A.n_coef = (G->sh_degree + 1) * (G->sh_degree + 1);
  const bool act = G->actor_id != nullptr;
  if (act) {
    SIMULI_REQUIRE(G->n_actors >= 1 && G->actor_pose, "simuli_project: actor_id needs n_actors >= 1 and actor_pose");
    static_assert(sizeof(simuli_pose) == 7 * sizeof(float), "simuli_pose must be 7 packed floats");
    A.actor_id = G->actor_id;
    A.actor_pose = reinterpret_cast<const float*>(G->actor_pose);
    A.n_actors = G->n_actors;
  }
  A.pose = make_pose_interp_f(make_pose_interp_d(P->pose_start, P->pose_end));
  A.K = P->rs_iterations;
  SIMULI_REQUIRE(ut_weights(P->ut_alpha, P->ut_beta, P->ut_kappa, &A.ut.spread, &A.ut.wm0, &A.ut.wmi, &A.ut.wc0,
                            &A.ut.wci),
                 "invalid UT parameters: alpha^2 (3 + kappa) must be > 0");
  A.ks = P->extent_sigma;
  depth_origin(P->pose_start, P->pose_end, A.o_mid);
  A.write_all = P->write_all_records;
  A.record = out->record; A.rect = out->tile_rect; A.key = out->depth_key; A.count = out->tile_count;
  A.view_dir = out->view_dir;
  const int threads = SIMULI_PROJ_THREADS;
  const unsigned blocks = static_cast<unsigned>((G->n + threads - 1) / threads);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (P->kind == SIMULI_SENSOR_LIDAR) {
    SIMULI_REQUIRE(P->lidar && P->tiling, "LiDAR projection needs lidar and tiling");
    const simuli_tiling_dev& T = *P->tiling;
    SIMULI_REQUIRE(T.elev_bounds && T.cull_row_scale && T.sat && T.n_phi >= 1 && T.n_theta >= 1,
                   "incomplete device tiling");
    SIMULI_REQUIRE(P->lidar->min_range_m > 0.f, "min_range_m must be > 0");
    A.az_start = P->lidar->azimuth_start_rad;
    A.dir = P->lidar->spin_direction;
    A.r_min = P->lidar->min_range_m;
    SIMULI_REQUIRE(P->lidar->beam_divergence_rad >= 0.f, "beam_divergence_rad must be >= 0");
    A.beam_div = P->lidar->beam_divergence_rad;
    {
      // launch constants of the sensor model: R0 = R(q0), t0, dt = t1 - t0, v = R0^T dt,
      // rotation axis k (in the start frame) and angle theta of R0^T R1 (host, double)
      const PoseInterpD pd = make_pose_interp_d(P->pose_start, P->pose_end);
      double R0d[9];
      {
        const double w = pd.q0[0], x = pd.q0[1], y = pd.q0[2], z = pd.q0[3];
        const double Rr[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                              2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                              2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
        for (int i = 0; i < 9; ++i) R0d[i] = Rr[i];
      }
      for (int i = 0; i < 9; ++i) A.R0[i] = static_cast<float>(R0d[i]);
      for (int i = 0; i < 3; ++i) {
        A.t0w[i] = P->pose_start.t[i];
        A.dtw[i] = static_cast<float>(pd.dt[i]);
        A.axis[i] = static_cast<float>(pd.axis[i]);
        A.v[i] = static_cast<float>(R0d[0 * 3 + i] * pd.dt[0] + R0d[1 * 3 + i] * pd.dt[1] + R0d[2 * 3 + i] * pd.dt[2]);
      }
      A.theta = static_cast<float>(2.0 * pd.half_theta);
      A.theta_d = 2.0 * pd.half_theta;
      for (int i = 0; i < 9; ++i) A.R0d[i] = R0d[i];
      for (int i = 0; i < 3; ++i) {
        A.t0d[i] = pd.t0[i];
        A.axis_d[i] = pd.axis[i];
        A.vd[i] = R0d[0 * 3 + i] * pd.dt[0] + R0d[1 * 3 + i] * pd.dt[1] + R0d[2 * 3 + i] * pd.dt[2];
      }
      A.small_rot = std::fabs(2.0 * pd.half_theta) <= 0.5 ? 1 : 0;
    }
    A.n_phi = T.n_phi; A.n_theta = T.n_theta; A.rows_per_tile = T.cull_rows_per_tile;
    A.az_cells = T.cull_az_cells; A.sat_cols = T.sat_cols; A.enable_cull = P->enable_culling;
    A.pi_f = T.pi_f; A.two_pi_f = T.two_pi_f; A.az_tile_scale = T.az_tile_scale; A.az_cell_scale = T.az_cell_scale;
    A.bounds = T.elev_bounds; A.row_scale = T.cull_row_scale; A.sat = T.sat;
    SIMULI_REQUIRE(P->enable_culling >= 0 && P->enable_culling <= 2, "simuli_project: enable_culling must be 0, 1 or 2");
    if (P->enable_culling == 2) {
      SIMULI_REQUIRE(T.beam_el_sorted && T.col_az_sorted && T.n_beams >= 1 && T.n_azimuth >= 1,
                     "simuli_project: exact culling needs beam_el_sorted / col_az_sorted");
      A.beam_sorted = T.beam_el_sorted; A.col_sorted = T.col_az_sorted;
      A.n_beams = T.n_beams; A.n_az = T.n_azimuth;
      A.col_step = (float)(T.n_azimuth / (2.0 * 3.14159265358979323846));
    }
    // rotation about the sensor z axis (yaw only): the planar sigma-point forms
    const bool yaw = A.axis[0] == 0.f && A.axis[1] == 0.f && std::fabs(A.axis[2]) == 1.f;
    if (A.beam_div > 0.f) {
      if (act) yaw ? launch_project<SIMULI_SENSOR_LIDAR, true, true, true>(A, blocks, threads, st)
                   : launch_project<SIMULI_SENSOR_LIDAR, true, true>(A, blocks, threads, st);
      else yaw ? launch_project<SIMULI_SENSOR_LIDAR, true, false, true>(A, blocks, threads, st)
               : launch_project<SIMULI_SENSOR_LIDAR, true, false>(A, blocks, threads, st);
    } else {
      if (act) yaw ? launch_project<SIMULI_SENSOR_LIDAR, false, true, true>(A, blocks, threads, st)
                   : launch_project<SIMULI_SENSOR_LIDAR, false, true>(A, blocks, threads, st);
      else yaw ? launch_project<SIMULI_SENSOR_LIDAR, false, false, true>(A, blocks, threads, st)
               : launch_project<SIMULI_SENSOR_LIDAR, false, false>(A, blocks, threads, st);
    }
  } else if (P->kind == SIMULI_SENSOR_CAMERA) {
    SIMULI_REQUIRE(P->camera, "camera projection needs camera");
    const simuli_camera& C = *P->camera;
    SIMULI_REQUIRE(C.width > 0 && C.height > 0 && C.fx > 0 && C.fy > 0, "invalid camera size / focal");
    if (C.tile_px != 8 && C.tile_px != 16) {  // the camera render / backward tile shapes
      set_error("simuli_project: camera tile_px %d not supported (8 or 16)", C.tile_px);
      return SIMULI_ERR_UNSUPPORTED;
    }
    SIMULI_REQUIRE(C.model == SIMULI_CAM_FISHEYE_KB || C.model == SIMULI_CAM_PINHOLE_RADTAN, "unknown camera model");
    A.cam_model = C.model; A.width = C.width; A.height = C.height; A.rolling = C.rolling_shutter;
    A.tile_px = C.tile_px; A.Wt = (C.width + C.tile_px - 1) / C.tile_px; A.Ht = (C.height + C.tile_px - 1) / C.tile_px;
    A.fx = C.fx; A.fy = C.fy; A.cx = C.cx; A.cy = C.cy;
    for (int i = 0; i < 5; ++i) A.k[i] = C.k[i];
    A.near_m = C.near_m; A.max_theta = C.max_theta_rad; A.inv_tile = 1.0f / (float)C.tile_px;
    if (act) launch_project<SIMULI_SENSOR_CAMERA, false, true>(A, blocks, threads, st);
    else launch_project<SIMULI_SENSOR_CAMERA, false, false>(A, blocks, threads, st);
  } else {
    set_error("simuli_project: unknown sensor kind %d", P->kind);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("simuli_project: launch failed: %s", cudaGetErrorString(e));
    return SIMULI_ERR_CUDA;
  }
  return SIMULI_OK;
}
