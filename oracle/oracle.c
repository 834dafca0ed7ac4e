/*
 * oracle.c -- CPU ORACLE FOR THE SIMULI HOT PATH.  TEST INFRASTRUCTURE ONLY.
 *
 * See oracle.h for the usage rule (tests / smoke / bench cpu_baseline only) and the
 * citation format.  Every function restates a passage of PAPER.md (P:n) in the paper's
 * order; where the paper is silent the SURVEY.md §8(c) reading is cited as "A<n>" and
 * listed in DESIGN.md §3.  Plain loops, double precision, no blocking or fusion.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC.
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py.  The whole
 * render on realistic scenes, which the paper gives no numbers for, is pinned by bitwise
 * scale covariance (2x lengths -> 2x depth, every other output identical), rigid
 * invariance, tiled == brute force and conservation.  O6's lens models
 * (KB fisheye, OpenCV radtan) and their inverses are pinned to OpenCV (cv2.fisheye /
 * cv2.projectPoints / undistortPoints, <= 1e-9 px, <= 1e-12 rad).  O8's exact culling mode
 * (A32) is pinned by brute force over every ray.  The NEXT-row
 * functions are pinned too: O0 (scipy + rigid invariance), O14 (constant map / identity
 * grid, texel centres, affine-field exactness), O15/O16 (central finite differences of the
 * forward, LiDAR and camera, with scene graph and per-ray SH; SH linearity; the opacity
 * scaling identity).
 */
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846
#define OR_TWO_PI (2.0 * OR_PI)

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
int or_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------
 * O1  Rotation and covariance.  Sigma = R S S^T R^T with R from a (normalised)
 *     quaternion (w,x,y,z) and S = diag(s)  -- P:73 §3.1; A26.
 * ---------------------------------------------------------------------------------- */
void or_quat_to_rot(const double q_in[4], double R[9]) {
  double n = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
  double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
}

void or_covariance(const double q[4], const double s[3], double Sigma[9]) {
  double R[9], RS[9];
  or_quat_to_rot(q, R);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) RS[i * 3 + k] = R[i * 3 + k] * s[k];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += RS[i * 3 + k] * RS[j * 3 + k];
      Sigma[i * 3 + j] = acc;
    }
}

/* ------------------------------------------------------------------------------------
 * O2  Unscented transform, 7 sigma points ("We project 7 sigma points").
 *     Scaled UT with (alpha, beta, kappa) (A1); square root of Sigma = R diag(s) (A2).
 *     lambda = alpha^2 (n + kappa) - n, n = 3;  spread = sqrt(n + lambda)
 *     wm0 = lambda/(n+lambda), wc0 = wm0 + 1 - alpha^2 + beta, wi = 1/(2(n+lambda)).
 * ---------------------------------------------------------------------------------- */
int or_ut_weights(const double ut[3], double* spread, double wm[7], double wc[7]) {
  const double n = 3.0;
  double alpha = ut[0], beta = ut[1], kappa = ut[2];
  double lambda = alpha * alpha * (n + kappa) - n;
  if (!(n + lambda > 0.0)) return -1;
  *spread = sqrt(n + lambda);
  wm[0] = lambda / (n + lambda);
  wc[0] = wm[0] + (1.0 - alpha * alpha + beta);
  for (int i = 1; i < 7; ++i) {
    wm[i] = 1.0 / (2.0 * (n + lambda));
    wc[i] = wm[i];
  }
  return 0;
}

int or_sigma_points(const double mu[3], const double q[4], const double s[3], const double ut[3],
                    double pts[21], double wm[7], double wc[7]) {
  double spread, R[9];
  if (or_ut_weights(ut, &spread, wm, wc)) return -1;
  or_quat_to_rot(q, R);
  for (int c = 0; c < 3; ++c) pts[c] = mu[c];
  for (int k = 0; k < 3; ++k) {      /* l_k = s_k * (column k of R) */
    for (int c = 0; c < 3; ++c) {
      double l = s[k] * R[c * 3 + k];
      pts[(1 + k) * 3 + c] = mu[c] + spread * l;
      pts[(4 + k) * 3 + c] = mu[c] - spread * l;
    }
  }
  return 0;
}

/* Sigma points from an arbitrary square root Lsq of the covariance (Lsq Lsq^T = Sigma):
 * mu, mu +- spread * (column k of Lsq).  Used with the Cholesky factor of the beam-
 * divergence covariance Sigma_hat (App. C; reading A27). */
int or_sigma_points_sqrt(const double mu[3], const double Lsq[9], const double ut[3], double pts[21], double wm[7],
                         double wc[7]) {
  double spread;
  if (or_ut_weights(ut, &spread, wm, wc)) return -1;
  for (int c = 0; c < 3; ++c) pts[c] = mu[c];
  for (int k = 0; k < 3; ++k)
    for (int c = 0; c < 3; ++c) {
      pts[(1 + k) * 3 + c] = mu[c] + spread * Lsq[c * 3 + k];
      pts[(4 + k) * 3 + c] = mu[c] - spread * Lsq[c * 3 + k];
    }
  return 0;
}

/* ------------------------------------------------------------------------------------
 * O2b Beam divergence (App. C): a 3D smoothing filter that widens
 *     each LiDAR particle by the beam footprint orthogonal to the viewing direction,
 *       Sigma_hat = Sigma + (theta_div r)^2 (I - d d^T),  d = (mu - o)/r,  r = |mu - o|,
 *     and the response uses Sigma_hat WITHOUT the opacity factor sqrt(|Sigma_perp| /
 *     |Sigma_hat_perp|) of AAA-Gaussians (the paper's modification).  o = sensor position
 *     at the firing time of the particle mean (the sigma-point-0 time of A17; reading A27).
 * ---------------------------------------------------------------------------------- */
void or_divergence_cov(const double Sigma[9], const double mu[3], const double o[3], double theta, double Sh[9]) {
  double d[3] = {mu[0] - o[0], mu[1] - o[1], mu[2] - o[2]};
  double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  double r = sqrt(r2);
  double w = (theta * r) * (theta * r);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double dd = r > 0.0 ? (d[i] / r) * (d[j] / r) : 0.0;
      Sh[i * 3 + j] = Sigma[i * 3 + j] + w * ((i == j ? 1.0 : 0.0) - dd);
    }
}

/* Cholesky factor of a symmetric positive definite 3x3 (textbook, row by row). */
int or_cholesky3(const double S[9], double L[9]) {
  for (int i = 0; i < 9; ++i) L[i] = 0.0;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j <= i; ++j) {
      double acc = S[i * 3 + j];
      for (int k = 0; k < j; ++k) acc -= L[i * 3 + k] * L[j * 3 + k];
      if (i == j) {
        if (!(acc > 0.0)) return -1;
        L[i * 3 + i] = sqrt(acc);
      } else {
        L[i * 3 + j] = acc / L[j * 3 + j];
      }
    }
  }
  return 0;
}

/* Inverse of a lower-triangular 3x3 by forward substitution on the identity columns. */
void or_lower_inverse3(const double L[9], double M[9]) {
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) {
      double acc = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) acc -= L[i * 3 + k] * M[k * 3 + c];
      M[i * 3 + c] = acc / L[i * 3 + i];
    }
}

/* UT moments of 7 projected 2-vectors ("estimate a 2D conic").  If wrap_a, the
 * first coordinate is an azimuth, unwrapped about sigma point 0 (A21). */
static void ut_moments(const double y[7][2], const double wm[7], const double wc[7], int wrap_a,
                       double mean[2], double cov[3]) {
  double yy[7][2];
  for (int i = 0; i < 7; ++i) {
    yy[i][0] = y[i][0];
    yy[i][1] = y[i][1];
    if (wrap_a) {
      double d = y[i][0] - y[0][0];
      while (d > OR_PI) d -= OR_TWO_PI;
      while (d <= -OR_PI) d += OR_TWO_PI;
      yy[i][0] = y[0][0] + d;
    }
  }
  mean[0] = mean[1] = 0.0;
  for (int i = 0; i < 7; ++i) {
    mean[0] += wm[i] * yy[i][0];
    mean[1] += wm[i] * yy[i][1];
  }
  cov[0] = cov[1] = cov[2] = 0.0;
  for (int i = 0; i < 7; ++i) {
    double da = yy[i][0] - mean[0], db = yy[i][1] - mean[1];
    cov[0] += wc[i] * da * da;
    cov[1] += wc[i] * da * db;
    cov[2] += wc[i] * db * db;
  }
}

/* UT through an affine "sensor" y = A x + b (pin: exact for affine maps). */
int or_ut_affine(const double mu[3], const double q[4], const double s[3], const double ut[3],
                 const double A[6], const double b[2], double mean[2], double cov[3]) {
  double pts[21], wm[7], wc[7], y[7][2];
  if (or_sigma_points(mu, q, s, ut, pts, wm, wc)) return -1;
  for (int i = 0; i < 7; ++i)
    for (int r = 0; r < 2; ++r)
      y[i][r] = A[r * 3 + 0] * pts[i * 3 + 0] + A[r * 3 + 1] * pts[i * 3 + 1] + A[r * 3 + 2] * pts[i * 3 + 2] + b[r];
  ut_moments(y, wm, wc, 0, mean, cov);
  return 0;
}

/* ------------------------------------------------------------------------------------
 * O3  Sensor pose at normalised firing time s in [0,1] ("incorporating camera
 *     motion into the projection function"; A4): t(s) = t0 + s (t1 - t0),
 *     R(s) = R0 Exp(s Log(R0^T R1)).  pose = (qw, qx, qy, qz, tx, ty, tz), sensor->world.
 * ---------------------------------------------------------------------------------- */
static void mat_mul(const double A[9], const double B[9], double C[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
}

static void so3_log(const double Rr[9], double w[3]) {
  double v[3] = {0.5 * (Rr[7] - Rr[5]), 0.5 * (Rr[2] - Rr[6]), 0.5 * (Rr[3] - Rr[1])};
  double sn = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  double c = 0.5 * (Rr[0] + Rr[4] + Rr[8] - 1.0);
  double th = atan2(sn, c);
  if (sn > 1e-300) {
    for (int i = 0; i < 3; ++i) w[i] = th * v[i] / sn;
  } else if (c > 0.0) {
    w[0] = w[1] = w[2] = 0.0;
  } else { /* rotation by pi: axis from (R + I)/2 */
    int k = 0;
    for (int i = 1; i < 3; ++i)
      if (Rr[i * 4] > Rr[k * 4]) k = i;
    double a[3];
    for (int i = 0; i < 3; ++i) a[i] = 0.5 * (Rr[i * 3 + k] + (i == k ? 1.0 : 0.0));
    double an = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    for (int i = 0; i < 3; ++i) w[i] = OR_PI * a[i] / an;
  }
}

static void so3_exp(const double w[3], double E[9]) {
  double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  for (int i = 0; i < 9; ++i) E[i] = (i % 4 == 0) ? 1.0 : 0.0;
  if (th == 0.0) return;
  double k[3] = {w[0] / th, w[1] / th, w[2] / th};
  double K[9] = {0, -k[2], k[1], k[2], 0, -k[0], -k[1], k[0], 0};
  double K2[9];
  mat_mul(K, K, K2);
  double sn = sin(th), cs = 1.0 - cos(th);
  for (int i = 0; i < 9; ++i) E[i] += sn * K[i] + cs * K2[i];
}

void or_pose_at(const double pose0[7], const double pose1[7], double s, double R[9], double t[3]) {
  double R0[9], R1[9], R0t[9], Rr[9], w[3], E[9];
  int same = 1;
  for (int i = 0; i < 7; ++i) same &= (pose0[i] == pose1[i]);
  or_quat_to_rot(pose0, R0);
  for (int c = 0; c < 3; ++c) t[c] = pose0[4 + c] + s * (pose1[4 + c] - pose0[4 + c]);
  if (same) {
    memcpy(R, R0, sizeof(double) * 9);
    return;
  }
  or_quat_to_rot(pose1, R1);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R0t[i * 3 + j] = R0[j * 3 + i];
  mat_mul(R0t, R1, Rr);
  so3_log(Rr, w);
  for (int c = 0; c < 3; ++c) w[c] *= s;
  so3_exp(w, E);
  mat_mul(R0, E, R);
}

/* world -> sensor frame: p = R^T (x - t) */
static void to_sensor(const double R[9], const double t[3], const double x[3], double p[3]) {
  double d[3] = {x[0] - t[0], x[1] - t[1], x[2] - t[2]};
  for (int i = 0; i < 3; ++i) p[i] = R[0 * 3 + i] * d[0] + R[1 * 3 + i] * d[1] + R[2 * 3 + i] * d[2];
}

/* ------------------------------------------------------------------------------------
 * O4  LiDAR point projection, Eq. 3: phi = atan2(y, x), omega = asin(z/r),
 *     r = |p|, in the sensor frame at the point's own firing time.  The
 *     firing time depends on the azimuth: K fixed-point iterations from s = 0 (A3, A5):
 *     s <- wrap_[0,2pi)(dir (phi - phi_start)) / 2pi.   out = (phi, omega, r, s).
 * ---------------------------------------------------------------------------------- */
/* seam_dist (optional): smallest angular distance of a firing-time update's azimuth to
 * the start of the sweep, where s jumps between 0 and 1 (an A23 threshold event) */
static void lidar_point_seam(const double x[3], const or_lidar* L, const double pose0[7], const double pose1[7],
                             int K, double out[4], double* seam_dist);

void or_lidar_point(const double x[3], const or_lidar* L, const double pose0[7], const double pose1[7],
                    int K, double out[4]) {
  lidar_point_seam(x, L, pose0, pose1, K, out, NULL);
}

static void lidar_point_seam(const double x[3], const or_lidar* L, const double pose0[7], const double pose1[7],
                             int K, double out[4], double* seam_dist) {
  double s = 0.0, R[9], t[3], p[3], r = 0, phi = 0, om = 0;
  if (seam_dist) *seam_dist = INFINITY;
  for (int i = 0; i <= K; ++i) {
    or_pose_at(pose0, pose1, s, R, t);
    to_sensor(R, t, x, p);
    r = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    phi = atan2(p[1], p[0]);
    double z = r > 0.0 ? p[2] / r : 0.0;
    if (z > 1.0) z = 1.0;
    if (z < -1.0) z = -1.0;
    om = asin(z);
    if (i < K) {
      double a = (double)L->dir * (phi - L->az_start);
      a = a - OR_TWO_PI * floor(a / OR_TWO_PI);
      s = a / OR_TWO_PI;
      if (seam_dist) {
        const double dseam = a < OR_TWO_PI - a ? a : OR_TWO_PI - a;
        if (dseam < *seam_dist) *seam_dist = dseam;
      }
    }
  }
  out[0] = phi;
  out[1] = om;
  out[2] = r;
  out[3] = s;
}

/* ------------------------------------------------------------------------------------
 * O6  Camera point projection (P:26, P:112, P:129 -- "arbitrary camera models";
 *     A22).  Camera frame = OpenCV (x right, y down, z forward).
 *     KB fisheye: theta = atan2(rho, z), theta_d = theta (1 + k1 th^2 + k2 th^4 + k3 th^6
 *     + k4 th^8), (u, v) = (fx theta_d x/rho + cx, fy theta_d y/rho + cy).
 *     Pinhole radtan: OpenCV k1 k2 p1 p2 k3.
 *     Rolling shutter: s <- clamp(v/H, 0, 1), K iterations from s = 0.
 * ---------------------------------------------------------------------------------- */
/* returns 1 valid, 0 computed but invalid (outside near / theta_max), -1 not computable */
static int cam_project_frame(const or_camera* C, const double p[3], double* u, double* v, int* edge) {
  double dist = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
  if (C->model == 1) {
    double rho = sqrt(p[0] * p[0] + p[1] * p[1]);
    double th = atan2(rho, p[2]);
    if (fabs(dist - C->near_m) < 1e-4 || fabs(th - C->max_theta) < 1e-5) *edge = 1;
    if (!(dist > 0.0)) return -1;
    double t2 = th * th;
    double thd = th * (1.0 + C->k[0] * t2 + C->k[1] * t2 * t2 + C->k[2] * t2 * t2 * t2 + C->k[3] * t2 * t2 * t2 * t2);
    double sc = rho > 0.0 ? thd / rho : 0.0;
    *u = C->fx * sc * p[0] + C->cx;
    *v = C->fy * sc * p[1] + C->cy;
    return (dist >= C->near_m && th <= C->max_theta) ? 1 : 0;
  } else {
    double th = atan2(sqrt(p[0] * p[0] + p[1] * p[1]), p[2]);
    if (fabs(p[2] - C->near_m) < 1e-4 || fabs(th - C->max_theta) < 1e-5) *edge = 1;
    if (!(p[2] > 0.0)) return -1;
    double xp = p[0] / p[2], yp = p[1] / p[2];
    double r2 = xp * xp + yp * yp;
    double k1 = C->k[0], k2 = C->k[1], p1 = C->k[2], p2 = C->k[3], k3 = C->k[4];
    double radial = 1.0 + k1 * r2 + k2 * r2 * r2 + k3 * r2 * r2 * r2;
    double xd = xp * radial + 2.0 * p1 * xp * yp + p2 * (r2 + 2.0 * xp * xp);
    double yd = yp * radial + p1 * (r2 + 2.0 * yp * yp) + 2.0 * p2 * xp * yp;
    *u = C->fx * xd + C->cx;
    *v = C->fy * yd + C->cy;
    return (p[2] >= C->near_m && th <= C->max_theta) ? 1 : 0;
  }
}

/* out = (u, v, |p|, s).  Returns 1 valid, 0 invalid but computed, -1 not computable.
 * A point is valid only if every fixed-point iteration projects validly. */
static int camera_point_edge(const double x[3], const or_camera* C, const double pose0[7], const double pose1[7],
                             int K, double out[4], int* edge) {
  double s = 0.0, R[9], t[3], p[3] = {0, 0, 0}, u = 0, v = 0;
  int valid = 1;
  for (int i = 0; i <= K; ++i) {
    or_pose_at(pose0, pose1, s, R, t);
    to_sensor(R, t, x, p);
    int st = cam_project_frame(C, p, &u, &v, edge);
    if (st < 0) return -1;
    if (st == 0) valid = 0;
    if (i < K) {
      if (C->rolling) {
        s = v / (double)C->height;
        if (s < 0.0) s = 0.0;
        if (s > 1.0) s = 1.0;
      } else {
        s = 0.0;
      }
    }
  }
  out[0] = u;
  out[1] = v;
  out[2] = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
  out[3] = s;
  return valid;
}

int or_camera_point(const double x[3], const or_camera* C, const double pose0[7], const double pose1[7], int K,
                    double out[4]) {
  int edge = 0;
  return camera_point_edge(x, C, pose0, pose1, K, out, &edge) == 1;
}

/* Inverse lens model for pixel rays (A22): KB by Newton on theta_d(theta) = r_d, radtan
 * by fixed-point undistortion; iterated to convergence in double. */
int or_camera_unproject(const or_camera* C, double u, double v, double dir[3]) {
  double mx = (u - C->cx) / C->fx, my = (v - C->cy) / C->fy;
  if (C->model == 1) {
    double rd = sqrt(mx * mx + my * my);
    if (rd == 0.0) {
      dir[0] = 0.0; dir[1] = 0.0; dir[2] = 1.0;
      return 1;
    }
    double th = rd;
    int ok = 0;
    for (int it = 0; it < 100; ++it) {
      double t2 = th * th;
      double f = th * (1.0 + C->k[0] * t2 + C->k[1] * t2 * t2 + C->k[2] * t2 * t2 * t2 + C->k[3] * t2 * t2 * t2 * t2) - rd;
      double fp = 1.0 + 3.0 * C->k[0] * t2 + 5.0 * C->k[1] * t2 * t2 + 7.0 * C->k[2] * t2 * t2 * t2 +
                  9.0 * C->k[3] * t2 * t2 * t2 * t2;
      double step = f / fp;
      th -= step;
      if (fabs(step) < 1e-15 * (1.0 + fabs(th))) {
        ok = 1;
        break;
      }
    }
    if (!ok || !(th >= 0.0) || th > C->max_theta) return 0;
    double sn = sin(th);
    dir[0] = sn * mx / rd;
    dir[1] = sn * my / rd;
    dir[2] = cos(th);
    return 1;
  } else {
    double x = mx, y = my;
    double k1 = C->k[0], k2 = C->k[1], p1 = C->k[2], p2 = C->k[3], k3 = C->k[4];
    for (int it = 0; it < 200; ++it) {
      double r2 = x * x + y * y;
      double radial = 1.0 + k1 * r2 + k2 * r2 * r2 + k3 * r2 * r2 * r2;
      double dx = 2.0 * p1 * x * y + p2 * (r2 + 2.0 * x * x);
      double dy = p1 * (r2 + 2.0 * y * y) + 2.0 * p2 * x * y;
      double nx = (mx - dx) / radial, ny = (my - dy) / radial;
      double ch = fabs(nx - x) + fabs(ny - y);
      x = nx;
      y = ny;
      if (ch < 1e-16) break;
    }
    double n = sqrt(x * x + y * y + 1.0);
    dir[0] = x / n;
    dir[1] = y / n;
    dir[2] = 1.0 / n;
    return atan(sqrt(x * x + y * y)) <= C->max_theta;
  }
}

/* ------------------------------------------------------------------------------------
 * O9  Degree-3 real spherical harmonics, 48 coefficients [16][3] (§3.1), with the
 *     3DGS normalisation constants (Y00 = 0.28209479177387814).
 * ---------------------------------------------------------------------------------- */
void or_sh_eval(const double* sh, int degree, const double dir[3], double out[3]) {
  const double C0 = 0.28209479177387814;
  const double C1 = 0.4886025119029199;
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                        0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                        -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
  double x = dir[0], y = dir[1], z = dir[2];
  double basis[16];
  int nb = (degree + 1) * (degree + 1);
  basis[0] = C0;
  if (degree >= 1) {
    basis[1] = -C1 * y;
    basis[2] = C1 * z;
    basis[3] = -C1 * x;
  }
  if (degree >= 2) {
    double xx = x * x, yy = y * y, zz = z * z;
    basis[4] = C2[0] * x * y;
    basis[5] = C2[1] * y * z;
    basis[6] = C2[2] * (2.0 * zz - xx - yy);
    basis[7] = C2[3] * x * z;
    basis[8] = C2[4] * (xx - yy);
  }
  if (degree >= 3) {
    double xx = x * x, yy = y * y, zz = z * z;
    basis[9] = C3[0] * y * (3.0 * xx - yy);
    basis[10] = C3[1] * x * y * z;
    basis[11] = C3[2] * y * (4.0 * zz - xx - yy);
    basis[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    basis[13] = C3[4] * x * (4.0 * zz - xx - yy);
    basis[14] = C3[5] * z * (xx - yy);
    basis[15] = C3[6] * x * (xx - 3.0 * yy);
  }
  for (int c = 0; c < 3; ++c) {
    double acc = 0.0;
    for (int k = 0; k < nb; ++k) acc += basis[k] * sh[k * 3 + c];
    out[c] = acc;
  }
}

/* ------------------------------------------------------------------------------------
 * O12 response (3DGRT): tau_max = argmax_tau rho(o + tau d).  In canonical space
 *     o' = M (o - mu), d' = M d with M = diag(1/s) R^T:
 *     tau = -(o'.d')/|d'|^2,  delta^2 = |(d'/|d'|) x o'|^2 = min_tau |o' + tau d'|^2.
 * ---------------------------------------------------------------------------------- */
void or_response(const double mu[3], const double Mr[9], const double o[3], const double d[3], double out[2]) {
  double pd[3] = {o[0] - mu[0], o[1] - mu[1], o[2] - mu[2]};
  double op[3], dp[3];
  for (int k = 0; k < 3; ++k) {
    op[k] = Mr[k * 3] * pd[0] + Mr[k * 3 + 1] * pd[1] + Mr[k * 3 + 2] * pd[2];
    dp[k] = Mr[k * 3] * d[0] + Mr[k * 3 + 1] * d[1] + Mr[k * 3 + 2] * d[2];
  }
  double dd = dp[0] * dp[0] + dp[1] * dp[1] + dp[2] * dp[2];
  double tau = -(op[0] * dp[0] + op[1] * dp[1] + op[2] * dp[2]) / dd;
  double dn = sqrt(dd);
  double u[3] = {dp[0] / dn, dp[1] / dn, dp[2] / dn};
  double cx = u[1] * op[2] - u[2] * op[1];
  double cy = u[2] * op[0] - u[0] * op[2];
  double cz = u[0] * op[1] - u[1] * op[0];
  out[0] = tau;
  out[1] = cx * cx + cy * cy + cz * cz;
}

/* LiDAR feature decode: gamma = zeta_0; beta = softmax(zeta_1 (hit), zeta_2 (drop)),
 * reported as (gamma, beta_drop) with the stable form of 1/(1 + exp(z1 - z2)) (A18). */
void or_decode_lidar(const double zeta[3], double out[2]) {
  double z = zeta[1] - zeta[2];
  double bd;
  if (z >= 0.0) {
    double e = exp(-z);
    bd = e / (1.0 + e);
  } else {
    bd = 1.0 / (1.0 + exp(z));
  }
  out[0] = zeta[0];
  out[1] = bd;
}

/* ------------------------------------------------------------------------------------
 * O7  Automated elevation tiling, Proc. ElevationTiling with the
 *     A8 corrections: (i) scan all r bins, (ii) partition = bins <= crossing bin, boundary
 *     at the float32 gap midpoint, (iii) +Phi_min, (iv) N_theta = ceil(H_max / M),
 *     (v) per-ray histogram (each beam weighted by A), (vi) integer crossing test
 *     c_i N_phi >= b total, (vii) one crossing per bin; empty partitions dropped.
 *     Dense culling grid: 1600 azimuth cells x 8 rows per elevation tile (A10),
 *     ray mask and zero-padded summed-area table.
 * ---------------------------------------------------------------------------------- */
int32_t or_elev_tile(const or_tiling* t, float w) {
  int32_t e = 0;
  for (int k = 1; k < t->n_phi; ++k)
    if (t->bounds[k] <= w) e++;
  return e;
}

static int32_t float_index(float u, int32_t n) {
  if (!(u >= 0.0f)) return 0;
  if (u >= (float)n) return n - 1;
  int32_t c = (int32_t)floorf(u);
  return c > n - 1 ? n - 1 : c;
}

int32_t or_az_col(const or_tiling* t, float phi) {
  volatile float a = phi + t->pi_f; /* correctly rounded float32 add, then multiply */
  float u = a * t->az_tile_scale;
  return float_index(u, t->n_theta);
}

int32_t or_dense_cell(const or_tiling* t, float phi) {
  volatile float a = phi + t->pi_f;
  float u = a * t->az_cell_scale;
  return float_index(u, t->cull_az_cells);
}

int32_t or_dense_row(const or_tiling* t, float w) {
  int32_t e = or_elev_tile(t, w);
  volatile float a = w - t->bounds[e];
  float u = a * t->cull_row_scale[e];
  return e * t->cull_rows_per_tile + float_index(u, t->cull_rows_per_tile);
}

void or_free_tiling(or_tiling* t) {
  free(t->bounds); free(t->cull_row_scale); free(t->ray_az); free(t->ray_el); free(t->ray_s);
  free(t->ray_tile); free(t->tile_ray_offsets); free(t->tile_rays); free(t->sat);
  free(t->ray_cell_row); free(t->ray_cell_col);
  memset(t, 0, sizeof(*t));
}

int or_build_tiling(const or_lidar* L, int32_t n_phi, int32_t M, int32_t r, int32_t cull_az, int32_t cull_rows,
                    or_tiling* out) {
  memset(out, 0, sizeof(*out));
  int32_t B = L->n_beams, A = L->n_az;
  if (B < 1 || A < 1 || n_phi < 1 || M < 1 || r < 1 || cull_az < 1 || cull_rows < 1) return -1;
  if (n_phi > r) return -1; /* "tile count exceeds histogram resolution" */
  double emin = L->elev[0], emax = L->elev[0];
  for (int b = 0; b < B; ++b) {
    if (!(fabs((double)L->elev[b]) < OR_PI / 2)) return -1;
    if (L->elev[b] < emin) emin = L->elev[b];
    if (L->elev[b] > emax) emax = L->elev[b];
  }
  int32_t* part = (int32_t*)calloc(B, sizeof(int32_t)); /* partition of each beam */
  int32_t nparts = 1;
  if (emax > emin) {
    /* lines 1-4: histogram of per-ray elevations (each beam weighted by A), cumulative sum */
    int64_t* H = (int64_t*)calloc(r, sizeof(int64_t));
    int32_t* bin_of = (int32_t*)calloc(B, sizeof(int32_t));
    for (int b = 0; b < B; ++b) {
      int32_t bin = (int32_t)floor(((double)L->elev[b] - emin) / (emax - emin) * (double)r);
      if (bin > r - 1) bin = r - 1;
      bin_of[b] = bin;
      H[bin] += A;
    }
    int64_t total = (int64_t)B * A, c = 0, bidx = 1;
    /* lines 5-11: one crossing per bin where C(i) >= b (integer-exact form) */
    int32_t* cross_of_bin = (int32_t*)calloc(r, sizeof(int32_t)); /* partition index of each bin */
    int32_t ncross = 0;
    for (int i = 0; i < r; ++i) {
      c += H[i];
      cross_of_bin[i] = ncross; /* bins up to and including a crossing bin belong to it */
      if (c * (int64_t)n_phi >= bidx * total) {
        ncross++;
        bidx++;
      }
    }
    /* drop empty partitions: renumber by occupied partitions in order */
    int32_t* used = (int32_t*)calloc(r + 1, sizeof(int32_t));
    for (int b = 0; b < B; ++b) used[cross_of_bin[bin_of[b]]] = 1;
    int32_t* renum = (int32_t*)calloc(r + 1, sizeof(int32_t));
    nparts = 0;
    for (int k = 0; k <= r; ++k) {
      renum[k] = nparts;
      if (used[k]) nparts++;
    }
    for (int b = 0; b < B; ++b) part[b] = renum[cross_of_bin[bin_of[b]]];
    free(H); free(bin_of); free(cross_of_bin); free(used); free(renum);
  }
  out->n_phi = nparts;
  out->bounds = (float*)malloc(sizeof(float) * (nparts + 1));
  out->bounds[0] = (float)emin;
  out->bounds[nparts] = (float)emax;
  for (int k = 0; k + 1 < nparts; ++k) {
    double a = -INFINITY, cc = INFINITY; /* largest beam of k, smallest beam of k+1 */
    for (int b = 0; b < B; ++b) {
      if (part[b] == k && L->elev[b] > a) a = L->elev[b];
      if (part[b] == k + 1 && L->elev[b] < cc) cc = L->elev[b];
    }
    float m = (float)((a + cc) / 2.0);
    if (m <= (float)a) m = (float)cc;
    out->bounds[k + 1] = m;
  }
  out->pi_f = (float)OR_PI;
  out->two_pi_f = (float)OR_TWO_PI;
  out->cull_rows_per_tile = cull_rows;
  out->cull_az_cells = cull_az;
  out->cull_row_scale = (float*)malloc(sizeof(float) * nparts);
  for (int k = 0; k < nparts; ++k) {
    double wdt = (double)out->bounds[k + 1] - (double)out->bounds[k];
    out->cull_row_scale[k] = wdt > 0.0 ? (float)((double)cull_rows / wdt) : 0.0f;
  }
  /* every beam's float32 tile must equal its integer partition */
  for (int b = 0; b < B; ++b) {
    if (or_elev_tile(out, L->elev[b]) != part[b]) {
      free(part);
      or_free_tiling(out);
      return -2;
    }
  }
  /* lines 12-13: re-histogram over T, H_max, N_theta = ceil(H_max / M), clamped to [1, A] */
  int64_t nbmax = 0;
  for (int k = 0; k < nparts; ++k) {
    int64_t cnt = 0;
    for (int b = 0; b < B; ++b) cnt += (part[b] == k);
    if (cnt > nbmax) nbmax = cnt;
  }
  int64_t Hmax = nbmax * A;
  int64_t nth = (Hmax + M - 1) / M;
  if (nth < 1) nth = 1;
  if (nth > A) nth = A;
  out->n_theta = (int32_t)nth;
  out->n_tiles = nparts * out->n_theta;
  out->az_tile_scale = (float)((double)out->n_theta / OR_TWO_PI);
  out->az_cell_scale = (float)((double)cull_az / OR_TWO_PI);
  free(part);

  /* ray table: ray (b, j) fires at column j: phi_j = phi_start + dir (j + 0.5) 2pi/A,
   * s_j = (j + 0.5)/A (A5); omega_b as given. */
  int32_t R = B * A;
  out->n_rays = R;
  out->n_beams = B;
  out->n_az = A;
  out->ray_az = (float*)malloc(sizeof(float) * R);
  out->ray_el = (float*)malloc(sizeof(float) * R);
  out->ray_s = (float*)malloc(sizeof(float) * R);
  out->ray_tile = (int32_t*)malloc(sizeof(int32_t) * R);
  out->ray_cell_row = (int32_t*)malloc(sizeof(int32_t) * R);
  out->ray_cell_col = (int32_t*)malloc(sizeof(int32_t) * R);
  for (int b = 0; b < B; ++b) {
    for (int j = 0; j < A; ++j) {
      int32_t id = b * A + j;
      double phi = L->az_start + (double)L->dir * (((double)j + 0.5) * (OR_TWO_PI / (double)A));
      if (phi >= OR_PI) phi -= OR_TWO_PI;
      else if (phi < -OR_PI) phi += OR_TWO_PI;
      out->ray_az[id] = (float)phi;
      out->ray_el[id] = L->elev[b];
      out->ray_s[id] = (float)(((double)j + 0.5) / (double)A);
      out->ray_tile[id] = or_elev_tile(out, L->elev[b]) * out->n_theta + or_az_col(out, out->ray_az[id]);
      out->ray_cell_row[id] = or_dense_row(out, L->elev[b]);
      out->ray_cell_col[id] = or_dense_cell(out, out->ray_az[id]);
    }
  }
  /* tile -> rays CSR, rays in increasing id */
  out->tile_ray_offsets = (int32_t*)calloc(out->n_tiles + 1, sizeof(int32_t));
  out->tile_rays = (int32_t*)malloc(sizeof(int32_t) * R);
  for (int i = 0; i < R; ++i) out->tile_ray_offsets[out->ray_tile[i] + 1]++;
  out->max_rays_in_tile = 0;
  for (int t = 0; t < out->n_tiles; ++t) {
    if (out->tile_ray_offsets[t + 1] > out->max_rays_in_tile) out->max_rays_in_tile = out->tile_ray_offsets[t + 1];
    out->tile_ray_offsets[t + 1] += out->tile_ray_offsets[t];
  }
  int32_t* fill = (int32_t*)calloc(out->n_tiles, sizeof(int32_t));
  for (int i = 0; i < R; ++i) {
    int32_t t = out->ray_tile[i];
    out->tile_rays[out->tile_ray_offsets[t] + fill[t]++] = i;
  }
  free(fill);
  /* dense ray mask and summed-area table: sat[i][j] = #occupied cells in [0,i) x [0,j) */
  int32_t rows = cull_rows * nparts, cols = cull_az;
  out->sat_rows = rows + 1;
  out->sat_cols = cols + 1;
  uint8_t* mask = (uint8_t*)calloc((size_t)rows * cols, 1);
  for (int i = 0; i < R; ++i) mask[(size_t)out->ray_cell_row[i] * cols + out->ray_cell_col[i]] = 1;
  out->sat = (int32_t*)calloc((size_t)out->sat_rows * out->sat_cols, sizeof(int32_t));
  for (int i = 1; i <= rows; ++i)
    for (int j = 1; j <= cols; ++j)
      out->sat[(size_t)i * out->sat_cols + j] = mask[(size_t)(i - 1) * cols + (j - 1)] +
                                                out->sat[(size_t)(i - 1) * out->sat_cols + j] +
                                                out->sat[(size_t)i * out->sat_cols + (j - 1)] -
                                                out->sat[(size_t)(i - 1) * out->sat_cols + (j - 1)];
  free(mask);
  return 0;
}

/* Proc. RayOccupancyCount: n = A - B - C + D over the inclusive dense
 * rectangle [r_lo, r_hi] x [c_lo, c_hi] with the +1 upper offsets of P:534-537. */
int or_sat_query(const int32_t* sat, int32_t sc, int32_t r_lo, int32_t r_hi, int32_t c_lo, int32_t c_hi) {
  int32_t A = sat[(size_t)(r_hi + 1) * sc + (c_hi + 1)];
  int32_t B = sat[(size_t)r_lo * sc + (c_hi + 1)];
  int32_t C = sat[(size_t)(r_hi + 1) * sc + c_lo];
  int32_t D = sat[(size_t)r_lo * sc + c_lo];
  return A - B - C + D;
}

/* ------------------------------------------------------------------------------------
 * O5 + O9 + O10: per-Gaussian projection.
 * ---------------------------------------------------------------------------------- */
static float round_down_f(double x) {
  float f = (float)x;
  if ((double)f > x) f = nextafterf(f, -INFINITY);
  return f;
}
static float round_up_f(double x) {
  float f = (float)x;
  if ((double)f < x) f = nextafterf(f, INFINITY);
  return f;
}

/* O10 depth key: float32 distance from o_mid = t0 + 0.5 (t1 - t0), fixed op order, no FMA. */
static float depth_key(const float mu[3], const double pose0[7], const double pose1[7]) {
  volatile float d[3];
  for (int c = 0; c < 3; ++c) {
    volatile float t0 = (float)pose0[4 + c], t1 = (float)pose1[4 + c];
    volatile float h = t1 - t0;
    volatile float hm = 0.5f * h;
    volatile float om = t0 + hm;
    d[c] = mu[c] - om;
  }
  volatile float xx = d[0] * d[0], yy = d[1] * d[1], zz = d[2] * d[2];
  volatile float s1 = xx + yy;
  volatile float s2 = s1 + zz;
  return sqrtf(s2);
}

static void write_invalid(or_proj_out* out, int64_t g) {
  out->valid[g] = 0;
  for (int c = 0; c < 4; ++c) out->box[g * 4 + c] = NAN;
  for (int c = 0; c < 2; ++c) out->mean2d[g * 2 + c] = NAN;
  for (int c = 0; c < 3; ++c) out->cov2d[g * 3 + c] = NAN;
}

typedef int (*point_fn)(const double x[3], const void* sensor, const double p0[7], const double p1[7], int K,
                        double out[4], int* edge);

static int lidar_point_fn(const double x[3], const void* sensor, const double p0[7], const double p1[7], int K,
                          double out[4], int* edge) {
  const or_lidar* L = (const or_lidar*)sensor;
  double seam = INFINITY;
  const int moving = memcmp(p0, p1, 7 * sizeof(double)) != 0;
  lidar_point_seam(x, L, p0, p1, K, out, &seam);
  if (fabs(out[2] - L->r_min) < 1e-4) *edge = 1;
  if (moving && seam < 1e-5) *edge = 1; /* firing time s ~ 0 vs ~ 1: float32 may decide otherwise */
  return out[2] >= L->r_min;
}

static int camera_point_fn(const double x[3], const void* sensor, const double p0[7], const double p1[7], int K,
                           double out[4], int* edge) {
  return camera_point_edge(x, (const or_camera*)sensor, p0, p1, K, out, edge);
}

static int project_common(const or_gaussians* G, const void* sensor, int wrap_a, point_fn fn, const double pose0[7],
                          const double pose1[7], int K, const double ut[3], double ks, or_proj_out* out) {
  double spread, wm[7], wc[7];
  if (or_ut_weights(ut, &spread, wm, wc)) return -1;
  int64_t n = G->n;
  int ncoef = (G->sh_degree + 1) * (G->sh_degree + 1);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t g = 0; g < n; ++g) {
    double mu[3], q[4], s[3], R[9];
    float muf[3];
    for (int c = 0; c < 3; ++c) {
      muf[c] = G->means[g * 3 + c];
      mu[c] = muf[c];
      s[c] = G->scales[g * 3 + c];
    }
    for (int c = 0; c < 4; ++c) q[c] = G->quats[g * 4 + c];
    out->key[g] = depth_key(muf, pose0, pose1);
    out->ambiguous[g] = 0;
    out->minrange[g] = NAN;
    double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    int ok = qn > 0.0 && isfinite(qn);
    for (int c = 0; c < 3; ++c) ok &= (s[c] > 0.0 && isfinite(s[c]) && isfinite(mu[c]));
    if (!ok) {
      write_invalid(out, g);
      continue;
    }
    or_quat_to_rot(q, R);
    double pts[21], w1[7], w2[7];
    /* beam divergence (LiDAR, App. C): Sigma_hat, its Cholesky factor as the sigma-point
     * square root and M_hat = L_hat^-1 as the canonical transform (Sigma_hat^-1 = M^T M) */
    const double theta = wrap_a ? ((const or_lidar*)sensor)->beam_div : 0.0;
    double Mdiv[9];
    if (theta > 0.0) {
      double o4[4], Rs0[9], ts0[3], Sig[9], Sh[9], Lh[9];
      int e_unused = 0;
      fn(mu, sensor, pose0, pose1, K, o4, &e_unused); /* firing time of the mean */
      or_pose_at(pose0, pose1, o4[3], Rs0, ts0);
      or_covariance(q, s, Sig);
      or_divergence_cov(Sig, mu, ts0, theta, Sh);
      if (or_cholesky3(Sh, Lh)) {
        write_invalid(out, g);
        continue;
      }
      or_sigma_points_sqrt(mu, Lh, ut, pts, w1, w2);
      or_lower_inverse3(Lh, Mdiv);
    } else {
      or_sigma_points(mu, q, s, ut, pts, w1, w2);
    }
    double y[7][2], s0 = 0.0, minr = INFINITY;
    int valid = 1, edge = 0, computable = 1;
    for (int i = 0; i < 7; ++i) {
      double o4[4] = {0, 0, 0, 0};
      int v = fn(&pts[i * 3], sensor, pose0, pose1, K, o4, &edge);
      if (v < 0) computable = 0;
      valid &= (v == 1);
      y[i][0] = o4[0];
      y[i][1] = o4[1];
      if (o4[2] < minr) minr = o4[2];
      if (i == 0) s0 = o4[3];
    }
    out->minrange[g] = minr;
    double mean[2], cov[3];
    ut_moments(y, wm, wc, wrap_a, mean, cov);
    double det = cov[0] * cov[2] - cov[1] * cov[1];
    int boxok = computable && isfinite(mean[0]) && isfinite(mean[1]) && cov[0] > 0.0 && cov[2] > 0.0 && det > 0.0 &&
                isfinite(det);
    if (boxok && det < 1e-5 * cov[0] * cov[2]) edge = 1;
    if (!boxok) {
      write_invalid(out, g);
      out->ambiguous[g] = 0;
      continue;
    }
    if (wrap_a) { /* azimuth mean normalised into [-pi, pi) */
      if (mean[0] >= OR_PI) mean[0] -= OR_TWO_PI;
      else if (mean[0] < -OR_PI) mean[0] += OR_TWO_PI;
    }
    out->valid[g] = valid;
    out->ambiguous[g] = edge;
    out->mean2d[g * 2] = mean[0];
    out->mean2d[g * 2 + 1] = mean[1];
    for (int c = 0; c < 3; ++c) out->cov2d[g * 3 + c] = cov[c];
    double ha = ks * sqrt(cov[0]), hb = ks * sqrt(cov[2]);
    out->box[g * 4 + 0] = round_down_f(mean[0] - ha);
    out->box[g * 4 + 1] = round_up_f(mean[0] + ha);
    out->box[g * 4 + 2] = round_down_f(mean[1] - hb);
    out->box[g * 4 + 3] = round_up_f(mean[1] + hb);
    if (theta > 0.0) {
      for (int i = 0; i < 9; ++i) out->Mrows[g * 9 + i] = Mdiv[i];
    } else {
      for (int k = 0; k < 3; ++k) /* M = diag(1/s) R^T : row k = (column k of R)/s_k */
        for (int i = 0; i < 3; ++i) out->Mrows[g * 9 + k * 3 + i] = R[i * 3 + k] / s[k];
    }
    /* O9: SH features, direction from the sensor position at sigma point 0's firing time (A17) */
    double Rs[9], ts[3], v[3], shd[48];
    or_pose_at(pose0, pose1, s0, Rs, ts);
    for (int c = 0; c < 3; ++c) v[c] = mu[c] - ts[c];
    if (out->viewdir) /* the view vector mu - o(s0), unnormalised (backward, A31) */
      for (int c = 0; c < 3; ++c) out->viewdir[g * 3 + c] = v[c];
    double vn = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int c = 0; c < 3; ++c) v[c] /= vn;
    for (int k = 0; k < ncoef * 3; ++k) shd[k] = G->sh[g * ncoef * 3 + k];
    or_sh_eval(shd, G->sh_degree, v, &out->feat[g * 3]);
  }
  return 0;
}

int or_project_lidar(const or_gaussians* G, const or_lidar* L, const double pose0[7], const double pose1[7], int K,
                     const double ut[3], double extent_sigma, or_proj_out* out) {
  return project_common(G, L, 1, lidar_point_fn, pose0, pose1, K, ut, extent_sigma, out);
}

int or_project_camera(const or_gaussians* G, const or_camera* C, const double pose0[7], const double pose1[7], int K,
                      const double ut[3], double extent_sigma, or_proj_out* out) {
  return project_common(G, C, 0, camera_point_fn, pose0, pose1, K, ut, extent_sigma, out);
}

/* ------------------------------------------------------------------------------------
 * O8  Culling (Proc. ProjectParticles) and render-tile rectangle.
 *     rect = (row_lo, row_hi, col_start, n_cols); the columns are the circular interval
 *     col_start, col_start+1, ... (mod N_theta).  Column/cell sets are built from the
 *     float32 box edges shifted by 2pi_f (never shifted rays), A12.
 * ---------------------------------------------------------------------------------- */
typedef int32_t (*idx_fn)(const or_tiling*, float);

/* Set of azimuth indices covered by [lo, hi] as a bitmap over n entries. */
static void az_set(const or_tiling* t, float lo, float hi, idx_fn f, int32_t n, uint8_t* set) {
  memset(set, 0, n);
  volatile float width = hi - lo;
  if (width >= t->two_pi_f) {
    memset(set, 1, n);
    return;
  }
  float a = lo > -t->pi_f ? lo : -t->pi_f;
  float b = hi < t->pi_f ? hi : t->pi_f;
  if (a <= b)
    for (int32_t i = f(t, a); i <= f(t, b); ++i) set[i] = 1;
  if (lo < -t->pi_f) {
    volatile float l2 = lo + t->two_pi_f;
    for (int32_t i = f(t, l2); i <= n - 1; ++i) set[i] = 1;
  }
  if (hi > t->pi_f) {
    volatile float h2 = hi - t->two_pi_f;
    for (int32_t i = 0; i <= f(t, h2); ++i) set[i] = 1;
  }
}

static int in_interval_a(float lo, float hi, float x, int wrap, float pi_f, float two_pi_f);

/* circular interval (start, length) of a bitmap that is one circular run (or full) */
static int set_to_interval(const uint8_t* set, int32_t n, int32_t* start, int32_t* len) {
  int32_t cnt = 0;
  for (int i = 0; i < n; ++i) cnt += set[i];
  *len = cnt;
  if (cnt == n || cnt == 0) {
    *start = 0;
    return 0;
  }
  for (int i = 0; i < n; ++i)
    if (set[i] && !set[(i + n - 1) % n]) {
      *start = i;
      for (int k = 0; k < cnt; ++k)
        if (!set[(i + k) % n]) return -1; /* not a single run */
      return 0;
    }
  return -1;
}

int or_cull_lidar(int64_t n, const int32_t* valid, const float* box, const or_tiling* t, int enable_cull,
                  int32_t* count, int32_t* rect) {
  int err = 0;
#pragma omp parallel
  {
    uint8_t* cset = (uint8_t*)malloc(t->cull_az_cells);
    uint8_t* tset = (uint8_t*)malloc(t->n_theta);
    uint8_t* rset = (uint8_t*)malloc(t->n_phi);
#pragma omp for schedule(dynamic, 4096)
    for (int64_t g = 0; g < n; ++g) {
      count[g] = 0;
      for (int c = 0; c < 4; ++c) rect[g * 4 + c] = 0;
      if (!valid[g]) continue;
      float lo_a = box[g * 4], hi_a = box[g * 4 + 1], lo_b = box[g * 4 + 2], hi_b = box[g * 4 + 3];
      if (enable_cull == 2) {
        /* Exact ray containment per render tile (reading A32): the tiles holding at least one
         * ray (b, j) with lo_b <= omega_b <= hi_b and phi_j inside the azimuth interval under
         * the compositing membership rule (O12, A12).  Plain scans over every beam and every
         * column: a tile (elevation tile of b, azimuth tile of j) holds such a ray iff one of
         * its beams and one of its columns pass. */
        memset(rset, 0, t->n_phi);
        memset(tset, 0, t->n_theta);
        int any_b = 0, any_c = 0;
        for (int32_t b = 0; b < t->n_beams; ++b) {
          float w = t->ray_el[(int64_t)b * t->n_az];
          if (lo_b <= w && w <= hi_b) {
            rset[or_elev_tile(t, w)] = 1;
            any_b = 1;
          }
        }
        for (int32_t j = 0; j < t->n_az && any_b; ++j) {
          float p = t->ray_az[j];
          if (in_interval_a(lo_a, hi_a, p, 1, t->pi_f, t->two_pi_f)) {
            tset[or_az_col(t, p)] = 1;
            any_c = 1;
          }
        }
        if (!any_b || !any_c) continue; /* culled: no ray inside the extent */
        int32_t e_lo = 0, e_hi = t->n_phi - 1;
        while (!rset[e_lo]) ++e_lo;
        while (!rset[e_hi]) --e_hi;
        for (int32_t e = e_lo; e <= e_hi; ++e)
          if (!rset[e]) err = 1; /* elevation tiles of a beam interval are contiguous */
        int32_t cs, cl;
        if (set_to_interval(tset, t->n_theta, &cs, &cl)) {
          err = 1;
          continue;
        }
        rect[g * 4 + 0] = e_lo;
        rect[g * 4 + 1] = e_hi;
        rect[g * 4 + 2] = cs;
        rect[g * 4 + 3] = cl;
        count[g] = (e_hi - e_lo + 1) * cl;
        continue;
      }
      float b0 = t->bounds[0], bl = t->bounds[t->n_phi];
      if (hi_b < b0 || lo_b > bl) continue; /* box misses the beam band */
      if (enable_cull) {                     /* Proc. RayOccupancyCount over the dense rectangle */
        int32_t r_lo = or_dense_row(t, lo_b), r_hi = or_dense_row(t, hi_b);
        az_set(t, lo_a, hi_a, or_dense_cell, t->cull_az_cells, cset);
        int32_t cs, cl;
        if (set_to_interval(cset, t->cull_az_cells, &cs, &cl)) {
          err = 1;
          continue;
        }
        int64_t occ = 0;
        int32_t c_end = cs + cl - 1;
        if (c_end < t->cull_az_cells) {
          occ = or_sat_query(t->sat, t->sat_cols, r_lo, r_hi, cs, c_end);
        } else { /* seam split */
          occ = or_sat_query(t->sat, t->sat_cols, r_lo, r_hi, cs, t->cull_az_cells - 1) +
                or_sat_query(t->sat, t->sat_cols, r_lo, r_hi, 0, c_end - t->cull_az_cells);
        }
        if (occ == 0) continue; /* culled: no ray inside the extent */
      }
      int32_t e_lo = or_elev_tile(t, lo_b), e_hi = or_elev_tile(t, hi_b);
      az_set(t, lo_a, hi_a, or_az_col, t->n_theta, tset);
      int32_t cs, cl;
      if (set_to_interval(tset, t->n_theta, &cs, &cl)) {
        err = 1;
        continue;
      }
      rect[g * 4 + 0] = e_lo;
      rect[g * 4 + 1] = e_hi;
      rect[g * 4 + 2] = cs;
      rect[g * 4 + 3] = cl;
      count[g] = (e_hi - e_lo + 1) * cl;
    }
    free(cset);
    free(tset);
    free(rset);
  }
  return err ? -1 : 0;
}

int or_cull_camera(int64_t n, const int32_t* valid, const float* box, const or_camera* C, int32_t* count,
                   int32_t* rect) {
  int32_t tp = C->tile_px;
  int32_t Wt = (C->width + tp - 1) / tp, Ht = (C->height + tp - 1) / tp;
  float inv = 1.0f / (float)tp;
  float wmax = (float)C->width - 0.5f, hmax = (float)C->height - 0.5f;
  for (int64_t g = 0; g < n; ++g) {
    count[g] = 0;
    for (int c = 0; c < 4; ++c) rect[g * 4 + c] = 0;
    if (!valid[g]) continue;
    float lo_u = box[g * 4], hi_u = box[g * 4 + 1], lo_v = box[g * 4 + 2], hi_v = box[g * 4 + 3];
    if (hi_u < 0.5f || lo_u > wmax || hi_v < 0.5f || lo_v > hmax) continue; /* no pixel centre inside */
    volatile float a0 = lo_u * inv, a1 = hi_u * inv, b0 = lo_v * inv, b1 = hi_v * inv;
    int32_t c_lo = float_index(a0, Wt), c_hi = float_index(a1, Wt);
    int32_t r_lo = float_index(b0, Ht), r_hi = float_index(b1, Ht);
    rect[g * 4 + 0] = r_lo;
    rect[g * 4 + 1] = r_hi;
    rect[g * 4 + 2] = c_lo;
    rect[g * 4 + 3] = c_hi - c_lo + 1;
    count[g] = (r_hi - r_lo + 1) * (c_hi - c_lo + 1);
  }
  return 0;
}

/* ------------------------------------------------------------------------------------
 * O11 Tile-Gaussian pairs "as in 3DGS": one pair per (tile, Gaussian) overlap,
 *     key = (tile << 32) | bits(depth key); the per-tile lists ordered by (key, id).
 * ---------------------------------------------------------------------------------- */
typedef struct {
  uint64_t key;
  uint32_t id;
} or_pair;

static int pair_cmp(const void* a, const void* b) {
  const or_pair* x = (const or_pair*)a;
  const or_pair* y = (const or_pair*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

int64_t or_bin(int64_t n, const int32_t* count, const int32_t* rect, const float* key, int32_t n_tiles,
               int32_t n_cols_total, int64_t capacity, uint64_t* keys_out, uint32_t* ids_out, int32_t* ranges) {
  int64_t P = 0;
  for (int64_t g = 0; g < n; ++g) P += count[g];
  if (P > capacity || keys_out == NULL) return P;
  or_pair* pairs = (or_pair*)malloc(sizeof(or_pair) * (P > 0 ? P : 1));
  int64_t k = 0;
  for (int64_t g = 0; g < n; ++g) {
    if (count[g] == 0) continue;
    uint32_t kb;
    memcpy(&kb, &key[g], 4);
    for (int32_t row = rect[g * 4]; row <= rect[g * 4 + 1]; ++row)
      for (int32_t c = 0; c < rect[g * 4 + 3]; ++c) {
        int64_t tile = (int64_t)row * n_cols_total + (rect[g * 4 + 2] + c) % n_cols_total;
        pairs[k].key = ((uint64_t)tile << 32) | kb;
        pairs[k].id = (uint32_t)g;
        k++;
      }
  }
  qsort(pairs, (size_t)P, sizeof(or_pair), pair_cmp);
  for (int32_t t = 0; t < 2 * n_tiles; ++t) ranges[t] = 0;
  for (int64_t i = 0; i < P; ++i) {
    keys_out[i] = pairs[i].key;
    ids_out[i] = pairs[i].id;
    int32_t t = (int32_t)(pairs[i].key >> 32);
    if (i == 0 || (int32_t)(pairs[i - 1].key >> 32) != t) ranges[2 * t] = (int32_t)i;
    if (i == P - 1 || (int32_t)(pairs[i + 1].key >> 32) != t) ranges[2 * t + 1] = (int32_t)(i + 1);
  }
  free(pairs);
  return P;
}

/* ------------------------------------------------------------------------------------
 * O12 Front-to-back compositing, Eq. 1 with the 3D response at tau_max
 *     (P:129), LiDAR features.  Per ray, over its tile's list in order:
 *     membership (A12) -> response -> alpha = min(alpha_max, sigma rho) -> skip if
 *     alpha < alpha_min or tau < near -> T' = T (1 - alpha); stop if T' < T_min (A14)
 *     -> accumulate.   flag bits (A23): 1 box edge, 2 alpha_min, 4 T_min, 8 validity,
 *     16 near threshold.
 * ---------------------------------------------------------------------------------- */
static int in_interval_a(float lo, float hi, float x, int wrap, float pi_f, float two_pi_f) {
  if (!wrap) return lo <= x && x <= hi;
  volatile float width = hi - lo;
  if (width >= two_pi_f) return 1;
  if (lo <= x && x <= hi) return 1;
  if (lo < -pi_f) {
    volatile float l2 = lo + two_pi_f;
    if (l2 <= x) return 1;
  }
  if (hi > pi_f) {
    volatile float h2 = hi - two_pi_f;
    if (x <= h2) return 1;
  }
  return 0;
}

/* same test on a box grown (eps > 0) or shrunk (eps < 0) in double (flag mode) */
static int in_interval_a_d(double lo, double hi, double x, int wrap, double eps) {
  lo -= eps;
  hi += eps;
  if (!wrap) return lo <= x && x <= hi;
  if (hi - lo >= OR_TWO_PI) return 1;
  for (int k = -1; k <= 1; ++k) {
    double xx = x + k * OR_TWO_PI;
    if (lo <= xx && xx <= hi) return 1;
  }
  return 0;
}

int or_composite(int64_t n_gauss, const double* mu, const double* Mrows, const double* sigma, const double* feat,
                 const float* box, const int32_t* gamb, const uint32_t* ids, const int32_t* ranges, int32_t n_rays,
                 const int32_t* ray_tile, const float* ray_a, const float* ray_b, const double* ray_od,
                 const int32_t* ray_valid, const or_render_params* p, or_render_out* out) {
  (void)n_gauss;
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t r = 0; r < n_rays; ++r) {
    double T = 1.0, acc[3] = {0, 0, 0}, D = 0.0, w = 0.0;
    int32_t nc = 0, flag = 0;
    int64_t scanned = 0, inbox = 0;
    if (ray_valid == NULL || ray_valid[r]) {
      const double* o = &ray_od[(int64_t)r * 6];
      const double* d = o + 3;
      int32_t t = ray_tile[r];
      float xa = ray_a[r], xb = ray_b[r];
      for (int32_t i = ranges[2 * t]; i < ranges[2 * t + 1]; ++i) {
        uint32_t g = ids[i];
        const float* bx = &box[(int64_t)g * 4];
        scanned++;
        int member = in_interval_a(bx[0], bx[1], xa, p->wrap, p->pi_f, p->two_pi_f) && bx[2] <= xb && xb <= bx[3];
        if (p->flag_mode) {
          int loose = in_interval_a_d(bx[0], bx[1], xa, p->wrap, p->eps_a) &&
                      (double)bx[2] - p->eps_b <= xb && xb <= (double)bx[3] + p->eps_b;
          int strict = in_interval_a_d(bx[0], bx[1], xa, p->wrap, -p->eps_a) &&
                       (double)bx[2] + p->eps_b <= xb && xb <= (double)bx[3] - p->eps_b;
          /* validity-ambiguous particles (gamb): the float32 box may differ a lot (e.g. a
           * sigma point at the sweep seam) -> candidates are the live rays inside a
           * generously grown box; like box-edge flips they only count if they could matter */
          const int amb_box = gamb && gamb[g] && in_interval_a_d(bx[0], bx[1], xa, p->wrap, p->eps_amb_a) &&
                              (double)bx[2] - p->eps_amb_b <= xb && xb <= (double)bx[3] + p->eps_amb_b;
          if (loose != strict || amb_box) {
            /* ambiguous membership matters only if this particle could composite with a
             * weight alpha T above the impact threshold (its alpha if it were a member) */
            double rs0[2];
            or_response(&mu[(int64_t)g * 3], &Mrows[(int64_t)g * 9], o, d, rs0);
            double a0 = sigma[g] * exp(-0.5 * rs0[1]);
            if (!(isfinite(a0)) || (a0 >= p->alpha_min - p->eps_alpha && a0 * T > p->eps_impact))
              flag |= (loose != strict) ? 1 : 8;
          }
        }
        if (gamb && gamb[g] == 2) continue; /* listed for flagging only (oracle-invalid) */
        if (!member) continue;
        inbox++;
        double rs[2];
        or_response(&mu[(int64_t)g * 3], &Mrows[(int64_t)g * 9], o, d, rs);
        double tau = rs[0];
        double a = sigma[g] * exp(-0.5 * rs[1]);
        double alpha = a < p->alpha_max ? a : p->alpha_max;
        if (p->flag_mode) {
          if (fabs(tau - p->near_tau) < p->eps_tau) flag |= 16;
          if (fabs(a - p->alpha_min) < p->eps_alpha) flag |= 2;
        }
        if (tau < p->near_tau) continue;
        if (alpha < p->alpha_min) continue;
        double Tn = T * (1.0 - alpha);
        if (p->flag_mode && fabs(Tn - p->T_min) < p->eps_T_rel * p->T_min) flag |= 4;
        if (Tn < p->T_min) break;
        double f[3] = {feat[(int64_t)g * 3], feat[(int64_t)g * 3 + 1], feat[(int64_t)g * 3 + 2]};
        if (p->sh) { /* Eq. 1 literally: SH_i(d), d the ray's unit direction (A30) */
          const int nco = (p->sh_degree + 1) * (p->sh_degree + 1);
          double shd[48], dn[3];
          const double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
          for (int c = 0; c < 3; ++c) dn[c] = d[c] / dl;
          for (int k = 0; k < nco * 3; ++k) shd[k] = p->sh[(int64_t)g * nco * 3 + k];
          or_sh_eval(shd, p->sh_degree, dn, f);
        }
        for (int c = 0; c < 3; ++c) acc[c] += alpha * T * f[c];
        D += alpha * T * tau;
        w += alpha * T;
        nc++;
        T = Tn;
      }
    }
    for (int c = 0; c < 3; ++c) out->feat[(int64_t)r * 3 + c] = acc[c];
    out->opacity[r] = w;
    out->depth_accum[r] = D;
    out->depth[r] = w > 0.0 ? D / w : 0.0;
    out->T_final[r] = T;
    out->n_contrib[r] = nc;
    if (out->flag) out->flag[r] = flag;
    if (out->scanned) out->scanned[r] = scanned;
    if (out->inbox) out->inbox[r] = inbox;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------
 * Rays.  LiDAR ray (b, j): o = t(s_j), d = R(s_j) (cos w cos phi, cos w sin phi, sin w)
 * with (phi_j, omega_b, s_j) the float32 ray-table values (A5).  Camera pixel (i, j):
 * centre (i + 0.5, j + 0.5), row time s = (j + 0.5)/H if rolling (A22).
 * ---------------------------------------------------------------------------------- */
void or_lidar_rays(const or_tiling* t, const double pose0[7], const double pose1[7], double* od) {
#pragma omp parallel for schedule(static)
  for (int32_t r = 0; r < t->n_rays; ++r) {
    double R[9], tt[3];
    or_pose_at(pose0, pose1, (double)t->ray_s[r], R, tt);
    double phi = t->ray_az[r], om = t->ray_el[r];
    double u[3] = {cos(om) * cos(phi), cos(om) * sin(phi), sin(om)};
    for (int i = 0; i < 3; ++i) {
      od[(int64_t)r * 6 + i] = tt[i];
      od[(int64_t)r * 6 + 3 + i] = R[i * 3] * u[0] + R[i * 3 + 1] * u[1] + R[i * 3 + 2] * u[2];
    }
  }
}

void or_camera_rays(const or_camera* C, const double pose0[7], const double pose1[7], double* od, int32_t* valid,
                    float* pix_u, float* pix_v, int32_t* ray_tile) {
  int32_t W = C->width, H = C->height, tp = C->tile_px;
  int32_t Wt = (W + tp - 1) / tp;
#pragma omp parallel for schedule(static)
  for (int32_t j = 0; j < H; ++j) {
    for (int32_t i = 0; i < W; ++i) {
      int64_t r = (int64_t)j * W + i;
      double u = i + 0.5, v = j + 0.5, dc[3], R[9], tt[3];
      double s = C->rolling ? v / (double)H : 0.0;
      valid[r] = or_camera_unproject(C, u, v, dc);
      or_pose_at(pose0, pose1, s, R, tt);
      for (int k = 0; k < 3; ++k) {
        od[r * 6 + k] = tt[k];
        od[r * 6 + 3 + k] = valid[r] ? R[k * 3] * dc[0] + R[k * 3 + 1] * dc[1] + R[k * 3 + 2] * dc[2] : 0.0;
      }
      pix_u[r] = (float)u;
      pix_v[r] = (float)v;
      ray_tile[r] = (j / tp) * Wt + (i / tp);
    }
  }
}

/* ------------------------------------------------------------------------------------
 * O14 Camera final colour, Eq. 2:  c = A(omega c_f + (1 - omega) c_b(d)).
 *     c_b: learned environment map -- reading A28: an equirectangular texture in
 *     the world frame (z up), longitude atan2(d_y, d_x) over [-pi, pi) -> [0, W_e), colatitude
 *     acos(d_z) over [0, pi] -> [0, H_e), texel centres at +0.5, bilinear, wrapping in
 *     longitude, clamped in colatitude.  A: learned bilateral grid -- a grid of 3x4
 *     affine matrices over (x / W, y / H, luminance) with luminance = 0.299 r + 0.587 g +
 *     0.114 b of the blended colour (clamped to [0, 1]), cell centres at +0.5, trilinear,
 *     clamped at the borders; c = M[:, :3] c_in + M[:, 3].  d = the pixel's unit ray
 *     direction (world).  env == NULL: c_b = 0; grid == NULL: A = identity.
 *     rgb_fg is Eq. 1's sum SH alpha T = omega * (normalised c_f), so "omega c_f" of Eq. 2 is
 *     rgb_fg itself (A28: the step is alpha compositing).
 * ---------------------------------------------------------------------------------- */
static void env_lookup(const float* env, int32_t He, int32_t We, const double d[3], double out[3]) {
  double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  double lon = atan2(d[1], d[0]);
  double z = n > 0.0 ? d[2] / n : 1.0;
  if (z > 1.0) z = 1.0;
  if (z < -1.0) z = -1.0;
  double colat = acos(z);
  double u = (lon + OR_PI) / OR_TWO_PI * We - 0.5;
  double v = colat / OR_PI * He - 0.5;
  double fu = floor(u), fv = floor(v);
  double au = u - fu, av = v - fv;
  int64_t u0 = (int64_t)fu, v0 = (int64_t)fv;
  for (int c = 0; c < 3; ++c) out[c] = 0.0;
  for (int dv = 0; dv <= 1; ++dv)
    for (int du = 0; du <= 1; ++du) {
      int64_t uu = ((u0 + du) % We + We) % We;
      int64_t vv = v0 + dv;
      if (vv < 0) vv = 0;
      if (vv > He - 1) vv = He - 1;
      double w = (du ? au : 1.0 - au) * (dv ? av : 1.0 - av);
      for (int c = 0; c < 3; ++c) out[c] += w * env[(vv * We + uu) * 3 + c];
    }
}

static void grid_apply(const float* grid, int32_t gh, int32_t gw, int32_t gd, double x, double y, const double cin[3],
                       double out[3]) {
  double lum = 0.299 * cin[0] + 0.587 * cin[1] + 0.114 * cin[2];
  if (lum < 0.0) lum = 0.0;
  if (lum > 1.0) lum = 1.0;
  double g[3] = {x * gw - 0.5, y * gh - 0.5, lum * gd - 0.5};
  int32_t n[3] = {gw, gh, gd};
  int64_t i0[3];
  double a[3];
  for (int k = 0; k < 3; ++k) {
    double c = g[k];
    if (c < 0.0) c = 0.0;
    if (c > n[k] - 1) c = n[k] - 1;
    double f = floor(c);
    i0[k] = (int64_t)f;
    a[k] = c - f;
  }
  double M[12] = {0};
  for (int dz = 0; dz <= 1; ++dz)
    for (int dy = 0; dy <= 1; ++dy)
      for (int dx = 0; dx <= 1; ++dx) {
        int64_t xi = i0[0] + dx, yi = i0[1] + dy, zi = i0[2] + dz;
        if (xi > gw - 1) xi = gw - 1;
        if (yi > gh - 1) yi = gh - 1;
        if (zi > gd - 1) zi = gd - 1;
        double w = (dx ? a[0] : 1.0 - a[0]) * (dy ? a[1] : 1.0 - a[1]) * (dz ? a[2] : 1.0 - a[2]);
        const float* m = &grid[((zi * gh + yi) * gw + xi) * 12];
        for (int q = 0; q < 12; ++q) M[q] += w * m[q];
      }
  for (int r = 0; r < 3; ++r) out[r] = M[r * 4] * cin[0] + M[r * 4 + 1] * cin[1] + M[r * 4 + 2] * cin[2] + M[r * 4 + 3];
}

int or_compose_camera(const or_camera* C, const double* ray_od, const double* rgb_fg, const double* omega,
                      const float* env, int32_t He, int32_t We, const float* grid, int32_t gh, int32_t gw,
                      int32_t gd, double* rgb_out) {
  int32_t W = C->width, H = C->height;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)W * H; ++r) {
    const double* d = &ray_od[r * 6 + 3];
    double cb[3] = {0, 0, 0}, cin[3];
    if (env) env_lookup(env, He, We, d, cb);
    for (int c = 0; c < 3; ++c) cin[c] = rgb_fg[r * 3 + c] + (1.0 - omega[r]) * cb[c];
    if (grid) {
      double x = ((double)(r % W) + 0.5) / W, y = ((double)(r / W) + 0.5) / H;
      grid_apply(grid, gh, gw, gd, x, y, cin, &rgb_out[r * 3]);
    } else {
      for (int c = 0; c < 3; ++c) rgb_out[r * 3 + c] = cin[c];
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------
 * O0 Scene graph (reading A29): particles of a dynamic object live in the object's
 *     local frame and are "transformed to world coordinates by applying the SE(3)
 *     transformation corresponding to the timestamp t":  mu_w = R_a mu + t_a,
 *     Sigma_w = R_a Sigma R_a^T, i.e. the rotation R_a R(q) = R(q_a (x) q) with S unchanged.
 *     The world particle is a float32 particle (mu_w rounded once from double, q_w the
 *     normalised double product rounded to float32).  actor_id -1: static (copied);
 *     outside [-1, n_actors): the particle is made degenerate (zero quaternion -> invalid,
 *     A20).  actor_pose [n_actors][7] = (q w,x,y,z, t), object -> world at t.
 * ---------------------------------------------------------------------------------- */
void or_actors_to_world(int64_t n, const float* means, const float* quats, const int32_t* actor_id,
                        int32_t n_actors, const double* actor_pose, float* means_w, float* quats_w) {
  for (int64_t i = 0; i < n; ++i) {
    const int32_t a = actor_id[i];
    if (a == -1) {
      for (int c = 0; c < 3; ++c) means_w[3 * i + c] = means[3 * i + c];
      for (int c = 0; c < 4; ++c) quats_w[4 * i + c] = quats[4 * i + c];
      continue;
    }
    if (a < -1 || a >= n_actors) {
      for (int c = 0; c < 3; ++c) means_w[3 * i + c] = means[3 * i + c];
      for (int c = 0; c < 4; ++c) quats_w[4 * i + c] = 0.0f;
      continue;
    }
    const double* P = actor_pose + 7 * (int64_t)a;
    double Ra[9];
    or_quat_to_rot(P, Ra);
    for (int r = 0; r < 3; ++r) {
      double acc = P[4 + r];
      for (int c = 0; c < 3; ++c) acc += Ra[3 * r + c] * (double)means[3 * i + c];
      means_w[3 * i + r] = (float)acc;
    }
    /* Hamilton product q_a (x) q of the unit quaternions */
    double qa[4], q[4], na = 0.0, nq = 0.0;
    for (int c = 0; c < 4; ++c) {
      qa[c] = P[c];
      q[c] = quats[4 * i + c];
      na += qa[c] * qa[c];
      nq += q[c] * q[c];
    }
    if (!(na > 0.0) || !(nq > 0.0)) {
      for (int c = 0; c < 4; ++c) quats_w[4 * i + c] = 0.0f;
      continue;
    }
    na = sqrt(na);
    nq = sqrt(nq);
    for (int c = 0; c < 4; ++c) {
      qa[c] /= na;
      q[c] /= nq;
    }
    const double w = qa[0] * q[0] - qa[1] * q[1] - qa[2] * q[2] - qa[3] * q[3];
    const double x = qa[0] * q[1] + qa[1] * q[0] + qa[2] * q[3] - qa[3] * q[2];
    const double y = qa[0] * q[2] - qa[1] * q[3] + qa[2] * q[0] + qa[3] * q[1];
    const double z = qa[0] * q[3] + qa[1] * q[2] - qa[2] * q[1] + qa[3] * q[0];
    quats_w[4 * i + 0] = (float)w;
    quats_w[4 * i + 1] = (float)x;
    quats_w[4 * i + 2] = (float)y;
    quats_w[4 * i + 3] = (float)z;
  }
}

/* ------------------------------------------------------------------------------------
 * O15 backward of Eq. 1 (reading A31).  For one ray with contributions
 * k = 1..K in list order (the members or_composite composites: not skipped, before the
 * terminating particle):
 *   w_k = alpha_k T_k,  T_k = prod_{j<k} (1 - alpha_j),
 *   zeta = sum w_k f_k,  omega = sum w_k,  D = sum w_k tau_k.
 * With upstream gradients (Gz, Go, GD) and suffix sums S_k(x) = sum_{i>k} w_i x_i:
 *   dL/dalpha_k = T_k (Gz.f_k + Go + GD tau_k) - (Gz.S_k(f) + Go S_k(1) + GD S_k(tau)) / (1 - alpha_k)
 *   dL/dtau_k = GD w_k,   dL/df_k = Gz w_k.
 * alpha = min(alpha_max, sigma rho), rho = exp(-delta^2 / 2): if not clamped,
 *   dL/dsigma = dL/dalpha rho,  dL/d(delta^2) = -dL/dalpha alpha / 2 (clamped: 0).
 * Response (O12) with u = M d, w = M (o - mu), n2 = |u|^2:
 *   tau = -(w.u)/n2,  delta^2 = |w|^2 - (w.u)^2/n2
 *   d(delta^2)/dw = 2 (w + tau u),  d(delta^2)/du = 2 tau (w + tau u)
 *   dtau/dw = -u/n2,               dtau/du = -(w + 2 tau u)/n2
 *   dL/dM = gw (o - mu)^T + gu d^T,  dL/dmu = -M^T gw.
 * Membership, skips and termination are discrete: no gradient through them.
 * ---------------------------------------------------------------------------------- */
int or_backward_composite(const double* mu, const double* Mrows, const double* sigma, const double* feat,
                          const float* box, const uint32_t* ids, const int32_t* ranges, int32_t n_rays,
                          const int32_t* ray_tile, const float* ray_a, const float* ray_b, const double* ray_od,
                          const int32_t* ray_valid, const or_render_params* p, const double* g_feat,
                          const double* g_opacity, const double* g_daccum, double* d_mu, double* d_M,
                          double* d_sigma, double* d_feat, double* d_sh) {
  int64_t max_len = 0;
  for (int32_t r = 0; r < n_rays; ++r) {
    const int32_t t = ray_tile[r];
    if (ranges[2 * t + 1] - ranges[2 * t] > max_len) max_len = ranges[2 * t + 1] - ranges[2 * t];
  }
  int fail = 0;
#pragma omp parallel
  {
    uint32_t* kg = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(max_len + 1));
    double* ka = (double*)malloc(sizeof(double) * (size_t)(max_len + 1) * 4); /* alpha, tau, T, rho */
    int* kc = (int*)malloc(sizeof(int) * (size_t)(max_len + 1));              /* clamped */
    if (!kg || !ka || !kc) {
#pragma omp atomic write
      fail = 1;
    } else {
#pragma omp for schedule(dynamic, 64)
      for (int32_t r = 0; r < n_rays; ++r) {
        if (ray_valid && !ray_valid[r]) continue;
        const double* o = &ray_od[(int64_t)r * 6];
        const double* d = o + 3;
        const int32_t t = ray_tile[r];
        const float xa = ray_a[r], xb = ray_b[r];
        /* forward: the contributions in list order (or_composite's rules) */
        int K = 0;
        double T = 1.0;
        for (int32_t i = ranges[2 * t]; i < ranges[2 * t + 1]; ++i) {
          const uint32_t g = ids[i];
          const float* bx = &box[(int64_t)g * 4];
          if (!(in_interval_a(bx[0], bx[1], xa, p->wrap, p->pi_f, p->two_pi_f) && bx[2] <= xb && xb <= bx[3]))
            continue;
          double rs[2];
          or_response(&mu[(int64_t)g * 3], &Mrows[(int64_t)g * 9], o, d, rs);
          const double rho = exp(-0.5 * rs[1]);
          const double a = sigma[g] * rho;
          const double alpha = a < p->alpha_max ? a : p->alpha_max;
          if (rs[0] < p->near_tau || alpha < p->alpha_min) continue;
          const double Tn = T * (1.0 - alpha);
          if (Tn < p->T_min) break;
          kg[K] = g;
          ka[4 * K] = alpha;
          ka[4 * K + 1] = rs[0];
          ka[4 * K + 2] = T;
          ka[4 * K + 3] = rho;
          kc[K] = !(a < p->alpha_max);
          ++K;
          T = Tn;
        }
        const double Gz[3] = {g_feat ? g_feat[3 * (int64_t)r] : 0.0, g_feat ? g_feat[3 * (int64_t)r + 1] : 0.0,
                              g_feat ? g_feat[3 * (int64_t)r + 2] : 0.0};
        const double Go = g_opacity ? g_opacity[r] : 0.0, GD = g_daccum ? g_daccum[r] : 0.0;
        /* backward, last contribution first, carrying the suffix sums */
        double Sf = 0.0, S1 = 0.0, St = 0.0; /* Gz.S(f), S(1), S(tau) */
        for (int k = K - 1; k >= 0; --k) {
          const uint32_t g = kg[k];
          const double alpha = ka[4 * k], tau = ka[4 * k + 1], Tk = ka[4 * k + 2], rho = ka[4 * k + 3];
          double f[3] = {feat[(int64_t)g * 3], feat[(int64_t)g * 3 + 1], feat[(int64_t)g * 3 + 2]};
          double Y[16];
          const int nco = p->sh ? (p->sh_degree + 1) * (p->sh_degree + 1) : 0;
          if (p->sh) { /* per-ray SH (A30): f = SH_g(d) and the basis Y_k(d), through O9 */
            double dn[3], shd[48];
            const double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            for (int c = 0; c < 3; ++c) dn[c] = d[c] / dl;
            for (int q = 0; q < nco * 3; ++q) shd[q] = p->sh[(int64_t)g * nco * 3 + q];
            or_sh_eval(shd, p->sh_degree, dn, f);
            for (int q = 0; q < nco; ++q) {
              double e[48] = {0}, yq[3];
              e[3 * q] = 1.0;
              or_sh_eval(e, p->sh_degree, dn, yq);
              Y[q] = yq[0];
            }
          }
          const double wk = alpha * Tk;
          const double gzf = Gz[0] * f[0] + Gz[1] * f[1] + Gz[2] * f[2];
          const double dalpha = Tk * (gzf + Go + GD * tau) - (Sf + Go * S1 + GD * St) / (1.0 - alpha);
          const double dtau = GD * wk;
          double dsig = 0.0, dd2 = 0.0;
          if (!kc[k]) {
            dsig = dalpha * rho;
            dd2 = -0.5 * dalpha * alpha;
          }
          /* response gradients */
          const double* M = &Mrows[(int64_t)g * 9];
          const double pw[3] = {o[0] - mu[g * 3], o[1] - mu[g * 3 + 1], o[2] - mu[g * 3 + 2]};
          double u[3], w[3];
          for (int a = 0; a < 3; ++a) {
            u[a] = M[3 * a] * d[0] + M[3 * a + 1] * d[1] + M[3 * a + 2] * d[2];
            w[a] = M[3 * a] * pw[0] + M[3 * a + 1] * pw[1] + M[3 * a + 2] * pw[2];
          }
          const double n2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
          const double tr = -(w[0] * u[0] + w[1] * u[1] + w[2] * u[2]) / n2; /* = tau */
          double gw[3], gu[3];
          for (int a = 0; a < 3; ++a) {
            const double h = w[a] + tr * u[a];
            gw[a] = dd2 * 2.0 * h + dtau * (-u[a] / n2);
            gu[a] = dd2 * 2.0 * tr * h + dtau * (-(w[a] + 2.0 * tr * u[a]) / n2);
          }
#pragma omp critical(or_bwd_acc)
          {
            for (int a = 0; a < 3; ++a) {
              for (int b = 0; b < 3; ++b) d_M[(int64_t)g * 9 + 3 * a + b] += gw[a] * pw[b] + gu[a] * d[b];
              double mt = 0.0;
              for (int b = 0; b < 3; ++b) mt += M[3 * b + a] * gw[b];
              d_mu[(int64_t)g * 3 + a] -= mt;
              d_feat[(int64_t)g * 3 + a] += Gz[a] * wk;
            }
            d_sigma[g] += dsig;
            if (p->sh && d_sh) /* dL/dc_qc = Y_q(d) Gz_c w (A30, A31) */
              for (int q = 0; q < nco; ++q)
                for (int c = 0; c < 3; ++c) d_sh[((int64_t)g * nco + q) * 3 + c] += Y[q] * Gz[c] * wk;
          }
          Sf += wk * gzf;
          S1 += wk;
          St += wk * tau;
        }
      }
    }
    free(kg);
    free(ka);
    free(kc);
  }
  return fail ? -1 : 0;
}

/* ------------------------------------------------------------------------------------
 * O16 with the scene graph (A29, A31).  For a particle of object a:
 *   R_w = R_a R_l,  mu_w = R_a mu_l + t_a  (O0)
 *   dL/dR_w = G from dL/dM: M[k][j] = R_w[j][k] / s_k gives G[j][k] = dL/dM[k][j] / s_k and
 *   dL/ds_k = -sum_j dL/dM[k][j] R_w[j][k] / s_k^2 (with beam divergence: the Cholesky chain below),
 *   dL/dR_l = R_a^T G,   dL/dmu_l = R_a^T dL/dmu_w,
 *   dL/dR_a += G R_l^T + dL/dmu_w mu_l^T,   dL/dt_a += dL/dmu_w,
 * each rotation gradient taken to its (unnormalised) quaternion by the O1 chain.  Static
 * particles (id -1, or actor_id NULL) have R_a = I, t_a = 0; ids outside [-1, n_actors) get zeros.
 * dR -> dq of the unnormalised quaternion by differentiating O1's entries, then
 * dL/dq = (dL/dq^ - q^ (q^ . dL/dq^)) / |q|; f = sum_k Y_k(v) c_k (O9): dL/dc_k = Y_k(v) dL/df.
 * g_actor [n_actors][7] = (dL/dq_a, dL/dt_a), accumulated over the object's particles.
 * ---------------------------------------------------------------------------------- */
static void rot_grad_to_quat(const double G[9], const double q_in[4], double dq_out[4]) {
  double qn = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
  const double w = q_in[0] / qn, x = q_in[1] / qn, y = q_in[2] / qn, z = q_in[3] / qn;
  const double dw = 2.0 * (-z * G[1] + y * G[2] + z * G[3] - x * G[5] - y * G[6] + x * G[7]);
  const double dx = 2.0 * (y * G[1] + z * G[2] + y * G[3] - 2.0 * x * G[4] - w * G[5] + z * G[6] + w * G[7] -
                           2.0 * x * G[8]);
  const double dy = 2.0 * (-2.0 * y * G[0] + x * G[1] + w * G[2] + x * G[3] + z * G[5] - w * G[6] + z * G[7] -
                           2.0 * y * G[8]);
  const double dz = 2.0 * (-2.0 * z * G[0] - w * G[1] + x * G[2] + w * G[3] - 2.0 * z * G[4] + y * G[5] +
                           x * G[6] + y * G[7]);
  const double dq[4] = {dw, dx, dy, dz}, qh[4] = {w, x, y, z};
  const double dot = dw * w + dx * x + dy * y + dz * z;
  for (int c = 0; c < 4; ++c) dq_out[c] = (dq[c] - qh[c] * dot) / qn;
}

void or_backward_params_sg(int64_t n, const float* means, const float* quats, const float* scales,
                           const double* viewdir, int32_t sh_degree, const int32_t* actor_id, int32_t n_actors,
                           const double* actor_pose, double beam_div, const double* d_mu, const double* d_M,
                           const double* d_feat, double* g_means, double* g_quats, double* g_scales, double* g_sh,
                           double* g_actor) {
  const int nco = (sh_degree + 1) * (sh_degree + 1);
  double* Ga = (double*)calloc((size_t)(n_actors > 0 ? n_actors : 1) * 12, sizeof(double)); /* dR_a 9, dt_a 3 */
  for (int64_t g = 0; g < n; ++g) {
    for (int c = 0; c < 3; ++c) g_means[3 * g + c] = 0.0;
    for (int c = 0; c < 4; ++c) g_quats[4 * g + c] = 0.0;
    for (int c = 0; c < 3; ++c) g_scales[3 * g + c] = 0.0;
    for (int k = 0; k < nco * 3; ++k) g_sh[(int64_t)g * nco * 3 + k] = 0.0;
    const int32_t a = actor_id ? actor_id[g] : -1;
    if (a < -1 || a >= n_actors) continue;
    double ql[4], qn = 0.0;
    for (int c = 0; c < 4; ++c) {
      ql[c] = quats[4 * g + c];
      qn += ql[c] * ql[c];
    }
    if (!(qn > 0.0) || !isfinite(qn)) continue;
    double Rl[9], Ra[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    or_quat_to_rot(ql, Rl);
    if (a >= 0) or_quat_to_rot(&actor_pose[7 * a], Ra);
    double Rw[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += Ra[3 * i + k] * Rl[3 * k + j];
        Rw[3 * i + j] = acc;
      }
    double G[9];     /* dL/dR_w[j][k] */
    double dmu_w[3] = {d_mu[3 * g], d_mu[3 * g + 1], d_mu[3 * g + 2]};
    if (beam_div > 0.0) {
      /* App. C (A27): M_hat = chol(Sigma_hat)^-1, Sigma_hat = R S^2 R^T + theta^2 (r^2 I - v v^T),
       * v = mu - o (o held at the mean's firing time, A31).  Backward: Mbar (lower) ->
       * Lbar = -M^T Mbar M^T (lower) -> Sigma_bar = sym(M^T Phi(L^T Lbar) M), Phi = lower
       * triangle with the diagonal halved (Cholesky backward) -> v, R, s. */
      const double* v = &viewdir[3 * g];
      const double t2 = beam_div * beam_div, r2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
      double Sh[9], Lh[9], Mh[9], s2[3];
      for (int k = 0; k < 3; ++k) s2[k] = (double)scales[3 * g + k] * (double)scales[3 * g + k];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double acc = 0.0;
          for (int k = 0; k < 3; ++k) acc += Rw[3 * i + k] * s2[k] * Rw[3 * j + k];
          Sh[3 * i + j] = acc + t2 * ((i == j ? r2 : 0.0) - v[i] * v[j]);
        }
      if (or_cholesky3(Sh, Lh)) {
        for (int c = 0; c < 3; ++c) g_scales[3 * g + c] = 0.0;
        continue;
      }
      or_lower_inverse3(Lh, Mh);
      double Mb[9], Lb[9], X[9], P[9], S[9], Sb[9];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Mb[3 * i + j] = j <= i ? d_M[g * 9 + 3 * i + j] : 0.0;
      for (int i = 0; i < 3; ++i) /* Lbar = -(M^T Mbar M^T), lower part */
        for (int j = 0; j < 3; ++j) {
          double acc = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) acc += Mh[3 * a + i] * Mb[3 * a + b] * Mh[3 * j + b];
          Lb[3 * i + j] = j <= i ? -acc : 0.0;
        }
      for (int i = 0; i < 3; ++i) /* X = L^T Lbar */
        for (int j = 0; j < 3; ++j) {
          double acc = 0.0;
          for (int a = 0; a < 3; ++a) acc += Lh[3 * a + i] * Lb[3 * a + j];
          X[3 * i + j] = acc;
        }
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) P[3 * i + j] = j < i ? X[3 * i + j] : (j == i ? 0.5 * X[3 * i + j] : 0.0);
      for (int i = 0; i < 3; ++i) /* S = M^T P M */
        for (int j = 0; j < 3; ++j) {
          double acc = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) acc += Mh[3 * a + i] * P[3 * a + b] * Mh[3 * b + j];
          S[3 * i + j] = acc;
        }
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Sb[3 * i + j] = 0.5 * (S[3 * i + j] + S[3 * j + i]);
      const double tr = Sb[0] + Sb[4] + Sb[8];
      for (int i = 0; i < 3; ++i) { /* dv = 2 theta^2 (tr(Sb) v - Sb v) */
        double sv = 0.0;
        for (int j = 0; j < 3; ++j) sv += Sb[3 * i + j] * v[j];
        dmu_w[i] += 2.0 * t2 * (tr * v[i] - sv);
      }
      for (int i = 0; i < 3; ++i) /* dR = 2 Sb R S^2 */
        for (int k = 0; k < 3; ++k) {
          double acc = 0.0;
          for (int j = 0; j < 3; ++j) acc += Sb[3 * i + j] * Rw[3 * j + k];
          G[3 * i + k] = 2.0 * acc * s2[k];
        }
      for (int k = 0; k < 3; ++k) { /* ds_k = 2 s_k (R^T Sb R)_kk */
        double acc = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) acc += Rw[3 * i + k] * Sb[3 * i + j] * Rw[3 * j + k];
        g_scales[3 * g + k] = 2.0 * (double)scales[3 * g + k] * acc;
      }
    } else {
      for (int k = 0; k < 3; ++k) {
        const double s = scales[3 * g + k];
        double ds = 0.0;
        for (int j = 0; j < 3; ++j) {
          const double dm = d_M[g * 9 + 3 * k + j];
          G[3 * j + k] = dm / s;
          ds -= dm * Rw[3 * j + k] / (s * s);
        }
        g_scales[3 * g + k] = ds;
      }
    }
    double Gl[9], dmu_l[3];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += Ra[3 * k + i] * G[3 * k + j]; /* R_a^T G */
        Gl[3 * i + j] = acc;
      }
      double m = 0.0;
      for (int k = 0; k < 3; ++k) m += Ra[3 * k + i] * dmu_w[k];
      dmu_l[i] = m;
    }
    rot_grad_to_quat(Gl, ql, &g_quats[4 * g]);
    for (int c = 0; c < 3; ++c) g_means[3 * g + c] = dmu_l[c];
    if (a >= 0) {
      double* A = &Ga[12 * a];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double acc = dmu_w[i] * (double)means[3 * g + j]; /* dL/dmu_w mu_l^T */
          for (int k = 0; k < 3; ++k) acc += G[3 * i + k] * Rl[3 * j + k]; /* G R_l^T */
          A[3 * i + j] += acc;
        }
      for (int c = 0; c < 3; ++c) A[9 + c] += dmu_w[c];
    }
    double vu[3];
    const double vl = sqrt(viewdir[3 * g] * viewdir[3 * g] + viewdir[3 * g + 1] * viewdir[3 * g + 1] +
                           viewdir[3 * g + 2] * viewdir[3 * g + 2]);
    for (int c = 0; c < 3; ++c) vu[c] = vl > 0.0 ? viewdir[3 * g + c] / vl : 0.0;
    for (int k = 0; k < nco; ++k) {
      double e[48] = {0}, yk[3];
      e[3 * k] = 1.0;
      or_sh_eval(e, sh_degree, vu, yk);
      for (int c = 0; c < 3; ++c) g_sh[(int64_t)g * nco * 3 + 3 * k + c] = yk[0] * d_feat[3 * g + c];
    }
  }
  for (int a = 0; a < n_actors; ++a) {
    rot_grad_to_quat(&Ga[12 * a], &actor_pose[7 * a], &g_actor[7 * a]);
    for (int c = 0; c < 3; ++c) g_actor[7 * a + 4 + c] = Ga[12 * a + 9 + c];
  }
  free(Ga);
}
