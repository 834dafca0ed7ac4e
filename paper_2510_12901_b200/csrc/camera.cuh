// Camera arguments and the inverse lens model shared by the camera render, Eq. 2 composition
// (render.cu) and the camera backward (backward.cu).
#pragma once
#include <cstdint>

#include "common.cuh"

namespace simuli {

// ------------------------------------------------------------------ camera
struct CameraArgs {
  const float4* record;
  const uint32_t* ids;
  const int2* ranges;
  const int* order;  // longest-first tile order (bin_sort) or NULL
  int model, width, height, rolling, tile_px, Wt;
  double fx, fy, cx, cy, k[5], max_theta;
  PoseInterpD pose;
  float near_tau, alpha_min, alpha_max, T_min;
  float *rgb, *opacity, *depth_accum, *depth, *final_T;
  int* n_contrib;
  double* ray_od;
  int *n_visited, *n_inbox;
  const float* sh;  // per-ray SH (A30) or NULL
  int sh_ncoef;
};

// inverse lens model in double (A22): KB by Newton on theta_d(theta) = r_d, radtan by
// fixed-point undistortion.  Returns false outside the model's validity.
__device__ inline bool unproject(const CameraArgs& A, double u, double v, double dir[3]) {
  const double mx = (u - A.cx) / A.fx, my = (v - A.cy) / A.fy;
  if (A.model == SIMULI_CAM_FISHEYE_KB) {
    const double rd = sqrt(mx * mx + my * my);
    if (rd == 0.0) {
      dir[0] = 0.0; dir[1] = 0.0; dir[2] = 1.0;
      return true;
    }
    double th = rd;
    bool conv = false;
    for (int it = 0; it < 30; ++it) {
      const double t2 = th * th;
      const double f = th * (1.0 + t2 * (A.k[0] + t2 * (A.k[1] + t2 * (A.k[2] + t2 * A.k[3])))) - rd;
      const double fp = 1.0 + t2 * (3.0 * A.k[0] + t2 * (5.0 * A.k[1] + t2 * (7.0 * A.k[2] + t2 * 9.0 * A.k[3])));
      const double step = f / fp;
      th -= step;
      if (fabs(step) < 1e-15 * (1.0 + fabs(th))) {
        conv = true;
        break;
      }
    }
    if (!conv || !(th >= 0.0) || th > A.max_theta) return false;
    double sn, cs;
    sincos(th, &sn, &cs);
    dir[0] = sn * mx / rd;
    dir[1] = sn * my / rd;
    dir[2] = cs;
    return true;
  }
  double x = mx, y = my;
  for (int it = 0; it < 60; ++it) {
    const double r2 = x * x + y * y;
    const double radial = 1.0 + r2 * (A.k[0] + r2 * (A.k[1] + r2 * A.k[4]));
    const double dx = 2.0 * A.k[2] * x * y + A.k[3] * (r2 + 2.0 * x * x);
    const double dy = A.k[2] * (r2 + 2.0 * y * y) + 2.0 * A.k[3] * x * y;
    const double nx = (mx - dx) / radial, ny = (my - dy) / radial;
    const double ch = fabs(nx - x) + fabs(ny - y);
    x = nx;
    y = ny;
    if (ch < 1e-16) break;
  }
  const double n = sqrt(x * x + y * y + 1.0);
  dir[0] = x / n;
  dir[1] = y / n;
  dir[2] = 1.0 / n;
  return atan(sqrt(x * x + y * y)) <= A.max_theta;
}

}  // namespace simuli
