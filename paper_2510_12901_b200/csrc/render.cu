// simuli_render_lidar / simuli_render_camera: per-ray front-to-back compositing (sm_100a).
//
// Eq. 1: c_f = sum f_i alpha_i T_i, omega = sum alpha_i T_i,
// alpha_i = sigma_i rho_i(o + tau_max d), T_i = prod_{j<i} (1 - alpha_j); the 3D response
// at tau_max; LiDAR features zeta -> intensity gamma = zeta_0 and ray drop
// softmax(zeta_1, zeta_2).  A listed particle contributes to a ray only if its box
// contains the ray (A12), which makes the result independent of tiling and culling.
//
// LiDAR: one warp per (tile, chunk of <= 32 rays), lane = ray.  Each warp stages batches of
// 32 records (32 x 80 B) of its tile's sorted list in shared memory, every lane walks the
// batch front to back, and the warp leaves the list once every ray has terminated
// (T (1 - alpha) < T_min; warp vote).  Rays are generated in double (pose at the column's
// firing time) and split into float hi/lo parts for the compensated response.
// Camera: one CTA of tile_px^2 threads per tile (pixel per thread), 256-record batches in
// shared memory, CTA-wide early exit; pixel rays by the inverse lens model in double.
#include <cstdint>

#include "abi_util.h"
#include "common.cuh"

namespace simuli {
namespace {

constexpr int kWarpsPerCta = 4;

struct LidarArgs {
  const float4* record;
  const uint32_t* ids;
  const int2* ranges;
  const int* tile_ray_offsets;
  const int* tile_rays;
  const float *ray_az, *ray_el, *ray_s;
  int n_tiles, chunks_per_tile;
  PoseInterpD pose;
  float pi_f, two_pi_f, near_tau, alpha_min, alpha_max, T_min;
  float *zeta, *opacity, *depth_accum, *depth, *intensity, *raydrop, *final_T;
  int* n_contrib;
  double* ray_od;
  int *n_visited, *n_inbox;
};

__global__ void __launch_bounds__(32 * kWarpsPerCta) k_render_lidar(const LidarArgs A) {
  __shared__ float4 s_rec[kWarpsPerCta][32][5];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wg = (int64_t)blockIdx.x * kWarpsPerCta + warp;
  const int tile = (int)(wg / A.chunks_per_tile);
  const int chunk = (int)(wg % A.chunks_per_tile);
  if (tile >= A.n_tiles) return;
  const int r_begin = __ldg(A.tile_ray_offsets + tile) + chunk * 32;
  const int r_end = __ldg(A.tile_ray_offsets + tile + 1);
  if (r_begin >= r_end) return;  // warp-uniform
  const bool active = r_begin + lane < r_end;
  const int ray = active ? __ldg(A.tile_rays + r_begin + lane) : 0;

  // ---- ray o(s_j), d(s_j) in double (A5): pose at the column firing time
  RayF rf;
  float ra = 0.f, rb = 0.f;
  double o[3] = {0, 0, 0}, dd[3] = {1, 0, 0};
  if (active) {
    ra = __ldg(A.ray_az + ray);
    rb = __ldg(A.ray_el + ray);
    double R[9];
    pose_at_d(A.pose, (double)__ldg(A.ray_s + ray), R, o);
    double sa, ca, se, ce;
    sincos((double)ra, &sa, &ca);
    sincos((double)rb, &se, &ce);
    const double u[3] = {ce * ca, ce * sa, se};
#pragma unroll
    for (int i = 0; i < 3; ++i) dd[i] = R[3 * i] * u[0] + R[3 * i + 1] * u[1] + R[3 * i + 2] * u[2];
  }
  split_ray(o, dd, rf);

  float T = 1.f, acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, D = 0.f, W = 0.f;
  int nc = 0, nv = 0, ni = 0;
  bool done = !active;
  const int2 rg = __ldg(A.ranges + tile);
  for (int b = rg.x; b < rg.y; b += 32) {
    const int nb = min(32, rg.y - b);
    if (lane < nb) {
      const uint32_t g = __ldg(A.ids + b + lane);
      const float4* src = A.record + (size_t)g * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) s_rec[warp][lane][c] = __ldg(src + c);
    }
    __syncwarp();
    if (!done) {
      for (int j = 0; j < nb; ++j) {
        const float4 bx = s_rec[warp][j][4];
        ++nv;
        if (!in_box_wrap(bx.x, bx.y, bx.z, bx.w, ra, rb, A.pi_f, A.two_pi_f)) continue;
        ++ni;
        const float4 r0 = s_rec[warp][j][0], r1 = s_rec[warp][j][1], r2 = s_rec[warp][j][2],
                     r3 = s_rec[warp][j][3];
        const float mu[3] = {r0.x, r0.y, r0.z};
        const float M[9] = {r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
        float tau, d2;
        response(rf, mu, M, &tau, &d2);
        const float alpha = fminf(A.alpha_max, r3.x * expf(-0.5f * d2));
        if (tau < A.near_tau || alpha < A.alpha_min) continue;
        const float Tn = T * (1.f - alpha);
        if (Tn < A.T_min) {
          done = true;
          break;
        }
        const float w = alpha * T;
        acc0 = fmaf(w, r3.y, acc0);
        acc1 = fmaf(w, r3.z, acc1);
        acc2 = fmaf(w, r3.w, acc2);
        D = fmaf(w, tau, D);
        W += w;
        ++nc;
        T = Tn;
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    __syncwarp();
  }
  if (!active) return;
  if (A.zeta) {
    A.zeta[3 * (size_t)ray] = acc0;
    A.zeta[3 * (size_t)ray + 1] = acc1;
    A.zeta[3 * (size_t)ray + 2] = acc2;
  }
  if (A.opacity) A.opacity[ray] = W;
  if (A.depth_accum) A.depth_accum[ray] = D;
  if (A.depth) A.depth[ray] = W > 0.f ? D / W : 0.f;
  if (A.intensity) A.intensity[ray] = acc0;
  if (A.raydrop) A.raydrop[ray] = raydrop_prob(acc1, acc2);
  if (A.final_T) A.final_T[ray] = T;
  if (A.n_contrib) A.n_contrib[ray] = nc;
  if (A.n_visited) A.n_visited[ray] = nv;
  if (A.n_inbox) A.n_inbox[ray] = ni;
  if (A.ray_od) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      A.ray_od[6 * (size_t)ray + i] = o[i];
      A.ray_od[6 * (size_t)ray + 3 + i] = dd[i];
    }
  }
}

// ------------------------------------------------------------------ camera
struct CameraArgs {
  const float4* record;
  const uint32_t* ids;
  const int2* ranges;
  int model, width, height, rolling, tile_px, Wt;
  double fx, fy, cx, cy, k[5], max_theta;
  PoseInterpD pose;
  float near_tau, alpha_min, alpha_max, T_min;
  float *rgb, *opacity, *depth_accum, *depth, *final_T;
  int* n_contrib;
  double* ray_od;
  int *n_visited, *n_inbox;
};

// inverse lens model in double (A22): KB by Newton on theta_d(theta) = r_d, radtan by
// fixed-point undistortion.  Returns false outside the model's validity.
__device__ bool unproject(const CameraArgs& A, double u, double v, double dir[3]) {
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

template <int TP>
__global__ void __launch_bounds__(TP* TP) k_render_camera(const CameraArgs A) {
  constexpr int NT = TP * TP;
  __shared__ float4 s_rec[NT][5];
  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int ty = tile / A.Wt, tx = tile % A.Wt;
  const int i = tx * TP + (tid % TP), j = ty * TP + (tid / TP);
  const bool inside = i < A.width && j < A.height;
  const float pu = (float)i + 0.5f, pv = (float)j + 0.5f;
  double o[3] = {0, 0, 0}, d[3] = {0, 0, 0};
  bool valid = false;
  if (inside) {
    double dc[3];
    valid = unproject(A, (double)i + 0.5, (double)j + 0.5, dc);
    const double s = A.rolling ? ((double)j + 0.5) / (double)A.height : 0.0;
    double R[9];
    pose_at_d(A.pose, s, R, o);
    if (valid)
      for (int k = 0; k < 3; ++k) d[k] = R[3 * k] * dc[0] + R[3 * k + 1] * dc[1] + R[3 * k + 2] * dc[2];
  }
  RayF rf;
  split_ray(o, d, rf);
  float T = 1.f, acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, D = 0.f, W = 0.f;
  int nc = 0, nv = 0, ni = 0;
  bool done = !(inside && valid);
  const int2 rg = __ldg(A.ranges + tile);
  for (int b = rg.x; b < rg.y; b += NT) {
    if (__syncthreads_count(!done) == 0) break;
    const int nb = min(NT, rg.y - b);
    if (tid < nb) {
      const uint32_t g = __ldg(A.ids + b + tid);
      const float4* src = A.record + (size_t)g * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) s_rec[tid][c] = __ldg(src + c);
    }
    __syncthreads();
    if (!done) {
      for (int jj = 0; jj < nb; ++jj) {
        const float4 bx = s_rec[jj][4];
        ++nv;
        if (!(bx.x <= pu && pu <= bx.y && bx.z <= pv && pv <= bx.w)) continue;
        ++ni;
        const float4 r0 = s_rec[jj][0], r1 = s_rec[jj][1], r2 = s_rec[jj][2], r3 = s_rec[jj][3];
        const float mu[3] = {r0.x, r0.y, r0.z};
        const float M[9] = {r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
        float tau, d2;
        response(rf, mu, M, &tau, &d2);
        const float alpha = fminf(A.alpha_max, r3.x * expf(-0.5f * d2));
        if (tau < A.near_tau || alpha < A.alpha_min) continue;
        const float Tn = T * (1.f - alpha);
        if (Tn < A.T_min) {
          done = true;
          break;
        }
        const float w = alpha * T;
        acc0 = fmaf(w, r3.y, acc0);
        acc1 = fmaf(w, r3.z, acc1);
        acc2 = fmaf(w, r3.w, acc2);
        D = fmaf(w, tau, D);
        W += w;
        ++nc;
        T = Tn;
      }
    }
    __syncthreads();
  }
  if (!inside) return;
  const size_t p = (size_t)j * A.width + i;
  if (A.rgb) {
    A.rgb[3 * p] = acc0;
    A.rgb[3 * p + 1] = acc1;
    A.rgb[3 * p + 2] = acc2;
  }
  if (A.opacity) A.opacity[p] = W;
  if (A.depth_accum) A.depth_accum[p] = D;
  if (A.depth) A.depth[p] = W > 0.f ? D / W : 0.f;
  if (A.final_T) A.final_T[p] = T;
  if (A.n_contrib) A.n_contrib[p] = nc;
  if (A.n_visited) A.n_visited[p] = nv;
  if (A.n_inbox) A.n_inbox[p] = ni;
  if (A.ray_od)
    for (int k = 0; k < 3; ++k) {
      A.ray_od[6 * p + k] = o[k];
      A.ray_od[6 * p + 3 + k] = d[k];
    }
}

int32_t launch_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return SIMULI_ERR_CUDA;
  }
  return SIMULI_OK;
}

}  // namespace
}  // namespace simuli

extern "C" int32_t simuli_render_lidar(const simuli_projected* proj, const uint32_t* sorted_ids,
                                       const int32_t* tile_ranges, const simuli_project_params* P,
                                       const simuli_render_params* rp, simuli_lidar_out* out, void* stream) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(proj && proj->record && sorted_ids && tile_ranges && P && rp && out, "simuli_render_lidar: NULL argument");
  SIMULI_REQUIRE(P->kind == SIMULI_SENSOR_LIDAR && P->lidar && P->tiling, "simuli_render_lidar: needs LiDAR params");
  const simuli_tiling_dev& T = *P->tiling;
  SIMULI_REQUIRE(T.tile_ray_offsets && T.tile_rays && T.ray_az && T.ray_el && T.ray_s && T.n_tiles >= 1,
                 "simuli_render_lidar: incomplete device tiling");
  SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(proj->record) % 16 == 0, "record must be 16-byte aligned");
  LidarArgs A{};
  A.record = reinterpret_cast<const float4*>(proj->record);
  A.ids = sorted_ids;
  A.ranges = reinterpret_cast<const int2*>(tile_ranges);
  A.tile_ray_offsets = T.tile_ray_offsets;
  A.tile_rays = T.tile_rays;
  A.ray_az = T.ray_az; A.ray_el = T.ray_el; A.ray_s = T.ray_s;
  A.n_tiles = T.n_tiles;
  A.chunks_per_tile = (T.max_rays_in_tile + 31) / 32;
  if (A.chunks_per_tile < 1) A.chunks_per_tile = 1;
  A.pose = make_pose_interp_d(P->pose_start, P->pose_end);
  A.pi_f = T.pi_f; A.two_pi_f = T.two_pi_f;
  A.near_tau = P->lidar->min_range_m;
  A.alpha_min = rp->alpha_min; A.alpha_max = rp->alpha_max; A.T_min = rp->T_min;
  A.zeta = out->zeta; A.opacity = out->opacity; A.depth_accum = out->depth_accum; A.depth = out->depth;
  A.intensity = out->intensity; A.raydrop = out->raydrop; A.final_T = out->final_T; A.n_contrib = out->n_contrib;
  A.ray_od = out->ray_od;
  A.n_visited = out->n_visited;
  A.n_inbox = out->n_inbox;
  const int64_t warps = (int64_t)T.n_tiles * A.chunks_per_tile;
  const unsigned blocks = (unsigned)((warps + kWarpsPerCta - 1) / kWarpsPerCta);
  k_render_lidar<<<blocks, 32 * kWarpsPerCta, 0, reinterpret_cast<cudaStream_t>(stream)>>>(A);
  return launch_check("simuli_render_lidar");
}

extern "C" int32_t simuli_render_camera(const simuli_projected* proj, const uint32_t* sorted_ids,
                                        const int32_t* tile_ranges, const simuli_project_params* P,
                                        const simuli_render_params* rp, simuli_camera_out* out, void* stream) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(proj && proj->record && sorted_ids && tile_ranges && P && rp && out,
                 "simuli_render_camera: NULL argument");
  SIMULI_REQUIRE(P->kind == SIMULI_SENSOR_CAMERA && P->camera, "simuli_render_camera: needs camera params");
  const simuli_camera& C = *P->camera;
  if (C.tile_px != 8 && C.tile_px != 16) {
    set_error("simuli_render_camera: tile_px %d not supported (8 or 16)", C.tile_px);
    return SIMULI_ERR_UNSUPPORTED;
  }
  SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(proj->record) % 16 == 0, "record must be 16-byte aligned");
  CameraArgs A{};
  A.record = reinterpret_cast<const float4*>(proj->record);
  A.ids = sorted_ids;
  A.ranges = reinterpret_cast<const int2*>(tile_ranges);
  A.model = C.model; A.width = C.width; A.height = C.height; A.rolling = C.rolling_shutter; A.tile_px = C.tile_px;
  A.Wt = (C.width + C.tile_px - 1) / C.tile_px;
  const int Ht = (C.height + C.tile_px - 1) / C.tile_px;
  A.fx = C.fx; A.fy = C.fy; A.cx = C.cx; A.cy = C.cy;
  for (int i = 0; i < 5; ++i) A.k[i] = C.k[i];
  A.max_theta = C.max_theta_rad;
  A.pose = make_pose_interp_d(P->pose_start, P->pose_end);
  A.near_tau = C.near_m;
  A.alpha_min = rp->alpha_min; A.alpha_max = rp->alpha_max; A.T_min = rp->T_min;
  A.rgb = out->rgb; A.opacity = out->opacity; A.depth_accum = out->depth_accum; A.depth = out->depth;
  A.final_T = out->final_T; A.n_contrib = out->n_contrib; A.ray_od = out->ray_od;
  A.n_visited = out->n_visited; A.n_inbox = out->n_inbox;
  const unsigned blocks = (unsigned)(A.Wt * Ht);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (C.tile_px) {
    case 8: k_render_camera<8><<<blocks, 64, 0, st>>>(A); break;
    default: k_render_camera<16><<<blocks, 256, 0, st>>>(A); break;
  }
  return launch_check("simuli_render_camera");
}
