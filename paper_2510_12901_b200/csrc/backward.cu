// simuli_backward_lidar / simuli_backward_camera: gradients of the render path (sm_100a).
#include <cstdint>
#include <cstdlib>

#include "abi_util.h"
#include "camera.cuh"
#include "common.cuh"

// ====================================================================== backward (A31)
// Gradients of the compositing (Eq. 1) and of the response with respect
// to the particle records, chained to the parameters.  Per ray the tile's list is
// replayed with the forward kernels' float32 arithmetic, so every discrete decision
// (membership, skips, termination) is the forward's -- except that a LiDAR ray enters list
// segment s > 0 with the product of the earlier segments' products, which can round
// differently from the forward's running product (a T_min crossing within ulps of the
// threshold may move by one member; simuli.h); per contribution k, with suffix sums
// S_k = total - prefix_k:
//   dL/dalpha_k = T_k (Gz.f_k + Go + GD tau_k) - (Gz.S_k(f) + Go S_k(1) + GD S_k(tau)) / (1 - alpha_k)
// (oracle O15).  The totals come from the forward's outputs (or a first list pass).  All
// lanes of a warp walk the same list entry, so a contribution's 16 gradient values (dmu 3,
// dM 9, dsigma, df 3) are warp-reduced by a reduce-scatter butterfly and added with one set
// of float atomics per entry.  LiDAR lists are cut into 512-entry segments (a stats pass of
// per-segment transmittance products, then the gradient pass); k_backward_params chains
// (dmu, dM, dsigma, df) to the particle parameters, the object poses (scene graph) and,
// with beam divergence, through the Cholesky factor of Sigma_hat.
namespace simuli {
namespace {

struct BwdArgs {
  const float4* record;
  const uint32_t* ids;
  const int2* ranges;
  const int* order;  // longest-first tile order or NULL
  const int *tile_ray_off, *tile_rays;  // LiDAR
  const float *ray_az, *ray_el, *ray_s;
  int n_az, chunks;
  float pi_f, two_pi_f;
  CameraArgs cam;  // camera geometry (unproject, pose)
  PoseInterpD pose;
  float near_tau, alpha_min, alpha_max, T_min;
  const float *g_feat, *g_opacity, *g_daccum, *g_depth, *g_intensity, *g_raydrop;
  const float *f_feat, *f_opacity, *f_daccum;  // forward totals (optional: skip pass 1)
  const float* sh;  // per-ray SH (A30) or NULL
  int sh_ncoef;
  float* dsh;       // per-ray SH: dL/dSH accumulated here (the caller's gradient array)
  float* ws;  // [n][16]
  int64_t n;
};

constexpr int kBwdVals = 16;

// d(tau, delta^2) -> d(mu, M) for one (ray, particle); p = o - mu compensated as in
// response(), a = M (p - t d), u = M d:  h = a + tau_s u (= w + tau u),
//   gw = 2 dd2 h - dtau u / n2,  gu = 2 dd2 tau h - dtau (w + 2 tau u) / n2,
//   dL/dM = gw p^T + gu d^T,  dL/dmu = -M^T gw.
__device__ __forceinline__ void response_grad(const RayF& r, const float mu[3], const float M[9], float dtau,
                                              float dd2, float g[12]) {
  float ph[3], pl[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float a = r.o_hi[k], b = -mu[k];
    const float s = __fadd_rn(a, b);
    const float bb = __fsub_rn(s, a);
    const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
    ph[k] = s;
    pl[k] = err + r.o_lo[k];
  }
  const float t = ph[0] * r.d_hi[0] + ph[1] * r.d_hi[1] + ph[2] * r.d_hi[2];
  float pp[3], p[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    pp[k] = fmaf(-t, r.d_hi[k], ph[k]) + fmaf(-t, r.d_lo[k], pl[k]);
    p[k] = ph[k] + pl[k];
  }
  float a[3], u[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    a[k] = M[3 * k] * pp[0] + M[3 * k + 1] * pp[1] + M[3 * k + 2] * pp[2];
    u[k] = M[3 * k] * r.d_hi[0] + M[3 * k + 1] * r.d_hi[1] + M[3 * k + 2] * r.d_hi[2];
  }
  const float inv = 1.0f / (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  const float ts = -(a[0] * u[0] + a[1] * u[1] + a[2] * u[2]) * inv;
  const float tau = ts - t;
  float gw[3], gu[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float h = fmaf(ts, u[k], a[k]);
    const float w = fmaf(t, u[k], a[k]);
    gw[k] = 2.f * dd2 * h - dtau * u[k] * inv;
    gu[k] = 2.f * dd2 * tau * h - dtau * fmaf(2.f * tau, u[k], w) * inv;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = -(M[k] * gw[0] + M[3 + k] * gw[1] + M[6 + k] * gw[2]);
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j) g[3 + 3 * k + j] = gw[k] * p[j] + gu[k] * r.d_hi[j];
}

// One lane's ray against one list entry, forward rules: 0 = no contribution, 1 = contributes
// (alpha, tau, rho, clamped filled), 2 = terminates the ray.
__device__ __forceinline__ int bwd_step(const BwdArgs& A, const RayF& rf, const float4 r[4], float T, float* alpha,
                                        float* tau, float* rho, bool* clamped) {
  const float mu[3] = {r[0].x, r[0].y, r[0].z};
  const float M[9] = {r[0].w, r[1].x, r[1].y, r[1].z, r[1].w, r[2].x, r[2].y, r[2].z, r[2].w};
  float d2;
  response(rf, mu, M, tau, &d2);
  *rho = __expf(-0.5f * d2);  // same as the render kernels (__expf)
  const float av = r[3].x * *rho;
  *alpha = fminf(A.alpha_max, av);
  *clamped = !(av < A.alpha_max);
  if (*tau < A.near_tau || *alpha < A.alpha_min) return 0;
  if (T * (1.f - *alpha) < A.T_min) return 2;
  return 1;
}

// Walks the list [rg.x, rg.y) in order for a warp whose lanes hold rays (ray lane r has
// coordinates (ra[r], rb[r]) in shared memory: LiDAR azimuth / elevation, camera pixel
// centre).  32 entries at a time are fetched in parallel (lane = entry: id + 80-byte
// record) and each lane tests its entry against all 32 rays (member(bx, a, b), the A12 box
// test), so entries that hold none of the warp's rays cost nothing further; the others are
// visited in list order with the record broadcast by shuffles.  body(member, id, rec) runs
// on all lanes (it may use warp collectives); the walk ends once every lane is done.
template <typename Member, typename Body>
__device__ __forceinline__ void walk_list(const BwdArgs& A, int2 rg, const bool& done, const float* ra,
                                          const float* rb, float4 (*srec)[5], Member member, Body body) {
  const int lane = threadIdx.x & 31;
  for (int base = rg.x; base < rg.y; base += 32) {
    const uint32_t open = __ballot_sync(0xffffffffu, !done);
    if (open == 0u) return;
    const int i = base + lane;
    uint32_t g = 0, mm = 0;
    float4 q[5] = {};
    __syncwarp();  // the previous batch's records are no longer read
    if (i < rg.y) {
      g = __ldg(A.ids + i);
      SIMULI_CHECK((int64_t)g < A.n, g, A.n);
      const float4* src = A.record + (size_t)g * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) q[c] = __ldg(src + c);
#pragma unroll
      for (int c = 0; c < 4; ++c) srec[lane][c] = q[c];
      for (uint32_t o = open; o; o &= o - 1u) {
        const int r = __ffs(o) - 1;
        mm |= (uint32_t)member(q[4], ra[r], rb[r]) << r;
      }
    }
    __syncwarp();
    uint32_t ent = __ballot_sync(0xffffffffu, mm != 0u);
    while (ent) {
      const int k = __ffs(ent) - 1;
      ent &= ent - 1u;
      const uint32_t mk = __shfl_sync(0xffffffffu, mm, k);  // all lanes (not under a short circuit)
      const uint32_t gk = __shfl_sync(0xffffffffu, g, k);
      const bool m = !done && ((mk >> lane) & 1u);
      if (!__any_sync(0xffffffffu, m)) continue;
      float4 r[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) r[c] = srec[k][c];
      body(m, gk, r);
      if (__all_sync(0xffffffffu, done)) return;
    }
  }
}

// Sum of 16 values over the warp as a reduce-scatter butterfly (16 shuffles instead of
// 5 x 16): afterwards lanes 2i and 2i + 1 hold the total of value i' where i' is lane's
// bits 4..1 read as (8, 4, 2, 1).
__device__ __forceinline__ float warp_reduce16(float v[16], int lane) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool up = lane & 16;
    const float send = up ? v[j] : v[j + 8];
    const float keep = up ? v[j + 8] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool up = lane & 8;
    const float send = up ? v[j] : v[j + 4];
    const float keep = up ? v[j + 4] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool up = lane & 4;
    const float send = up ? v[j] : v[j + 2];
    const float keep = up ? v[j + 2] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const float send = up ? v[0] : v[1];
    const float keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Gradient walk over [rg.x, rg.y) (the whole list, or one segment of it): T starts at T0
// and the prefix sums (Gz.zeta, omega, D) at (pzf, pW, pD) -- 1 and 0 for a whole list, the
// transmittance and sums of the earlier segments otherwise; (tot_f, W, D) are the ray's
// totals.  The forward's decisions are replayed with the running T.
template <typename Member>
__device__ __forceinline__ void bwd_grad_walk(const BwdArgs& A, const RayF& rf, bool live, int2 rg, const float* ra,
                                              const float* rb, float4 (*srec)[5], const float shb[16], Member member,
                                              float T, float pzf, float pW, float pD, float tot_f, float W, float D,
                                              const float Gz[3], float Go, float GD) {
  const int lane = threadIdx.x & 31;
  bool done = !live || T < A.T_min;
  walk_list(A, rg, done, ra, rb, srec, member, [&](bool m, uint32_t g, const float4 r[4]) {
    float v[kBwdVals];
#pragma unroll
    for (int q = 0; q < kBwdVals; ++q) v[q] = 0.f;
    bool contributed = false;
    float wsh = 0.f;  // this lane's weight alpha T (per-ray SH gradient)
    if (m) {
      float alpha, tau, rho;
      bool cl;
      const int st = bwd_step(A, rf, r, T, &alpha, &tau, &rho, &cl);
      if (st == 2) done = true;
      if (st == 1) {
        contributed = true;
        const float w = alpha * T;
        float f[3] = {r[3].y, r[3].z, r[3].w};
        if (A.sh) sh_dot(A.sh + (size_t)g * A.sh_ncoef * 3, A.sh_ncoef, shb, f);
        const float gzf = Gz[0] * f[0] + Gz[1] * f[1] + Gz[2] * f[2];
        pzf = fmaf(w, gzf, pzf);
        pD = fmaf(w, tau, pD);
        pW += w;
        wsh = w;
        const float suf = (tot_f - pzf) + Go * (W - pW) + GD * (D - pD);
        const float dalpha = T * (gzf + Go + GD * tau) - suf / (1.f - alpha);
        const float dtau = GD * w;
        float dd2 = 0.f;
        if (!cl) {
          v[12] = dalpha * rho;
          dd2 = -0.5f * dalpha * alpha;
        }
        const float mu[3] = {r[0].x, r[0].y, r[0].z};
        const float M[9] = {r[0].w, r[1].x, r[1].y, r[1].z, r[1].w, r[2].x, r[2].y, r[2].z, r[2].w};
        float g12[12];
        response_grad(rf, mu, M, dtau, dd2, g12);
#pragma unroll
        for (int q = 0; q < 12; ++q) v[q] = g12[q];
        if (!A.sh) {
          v[13] = Gz[0] * w;
          v[14] = Gz[1] * w;
          v[15] = Gz[2] * w;
        }
        T = T * (1.f - alpha);
      }
    }
    if (__any_sync(0xffffffffu, contributed)) {
      const float tot = warp_reduce16(v, lane);
      const int q = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
      SIMULI_CHECK((int64_t)g < A.n, g, A.n);
      if (!(lane & 1)) atomicAdd(A.ws + (size_t)g * kBwdVals + q, tot);
      if (A.sh) {  // per-ray SH: dL/dc_kc = Y_k(d) Gz_c w, summed over the warp's rays
#pragma unroll 1
        for (int c = 0; c < 3; ++c) {
          float u[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) u[k] = k < A.sh_ncoef ? shb[k] * Gz[c] * wsh : 0.f;
          const float t = warp_reduce16(u, lane);
          if (!(lane & 1) && q < A.sh_ncoef) atomicAdd(A.dsh + ((size_t)g * A.sh_ncoef + q) * 3 + c, t);
        }
      }
    }
  });
}

// Upstream gradients of the decoded outputs -> (Gz, Go, GD) from the ray's totals
template <bool LIDAR>
__device__ __forceinline__ void bwd_fold(const BwdArgs& A, bool live, int ray, float z0, float z1, float z2, float W,
                                         float D, float Gz[3], float* Go_, float* GD_) {
  float Go = 0.f, GD = 0.f;
  Gz[0] = Gz[1] = Gz[2] = 0.f;
  if (live) {
    if (A.g_feat)
#pragma unroll
      for (int c = 0; c < 3; ++c) Gz[c] = __ldg(A.g_feat + 3 * (size_t)ray + c);
    if (A.g_opacity) Go = __ldg(A.g_opacity + ray);
    if (A.g_daccum) GD = __ldg(A.g_daccum + ray);
    if (A.g_depth && W > 0.f) {
      const float gd = __ldg(A.g_depth + ray);
      GD += gd / W;
      Go -= gd * D / (W * W);
    }
    if (LIDAR) {
      if (A.g_intensity) Gz[0] += __ldg(A.g_intensity + ray);
      if (A.g_raydrop) {
        const float beta = raydrop_prob(z1, z2);
        const float gr = __ldg(A.g_raydrop + ray) * beta * (1.f - beta);
        Gz[1] -= gr;
        Gz[2] += gr;
      }
    }
  }
  *Go_ = Go;
  *GD_ = GD;
}

// The two passes of one warp whose lanes hold rays (LiDAR / camera: the same tile) over the
// tile's list; member(bx) is the lane's A12 box test.
template <bool LIDAR, typename Member>
__device__ __forceinline__ void bwd_ray_pair_passes(const BwdArgs& A, const RayF& rf, bool live, int ray,
                                                    int2 rg, const float* ra, const float* rb, float4 (*srec)[5],
                                                    const float shb[16], Member member) {
  const int lane = threadIdx.x & 31;
  // ---- pass 1: totals
  float T = 1.f, z0 = 0.f, z1 = 0.f, z2 = 0.f, D = 0.f, W = 0.f;
  bool done = !live;
  if (A.f_feat) {  // the forward's own totals of this frame
    if (live) {
      z0 = __ldg(A.f_feat + 3 * (size_t)ray);
      z1 = __ldg(A.f_feat + 3 * (size_t)ray + 1);
      z2 = __ldg(A.f_feat + 3 * (size_t)ray + 2);
      W = __ldg(A.f_opacity + ray);
      D = __ldg(A.f_daccum + ray);
    }
  } else walk_list(A, rg, done, ra, rb, srec, member, [&](bool m, uint32_t gid, const float4 r[4]) {
    if (!m) return;
    float alpha, tau, rho;
    bool cl;
    const int st = bwd_step(A, rf, r, T, &alpha, &tau, &rho, &cl);
    if (st == 0) return;
    if (st == 2) {
      done = true;
      return;
    }
    const float w = alpha * T;
    float f[3] = {r[3].y, r[3].z, r[3].w};
    if (A.sh) sh_dot(A.sh + (size_t)gid * A.sh_ncoef * 3, A.sh_ncoef, shb, f);  // as the per-ray forward
    z0 = fmaf(w, f[0], z0);
    z1 = fmaf(w, f[1], z1);
    z2 = fmaf(w, f[2], z2);
    D = fmaf(w, tau, D);
    W += w;
    T = T * (1.f - alpha);
  });
  float Gz[3], Go, GD;
  bwd_fold<LIDAR>(A, live, ray, z0, z1, z2, W, D, Gz, &Go, &GD);
  // ---- pass 2: gradients
  bwd_grad_walk(A, rf, live, rg, ra, rb, srec, shb, member, 1.f, 0.f, 0.f, 0.f, Gz[0] * z0 + Gz[1] * z1 + Gz[2] * z2,
                W, D, Gz, Go, GD);
}

// The rays of one warp, exactly as the render kernels build them.  LiDAR: rays chunk*32 +
// lane of the tile (ra, rb = azimuth, elevation); camera: pixels strip*32 + lane of the TP x TP
// tile (ra, rb = pixel centre).  Returns this lane's liveness; ray = output index.
__device__ __forceinline__ bool lidar_ray_setup(const BwdArgs& A, int tile, int chunk, int lane, RayF& rf,
                                                float shb[16], float* s_a, float* s_b, int& ray) {
  const int off0 = __ldg(A.tile_ray_off + tile), off1 = __ldg(A.tile_ray_off + tile + 1);
  const int k = off0 + chunk * 32 + lane;
  const bool live = k < off1;
  ray = live ? __ldg(A.tile_rays + k) : 0;
  const int b = ray / A.n_az, j = ray % A.n_az;
  const float phi = live ? __ldg(A.ray_az + j) : 0.f, el = live ? __ldg(A.ray_el + (size_t)b * A.n_az) : 0.f;
  double o[3] = {0, 0, 0}, dd[3] = {1, 0, 0};
  if (live) {
    double Rm[9];
    pose_at_d(A.pose, (double)__ldg(A.ray_s + j), Rm, o);
    double sa, ca, se, ce;
    sincos((double)phi, &sa, &ca);
    sincos((double)el, &se, &ce);
    const double u[3] = {ce * ca, ce * sa, se};
#pragma unroll
    for (int i = 0; i < 3; ++i) dd[i] = Rm[3 * i] * u[0] + Rm[3 * i + 1] * u[1] + Rm[3 * i + 2] * u[2];
  }
  split_ray(o, dd, rf);
  if (A.sh) sh_basis3((float)dd[0], (float)dd[1], (float)dd[2], shb);
  __syncwarp();
  s_a[lane] = phi;
  s_b[lane] = el;
  __syncwarp();
  return live;
}

template <int TP>
__device__ __forceinline__ bool camera_ray_setup(const BwdArgs& A, int tile, int strip, int lane, RayF& rf,
                                                 float shb[16], float* s_a, float* s_b, int& ray) {
  const CameraArgs& C = A.cam;
  const int ty = tile / C.Wt, tx = tile % C.Wt;
  const int idx = strip * 32 + lane;
  const int i = tx * TP + (idx % TP), j = ty * TP + (idx / TP);
  const bool inside = i < C.width && j < C.height;
  double o[3] = {0, 0, 0}, d[3] = {0, 0, 0};
  bool valid = false;
  if (inside) {
    double dc[3];
    valid = unproject(C, (double)i + 0.5, (double)j + 0.5, dc);
    const double s = C.rolling ? ((double)j + 0.5) / (double)C.height : 0.0;
    double R[9];
    pose_at_d(C.pose, s, R, o);
    if (valid)
      for (int k = 0; k < 3; ++k) d[k] = R[3 * k] * dc[0] + R[3 * k + 1] * dc[1] + R[3 * k + 2] * dc[2];
  }
  split_ray(o, d, rf);
  if (A.sh) sh_basis3((float)d[0], (float)d[1], (float)d[2], shb);
  ray = inside ? j * C.width + i : 0;
  __syncwarp();
  s_a[lane] = (float)i + 0.5f;
  s_b[lane] = (float)j + 0.5f;
  __syncwarp();
  return inside && valid;
}

struct LidarMember {  // k_render_lidar's column x beam test
  float pi_f, two_pi_f;
  __device__ __forceinline__ bool operator()(const float4 bx, float p, float w) const {
    bool col;
    if (__fsub_rn(bx.y, bx.x) >= two_pi_f) {
      col = true;
    } else {
      const float lo2 = bx.x < -pi_f ? __fadd_rn(bx.x, two_pi_f) : INFINITY;
      const float hi2 = bx.y > pi_f ? __fsub_rn(bx.y, two_pi_f) : -INFINITY;
      col = (bx.x <= p && p <= bx.y) || lo2 <= p || p <= hi2;
    }
    return col && bx.z <= w && w <= bx.w;
  }
};
struct CameraMember {
  __device__ __forceinline__ bool operator()(const float4 bx, float pu, float pv) const {
    return bx.x <= pu && pu <= bx.y && bx.z <= pv && pv <= bx.w;
  }
};

// unsegmented: one warp per (tile, 32 rays) walks the whole list twice (no forward totals)
__global__ void __launch_bounds__(32) k_backward_lidar(const BwdArgs A) {
  const int slot = (int)(blockIdx.x / A.chunks), chunk = (int)(blockIdx.x % A.chunks);
  const int tile = A.order ? __ldg(A.order + slot) : slot;
  __shared__ float s_a[32], s_b[32];
  __shared__ float4 s_rec[32][5];
  RayF rf;
  float shb[16];
  int ray;
  const bool live = lidar_ray_setup(A, tile, chunk, threadIdx.x, rf, shb, s_a, s_b, ray);
  if (__ballot_sync(0xffffffffu, live) == 0u) return;
  bwd_ray_pair_passes<true>(A, rf, live, ray, __ldg(A.ranges + tile), s_a, s_b, s_rec, shb,
                            LidarMember{A.pi_f, A.two_pi_f});
}

template <int TP>
__global__ void __launch_bounds__(32) k_backward_camera(const BwdArgs A) {
  constexpr int STRIPS = TP * TP / 32;
  const int slot = (int)(blockIdx.x / STRIPS), strip = (int)(blockIdx.x % STRIPS);
  const int tile = A.order ? __ldg(A.order + slot) : slot;
  __shared__ float s_a[32], s_b[32];
  __shared__ float4 s_rec[32][5];
  RayF rf;
  float shb[16];
  int ray;
  const bool live = camera_ray_setup<TP>(A, tile, strip, threadIdx.x, rf, shb, s_a, s_b, ray);
  if (__ballot_sync(0xffffffffu, live) == 0u) return;
  bwd_ray_pair_passes<false>(A, rf, live, ray, __ldg(A.ranges + tile), s_a, s_b, s_rec, shb, CameraMember{});
}

// ---------------------------------------------------------------- segmented backward
// With the forward's totals the first pass is not needed, and a long list can be cut into
// segments of kBwdSeg entries walked by different warps: a stats pass gives each
// (segment, ray) its transmittance product and local sums (no termination), and the
// gradient pass of segment s starts from the product / sums of segments 0..s-1 of its tile
// (A31; termination is replayed with the running T: a ray that stopped in an earlier
// segment enters later ones with T < T_min).  Work items (slot, ray group, segment) are
// numbered longest tile first and taken from an atomic counter by persistent warps.
constexpr int kBwdSeg = 512;
constexpr int kBwdGroupsMax = 8;  // ray groups (LiDAR chunks / camera strips) per tile, upper bound

struct SegPlan {  // device scalars at the head of the segment area
  int total, counter_stats, counter_grad, segmented;
};

__global__ void __launch_bounds__(1024) k_bwd_plan(const BwdArgs A, int n_tiles, int groups, int cap_items,
                                                   int* item_off, SegPlan* plan) {
  __shared__ int s_warp[32];
  __shared__ int s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  int seg = 1;
  for (int pass = 0; pass < 2; ++pass) {  // pass 1 only if pass 0 overflowed: one segment per tile
    for (int base = 0; base < n_tiles; base += 1024) {
      const int slot = base + threadIdx.x;
      int items = 0;
      if (slot < n_tiles) {
        const int tile = A.order ? __ldg(A.order + slot) : slot;
        const int2 rg = __ldg(A.ranges + tile);
        const int nseg = seg ? max(1, (rg.y - rg.x + kBwdSeg - 1) / kBwdSeg) : 1;
        items = nseg * groups;
      }
      int incl = items;
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) s_warp[w] = incl;
      __syncthreads();
      int wo = 0;
      for (int k = 0; k < w; ++k) wo += s_warp[k];
      const int carry = s_carry;
      if (slot < n_tiles) item_off[slot] = carry + wo + incl - items;
      __syncthreads();
      if (threadIdx.x == 1023) s_carry = carry + wo + incl;
      __syncthreads();
    }
    if (s_carry <= cap_items || !seg) break;
    seg = 0;
    __syncthreads();
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    item_off[n_tiles] = s_carry;
    plan->total = s_carry;
    plan->counter_stats = 0;
    plan->counter_grad = 0;
    plan->segmented = seg;
  }
}

template <bool LIDAR, int TP, bool STATS>
__global__ void __launch_bounds__(32) k_bwd_seg(const BwdArgs A, int n_tiles, int groups, const int* item_off,
                                                SegPlan* plan, float4* stats) {
  __shared__ float s_a[32], s_b[32];
  __shared__ float4 s_rec[32][5];
  const int lane = threadIdx.x;
  const int total = *reinterpret_cast<volatile int*>(&plan->total);
  const bool segmented = plan->segmented != 0;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(STATS ? &plan->counter_stats : &plan->counter_grad, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= total) return;
    int lo = 0, hi = n_tiles;  // slot: last with item_off[slot] <= item
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(item_off + mid) <= item) lo = mid;
      else hi = mid;
    }
    const int slot = lo, tile = A.order ? __ldg(A.order + slot) : slot;
    const int2 rg = __ldg(A.ranges + tile);
    const int nseg = segmented ? max(1, (rg.y - rg.x + kBwdSeg - 1) / kBwdSeg) : 1;
    const int local = item - __ldg(item_off + slot), group = local / nseg, sgi = local % nseg;
    if (STATS && sgi == nseg - 1) continue;  // the last segment's stats are never read
    RayF rf;
    float shb[16];
    int ray;
    const bool live = LIDAR ? lidar_ray_setup(A, tile, group, lane, rf, shb, s_a, s_b, ray)
                            : camera_ray_setup<TP>(A, tile, group, lane, rf, shb, s_a, s_b, ray);
    if (__ballot_sync(0xffffffffu, live) == 0u) continue;
    const int2 seg = make_int2(rg.x + sgi * kBwdSeg, min(rg.y, rg.x + (sgi + 1) * kBwdSeg));
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, W = 0.f, D = 0.f;
    if (live) {
      z0 = __ldg(A.f_feat + 3 * (size_t)ray);
      z1 = __ldg(A.f_feat + 3 * (size_t)ray + 1);
      z2 = __ldg(A.f_feat + 3 * (size_t)ray + 2);
      W = __ldg(A.f_opacity + ray);
      D = __ldg(A.f_daccum + ray);
    }
    float Gz[3], Go, GD;
    bwd_fold<LIDAR>(A, live, ray, z0, z1, z2, W, D, Gz, &Go, &GD);
    const int base_item = __ldg(item_off + slot) + group * nseg;  // segment 0 of this ray group
    if (STATS) {
      float P = 1.f, Af = 0.f, Wl = 0.f, Dl = 0.f, T = 1.f;
      bool done = !live;
      const auto mem = [&](const float4 bx, float a, float b) {
        if (LIDAR) return LidarMember{A.pi_f, A.two_pi_f}(bx, a, b);
        return CameraMember{}(bx, a, b);
      };
      walk_list(A, seg, done, s_a, s_b, s_rec, mem, [&](bool m, uint32_t g, const float4 r[4]) {
        if (!m) return;
        float alpha, tau, rho;
        bool cl;
        bwd_step(A, rf, r, 1.f, &alpha, &tau, &rho, &cl);  // skip rules only (T = 1: no stop)
        if (tau < A.near_tau || alpha < A.alpha_min) return;
        float f[3] = {r[3].y, r[3].z, r[3].w};
        if (A.sh) sh_dot(A.sh + (size_t)g * A.sh_ncoef * 3, A.sh_ncoef, shb, f);
        const float w = alpha * T;
        Af = fmaf(w, Gz[0] * f[0] + Gz[1] * f[1] + Gz[2] * f[2], Af);
        Wl += w;
        Dl = fmaf(w, tau, Dl);
        T = T * (1.f - alpha);
        P = T;
        // below T_min the ray stops in this segment or earlier: later segments only need
        // T_in < T_min, which any partial product below T_min already guarantees
        if (T < A.T_min) done = true;
      });
      stats[(size_t)item * 32 + lane] = make_float4(P, Af, Wl, Dl);
    } else {
      float T = 1.f, pzf = 0.f, pW = 0.f, pD = 0.f;
      for (int s2 = 0; s2 < sgi; ++s2) {  // earlier segments of this ray group
        const float4 st = stats[(size_t)(base_item + s2) * 32 + lane];
        pzf = fmaf(T, st.y, pzf);
        pW = fmaf(T, st.z, pW);
        pD = fmaf(T, st.w, pD);
        T *= st.x;
      }
      const float tot_f = Gz[0] * z0 + Gz[1] * z1 + Gz[2] * z2;
      if (LIDAR)
        bwd_grad_walk(A, rf, live, seg, s_a, s_b, s_rec, shb, LidarMember{A.pi_f, A.two_pi_f}, T, pzf, pW, pD, tot_f,
                      W, D, Gz, Go, GD);
      else
        bwd_grad_walk(A, rf, live, seg, s_a, s_b, s_rec, shb, CameraMember{}, T, pzf, pW, pD, tot_f, W, D, Gz, Go,
                      GD);
    }
  }
}

// dL/dR (row-major 3x3) -> dL/dq of the unnormalised quaternion q behind R = R(q / |q|) (O1)
__device__ __forceinline__ void rot_grad_to_quat(const float G[9], const float q[4], float inv, float dq_out[4]) {
  const float w = q[0], x = q[1], y = q[2], z = q[3];  // normalised
  const float dq[4] = {
      2.f * (-z * G[1] + y * G[2] + z * G[3] - x * G[5] - y * G[6] + x * G[7]),
      2.f * (y * G[1] + z * G[2] + y * G[3] - 2.f * x * G[4] - w * G[5] + z * G[6] + w * G[7] - 2.f * x * G[8]),
      2.f * (-2.f * y * G[0] + x * G[1] + w * G[2] + x * G[3] + z * G[5] - w * G[6] + z * G[7] - 2.f * y * G[8]),
      2.f * (-2.f * z * G[0] - w * G[1] + x * G[2] + w * G[3] - 2.f * z * G[4] + y * G[5] + x * G[6] + y * G[7])};
  const float dot = dq[0] * w + dq[1] * x + dq[2] * y + dq[3] * z;
#pragma unroll
  for (int c = 0; c < 4; ++c) dq_out[c] = (dq[c] - q[c] * dot) * inv;
}

struct ParamsArgs {
  const float *ws, *means, *quats, *scales, *view_dir;
  const int* actor_id;
  const float* actor_pose;  // [n_actors][7]
  int n_actors, ncoef;
  int per_ray_sh;  // the SH gradient was accumulated by the list walk (A30)
  float beam_div;  // App. C theta (LiDAR), 0 = off
  int64_t n;
};

// parameter chain (O16): M = diag(1/s) R_w^T with R_w = R_a R(q_l^) (R_a = I for static
// particles), mu_w = R_a mu_l + t_a -> (mu_l, q_l, s) and the object poses (atomics into
// out.actor_pose, each particle's share being linear in its own dL/dR_a, dL/dmu_w);
// f = SH(v) -> SH coefficients
__global__ void __launch_bounds__(256) k_backward_params(const ParamsArgs P, simuli_gaussian_grads out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.n) return;
  float v[kBwdVals];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(P.ws) + g * 4 + c);
    v[4 * c] = x.x; v[4 * c + 1] = x.y; v[4 * c + 2] = x.z; v[4 * c + 3] = x.w;
  }
  out.opacity[g] = v[12];
  int a = -1;
  if (P.actor_id) a = __ldg(P.actor_id + g);
  const bool in_range = a >= -1 && a < P.n_actors;
  const float4 q4 = __ldg(reinterpret_cast<const float4*>(P.quats) + g);
  const float qn2 = q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w;
  float gq[4] = {0.f, 0.f, 0.f, 0.f}, gs[3] = {0.f, 0.f, 0.f}, gm[3] = {v[0], v[1], v[2]};
  if (in_range && qn2 > 0.f && isfinite(qn2)) {
    const float inv = rsqrtf(qn2);
    const float q[4] = {q4.x * inv, q4.y * inv, q4.z * inv, q4.w * inv};
    float Rl[9], Ra[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f}, qa[4] = {1.f, 0.f, 0.f, 0.f}, inva = 1.f;
    quat_rot(q, Rl);
    const float* ap = nullptr;
    if (a >= 0) {
      ap = P.actor_pose + 7 * (size_t)a;
      const float qa4[4] = {__ldg(ap), __ldg(ap + 1), __ldg(ap + 2), __ldg(ap + 3)};
      inva = rsqrtf(qa4[0] * qa4[0] + qa4[1] * qa4[1] + qa4[2] * qa4[2] + qa4[3] * qa4[3]);
#pragma unroll
      for (int c = 0; c < 4; ++c) qa[c] = qa4[c] * inva;
      quat_rot(qa, Ra);
    }
    float Rw[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Rw[3 * i + j] = Ra[3 * i] * Rl[j] + Ra[3 * i + 1] * Rl[3 + j] + Ra[3 * i + 2] * Rl[6 + j];
    float G[9];  // dL/dR_w[j][k]
    if (P.beam_div > 0.f) {
      // App. C (A27): M = chol(Sigma_hat)^-1 -> Lbar = -(M^T Mbar M^T) (lower) -> Sigma_bar =
      // sym(M^T Phi(L^T Lbar) M), Phi = lower triangle with the diagonal halved -> dv, dR, ds
      const float vv[3] = {__ldg(P.view_dir + 3 * g), __ldg(P.view_dir + 3 * g + 1), __ldg(P.view_dir + 3 * g + 2)};
      const float t2 = P.beam_div * P.beam_div, r2 = vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2];
      float s2[3], Sh[9];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float sk = __ldg(P.scales + 3 * g + k);
        s2[k] = sk * sk;
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          Sh[3 * i + j] = Rw[3 * i] * s2[0] * Rw[3 * j] + Rw[3 * i + 1] * s2[1] * Rw[3 * j + 1] +
                          Rw[3 * i + 2] * s2[2] * Rw[3 * j + 2] + t2 * ((i == j ? r2 : 0.f) - vv[i] * vv[j]);
      float Lh[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      Lh[0] = sqrtf(Sh[0]);
      Lh[3] = Sh[3] / Lh[0];
      Lh[6] = Sh[6] / Lh[0];
      Lh[4] = sqrtf(Sh[4] - Lh[3] * Lh[3]);
      Lh[7] = (Sh[7] - Lh[6] * Lh[3]) / Lh[4];
      Lh[8] = sqrtf(Sh[8] - Lh[6] * Lh[6] - Lh[7] * Lh[7]);
      float Mh[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // L^-1 (lower)
      Mh[0] = 1.f / Lh[0];
      Mh[4] = 1.f / Lh[4];
      Mh[8] = 1.f / Lh[8];
      Mh[3] = -Lh[3] * Mh[0] * Mh[4];
      Mh[7] = -Lh[7] * Mh[4] * Mh[8];
      Mh[6] = -(Lh[6] * Mh[0] + Lh[7] * Mh[3]) * Mh[8];
      float Lb[9], X[9], Pm[9], S[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          float acc = 0.f;
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) acc += Mh[3 * a + i] * v[3 + 3 * a + b] * Mh[3 * j + b];
          Lb[3 * i + j] = j <= i ? -acc : 0.f;
        }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) X[3 * i + j] = Lh[i] * Lb[j] + Lh[3 + i] * Lb[3 + j] + Lh[6 + i] * Lb[6 + j];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Pm[3 * i + j] = j < i ? X[3 * i + j] : (j == i ? 0.5f * X[3 * i + j] : 0.f);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          float acc = 0.f;
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) acc += Mh[3 * a + i] * Pm[3 * a + b] * Mh[3 * b + j];
          S[3 * i + j] = acc;
        }
      float Sb[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Sb[3 * i + j] = 0.5f * (S[3 * i + j] + S[3 * j + i]);
      const float tr = Sb[0] + Sb[4] + Sb[8];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        v[i] += 2.f * t2 * (tr * vv[i] - (Sb[3 * i] * vv[0] + Sb[3 * i + 1] * vv[1] + Sb[3 * i + 2] * vv[2]));
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
          G[3 * i + k] = 2.f * (Sb[3 * i] * Rw[k] + Sb[3 * i + 1] * Rw[3 + k] + Sb[3 * i + 2] * Rw[6 + k]) * s2[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) acc += Rw[3 * i + k] * Sb[3 * i + j] * Rw[3 * j + k];
        gs[k] = 2.f * __ldg(P.scales + 3 * g + k) * acc;
      }
      if (!isfinite(Lh[8]) || !(Lh[8] > 0.f)) {
#pragma unroll
        for (int q = 0; q < 9; ++q) G[q] = 0.f;
        gs[0] = gs[1] = gs[2] = 0.f;
      }
      gm[0] = v[0]; gm[1] = v[1]; gm[2] = v[2];
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float s = __ldg(P.scales + 3 * g + k);
        float ds = 0.f;
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          const float dm = v[3 + 3 * k + jj];
          G[3 * jj + k] = dm / s;
          ds -= dm * Rw[3 * jj + k] / (s * s);
        }
        gs[k] = ds;
      }
    }
    if (a < 0) {
      rot_grad_to_quat(G, q, inv, gq);
    } else {
      float Gl[9];  // R_a^T G
#pragma unroll
      for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) Gl[3 * i + j] = Ra[i] * G[j] + Ra[3 + i] * G[3 + j] + Ra[6 + i] * G[6 + j];
        gm[i] = Ra[i] * v[0] + Ra[3 + i] * v[1] + Ra[6 + i] * v[2];
      }
      rot_grad_to_quat(Gl, q, inv, gq);
      if (out.actor_pose) {
        const float ml[3] = {__ldg(P.means + 3 * g), __ldg(P.means + 3 * g + 1), __ldg(P.means + 3 * g + 2)};
        float Ga[9];  // G R_l^T + dL/dmu_w mu_l^T
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            Ga[3 * i + j] = G[3 * i] * Rl[3 * j] + G[3 * i + 1] * Rl[3 * j + 1] + G[3 * i + 2] * Rl[3 * j + 2] +
                            v[i] * ml[j];
        float dqa[4];
        rot_grad_to_quat(Ga, qa, inva, dqa);
        float* o = out.actor_pose + 7 * (size_t)a;
        if (dqa[0] != 0.f || dqa[1] != 0.f || dqa[2] != 0.f || dqa[3] != 0.f || v[0] != 0.f || v[1] != 0.f ||
            v[2] != 0.f) {
#pragma unroll
          for (int c = 0; c < 4; ++c) atomicAdd(o + c, dqa[c]);
#pragma unroll
          for (int c = 0; c < 3; ++c) atomicAdd(o + 4 + c, v[c]);
        }
      }
    }
  }
  if (!in_range) gm[0] = gm[1] = gm[2] = 0.f;
  for (int c = 0; c < 3; ++c) out.means[3 * g + c] = gm[c];
  reinterpret_cast<float4*>(out.quats)[g] = make_float4(gq[0], gq[1], gq[2], gq[3]);
  for (int c = 0; c < 3; ++c) out.scales[3 * g + c] = gs[c];
  if (P.per_ray_sh || P.ncoef == 16) return;  // degree 3: k_backward_sh16
  float b[16];
  {
    const float vx = __ldg(P.view_dir + 3 * g), vy = __ldg(P.view_dir + 3 * g + 1), vz = __ldg(P.view_dir + 3 * g + 2);
    const float l2 = vx * vx + vy * vy + vz * vz;
    const float iv = l2 > 0.f ? rsqrtf(l2) : 0.f;
    sh_basis3(vx * iv, vy * iv, vz * iv, b);
  }
  float* o = out.sh + (size_t)g * P.ncoef * 3;
  for (int k = 0; k < P.ncoef; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) o[3 * k + c] = b[k] * v[13 + c];
}

// dL/dSH = Y_k(v) dL/df for degree 3: each thread builds its particle's 48 values in
// shared memory, then the warp stores its 32 particles' 6 KB as coalesced float4 rows
__global__ void __launch_bounds__(256) k_backward_sh16(const float* __restrict__ ws,
                                                       const float* __restrict__ view_dir, int64_t n,
                                                       float* __restrict__ gsh) {
  __shared__ float4 s_rows[256 * 12];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w0 = threadIdx.x & ~31;
  if (g < n) {
    const float vx = __ldg(view_dir + 3 * g), vy = __ldg(view_dir + 3 * g + 1), vz = __ldg(view_dir + 3 * g + 2);
    const float l2 = vx * vx + vy * vy + vz * vz;
    const float iv = l2 > 0.f ? rsqrtf(l2) : 0.f;
    float b[16];
    sh_basis3(vx * iv, vy * iv, vz * iv, b);
    const float df[3] = {__ldg(ws + g * kBwdVals + 13), __ldg(ws + g * kBwdVals + 14), __ldg(ws + g * kBwdVals + 15)};
    float4* row = s_rows + threadIdx.x * 12;
#pragma unroll
    for (int j = 0; j < 12; ++j)  // element q = 4 j + e: coefficient q / 3, channel q % 3
      row[j] = make_float4(b[(4 * j) / 3] * df[(4 * j) % 3], b[(4 * j + 1) / 3] * df[(4 * j + 1) % 3],
                           b[(4 * j + 2) / 3] * df[(4 * j + 2) % 3], b[(4 * j + 3) / 3] * df[(4 * j + 3) % 3]);
  }
  __syncwarp();
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + w0;
  const int np = n - g0 >= 32 ? 32 : (int)(n - g0);
  float4* dst = reinterpret_cast<float4*>(gsh) + g0 * 12;
  const float4* src = s_rows + w0 * 12;
  for (int t = lane; t < np * 12; t += 32) dst[t] = src[t];
}

int32_t bwd_common_checks(const simuli_gaussians* G, const simuli_projected* proj, const uint32_t* ids,
                          const int32_t* ranges, const simuli_project_params* P, const simuli_render_params* rp,
                          const simuli_gaussian_grads* gout, void* ws, size_t ws_bytes, const char* what) {
  if (G && G->n == 0) return SIMULI_OK;  // nothing to differentiate (callers return before any launch)
  if (!(G && proj && proj->record && ids && ranges && P && rp && gout && ws)) {
    set_error("%s: NULL argument", what);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  if (!proj->view_dir) {
    set_error("%s: proj->view_dir was not written (simuli_project with a view_dir buffer)", what);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  if (!(gout->means && gout->quats && gout->scales && gout->opacity && gout->sh)) {
    set_error("%s: NULL gradient output", what);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  if (ws_bytes < (size_t)G->n * kBwdVals * sizeof(float) || reinterpret_cast<uintptr_t>(ws) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(gout->quats) % 16 != 0) {
    set_error("%s: workspace too small / workspace or quats gradient not 16-byte aligned", what);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  if (rp->sh && (reinterpret_cast<uintptr_t>(rp->sh) % 16 != 0 || rp->sh_degree != G->sh_degree)) {
    set_error("%s: per-ray SH must be 16-byte aligned and of the particles' degree", what);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  if (G->actor_id && (G->n_actors < 1 || !G->actor_pose)) {
    set_error("%s: actor_id needs n_actors >= 1 and actor_pose", what);
    return SIMULI_ERR_INVALID_ARGUMENT;
  }
  if (G->sh_degree < 0 || G->sh_degree > 3) {
    set_error("%s: sh_degree not in 0..3", what);
    return SIMULI_ERR_UNSUPPORTED;
  }
  return SIMULI_OK;
}

void bwd_fill_common(BwdArgs& A, const simuli_projected* proj, const uint32_t* ids, const int32_t* ranges,
                     const simuli_project_params* P, const simuli_render_params* rp, void* ws, int64_t n) {
  A.n = n;
  A.record = reinterpret_cast<const float4*>(proj->record);
  A.ids = ids;
  A.ranges = reinterpret_cast<const int2*>(ranges);
  A.pose = make_pose_interp_d(P->pose_start, P->pose_end);
  A.alpha_min = rp->alpha_min; A.alpha_max = rp->alpha_max; A.T_min = rp->T_min;
  A.ws = static_cast<float*>(ws);
  if (rp->sh) {
    A.sh = rp->sh;
    A.sh_ncoef = (rp->sh_degree + 1) * (rp->sh_degree + 1);
  }
}

int32_t bwd_params(const simuli_gaussians* G, const simuli_projected* proj, const simuli_gaussian_grads* gout,
                   const float* ws, bool per_ray_sh, float beam_div, cudaStream_t st, const char* what) {
  ParamsArgs P{};
  P.per_ray_sh = per_ray_sh ? 1 : 0;
  P.beam_div = beam_div;
  P.ws = ws; P.means = G->means; P.quats = G->quats; P.scales = G->scales; P.view_dir = proj->view_dir;
  P.ncoef = (G->sh_degree + 1) * (G->sh_degree + 1);
  P.n = G->n;
  simuli_gaussian_grads o = *gout;
  if (G->actor_id) {
    P.actor_id = G->actor_id;
    P.actor_pose = reinterpret_cast<const float*>(G->actor_pose);
    P.n_actors = G->n_actors;
    if (o.actor_pose) cudaMemsetAsync(o.actor_pose, 0, sizeof(float) * 7 * (size_t)G->n_actors, st);
  } else {
    o.actor_pose = nullptr;
  }
  if (G->n > 0) {
    k_backward_params<<<(unsigned)((G->n + 255) / 256), 256, 0, st>>>(P, o);
    if (!per_ray_sh && P.ncoef == 16)
      k_backward_sh16<<<(unsigned)((G->n + 255) / 256), 256, 0, st>>>(ws, proj->view_dir, G->n, o.sh);
  }
  return launch_check(what);
}

}  // namespace
}  // namespace simuli

namespace simuli {
namespace {
// segment area of the backward workspace, after the n x 16 gradient floats:
// SegPlan | item_off [n_tiles + 1] (16-byte padded) | stats [items][32] float4
size_t seg_area_fixed(int32_t n_tiles) { return 16 + (((size_t)n_tiles + 1) * 4 + 15) / 16 * 16; }

// runs the segmented walk if the forward totals are given and the workspace holds at least
// one item per (tile, ray group); returns false to use the unsegmented kernels
template <bool LIDAR, int TP>
bool launch_segmented(BwdArgs A, int32_t n_tiles, int groups, int64_t n, void* workspace, size_t workspace_bytes,
                      cudaStream_t st) {
  if (!A.f_feat) return false;
  const size_t head = (size_t)n * kBwdVals * sizeof(float);
  if (workspace_bytes < head + seg_area_fixed(n_tiles)) return false;
  const size_t cap = (workspace_bytes - head - seg_area_fixed(n_tiles)) / (32 * sizeof(float4));
  if (cap < (size_t)n_tiles * groups) return false;
  char* area = static_cast<char*>(workspace) + head;
  SegPlan* plan = reinterpret_cast<SegPlan*>(area);
  int* item_off = reinterpret_cast<int*>(area + 16);
  float4* stats = reinterpret_cast<float4*>(area + seg_area_fixed(n_tiles));
  const int cap_items = cap > (size_t)INT32_MAX ? INT32_MAX : (int)cap;
  k_bwd_plan<<<1, 1024, 0, st>>>(A, n_tiles, groups, cap_items, item_off, plan);
  const unsigned grid = 148 * 32;  // persistent warps, a full device
  k_bwd_seg<LIDAR, TP, true><<<grid, 32, 0, st>>>(A, n_tiles, groups, item_off, plan, stats);
  k_bwd_seg<LIDAR, TP, false><<<grid, 32, 0, st>>>(A, n_tiles, groups, item_off, plan, stats);
  return true;
}
}  // namespace
}  // namespace simuli

extern "C" int32_t simuli_backward_workspace_size(int64_t n, int64_t pair_capacity, int32_t n_tiles, size_t* bytes) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(n >= 0 && pair_capacity >= 0 && n_tiles >= 0 && bytes, "simuli_backward_workspace_size: bad argument");
  const size_t items = ((size_t)n_tiles + (size_t)pair_capacity / kBwdSeg + 1) * kBwdGroupsMax;
  *bytes = (size_t)n * kBwdVals * sizeof(float) + seg_area_fixed(n_tiles) + items * 32 * sizeof(float4);
  return SIMULI_OK;
}

extern "C" int32_t simuli_backward_lidar(const simuli_gaussians* G, const simuli_projected* proj,
                                         const uint32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order,
                                         const simuli_project_params* P, const simuli_render_params* rp,
                                         const simuli_lidar_grad_in* gin, simuli_gaussian_grads* gout,
                                         void* workspace, size_t workspace_bytes, void* stream) {
  using namespace simuli;
  clear_error();
  const int32_t rc = bwd_common_checks(G, proj, sorted_ids, tile_ranges, P, rp, gout, workspace, workspace_bytes,
                                       "simuli_backward_lidar");
  if (rc != SIMULI_OK || G->n == 0) return rc;
  SIMULI_REQUIRE(gin, "simuli_backward_lidar: NULL grad_in");
  SIMULI_REQUIRE(P->kind == SIMULI_SENSOR_LIDAR && P->lidar && P->tiling, "simuli_backward_lidar: needs LiDAR params");

  const simuli_tiling_dev& T = *P->tiling;
  SIMULI_REQUIRE(T.tile_ray_offsets && T.tile_rays && T.ray_az && T.ray_el && T.ray_s && T.n_tiles >= 1,
                 "simuli_backward_lidar: incomplete device tiling");
  BwdArgs A{};
  bwd_fill_common(A, proj, sorted_ids, tile_ranges, P, rp, workspace, G->n);
  A.order = tile_order;
  A.tile_ray_off = T.tile_ray_offsets; A.tile_rays = T.tile_rays;
  A.ray_az = T.ray_az; A.ray_el = T.ray_el; A.ray_s = T.ray_s;
  A.n_az = T.n_azimuth;
  A.chunks = (T.max_rays_in_tile + 31) / 32;
  A.pi_f = T.pi_f; A.two_pi_f = T.two_pi_f;
  A.near_tau = P->lidar->min_range_m;
  A.g_feat = gin->zeta; A.g_opacity = gin->opacity; A.g_daccum = gin->depth_accum; A.g_depth = gin->depth;
  A.g_intensity = gin->intensity; A.g_raydrop = gin->raydrop;
  if (gin->fwd_zeta && gin->fwd_opacity && gin->fwd_depth_accum) {
    A.f_feat = gin->fwd_zeta; A.f_opacity = gin->fwd_opacity; A.f_daccum = gin->fwd_depth_accum;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (G->n == 0) return SIMULI_OK;
  cudaMemsetAsync(workspace, 0, (size_t)G->n * kBwdVals * sizeof(float), st);
  if (A.sh) {
    A.dsh = gout->sh;
    cudaMemsetAsync(gout->sh, 0, sizeof(float) * 3 * A.sh_ncoef * (size_t)G->n, st);
  }
  if (!launch_segmented<true, 16>(A, T.n_tiles, A.chunks, G->n, workspace, workspace_bytes, st))
    k_backward_lidar<<<(unsigned)(T.n_tiles * A.chunks), 32, 0, st>>>(A);
  const int32_t lc = launch_check("simuli_backward_lidar");
  if (lc != SIMULI_OK) return lc;
  return bwd_params(G, proj, gout, static_cast<const float*>(workspace), A.sh != nullptr,
                    P->lidar->beam_divergence_rad, st, "simuli_backward_lidar (params)");
}

extern "C" int32_t simuli_backward_camera(const simuli_gaussians* G, const simuli_projected* proj,
                                          const uint32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order,
                                          const simuli_project_params* P, const simuli_render_params* rp,
                                          const simuli_camera_grad_in* gin, simuli_gaussian_grads* gout,
                                          void* workspace, size_t workspace_bytes, void* stream) {
  using namespace simuli;
  clear_error();
  const int32_t rc = bwd_common_checks(G, proj, sorted_ids, tile_ranges, P, rp, gout, workspace, workspace_bytes,
                                       "simuli_backward_camera");
  if (rc != SIMULI_OK || G->n == 0) return rc;
  SIMULI_REQUIRE(gin, "simuli_backward_camera: NULL grad_in");
  SIMULI_REQUIRE(P->kind == SIMULI_SENSOR_CAMERA && P->camera, "simuli_backward_camera: needs camera params");
  const simuli_camera& C = *P->camera;
  if (C.tile_px != 8 && C.tile_px != 16) {
    set_error("simuli_backward_camera: tile_px %d not supported (8 or 16)", C.tile_px);
    return SIMULI_ERR_UNSUPPORTED;
  }
  BwdArgs A{};
  bwd_fill_common(A, proj, sorted_ids, tile_ranges, P, rp, workspace, G->n);
  A.order = tile_order;
  CameraArgs& K = A.cam;
  K.model = C.model; K.width = C.width; K.height = C.height; K.rolling = C.rolling_shutter; K.tile_px = C.tile_px;
  K.Wt = (C.width + C.tile_px - 1) / C.tile_px;
  K.fx = C.fx; K.fy = C.fy; K.cx = C.cx; K.cy = C.cy;
  for (int i = 0; i < 5; ++i) K.k[i] = C.k[i];
  K.max_theta = C.max_theta_rad;
  K.pose = A.pose;
  A.near_tau = C.near_m;
  A.g_feat = gin->rgb; A.g_opacity = gin->opacity; A.g_daccum = gin->depth_accum; A.g_depth = gin->depth;
  if (gin->fwd_rgb && gin->fwd_opacity && gin->fwd_depth_accum) {
    A.f_feat = gin->fwd_rgb; A.f_opacity = gin->fwd_opacity; A.f_daccum = gin->fwd_depth_accum;
  }
  const int Ht = (C.height + C.tile_px - 1) / C.tile_px;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (G->n == 0) return SIMULI_OK;
  cudaMemsetAsync(workspace, 0, (size_t)G->n * kBwdVals * sizeof(float), st);
  if (A.sh) {
    A.dsh = gout->sh;
    cudaMemsetAsync(gout->sh, 0, sizeof(float) * 3 * A.sh_ncoef * (size_t)G->n, st);
  }
  const unsigned tiles = (unsigned)(K.Wt * Ht);
  // camera: the unsegmented walk (its rays stop early behind opaque surfaces, which a
  // segment's stats pass cannot know; config D: 2.42 ms unsegmented vs 2.88 ms segmented)
  if (C.tile_px == 8) k_backward_camera<8><<<tiles * 2, 32, 0, st>>>(A);
  else k_backward_camera<16><<<tiles * 8, 32, 0, st>>>(A);
  const int32_t lc = launch_check("simuli_backward_camera");
  if (lc != SIMULI_OK) return lc;
  return bwd_params(G, proj, gout, static_cast<const float*>(workspace), A.sh != nullptr, 0.f, st,
                    "simuli_backward_camera (params)");
}
