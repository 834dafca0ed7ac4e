// simuli_render_lidar / simuli_render_camera: per-ray front-to-back compositing (sm_100a).
//
// Eq. 1: c_f = sum f_i alpha_i T_i, omega = sum alpha_i T_i,
// alpha_i = sigma_i rho_i(o + tau_max d), T_i = prod_{j<i} (1 - alpha_j); the 3D response
// at tau_max; LiDAR features zeta -> intensity gamma = zeta_0 and ray drop
// softmax(zeta_1, zeta_2).  A listed particle contributes to a ray only if its box
// contains the ray (A12), which makes the result independent of tiling and culling.
//
// LiDAR (k_render_lidar): one CTA per work item = (tile, beam group, column group) of <= 32
// rays, items scheduled longest-list-first.  Warp-specialised pipeline over rounds of
// E = 32 NP list entries (NP = 4 producer warps, one consumer warp):
//  * producers (NP warps, thread = list entry): the round's 80-byte records arrive by
//    cp.async, issued STAGES - 1 rounds ahead (a ring of record stages); each entry's
//    exact A12 ray mask, factorised as (columns inside the azimuth interval) x (beams inside
//    the elevation interval); a 32x32 bit transpose gives every ray its member entries; the
//    member pairs are compacted and their responses (alpha, tau) computed with every lane
//    busy, written ray-major (slot k of ray r = the k-th member of r in list order; E slots
//    per ray, so no member ever overflows);
//  * consumer (one warp, lane = ray): streams its ray's slots front to back -- first the
//    transmittance chain, then the weighted sums -- and reports terminated rays, whose
//    member pairs the producers skip from then on; the item ends once every ray has
//    terminated.
// The per-ray arithmetic (order and operands) does not depend on the tiling, on culling or
// on the round structure, so results are bit-identical across (N_phi, M) and culling on/off.
// Rays are generated in double (pose at the column's firing time) and split into float
// hi / lo parts for the compensated response (common.cuh).
// Camera (k_render_camera): one CTA per (16x16 tile, band of 4 pixel rows) -- a tile's four
// bands share its list, so the long near-field lists are spread over four CTAs -- items
// longest-list-first, pixel per thread, 128-record batches in shared memory; each warp
// ballots which entries overlap its 2 x 16 pixel strip and walks only those; CTA-wide early
// exit.  Config D (1920x1080 fisheye, 2M particles) render: 2.31 ms (one 256-thread CTA per
// tile) -> 2.01 (strip pre-cull) -> 1.08 (4 bands; 8 bands: 1.15).  Pixel rays by the inverse
// lens model in double.
#include <cstdint>
#include <cstdlib>
#include <string>

#include "abi_util.h"
#include "common.cuh"

namespace simuli {
namespace {

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

// One CTA per (tile, band of TP / SPLIT pixel rows): the bands of a tile read the same list,
// so a long list (near-field particles covering many pixels) is spread over SPLIT CTAs
// instead of one; items are scheduled longest list first (tile_order).
template <int TP, int SPLIT, bool PRAY>
__global__ void __launch_bounds__(TP* TP / SPLIT) k_render_camera(const CameraArgs A) {
  constexpr int NTH = TP * TP / SPLIT;  // threads = pixels of the band
  constexpr int NT = 128;               // list entries staged per batch
  __shared__ float4 s_rec[NT][5];
  __shared__ uint32_t s_id[PRAY ? NT : 1];  // particle ids of the batch (per-ray SH)
  const int tid = threadIdx.x;
  const int slot = (int)(blockIdx.x / SPLIT), band = (int)(blockIdx.x % SPLIT);
  const int tile = A.order ? __ldg(A.order + slot) : slot;
  const int ty = tile / A.Wt, tx = tile % A.Wt;
  const int i = tx * TP + (tid % TP), j = ty * TP + band * (TP / SPLIT) + (tid / TP);
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
  float shb[16];
  if (PRAY) sh_basis3((float)d[0], (float)d[1], (float)d[2], shb);
  float T = 1.f, acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, D = 0.f, W = 0.f;
  int nc = 0, nv = 0, ni = 0, term_at = -1;
  bool done = !(inside && valid);
  const int2 rg = __ldg(A.ranges + tile);
  for (int b = rg.x; b < rg.y; b += NT) {
    if (__syncthreads_count(!done) == 0) break;
    const int nb = min(NT, rg.y - b);
    for (int e = tid; e < nb; e += NTH) {
      const uint32_t g = __ldg(A.ids + b + e);
      const float4* src = A.record + (size_t)g * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) s_rec[e][c] = __ldg(src + c);
      if (PRAY) s_id[e] = g;
    }
    __syncthreads();
    // warp-level pre-cull: the warp's pixels form a strip of 32 / TP rows x TP columns; an
    // entry whose box misses the strip's pixel-centre rectangle cannot contain any of them,
    // so the warp walks only the entries that overlap it (ballots over the batch, in order)
    const int lane = tid & 31;
    const float su0 = (float)(tx * TP) + 0.5f, su1 = (float)(tx * TP + TP - 1) + 0.5f;
    const int row0 = ty * TP + band * (TP / SPLIT) + (tid - lane) / TP;
    const float sv0 = (float)row0 + 0.5f, sv1 = (float)(row0 + 32 / TP - 1) + 0.5f;
    const bool warp_live = __any_sync(0xffffffffu, !done);
    if (warp_live) {
      for (int k0 = 0; k0 < nb; k0 += 32) {
        const int jl = k0 + lane;
        bool ov = false;
        if (jl < nb) {
          const float4 bx = s_rec[jl][4];
          ov = bx.x <= su1 && su0 <= bx.y && bx.z <= sv1 && sv0 <= bx.w;
        }
        uint32_t mask = __ballot_sync(0xffffffffu, ov);
        while (mask) {
          const int jj = k0 + __ffs(mask) - 1;
          mask &= mask - 1u;
          if (done) continue;
          const float4 bx = s_rec[jj][4];
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
            term_at = b - rg.x + jj;
            continue;
          }
          const float w = alpha * T;
          float f[3] = {r3.y, r3.z, r3.w};
          if (PRAY) sh_dot(A.sh + (size_t)s_id[jj] * A.sh_ncoef * 3, A.sh_ncoef, shb, f);
          acc0 = fmaf(w, f[0], acc0);
          acc1 = fmaf(w, f[1], acc1);
          acc2 = fmaf(w, f[2], acc2);
          D = fmaf(w, tau, D);
          W += w;
          ++nc;
          T = Tn;
        }
      }
    }
    __syncthreads();
  }
  // entries visited: up to and including the terminating one, else the whole list
  nv = (inside && valid) ? (term_at >= 0 ? term_at + 1 : rg.y - rg.x) : 0;
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


// ------------------------------------------------------------------ LiDAR
struct LidarArgs {
  const float4* record;
  const uint32_t* ids;
  const int2* ranges;
  const int* order;
  const int *etb_off, *etb, *atc_off, *atc;
  const float *ray_az, *ray_el, *ray_s;
  int n_theta, n_az, items_per_tile, cg, bg, n_cg;
  int64_t n_items;
  PoseInterpD pose;
  float pi_f, two_pi_f, near_tau, alpha_min, alpha_max, T_min;
  float *zeta, *opacity, *depth_accum, *depth, *intensity, *raydrop, *final_T;
  int* n_contrib;
  double* ray_od;
  int *n_visited, *n_inbox;
  const float* sh;  // per-ray SH (A30) or NULL
  int sh_ncoef;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 32x32 bit-matrix transpose across a warp: in: lane i holds row i; out: lane r holds
// the word whose bit e is bit r of row e (5-stage shuffle butterfly).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t lm[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~lm[s]) | ((y & ~lm[s]) >> j)) : ((x & lm[s]) | ((y & lm[s]) << j));
  }
  return x;
}

template <int NP, int STAGES, int SLOTB>
struct LidarSmem {
  float4 rec[STAGES][32 * NP][5];  // record ring (cp.async, STAGES - 1 rounds ahead)
  // ray-major slots, rows padded so that the consumer's lane-per-ray accesses (lane r reads
  // row r) hit distinct banks: without the pad every row starts in the same bank and each
  // consumer load / store was a 32-way conflict
  float2 at[SLOTB][32][32 * NP + 1];   // (alpha, tau) of member pairs, per slot buffer
  uint8_t ent[SLOTB][32][32 * NP + 4]; // entry index within the round
  float4 feat[SLOTB][32 * NP];     // (sigma, features) of the round's entries
  uint32_t pid[SLOTB][32 * NP];    // particle ids of the round's entries (per-ray SH)
  uint32_t memb[SLOTB][NP][32];    // [warp][ray] member entries of the warp's 32
  int rowoff[NP][32];              // members of ray r in warps before w (current round)
  uint16_t plist[NP][1024];        // the warp's member pairs (entry << 5 | ray)
  float ray_oh[32][3], ray_ol[32][3], ray_dh[32][3], ray_dl[32][3];
  float col_phi[32], beam_el[32];
  int col_id[32], beam_id[32];
  int stop_at[2];
  uint32_t done_mask[2];  // rays terminated by the end of the round that released buffer b
};

#ifdef SIMULI_RENDER_PROFILE
__device__ long long g_render_prof[1 << 20];  // per item: start ns, end ns, rounds run, list length | smid << 32
__device__ long long g_render_trace[64][16];  // item traced: clock64 marks per round (see RMARK)
__device__ int g_render_trace_item;
#define RMARK(r, k)                                                                                  \
  do {                                                                                               \
    if (blockIdx.x == (unsigned)g_render_trace_item && (r) < 64 && (threadIdx.x & 31) == 0) g_render_trace[(r)][(k)] = clock64(); \
  } while (0)
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define RMARK(r, k) \
  do {              \
  } while (0)
#endif

// LiDAR pipeline shape: 4 producer warps (128 list entries per round), 2 record stages, one
// slot buffer (~69 KB shared memory, 3 CTAs per SM).  Render-only means over 10 poses of the
// B-batch trajectory, L2 flushed (NP, stages, slot buffers):
//   config B: (4,2,1) 260 us [252-275], (3,2,1) 254 [215-305], (2,2,2) 266 [211-324],
//             (2,2,1) 296, (2,3,1) 295, (4,2,2) 298;
//   config C: (4,2,1) 489 us, (3,2,1) 554, (2,2,2) 664.
// Fewer, larger rounds keep the long near-field lists off the critical path.
constexpr int kLidarNP = 4, kLidarStages = 2, kLidarSlotBuffers = 1;

// SLOTB = 2: double-buffered slots, producers up to two rounds ahead of the consumer;
// SLOTB = 1: one slot buffer (less shared memory, more CTAs per SM), producers wait for the
// consumer's previous round after their box tests, before writing the slots.
template <int NP, int STAGES, int SLOTB, bool PRAY>
__global__ void __launch_bounds__(32 * (NP + 1), 1) k_render_lidar(const LidarArgs A) {
  constexpr int E = 32 * NP;
  constexpr int NT = 32 * (NP + 1);
  constexpr int BAR_PROD = 1, BAR_FULL = 2, BAR_EMPTY = 4, BAR_RAYS = 6;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LidarSmem<NP, STAGES, SLOTB>& S = *reinterpret_cast<LidarSmem<NP, STAGES, SLOTB>*>(smem_raw);
  // per-ray SH (A30), degree 3: the round's member entries' 192-byte coefficient blocks,
  // staged by the producers after the box tests (one slot buffer: written only once the
  // consumer has released the previous round)
  static_assert(!PRAY || SLOTB == 1, "per-ray SH staging assumes one slot buffer");
  float4* s_sh = reinterpret_cast<float4*>(smem_raw + sizeof(LidarSmem<NP, STAGES, SLOTB>));
  const bool sh_smem = PRAY && A.sh_ncoef == 16;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef SIMULI_RENDER_PROFILE
  const long long t_start = gtime();
  int rounds_run = 0;
#endif
  const int64_t item = blockIdx.x;
  const int tslot = (int)(item / A.items_per_tile), sub = (int)(item % A.items_per_tile);
  const int tile = A.order ? __ldg(A.order + tslot) : tslot;
  const int et = tile / A.n_theta, at_ = tile % A.n_theta;
  const int bgi = sub / A.n_cg, cgi = sub % A.n_cg;
  const int b0 = __ldg(A.etb_off + et) + bgi * A.bg, b1 = min(__ldg(A.etb_off + et + 1), b0 + A.bg);
  const int c0 = __ldg(A.atc_off + at_) + cgi * A.cg, c1 = min(__ldg(A.atc_off + at_ + 1), c0 + A.cg);
  const int nb = b1 - b0, nc = c1 - c0;
  if (nb <= 0 || nc <= 0) return;  // CTA-uniform
  const int R = nb * nc;
  if (tid < nc) {
    const int j = __ldg(A.atc + c0 + tid);
    S.col_id[tid] = j;
    S.col_phi[tid] = __ldg(A.ray_az + j);
  }
  if (tid >= 32 && tid < 32 + nb) {
    const int b = __ldg(A.etb + b0 + tid - 32);
    S.beam_id[tid - 32] = b;
    S.beam_el[tid - 32] = __ldg(A.ray_el + (size_t)b * A.n_az);
  }
  if (tid < 2) S.stop_at[tid] = 0;
  __syncthreads();
  const int2 rg = __ldg(A.ranges + tile);
  const int n_rounds = (rg.y - rg.x + E - 1) / E;

  if (warp == NP) {
    // ================= consumer: lane = ray
    int ray = 0;
    double o[3] = {0, 0, 0}, dd[3] = {1, 0, 0};
    RayF rf;
    if (lane < R) {
      const int bi = lane / nc, ci = lane % nc;
      const int j = S.col_id[ci];
      ray = S.beam_id[bi] * A.n_az + j;
      double Rm[9];
      pose_at_d(A.pose, (double)__ldg(A.ray_s + j), Rm, o);
      double sa, ca, se, ce;
      sincos((double)S.col_phi[ci], &sa, &ca);
      sincos((double)S.beam_el[bi], &se, &ce);
      const double u[3] = {ce * ca, ce * sa, se};
#pragma unroll
      for (int i = 0; i < 3; ++i) dd[i] = Rm[3 * i] * u[0] + Rm[3 * i + 1] * u[1] + Rm[3 * i + 2] * u[2];
    }
    split_ray(o, dd, rf);
    if (lane < R) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        S.ray_oh[lane][i] = rf.o_hi[i];
        S.ray_ol[lane][i] = rf.o_lo[i];
        S.ray_dh[lane][i] = rf.d_hi[i];
        S.ray_dl[lane][i] = rf.d_lo[i];
      }
    }
    __threadfence_block();
    named_arrive(BAR_RAYS, NT);
    float shb[16];
    if (PRAY) sh_basis3((float)dd[0], (float)dd[1], (float)dd[2], shb);
    float T = 1.f, acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, D = 0.f, W = 0.f;
    int ncontrib = 0, nv = 0, ni = 0;
    bool done = lane >= R;
    for (int r = 0; r < n_rounds; ++r) {
      const int b = r & 1, sb = SLOTB == 2 ? b : 0;
      RMARK(r, 8);
      named_sync(BAR_FULL + b, NT);
      RMARK(r, 9);
      const int start = rg.x + r * E;
      if (!done) {
        const int n_in = min(E, rg.y - start);
        int cnt = 0;
#pragma unroll
        for (int w = 0; w < NP; ++w) cnt += __popc(S.memb[sb][w][lane]);
        bool stopped = false;
        // one pass over the ray's slots in list order; the slot loads run two members ahead
        // and the feature load (indexed by the entry) one ahead, off the transmittance chain
        int stop_k = -1, stop_e = 0;
        if (cnt > 0) {
          float2 a1 = S.at[sb][lane][0], a2 = make_float2(0.f, 0.f);
          int e1 = S.ent[sb][lane][0], e2 = 0;
          if (cnt > 1) {
            a2 = S.at[sb][lane][1];
            e2 = S.ent[sb][lane][1];
          }
          float4 f1 = S.feat[sb][e1];
          for (int k = 0; k < cnt; ++k) {
            const float2 a = a1;
            const float4 f = f1;
            const int e = e1;
            a1 = a2;
            e1 = e2;
            if (k + 2 < cnt) {
              a2 = S.at[sb][lane][k + 2];
              e2 = S.ent[sb][lane][k + 2];
            }
            if (k + 1 < cnt) f1 = S.feat[sb][e1];
            if (a.y < A.near_tau || a.x < A.alpha_min) continue;  // skipped member
            const float Tn = T * (1.f - a.x);
            if (Tn < A.T_min) {  // terminated: this member is not composited (A14)
              stop_k = k;
              stop_e = e;
              break;
            }
            const float w = a.x * T;
            float fv[3] = {f.y, f.z, f.w};
            if (PRAY) {
              if (sh_smem) sh_dot16(s_sh + e * 12, shb, fv);
              else sh_dot(A.sh + (size_t)S.pid[sb][e] * A.sh_ncoef * 3, A.sh_ncoef, shb, fv);
            }
            acc0 = fmaf(w, fv[0], acc0);
            acc1 = fmaf(w, fv[1], acc1);
            acc2 = fmaf(w, fv[2], acc2);
            D = fmaf(w, a.y, D);
            W += w;
            ++ncontrib;
            T = Tn;
          }
        }
        RMARK(r, 10);
        if (stop_k >= 0) {
          stopped = true;
          nv += stop_e + 1;
          ni += stop_k + 1;
        }
        if (stopped) done = true;
        else {
          nv += n_in;
          ni += cnt;
        }
      }
      const uint32_t dmask = __ballot_sync(0xffffffffu, done);
      const bool all = dmask == 0xffffffffu;
      RMARK(r, 11);
#ifdef SIMULI_RENDER_PROFILE
      rounds_run = r + 1;
#endif
      if (r + SLOTB < n_rounds) {
        if (lane == 0) {
          S.stop_at[b] = all ? 1 : 0;
          S.done_mask[b] = dmask;
        }
        __threadfence_block();
        named_arrive(BAR_EMPTY + b, NT);
      }
      if (all) {
        if (SLOTB == 2 && r + 1 < n_rounds) named_sync(BAR_FULL + (b ^ 1), NT);  // drain the round in flight
        break;
      }
    }
#ifdef SIMULI_RENDER_PROFILE
    if (lane == 0 && item < (1 << 18)) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_render_prof[4 * item] = t_start;
      g_render_prof[4 * item + 1] = gtime();
      g_render_prof[4 * item + 2] = rounds_run;
      g_render_prof[4 * item + 3] = (long long)(rg.y - rg.x) | ((long long)smid << 32);
    }
#endif
    if (lane >= R) return;
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
    if (A.n_contrib) A.n_contrib[ray] = ncontrib;
    if (A.n_visited) A.n_visited[ray] = nv;
    if (A.n_inbox) A.n_inbox[ray] = ni;
    if (A.ray_od) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        A.ray_od[6 * (size_t)ray + i] = o[i];
        A.ray_od[6 * (size_t)ray + 3 + i] = dd[i];
      }
    }
    return;
  }

  // ================= producers: thread = list entry of the round
  constexpr int D = STAGES - 1;  // record prefetch distance (rounds)
  auto issue = [&](int round, uint32_t id) {
    if (round < n_rounds && rg.x + round * E + tid < rg.y) {
      const float4* src = A.record + (size_t)id * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) cp_async16(&S.rec[round % STAGES][tid][c], src + c);
    }
    cp_async_commit();  // one group per round, empty or not (keeps the wait_group count exact)
  };
  auto load_id = [&](int round) -> uint32_t {
    const int e = rg.x + round * E + tid;
    return (round < n_rounds && e < rg.y) ? __ldg(A.ids + e) : 0u;
  };
  {
    uint32_t ids[D];
#pragma unroll
    for (int q = 0; q < D; ++q) ids[q] = load_id(q);
#pragma unroll
    for (int q = 0; q < D; ++q) issue(q, ids[q]);
  }
  uint32_t id_pf = load_id(D);
  // the item's first 8 column azimuths / 4 beam elevations in registers (the usual item;
  // unused slots are masked by nc / nb below)
  float cphi[8], bel[4];
#pragma unroll
  for (int ci = 0; ci < 8; ++ci) cphi[ci] = S.col_phi[ci];
#pragma unroll
  for (int bi = 0; bi < 4; ++bi) bel[bi] = S.beam_el[bi];
  named_sync(BAR_RAYS, NT);
  uint32_t alive = 0xffffffffu;  // rays the consumer has not terminated (2 rounds behind)
  for (int r = 0; r < n_rounds; ++r) {
    const int b = r & 1, st = r % STAGES, sb = SLOTB == 2 ? b : 0;
    if (warp == 0) RMARK(r, 0);
    if (SLOTB == 2 && r >= 2) {
      named_sync(BAR_EMPTY + b, NT);
      if (S.stop_at[b]) break;
      alive = ~S.done_mask[b];
    }
    const int start = rg.x + r * E;
    cp_async_wait<D - 1>();   // this thread's copies of round r have landed
    if (warp == 0) RMARK(r, 1);
    named_sync(BAR_PROD, E);  // everyone's: round r's records visible; stage of round r - 1 and rowoff free
    if (warp == 0) RMARK(r, 2);
    issue(r + D, id_pf);
    id_pf = load_id(r + D + 1);
    const bool valid = start + tid < rg.y;
    uint32_t m = 0;
    if (valid) {
      const float4 bx = S.rec[st][tid][4];
      uint32_t colbits = 0;
      if (__fsub_rn(bx.y, bx.x) >= A.two_pi_f) {
        colbits = (nc == 32) ? 0xffffffffu : ((1u << nc) - 1u);
      } else {
        const float lo2 = bx.x < -A.pi_f ? __fadd_rn(bx.x, A.two_pi_f) : INFINITY;
        const float hi2 = bx.y > A.pi_f ? __fsub_rn(bx.y, A.two_pi_f) : -INFINITY;
        // the usual item has <= 8 columns and <= 4 beams: fixed-trip unrolled, independent
        // compares (general shapes fall through to the loops)
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
          const float p = cphi[ci];
          const bool in = ci < nc && ((bx.x <= p && p <= bx.y) || lo2 <= p || p <= hi2);
          colbits |= (uint32_t)in << ci;
        }
        for (int ci = 8; ci < nc; ++ci) {
          const float p = S.col_phi[ci];
          const bool in = (bx.x <= p && p <= bx.y) || lo2 <= p || p <= hi2;
          colbits |= (uint32_t)in << ci;
        }
      }
      if (colbits) {
        uint32_t beambits = 0;
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
          const float w = bel[bi];
          beambits |= (uint32_t)(bi < nb && bx.z <= w && w <= bx.w) << bi;
        }
        for (int bi = 4; bi < nb; ++bi) {
          const float w = S.beam_el[bi];
          beambits |= (uint32_t)(bx.z <= w && w <= bx.w) << bi;
        }
        for (uint32_t bb = beambits; bb; bb &= bb - 1u) m |= colbits << ((__ffs(bb) - 1) * nc);
      }
    }
    if (warp == 0) RMARK(r, 3);
    if (SLOTB == 1 && r >= 1) {  // the consumer is done with round r - 1's slots
      named_sync(BAR_EMPTY + (b ^ 1), NT);
      if (S.stop_at[b ^ 1]) break;
      alive = ~S.done_mask[b ^ 1];
    }
    if (warp == 0) RMARK(r, 4);
    uint32_t pid = 0;
    if (valid) {
      S.feat[sb][tid] = S.rec[st][tid][3];
      if (PRAY) {
        pid = __ldg(A.ids + start + tid);
        S.pid[sb][tid] = pid;
      }
    }
    m &= alive;  // no member pairs for terminated rays
    if (sh_smem) {  // asynchronous: lands while the round's responses are computed
      if (m != 0u) {
        const float4* src = reinterpret_cast<const float4*>(A.sh) + (size_t)pid * 12;
#pragma unroll
        for (int c = 0; c < 12; ++c) cp_async16(s_sh + tid * 12 + c, src + c);
      }
      cp_async_commit();
    }
    const uint32_t my = warp_transpose32(m, lane);  // lane r: entries of this warp holding ray r
    S.memb[sb][warp][lane] = my;
    const int k = __popc(m);
    int inc = k;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += t;
    }
    const int K = __shfl_sync(0xffffffffu, inc, 31);
    const int ex = inc - k;
    {
      int pos = ex;
      uint32_t mm = m;
      while (mm) {
        const int rr = __ffs(mm) - 1;
        mm &= mm - 1u;
        S.plist[warp][pos++] = (uint16_t)((lane << 5) | rr);
      }
    }
    if (warp == 0) RMARK(r, 5);
    named_sync(BAR_PROD, E);  // every producer warp's member words are in
    if (warp == 0) RMARK(r, 6);
    {
      int off = 0;
#pragma unroll
      for (int w = 0; w < NP; ++w)
        if (w < warp) off += __popc(S.memb[sb][w][lane]);
      S.rowoff[warp][lane] = off;
    }
    __syncwarp();
    for (int idx = lane; idx < K; idx += 32) {
      const int v = S.plist[warp][idx];
      const int rr = v & 31, el = v >> 5, e = warp * 32 + el;
      const int slot = S.rowoff[warp][rr] + __popc(S.memb[sb][warp][rr] & ((1u << el) - 1u));
      const float4 r0 = S.rec[st][e][0], r1 = S.rec[st][e][1], r2 = S.rec[st][e][2], r3 = S.rec[st][e][3];
      const float mu[3] = {r0.x, r0.y, r0.z};
      const float M[9] = {r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
      RayF rf;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        rf.o_hi[i] = S.ray_oh[rr][i];
        rf.o_lo[i] = S.ray_ol[rr][i];
        rf.d_hi[i] = S.ray_dh[rr][i];
        rf.d_lo[i] = S.ray_dl[rr][i];
      }
      float tau, d2;
      response(rf, mu, M, &tau, &d2);
      S.at[sb][rr][slot] = make_float2(fminf(A.alpha_max, r3.x * expf(-0.5f * d2)), tau);
      S.ent[sb][rr][slot] = (uint8_t)e;
    }
    if (sh_smem) cp_async_wait<0>();  // the staged SH (and the record prefetch issued before it)
    __syncwarp();
    __threadfence_block();
    if (warp == 0) RMARK(r, 7);
    named_arrive(BAR_FULL + b, NT);
  }
  cp_async_wait<0>();
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
                                       const int32_t* tile_ranges, const int32_t* tile_order,
                                       const simuli_project_params* P, const simuli_render_params* rp,
                                       simuli_lidar_out* out, void* stream) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(proj && proj->record && sorted_ids && tile_ranges && P && rp && out, "simuli_render_lidar: NULL argument");
  SIMULI_REQUIRE(P->kind == SIMULI_SENSOR_LIDAR && P->lidar && P->tiling, "simuli_render_lidar: needs LiDAR params");
  const simuli_tiling_dev& T = *P->tiling;
  SIMULI_REQUIRE(T.tile_ray_offsets && T.tile_rays && T.ray_az && T.ray_el && T.ray_s && T.n_tiles >= 1,
                 "simuli_render_lidar: incomplete device tiling");
  SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(proj->record) % 16 == 0, "record must be 16-byte aligned");
  SIMULI_REQUIRE(T.elev_tile_beam_offsets && T.elev_tile_beams && T.az_tile_col_offsets && T.az_tile_cols,
                 "simuli_render_lidar: device tiling lacks the beam / column CSR");
  SIMULI_REQUIRE(T.max_beams_per_elev_tile >= 1 && T.max_cols_per_az_tile >= 1,
                 "simuli_render_lidar: tiling maxima missing");
  LidarArgs A{};
  A.record = reinterpret_cast<const float4*>(proj->record);
  A.ids = sorted_ids;
  A.ranges = reinterpret_cast<const int2*>(tile_ranges);
  A.order = tile_order;
  A.etb_off = T.elev_tile_beam_offsets; A.etb = T.elev_tile_beams;
  A.atc_off = T.az_tile_col_offsets; A.atc = T.az_tile_cols;
  A.ray_az = T.ray_az; A.ray_el = T.ray_el; A.ray_s = T.ray_s;
  A.n_theta = T.n_theta; A.n_az = T.n_azimuth;
  // work items: beam groups x column groups of <= 32 rays per tile, uniform over tiles
  A.cg = T.max_cols_per_az_tile < 32 ? T.max_cols_per_az_tile : 32;
  A.bg = 32 / A.cg;
  A.n_cg = (T.max_cols_per_az_tile + A.cg - 1) / A.cg;
  const int nbg = (T.max_beams_per_elev_tile + A.bg - 1) / A.bg;
  A.items_per_tile = A.n_cg * nbg;
  A.n_items = (int64_t)T.n_tiles * A.items_per_tile;
  A.pose = make_pose_interp_d(P->pose_start, P->pose_end);
  A.pi_f = T.pi_f; A.two_pi_f = T.two_pi_f;
  A.near_tau = P->lidar->min_range_m;
  A.alpha_min = rp->alpha_min; A.alpha_max = rp->alpha_max; A.T_min = rp->T_min;
  A.zeta = out->zeta; A.opacity = out->opacity; A.depth_accum = out->depth_accum; A.depth = out->depth;
  A.intensity = out->intensity; A.raydrop = out->raydrop; A.final_T = out->final_T; A.n_contrib = out->n_contrib;
  A.ray_od = out->ray_od; A.n_visited = out->n_visited; A.n_inbox = out->n_inbox;
  if (rp->sh) {
    SIMULI_REQUIRE(rp->sh_degree >= 0 && rp->sh_degree <= 3, "simuli_render_lidar: sh_degree not in 0..3");
    SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(rp->sh) % 16 == 0, "simuli_render_lidar: sh must be 16-byte aligned");
    A.sh = rp->sh;
    A.sh_ncoef = (rp->sh_degree + 1) * (rp->sh_degree + 1);
  }
  if (A.n_items == 0) return SIMULI_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto launch = [&](auto np_tag, auto stages_tag, auto slot_tag) {
    constexpr int NP = decltype(np_tag)::value, STG = decltype(stages_tag)::value, SB = decltype(slot_tag)::value;
    constexpr size_t smem = sizeof(LidarSmem<NP, STG, SB>);
    cudaFuncSetAttribute(k_render_lidar<NP, STG, SB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_render_lidar<NP, STG, SB, false><<<(unsigned)A.n_items, 32 * (NP + 1), smem, st>>>(A);
  };
  if (A.sh) {  // per-ray SH (A30): the default pipeline shape only
    const size_t smem = sizeof(LidarSmem<kLidarNP, kLidarStages, kLidarSlotBuffers>) +
                        (A.sh_ncoef == 16 ? sizeof(float4) * 12 * 32 * kLidarNP : 0);
    auto kern = k_render_lidar<kLidarNP, kLidarStages, kLidarSlotBuffers, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)A.n_items, 32 * (kLidarNP + 1), smem, st>>>(A);
    return launch_check("simuli_render_lidar");
  }
  using std::integral_constant;
  static const int variant = [] {
    const char* v = getenv("SIMULI_LIDAR_VARIANT");  // tuning only
    return v ? atoi(v) : 0;
  }();
  using I1 = integral_constant<int, 1>;
  using I2 = integral_constant<int, 2>;
  using I3 = integral_constant<int, 3>;
  using I4 = integral_constant<int, 4>;
  switch (variant) {  // NP * 100 + STAGES * 10 + SLOTB
    case 221: launch(I2{}, I2{}, I1{}); break;
    case 231: launch(I2{}, I3{}, I1{}); break;
    case 421: launch(I4{}, I2{}, I1{}); break;
    case 321: launch(I3{}, I2{}, I1{}); break;
    case 422: launch(I4{}, I2{}, I2{}); break;
    case 222: launch(I2{}, I2{}, I2{}); break;
    default: launch(integral_constant<int, kLidarNP>{}, integral_constant<int, kLidarStages>{},
                    integral_constant<int, kLidarSlotBuffers>{}); break;
  }
  return launch_check("simuli_render_lidar");
}

extern "C" int32_t simuli_render_camera(const simuli_projected* proj, const uint32_t* sorted_ids,
                                        const int32_t* tile_ranges, const int32_t* tile_order,
                                        const simuli_project_params* P, const simuli_render_params* rp,
                                        simuli_camera_out* out, void* stream) {
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
  A.order = tile_order;
  A.n_visited = out->n_visited; A.n_inbox = out->n_inbox;
  if (rp->sh) {
    SIMULI_REQUIRE(rp->sh_degree >= 0 && rp->sh_degree <= 3, "simuli_render_camera: sh_degree not in 0..3");
    SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(rp->sh) % 16 == 0, "simuli_render_camera: sh must be 16-byte aligned");
    A.sh = rp->sh;
    A.sh_ncoef = (rp->sh_degree + 1) * (rp->sh_degree + 1);
  }
  const unsigned blocks = (unsigned)(A.Wt * Ht);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (A.sh) {
    switch (C.tile_px) {
      case 8: k_render_camera<8, 1, true><<<blocks, 64, 0, st>>>(A); break;
      default: k_render_camera<16, 4, true><<<blocks * 4, 64, 0, st>>>(A); break;
    }
  } else {
    switch (C.tile_px) {
      case 8: k_render_camera<8, 1, false><<<blocks, 64, 0, st>>>(A); break;
      default: k_render_camera<16, 4, false><<<blocks * 4, 64, 0, st>>>(A); break;
    }
  }
  return launch_check("simuli_render_camera");
}

#ifdef SIMULI_RENDER_PROFILE
extern "C" int32_t simuli_debug_render_trace(long long* host, int item) {
  cudaMemcpyToSymbol(simuli::g_render_trace_item, &item, sizeof(int));
  return cudaMemcpyFromSymbol(host, simuli::g_render_trace, sizeof(long long) * 64 * 16) == cudaSuccess ? 0 : 3;
}
extern "C" int32_t simuli_debug_render_prof(long long* host, int64_t n) {
  return cudaMemcpyFromSymbol(host, simuli::g_render_prof, sizeof(long long) * 4 * n) == cudaSuccess ? 0 : 3;
}
#endif

namespace simuli {
namespace {

// ------------------------------------------------------------------ camera Eq. 2
struct ComposeArgs {
  CameraArgs cam;  // lens model + poses (ray directions)
  const float* env;
  int He, We;
  const float* grid;
  int gh, gw, gd;
  const float* rgb_fg;
  const float* opacity;
  float* rgb_out;
};

__device__ void env_lookup(const ComposeArgs& A, const double d[3], float out[3]) {
  const double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  const double lon = atan2(d[1], d[0]);
  const double z = n > 0.0 ? fmin(1.0, fmax(-1.0, d[2] / n)) : 1.0;
  const double colat = acos(z);
  const double u = (lon + 3.141592653589793) / 6.283185307179586 * A.We - 0.5;
  const double v = colat / 3.141592653589793 * A.He - 0.5;
  const double fu = floor(u), fv = floor(v);
  const float au = (float)(u - fu), av = (float)(v - fv);
  const int u0 = (int)fu, v0 = (int)fv;
  float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int dv = 0; dv <= 1; ++dv)
#pragma unroll
    for (int du = 0; du <= 1; ++du) {
      const int uu = ((u0 + du) % A.We + A.We) % A.We;
      const int vv = min(max(v0 + dv, 0), A.He - 1);
      const float w = (du ? au : 1.f - au) * (dv ? av : 1.f - av);
      const float* t = A.env + ((size_t)vv * A.We + uu) * 3;
      acc[0] = fmaf(w, __ldg(t), acc[0]);
      acc[1] = fmaf(w, __ldg(t + 1), acc[1]);
      acc[2] = fmaf(w, __ldg(t + 2), acc[2]);
    }
  out[0] = acc[0]; out[1] = acc[1]; out[2] = acc[2];
}

// thread per pixel: ray direction, environment map, blend, bilateral-grid affine
// grid (ceil(W / 256), H): a CTA covers 256 pixels of one row, whose (rolling-shutter) pose
// is computed once per CTA
__global__ void __launch_bounds__(256) k_compose_camera(const ComposeArgs A) {
  const int W = A.cam.width, H = A.cam.height;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  __shared__ double s_R[9];
  if (A.env) {
    if (threadIdx.x == 0) {
      const double s = A.cam.rolling ? ((double)j + 0.5) / (double)H : 0.0;
      double R[9], o[3];
      pose_at_d(A.cam.pose, s, R, o);
      for (int k = 0; k < 9; ++k) s_R[k] = R[k];
    }
    __syncthreads();
  }
  if (i >= W) return;
  const int64_t p = (int64_t)j * W + i;
  float cb[3] = {0.f, 0.f, 0.f};
  if (A.env) {
    double dc[3], d[3] = {0.0, 0.0, 0.0};
    if (unproject(A.cam, (double)i + 0.5, (double)j + 0.5, dc))
      for (int k = 0; k < 3; ++k) d[k] = s_R[3 * k] * dc[0] + s_R[3 * k + 1] * dc[1] + s_R[3 * k + 2] * dc[2];
    env_lookup(A, d, cb);
  }
  const float om = __ldg(A.opacity + p);
  float cin[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) cin[c] = __ldg(A.rgb_fg + 3 * p + c) + (1.f - om) * cb[c];
  float out[3] = {cin[0], cin[1], cin[2]};
  if (A.grid) {
    const float lum = fminf(1.f, fmaxf(0.f, 0.299f * cin[0] + 0.587f * cin[1] + 0.114f * cin[2]));
    const float g[3] = {((float)i + 0.5f) / W * A.gw - 0.5f, ((float)j + 0.5f) / H * A.gh - 0.5f, lum * A.gd - 0.5f};
    const int n[3] = {A.gw, A.gh, A.gd};
    int i0[3];
    float a[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float c = fminf(fmaxf(g[k], 0.f), (float)(n[k] - 1));
      const float f = floorf(c);
      i0[k] = (int)f;
      a[k] = c - f;
    }
    float M[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) M[q] = 0.f;
#pragma unroll
    for (int dz = 0; dz <= 1; ++dz)
#pragma unroll
      for (int dy = 0; dy <= 1; ++dy)
#pragma unroll
        for (int dx = 0; dx <= 1; ++dx) {
          const int xi = min(i0[0] + dx, A.gw - 1), yi = min(i0[1] + dy, A.gh - 1), zi = min(i0[2] + dz, A.gd - 1);
          const float w = (dx ? a[0] : 1.f - a[0]) * (dy ? a[1] : 1.f - a[1]) * (dz ? a[2] : 1.f - a[2]);
          const float4* m = reinterpret_cast<const float4*>(A.grid + (((size_t)zi * A.gh + yi) * A.gw + xi) * 12);
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 v = __ldg(m + q);
            M[4 * q] = fmaf(w, v.x, M[4 * q]);
            M[4 * q + 1] = fmaf(w, v.y, M[4 * q + 1]);
            M[4 * q + 2] = fmaf(w, v.z, M[4 * q + 2]);
            M[4 * q + 3] = fmaf(w, v.w, M[4 * q + 3]);
          }
        }
#pragma unroll
    for (int r = 0; r < 3; ++r) out[r] = M[4 * r] * cin[0] + M[4 * r + 1] * cin[1] + M[4 * r + 2] * cin[2] + M[4 * r + 3];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) A.rgb_out[3 * p + c] = out[c];
}

}  // namespace
}  // namespace simuli

extern "C" int32_t simuli_compose_camera(const simuli_project_params* P, const simuli_camera_compose* comp,
                                         const float* rgb_fg, const float* opacity, float* rgb_out, void* stream) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(P && comp && rgb_fg && opacity && rgb_out, "simuli_compose_camera: NULL argument");
  SIMULI_REQUIRE(P->kind == SIMULI_SENSOR_CAMERA && P->camera, "simuli_compose_camera: needs camera params");
  SIMULI_REQUIRE(!comp->env_map || (comp->env_h > 0 && comp->env_w > 0), "simuli_compose_camera: bad env map size");
  SIMULI_REQUIRE(!comp->grid || (comp->grid_h > 0 && comp->grid_w > 0 && comp->grid_d > 0),
                 "simuli_compose_camera: bad grid size");
  SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(comp->grid) % 16 == 0, "simuli_compose_camera: grid must be 16-byte aligned");
  const simuli_camera& C = *P->camera;
  ComposeArgs A{};
  A.cam.model = C.model; A.cam.width = C.width; A.cam.height = C.height; A.cam.rolling = C.rolling_shutter;
  A.cam.fx = C.fx; A.cam.fy = C.fy; A.cam.cx = C.cx; A.cam.cy = C.cy;
  for (int i = 0; i < 5; ++i) A.cam.k[i] = C.k[i];
  A.cam.max_theta = C.max_theta_rad;
  A.cam.pose = make_pose_interp_d(P->pose_start, P->pose_end);
  A.env = comp->env_map; A.He = comp->env_h; A.We = comp->env_w;
  A.grid = comp->grid; A.gh = comp->grid_h; A.gw = comp->grid_w; A.gd = comp->grid_d;
  A.rgb_fg = rgb_fg; A.opacity = opacity; A.rgb_out = rgb_out;
  const int64_t n = (int64_t)C.width * C.height;
  if (n == 0) return SIMULI_OK;
  k_compose_camera<<<dim3((unsigned)((C.width + 255) / 256), (unsigned)C.height), 256, 0,
                     reinterpret_cast<cudaStream_t>(stream)>>>(A);
  return launch_check("simuli_compose_camera");
}

// ====================================================================== backward (A31)
// Gradients of the compositing (Eq. 1) and of the response with respect
// to the particle records, chained to the parameters.  Per ray the tile's list is
// replayed with the forward kernels' float32 arithmetic, so every discrete decision
// (membership, skips, termination) is the forward's; per contribution k, with suffix sums
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
  *rho = expf(-0.5f * d2);
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
#ifdef SIMULI_BWD_CHECK
      if ((int64_t)g >= A.n) {
        printf("bwd: entry %d id %u >= n %lld (range %d..%d)\n", i, g, (long long)A.n, rg.x, rg.y);
        __trap();
      }
#endif
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
