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
// longest-list-first, pixel per thread, 128-record batches in shared memory, double-buffered
// (batch k + 1 arrives by cp.async, its ids prefetched a batch earlier, while batch k is
// walked); each warp ballots which entries overlap its 2 x 16 pixel strip and walks only
// those; CTA-wide early exit.  Config D (1920x1080 fisheye, 2M particles) render: 2.31 ms
// (one 256-thread CTA per tile) -> 2.01 (strip pre-cull) -> 1.08 (4 bands; 8 bands: 1.15)
// -> 0.97 (double-buffered batches).  Pixel rays by the inverse lens model in double.
#include <cstdint>
#include <cstdlib>
#include <string>

#include "abi_util.h"
#include "camera.cuh"
#include "common.cuh"

namespace simuli {
namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One CTA per (tile, band of TP / SPLIT pixel rows): the bands of a tile read the same list,
// so a long list (near-field particles covering many pixels) is spread over SPLIT CTAs
// instead of one; items are scheduled longest list first (tile_order).
template <int TP, int SPLIT, bool PRAY>
__global__ void __launch_bounds__(TP* TP / SPLIT) k_render_camera(const CameraArgs A) {
  constexpr int NTH = TP * TP / SPLIT;  // threads = pixels of the band
  constexpr int NT = 128;               // list entries staged per batch
  constexpr int PER = NT / NTH;         // entries per thread per batch
  // two batch buffers: batch k + 1's records are copied (cp.async) while batch k is walked
  // (per-ray SH keeps one buffer: its extra registers leave no room for the second)
  constexpr int NBUF = PRAY ? 1 : 2;
  __shared__ float4 s_rec2[NBUF][NT][5];
  __shared__ uint32_t s_id2[NBUF][PRAY ? NT : 1];  // particle ids of the batch (per-ray SH)
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
  const int nbatch = (rg.y - rg.x + NT - 1) / NT;
  auto load_ids = [&](int bi, uint32_t out[PER]) {  // ids of batch bi (registers; used a batch later)
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int pos = rg.x + bi * NT + tid + q * NTH;
      out[q] = (bi < nbatch && pos < rg.y) ? __ldg(A.ids + pos) : 0u;
    }
  };
  auto issue = [&](int bi, const uint32_t idv[PER]) {  // batch bi's records into buffer bi & 1
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NTH, pos = rg.x + bi * NT + e;
      if (bi < nbatch && pos < rg.y) {
        const float4* src = A.record + (size_t)idv[q] * 5;
#pragma unroll
        for (int c = 0; c < 5; ++c) cp_async16(&s_rec2[bi % NBUF][e][c], src + c);
        if (PRAY) s_id2[bi % NBUF][e] = idv[q];
      }
    }
    cp_async_commit();
  };
  uint32_t idn[PER];
  if (NBUF == 2) {
    load_ids(0, idn);
    issue(0, idn);
    load_ids(1, idn);
  }
  for (int bi = 0; bi < nbatch; ++bi) {
    // the count barrier also means every thread is done with batch bi - 1, whose buffer
    // batch bi + 1 reuses
    if (__syncthreads_count(!done) == 0) break;
    if (NBUF == 2) {
      issue(bi + 1, idn);
      load_ids(bi + 2, idn);
      cp_async_wait<1>();  // this thread's copies of batch bi have landed
    } else {
      load_ids(bi, idn);
      issue(bi, idn);
      cp_async_wait<0>();
    }
    __syncthreads();
    const int b = rg.x + bi * NT;
    const int nb = min(NT, rg.y - b);
    float4 (*s_rec)[5] = s_rec2[bi % NBUF];
    const uint32_t* s_id = s_id2[bi % NBUF];
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
  }
  cp_async_wait<0>();
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
