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
// walked); each warp ballots which entries overlap its 2 x 16 pixel strip; the pixel lanes'
// member masks over those come from the entry lanes' strip masks (the per-pixel box test on
// the strip's column and row centres) by a 32 x 32 bit transpose, and the lanes walk their
// own members in list order (one member per live lane per step: 11 of 32 lanes were busy
// when the warp walked the strip's entries together); CTA-wide early exit.  Config D
// (1920x1080 fisheye, 2M particles) render: 2.31 ms (one 256-thread CTA per tile) -> 2.01
// (strip pre-cull) -> 1.08 (4 bands; 8 bands: 1.15) -> 0.97 (double-buffered batches) ->
// 0.78 (per-lane member walk; per-ray SH 2.26 -> 1.42) -> 0.59 (transposed member masks:
// the near-field lists of 20k entries were the render's tail; per-ray SH 1.34).  Pixel
// rays by the inverse lens model in double.
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

#ifndef SIMULI_CAM_DENSE
#define SIMULI_CAM_DENSE 2  // strip-overlapping entries of a group from which the masks are transposed
#endif
// One CTA per (tile, band of TP / SPLIT pixel rows): the bands of a tile read the same list,
// so a long list (near-field particles covering many pixels) is spread over SPLIT CTAs
// instead of one; items are scheduled longest list first (tile_order).
template <int TP, int SPLIT, bool PRAY>
__global__ void __launch_bounds__(TP* TP / SPLIT) k_render_camera(const CameraArgs A) {
  pdl_wait();
  pdl_trigger();
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
  SIMULI_CHECK(tile >= 0 && tile < A.Wt * ((A.height + A.tile_px - 1) / A.tile_px), tile, A.Wt);
  const int2 rg = __ldg(A.ranges + tile);
  SIMULI_CHECK(rg.x >= 0 && rg.x <= rg.y, rg.x, rg.y);
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
        // this pixel's member entries among those (the same box test per entry as the walk
        // over the strip's entries); then every lane walks its own members in list order, so
        // a step evaluates one member per live lane instead of one entry for the lanes it
        // covers
        uint32_t mine = 0u;
        const uint32_t strip = __ballot_sync(0xffffffffu, ov);  // all lanes (done or not)
        if (__popc(strip) >= SIMULI_CAM_DENSE) {  // warp-uniform: a dense group (near-field lists)
          // lane = entry: the strip pixels inside its box (the same comparisons, column and
          // row centres of the strip), then a 32 x 32 bit transpose gives every pixel lane
          // its member entries
          uint32_t pm = 0u;
          if (ov) {
            const float4 bx = s_rec[jl][4];
            uint32_t colmask = 0u;
#pragma unroll
            for (int cc = 0; cc < TP; ++cc) {
              const float u = (float)(tx * TP + cc) + 0.5f;
              colmask |= (uint32_t)(bx.x <= u && u <= bx.y) << cc;
            }
#pragma unroll
            for (int rr = 0; rr < 32 / TP; ++rr) {
              const float v = (float)(row0 + rr) + 0.5f;
              if (bx.z <= v && v <= bx.w) pm |= colmask << (rr * TP);
            }
          }
          mine = warp_transpose32(pm, lane);
          if (done) mine = 0u;
        } else if (!done) {
          for (uint32_t t = strip; t; t &= t - 1u) {
            const int e = __ffs(t) - 1;
            const float4 bx = s_rec[k0 + e][4];
            if (bx.x <= pu && pu <= bx.y && bx.z <= pv && pv <= bx.w) mine |= 1u << e;
          }
        }
        while (mine) {
          const int jj = k0 + __ffs(mine) - 1;
          mine &= mine - 1u;
          ++ni;
          const float4 r0 = s_rec[jj][0], r1 = s_rec[jj][1], r2 = s_rec[jj][2], r3 = s_rec[jj][3];
          const float mu[3] = {r0.x, r0.y, r0.z};
          const float M[9] = {r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
          float tau, d2;
          response(rf, mu, M, &tau, &d2);
          const float alpha = fminf(A.alpha_max, r3.x * __expf(-0.5f * d2));
          if (tau < A.near_tau || alpha < A.alpha_min) continue;
          const float Tn = T * (1.f - alpha);
          if (Tn < A.T_min) {
            done = true;
            mine = 0u;
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
  int64_t n_long;  // hybrid render: items taken by the producer / consumer path
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

// mbarriers (CTA scope): the LiDAR render's chunk-slot ring between producers and consumer.
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(b))),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(b)))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
  unsigned ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 10000000;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(a), "r"(parity)
                 : "memory");
  } while (!ok);
}

// LiDAR render: one CTA per work item (<= 32 rays of one tile) = P producer warps + one
// consumer warp over the item's list in 32-entry chunks (producer p takes chunks p, p + P,
// ...), handed over through a ring of NS chunk slots with one full / empty mbarrier pair
// per slot:
//  producer, per chunk (lane = entry):
//   [A] the entry's box (16 B, cp.async two chunks ahead) against the item's columns and
//       beams -> the exact A12 ray mask m; only entries with m != 0 fetch the rest of their
//       record (64 B: mu, M, opacity, features) -- most listed entries contain none of the
//       tile's rays;
//   [B] (one chunk later, when that fetch has landed) the producer claims the chunk's slot
//       (the consumer has released the chunk NS before), a 32x32 bit transpose gives every ray
//       its member entries; the pairs are numbered ray-major (ray r's k-th member = pair
//       off_r + k), listed by the ray lanes, and their responses (alpha, tau) computed with
//       every lane busy; up to CAP per chunk (the rare rest: the consumer, from the
//       record); the member entries' (opacity, features) go to the slot;
//  consumer (lane = ray): the transmittance chain over the ray's members in list order,
//       state in registers; it publishes the terminated rays (later box tests skip them)
//       and ends the item once all have terminated.
// The per-ray arithmetic (responses, chain order and operands) does not depend on the
// tiling, on culling or on the chunking, so results are bit-identical across (N_phi, M)
// and culling on/off.
// pipeline shape: P producers, NS chunk slots (a producer claims its chunk's slot one
// iteration after the box test), CAP pairs per slot, chosen per call
// (simuli_render_params.lidar_producers): 3 -> (3, 3, 384), the latency shape (one config-B
// scan alone: 173 us; round 1's (3, 6, 512): 182 us), 2 -> (2, 3, 384), 1 -> (1, 2, 256);
// 4 -> k_render_lidar_w below, one warp per item, the leanest (config B with scans in
// flight: 258 / 289 / 311 M rays/s for 3 producers / 1 producer / warp per item; one scan
// alone 176 / 345 / 331 us); 0 (default) -> k_render_lidar_h, the hybrid: one (3, 3, 384)
// producer / consumer item per SM for the longest lists, one warp per item for the rest
// (305 M rays/s in flight, 175 us alone).  SIMULI_LIDAR_VARIANT (P * 10000 + NS * 1000 +
// CAP, 1..8 warp-per-item shapes, 9 hybrid with SIMULI_LIDAR_NLONG) overrides it for sweeps.

template <int CAP>
struct LidarSlot {
  float2 at[CAP];   // (alpha, tau) of the chunk's pairs, ray-major
  float4 f[32];          // (opacity, features) of the chunk's member entries
  uint32_t my[32];       // ray r: member entries of the chunk
  int off[32];           // ray r: index of its first pair
  uint32_t pid[32];      // particle ids of the member entries
};
template <int P, int NS, int CAP>
struct LidarSmem {
  float4 ray[32][3];        // o_hi, o_lo, d_hi, d_lo packed
  float4 rest[P][2][32][4];  // producer p: mu, M, opacity, f of the member entries (two chunks)
  float4 box[P][3][32];      // producer p: chunk boxes (prefetched two chunks ahead)
  uint16_t pairs[P][CAP];  // producer p: the chunk's pairs (ray << 5 | entry), ray-major
  LidarSlot<CAP> slot[NS];
  float col_phi[32], beam_el[32];
  int col_id[32], beam_id[32];
  unsigned long long full[NS], empty[NS];
  uint32_t done_mask;
  int stop;
};

__device__ __forceinline__ void unpack_ray(const float4* q, RayF& r) {
  const float4 a = q[0], b = q[1], c = q[2];
  r.o_hi[0] = a.x; r.o_hi[1] = a.y; r.o_hi[2] = a.z; r.o_lo[0] = a.w;
  r.o_lo[1] = b.x; r.o_lo[2] = b.y; r.d_hi[0] = b.z; r.d_hi[1] = b.w;
  r.d_hi[2] = c.x; r.d_lo[0] = c.y; r.d_lo[1] = c.z; r.d_lo[2] = c.w;
}

// producer-side wait for a slot release that also gives up once the consumer has stopped
// (the consumer ends an item early, without draining, when all its rays have terminated);
// a non-blocking test + nanosleep: a suspended try_wait (NANOSLEEP.SYNCS) wakes on every
// barrier event of the SM, and the spinning producers took the consumer's issue slots
__device__ __forceinline__ bool mbar_wait_or_stop(unsigned long long* b, unsigned parity, volatile int* stop) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
  for (;;) {
    unsigned ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(a), "r"(parity)
                 : "memory");
    if (ok) return true;
    if (*stop) return false;
    __nanosleep(256);  // a waiting producer is ahead of the consumer: poll slowly, leave it the issue slots
  }
}

__device__ __forceinline__ float pair_alpha(const float4* rec, const RayF& rf, float alpha_max, float* tau) {
  const float4 r0 = rec[0], r1 = rec[1], r2 = rec[2];
  const float sig = rec[3].x;
  const float mu[3] = {r0.x, r0.y, r0.z};
  const float M[9] = {r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
  float d2;
  response(rf, mu, M, tau, &d2);
  return fminf(alpha_max, sig * __expf(-0.5f * d2));
}

#ifdef SIMULI_RENDER_PROFILE
// profiling builds only: per item start ns, end ns, chunks run, list length | smid << 32
__device__ long long g_render_prof[1 << 20];
// clock64 cycles summed over all items: [0] consumer waiting full, [1] consumer chain,
// [2] producer waiting cp.async, [3] producer [A], [4] producer waiting empty, [5] producer [B]
__device__ unsigned long long g_render_phase[8];
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(i, t0) if (lane == 0) atomicAdd(&g_render_phase[i], (unsigned long long)(clock64() - (t0)))
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define PROF_T(v)
#define PROF_ADD(i, t0)
#endif

template <int P, int NS, int CAP, bool PRAY>
__device__ __forceinline__ void pc_item(const LidarArgs& A, const int64_t item, unsigned char* smem_raw) {
  LidarSmem<P, NS, CAP>& S = *reinterpret_cast<LidarSmem<P, NS, CAP>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tslot = (int)(item / A.items_per_tile), sub = (int)(item % A.items_per_tile);
  const int tile = A.order ? __ldg(A.order + tslot) : tslot;
  SIMULI_CHECK(tile >= 0 && (int64_t)tile * A.items_per_tile < A.n_items, tile, A.n_items);
  const int et = tile / A.n_theta, at_ = tile % A.n_theta;
  const int bgi = sub / A.n_cg, cgi = sub % A.n_cg;
  const int b0 = __ldg(A.etb_off + et) + bgi * A.bg, b1 = min(__ldg(A.etb_off + et + 1), b0 + A.bg);
  const int c0 = __ldg(A.atc_off + at_) + cgi * A.cg, c1 = min(__ldg(A.atc_off + at_ + 1), c0 + A.cg);
  const int nb = b1 - b0, nc = c1 - c0;
  if (nb <= 0 || nc <= 0) return;  // CTA-uniform
  const int R = nb * nc;
  SIMULI_CHECK(R <= 32, nb, nc);
#ifdef SIMULI_RENDER_PROFILE
  const long long t_start = gtime();
#endif
  if (warp == P) {
    const int j = lane < nc ? __ldg(A.atc + c0 + lane) : 0;
    S.col_id[lane] = j;
    S.col_phi[lane] = lane < nc ? __ldg(A.ray_az + j) : 0.f;
    const int b = lane < nb ? __ldg(A.etb + b0 + lane) : 0;
    S.beam_id[lane] = b;
    S.beam_el[lane] = lane < nb ? __ldg(A.ray_el + (size_t)b * A.n_az) : 0.f;
  }
  if (tid < NS) {
    mbar_init(&S.full[tid], 1);
    mbar_init(&S.empty[tid], 1);
  }
  if (tid == 0) {
    S.stop = 0;
    S.done_mask = R == 32 ? 0u : ~((1u << R) - 1u);  // lanes >= R: no ray
  }
  __syncthreads();
  const int2 rg = __ldg(A.ranges + tile);
  SIMULI_CHECK(rg.x >= 0 && rg.x <= rg.y, rg.x, rg.y);
  const int len = rg.y - rg.x;
  const int nchunks = (len + 31) >> 5;
  volatile uint32_t* vdone = &S.done_mask;
  volatile int* vstop = &S.stop;

  if (warp == P) {
    // ================= consumer: lane = ray
    int ray = 0;
    RayF rf;
    {
      double o[3] = {0, 0, 0}, dd[3] = {0, 0, 0};
      if (lane < R) {
        // rays in double: origin t(s_j), direction R(s_j) u(phi_j, omega_b) (A5), split hi / lo
        const int bi = lane / nc, ci = lane % nc;
        const int j = S.col_id[ci];
        ray = S.beam_id[bi] * A.n_az + j;
        SIMULI_CHECK(j >= 0 && j < A.n_az && ray >= 0, j, ray);
        double Rm[9];
        pose_at_d(A.pose, (double)__ldg(A.ray_s + j), Rm, o);
        double sa, ca, se, ce;
        sincos((double)S.col_phi[ci], &sa, &ca);
        sincos((double)S.beam_el[bi], &se, &ce);
        const double u[3] = {ce * ca, ce * sa, se};
#pragma unroll
        for (int i = 0; i < 3; ++i) dd[i] = Rm[3 * i] * u[0] + Rm[3 * i + 1] * u[1] + Rm[3 * i + 2] * u[2];
        if (A.ray_od) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            A.ray_od[6 * (size_t)ray + i] = o[i];
            A.ray_od[6 * (size_t)ray + 3 + i] = dd[i];
          }
        }
      }
      split_ray(o, dd, rf);
      S.ray[lane][0] = make_float4(rf.o_hi[0], rf.o_hi[1], rf.o_hi[2], rf.o_lo[0]);
      S.ray[lane][1] = make_float4(rf.o_lo[1], rf.o_lo[2], rf.d_hi[0], rf.d_hi[1]);
      S.ray[lane][2] = make_float4(rf.d_hi[2], rf.d_lo[0], rf.d_lo[1], rf.d_lo[2]);
    }
    float shb[PRAY ? 16 : 1];
    if (PRAY) {
      const float dx = rf.d_hi[0] + rf.d_lo[0], dy = rf.d_hi[1] + rf.d_lo[1], dz = rf.d_hi[2] + rf.d_lo[2];
      sh_basis3(dx, dy, dz, shb);
    }
    named_sync(1, 32 * (P + 1));  // rays visible to the producers
    float T = 1.f, z0 = 0.f, z1 = 0.f, z2 = 0.f, D = 0.f, Wt = 0.f;
    int ncon = 0, ni = 0, nv = len;
    bool done = lane >= R;
    uint32_t dmask = *vdone;
    int c = 0;
    for (; c < nchunks; ++c) {
      const int s = c % NS;
      LidarSlot<CAP>& sl = S.slot[s];
      PROF_T(t_w);
      mbar_wait(&S.full[s], (unsigned)((c / NS) & 1));
      PROF_ADD(0, t_w);
      PROF_T(t_c);
      uint32_t rem = done ? 0u : sl.my[lane];
      int idx = sl.off[lane];
      if (!PRAY) {
        // branch-free over the ray's members in list order; the next member's (alpha, tau)
        // and features are loaded one ahead, off the transmittance chain
        int e = rem ? __ffs(rem) - 1 : 0;
        float2 a = sl.at[min(idx, CAP - 1)];
        float4 f = sl.f[e];
        while (__any_sync(0xffffffffu, rem != 0u)) {
          const bool has = rem != 0u;
          const uint32_t rem2 = rem & (rem - 1u);
          const int e2 = rem2 ? __ffs(rem2) - 1 : e;
          const float2 a2 = sl.at[min(idx + 1, CAP - 1)];
          const float4 f2 = sl.f[e2];
          if (has && idx >= CAP) {  // beyond the slot's pair capacity (dense chunks, rare)
            const float4* rec = A.record + (size_t)sl.pid[e] * 5;
            const float4 q[4] = {__ldg(rec), __ldg(rec + 1), __ldg(rec + 2), __ldg(rec + 3)};
            a.x = pair_alpha(q, rf, A.alpha_max, &a.y);
          }
          const bool valid = has && !(a.y < A.near_tau || a.x < A.alpha_min);  // A13, A15
          const float Tn = T * (1.f - a.x);
          const bool term = valid && Tn < A.T_min;  // terminated: not composited (A14)
          const bool comp = valid && !term;
          const float w = a.x * T;
          z0 = comp ? fmaf(w, f.y, z0) : z0;
          z1 = comp ? fmaf(w, f.z, z1) : z1;
          z2 = comp ? fmaf(w, f.w, z2) : z2;
          D = comp ? fmaf(w, a.y, D) : D;
          Wt = comp ? Wt + w : Wt;
          T = comp ? Tn : T;
          ncon += comp ? 1 : 0;
          ni += has ? 1 : 0;
          if (term) {
            done = true;
            nv = 32 * c + e + 1;
          }
          rem = term ? 0u : rem2;
          e = e2;
          a = a2;
          f = f2;
          ++idx;
        }
      } else {
        while (__any_sync(0xffffffffu, rem != 0u)) {
          if (rem != 0u) {
            const int e = __ffs(rem) - 1;
            rem &= rem - 1u;
            float2 a;
            if (idx < CAP) {
              a = sl.at[idx];
            } else {  // beyond the slot's pair capacity (dense chunks, rare): from the record
              const float4* rec = A.record + (size_t)sl.pid[e] * 5;
              const float4 q[4] = {__ldg(rec), __ldg(rec + 1), __ldg(rec + 2), __ldg(rec + 3)};
              a.x = pair_alpha(q, rf, A.alpha_max, &a.y);
            }
            ++idx;
            ++ni;
            if (!(a.y < A.near_tau || a.x < A.alpha_min)) {  // skipped member (A13, A15)
              const float Tn = T * (1.f - a.x);
              if (Tn < A.T_min) {  // terminated: this member is not composited (A14)
                done = true;
                rem = 0u;
                nv = 32 * c + e + 1;
              } else {
                const float w = a.x * T;
                float fv[3];
                if (PRAY) {
                  sh_dot(A.sh + (size_t)sl.pid[e] * A.sh_ncoef * 3, A.sh_ncoef, shb, fv);
                } else {
                  const float4 f = sl.f[e];
                  fv[0] = f.y; fv[1] = f.z; fv[2] = f.w;
                }
                z0 = fmaf(w, fv[0], z0);
                z1 = fmaf(w, fv[1], z1);
                z2 = fmaf(w, fv[2], z2);
                D = fmaf(w, a.y, D);
                Wt += w;
                ++ncon;
                T = Tn;
              }
            }
          }
        }
      }
      PROF_ADD(1, t_c);
      const uint32_t dm = __ballot_sync(0xffffffffu, done);
      const bool all = dm == 0xffffffffu;
      if (dm != dmask) {
        dmask = dm;
        if (lane == 0) {
          *vdone = dm;
          if (all) *vstop = 1;
        }
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        mbar_arrive(&S.empty[s]);
      }
      if (all) break;
    }
#ifdef SIMULI_RENDER_PROFILE
    if (lane == 0 && item < (1 << 18)) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_render_prof[4 * item] = t_start;
      g_render_prof[4 * item + 1] = gtime();
      g_render_prof[4 * item + 2] = c < nchunks ? c + 1 : nchunks;
      g_render_prof[4 * item + 3] = (long long)len | ((long long)smid << 32);
    }
#endif
    if (lane >= R) return;
    if (A.zeta) {
      A.zeta[3 * (size_t)ray] = z0;
      A.zeta[3 * (size_t)ray + 1] = z1;
      A.zeta[3 * (size_t)ray + 2] = z2;
    }
    if (A.opacity) A.opacity[ray] = Wt;
    if (A.depth_accum) A.depth_accum[ray] = D;
    if (A.depth) A.depth[ray] = Wt > 0.f ? D / Wt : 0.f;
    if (A.intensity) A.intensity[ray] = z0;
    if (A.raydrop) A.raydrop[ray] = raydrop_prob(z1, z2);
    if (A.final_T) A.final_T[ray] = T;
    if (A.n_contrib) A.n_contrib[ray] = ncon;
    if (A.n_visited) A.n_visited[ray] = nv;
    if (A.n_inbox) A.n_inbox[ray] = ni;
    return;
  }

  // ================= producers: lane = entry of the chunk
  float4(&pbox)[3][32] = S.box[warp];
  float4(&prest)[2][32][4] = S.rest[warp];
  uint16_t* ppair = S.pairs[warp];
  auto load_id = [&](int c) -> uint32_t {
    const int p = 32 * c + lane;
    return (c < nchunks && p < len) ? __ldg(A.ids + rg.x + p) : 0u;
  };
  auto issue_box = [&](int c, uint32_t id, int b) {
    if (c < nchunks && 32 * c + lane < len) cp_async16(&pbox[b][lane], A.record + (size_t)id * 5 + 4);
    cp_async_commit();  // one group per call (empty or not): keeps the wait_group count exact
  };
  uint32_t id_c = load_id(warp);      // chunk c_k (this lane's entry)
  uint32_t id_n = load_id(warp + P);  // chunk c_{k+1}
  issue_box(warp, id_c, 0);
  issue_box(warp + P, id_n, 1);
  uint32_t id_nn = load_id(warp + 2 * P);  // chunk c_{k+2}
  // the item's first 8 column azimuths / 4 beam elevations in registers (the usual item;
  // unused slots are masked by nc / nb below)
  float cphi[8], bel[4];
#pragma unroll
  for (int ci = 0; ci < 8; ++ci) cphi[ci] = S.col_phi[ci];
#pragma unroll
  for (int bi = 0; bi < 4; ++bi) bel[bi] = S.beam_el[bi];
  auto box_mask = [&](const float4 bx) -> uint32_t {
    uint32_t colbits = 0;
    if (__fsub_rn(bx.y, bx.x) >= A.two_pi_f) {
      colbits = (nc == 32) ? 0xffffffffu : ((1u << nc) - 1u);
    } else {
      const float lo2 = bx.x < -A.pi_f ? __fadd_rn(bx.x, A.two_pi_f) : INFINITY;
      const float hi2 = bx.y > A.pi_f ? __fsub_rn(bx.y, A.two_pi_f) : -INFINITY;
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
    uint32_t m = 0;
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
    return m;
  };
  named_sync(1, 32 * (P + 1));  // rays (consumer) visible

  uint32_t m_prev = 0, id_p = 0;  // ray mask and particle id of chunk c_{k-1} (this lane's entry)
  for (int k = 0;; ++k) {
    const int cc = warp + k * P;  // chunk c_k: [A] this iteration
    const int cp = cc - P;        // chunk c_{k-1}: [B] this iteration
    if (*vstop) break;
    const bool has_cur = cc < nchunks;
    if (!has_cur && k == 0) break;
    PROF_T(t_cp);
    cp_async_wait<1>();  // box(c_k) and rest(c_{k-1}) (this lane's copies; box(c_{k+1}) may fly)
    __syncwarp();
    PROF_ADD(2, t_cp);
    PROF_T(t_a);
    uint32_t m_cur = 0;
    const uint32_t id_k = id_c;
    if (has_cur) {
      // ---- [A] chunk c_k: box test, fetch the member entries' records (one chunk ahead)
      if (32 * cc + lane < len) m_cur = box_mask(pbox[k % 3][lane]) & ~*vdone;
      if (m_cur) {
        const float4* src = A.record + (size_t)id_c * 5;
#pragma unroll
        for (int q = 0; q < 4; ++q) cp_async16(&prest[k & 1][lane][q], src + q);
      }
      cp_async_commit();
      issue_box(cc + 2 * P, id_nn, (k + 2) % 3);
      id_c = id_n;
      id_n = id_nn;
      id_nn = load_id(cc + 3 * P);
    }
    PROF_ADD(3, t_a);
    if (k >= 1) {
      // ---- [B] chunk c_{k-1}: claim its slot, pairs (ray-major) and their responses
      const int s = cp % NS;
      PROF_T(t_e);
      if (cp >= NS) {
        if (!mbar_wait_or_stop(&S.empty[s], (unsigned)((cp / NS - 1) & 1), vstop)) break;
        if (*vstop) break;
      }
      PROF_ADD(4, t_e);
      PROF_T(t_b);
      LidarSlot<CAP>& sl = S.slot[s];
      const float4(&rest)[32][4] = prest[(k - 1) & 1];
      const uint32_t my = warp_transpose32(m_prev, lane);  // lane r: the chunk's entries holding ray r
      const int cnt = __popc(my);
      int inc = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
      }
      const int off_r = inc - cnt;
      const int K = min(__shfl_sync(0xffffffffu, inc, 31), CAP);
      sl.my[lane] = my;
      sl.off[lane] = off_r;
      if (m_prev) {
        sl.f[lane] = rest[lane][3];
        sl.pid[lane] = id_p;
      }
      // the pair list, ray-major: ray r's k-th member e -> pairs[off_r + k] = r << 5 | e
      {
        int i = off_r;
        for (uint32_t t = my; t && i < CAP; t &= t - 1u, ++i) ppair[i] = (uint16_t)((lane << 5) | (__ffs(t) - 1));
      }
      SIMULI_CHECK(K >= 0 && K <= CAP && off_r >= 0, K, off_r);
      __syncwarp();
      for (int i = lane; i < K; i += 32) {
        const int v = ppair[i];
        const int r = v >> 5, e = v & 31;
        RayF rf;
        unpack_ray(S.ray[r], rf);
        float tau;
        const float a = pair_alpha(rest[e], rf, A.alpha_max, &tau);
        sl.at[i] = make_float2(a, tau);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        mbar_arrive(&S.full[s]);
      }
      PROF_ADD(5, t_b);
    }
    m_prev = m_cur;
    id_p = id_k;
    if (!has_cur) break;
  }
  cp_async_wait<0>();
}

template <int P, int NS, int CAP, bool PRAY>
__global__ void __launch_bounds__(32 * (P + 1)) k_render_lidar(const LidarArgs A) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pc_item<P, NS, CAP, PRAY>(A, blockIdx.x, smem_raw);
}


// ---------------------------------------------------------------- LiDAR, warp per item
// One warp per work item, W items per CTA, no inter-warp hand-off: the warp walks the
// item's list in 32-entry chunks with a software pipeline -- box(c + 3) by cp.async (ids a
// chunk earlier), the exact A12 masks of chunk c + 1 and its member entries' records by
// cp.async, while chunk c is finished (transpose, member pairs ray-major, responses with
// every lane busy, then the per-ray chain).  Same responses, chain order and operands as
// k_render_lidar: identical outputs.  The fewest SM resources per item; the longest lists
// become a serial chain (one scan alone: 348 us).
template <int CAP>
struct WarpItemSmem {
  float4 ray[32][3];
  float4 box[3][32];
  float4 rec[2][32][4];
  float2 at[CAP];
  uint16_t pairs[CAP];
  uint32_t pid[2][32];
  float col_phi[32], beam_el[32];
  int col_id[32], beam_id[32];
};

template <int CAP, bool PRAY>
__device__ __forceinline__ void w_item(const LidarArgs& A, const int64_t item, WarpItemSmem<CAP>& S) {
  const int lane = threadIdx.x & 31;
  if (item >= A.n_items) return;  // warp-uniform
  const int tslot = (int)(item / A.items_per_tile), sub = (int)(item % A.items_per_tile);
  const int tile = A.order ? __ldg(A.order + tslot) : tslot;
  const int et = tile / A.n_theta, at_ = tile % A.n_theta;
  const int bgi = sub / A.n_cg, cgi = sub % A.n_cg;
  const int b0 = __ldg(A.etb_off + et) + bgi * A.bg, b1 = min(__ldg(A.etb_off + et + 1), b0 + A.bg);
  const int c0 = __ldg(A.atc_off + at_) + cgi * A.cg, c1 = min(__ldg(A.atc_off + at_ + 1), c0 + A.cg);
  const int nb = b1 - b0, nc = c1 - c0;
  if (nb <= 0 || nc <= 0) return;  // warp-uniform
  const int R = nb * nc;
  {
    const int j = lane < nc ? __ldg(A.atc + c0 + lane) : 0;
    S.col_id[lane] = j;
    S.col_phi[lane] = lane < nc ? __ldg(A.ray_az + j) : 0.f;
    const int b = lane < nb ? __ldg(A.etb + b0 + lane) : 0;
    S.beam_id[lane] = b;
    S.beam_el[lane] = lane < nb ? __ldg(A.ray_el + (size_t)b * A.n_az) : 0.f;
  }
  const int2 rg = __ldg(A.ranges + tile);
  const int len = rg.y - rg.x;
  const int nchunks = (len + 31) >> 5;
  auto ld_id = [&](int c) -> uint32_t {
    const int p = 32 * c + lane;
    return (c < nchunks && p < len) ? __ldg(A.ids + rg.x + p) : 0u;
  };
  auto issue_box = [&](int c, uint32_t id) {
    if (c < nchunks && 32 * c + lane < len) cp_async16(&S.box[c % 3][lane], A.record + (size_t)id * 5 + 4);
  };
  uint32_t idq0 = ld_id(0), idq1 = ld_id(1), idq2 = ld_id(2);
  issue_box(0, idq0);
  issue_box(1, idq1);
  cp_async_commit();
  __syncwarp();
  int ray = 0;
  RayF rf;
  {
    double o[3] = {0, 0, 0}, dd[3] = {0, 0, 0};
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
      if (A.ray_od) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          A.ray_od[6 * (size_t)ray + i] = o[i];
          A.ray_od[6 * (size_t)ray + 3 + i] = dd[i];
        }
      }
    }
    split_ray(o, dd, rf);
    S.ray[lane][0] = make_float4(rf.o_hi[0], rf.o_hi[1], rf.o_hi[2], rf.o_lo[0]);
    S.ray[lane][1] = make_float4(rf.o_lo[1], rf.o_lo[2], rf.d_hi[0], rf.d_hi[1]);
    S.ray[lane][2] = make_float4(rf.d_hi[2], rf.d_lo[0], rf.d_lo[1], rf.d_lo[2]);
  }
  float shb[PRAY ? 16 : 1];
  if (PRAY) {
    const float dx = rf.d_hi[0] + rf.d_lo[0], dy = rf.d_hi[1] + rf.d_lo[1], dz = rf.d_hi[2] + rf.d_lo[2];
    sh_basis3(dx, dy, dz, shb);
  }
  float cphi[8], bel[4];
#pragma unroll
  for (int ci = 0; ci < 8; ++ci) cphi[ci] = S.col_phi[ci];
#pragma unroll
  for (int bi = 0; bi < 4; ++bi) bel[bi] = S.beam_el[bi];
  auto box_mask = [&](const float4 bx) -> uint32_t {
    uint32_t colbits = 0;
    if (__fsub_rn(bx.y, bx.x) >= A.two_pi_f) {
      colbits = (nc == 32) ? 0xffffffffu : ((1u << nc) - 1u);
    } else {
      const float lo2 = bx.x < -A.pi_f ? __fadd_rn(bx.x, A.two_pi_f) : INFINITY;
      const float hi2 = bx.y > A.pi_f ? __fsub_rn(bx.y, A.two_pi_f) : -INFINITY;
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
    uint32_t m = 0;
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
    return m;
  };
  auto fetch_rec = [&](int c, uint32_t m, uint32_t id) {
    if (m) {
      const float4* src = A.record + (size_t)id * 5;
#pragma unroll
      for (int q = 0; q < 4; ++q) cp_async16(&S.rec[c & 1][lane][q], src + q);
    }
    S.pid[c & 1][lane] = id;
  };
  uint32_t done_mask = R == 32 ? 0u : ~((1u << R) - 1u);
  cp_async_wait<0>();
  __syncwarp();
  uint32_t m_next = (nchunks > 0 && lane < len) ? box_mask(S.box[0][lane]) : 0u;
  fetch_rec(0, m_next, idq0);
  issue_box(2, idq2);
  cp_async_commit();
  uint32_t idq3 = ld_id(3);
  float T = 1.f, z0 = 0.f, z1 = 0.f, z2 = 0.f, D = 0.f, Wt = 0.f;
  int ncon = 0, ni = 0, nv = len;
  bool done = lane >= R;
  for (int c = 0; c < nchunks; ++c) {
    const uint32_t m_cur = m_next;
    m_next = 0u;
    if (c + 1 < nchunks) {
      if (32 * (c + 1) + lane < len) m_next = box_mask(S.box[(c + 1) % 3][lane]) & ~done_mask;
      fetch_rec(c + 1, m_next, idq1);
      issue_box(c + 3, idq3);
    }
    cp_async_commit();
    idq1 = idq2;
    idq2 = idq3;
    idq3 = ld_id(c + 4);
    cp_async_wait<1>();
    __syncwarp();
    const uint32_t my = warp_transpose32(m_cur, lane);
    const uint32_t mine = done ? 0u : my;
    const int cnt = __popc(mine);
    int inc = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += t;
    }
    const int off_r = inc - cnt;
    const int K = min(__shfl_sync(0xffffffffu, inc, 31), CAP);
    {
      int i = off_r;
      for (uint32_t t = mine; t && i < CAP; t &= t - 1u, ++i) S.pairs[i] = (uint16_t)((lane << 5) | (__ffs(t) - 1));
    }
    __syncwarp();
    const float4(&rec)[32][4] = S.rec[c & 1];
    for (int i = lane; i < K; i += 32) {
      const int v = S.pairs[i];
      RayF rr;
      unpack_ray(S.ray[v >> 5], rr);
      float tau;
      const float a = pair_alpha(rec[v & 31], rr, A.alpha_max, &tau);
      S.at[i] = make_float2(a, tau);
    }
    __syncwarp();
    uint32_t rem = mine;
    int idx = off_r;
    if (!PRAY) {
      // branch-free, two members per step: both members' loads issued together, only T
      // carries a dependency (same operations and order as the per-member form)
      while (__any_sync(0xffffffffu, rem != 0u)) {
        int e2[2];
        bool h2[2];
        float2 a2[2];
        float4 f2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          h2[u] = rem != 0u;
          e2[u] = h2[u] ? __ffs(rem) - 1 : 0;
          rem &= rem - 1u;
          a2[u] = S.at[min(idx + u, CAP - 1)];
          f2[u] = rec[e2[u]][3];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const bool has = h2[u] && !done;
          float2 a = a2[u];
          if (has && idx >= CAP) a.x = pair_alpha(rec[e2[u]], rf, A.alpha_max, &a.y);
          const bool valid = has && !(a.y < A.near_tau || a.x < A.alpha_min);  // A13, A15
          const float Tn = T * (1.f - a.x);
          const bool term = valid && Tn < A.T_min;  // A14
          const bool comp = valid && !term;
          const float w = a.x * T;
          z0 = comp ? fmaf(w, f2[u].y, z0) : z0;
          z1 = comp ? fmaf(w, f2[u].z, z1) : z1;
          z2 = comp ? fmaf(w, f2[u].w, z2) : z2;
          D = comp ? fmaf(w, a.y, D) : D;
          Wt = comp ? Wt + w : Wt;
          T = comp ? Tn : T;
          ncon += comp ? 1 : 0;
          ni += has ? 1 : 0;
          if (term) {
            done = true;
            nv = 32 * c + e2[u] + 1;
          }
          idx += has ? 1 : 0;
        }
        if (done) rem = 0u;
      }
    } else
    while (rem) {
      const int e = __ffs(rem) - 1;
      rem &= rem - 1u;
      float2 a;
      if (idx < CAP) {
        a = S.at[idx];
      } else {
        a.x = pair_alpha(rec[e], rf, A.alpha_max, &a.y);
      }
      ++idx;
      ++ni;
      if (!(a.y < A.near_tau || a.x < A.alpha_min)) {
        const float Tn = T * (1.f - a.x);
        if (Tn < A.T_min) {
          done = true;
          rem = 0u;
          nv = 32 * c + e + 1;
        } else {
          const float w = a.x * T;
          float fv[3];
          if (PRAY) {
            sh_dot(A.sh + (size_t)S.pid[c & 1][e] * A.sh_ncoef * 3, A.sh_ncoef, shb, fv);
          } else {
            const float4 f = rec[e][3];
            fv[0] = f.y; fv[1] = f.z; fv[2] = f.w;
          }
          z0 = fmaf(w, fv[0], z0);
          z1 = fmaf(w, fv[1], z1);
          z2 = fmaf(w, fv[2], z2);
          D = fmaf(w, a.y, D);
          Wt += w;
          ++ncon;
          T = Tn;
        }
      }
    }
    done_mask = __ballot_sync(0xffffffffu, done);
    if (done_mask == 0xffffffffu) break;
    __syncwarp();
  }
  cp_async_wait<0>();
  if (lane >= R) return;
  if (A.zeta) {
    A.zeta[3 * (size_t)ray] = z0;
    A.zeta[3 * (size_t)ray + 1] = z1;
    A.zeta[3 * (size_t)ray + 2] = z2;
  }
  if (A.opacity) A.opacity[ray] = Wt;
  if (A.depth_accum) A.depth_accum[ray] = D;
  if (A.depth) A.depth[ray] = Wt > 0.f ? D / Wt : 0.f;
  if (A.intensity) A.intensity[ray] = z0;
  if (A.raydrop) A.raydrop[ray] = raydrop_prob(z1, z2);
  if (A.final_T) A.final_T[ray] = T;
  if (A.n_contrib) A.n_contrib[ray] = ncon;
  if (A.n_visited) A.n_visited[ray] = nv;
  if (A.n_inbox) A.n_inbox[ray] = ni;
}

template <int W, int CAP, bool PRAY>
__global__ void __launch_bounds__(32 * W) k_render_lidar_w(const LidarArgs A) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  w_item<CAP, PRAY>(A, (int64_t)blockIdx.x * W + warp, reinterpret_cast<WarpItemSmem<CAP>*>(smem_raw)[warp]);
}

// Hybrid: the n_long longest items (the first ones: items follow the longest-first tile
// order) by the producer / consumer pipeline (3 producers, its shortest critical path), the
// rest one warp per item (the least resources): one scan alone is then bounded by the P/C
// time of the longest lists while most items keep the lean path.
// tuning only: SIMULI_RENDER_H_MINB sets a minimum of resident CTAs per SM (without it,
// 96 registers; an explicit minimum of 1 lets ptxas take 112 and runs slower --
// profiles/r02_experiments.md)
template <int CAP, int WCAP, bool PRAY>
#ifdef SIMULI_RENDER_H_MINB
__global__ void __launch_bounds__(128, SIMULI_RENDER_H_MINB) k_render_lidar_h(const LidarArgs A) {
#else
__global__ void __launch_bounds__(128) k_render_lidar_h(const LidarArgs A) {
#endif
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if ((int64_t)blockIdx.x < A.n_long) {
    pc_item<3, 3, CAP, PRAY>(A, blockIdx.x, smem_raw);
  } else {
    const int warp = threadIdx.x >> 5;
    w_item<WCAP, PRAY>(A, A.n_long + ((int64_t)blockIdx.x - A.n_long) * 4 + warp,
                       reinterpret_cast<WarpItemSmem<WCAP>*>(smem_raw)[warp]);
  }
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
  static const int item_rays = [] {
    const char* v = getenv("SIMULI_LIDAR_ITEM_RAYS");  // tuning only: rays per work item (<= 32)
    const int r = v ? atoi(v) : 32;
    return r >= 1 && r <= 32 ? r : 32;
  }();
  A.cg = T.max_cols_per_az_tile < item_rays ? T.max_cols_per_az_tile : item_rays;
  A.bg = item_rays / A.cg;
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
  auto launch = [&](auto p_tag, auto ns_tag, auto cap_tag) {
    constexpr int P_ = decltype(p_tag)::value, NS_ = decltype(ns_tag)::value, CAP_ = decltype(cap_tag)::value;
    constexpr size_t smem = sizeof(LidarSmem<P_, NS_, CAP_>);
    auto kern = A.sh ? k_render_lidar<P_, NS_, CAP_, true> : k_render_lidar<P_, NS_, CAP_, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, (unsigned)A.n_items, 32 * (P_ + 1), smem, st, A);
  };
  using std::integral_constant;
  static const int variant = [] {
    const char* v = getenv("SIMULI_LIDAR_VARIANT");  // tuning only: P * 10000 + NS * 1000 + CAP
    return v ? atoi(v) : 0;
  }();
  using I2 = integral_constant<int, 2>;
  using I3 = integral_constant<int, 3>;
  using I4 = integral_constant<int, 4>;
  using I6 = integral_constant<int, 6>;
  using I8 = integral_constant<int, 8>;
  auto launch_w = [&](auto w_tag, auto cap_tag) {
    constexpr int W_ = decltype(w_tag)::value, CAP_ = decltype(cap_tag)::value;
    constexpr size_t smem = sizeof(WarpItemSmem<CAP_>) * W_;
    auto kern = A.sh ? k_render_lidar_w<W_, CAP_, true> : k_render_lidar_w<W_, CAP_, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, (unsigned)((A.n_items + W_ - 1) / W_), 32 * W_, smem, st, A);
  };
  auto launch_h = [&](int64_t n_long) {
    constexpr int CAP_ = 384, WCAP_ = 128;
    constexpr size_t s1 = sizeof(LidarSmem<3, 3, CAP_>), s2 = sizeof(WarpItemSmem<WCAP_>) * 4;
    constexpr size_t smem = s1 > s2 ? s1 : s2;
    A.n_long = n_long < A.n_items ? n_long : A.n_items;
    auto kern = A.sh ? k_render_lidar_h<CAP_, WCAP_, true> : k_render_lidar_h<CAP_, WCAP_, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, (unsigned)(A.n_long + (A.n_items - A.n_long + 3) / 4), 128, smem, st, A);
  };
  static const int64_t n_long_env = [] {
    const char* v = getenv("SIMULI_LIDAR_NLONG");  // tuning only
    return v ? (int64_t)atoll(v) : (int64_t)-1;
  }();
  // hybrid default: one producer / consumer item per SM (the longest lists), the rest one
  // warp per item
  static const int64_t n_long_default = [] {
    int d = 0, v = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return (int64_t)v;
  }();
  SIMULI_REQUIRE(rp->lidar_producers >= 0 && rp->lidar_producers <= 4,
                 "simuli_render_lidar: lidar_producers must be 0..4");
  if (variant == 0) {
    switch (rp->lidar_producers) {
      case 3: launch(I3{}, I3{}, integral_constant<int, 384>{}); break;  // latency
      case 2: launch(I2{}, I3{}, integral_constant<int, 384>{}); break;
      case 1: launch(integral_constant<int, 1>{}, I2{}, integral_constant<int, 256>{}); break;
      case 4: launch_w(I4{}, integral_constant<int, 128>{}); break;     // warp per item only
      default: launch_h(n_long_env >= 0 ? n_long_env : n_long_default); break;  // hybrid
    }
    return launch_check("simuli_render_lidar");
  }
  switch (variant) {
    case 9: launch_h(n_long_env >= 0 ? n_long_env : n_long_default); break;
    case 1: launch_w(I4{}, integral_constant<int, 256>{}); break;
    case 2: launch_w(I2{}, integral_constant<int, 256>{}); break;
    case 3: launch_w(I4{}, integral_constant<int, 128>{}); break;
    case 4: launch_w(I8{}, integral_constant<int, 128>{}); break;
    case 5: launch_w(I4{}, integral_constant<int, 64>{}); break;
    case 6: launch_w(I2{}, integral_constant<int, 128>{}); break;
    case 7: launch_w(integral_constant<int, 1>{}, integral_constant<int, 128>{}); break;
    case 8: launch_w(I8{}, integral_constant<int, 64>{}); break;
    case 24512: launch(I2{}, I4{}, integral_constant<int, 512>{}); break;
    case 24384: launch(I2{}, I4{}, integral_constant<int, 384>{}); break;
    case 48256: launch(I4{}, I8{}, integral_constant<int, 256>{}); break;
    case 48384: launch(I4{}, I8{}, integral_constant<int, 384>{}); break;
    case 36384: launch(I3{}, I6{}, integral_constant<int, 384>{}); break;
    case 36256: launch(I3{}, I6{}, integral_constant<int, 256>{}); break;
    case 33256: launch(I3{}, I3{}, integral_constant<int, 256>{}); break;
    case 33384: launch(I3{}, I3{}, integral_constant<int, 384>{}); break;
    case 44256: launch(I4{}, I4{}, integral_constant<int, 256>{}); break;
    case 26256: launch(I2{}, I6{}, integral_constant<int, 256>{}); break;
    case 24256: launch(I2{}, I4{}, integral_constant<int, 256>{}); break;
    case 22384: launch(I2{}, I2{}, integral_constant<int, 384>{}); break;
    case 23384: launch(I2{}, I3{}, integral_constant<int, 384>{}); break;
    case 12384: launch(integral_constant<int, 1>{}, I2{}, integral_constant<int, 384>{}); break;
    case 13384: launch(integral_constant<int, 1>{}, I3{}, integral_constant<int, 384>{}); break;
    case 12256: launch(integral_constant<int, 1>{}, I2{}, integral_constant<int, 256>{}); break;
    default:
      set_error("simuli_render_lidar: unknown SIMULI_LIDAR_VARIANT %d", variant);
      return SIMULI_ERR_INVALID_ARGUMENT;
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
      case 8: launch_pdl(k_render_camera<8, 1, true>, blocks, 64, 0, st, A); break;
      default: launch_pdl(k_render_camera<16, 4, true>, blocks * 4, 64, 0, st, A); break;
    }
  } else {
    switch (C.tile_px) {
      case 8: launch_pdl(k_render_camera<8, 1, false>, blocks, 64, 0, st, A); break;
      default: launch_pdl(k_render_camera<16, 4, false>, blocks * 4, 64, 0, st, A); break;
    }
  }
  return launch_check("simuli_render_camera");
}

#ifdef SIMULI_RENDER_PROFILE
extern "C" int32_t simuli_debug_render_phase(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, simuli::g_render_phase, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 3;
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
