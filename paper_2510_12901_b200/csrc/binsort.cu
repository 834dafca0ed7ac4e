// simuli_bin_sort: tile-Gaussian duplication + radix sort + tile ranges (sm_100a).
//
// "we ... estimate a 2D conic before applying tiling and culling as in 3DGS": one
// (tile, particle) pair per render tile a particle's box overlaps, ordered so that every
// tile's list runs front to back by the float32 depth key, ties by particle id (A19) --
// the "Sort" kernel of tab:culling.
//
// B200 design: instead of sorting P 64-bit (tile | depth) keys over 6 digit passes, the
// order is built in two stable LSD stages that move 8 bytes per element:
//   1. depth sort of the V visible particles (32-bit depth bits + 32-bit id, 4 passes);
//   2. duplication in that depth order into (tile, id) pairs, then a stable sort of the
//      P pairs by tile (ceil(log2 n_tiles / 8) passes: 2 for up to 65536 tiles).
// Stability makes the result identical to sorting (tile << 32 | depth bits, id).
// Every pass is a hand-written onesweep: per partition a warp-level ballot multisplit
// ranks the keys, a decoupled look-back over partitions (dynamic partition ids for
// forward progress) gives the global digit offsets, keys are staged in shared memory in
// digit order and written out coalesced.  Digit histograms of all passes are accumulated
// by the kernels that produce the keys (no separate histogram sweep).
//
// Launches (caller's stream; no host sync when pair_capacity >= 0):
//   k_count_reduce, k_count_top        scan of tile counts and of visibility (id order)
//   k_compact                          visible (depth bits, id) in id order + depth histograms
//   k_onesweep<u32> x 4                depth sort
//   k_vcount_reduce, k_vcount_top      scan of tile counts in depth order
//   k_duplicate                        balanced, coalesced pair emission + tile histograms
//   k_onesweep<u32> x ceil(tile bits / 8)   stable tile sort
//   k_ranges, [k_keys64], [k_tile_order]
#include <cstdint>

#include "abi_util.h"
#include "common.cuh"

namespace simuli {
namespace {

constexpr int kBlkThreads = 256;
constexpr int kBlkItems = 4;
constexpr int kBlk = kBlkThreads * kBlkItems;  // elements per scan / duplication block
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kPart = kSortThreads * kSortItems;  // keys per onesweep partition
constexpr int kDepthPasses = 4;
constexpr int kMaxPasses = 8;  // 4 depth + up to 4 tile passes
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int tile_passes(int32_t n_tiles) {
  int bits = 0;
  while (bits < 31 && (1ll << bits) < (int64_t)n_tiles) ++bits;
  return (bits + 7) / 8;
}

struct Workspace {
  int64_t* blk_pairs;  // [nb+1] tile-count block sums -> offsets (id order)
  int32_t* blk_vis;    // [nb+1] visible-count block sums -> offsets
  int64_t* vblk;       // [nb+1] tile-count block sums in depth order
  int64_t* scal;       // [0] = P, [1] = V
  uint32_t* hist;      // [kMaxPasses][256]
  uint32_t* counters;  // [kMaxPasses]
  uint32_t* status;    // [kMaxPasses][max parts][256]
  uint32_t* vk[2];     // [n] depth bits
  uint32_t* vi[2];     // [n] particle ids
  uint32_t* tk[2];     // [cap] tile keys
  uint32_t* ti_alt;    // [cap] ids (ping-pong partner of sorted_ids)
  int64_t max_parts;
  size_t bytes;
};

Workspace carve(void* base, int64_t n, int64_t cap) {
  Workspace w{};
  const int64_t nb = (n + kBlk - 1) / kBlk;
  const int64_t parts_v = (n + kPart - 1) / kPart, parts_p = (cap + kPart - 1) / kPart;
  w.max_parts = parts_v > parts_p ? parts_v : parts_p;
  if (w.max_parts < 1) w.max_parts = 1;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off += align_up(bytes > 0 ? bytes : 1);
    return r;
  };
  w.blk_pairs = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (nb + 1)));
  w.blk_vis = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (nb + 1)));
  w.vblk = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (nb + 1)));
  w.scal = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * 4));
  w.hist = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses * 256));
  w.counters = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses));
  w.status = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses * w.max_parts * 256));
  for (int i = 0; i < 2; ++i) w.vk[i] = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * n));
  for (int i = 0; i < 2; ++i) w.vi[i] = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * n));
  for (int i = 0; i < 2; ++i) w.tk[i] = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * cap));
  w.ti_alt = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * cap));
  w.bytes = off;
  return w;
}

// ------------------------------------------------------------------ block scan helpers
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// exclusive scan of one value per thread over a 256-thread block; *total = block sum.
// scratch: >= 8 ints of shared memory.
__device__ __forceinline__ int block_excl_scan256(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  int wpre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const int s = scratch[w];
    if (w < warp) wpre += s;
    tot += s;
  }
  __syncthreads();
  *total = tot;
  return wpre + inc - v;
}

// single-CTA exclusive scan of nb int64 (or int32) block sums in place; writes the total
// to sums[nb] and to *total_out.
template <typename T>
__device__ void cta_scan_inplace(T* sums, int64_t nb, int64_t* total_out) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < nb ? (int64_t)sums[i] : 0;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    int64_t wpre = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) wpre += warp_tot[w];
      tot += warp_tot[w];
    }
    if (i < nb) sums[i] = (T)(carry + wpre + inc - v);
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sums[nb] = (T)carry;
    *total_out = carry;
  }
}

// ------------------------------------------------------------------ stage 0: counts
__global__ void __launch_bounds__(kBlkThreads) k_count_reduce(const int* __restrict__ count, int64_t n,
                                                              int64_t* __restrict__ blk_pairs,
                                                              int32_t* __restrict__ blk_vis) {
  __shared__ int scratch[8];
  const int64_t base = (int64_t)blockIdx.x * kBlk;
  int s = 0, v = 0;
#pragma unroll
  for (int i = 0; i < kBlkItems; ++i) {
    const int64_t g = base + i * kBlkThreads + threadIdx.x;
    if (g < n) {
      const int c = __ldg(count + g);
      s += c;
      v += c > 0;
    }
  }
  int tot, totv;
  block_excl_scan256(s, scratch, &tot);
  block_excl_scan256(v, scratch, &totv);
  if (threadIdx.x == 0) {
    blk_pairs[blockIdx.x] = tot;
    blk_vis[blockIdx.x] = totv;
  }
}

__global__ void __launch_bounds__(1024) k_count_top(int64_t* __restrict__ blk_pairs, int32_t* __restrict__ blk_vis,
                                                    int64_t nb, int64_t* __restrict__ scal,
                                                    int64_t* __restrict__ n_pairs, uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ counters) {
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x < kMaxPasses) counters[threadIdx.x] = 0;
  cta_scan_inplace(blk_pairs, nb, &scal[0]);
  __syncthreads();
  cta_scan_inplace(blk_vis, nb, &scal[1]);
  __syncthreads();
  if (threadIdx.x == 0) *n_pairs = scal[0];
}

// visible particles (count > 0) in id order -> (depth bits, id); depth-pass histograms
__global__ void __launch_bounds__(kBlkThreads) k_compact(const int* __restrict__ count, const float* __restrict__ key,
                                                         int64_t n, const int32_t* __restrict__ blk_vis,
                                                         uint32_t* __restrict__ vk, uint32_t* __restrict__ vi,
                                                         uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[kDepthPasses * 256];
  __shared__ int scratch[8];
  const int tid = threadIdx.x;
  for (int i = tid; i < kDepthPasses * 256; i += kBlkThreads) s_hist[i] = 0;
  const int64_t g0 = (int64_t)blockIdx.x * kBlk + tid * kBlkItems;  // blocked: thread owns 4 consecutive
  int flag[kBlkItems], v = 0;
#pragma unroll
  for (int i = 0; i < kBlkItems; ++i) {
    const int64_t g = g0 + i;
    flag[i] = (g < n && __ldg(count + g) > 0) ? 1 : 0;
    v += flag[i];
  }
  int tot;
  int ex = block_excl_scan256(v, scratch, &tot) + blk_vis[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kBlkItems; ++i) {
    if (!flag[i]) continue;
    const int64_t g = g0 + i;
    const uint32_t kb = __float_as_uint(__ldg(key + g));
    vk[ex] = kb;
    vi[ex] = (uint32_t)g;
    ++ex;
#pragma unroll
    for (int p = 0; p < kDepthPasses; ++p) atomicAdd(&s_hist[p * 256 + ((kb >> (8 * p)) & 0xFF)], 1u);
  }
  __syncthreads();
  for (int i = tid; i < kDepthPasses * 256; i += kBlkThreads)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// tile counts of the depth-sorted visible particles, per 1024-block
__global__ void __launch_bounds__(kBlkThreads) k_vcount_reduce(const int* __restrict__ count,
                                                               const uint32_t* __restrict__ vi,
                                                               const int64_t* __restrict__ scal,
                                                               int64_t* __restrict__ vblk) {
  __shared__ int scratch[8];
  const int64_t V = scal[1];
  const int64_t base = (int64_t)blockIdx.x * kBlk;
  if (base >= V && blockIdx.x > 0) return;
  int s = 0;
#pragma unroll
  for (int i = 0; i < kBlkItems; ++i) {
    const int64_t j = base + i * kBlkThreads + threadIdx.x;
    if (j < V) s += __ldg(count + vi[j]);
  }
  int tot;
  block_excl_scan256(s, scratch, &tot);
  if (threadIdx.x == 0) vblk[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_vcount_top(int64_t* __restrict__ vblk, const int64_t* __restrict__ scal,
                                                     int64_t* __restrict__ scratch_total) {
  const int64_t nvb = (scal[1] + kBlk - 1) / kBlk;
  cta_scan_inplace(vblk, nvb, scratch_total);
}

// ------------------------------------------------------------------ duplication (depth order)
struct DupArgs {
  const int* count;
  const int4* rect;
  const uint32_t* vi;
  const int64_t* scal;
  const int64_t* vblk;
  int64_t capacity;
  int n_cols_total, passes;
  uint32_t* tk_out;
  uint32_t* ti_out;
  uint32_t* hist;  // [passes][256] of the tile passes
};

__global__ void __launch_bounds__(kBlkThreads) k_duplicate(const DupArgs A) {
  __shared__ int s_excl[kBlk + 1];
  __shared__ int4 s_rect[kBlk];
  __shared__ uint32_t s_id[kBlk];
  __shared__ uint32_t s_hist[4 * 256];
  __shared__ int scratch[8];
  const int tid = threadIdx.x;
  const int64_t V = A.scal[1];
  const int64_t j0 = (int64_t)blockIdx.x * kBlk;
  if (j0 >= V) return;  // block-uniform
  for (int i = tid; i < A.passes * 256; i += kBlkThreads) s_hist[i] = 0;
  int c[kBlkItems], run = 0;
#pragma unroll
  for (int i = 0; i < kBlkItems; ++i) {
    const int64_t j = j0 + tid * kBlkItems + i;
    c[i] = 0;
    if (j < V) {
      const uint32_t g = A.vi[j];
      c[i] = __ldg(A.count + g);
      s_id[tid * kBlkItems + i] = g;
      s_rect[tid * kBlkItems + i] = __ldg(A.rect + g);
    }
    run += c[i];
  }
  int tot;
  int ex = block_excl_scan256(run, scratch, &tot);
#pragma unroll
  for (int i = 0; i < kBlkItems; ++i) {
    s_excl[tid * kBlkItems + i] = ex;
    ex += c[i];
  }
  if (tid == 0) s_excl[kBlk] = tot;
  __syncthreads();
  const int64_t out0 = A.vblk[blockIdx.x];
  for (int k = tid; k < tot; k += kBlkThreads) {
    int lo = 0, hi = kBlk;  // last li with s_excl[li] <= k
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_excl[mid] <= k) lo = mid;
      else hi = mid;
    }
    const int j = k - s_excl[lo];
    const int4 r = s_rect[lo];
    const int row = r.x + j / r.w;
    int col = r.z + j % r.w;
    if (col >= A.n_cols_total) col -= A.n_cols_total;
    const uint32_t tile = (uint32_t)row * (uint32_t)A.n_cols_total + (uint32_t)col;
    const int64_t pos = out0 + k;
    if (pos < A.capacity) {
      A.tk_out[pos] = tile;
      A.ti_out[pos] = s_id[lo];
      for (int p = 0; p < A.passes; ++p) atomicAdd(&s_hist[p * 256 + ((tile >> (8 * p)) & 0xFF)], 1u);
    }
  }
  __syncthreads();
  for (int i = tid; i < A.passes * 256; i += kBlkThreads)
    if (s_hist[i]) atomicAdd(&A.hist[i], s_hist[i]);
}

// ------------------------------------------------------------------ onesweep pass (u32 keys)
struct SweepArgs {
  const uint32_t* keys_in;
  const uint32_t* vals_in;
  uint32_t* keys_out;
  uint32_t* vals_out;
  const int64_t* count;  // device element count (P or V)
  int64_t capacity;
  int shift;
  const uint32_t* hist;  // [256] of this pass
  uint32_t* status;      // [n_parts][256] of this pass
  uint32_t* counter;
};

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kSortThreads) k_onesweep(const SweepArgs A) {
  __shared__ uint32_t s_part;
  __shared__ uint32_t s_warp_hist[8][256];
  __shared__ uint32_t s_digit_excl[256];
  __shared__ uint32_t s_global[256];
  __shared__ uint32_t s_keys[kPart];
  __shared__ uint32_t s_vals[kPart];
  __shared__ int scratch[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_part = atomicAdd(A.counter, 1u);
  for (int i = tid; i < 8 * 256; i += kSortThreads) (&s_warp_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t P = min(*A.count, A.capacity);
  const int64_t n_parts = (P + kPart - 1) / kPart;
  const int64_t part = s_part;
  if (part >= n_parts) return;
  const int64_t base = part * kPart;
  const int valid = (int)min((int64_t)kPart, P - base);

  uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
  const int64_t wbase = base + warp * (32 * kSortItems);
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    if (idx < P) {
      k[i] = A.keys_in[idx];
      v[i] = A.vals_in[idx];
    } else {
      k[i] = 0xffffffffu;  // padding: digit 0xFF, ranked after every real key
      v[i] = 0;
    }
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = (k[i] >> A.shift) & 0xFFu;
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
    const uint32_t before = __popc(peers & lt_mask);
    const uint32_t prev = s_warp_hist[warp][d];
    __syncwarp();
    if (before == 0) s_warp_hist[warp][d] = prev + __popc(peers);
    __syncwarp();
    rank[i] = prev + before;
  }
  __syncthreads();
  const int d = tid;
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t c = s_warp_hist[w][d];
    s_warp_hist[w][d] = run;
    run += c;
  }
  const uint32_t pad = (uint32_t)(kPart - valid);
  const uint32_t cnt_pub = run - (d == 255 ? pad : 0u);
  uint32_t* st = A.status + part * 256 + d;
  if (part == 0) st_relaxed(st, kFlagInc | cnt_pub);
  else st_relaxed(st, kFlagAgg | cnt_pub);
  int tot;
  s_digit_excl[d] = (uint32_t)block_excl_scan256((int)run, scratch, &tot);
  int htot;
  const int hex = block_excl_scan256((int)A.hist[d], scratch, &htot);
  uint32_t excl = 0;
  if (part > 0) {
    int64_t p = part - 1;
    while (true) {
      const uint32_t s = ld_relaxed(A.status + p * 256 + d);
      if ((s & ~kValMask) == 0) continue;  // not yet published
      excl += s & kValMask;
      if ((s & ~kValMask) == kFlagInc) break;
      --p;
    }
    st_relaxed(st, kFlagInc | (excl + cnt_pub));
  }
  s_global[d] = (uint32_t)hex + excl;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t dd = (k[i] >> A.shift) & 0xFFu;
    const uint32_t pos = s_digit_excl[dd] + s_warp_hist[warp][dd] + rank[i];
    s_keys[pos] = k[i];
    s_vals[pos] = v[i];
  }
  __syncthreads();
  for (int j = tid; j < valid; j += kSortThreads) {
    const uint32_t key = s_keys[j];
    const uint32_t dd = (key >> A.shift) & 0xFFu;
    const int64_t out = (int64_t)s_global[dd] + (j - (int64_t)s_digit_excl[dd]);
    A.keys_out[out] = key;
    A.vals_out[out] = s_vals[j];
  }
}

// ------------------------------------------------------------------ ranges, keys, order
__global__ void k_ranges(const uint32_t* __restrict__ tk, const int64_t* __restrict__ n_pairs, int64_t capacity,
                         int2* __restrict__ ranges) {
  const int64_t P = min(*n_pairs, capacity);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = tk[i];
    if (i == 0 || tk[i - 1] != t) ranges[t].x = (int)i;
    if (i == P - 1 || tk[i + 1] != t) ranges[t].y = (int)(i + 1);
  }
}

__global__ void k_keys64(const uint32_t* __restrict__ tk, const uint32_t* __restrict__ ids,
                         const float* __restrict__ key, const int64_t* __restrict__ n_pairs, int64_t capacity,
                         uint64_t* __restrict__ out) {
  const int64_t P = min(*n_pairs, capacity);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ((uint64_t)tk[i] << 32) | (uint64_t)__float_as_uint(__ldg(key + ids[i]));
}

// Longest-first schedule: tiles bucketed by floor(log2(list length)), decreasing (a
// counting sort; order inside a bucket is whatever the atomics give -- it only affects
// scheduling, never results).  One CTA.
__global__ void __launch_bounds__(1024) k_tile_order(const int2* __restrict__ ranges, int n_tiles,
                                                     int* __restrict__ order) {
  __shared__ int s_hist[33];
  __shared__ int s_off[33];
  for (int i = threadIdx.x; i < 33; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    const int len = r.y - r.x;
    atomicAdd(&s_hist[len > 0 ? 32 - __clz(len) : 0], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int b = 32; b >= 0; --b) {
      s_off[b] = run;
      run += s_hist[b];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    const int len = r.y - r.x;
    order[atomicAdd(&s_off[len > 0 ? 32 - __clz(len) : 0], 1)] = t;
  }
}

}  // namespace
}  // namespace simuli

extern "C" int32_t simuli_bin_sort_workspace_size(int64_t n, int64_t cap, int32_t n_tiles, size_t* bytes) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(bytes && n >= 0 && n_tiles >= 1, "simuli_bin_sort_workspace_size: bad argument");
  if (cap < 0) cap = -cap;
  *bytes = carve(nullptr, n, cap).bytes;
  return SIMULI_OK;
}

extern "C" int32_t simuli_bin_sort(const simuli_projected* proj, int64_t n, int32_t n_tiles, int32_t n_cols_total,
                                   void* workspace, size_t ws_bytes, int64_t pair_capacity, uint64_t* sorted_keys,
                                   uint32_t* sorted_ids, int32_t* tile_ranges, int32_t* tile_order,
                                   int64_t* n_pairs_dev, int64_t* pairs_required, void* stream) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(proj && n >= 0 && n_tiles >= 1 && n_cols_total >= 1 && n_cols_total <= n_tiles,
                 "simuli_bin_sort: bad argument");
  SIMULI_REQUIRE(n <= 0x7fffffffLL, "simuli_bin_sort: n must fit in 32 bits (particle ids are u32)");
  SIMULI_REQUIRE(tile_ranges && n_pairs_dev && sorted_ids, "simuli_bin_sort: NULL output");
  SIMULI_REQUIRE(proj->tile_count && proj->tile_rect && proj->depth_key, "simuli_bin_sort: NULL projection array");
  const bool sync_mode = pair_capacity < 0;
  const int64_t cap = sync_mode ? -pair_capacity : pair_capacity;
  SIMULI_REQUIRE(cap < (1ll << 30), "pair capacity must be < 2^30");
  const Workspace need = carve(nullptr, n, cap);
  SIMULI_REQUIRE(workspace && ws_bytes >= need.bytes, "workspace too small: need %zu bytes", need.bytes);
  Workspace w = carve(workspace, n, cap);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int tpasses = tile_passes(n_tiles);
  const int64_t nb = (n + kBlk - 1) / kBlk;
  auto check = [&](const char* what) -> int32_t {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("simuli_bin_sort: %s: %s", what, cudaGetErrorString(e));
      return SIMULI_ERR_CUDA;
    }
    return SIMULI_OK;
  };
  if (cudaMemsetAsync(tile_ranges, 0, sizeof(int32_t) * 2 * (size_t)n_tiles, st) != cudaSuccess)
    return check("memset ranges");
  if (nb > 0)
    k_count_reduce<<<(unsigned)nb, kBlkThreads, 0, st>>>(proj->tile_count, n, w.blk_pairs, w.blk_vis);
  k_count_top<<<1, 1024, 0, st>>>(w.blk_pairs, w.blk_vis, nb, w.scal, n_pairs_dev, w.hist, w.counters);
  if (int32_t e = check("scan")) return e;
  if (sync_mode) {
    int64_t P = 0;
    if (cudaMemcpyAsync(&P, n_pairs_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return check("pair count readback");
    if (pairs_required) *pairs_required = P;
    if (P > cap) {
      set_error("simuli_bin_sort: %lld pairs exceed capacity %lld", (long long)P, (long long)cap);
      return SIMULI_ERR_CAPACITY;
    }
  }
  if (cudaMemsetAsync(w.status, 0, sizeof(uint32_t) * (kDepthPasses + tpasses) * w.max_parts * 256, st) !=
      cudaSuccess)
    return check("memset status");
  auto sweep = [&](int pass_slot, const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                   const int64_t* count, int64_t capacity, int shift) {
    const int64_t parts = (capacity + kPart - 1) / kPart;
    if (parts <= 0) return;
    SweepArgs S{kin, vin, kout, vout, count, capacity, shift, w.hist + pass_slot * 256,
                w.status + (size_t)pass_slot * w.max_parts * 256, w.counters + pass_slot};
    k_onesweep<<<(unsigned)parts, kSortThreads, 0, st>>>(S);
  };
  // ---- stage 1: depth sort of the visible particles (result back in vk[0] / vi[0])
  if (nb > 0) {
    k_compact<<<(unsigned)nb, kBlkThreads, 0, st>>>(proj->tile_count, proj->depth_key, n, w.blk_vis, w.vk[0],
                                                    w.vi[0], w.hist);
    for (int p = 0; p < kDepthPasses; ++p)
      sweep(p, w.vk[p & 1], w.vi[p & 1], w.vk[(p + 1) & 1], w.vi[(p + 1) & 1], w.scal + 1, n, 8 * p);
    if (int32_t e = check("depth sort")) return e;
    // ---- stage 2: duplication in depth order, stable tile sort
    k_vcount_reduce<<<(unsigned)nb, kBlkThreads, 0, st>>>(proj->tile_count, w.vi[0], w.scal, w.vblk);
    k_vcount_top<<<1, 1024, 0, st>>>(w.vblk, w.scal, w.scal + 2);
    uint32_t* ti[2] = {sorted_ids, w.ti_alt};
    int cur = (tpasses % 2 == 0) ? 0 : 1;  // the last pass must land in sorted_ids
    if (cap > 0) {
      DupArgs D{proj->tile_count, reinterpret_cast<const int4*>(proj->tile_rect), w.vi[0], w.scal, w.vblk, cap,
                n_cols_total, tpasses, w.tk[cur], ti[cur], w.hist + kDepthPasses * 256};
      k_duplicate<<<(unsigned)nb, kBlkThreads, 0, st>>>(D);
      for (int p = 0; p < tpasses; ++p) {
        sweep(kDepthPasses + p, w.tk[cur], ti[cur], w.tk[cur ^ 1], ti[cur ^ 1], w.scal, cap, 8 * p);
        cur ^= 1;
      }
      if (int32_t e = check("tile sort")) return e;
      k_ranges<<<148 * 4, 256, 0, st>>>(w.tk[cur], n_pairs_dev, cap, reinterpret_cast<int2*>(tile_ranges));
      if (sorted_keys)
        k_keys64<<<148 * 4, 256, 0, st>>>(w.tk[cur], sorted_ids, proj->depth_key, n_pairs_dev, cap, sorted_keys);
      if (int32_t e = check("ranges")) return e;
    }
  }
  if (tile_order) {
    k_tile_order<<<1, 1024, 0, st>>>(reinterpret_cast<const int2*>(tile_ranges), n_tiles, tile_order);
    if (int32_t e = check("tile order")) return e;
  }
  return SIMULI_OK;
}
