// simuli_bin_sort: tile-Gaussian duplication + onesweep radix sort + tile ranges (sm_100a).
//
// "we ... estimate a 2D conic before applying tiling and culling as in 3DGS": one
// (tile << 32 | depth-key bits, particle id) pair per tile a particle overlaps, sorted so
// every tile's list is depth ordered (the "Sort" kernel of tab:culling).
//
// Launch sequence (all on the caller's stream, no host sync when pair_capacity >= 0):
//   k_count_reduce  per-1024-particle tile-count sums
//   k_count_top     exclusive scan of the block sums (1 CTA) -> P (n_pairs_dev)
//   k_duplicate     block-local scan, balanced + coalesced pair emission (each thread
//                   emits pairs, binary-searching its owner in shared memory), and the
//                   per-pass digit histograms of every emitted key (shared -> global atomics)
//   k_onesweep x passes  stable LSD onesweep (8-bit digits): per 3072-key partition a
//                   warp-level ballot multisplit ranks keys, decoupled look-back over
//                   partitions (dynamic partition ids for forward progress) gives the
//                   global digit offsets, keys are staged in shared memory in digit order
//                   and written out coalesced.
//   k_ranges        [begin, end) per tile from key changes.
#include <cstdint>

#include "abi_util.h"
#include "common.cuh"

namespace simuli {
namespace {

constexpr int kDupThreads = 256;
constexpr int kDupItems = 4;
constexpr int kDupBlock = kDupThreads * kDupItems;  // particles per duplication block
constexpr int kSortThreads = 256;
constexpr int kSortItems = 12;
constexpr int kPart = kSortThreads * kSortItems;  // keys per onesweep partition
constexpr int kMaxPasses = 8;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Workspace {
  int64_t* block_sums;   // [n_dup_blocks] -> exclusive offsets
  uint32_t* hist;        // [kMaxPasses][256]
  uint32_t* status;      // [kMaxPasses][n_parts][256]
  uint32_t* counters;    // [kMaxPasses]
  uint64_t* keys_alt;    // [capacity]
  uint32_t* vals_alt;    // [capacity]
  size_t bytes;
};

Workspace carve(void* base, int64_t n, int64_t cap) {
  Workspace w{};
  const int64_t nb = (n + kDupBlock - 1) / kDupBlock;
  const int64_t parts = (cap + kPart - 1) / kPart;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off += align_up(bytes);
    return r;
  };
  w.block_sums = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (nb + 1)));
  w.hist = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses * 256));
  w.counters = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses));
  w.status = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses * (parts > 0 ? parts : 1) * 256));
  w.keys_alt = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * (cap > 0 ? cap : 1)));
  w.vals_alt = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * (cap > 0 ? cap : 1)));
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

// exclusive scan of one value per thread over a 256-thread block; returns exclusive prefix,
// *total = block sum.  scratch: >= 8 ints of shared memory.
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

// ------------------------------------------------------------------ scan of tile counts
__global__ void __launch_bounds__(kDupThreads) k_count_reduce(const int* __restrict__ count, int64_t n,
                                                              int64_t* __restrict__ block_sums) {
  __shared__ int scratch[8];
  const int64_t base = (int64_t)blockIdx.x * kDupBlock;
  int s = 0;
#pragma unroll
  for (int i = 0; i < kDupItems; ++i) {
    const int64_t g = base + i * kDupThreads + threadIdx.x;
    if (g < n) s += __ldg(count + g);
  }
  int tot;
  block_excl_scan256(s, scratch, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_count_top(int64_t* __restrict__ block_sums, int64_t nb,
                                                    int64_t* __restrict__ n_pairs, uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ counters) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x < kMaxPasses) counters[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    int64_t v = i < nb ? block_sums[i] : 0, inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    int64_t wpre = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < warp) wpre += warp_tot[w];
      tot += warp_tot[w];
    }
    if (i < nb) block_sums[i] = carry + wpre + inc - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    block_sums[nb] = carry;
    *n_pairs = carry;
  }
}

// ------------------------------------------------------------------ duplication
struct DupArgs {
  const int* count;
  const int4* rect;
  const float* key;
  int64_t n, capacity;
  const int64_t* block_offsets;
  int n_cols_total, passes;
  uint64_t* keys_out;
  uint32_t* vals_out;
  uint32_t* hist;  // [passes][256]
};

__global__ void __launch_bounds__(kDupThreads) k_duplicate(const DupArgs A) {
  __shared__ int s_excl[kDupBlock + 1];
  __shared__ int4 s_rect[kDupBlock];
  __shared__ uint32_t s_key[kDupBlock];
  __shared__ uint32_t s_hist[kMaxPasses * 256];
  __shared__ int scratch[8];
  const int tid = threadIdx.x;
  const int64_t g0 = (int64_t)blockIdx.x * kDupBlock;
  for (int i = tid; i < A.passes * 256; i += kDupThreads) s_hist[i] = 0;
  // blocked arrangement: thread t owns particles [t*items, (t+1)*items) of the block
  int c[kDupItems], run = 0;
#pragma unroll
  for (int i = 0; i < kDupItems; ++i) {
    const int64_t g = g0 + tid * kDupItems + i;
    c[i] = g < A.n ? __ldg(A.count + g) : 0;
    run += c[i];
  }
  int tot;
  int ex = block_excl_scan256(run, scratch, &tot);
#pragma unroll
  for (int i = 0; i < kDupItems; ++i) {
    const int li = tid * kDupItems + i;
    const int64_t g = g0 + li;
    s_excl[li] = ex;
    ex += c[i];
    if (c[i] > 0) {
      s_rect[li] = __ldg(A.rect + g);
      s_key[li] = __float_as_uint(__ldg(A.key + g));
    }
  }
  if (tid == 0) s_excl[kDupBlock] = tot;
  __syncthreads();
  const int64_t out0 = A.block_offsets[blockIdx.x];
  for (int k = tid; k < tot; k += kDupThreads) {
    // owner: last li with s_excl[li] <= k (and c > 0, implied by s_excl[li+1] > k)
    int lo = 0, hi = kDupBlock;  // invariant s_excl[lo] <= k < s_excl[hi]
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
    const uint64_t tile = (uint64_t)row * (uint64_t)A.n_cols_total + (uint64_t)col;
    const uint64_t key = (tile << 32) | (uint64_t)s_key[lo];
    const int64_t pos = out0 + k;
    if (pos < A.capacity) {
      A.keys_out[pos] = key;
      A.vals_out[pos] = (uint32_t)(g0 + lo);
      for (int p = 0; p < A.passes; ++p) atomicAdd(&s_hist[p * 256 + (int)((key >> (8 * p)) & 0xFF)], 1u);
    }
  }
  __syncthreads();
  for (int i = tid; i < A.passes * 256; i += kDupThreads)
    if (s_hist[i]) atomicAdd(&A.hist[i], s_hist[i]);
}

// ------------------------------------------------------------------ onesweep pass
struct SweepArgs {
  const uint64_t* keys_in;
  const uint32_t* vals_in;
  uint64_t* keys_out;
  uint32_t* vals_out;
  const int64_t* n_pairs;
  int64_t capacity;
  int shift;
  const uint32_t* hist;  // [256] of this pass
  uint32_t* status;      // [n_parts][256] of this pass
  uint32_t* counter;
};

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
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
  __shared__ uint64_t s_keys[kPart];
  __shared__ uint32_t s_vals[kPart];
  __shared__ int scratch[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_part = atomicAdd(A.counter, 1u);
  for (int i = tid; i < 8 * 256; i += kSortThreads) (&s_warp_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t P = min(*A.n_pairs, A.capacity);
  const int64_t n_parts = (P + kPart - 1) / kPart;
  const int64_t part = s_part;
  if (part >= n_parts) return;
  const int64_t base = part * kPart;
  const int valid = (int)min((int64_t)kPart, P - base);

  uint64_t k[kSortItems];
  uint32_t v[kSortItems];
  uint32_t rank[kSortItems];
  const int64_t wbase = base + warp * (32 * kSortItems);
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    if (idx < P) {
      k[i] = A.keys_in[idx];
      v[i] = A.vals_in[idx];
    } else {
      k[i] = ~0ull;  // padding: digit 0xFF, ranked after every real key of the partition
      v[i] = 0;
    }
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = (uint32_t)(k[i] >> A.shift) & 0xFFu;
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
  // thread = digit: exclusive prefix over warps, partition count
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
  const int dex = block_excl_scan256((int)run, scratch, &tot);
  s_digit_excl[d] = (uint32_t)dex;
  // global digit base of this pass (exclusive prefix of the histogram)
  int htot;
  const int hex = block_excl_scan256((int)A.hist[d], scratch, &htot);
  // decoupled look-back
  uint32_t excl = 0;
  if (part > 0) {
    int64_t p = part - 1;
    while (true) {
      const uint32_t s = ld_volatile(A.status + p * 256 + d);
      if ((s & ~kValMask) == 0) continue;  // not yet published
      excl += s & kValMask;
      if ((s & ~kValMask) == kFlagInc) break;
      --p;
    }
    st_relaxed(st, kFlagInc | (excl + cnt_pub));
  }
  s_global[d] = (uint32_t)hex + excl;
  __syncthreads();
  // stage in digit order
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t dd = (uint32_t)(k[i] >> A.shift) & 0xFFu;
    const uint32_t pos = s_digit_excl[dd] + s_warp_hist[warp][dd] + rank[i];
    s_keys[pos] = k[i];
    s_vals[pos] = v[i];
  }
  __syncthreads();
  for (int j = tid; j < valid; j += kSortThreads) {
    const uint64_t key = s_keys[j];
    const uint32_t dd = (uint32_t)(key >> A.shift) & 0xFFu;
    const int64_t out = (int64_t)s_global[dd] + (j - (int64_t)s_digit_excl[dd]);
    A.keys_out[out] = key;
    A.vals_out[out] = s_vals[j];
  }
}

// ------------------------------------------------------------------ tile ranges
__global__ void k_ranges(const uint64_t* __restrict__ keys, const int64_t* __restrict__ n_pairs, int64_t capacity,
                         int2* __restrict__ ranges) {
  const int64_t P = min(*n_pairs, capacity);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(keys[i] >> 32);
    if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (int)i;
    if (i == P - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (int)(i + 1);
  }
}

// Longest-first schedule: tiles bucketed by floor(log2(list length)) in decreasing order
// (a counting sort; the order inside a bucket is whatever the atomics give -- it only
// affects scheduling, never results).  One CTA.
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

int sort_passes(int32_t n_tiles) {
  int tile_bits = 0;
  while (tile_bits < 31 && (1ll << tile_bits) < (int64_t)n_tiles) ++tile_bits;
  const int bits = 31 + tile_bits;  // depth keys are non-negative floats: bit 31 is zero
  // digits cover bits [0, 8*passes); tile bits start at bit 32
  int passes = (32 + tile_bits + 7) / 8;
  (void)bits;
  return passes;
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
  SIMULI_REQUIRE(tile_ranges && n_pairs_dev && sorted_keys && sorted_ids, "simuli_bin_sort: NULL output");
  SIMULI_REQUIRE(proj->tile_count && proj->tile_rect && proj->depth_key, "simuli_bin_sort: NULL projection array");
  const bool sync_mode = pair_capacity < 0;
  const int64_t cap = sync_mode ? -pair_capacity : pair_capacity;
  SIMULI_REQUIRE(cap < (1ll << 30), "pair capacity must be < 2^30");
  const Workspace need = carve(nullptr, n, cap);
  SIMULI_REQUIRE(workspace && ws_bytes >= need.bytes, "workspace too small: need %zu bytes", need.bytes);
  Workspace w = carve(workspace, n, cap);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int passes = sort_passes(n_tiles);
  const int64_t nb = (n + kDupBlock - 1) / kDupBlock;
  const int64_t parts = (cap + kPart - 1) / kPart;
  auto check = [&](const char* what) -> int32_t {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("simuli_bin_sort: %s: %s", what, cudaGetErrorString(e));
      return SIMULI_ERR_CUDA;
    }
    return SIMULI_OK;
  };
  if (cudaMemsetAsync(tile_ranges, 0, sizeof(int32_t) * 2 * (size_t)n_tiles, st) != cudaSuccess) return check("memset");
  if (n > 0) k_count_reduce<<<(unsigned)nb, kDupThreads, 0, st>>>(proj->tile_count, n, w.block_sums);
  k_count_top<<<1, 1024, 0, st>>>(w.block_sums, nb, n_pairs_dev, w.hist, w.counters);
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
  if (parts > 0 && cudaMemsetAsync(w.status, 0, sizeof(uint32_t) * kMaxPasses * parts * 256, st) != cudaSuccess)
    return check("memset status");
  // the last pass must land in (sorted_keys, sorted_ids)
  uint64_t* kbuf[2] = {sorted_keys, w.keys_alt};
  uint32_t* vbuf[2] = {sorted_ids, w.vals_alt};
  int cur = (passes % 2 == 0) ? 0 : 1;
  if (n > 0) {
    DupArgs D{proj->tile_count, reinterpret_cast<const int4*>(proj->tile_rect), proj->depth_key, n, cap,
              w.block_sums, n_cols_total, passes, kbuf[cur], vbuf[cur], w.hist};
    k_duplicate<<<(unsigned)nb, kDupThreads, 0, st>>>(D);
    if (int32_t e = check("duplicate")) return e;
  }
  for (int p = 0; p < passes && parts > 0; ++p) {
    SweepArgs S{kbuf[cur], vbuf[cur], kbuf[cur ^ 1], vbuf[cur ^ 1], n_pairs_dev, cap, 8 * p,
                w.hist + p * 256, w.status + (size_t)p * parts * 256, w.counters + p};
    k_onesweep<<<(unsigned)parts, kSortThreads, 0, st>>>(S);
    if (int32_t e = check("onesweep")) return e;
    cur ^= 1;
  }
  if (cap > 0) {
    k_ranges<<<148 * 4, 256, 0, st>>>(sorted_keys, n_pairs_dev, cap, reinterpret_cast<int2*>(tile_ranges));
    if (int32_t e = check("ranges")) return e;
  }
  if (tile_order) {
    k_tile_order<<<1, 1024, 0, st>>>(reinterpret_cast<const int2*>(tile_ranges), n_tiles, tile_order);
    if (int32_t e = check("tile order")) return e;
  }
  return SIMULI_OK;
}
