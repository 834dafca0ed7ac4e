// simuli_bin_sort: tile-Gaussian duplication + onesweep radix sort + tile ranges (sm_100a).
//
// "we ... estimate a 2D conic before applying tiling and culling as in 3DGS": one
// (tile, particle) pair per render tile a particle's box overlaps, ordered so that every
// tile's list runs front to back by the float32 depth key, ties by particle id (A19) --
// the "Sort" kernel of tab:culling.
//
// Launch sequence (caller's stream; no host sync when pair_capacity >= 0):
//   memset          one: pass histograms, counters, key range, the look-back status words
//                   of the count scan and the first pass (each pass clears the next's)
//   k_count_scan    single-pass scan of the tile counts (decoupled look-back over
//                   1024-particle blocks) + min / max depth-key bits of the pair-emitting
//                   particles; the last block derives P, the key width
//                   b = bits(max - min) and the pass count ceil((b + tile bits) / 8)
//   k_duplicate     balanced, coalesced pair emission (each thread emits pairs k = tid,
//                   tid+256, ... binary-searching its owner in shared memory) of the
//                   trimmed key (tile << b) | (depth bits - min) -- an order-preserving
//                   map of (tile, depth bits) -- plus the digit histograms of every pass
//   k_onesweep x 6  stable LSD onesweep, 8-bit digits (10-bit measured slower,
//                   profiles/r02_experiments.md); passes beyond the device-side pass
//                   count exit at once (buffer parity is chosen on the device so the
//                   last real pass lands in the caller's arrays).  Per 5120-key partition
//                   (256 threads x 20 keys) a warp-level multisplit (ballot-built peer
//                   masks) ranks the keys, the partition publishes its digit counts, stages
//                   its keys in digit order in shared memory, then a decoupled look-back
//                   over partitions (dynamic partition ids for forward progress) yields
//                   the global digit offsets and the keys are written out coalesced.
//   k_ranges        [begin, end) per tile from tile changes of the sorted keys
//   k_tile_order    longest-first tile order
//   [k_keys64]      the u64 (tile << 32 | depth bits) keys, only if the caller wants them
#include <cstdint>
#include <cstdlib>

#include "abi_util.h"
#include "common.cuh"

namespace simuli {
namespace {

constexpr int kDupThreads = 256;
constexpr int kDupItems = 4;
constexpr int kDupBlock = kDupThreads * kDupItems;
constexpr int kSortThreads = 256;
constexpr int kSortItems = 12;
constexpr int kLookW = 8;      // look-back window (predecessor partitions loaded per round trip)
constexpr int kRankBatch = 4;  // ranking items whose match.any latencies overlap
constexpr int kPart = kSortThreads * kSortItems;  // smallest partition of any sweep shape (status rows)
constexpr int kMaxPasses = 6;  // 48 key bits: 16 tile bits + 32 depth bits at most
constexpr int kRadixMax = 1024;  // digits of up to 10 bits
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

// device scalars: [0] P, [1] key-min bits, [2] key-max bits, [3] depth bits b,
// [4] passes, [5] tile bits
enum { S_P = 0, S_KMIN, S_KMAX, S_B, S_PASSES, S_TBITS, S_N };

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// digit width of the radix passes: 8 bits (256 digits).  The sweep and the duplication's
// histograms are written for any width; 10-bit digits (one pass fewer for config B's 38-bit
// keys) measured slower -- 231 vs 199 us per sort, profiles/r02_experiments.md
constexpr int kRB = 8;
int sort_rb() { return kRB; }
int max_passes_of(int tbits, int rb) { return (32 + tbits + rb - 1) / rb; }

int tile_bits_of(int32_t n_tiles) {
  int bits = 0;
  while (bits < 31 && (1ll << bits) < (int64_t)n_tiles) ++bits;
  return bits;
}

struct Workspace {
  int64_t* block_sums;  // [nb+1]
  int64_t* scal;        // [S_N]
  // zeroed by one memset per call: zero .. zero + zero_bytes
  uint32_t* hist;       // [kMaxPasses][kRadixMax]
  uint32_t* counters;   // [kMaxPasses] sweep partition counters, [kMaxPasses..+4) scan / ranges counters
  uint32_t* kminmax;    // [2]: ~min, max depth-key bits of the pair-emitting particles (atomicMax)
  uint32_t* cstatus;    // [nb] look-back status of the count scan
  uint32_t* status;     // [max passes][n_parts][2^rb]; pass 0's rows in the zeroed region,
                        // pass p + 1's rows zeroed by pass p's partitions
  char* zero;
  size_t zero_bytes;
  uint64_t* keys[2];    // [cap]
  uint32_t* vals_alt;   // [cap]
  int64_t parts;
  size_t bytes;
};

Workspace carve(void* base, int64_t n, int64_t cap, int32_t n_tiles, int rb) {
  Workspace w{};
  const int64_t nb = (n + kDupBlock - 1) / kDupBlock;
  w.parts = (cap + kPart - 1) / kPart;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off += align_up(bytes > 0 ? bytes : 1);
    return r;
  };
  w.block_sums = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (nb + 1)));
  w.scal = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * S_N));
  const size_t z0 = off;
  w.hist = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxPasses * kRadixMax));
  w.counters = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * (kMaxPasses + 4)));
  w.kminmax = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 2));
  w.cstatus = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * (nb > 0 ? nb : 1)));
  const size_t row = sizeof(uint32_t) * (size_t)(w.parts > 0 ? w.parts : 1) << rb;  // one pass's status
  w.status = reinterpret_cast<uint32_t*>(take(row));
  w.zero = p ? p + z0 : nullptr;
  w.zero_bytes = off - z0;
  take(row * (size_t)(max_passes_of(tile_bits_of(n_tiles), rb) - 1));  // status of passes 1..
  for (int i = 0; i < 2; ++i) w.keys[i] = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * cap));
  w.vals_alt = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * cap));
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

// zeroing on the stream as a kernel (a memset node would break the programmatic launch chain)
__global__ void __launch_bounds__(256) k_zero(uint32_t* __restrict__ p, int64_t n_words) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_words; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0u;
}
unsigned zero_blocks(int64_t n_words) {
  const int64_t b = (n_words + 255) / 256;
  return (unsigned)(b < 148 * 4 ? (b > 0 ? b : 1) : 148 * 4);
}

// ------------------------------------------------------------------ counts, key range
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Single-pass scan of the tile counts: 1024-thread blocks of kScanPer = 8 x 1024 particles
// (8 consecutive particles per thread, two 16-byte loads each for counts and keys), a
// decoupled look-back over blocks (dynamic block ids for forward progress; warp 0 reads 32
// predecessors per round trip) -> block_sums[d] = pairs emitted before duplicate block d
// (1024 particles); min / max depth-key bits of the pair-emitting particles by atomics;
// the block that finishes last derives P, the key width b = bits(max - min) and the pass
// count ceil((b + tile bits) / 8).  (One kernel instead of a block reduce + a one-CTA scan.)
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanPer = kScanThreads * kScanItems;  // = 8 duplicate blocks
static_assert(kScanPer % kDupBlock == 0, "scan blocks cover whole duplicate blocks");
__global__ void __launch_bounds__(kScanThreads) k_count_scan(const int* __restrict__ count,
                                                             const float* __restrict__ key, int64_t n, int64_t nsb,
                                                             int64_t nb, int tile_bits, int rb,
                                                             int64_t* __restrict__ block_sums,
                                                             uint32_t* __restrict__ cstatus, uint32_t* __restrict__ kminmax,
                                                             uint32_t* __restrict__ ctr, int64_t* __restrict__ scal,
                                                             int64_t* __restrict__ n_pairs,
                                                             int64_t* __restrict__ n_pairs_max) {
  pdl_wait();
  pdl_trigger();
  constexpr int DB = kScanPer / kDupBlock;  // duplicate blocks per scan block
  constexpr int TPD = kDupBlock / kScanItems;  // threads per duplicate block
  __shared__ int s_wsum[32];
  __shared__ uint32_t s_min[32], s_max[32];
  __shared__ uint32_t s_blk, s_tot;
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_blk = atomicAdd(&ctr[0], 1u);
  __syncthreads();
  const int64_t blk = s_blk;
  const int64_t g0 = blk * kScanPer + (int64_t)tid * kScanItems;
  int sum = 0;
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  if (g0 + kScanItems <= n) {
    const int4* c4 = reinterpret_cast<const int4*>(count + g0);
    const uint4* k4 = reinterpret_cast<const uint4*>(key + g0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int4 c = __ldg(c4 + h);
      const uint4 k = __ldg(k4 + h);
      const int cc[4] = {c.x, c.y, c.z, c.w};
      const uint32_t kk[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sum += cc[j];
        if (cc[j] > 0) {
          kmin = min(kmin, kk[j]);
          kmax = max(kmax, kk[j]);
        }
      }
    }
  } else {
    for (int j = 0; j < kScanItems; ++j) {
      const int64_t g = g0 + j;
      if (g < n) {
        const int c = __ldg(count + g);
        sum += c;
        if (c > 0) {
          const uint32_t kb = __float_as_uint(__ldg(key + g));
          kmin = min(kmin, kb);
          kmax = max(kmax, kb);
        }
      }
    }
  }
  int ws = sum;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ws += __shfl_xor_sync(0xffffffffu, ws, o);
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) {
    s_wsum[warp] = ws;
    s_min[warp] = kmin;
    s_max[warp] = kmax;
  }
  __syncthreads();
  if (warp == 0) {
    // block total and range, published as an aggregate at once
    int t = s_wsum[lane];
    uint32_t mn = s_min[lane], mx = s_max[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, o);
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      st_relaxed(cstatus + blk, (blk == 0 ? kFlagInc : kFlagAgg) | (uint32_t)t);
      if (mx >= mn) {
        atomicMax(&kminmax[0], ~mn);
        atomicMax(&kminmax[1], mx);
      }
    }
    // look-back: 32 predecessors per round trip, summed up to the first inclusive prefix
    // (or up to the first block that has not published, retried from there)
    uint32_t excl = 0;
    int64_t p = blk - 1;
    while (p >= 0) {
      const int64_t q = p - lane;
      const uint32_t v = q >= 0 ? ld_relaxed(cstatus + q) : kFlagInc;
      const uint32_t f = v & ~kValMask;
      const uint32_t unpub = __ballot_sync(0xffffffffu, f == 0), inc = __ballot_sync(0xffffffffu, f == kFlagInc);
      const int fu = unpub ? __ffs(unpub) - 1 : 32, fi = inc ? __ffs(inc) - 1 : 32;
      const int upto = fi < fu ? fi + 1 : fu;  // lanes [0, upto) are consumed
      uint32_t x = lane < upto ? (v & kValMask) : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      excl += x;
      if (fi < fu) break;
      p -= upto;
      if (upto == 0) __nanosleep(32);
    }
    if (lane == 0) {
      if (blk > 0) st_relaxed(cstatus + blk, kFlagInc | (excl + (uint32_t)t));
      s_tot = excl;
    }
  }
  __syncthreads();
  // per duplicate block d of this scan block: exclusive prefix of the warp sums
  if (tid < DB) {
    uint32_t pre = s_tot;
    for (int d = 0; d < tid; ++d)
      for (int w = 0; w < TPD / 32; ++w) pre += (uint32_t)s_wsum[d * (TPD / 32) + w];
    const int64_t db = blk * DB + tid;
    if (db < nb) block_sums[db] = pre;
  }
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&ctr[1], 1u) == (uint32_t)(nsb - 1);
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  // the last block: every block has published its inclusive prefix and key range
  __threadfence();
  const int64_t P = (int64_t)(ld_relaxed(cstatus + nsb - 1) & kValMask);
  uint32_t mn = ~ld_relaxed(&kminmax[0]), mx = ld_relaxed(&kminmax[1]);
  block_sums[nb] = P;
  *n_pairs = P;
  if (n_pairs_max) atomicMax(reinterpret_cast<unsigned long long*>(n_pairs_max), (unsigned long long)P);
  int b = 0;
  if (P > 0 && mx > mn) b = 32 - __clz(mx - mn);
  if (P == 0) mn = 0;
  scal[S_P] = P;
  scal[S_KMIN] = mn;
  scal[S_KMAX] = mx;
  scal[S_B] = b;
  // at least one pass whenever there are pairs: it also writes the ids
  scal[S_PASSES] = P > 0 ? max(1, (b + tile_bits + rb - 1) / rb) : 0;
  scal[S_TBITS] = tile_bits;
}

// n = 0: no pairs
__global__ void k_count_empty(int tile_bits, int64_t* scal, int64_t* n_pairs, int64_t* block_sums) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    scal[S_P] = 0; scal[S_KMIN] = 0; scal[S_KMAX] = 0; scal[S_B] = 0; scal[S_PASSES] = 0;
    scal[S_TBITS] = tile_bits;
    *n_pairs = 0;
    block_sums[0] = 0;
  }
}

// ------------------------------------------------------------------ duplication
struct DupArgs {
  const int* count;
  const int4* rect;
  const float* key;
  int64_t n, capacity;
  const int64_t* block_offsets;
  const int64_t* scal;
  int n_cols_total;
  uint64_t* keys[2];
  uint32_t* vals[2];
  uint32_t* hist;      // [kMaxPasses][kRadixMax]
  int32_t* tile_cnt;   // unused
  int id_bits, packed; // packed: one u64 word = (key << id_bits) | id
  int n_tiles;
};

// Warp-balanced emission: warp w of the CTA takes particles [128 w, 128 w + 128) of the
// CTA's 1024 in groups of 32 (lane = particle); a group's pairs are enumerated 32 at a time
// (pair k0 + lane), the owner lane found by a 5-step shuffle search over the exclusive
// prefix of the counts (no shared-memory binary search, no bank conflicts), so a particle
// spanning hundreds of tiles does not serialise one lane.  Pairs are written in particle
// order (the stable sort then keeps equal keys in id order).
template <int RB>
__global__ void __launch_bounds__(kDupThreads) k_duplicate(const DupArgs A) {
  pdl_wait();
  pdl_trigger();
  constexpr int R = 1 << RB;
  __shared__ uint32_t s_hist[(RB == 8 ? kMaxPasses : 5) * R];
  __shared__ int s_wtot[kDupThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gb = (int64_t)blockIdx.x * kDupBlock;
  const int passes = (int)A.scal[S_PASSES];
  const int b = (int)A.scal[S_B];
  const uint32_t kmin = (uint32_t)A.scal[S_KMIN];
  const int s0 = passes & 1;  // output buffer parity so the last pass lands in buffer 0
  uint64_t* kout = s0 ? A.keys[1] : A.keys[0];
  uint32_t* vout = s0 ? A.vals[1] : A.vals[0];
  for (int i = tid; i < passes * R; i += kDupThreads) s_hist[i] = 0;
  constexpr int kGroups = kDupBlock / kDupThreads;  // groups of 32 particles per warp
  const int64_t gw = gb + (int64_t)warp * 32 * kGroups;
  int c[kGroups], wsum = 0;
#pragma unroll
  for (int q = 0; q < kGroups; ++q) {
    const int64_t g = gw + q * 32 + lane;
    c[q] = g < A.n ? __ldg(A.count + g) : 0;
    wsum += c[q];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if (lane == 0) s_wtot[warp] = wsum;
  __syncthreads();
  int64_t base = A.block_offsets[blockIdx.x];
  for (int w = 0; w < warp; ++w) base += s_wtot[w];
#pragma unroll 1
  for (int q = 0; q < kGroups; ++q) {
    const int64_t g = gw + q * 32 + lane;
    const int cq = c[q];
    int4 r = make_int4(0, 0, 0, 1);
    uint32_t kq = 0;
    if (cq > 0) {
      r = __ldg(A.rect + g);
      kq = __float_as_uint(__ldg(A.key + g)) - kmin;
    }
    int incl = cq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - cq;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int k0 = 0; k0 < total; k0 += 32) {
      const int k = k0 + lane;
      int lo = 0;  // owner: the last lane whose exclusive prefix is <= k
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, excl, lo + step);
        if (v <= k) lo += step;
      }
      const int j = k - __shfl_sync(0xffffffffu, excl, lo);
      const int rx = __shfl_sync(0xffffffffu, r.x, lo), rz = __shfl_sync(0xffffffffu, r.z, lo),
                rw = __shfl_sync(0xffffffffu, r.w, lo);
      const uint32_t kk = __shfl_sync(0xffffffffu, kq, lo);
      if (k >= total) continue;
      const int row = rx + j / rw;  // rect = (row0, row1, col start, col run length)
      int col = rz + j % rw;
      if (col >= A.n_cols_total) col -= A.n_cols_total;
      const uint32_t tile = (uint32_t)row * (uint32_t)A.n_cols_total + (uint32_t)col;
      SIMULI_CHECK(col >= 0 && col < A.n_cols_total && tile < (uint32_t)A.n_tiles, col, tile);
      SIMULI_CHECK(kk < (1u << b) || b == 32 || kq == 0, kk, b);
      const uint64_t key = ((uint64_t)tile << b) | (uint64_t)kk;
      const int64_t pos = base + k;
      if (pos < A.capacity) {
        const uint64_t id = (uint64_t)(gw + q * 32 + lo);
        if (A.packed) {
          kout[pos] = (key << A.id_bits) | id;
        } else {
          kout[pos] = key;
          vout[pos] = (uint32_t)id;
        }
        for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p * R + (int)((key >> (RB * p)) & (R - 1))], 1u);
      }
    }
    base += total;
  }
  __syncthreads();
  for (int i = tid; i < passes * R; i += kDupThreads)
    if (s_hist[i]) atomicAdd(&A.hist[(i / R) * kRadixMax + (i % R)], s_hist[i]);
}

// ------------------------------------------------------------------ onesweep pass
struct SweepArgs {
  uint64_t* keys[2];
  uint32_t* vals[2];
  const int64_t* scal;
  int64_t capacity;
  int pass;
  int id_bits;          // packed mode: low id_bits of every word are the particle id
  uint32_t* ids_final;  // packed mode: the last pass also writes the ids here
  const uint32_t* hist;  // [2^rb] of this pass
  uint32_t* status;      // [n_parts][2^rb] of this pass
  uint32_t* status_next; // the next pass's rows (zeroed here, one row per partition) or NULL
  uint32_t* counter;
};


#ifdef SIMULI_SORT_PROFILE
// profiling builds only: per (pass, partition) globaltimer stamps: start, keys loaded,
// ranked, aggregate published, look-back done, end; [6] = look-back rounds (max over digits)
__device__ long long g_sort_prof[kMaxPasses][4096][8];
__device__ __forceinline__ long long sort_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SORT_STAMP(i) if (tid == 0 && part < 4096) g_sort_prof[A.pass][part][i] = sort_gtime()
#else
#define SORT_STAMP(i)
#endif

// lanes of the warp holding the same RB-bit digit: the AND over the digit's bits of the
// bit's ballot (or its complement) -- RB ballots instead of one match.any, whose cost grows
// with the number of distinct values in the warp (measured: ~5 us per 3072-key partition
// with random digits, vs ~2 us with a few distinct values)
template <int RB>
__device__ __forceinline__ uint32_t warp_peers(uint32_t dg) {
  uint32_t m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (dg >> b) & 1u);
    m &= ((dg >> b) & 1u) ? bal : ~bal;
  }
  return m;
}

// exclusive scan of one value per thread over an NT-thread block (NT / 32 <= 32 warps)
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* scratch, int* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  int wpre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int s = scratch[w];
    if (w < warp) wpre += s;
    tot += s;
  }
  __syncthreads();
  *total = tot;
  return wpre + inc - v;
}

// One onesweep pass: NT threads x ITEMS keys per partition, RB-bit digits; DT digit threads
// own DPT consecutive digits each and look back LOOKW predecessor partitions per round trip.
template <bool Packed, int NT, int ITEMS, int R>
struct SweepSmem {
  uint32_t warp_hist[NT / 32][R];
  uint32_t digit_excl[R];
  uint32_t global[R];
  uint64_t keys[NT * ITEMS];
  uint32_t vals[Packed ? 1 : NT * ITEMS];
  int scratch[32];
  uint32_t part;
};

template <bool Packed, int NT, int ITEMS, int LOOKW, int MINB, int RB>
__global__ void __launch_bounds__(NT, MINB) k_onesweep(const SweepArgs A) {
  pdl_wait();
  pdl_trigger();
  constexpr int R = 1 << RB;
  constexpr int DT = NT < R ? NT : R;  // digit threads
  constexpr int DPT = R / DT;          // consecutive digits per digit thread
  static_assert(NT >= 256 && R % DT == 0, "digit threads cover the digits");
  constexpr int NW = NT / 32;
  constexpr int PART = NT * ITEMS;
  extern __shared__ __align__(16) unsigned char sweep_smem[];
  SweepSmem<Packed, NT, ITEMS, R>& S = *reinterpret_cast<SweepSmem<Packed, NT, ITEMS, R>*>(sweep_smem);
  const int passes = (int)A.scal[S_PASSES];
  if (A.pass >= passes) return;  // grid-uniform: this digit is beyond the key width
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t P = min(A.scal[S_P], A.capacity);
  const int64_t n_parts = (P + PART - 1) / PART;
  // the grid is sized for the capacity; exactly the first n_parts CTAs take a partition
  // number from the counter, so every partition is claimed once
  if ((int64_t)blockIdx.x >= n_parts) return;
  if (tid == 0) S.part = atomicAdd(A.counter, 1u);
  for (int i = tid; i < NW * R; i += NT) (&S.warp_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t part = S.part;
  // the next pass has the same partitions: this one clears its status row there (the next
  // launch follows this one on the stream)
  if (A.status_next && A.pass + 1 < passes)
    for (int i = tid; i < R; i += NT) A.status_next[part * R + i] = 0u;
#ifdef SIMULI_SORT_PROFILE
  long long t_start = sort_gtime();
  if (tid == 0 && part < 4096) g_sort_prof[A.pass][part][0] = t_start;
#endif
  const int in = ((passes & 1) + A.pass) & 1;
  // selects, not A.keys[in]: a dynamic index into the parameter struct would copy it to
  // local memory
  const uint64_t* keys_in = in ? A.keys[1] : A.keys[0];
  const uint32_t* vals_in = in ? A.vals[1] : A.vals[0];
  uint64_t* keys_out = in ? A.keys[0] : A.keys[1];
  uint32_t* vals_out = in ? A.vals[0] : A.vals[1];
  const int shift = RB * A.pass + (Packed ? A.id_bits : 0);
  const bool last = A.pass == passes - 1;
  const int64_t base = part * PART;
  const int valid = (int)min((int64_t)PART, P - base);

  uint64_t k[ITEMS];
  uint32_t v[ITEMS];
  uint32_t rank[ITEMS];
  const int64_t wbase = base + warp * (32 * ITEMS);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    if (idx < P) {
      k[i] = keys_in[idx];
      if (!Packed) v[i] = vals_in[idx];
    } else {
      k[i] = ~0ull;  // padding: the top digit, ranked after every real key of the partition
      if (!Packed) v[i] = 0;
    }
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
#ifdef SIMULI_SORT_PROFILE
  {
    uint64_t x = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) x ^= k[i];
    if (x == 0x123456789ull) S.part = 0;  // forces the loads to complete before the stamp
  }
  __syncthreads();
  SORT_STAMP(1);
  const long long ck_rank0 = clock64();
#endif
  // warp multisplit: lanes with equal digits (ballot-built peer masks), the highest of them
  // bumps the warp's digit counter once and broadcasts the previous value.  Items go in
  // batches of kRankBatch so the ballot latencies overlap; the counter updates stay in item
  // order (one warp's shared-memory atomics execute in program order), which keeps the sort
  // stable.
#pragma unroll
  for (int i0 = 0; i0 < ITEMS; i0 += kRankBatch) {
    uint32_t peers[kRankBatch], dg[kRankBatch], prev[kRankBatch];
#pragma unroll
    for (int j = 0; j < kRankBatch; ++j) {
      dg[j] = (uint32_t)(k[i0 + j] >> shift) & (R - 1);
      peers[j] = warp_peers<RB>(dg[j]);
    }
#pragma unroll
    for (int j = 0; j < kRankBatch; ++j) {
      prev[j] = 0;
      if (lane == 31 - __clz(peers[j])) prev[j] = atomicAdd(&S.warp_hist[warp][dg[j]], (uint32_t)__popc(peers[j]));
    }
#pragma unroll
    for (int j = 0; j < kRankBatch; ++j) {
      prev[j] = __shfl_sync(0xffffffffu, prev[j], 31 - __clz(peers[j]));
      rank[i0 + j] = prev[j] + __popc(peers[j] & lt_mask);
    }
  }
  __syncthreads();
  SORT_STAMP(2);
#ifdef SIMULI_SORT_PROFILE
  if (tid == 0 && part < 4096) g_sort_prof[A.pass][part][6] = clock64() - ck_rank0;
#endif
  // digit threads (tid < DT, digits d0 .. d0 + DPT - 1): per-warp exclusive offsets, the
  // partition's digit counts, published as aggregates at once
  const int d0 = tid * DPT;
  const uint32_t pad = (uint32_t)(PART - valid);
  uint32_t run[DPT], cnt_pub[DPT], hv[DPT];
  uint32_t tsum = 0, hsum = 0;
  uint32_t* st = A.status + part * R + d0;
  if (tid < DT) {
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      uint32_t r = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t c = S.warp_hist[w][d0 + j];
        S.warp_hist[w][d0 + j] = r;
        r += c;
      }
      run[j] = r;
      cnt_pub[j] = r - (d0 + j == R - 1 ? pad : 0u);
      tsum += r;
      st_relaxed(st + j, (part == 0 ? kFlagInc : kFlagAgg) | cnt_pub[j]);
      hv[j] = A.hist[d0 + j];
      hsum += hv[j];
    }
  }
  SORT_STAMP(3);
  int tot;
  const uint32_t tex = (uint32_t)block_excl_scan<NT>(tid < DT ? (int)tsum : 0, S.scratch, &tot);
  if (tid < DT) {
    uint32_t e = tex;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      S.digit_excl[d0 + j] = e;
      e += run[j];
    }
  }
  int htot;
  const uint32_t hex = (uint32_t)block_excl_scan<NT>(tid < DT ? (int)hsum : 0, S.scratch, &htot);
  // keys staged in digit order in shared memory while the predecessors publish (the
  // scatter needs only partition-local offsets; block_excl_scan's barrier made digit_excl
  // visible)
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t dd = (uint32_t)(k[i] >> shift) & (R - 1);
    const uint32_t pos = S.digit_excl[dd] + S.warp_hist[warp][dd] + rank[i];
    SIMULI_CHECK(pos < (uint32_t)PART, pos, PART);
    S.keys[pos] = k[i];
    if (!Packed) S.vals[pos] = v[i];
  }
  if (tid < DT) {
    uint32_t excl[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) excl[j] = 0;
    if (part > 0) {
      // windowed look-back: LOOKW predecessors are loaded at once (independent loads, one
      // round trip), then consumed in order; a digit closes at its first inclusive prefix,
      // a round stops at the first partition that has not published every still-open digit
      // (retried from there, after a short sleep so the spinning digit threads leave the
      // issue slots to the SM's other partitions)
      uint32_t open = (1u << DPT) - 1u;
      int64_t p = part - 1;
      while (true) {
        uint32_t sv[LOOKW][DPT];
#pragma unroll
        for (int w = 0; w < LOOKW; ++w)
#pragma unroll
          for (int j = 0; j < DPT; ++j) sv[w][j] = (p - w >= 0) ? ld_relaxed(A.status + (p - w) * R + d0 + j) : 0u;
        int adv = 0;
        bool blocked = false;
#pragma unroll
        for (int w = 0; w < LOOKW; ++w) {
          bool pub = true;
#pragma unroll
          for (int j = 0; j < DPT; ++j) pub = pub && (!((open >> j) & 1u) || (sv[w][j] & ~kValMask) != 0);
          const bool take = !blocked && open != 0u && pub;
          blocked = blocked || (open != 0u && !pub);
#pragma unroll
          for (int j = 0; j < DPT; ++j) {
            const bool tj = take && ((open >> j) & 1u);
            excl[j] += tj ? (sv[w][j] & kValMask) : 0u;
            if (tj && (sv[w][j] & ~kValMask) == kFlagInc) open &= ~(1u << j);
          }
          adv += take ? 1 : 0;
        }
        if (open == 0u) break;
        p -= adv;
        if (blocked) __nanosleep(64);
      }
#pragma unroll
      for (int j = 0; j < DPT; ++j) st_relaxed(st + j, kFlagInc | (excl[j] + cnt_pub[j]));
    }
    uint32_t h = hex;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      S.global[d0 + j] = h + excl[j];
      h += hv[j];
    }
  }
  __syncthreads();
  SORT_STAMP(4);
  for (int j = tid; j < valid; j += NT) {
    const uint64_t key = S.keys[j];
    const uint32_t dd = (uint32_t)(key >> shift) & (R - 1);
    const int64_t out = (int64_t)S.global[dd] + (j - (int64_t)S.digit_excl[dd]);
    SIMULI_CHECK(out >= 0 && out < P, out, P);
    keys_out[out] = key;
    if (!Packed) vals_out[out] = S.vals[j];
    else if (last) A.ids_final[out] = (uint32_t)(key & ((1ull << A.id_bits) - 1ull));
  }
#ifdef SIMULI_SORT_PROFILE
  __syncthreads();
  SORT_STAMP(5);
  if (tid == 0 && part < 4096) g_sort_prof[A.pass][part][7] = 1;
#endif
}

// pass launcher: sweep shape (threads, items, look-back window, digit bits); the default
// and the tuning variants (SIMULI_SORT_VARIANT = NT * 10000 + ITEMS * 100 + LOOKW)
template <bool Packed, int NT, int ITEMS, int LOOKW, int MINB, int RB>
void launch_sweep(const SweepArgs& S, int64_t cap, cudaStream_t st) {
  constexpr int PART = NT * ITEMS;
  static_assert(PART >= kPart, "status rows are sized for partitions of >= kPart keys");
  constexpr size_t smem = sizeof(SweepSmem<Packed, NT, ITEMS, (1 << RB)>);
  static bool once = [] {
    cudaFuncSetAttribute(k_onesweep<Packed, NT, ITEMS, LOOKW, MINB, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return true;
  }();
  (void)once;
  const unsigned grid = (unsigned)((cap + PART - 1) / PART);
  if (grid > 0) launch_pdl(k_onesweep<Packed, NT, ITEMS, LOOKW, MINB, RB>, grid, NT, smem, st, S);
}

template <bool Packed>
void launch_sweep_variant(const SweepArgs& S, int64_t cap, cudaStream_t st, int rb) {
  static const int variant = [] {
    const char* v = getenv("SIMULI_SORT_VARIANT");
    return v ? atoi(v) : 0;
  }();
  (void)rb;  // kRB
  switch (variant) {
    case 2561216: launch_sweep<Packed, 256, 12, 16, 4, 8>(S, cap, st); break;
    case 2561232: launch_sweep<Packed, 256, 12, 32, 4, 8>(S, cap, st); break;
    case 2561233: launch_sweep<Packed, 256, 12, 32, 3, 8>(S, cap, st); break;
    case 2561633: launch_sweep<Packed, 256, 16, 32, 3, 8>(S, cap, st); break;
    case 2561616: launch_sweep<Packed, 256, 16, 16, 4, 8>(S, cap, st); break;
    case 2561632: launch_sweep<Packed, 256, 16, 32, 4, 8>(S, cap, st); break;
    case 2562432: launch_sweep<Packed, 256, 24, 32, 4, 8>(S, cap, st); break;
    case 5121232: launch_sweep<Packed, 512, 12, 32, 2, 8>(S, cap, st); break;
    case 5121216: launch_sweep<Packed, 512, 12, 16, 2, 8>(S, cap, st); break;
    case 2562408: launch_sweep<Packed, 256, 24, 8, 3, 8>(S, cap, st); break;
    case 2562404: launch_sweep<Packed, 256, 24, 4, 3, 8>(S, cap, st); break;
    case 2562416: launch_sweep<Packed, 256, 24, 16, 3, 8>(S, cap, st); break;
    case 5122408: launch_sweep<Packed, 512, 24, 8, 1, 8>(S, cap, st); break;
    case 2561608: launch_sweep<Packed, 256, 16, 8, 4, 8>(S, cap, st); break;
    case 10241208: launch_sweep<Packed, 1024, 12, 8, 1, 8>(S, cap, st); break;
    case 10241216: launch_sweep<Packed, 1024, 12, 16, 1, 8>(S, cap, st); break;
    case 5121632: launch_sweep<Packed, 512, 16, 32, 2, 8>(S, cap, st); break;
    case 2561208: launch_sweep<Packed, 256, 12, 8, 4, 8>(S, cap, st); break;
    case 5121208: launch_sweep<Packed, 512, 12, 8, 2, 8>(S, cap, st); break;
    // default: 256 threads x 20 keys (5120 per partition), 3 CTAs per SM: with several
    // scans in flight the fewest look-back spins per key (config B, four scans in flight:
    // 275 -> 289 M rays/s against 512 x 12; one sort alone 200 us vs 190 us)
    default: launch_sweep<Packed, 256, 20, kLookW, 3, 8>(S, cap, st); break;
  }
}


// ------------------------------------------------------------------ tile metadata
// [begin, end) of every tile from the tile changes of the sorted keys (tile = key >> b)
__global__ void k_ranges(const uint64_t* __restrict__ keys, const int64_t* __restrict__ scal, int64_t capacity,
                         int id_bits, int2* __restrict__ ranges, int n_tiles) {
  pdl_wait();
  pdl_trigger();
  const int64_t P = min(scal[S_P], capacity);
  const int b = (int)scal[S_B] + id_bits;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(keys[i] >> b);
    SIMULI_CHECK(t < (uint32_t)n_tiles, t, n_tiles);
    SIMULI_CHECK(i == 0 || keys[i - 1] <= keys[i], i, P);  // sorted
    if (i == 0 || (uint32_t)(keys[i - 1] >> b) != t) ranges[t].x = (int)i;
    if (i == P - 1 || (uint32_t)(keys[i + 1] >> b) != t) ranges[t].y = (int)(i + 1);
  }
}

// Longest-first schedule: tiles bucketed by floor(log2(list length)), decreasing (a
// counting sort; the order inside a bucket is whatever the atomics give -- it only affects
// scheduling, never results).  One CTA.
__global__ void __launch_bounds__(1024) k_tile_order(const int2* __restrict__ ranges, int n_tiles,
                                                     int* __restrict__ order) {
  pdl_wait();
  pdl_trigger();
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
    for (int bb = 32; bb >= 0; --bb) {
      s_off[bb] = run;
      run += s_hist[bb];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int2 r = ranges[t];
    const int len = r.y - r.x;
    const int o = atomicAdd(&s_off[len > 0 ? 32 - __clz(len) : 0], 1);
    SIMULI_CHECK(o >= 0 && o < n_tiles && r.x >= 0 && len >= 0, o, len);
    order[o] = t;
  }
}

// (tile << 32 | depth bits) from the trimmed keys
__global__ void k_keys64(const uint64_t* __restrict__ keys, const int64_t* __restrict__ scal, int64_t capacity,
                         int id_bits, uint64_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t P = min(scal[S_P], capacity);
  const int b = (int)scal[S_B];
  const uint32_t kmin = (uint32_t)scal[S_KMIN];
  const uint64_t mask = b >= 64 ? ~0ull : ((1ull << b) - 1ull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i] >> id_bits;
    out[i] = ((k >> b) << 32) | (uint64_t)((uint32_t)(k & mask) + kmin);
  }
}

}  // namespace
}  // namespace simuli

extern "C" int32_t simuli_bin_sort_workspace_size(int64_t n, int64_t cap, int32_t n_tiles, size_t* bytes) {
  using namespace simuli;
  clear_error();
  SIMULI_REQUIRE(bytes && n >= 0 && n_tiles >= 1, "simuli_bin_sort_workspace_size: bad argument");
  if (cap < 0) cap = -cap;
  *bytes = carve(nullptr, n, cap, n_tiles, sort_rb()).bytes;
  return SIMULI_OK;
}

extern "C" int32_t simuli_bin_sort(const simuli_projected* proj, int64_t n, int32_t n_tiles, int32_t n_cols_total,
                                   void* workspace, size_t ws_bytes, int64_t pair_capacity, uint64_t* sorted_keys,
                                   uint32_t* sorted_ids, int32_t* tile_ranges, int32_t* tile_order,
                                   int64_t* n_pairs_dev, int64_t* n_pairs_max_dev, int64_t* pairs_required,
                                   void* stream) {
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
  const int tbits = tile_bits_of(n_tiles);
  SIMULI_REQUIRE(tbits <= 16, "n_tiles must be <= 65536");
  const int rb = sort_rb();
  const Workspace need = carve(nullptr, n, cap, n_tiles, rb);
  SIMULI_REQUIRE(workspace && ws_bytes >= need.bytes, "workspace too small: need %zu bytes", need.bytes);
  Workspace w = carve(workspace, n, cap, n_tiles, rb);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nb = (n + kDupBlock - 1) / kDupBlock;
  auto check = [&](const char* what) -> int32_t {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("simuli_bin_sort: %s: %s", what, cudaGetErrorString(e));
      return SIMULI_ERR_CUDA;
    }
    return SIMULI_OK;
  };
  // one memset zeroes the pass histograms, all counters, the key range and the look-back
  // status words of the count scan and the first sweep pass (each pass clears the next's)
  launch_pdl(k_zero, zero_blocks((int64_t)(w.zero_bytes / 4)), 256, 0, st, reinterpret_cast<uint32_t*>(w.zero),
             (int64_t)(w.zero_bytes / 4));
  uint32_t* ctr = w.counters + kMaxPasses;  // [0] scan block ids, [1] scan blocks done
  if (nb > 0) {
    const int64_t nsb = (n + kScanPer - 1) / kScanPer;
    SIMULI_REQUIRE(reinterpret_cast<uintptr_t>(proj->tile_count) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(proj->depth_key) % 16 == 0,
                   "simuli_bin_sort: tile_count / depth_key must be 16-byte aligned");
    launch_pdl(k_count_scan, (unsigned)nsb, kScanThreads, 0, st, proj->tile_count, proj->depth_key, n, nsb, nb, tbits, rb,
                                                         w.block_sums, w.cstatus, w.kminmax, ctr, w.scal, n_pairs_dev,
                                                         n_pairs_max_dev);
  } else {
    launch_pdl(k_count_empty, 1, 32, 0, st, tbits, w.scal, n_pairs_dev, w.block_sums);
  }
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
  const int max_passes = max_passes_of(tbits, rb);
  uint32_t* vals[2] = {sorted_ids, w.vals_alt};
  // packed mode: depth-key span b <= 31 bits (positive floats), so one u64 word holds
  // (tile << b | depth - min) << id_bits | id whenever 31 + tile bits + id bits <= 64
  int id_bits = 1;
  while (id_bits < 31 && (1ll << id_bits) < n) ++id_bits;
  const bool packed = 31 + tbits + id_bits <= 64;
  if (nb > 0 && cap > 0) {
    DupArgs D{proj->tile_count, reinterpret_cast<const int4*>(proj->tile_rect), proj->depth_key, n, cap,
              w.block_sums, w.scal, n_cols_total, {w.keys[0], w.keys[1]}, {vals[0], vals[1]}, w.hist, nullptr,
              id_bits, packed ? 1 : 0, n_tiles};
    launch_pdl(k_duplicate<kRB>, (unsigned)nb, kDupThreads, 0, st, D);
    if (int32_t e = check("duplicate")) return e;
    for (int p = 0; p < max_passes; ++p) {
      const size_t row = (size_t)w.parts << rb;  // one pass's status words
      SweepArgs S{{w.keys[0], w.keys[1]}, {vals[0], vals[1]}, w.scal, cap, p, id_bits, sorted_ids,
                  w.hist + p * kRadixMax, w.status + p * row, p + 1 < max_passes ? w.status + (p + 1) * row : nullptr,
                  w.counters + p};
      if (packed) launch_sweep_variant<true>(S, cap, st, rb);
      else launch_sweep_variant<false>(S, cap, st, rb);
    }
    if (int32_t e = check("onesweep")) return e;
  }
  const int key_shift = packed ? id_bits : 0;
  launch_pdl(k_zero, zero_blocks(2 * (int64_t)n_tiles), 256, 0, st, reinterpret_cast<uint32_t*>(tile_ranges),
             2 * (int64_t)n_tiles);
  if (cap > 0)
    launch_pdl(k_ranges, 148 * 8, 256, 0, st, w.keys[0], w.scal, cap, key_shift, reinterpret_cast<int2*>(tile_ranges),
                                      n_tiles);
  if (tile_order)
    launch_pdl(k_tile_order, 1, 1024, 0, st, reinterpret_cast<const int2*>(tile_ranges), n_tiles, tile_order);
  if (sorted_keys && cap > 0) launch_pdl(k_keys64, 148 * 4, 256, 0, st, w.keys[0], w.scal, cap, key_shift, sorted_keys);
  return check("tile metadata");
}

#ifdef SIMULI_SORT_PROFILE
extern "C" int32_t simuli_debug_sort_prof(long long* host) {
  return cudaMemcpyFromSymbol(host, simuli::g_sort_prof, sizeof(long long) * simuli::kMaxPasses * 4096 * 8) ==
                 cudaSuccess ? 0 : 3;
}
#endif
