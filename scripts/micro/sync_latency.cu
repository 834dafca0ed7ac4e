// Microbenchmark: producer/consumer hand-off latency between two warps of one CTA on
// sm_100a (mbarrier try_wait with / without suspend hint, volatile shared flag, named
// barrier).  Round trip = warp 0 signals warp 1, warp 1 signals back.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_latency sync_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("{.reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(sa(b)) : "memory");
}
template <int HINT>
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned par) {
  unsigned ok;
  do {
    if (HINT)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(sa(b)), "r"(par), "n"(HINT) : "memory");
    else
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  } while (!ok);
}

template <int MODE, int HINT>
__global__ void k_pingpong(int iters, long long* out, int busy_warps) {
  __shared__ unsigned long long bar[2];
  __shared__ volatile int flag[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mb_init(&bar[0]); mb_init(&bar[1]); flag[0] = flag[1] = -1; }
  __syncthreads();
  if (warp >= 2) {  // background load: dependent FMA chains
    float x = lane;
    for (int i = 0; i < iters * 64; ++i) x = fmaf(x, 1.0000001f, 0.5f);
    if (x == 12345.f) out[9] = 1;
    return;
  }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (warp == 0) {
      if (MODE == 0) { __syncwarp(); if (lane == 0) mb_arrive(&bar[0]); mb_wait<HINT>(&bar[1], i & 1); }
      if (MODE == 1) { __syncwarp(); if (lane == 0) flag[0] = i; while (flag[1] != i) {} }
      if (MODE == 2) { asm volatile("bar.arrive 1, 64;" ::: "memory"); asm volatile("bar.sync 2, 64;" ::: "memory"); }
    } else {
      if (MODE == 0) { mb_wait<HINT>(&bar[0], i & 1); __syncwarp(); if (lane == 0) mb_arrive(&bar[1]); }
      if (MODE == 1) { while (flag[0] != i) {} __syncwarp(); if (lane == 0) flag[1] = i; }
      if (MODE == 2) { asm volatile("bar.sync 1, 64;" ::: "memory"); asm volatile("bar.arrive 2, 64;" ::: "memory"); }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

template <int MODE, int HINT>
void run(const char* name, int busy) {
  long long* d; cudaMalloc(&d, 16 * sizeof(long long));
  k_pingpong<MODE, HINT><<<1, 64 + 32 * busy>>>(1000, d, busy);
  k_pingpong<MODE, HINT><<<1, 64 + 32 * busy>>>(10000, d, busy);
  long long h = 0; cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%-28s busy warps %2d: round trip %lld cycles %s\n", name, busy, h, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}
int main() {
  for (int busy : {0, 14}) {
    run<0, 0>("mbarrier try_wait", busy);
    run<0, 1000>("mbarrier try_wait hint 1us", busy);
    run<0, 10000000>("mbarrier try_wait hint 10ms", busy);
    run<1, 0>("volatile smem flag", busy);
    run<2, 0>("named barrier", busy);
  }
  return 0;
}
