// Reference timing only (not product code): CUB DeviceRadixSort on N random u64 keys with
// `bits` significant bits (begin_bit 0, end_bit bits), pairs (u64 key, u32 value) and
// keys-only, to compare against libsimuli's onesweep passes.  nvcc -O3 -arch=sm_100a
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 1750000;
  const int bits = argc > 2 ? atoi(argv[2]) : 38;
  std::vector<unsigned long long> h(n);
  std::mt19937_64 rng(1);
  for (auto& x : h) x = rng() & ((1ull << bits) - 1);
  unsigned long long *k0, *k1; unsigned *v0, *v1;
  cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  cudaMemcpy(k0, h.data(), n * 8, cudaMemcpyHostToDevice);
  size_t tb = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)n, 0, bits);
  cub::DeviceRadixSort::SortKeys(nullptr, tb2, k0, k1, (int)n, 0, bits);
  void* tmp; cudaMalloc(&tmp, tb > tb2 ? tb : tb2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int i = 0; i < 3; ++i) {
      if (mode == 0) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n, 0, bits);
      else cub::DeviceRadixSort::SortKeys(tmp, tb2, k0, k1, (int)n, 0, bits);
    }
    const int reps = 50;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) {
      if (mode == 0) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n, 0, bits);
      else cub::DeviceRadixSort::SortKeys(tmp, tb2, k0, k1, (int)n, 0, bits);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("CUB %s n=%ld bits=%d: %.1f us\n", mode == 0 ? "SortPairs(u64,u32)" : "SortKeys(u64)", n, bits, ms * 1e3 / reps);
  }
  return 0;
}
