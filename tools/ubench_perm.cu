// Microbenchmark for the CTA-local sorter's write pattern: every record of a
// bin (2^LB2 records, R bytes) is read coalesced into registers and written to
// a pseudo-random position inside the same bin (an odd-multiplier bijection),
// i.e. the pattern of a direct-to-final-position local sort with no smem
// staging.  Compared with a plain copy.  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

template <int R> struct V;
template <> struct V<8> { using T = uint2; };
template <> struct V<16> { using T = uint4; };

template <int R, int LB2, int B, int PERM>
__global__ void __launch_bounds__(B) k_perm(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint32_t nbins) {
  using T = typename V<R>::T;
  constexpr uint32_t N = 1u << LB2;
  constexpr int IL = (int)(N / B);
  for (uint32_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    const T* s = reinterpret_cast<const T*>(src + (size_t)b * N * R);
    T* d = reinterpret_cast<T*>(dst + (size_t)b * N * R);
    T r[IL];
#pragma unroll
    for (int i = 0; i < IL; ++i) r[i] = __ldg(s + i * B + threadIdx.x);
    __syncthreads();  // all loads of the bin land before any store (as in the sorter)
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const uint32_t idx = i * B + threadIdx.x;
      const uint32_t p = PERM ? ((idx * 0x9E3779B1u + b * 0x85EBCA6Bu) & (N - 1)) : idx;
      d[p] = r[i];
    }
  }
}

template <int R, int LB2, int B, int PERM>
int run(uint8_t* a, uint8_t* c, size_t bytes, int occ_per_sm, int sms) {
  const uint32_t nbins = (uint32_t)(bytes / ((size_t)R << LB2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int g = sms * occ_per_sm;
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_perm<R, LB2, B, PERM><<<g, B>>>(a, c, nbins);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("R=%2d bin=2^%d (%6zu B) B=%4d grid=%d perm=%d : %.3f ms  %.0f GB/s (r+w)\n", R, LB2, (size_t)R << LB2, B, g, PERM,
         best, 2.0 * nbins * ((size_t)R << LB2) / best / 1e6);
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 8ull << 30;
  uint8_t *a, *c;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&c, bytes));
  CK(cudaMemset(a, 1, bytes)); CK(cudaMemset(c, 0, bytes));
  for (int occ : {1, 2, 4}) {
    run<8, 14, 512, 0>(a, c, bytes, occ, sms);
    run<8, 14, 512, 1>(a, c, bytes, occ, sms);
    run<8, 14, 1024, 1>(a, c, bytes, occ, sms);
    run<16, 12, 512, 0>(a, c, bytes, occ, sms);
    run<16, 12, 512, 1>(a, c, bytes, occ, sms);
    run<16, 12, 256, 1>(a, c, bytes, occ, sms);
  }
  return 0;
}
