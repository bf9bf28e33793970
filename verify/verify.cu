// Test/bench-side checker kernels (NOT part of the sort): sortedness scan and
// an order-independent multiset digest of records.  Used for full-size
// (BASELINE.json) parity where the oracle cannot hold the data: a result is
// correct iff it is sorted by key and is a permutation of the input
// (DESIGN.md "Parity").  Shares no code with the product or the oracle.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ uint64_t mixv(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// key compare: words K/8-1 .. 0 (high word first), little-endian words
__device__ __forceinline__ bool gt(const uint64_t* a, const uint64_t* b, int KW) {
  for (int w = KW - 1; w >= 0; --w)
    if (a[w] != b[w]) return a[w] > b[w];
  return false;
}
__global__ void k_sorted(const uint64_t* __restrict__ r, uint64_t n, int RW, int KW, unsigned long long* bad,
                         unsigned long long* first_bad) {
  unsigned long long cnt = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (gt(r + i * RW, r + (i + 1) * RW, KW)) {
      ++cnt;
      atomicMin(first_bad, (unsigned long long)i);
    }
  }
  if (cnt) atomicAdd(bad, cnt);
}
__global__ void k_digest(const uint64_t* __restrict__ r, uint64_t n, int RW, unsigned long long* out) {
  uint64_t s = 0, x = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = 0x243F6A8885A308D3ull;
    for (int w = 0; w < RW; ++w) h = mixv(h ^ r[i * RW + w]);
    s += h;
    x ^= mixv(h + 0x13198A2E03707344ull);
  }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    x ^= __shfl_xor_sync(0xffffffffu, x, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], (unsigned long long)s);
    atomicXor(&out[1], (unsigned long long)x);
  }
}
}  // namespace

extern "C" {
// out[0] = number of adjacent key inversions, out[1] = first inversion index (or ~0)
int verify_sorted(const void* dev, uint64_t n, uint32_t R, uint32_t K, unsigned long long* host_out) {
  unsigned long long* d;
  if (cudaMalloc(&d, 16) != cudaSuccess) return 1;
  unsigned long long init[2] = {0, ~0ull};
  cudaMemcpy(d, init, 16, cudaMemcpyHostToDevice);
  if (n > 1) k_sorted<<<1184, 256>>>((const uint64_t*)dev, n, R / 8, K / 8, d, d + 1);
  cudaError_t e = cudaMemcpy(host_out, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? (int)cudaGetLastError() : (int)e;
}
// out[0] = sum of per-record hashes, out[1] = xor of re-mixed hashes
int verify_digest(const void* dev, uint64_t n, uint32_t R, unsigned long long* host_out) {
  unsigned long long* d;
  if (cudaMalloc(&d, 16) != cudaSuccess) return 1;
  cudaMemset(d, 0, 16);
  if (n) k_digest<<<1184, 256>>>((const uint64_t*)dev, n, R / 8, d);
  cudaError_t e = cudaMemcpy(host_out, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? (int)cudaGetLastError() : (int)e;
}
}
