// Microbenchmark (not part of the library): how fast can B200 HBM absorb a
// radix scatter that writes every record on its own, with no shared-memory
// staging?  Records of R bytes are read coalesced and each is stored at
// dest[i] * R, where dest is the stable partition of the records into F
// streams (stream = hash(i) mod F) inside segments of S records -- the write
// pattern of one radix pass with fan-out F over bins of S records.  F = 1 is a
// plain copy.  For R = 32 every record is one full 32-byte sector, so the
// question is whether L2 / HBM keep full speed when consecutive stores of a
// warp hit F different write fronts.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubs tools/ubench_scatter.cu && /tmp/ubs
#include <cub/cub.cuh>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// sort key: segment index (high bits) | stream (low bits); stable sort by it
// gives the pass's output order
__global__ void k_keys(uint64_t* key, uint32_t* idx, uint64_t n, uint64_t S, uint32_t F) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t seg = i / S;
    key[i] = (seg << 32) | (F > 1 ? (uint32_t)(mix64(i + 12345) % F) : 0u);
    idx[i] = (uint32_t)i;
  }
}
__global__ void k_inv(const uint32_t* order, uint32_t* dest, uint64_t n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    dest[order[j]] = (uint32_t)j;
}

template <int R> struct V;
template <> struct V<8> { using T = uint2; };
template <> struct V<16> { using T = uint4; };
template <> struct V<32> { struct T { uint4 a, b; }; };

template <int R, int U>
__global__ void __launch_bounds__(256) k_scatter(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                 const uint32_t* __restrict__ dest, uint64_t n) {
  using T = typename V<R>::T;
  const uint64_t stride = (uint64_t)gridDim.x * 256 * U;
  for (uint64_t b = (uint64_t)blockIdx.x * 256 * U; b < n; b += stride) {
    T r[U];
    uint32_t d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + u * 256 + threadIdx.x;
      if (i < n) {
        r[u] = reinterpret_cast<const T*>(src)[i];
        d[u] = __ldg(dest + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + u * 256 + threadIdx.x;
      if (i < n) reinterpret_cast<T*>(dst)[d[u]] = r[u];
    }
  }
}

template <int R>
void run(uint64_t n, uint8_t* a, uint8_t* c, uint64_t* key, uint64_t* key2, uint32_t* idx, uint32_t* idx2,
         uint32_t* dest, void* tmp, size_t tmpb, uint64_t S, uint32_t F, int sms) {
  k_keys<<<sms * 8, 256>>>(key, idx, n, S, F);
  size_t tb = tmpb;
  CK(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, (int64_t)n));
  k_inv<<<sms * 8, 256>>>(idx2, dest, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    cudaEventRecord(e0);
    k_scatter<R, 4><<<sms * 8, 256>>>(a, c, dest, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  const double rec = 2.0 * n * R / (best * 1e-3) / 1e9, all = (2.0 * n * R + 4.0 * n) / (best * 1e-3) / 1e9;
  printf("R=%2d n=%llu S=%-10llu F=%-6u %8.3f ms  records %6.0f GB/s  (+dest idx %6.0f GB/s)\n", R,
         (unsigned long long)n, (unsigned long long)S, F, best, rec, all);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t bytes = 8ull << 30;
  uint8_t *a, *c;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&c, bytes));
  CK(cudaMemset(a, 1, bytes));
  const uint64_t nmax = bytes / 8;
  uint64_t *key, *key2;
  uint32_t *idx, *idx2, *dest;
  CK(cudaMalloc(&key, nmax * 8));
  CK(cudaMalloc(&key2, nmax * 8));
  CK(cudaMalloc(&idx, nmax * 4));
  CK(cudaMalloc(&idx2, nmax * 4));
  CK(cudaMalloc(&dest, nmax * 4));
  size_t tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, key, key2, idx, idx2, (int64_t)nmax);
  void* tmp;
  CK(cudaMalloc(&tmp, tmpb));
  struct Cfg { uint64_t S; uint32_t F; };
  // whole array (level 0), 3.9 M-record segments (level 1 of 1 G), 15.3 K-record bins (local phase)
  const std::vector<Cfg> cfgs = {{~0ull >> 1, 1},   {~0ull >> 1, 256},  {~0ull >> 1, 2048}, {~0ull >> 1, 65536},
                                 {3906250, 256},    {3906250, 1024},    {3906250, 2048},    {3906250, 4096},
                                 {15259, 65536},    {15259, 16384},     {1907, 4096}};
  for (const Cfg& g : cfgs) run<32>(bytes / 32, a, c, key, key2, idx, idx2, dest, tmp, tmpb, g.S, g.F, sms);
  for (const Cfg& g : cfgs) run<16>(bytes / 16, a, c, key, key2, idx, idx2, dest, tmp, tmpb, g.S, g.F, sms);
  for (const Cfg& g : cfgs) run<8>(bytes / 8, a, c, key, key2, idx, idx2, dest, tmp, tmpb, g.S, g.F, sms);
  return 0;
}
