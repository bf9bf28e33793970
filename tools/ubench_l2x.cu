// Microbenchmark (not part of the library): the medium a cluster-local sort
// can move records between SMs through.  Every CTA holds 4096 records of 32 B
// (128 KB) and stores each one to a pseudo-random slot of its group's
// 4 x 128 KB region (the record's place in the sorted bin, owned by one of
// the 4 CTAs), then the group synchronises and repeats:
//   dsmem : the region is the 4 CTAs' shared memory (cluster of 4, DSMEM
//           stores) -- what k_local_cluster does today;
//   l2    : the region is a 512 KB global scratch per group (L2-resident:
//           148 x 128 KB = 19 MB), random 32-byte stores, then each CTA reads
//           its 128 KB back coalesced (the owner's slice);
//   l2seq : as l2 but the stores are coalesced (the bound for l2).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_l2x tools/ubench_l2x.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NB = 512, IL = 8, N = NB * IL;  // records per CTA
struct Rec { uint4 a, b; };

__device__ __forceinline__ uint32_t perm(uint32_t i, uint32_t it) {  // bijection on [0, 4N)
  return ((i * 0x9E3779B1u) + it * 0x85EBCA6Bu) & (4 * N - 1);
}

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(NB, 1) k_dsmem(int iters, uint64_t* sink) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ uint4 sm[];
  Rec* st = reinterpret_cast<Rec*>(sm);
  const uint32_t cr = cl.block_rank();
  Rec r[IL];
#pragma unroll
  for (int i = 0; i < IL; ++i) r[i] = {make_uint4(i, cr, threadIdx.x, 1), make_uint4(2, 3, 4, 5)};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const uint32_t g = perm(cr * N + i * NB + threadIdx.x, it);
      Rec* dst = cl.map_shared_rank(st, g / N);
      dst[g % N] = r[i];
    }
    cl.sync();
#pragma unroll
    for (int i = 0; i < IL; ++i) r[i] = st[i * NB + threadIdx.x];
    cl.sync();
  }
  uint64_t x = 0;
#pragma unroll
  for (int i = 0; i < IL; ++i) x += r[i].a.x + r[i].b.w;
  if (x == 12345) sink[0] = x;
}

template <bool SEQ>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(NB, 1) k_l2(Rec* scratch, int iters, uint64_t* sink) {
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t cr = cl.block_rank();
  Rec* reg = scratch + (size_t)(blockIdx.x / 4) * 4 * N;  // the group's 512 KB
  Rec r[IL];
#pragma unroll
  for (int i = 0; i < IL; ++i) r[i] = {make_uint4(i, cr, threadIdx.x, 1), make_uint4(2, 3, 4, 5)};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const uint32_t li = cr * N + i * NB + threadIdx.x;
      const uint32_t g = SEQ ? li : perm(li, it);
      __stcg(&reg[g].a, r[i].a);
      __stcg(&reg[g].b, r[i].b);
    }
    cl.sync();
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const Rec* p = reg + cr * N + i * NB + threadIdx.x;
      r[i].a = __ldcg(&p->a);
      r[i].b = __ldcg(&p->b);
    }
    cl.sync();
  }
  uint64_t x = 0;
#pragma unroll
  for (int i = 0; i < IL; ++i) x += r[i].a.x + r[i].b.w;
  if (x == 12345) sink[0] = x;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 400;
  Rec* scratch;
  uint64_t* sink;
  CK(cudaMalloc(&scratch, (size_t)sms * N * sizeof(Rec)));
  CK(cudaMalloc(&sink, 8));
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, N * 32));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto grid_of = [&](const void* f, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms, 1, 1);
    cfg.blockDim = dim3(NB, 1, 1);
    cfg.dynamicSmemBytes = smem;
    int nc = 0;
    cudaOccupancyMaxActiveClusters(&nc, f, &cfg);
    return nc * 4;
  };
  for (int mode = 0; mode < 3; ++mode) {
    const int g = mode == 0 ? grid_of((const void*)k_dsmem, N * 32)
                            : grid_of(mode == 1 ? (const void*)k_l2<false> : (const void*)k_l2<true>, 0);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_dsmem<<<g, NB, N * 32>>>(iters, sink);
      else if (mode == 1) k_l2<false><<<g, NB>>>(scratch, iters, sink);
      else k_l2<true><<<g, NB>>>(scratch, iters, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    const double moved = (double)g * iters * N * 32;  // bytes stored (and read back) per launch
    const double cyc = best * 1e-3 * 1.965e9 / iters;  // per iteration
    printf("%-6s CTAs %3d: %8.3f ms  %7.0f GB/s of records stored  %6.0f cycles per 128 KB per CTA (store + sync + read + sync)\n",
           mode == 0 ? "dsmem" : (mode == 1 ? "l2" : "l2seq"), g, best, moved / (best * 1e-3) / 1e9, cyc);
  }
  return 0;
}
