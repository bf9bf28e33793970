// radsort_tinybench: the GPU analog of the paper's tiny-sorter experiment
// (§4.1, Fig. 1: time per element of the tiny-array sorters
// for n = 2..64 and several record layouts), used to choose the size classes
// of the tiny-bin sorters (R4).
//
// `bins` arrays of n records each, keys sharing their most significant digit
// (as every bin at depth >= 1 does), are sorted in global memory by one of the
// library's own device sorters:
//   0  enumeration sort, one record per lane (es_rank; n <= 32)
//   1  warp bitonic network on packed sort keys (warp_tiny_sort)
//   2  warp tail sorter: counting pass on the next digit + ES among
//      the few colliders (warp_tail_sort; the k_children default)
//   3  insertion sort, one thread per bin (lane_insertion_sort)
// Timed with CUDA events; the output is checked on the device (every bin
// non-decreasing and a permutation of its input).  radsort_tinysort runs one
// sorter on caller-provided arrays (for the tests of each sorter).
// Benchmark / test infrastructure: not on the sort path.
#include "sorter.cuh"

namespace radsort {
namespace {

__device__ __forceinline__ uint64_t tb_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// record i of bin b: random key whose top byte is the bin's (shared) digit 0
template <int R, int K>
__global__ void tb_fill(uint8_t* buf, uint64_t total, uint32_t n, uint64_t seed) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  uint64_t* w = reinterpret_cast<uint64_t*>(buf + i * R);
  const uint64_t top = (uint64_t)(i / n & 255u) << 56;
  for (int j = 0; j < R / 8; ++j) w[j] = tb_mix(seed + i * 8 + j);
  w[K / 8 - 1] = (w[K / 8 - 1] & 0x00FFFFFFFFFFFFFFull) | top;
}

template <int R, int K>
__global__ void tb_sort_warp(const uint8_t* src, uint8_t* dst, uint64_t bins, uint32_t n, int algo) {
  __shared__ __align__(16) TailScratch<K> ws[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t b = blockIdx.x * 8ull + warp; b < bins; b += gridDim.x * 8ull) {
    const uint8_t* s = src + b * n * R;
    uint8_t* o = dst + b * n * R;
    if (algo == 0) {
      Rec<R> x;
      uint32_t rank = 0;
      if ((uint32_t)lane < n) {
        x = ld_rec<R>(s + (size_t)lane * R);
        rank = es_rank<R, K>(s, n, (uint32_t)lane, key_of<R, K>(x));
      }
      if ((uint32_t)lane < n) st_rec<R>(o + (size_t)rank * R, x);
    } else if (algo == 1) {
      warp_tiny_sort<R, K>(s, o, n, 1, lane);
    } else {
      warp_tail_sort<R, K>(s, o, n, 1, lane, ws[warp]);
    }
  }
}

template <int R, int K>
__global__ void tb_sort_thread(const uint8_t* src, uint8_t* dst, uint64_t bins, uint32_t n) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= bins) return;
  const uint8_t* s = src + b * n * R;
  uint8_t* o = dst + b * n * R;
  for (uint32_t i = 0; i < n; ++i) st_rec<R>(o + (size_t)i * R, ld_rec<R>(s + (size_t)i * R));
  lane_insertion_sort<R, K>(o, n);
}

// Output check of every array: keys non-decreasing, and the array is a
// permutation of its input (order-independent digests of the full records:
// sum and xor of a 64-bit mix of (word, word index) over the array).
template <int R, int K>
__global__ void tb_check(const uint8_t* in, const uint8_t* buf, uint64_t bins, uint32_t n, unsigned int* bad) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= bins) return;
  const uint8_t* s = buf + b * n * R;
  const uint8_t* x = in + b * n * R;
  for (uint32_t i = 1; i < n; ++i)
    if (key_lt(ld_key<R, K>(s + (size_t)i * R), ld_key<R, K>(s + (size_t)(i - 1) * R))) atomicAdd(bad, 1u);
  uint64_t sa = 0, xa = 0, sb = 0, xb = 0;
  for (uint32_t i = 0; i < n; ++i)
    for (int j = 0; j < R / 8; ++j) {
      const uint64_t u = tb_mix(reinterpret_cast<const uint64_t*>(s + (size_t)i * R)[j] ^ ((uint64_t)j << 56));
      const uint64_t v = tb_mix(reinterpret_cast<const uint64_t*>(x + (size_t)i * R)[j] ^ ((uint64_t)j << 56));
      sa += u; xa ^= u; sb += v; xb ^= v;
    }
  if (sa != sb || xa != xb) atomicAdd(bad, 1u);
}

template <int R, int K>
void tb_launch(const uint8_t* src, uint8_t* dst, uint64_t bins, uint32_t n, uint32_t algo, cudaStream_t st) {
  if (algo == 3) tb_sort_thread<R, K><<<(unsigned)((bins + 127) / 128), 128, 0, st>>>(src, dst, bins, n);
  else tb_sort_warp<R, K><<<(unsigned)std::min<uint64_t>((bins + 7) / 8, 148ull * 64), 256, 0, st>>>(src, dst, bins, n, (int)algo);
}

template <int R, int K>
radsort_status tinybench_t(uint32_t n, uint32_t algo, uint64_t bins, double* ns_per_record) {
  if (n < 2 || n > TINY_MAX || (algo == 0 && n > 32) || algo > 3) {
    set_detail("tinybench: n in [2, %u] (ES: n <= 32), algo in 0..3", TINY_MAX);
    return RADSORT_ERR_INVALID_ARG;
  }
  const uint64_t total = bins * n;
  uint8_t *src = nullptr, *dst = nullptr;
  unsigned int* bad = nullptr;
  RS_CUDA(cudaMalloc(&src, total * R));
  RS_CUDA(cudaMalloc(&dst, total * R));
  RS_CUDA(cudaMalloc(&bad, sizeof(unsigned int)));
  RS_CUDA(cudaMemset(bad, 0, sizeof(unsigned int)));
  tb_fill<R, K><<<(unsigned)((total + 255) / 256), 256>>>(src, total, n, 0x7B5ull);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    tb_launch<R, K>(src, dst, bins, n, algo, 0);
    cudaEventRecord(e1);
    RS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  tb_check<R, K><<<(unsigned)((bins + 255) / 256), 256>>>(src, dst, bins, n, bad);
  unsigned int h_bad = 0;
  RS_CUDA(cudaMemcpy(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(src);
  cudaFree(dst);
  cudaFree(bad);
  if (h_bad) {
    set_detail("tinybench: %u out-of-order pairs or non-permuted arrays (algo %u, n %u)", h_bad, algo, n);
    return RADSORT_ERR_CUDA;
  }
  *ns_per_record = (double)best * 1e6 / (double)total;
  return RADSORT_OK;
}

template <int R, int K>
radsort_status tinysort_t(uint32_t n, uint32_t algo, const uint8_t* in, uint8_t* out, uint64_t bins, cudaStream_t st) {
  if (n < 2 || n > TINY_MAX || (algo == 0 && n > 32) || algo > 3) {
    set_detail("tinysort: n in [2, %u] (ES: n <= 32), algo in 0..3", TINY_MAX);
    return RADSORT_ERR_INVALID_ARG;
  }
  tb_launch<R, K>(in, out, bins, n, algo, st);
  RS_CUDA(cudaGetLastError());
  return RADSORT_OK;
}

}  // namespace
}  // namespace radsort

using namespace radsort;

extern "C" radsort_status radsort_tinybench(uint32_t rec_size, uint32_t key_size, uint32_t n, uint32_t algo,
                                            uint64_t bins, double* ns_per_record) {
  if (!ns_per_record || bins == 0) {
    set_detail("tinybench: ns_per_record must be non-NULL and bins > 0");
    return RADSORT_ERR_INVALID_ARG;
  }
  if (rec_size == 8 && key_size == 8) return tinybench_t<8, 8>(n, algo, bins, ns_per_record);
  if (rec_size == 16 && key_size == 8) return tinybench_t<16, 8>(n, algo, bins, ns_per_record);
  if (rec_size == 16 && key_size == 16) return tinybench_t<16, 16>(n, algo, bins, ns_per_record);
  if (rec_size == 32 && key_size == 8) return tinybench_t<32, 8>(n, algo, bins, ns_per_record);
  if (rec_size == 32 && key_size == 16) return tinybench_t<32, 16>(n, algo, bins, ns_per_record);
  set_detail("tinybench: layout (%u,%u) not built", rec_size, key_size);
  return RADSORT_ERR_UNSUPPORTED;
}

extern "C" radsort_status radsort_tinysort(uint32_t rec_size, uint32_t key_size, uint32_t n, uint32_t algo,
                                           const void* dev_in, void* dev_out, uint64_t bins, void* stream) {
  if (bins == 0) return RADSORT_OK;
  if (!dev_in || !dev_out || dev_in == dev_out) {
    set_detail("tinysort: distinct non-NULL device buffers required");
    return RADSORT_ERR_INVALID_ARG;
  }
  const cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* in = (const uint8_t*)dev_in;
  uint8_t* out = (uint8_t*)dev_out;
  if (rec_size == 8 && key_size == 8) return tinysort_t<8, 8>(n, algo, in, out, bins, st);
  if (rec_size == 16 && key_size == 8) return tinysort_t<16, 8>(n, algo, in, out, bins, st);
  if (rec_size == 16 && key_size == 16) return tinysort_t<16, 16>(n, algo, in, out, bins, st);
  if (rec_size == 32 && key_size == 8) return tinysort_t<32, 8>(n, algo, in, out, bins, st);
  if (rec_size == 32 && key_size == 16) return tinysort_t<32, 16>(n, algo, in, out, bins, st);
  set_detail("tinysort: layout (%u,%u) not built", rec_size, key_size);
  return RADSORT_ERR_UNSUPPORTED;
}
