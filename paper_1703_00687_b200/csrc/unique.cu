// radsort_unique_count: run-length "unique key + count" over sorted records --
// the k-mer counting step the paper's sorter serves in KMC3 (PAPER.md:280-282
// §4.2).  Kernels over 4096-record tiles:
//   k_uc_count  run heads per tile (record i starts a run iff i == 0 or its key
//               differs from record i-1's) and the tile's head bitmask
//   k_uc_scan   exclusive scan of the tile counts (one CTA)
//   k_uc_write  the key and start index of every run, at its rank (reads the
//               bitmask and the keys of the heads only)
//   k_uc_len    run lengths from consecutive starts
#include "sorter.cuh"

namespace radsort {
namespace {

constexpr uint32_t UC_T = 4096, UC_B = 256;

template <int R, int K>
__device__ __forceinline__ bool uc_head(const uint8_t* recs, uint64_t i) {
  return i == 0 || !key_eq(ld_key<R, K>(recs + i * R), ld_key<R, K>(recs + (i - 1) * R));
}

template <int R, int K>
__global__ void __launch_bounds__(UC_B) k_uc_count(const uint8_t* __restrict__ recs, uint64_t n,
                                                   uint32_t* __restrict__ tile_cnt, uint32_t* __restrict__ heads) {
  // also writes the run-head bitmask of the tile (bit j of word j / 32: record
  // t0 + j starts a run), so that k_uc_write does not read the keys again
  const uint64_t t0 = (uint64_t)blockIdx.x * UC_T;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t c = 0;
  for (uint32_t j0 = 0; j0 < UC_T; j0 += UC_B) {
    const uint64_t i = t0 + j0 + threadIdx.x;
    const bool h = i < n && uc_head<R, K>(recs, i);
    const uint32_t b = __ballot_sync(0xffffffffu, h);
    if (lane == 0) heads[(size_t)blockIdx.x * (UC_T / 32) + (j0 >> 5) + w] = b;
    c += (uint32_t)h;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[UC_B / 32];
  if (lane == 0) ws[w] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int q = 0; q < UC_B / 32; ++q) s += ws[q];
    tile_cnt[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(1024) k_uc_scan(const uint32_t* __restrict__ tile_cnt, uint32_t ntiles,
                                                  unsigned long long* __restrict__ tile_off,
                                                  unsigned long long* __restrict__ total) {
  __shared__ unsigned long long ws[32];
  __shared__ unsigned long long carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < ntiles; b += 1024) {
    const unsigned long long v = b + tid < ntiles ? tile_cnt[b + tid] : 0ull;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    unsigned long long add = carry;
    for (int i = 0; i < w; ++i) add += ws[i];
    if (b + tid < ntiles) tile_off[b + tid] = add + x - v;
    __syncthreads();
    if (tid == 1023) carry = add + x;
    __syncthreads();
  }
  if (tid == 0) *total = carry;
}

template <int R, int K>
__global__ void __launch_bounds__(UC_T / 32) k_uc_write(const uint8_t* __restrict__ recs,
                                                        const unsigned long long* __restrict__ tile_off,
                                                        const uint32_t* __restrict__ heads, uint8_t* __restrict__ keys_out,
                                                        uint32_t* __restrict__ starts) {
  // one thread per 32-record word of the tile's head bitmask: exclusive scan of
  // the popcounts, then the key and start index of every head (the keys of
  // run heads only are read: ~1 record in 40 on the k-mer stream)
  constexpr int NT = UC_T / 32, NWP = NT / 32;
  __shared__ uint32_t ws[NWP];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t b = heads[(size_t)blockIdx.x * NT + tid];
  const uint32_t c = (uint32_t)__popc(b);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  uint32_t add = 0;
  for (int i = 0; i < w; ++i) add += ws[i];
  unsigned long long u = tile_off[blockIdx.x] + add + x - c;
  const uint64_t base = (uint64_t)blockIdx.x * UC_T + (uint64_t)tid * 32;
  while (b) {
    const uint32_t q = (uint32_t)__ffs(b) - 1u;
    b &= b - 1u;
    const uint64_t i = base + q;
    const Key<K> k = ld_key<R, K>(recs + i * R);
    uint64_t* ko = reinterpret_cast<uint64_t*>(keys_out + u * K);
    ko[0] = k.w0;
    if constexpr (K == 16) ko[1] = k.w1;
    starts[u] = (uint32_t)i;
    ++u;
  }
}

__global__ void k_uc_len(const uint32_t* __restrict__ starts, const unsigned long long* __restrict__ total,
                         uint64_t n, uint32_t* __restrict__ counts) {
  const unsigned long long U = *total;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < U; u += (uint64_t)gridDim.x * blockDim.x)
    counts[u] = (uint32_t)((u + 1 < U ? (uint64_t)starts[u + 1] : n) - starts[u]);
}

template <int R, int K>
radsort_status unique_t(Context* ctx, const uint8_t* recs, uint64_t n, uint8_t* keys_out, uint32_t* counts_out,
                        uint64_t* n_unique, cudaStream_t st) {
  const uint32_t ntiles = (uint32_t)((n + UC_T - 1) / UC_T);
  workspace_acquire(ctx, st);
  radsort_status rs;
  // tile counts + head bitmasks | tile offsets | total, then the run starts (reusing the multi-GPU scratch buffers)
  if ((rs = ensure(ctx->mlo, (size_t)ntiles * 4 + (size_t)ntiles * (UC_T / 8) + 16)) ||
      (rs = ensure(ctx->mlt, (size_t)ntiles * 8 + 16)) || (rs = ensure(ctx->mle, (size_t)n * 4 + 16)))
    return rs;
  uint32_t* tile_cnt = (uint32_t*)ctx->mlo.p;
  uint32_t* heads = tile_cnt + ntiles;
  unsigned long long* tile_off = (unsigned long long*)ctx->mlt.p;
  unsigned long long* total = tile_off + ntiles;
  uint32_t* starts = (uint32_t*)ctx->mle.p;
  k_uc_count<R, K><<<ntiles, UC_B, 0, st>>>(recs, n, tile_cnt, heads);
  k_uc_scan<<<1, 1024, 0, st>>>(tile_cnt, ntiles, tile_off, total);
  k_uc_write<R, K><<<ntiles, UC_T / 32, 0, st>>>(recs, tile_off, heads, keys_out, starts);
  k_uc_len<<<(unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sms * 8), 256, 0, st>>>(starts, total, n,
                                                                                                 counts_out);
  RS_CUDA(cudaGetLastError());
  unsigned long long h_total = 0;
  RS_CUDA(cudaMemcpyAsync(&h_total, total, sizeof h_total, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  workspace_release(ctx, st);
  *n_unique = h_total;
  return RADSORT_OK;
}

}  // namespace
}  // namespace radsort

using namespace radsort;

extern "C" radsort_status radsort_unique_count(const void* dev_sorted, uint64_t n, uint32_t rec_size,
                                               uint32_t key_size, void* dev_keys_out, uint32_t* dev_counts_out,
                                               uint64_t* n_unique, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!n_unique) {
    set_detail("unique_count: n_unique must be non-NULL");
    return RADSORT_ERR_INVALID_ARG;
  }
  *n_unique = 0;
  if (n == 0) return RADSORT_OK;
  if (!dev_sorted || !dev_keys_out || !dev_counts_out) {
    set_detail("unique_count: NULL device pointer with n > 0");
    return RADSORT_ERR_INVALID_ARG;
  }
  if (n >= (1ull << 32)) {
    set_detail("unique_count: n must be < 2^32");
    return RADSORT_ERR_INVALID_ARG;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  Context* ctx = get_or_create_ctx(dev);
  if (!ctx) return RADSORT_ERR_NOT_INITIALIZED;
  std::lock_guard<std::mutex> lk(ctx->mu);
  const uint8_t* r = (const uint8_t*)dev_sorted;
  uint8_t* k = (uint8_t*)dev_keys_out;
#define RS_UC(RR, KK) \
  if (rec_size == RR && key_size == KK) return unique_t<RR, KK>(ctx, r, n, k, dev_counts_out, n_unique, stream)
  RS_UC(8, 8);
  RS_UC(16, 8);
  RS_UC(16, 16);
  RS_UC(24, 8);
  RS_UC(24, 16);
  RS_UC(32, 8);
  RS_UC(32, 16);
  RS_UC(40, 16);
#undef RS_UC
  set_detail("unique_count: layout (%u,%u) not built", rec_size, key_size);
  return RADSORT_ERR_UNSUPPORTED;
}
