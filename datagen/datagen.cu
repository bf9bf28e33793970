// Seeded synthetic record generator -- device twin of datagen/host.py.
//
// Test/bench infrastructure only: it produces inputs for both the CUDA sort and
// the CPU oracle and contains none of the sort's arithmetic.  It shares no
// code with paper_1703_00687_b200/csrc (the product) nor with oracle/.
// The stream definition, distributions and record layout are documented in
// datagen/host.py and DESIGN.md ("Input recipe").
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr int W_DEFAULT = 8;
constexpr int W_ZIPF = 32;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t uw(uint64_t seed, uint64_t i, int w, int W) {
  return mix64(seed + ((uint64_t)W * i + (uint64_t)(w + 1)) * GOLDEN);
}

// Zipf rejection-inversion (Hoermann & Derflinger, ACM TOMACS 1996; helper1/2 in
// the form Apache Commons Math publishes), same constants as host.py
__device__ __forceinline__ double helper1(double x) {
  return fabs(x) > 1e-8 ? log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x));
}
__device__ __forceinline__ double helper2(double x) {
  return fabs(x) > 1e-8 ? expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
}
__device__ __forceinline__ double Hf(double x, double s) { double lx = log(x); return helper2((1.0 - s) * lx) * lx; }
__device__ __forceinline__ double hf(double x, double s) { return exp(-s * log(x)); }
__device__ __forceinline__ double Hinv(double x, double s) {
  double t = x * (1.0 - s);
  if (t < -1.0) t = -1.0;
  return exp(helper1(t) * x);
}

__device__ uint64_t zipf_rank(uint64_t seed, uint64_t i, double N, double s) {
  const double hx1 = Hf(1.5, s) - 1.0;
  const double hN = Hf(N + 0.5, s);
  const double sc = 2.0 - Hinv(Hf(2.5, s) - hf(2.0, s), s);
  double k = 1.0;
  for (int j = 0; j < W_ZIPF; ++j) {
    uint64_t w = uw(seed, i, j, W_ZIPF);
    double U = (double)(w >> 11) * (1.0 / 9007199254740992.0);
    double uu = hN + U * (hx1 - hN);
    double x = Hinv(uu, s);
    k = floor(x + 0.5);
    if (k < 1.0) k = 1.0;
    if (k > N) k = N;
    if (k - x <= sc || uu >= Hf(k + 0.5, s) - hf(k, s)) break;
  }
  return (uint64_t)k;
}

__device__ __forceinline__ uint64_t bytes_word(uint64_t r) {
  uint64_t acc = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    uint32_t sel = (uint32_t)(r >> (8 * b)) & 255u;
    uint64_t v = sel < 86 ? 0ull : (sel < 171 ? 1ull : 255ull);
    acc |= v << (8 * b);
  }
  return acc;
}

// k-mer stream (distribution 9, the KMC3 workload of PAPER.md:280-282): record
// i is the k-mer (k = 55 for 16-byte keys, 31 for 8-byte keys; 2 bits per base,
// first base most significant) read at a uniform position of a pseudo-random
// reference of KMER_L bases (circular); with probability 1/64 one base is
// substituted (a "sequencing error": mostly singleton k-mers).
constexpr uint64_t KMER_L = 1ull << 22;
__device__ __forceinline__ uint64_t kmer_base(uint64_t seed, uint64_t x) {
  return mix64(seed + 0x9E3779B97F4A7C15ull * (x + 0x100000000ull)) & 3ull;
}
__device__ void kmer_key(uint64_t seed, uint64_t i, int KW, uint64_t* key) {
  const int k = KW == 2 ? 55 : 31;
  const uint64_t p = uw(seed, i, 0, W_DEFAULT) % KMER_L, e = uw(seed, i, 1, W_DEFAULT);
  const bool err = (e & 63ull) == 0;
  const int epos = (int)((e >> 8) % (uint64_t)k);
  uint64_t hi = 0, lo = 0;
  for (int j = 0; j < k; ++j) {
    uint64_t b = kmer_base(seed, (p + (uint64_t)j) % KMER_L);
    if (err && j == epos) b = (b + 1ull + ((e >> 16) % 3ull)) & 3ull;
    hi = (hi << 2) | (lo >> 62);
    lo = (lo << 2) | b;
  }
  key[0] = lo;
  key[1] = hi;
}

__global__ void k_generate(uint64_t* __restrict__ out, uint64_t n, uint64_t first, int RW, int KW,
                           int dist, int payload, uint64_t seed) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = first + r;
    uint64_t key[2] = {0, 0};
    switch (dist) {
      case 0:
        if (KW == 1) key[0] = uw(seed, i, 0, W_DEFAULT);
        else { key[0] = uw(seed, i, 1, W_DEFAULT); key[1] = uw(seed, i, 0, W_DEFAULT); }
        break;
      case 2: {
        uint64_t k = zipf_rank(seed, i, 4294967296.0, 1.1);
        if (KW == 1) key[0] = mix64(k);
        else { key[0] = mix64(k + (1ull << 32)); key[1] = mix64(k); }
        break;
      }
      case 8:
        for (int kw = 0; kw < KW; ++kw) key[kw] = bytes_word(uw(seed, i, 4 + kw, W_DEFAULT));
        break;
      case 9:
        kmer_key(seed, i, KW, key);
        break;
      default: {
        uint64_t k;
        switch (dist) {
          case 1: k = uw(seed, i, 0, W_DEFAULT) >> 24; break;
          case 3: k = 0x5555AAAA5555AAAAull; break;
          case 4: k = i; break;
          case 5: k = ~i; break;
          case 6: k = mix64(uw(seed, i, 0, W_DEFAULT) % 7ull); break;
          default: k = (0xABCDEFull << 40) | (uw(seed, i, 0, W_DEFAULT) >> 24); break;  // 7
        }
        if (KW == 1) key[0] = k;
        else if (dist >= 3 && dist <= 6) { key[0] = k; key[1] = k; }
        else { key[0] = uw(seed, i, 1, W_DEFAULT); key[1] = k; }
      }
    }
    uint64_t* rec = out + r * (uint64_t)RW;
    for (int w = 0; w < KW; ++w) rec[w] = key[w];
    for (int w = KW; w < RW; ++w)
      rec[w] = (payload == 1 && w == KW) ? i : uw(seed, i, w, W_DEFAULT);
  }
}

}  // namespace

extern "C" {

// Fill dev_out[0..n) with records [first, first+n) of the given stream.
// Returns 0 on success, a cudaError_t value otherwise.
int datagen_fill(void* dev_out, uint64_t n, uint64_t first, uint32_t R, uint32_t K, int dist,
                 int payload, uint64_t seed, cudaStream_t stream) {
  if (n == 0) return 0;
  if (!dev_out || R % 8 || K % 8 || K < 8 || K > 16 || K > R || R > 64) return (int)cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (n + 255) / 256;
  unsigned grid = (unsigned)(want < (uint64_t)sms * 16 ? want : (uint64_t)sms * 16);
  k_generate<<<grid, 256, 0, stream>>>((uint64_t*)dev_out, n, first, (int)(R / 8), (int)(K / 8), dist,
                                       payload, seed);
  return (int)cudaGetLastError();
}

}
