// radsort device code: the MSD radix-sort hot path for sm_100a.
//
// PAPER.md:35 §1 (MSD radix sort: partition by the most significant digit,
// recurse into bins), §3.1 (1 B digits; whole-array pass,
// then small bins, then tiny bins), §3.2 (small-bin counting
// scatter; buffered, aligned scatter), §3.3 (tiny-bin
// sorters; <=256-record bins skip empty/singleton sub-bins).  The GPU mapping
// of each step is described in DESIGN.md §3 ("Kernels").
//
// Shares no code with oracle/ or datagen/.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace radsort {

constexpr int RADIX = 256;
constexpr uint32_t TINY_MAX = 128;     // warp tiny sorter ceiling ("up to about a hundred")
constexpr int HIST_B = 256;            // threads per histogram CTA
constexpr int CHILD_B = 256;           // threads per children CTA
constexpr int LOCAL_SMEM_BYTES = 131072;  // CTA-local sorter capacity in bytes

template <int R> __host__ __device__ constexpr uint32_t local_capacity() { return (uint32_t)(LOCAL_SMEM_BYTES / R); }
// Records per scatter/histogram tile of TB bytes: a multiple of the scatter CTA size SB.
template <int R, int TB, int SB> __host__ __device__ constexpr uint32_t tile_recs() { return (uint32_t)((TB / R) / SB * SB); }

enum : uint8_t { SRC_REC = 0, SRC_TMP = 1 };
enum : uint8_t { MODE_NONE = 0, MODE_SCATTER = 1, MODE_COPY = 2, MODE_SPLIT = 3, MODE_FILL = 4 };
enum : uint8_t { FLAG_EQUAL = 1, FLAG_FILL = 2, FLAG_CAND = 4 };  // CAND: sampled as possibly key-dominated
// Bits [4, 7) of Seg::flags: how many leading bits of digit `depth` the bin's
// keys already share (2 for the children of a 10-bit pass, DESIGN.md §3 "wide
// level"; 0 otherwise).  Only the CTA-local sorters read it (their composite
// digit starts below the shared bits); every other step is correct without it.
constexpr int FLAG_SKIP_SHIFT = 4;
constexpr uint8_t FLAG_SKIP_MASK = 7u << FLAG_SKIP_SHIFT;
__host__ __device__ __forceinline__ uint32_t seg_skip(uint8_t flags) { return (flags >> FLAG_SKIP_SHIFT) & 7u; }

// A bin ("bins that may be further processed independently"):
// record range [off, off+len) of buffer `src`, to be partitioned by digit `depth`.
// `aux`: for a FLAG_FILL bin, the index of its key in the probe-key table.
struct Seg {
  uint32_t off;
  uint32_t len;
  uint8_t depth;
  uint8_t src;
  uint8_t mode;
  uint8_t flags;
  uint32_t aux;
};
static_assert(sizeof(Seg) == 16, "Seg is 16 bytes");

// Device-resident control block; the host reads it once per MSD level.
struct Ctl {
  uint32_t n_large_next;   // entries appended to Large[nxt] this level
  uint32_t n_local[2];     // Local list counts (by parity)
  uint32_t max_local_len[2];
  uint32_t tiles_total;    // tiles of this level's Large list
  uint32_t scatter_ticket; // decoupled look-back tile ticket
  uint32_t d0;             // first digit of the level-0 pass (from k_sample)
  unsigned long long rec_hist, rec_scatter, rec_copy, rec_tiny, rec_local, rec_final;
  unsigned long long bins_large, bins_local, bins_tiny, bins_final;
  unsigned long long bins_split, rec_split;  // dominant-key three-way splits (segments, records of the key)
  uint32_t n_probe;                          // probe-key table entries used this sort
  uint32_t n_local_small[2];                 // Local list entries of <= small_cap<R>() records (by parity)
  uint32_t n_local_med[2];                   // ... of small_cap < len <= med_cap<R>() records
  uint32_t dup_est;                          // k_dupest: sampled keys that met an equal earlier sample
  unsigned long long rec_large_next;          // records of the entries appended to Large[nxt] this level
  unsigned long long prof[16];  // phase cycle counters (RADSORT_PHASE_PROF builds only)
};

// ------------------------------------------------------------------ records
template <int R> struct Rec;
template <> struct Rec<8> { uint2 a; };
template <> struct Rec<16> { uint4 a; };
template <> struct Rec<32> { uint4 a, b; };
template <> struct Rec<24> { uint2 a, b, c; };        // 8-byte aligned (SPEC.md:28-30 layouts (8,16), (16,8))
template <> struct Rec<40> { uint2 a, b, c, d, e; };  // 8-byte aligned (layout (16,24))

template <int R> __device__ __forceinline__ Rec<R> ld_rec(const uint8_t* p);
template <> __device__ __forceinline__ Rec<8> ld_rec<8>(const uint8_t* p) { return {*reinterpret_cast<const uint2*>(p)}; }
template <> __device__ __forceinline__ Rec<16> ld_rec<16>(const uint8_t* p) { return {*reinterpret_cast<const uint4*>(p)}; }
template <> __device__ __forceinline__ Rec<32> ld_rec<32>(const uint8_t* p) {
  return {reinterpret_cast<const uint4*>(p)[0], reinterpret_cast<const uint4*>(p)[1]};
}
template <> __device__ __forceinline__ Rec<24> ld_rec<24>(const uint8_t* p) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
  return {q[0], q[1], q[2]};
}
template <> __device__ __forceinline__ Rec<40> ld_rec<40>(const uint8_t* p) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
  return {q[0], q[1], q[2], q[3], q[4]};
}
template <int R> __device__ __forceinline__ void st_rec(uint8_t* p, const Rec<R>& r);
template <> __device__ __forceinline__ void st_rec<8>(uint8_t* p, const Rec<8>& r) { *reinterpret_cast<uint2*>(p) = r.a; }
template <> __device__ __forceinline__ void st_rec<16>(uint8_t* p, const Rec<16>& r) { *reinterpret_cast<uint4*>(p) = r.a; }
template <> __device__ __forceinline__ void st_rec<32>(uint8_t* p, const Rec<32>& r) {
  reinterpret_cast<uint4*>(p)[0] = r.a;
  reinterpret_cast<uint4*>(p)[1] = r.b;
}
template <> __device__ __forceinline__ void st_rec<24>(uint8_t* p, const Rec<24>& r) {
  uint2* q = reinterpret_cast<uint2*>(p);
  q[0] = r.a; q[1] = r.b; q[2] = r.c;
}
template <> __device__ __forceinline__ void st_rec<40>(uint8_t* p, const Rec<40>& r) {
  uint2* q = reinterpret_cast<uint2*>(p);
  q[0] = r.a; q[1] = r.b; q[2] = r.c; q[3] = r.d; q[4] = r.e;
}
// read-only, non-coherent path for the streaming source of a pass
template <int R> __device__ __forceinline__ Rec<R> ldg_rec(const uint8_t* p);
template <> __device__ __forceinline__ Rec<8> ldg_rec<8>(const uint8_t* p) { return {__ldg(reinterpret_cast<const uint2*>(p))}; }
template <> __device__ __forceinline__ Rec<16> ldg_rec<16>(const uint8_t* p) { return {__ldg(reinterpret_cast<const uint4*>(p))}; }
template <> __device__ __forceinline__ Rec<32> ldg_rec<32>(const uint8_t* p) {
  return {__ldg(reinterpret_cast<const uint4*>(p)), __ldg(reinterpret_cast<const uint4*>(p) + 1)};
}

template <> __device__ __forceinline__ Rec<24> ldg_rec<24>(const uint8_t* p) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
  return {__ldg(q), __ldg(q + 1), __ldg(q + 2)};
}
template <> __device__ __forceinline__ Rec<40> ldg_rec<40>(const uint8_t* p) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
  return {__ldg(q), __ldg(q + 1), __ldg(q + 2), __ldg(q + 3), __ldg(q + 4)};
}

// read-only 256-bit load for R = 32 (LDG.256: one request per 32-byte record);
// L2-only loads (ld.global.cg: no L1 allocation), for data read once
template <int R> __device__ __forceinline__ Rec<R> ldcg_rec(const uint8_t* p);
template <> __device__ __forceinline__ Rec<32> ldcg_rec<32>(const uint8_t* p) {
  Rec<32> r;
  asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.a.x), "=r"(r.a.y), "=r"(r.a.z), "=r"(r.a.w), "=r"(r.b.x), "=r"(r.b.y), "=r"(r.b.z), "=r"(r.b.w)
               : "l"(p)
               : "memory");
  return r;
}
template <> __device__ __forceinline__ Rec<16> ldcg_rec<16>(const uint8_t* p) { return {__ldcg(reinterpret_cast<const uint4*>(p))}; }
template <> __device__ __forceinline__ Rec<8> ldcg_rec<8>(const uint8_t* p) { return {__ldcg(reinterpret_cast<const uint2*>(p))}; }
template <> __device__ __forceinline__ Rec<24> ldcg_rec<24>(const uint8_t* p) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
  return {__ldcg(q), __ldcg(q + 1), __ldcg(q + 2)};
}
template <> __device__ __forceinline__ Rec<40> ldcg_rec<40>(const uint8_t* p) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
  return {__ldcg(q), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3), __ldcg(q + 4)};
}
// other sizes as ldg_rec.  Used where it was measured (ptxas 12.9 crashes on
// it in some kernels).
template <int R> __device__ __forceinline__ Rec<R> ldg_wide(const uint8_t* p) { return ldg_rec<R>(p); }
template <> __device__ __forceinline__ Rec<32> ldg_wide<32>(const uint8_t* p) {
  Rec<32> r;
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.a.x), "=r"(r.a.y), "=r"(r.a.z), "=r"(r.a.w), "=r"(r.b.x), "=r"(r.b.y), "=r"(r.b.z), "=r"(r.b.w)
               : "l"(p));
  return r;
}

// store to GLOBAL memory (p must be a global address): R = 32 is one 256-bit
// store (STG.256), other sizes as st_rec
template <int R> __device__ __forceinline__ void stg_rec(uint8_t* p, const Rec<R>& r) { st_rec<R>(p, r); }
template <> __device__ __forceinline__ void stg_rec<32>(uint8_t* p, const Rec<32>& r) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.a.x), "r"(r.a.y), "r"(r.a.z),
               "r"(r.a.w), "r"(r.b.x), "r"(r.b.y), "r"(r.b.z), "r"(r.b.w)
               : "memory");
}

__device__ __forceinline__ uint64_t u64of(uint32_t lo, uint32_t hi) { return (uint64_t)lo | ((uint64_t)hi << 32); }

// ---------------------------------------------------------------------- keys
// Key = bytes [0,K) as a little-endian unsigned integer (R1).
template <int K> struct Key;
template <> struct Key<8> { uint64_t w0; };
template <> struct Key<16> { uint64_t w0, w1; };  // w1 = high word (bytes 8..15)

template <int R, int K> __device__ __forceinline__ Key<K> key_of(const Rec<R>& r);
template <> __device__ __forceinline__ Key<8> key_of<8, 8>(const Rec<8>& r) { return {u64of(r.a.x, r.a.y)}; }
template <> __device__ __forceinline__ Key<8> key_of<16, 8>(const Rec<16>& r) { return {u64of(r.a.x, r.a.y)}; }
template <> __device__ __forceinline__ Key<8> key_of<32, 8>(const Rec<32>& r) { return {u64of(r.a.x, r.a.y)}; }
template <> __device__ __forceinline__ Key<16> key_of<16, 16>(const Rec<16>& r) { return {u64of(r.a.x, r.a.y), u64of(r.a.z, r.a.w)}; }
template <> __device__ __forceinline__ Key<16> key_of<32, 16>(const Rec<32>& r) { return {u64of(r.a.x, r.a.y), u64of(r.a.z, r.a.w)}; }
template <> __device__ __forceinline__ Key<8> key_of<24, 8>(const Rec<24>& r) { return {u64of(r.a.x, r.a.y)}; }
template <> __device__ __forceinline__ Key<16> key_of<24, 16>(const Rec<24>& r) { return {u64of(r.a.x, r.a.y), u64of(r.b.x, r.b.y)}; }
template <> __device__ __forceinline__ Key<16> key_of<40, 16>(const Rec<40>& r) { return {u64of(r.a.x, r.a.y), u64of(r.b.x, r.b.y)}; }

// The record whose bytes are exactly a key (R == K; used to fill final bins).
template <int R, int K> __device__ __forceinline__ Rec<R> rec_of_key(const Key<K>& k) {
  Rec<R> x{};
  if constexpr (R == 8 && K == 8) x.a = make_uint2((uint32_t)k.w0, (uint32_t)(k.w0 >> 32));
  if constexpr (R == 16 && K == 16)
    x.a = make_uint4((uint32_t)k.w0, (uint32_t)(k.w0 >> 32), (uint32_t)k.w1, (uint32_t)(k.w1 >> 32));
  return x;
}

// Digit d, d = 0 most significant ("1 B digits"): byte K-1-d.
__device__ __forceinline__ uint32_t digit_of(const Key<8>& k, uint32_t d) {
  return (uint32_t)(k.w0 >> (8u * (7u - d))) & 255u;
}
__device__ __forceinline__ uint32_t digit_of(const Key<16>& k, uint32_t d) {
  return d < 8 ? (uint32_t)(k.w1 >> (8u * (7u - d))) & 255u : (uint32_t)(k.w0 >> (8u * (15u - d))) & 255u;
}

// The 32 key bits starting sb < 8K bits below the most significant one (zero
// bits past the end of the key): one funnel shift of the two 32-bit key words
// that hold them (the word pair is selected by sb, uniform across a bin).
__device__ __forceinline__ uint32_t key_window(const Key<8>& k, uint32_t sb) {
  const uint32_t W0 = (uint32_t)(k.w0 >> 32), W1 = (uint32_t)k.w0;
  const bool j0 = sb < 32;
  return __funnelshift_l(j0 ? W1 : 0u, j0 ? W0 : W1, sb & 31u);
}
__device__ __forceinline__ uint32_t key_window(const Key<16>& k, uint32_t sb) {
  const uint32_t W0 = (uint32_t)(k.w1 >> 32), W1 = (uint32_t)k.w1, W2 = (uint32_t)(k.w0 >> 32), W3 = (uint32_t)k.w0;
  const uint32_t j = sb >> 5;
  const uint32_t a = j == 0 ? W0 : (j == 1 ? W1 : (j == 2 ? W2 : W3));
  const uint32_t b = j == 0 ? W1 : (j == 1 ? W2 : (j == 2 ? W3 : 0u));
  return __funnelshift_l(b, a, sb & 31u);
}
// 1 <= W <= 32 key bits starting sb bits below the most significant one
// (8-byte keys: one 64-bit shift pair, measured cheaper than the window).
__device__ __forceinline__ uint32_t key_bits(const Key<8>& k, uint32_t sb, uint32_t W) {
  return (uint32_t)((k.w0 << sb) >> (64u - W));
}
__device__ __forceinline__ uint32_t key_bits(const Key<16>& k, uint32_t sb, uint32_t W) {
  return key_window(k, sb) >> (32u - W);
}
// The radix digit of a pass of DB bits at depth d: DB = 8 is digit d (one key
// byte); DB = 10 is digit d followed by the two leading bits of
// digit d+1 (a "wide" level).
template <int DB, int K>
__device__ __forceinline__ uint32_t digit_w(const Key<K>& k, uint32_t d) {
  if constexpr (DB == 8) return digit_of(k, d);
  else return key_window(k, 8u * d) >> (32 - DB);
}

// First digit >= d whose byte differs between the AND and the OR of all keys
// of a bin (i.e. the first non-constant digit, "bins ... tend to
// shrink (except bins with all keys equal)"); returns K if none.
template <int K>
__device__ __forceinline__ uint32_t first_nonconst_digit(const uint64_t* andw, const uint64_t* orw, uint32_t d) {
  for (; d < (uint32_t)K; ++d) {
    uint32_t bi = (uint32_t)K - 1u - d;
    uint64_t x = (andw[bi >> 3] ^ orw[bi >> 3]) >> (8u * (bi & 7u));
    if (x & 255u) return d;
  }
  return (uint32_t)K;
}

// ---------------------------------------------------------- status words
// Decoupled look-back status (one per tile x digit): [63:48] epoch,
// [47:46] flag (1 = tile aggregate, 2 = inclusive prefix), [45:0] value.
constexpr uint64_t ST_AGG = 1ull << 46;
constexpr uint64_t ST_PREFIX = 2ull << 46;
constexpr uint64_t ST_VAL = (1ull << 46) - 1;

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------ TMA bulk copy / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared (16-byte aligned addresses, size % 16 == 0),
// completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// order this thread's earlier generic-proxy smem accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ----------------------------------------------------------- block helpers
// Exclusive scan of one value per thread for threads [0, 256); every thread
// of the block must call it (it contains barriers).  `ws` = 8 words of smem.
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* ws) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t x = v;
  if (tid < 256) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
  }
  __syncthreads();
  uint32_t add = 0;
  if (tid < 256) {
#pragma unroll
    for (int i = 0; i < 8; ++i) add += (i < w) ? ws[i] : 0u;
  }
  __syncthreads();
  return x - v + add;
}

// Exclusive scan of one value per thread over a block of NT threads (every
// thread calls it; it contains barriers).  `ws` = NT/32 words of smem.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* ws) {
  if constexpr (NT == 256) {
    return block_excl_scan256(v, ws);
  } else {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t t = lane < NW ? ws[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < NW) ws[lane] = t;
    }
    __syncthreads();
    const uint32_t add = w > 0 ? ws[w - 1] : 0u;
    __syncthreads();
    return x - v + add;
  }
}

// ------------------------------------------------------- warp tiny sorter
// Sort key for a tiny bin at depth `depth` >= 1: the `depth` leading digits
// are shared by the whole bin, so they are shifted out and the record's index
// inside the bin (< 128, 7 bits) is packed into the freed low byte.  Ordering
// the packed keys orders the records by key (ties by index), and the sort then
// moves each full record once -- the enumeration-sort idea of "n assignments"
// (§2.2, §3.3).
struct SK8 {
  uint64_t v;
  __device__ __forceinline__ bool lt(const SK8& o) const { return v < o.v; }
  __device__ __forceinline__ uint32_t idx() const { return (uint32_t)v & 255u; }
  __device__ __forceinline__ SK8 shfl(int m) const { return {__shfl_xor_sync(0xffffffffu, v, m)}; }
  static __device__ __forceinline__ SK8 maxv() { return {~0ull}; }
};
struct SK16 {
  uint64_t hi, lo;
  __device__ __forceinline__ bool lt(const SK16& o) const { return hi < o.hi || (hi == o.hi && lo < o.lo); }
  __device__ __forceinline__ uint32_t idx() const { return (uint32_t)lo & 255u; }
  __device__ __forceinline__ SK16 shfl(int m) const {
    return {__shfl_xor_sync(0xffffffffu, hi, m), __shfl_xor_sync(0xffffffffu, lo, m)};
  }
  static __device__ __forceinline__ SK16 maxv() { return {~0ull, ~0ull}; }
};
template <int K> struct SKT;
template <> struct SKT<8> { using T = SK8; };
template <> struct SKT<16> { using T = SK16; };

__device__ __forceinline__ SK8 make_sk(const Key<8>& k, uint32_t depth, uint32_t i) {
  return {(k.w0 << (8u * depth)) | i};
}
__device__ __forceinline__ SK16 make_sk(const Key<16>& k, uint32_t depth, uint32_t i) {
  const uint32_t s = 8u * depth;  // 8..120
  uint64_t hi, lo;
  if (s >= 64) { hi = k.w0 << (s - 64); lo = 0; }
  else { hi = (k.w1 << s) | (k.w0 >> (64 - s)); lo = k.w0 << s; }
  return {hi, lo | i};
}

// Bitonic sorting network over 32*E keys held E per lane (element i = lane*E+e),
// PAPER.md:96-100 §2.2 (sorting networks: fixed comparators, hard-coded indices).
template <class SK, int E>
__device__ __forceinline__ void warp_bitonic(SK (&x)[E], int lane) {
  constexpr int N = 32 * E;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = e ^ j;
          if (p > e) {
            const int i = lane * E + e;
            const bool asc = (i & k) == 0;
            SK a = x[e], b = x[p];
            const bool sw = asc ? b.lt(a) : a.lt(b);
            x[e] = sw ? b : a;
            x[p] = sw ? a : b;
          }
        }
      } else {
        const int lm = j / E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane * E + e;
          SK y = x[e].shfl(lm);
          const bool takemin = (((i & j) == 0) == ((i & k) == 0));
          const bool ylt = y.lt(x[e]);
          x[e] = (takemin == ylt) ? y : x[e];
        }
      }
    }
  }
}

template <int R, int K, int E>
__device__ __forceinline__ void tiny_sort_e(const uint8_t* src, uint8_t* dst, uint32_t n, uint32_t depth, int lane) {
  using SK = typename SKT<K>::T;
  SK x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)(lane * E + e);
    if (i < n) x[e] = make_sk(key_of<R, K>(ld_rec<R>(src + (size_t)i * R)), depth, i);
    else x[e] = SK::maxv();
  }
  warp_bitonic<SK, E>(x, lane);
  Rec<R> r[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)(lane * E + e);
    if (i < n) r[e] = ld_rec<R>(src + (size_t)x[e].idx() * R);
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)(lane * E + e);
    if (i < n) st_rec<R>(dst + (size_t)i * R, r[e]);
  }
}

// Sort a tiny bin of 2 <= n <= TINY_MAX records (one warp).  src and dst may
// alias (every lane gathers before any lane stores) and may point into smem.
template <int R, int K>
__device__ __forceinline__ void warp_tiny_sort(const uint8_t* src, uint8_t* dst, uint32_t n, uint32_t depth, int lane) {
  if (n <= 32) tiny_sort_e<R, K, 1>(src, dst, n, depth, lane);
  else if (n <= 64) tiny_sort_e<R, K, 2>(src, dst, n, depth, lane);
  else tiny_sort_e<R, K, 4>(src, dst, n, depth, lane);
}

template <int R>
__device__ __forceinline__ void warp_copy(const uint8_t* src, uint8_t* dst, uint32_t n, int lane) {
  for (uint32_t i = lane; i < n; i += 32) st_rec<R>(dst + (size_t)i * R, ld_rec<R>(src + (size_t)i * R));
}

__device__ __forceinline__ bool key_lt(const Key<8>& a, const Key<8>& b) { return a.w0 < b.w0; }
__device__ __forceinline__ bool key_lt(const Key<16>& a, const Key<16>& b) {
  return (a.w1 < b.w1) | ((a.w1 == b.w1) & (a.w0 < b.w0));
}

// Lane-serial insertion sort of c (<= 8) records in place (§2.2,
// PAPER.md:177 §3.3 insertion sort as the fix-up stage).
template <int R, int K>
__device__ __forceinline__ void lane_insertion_sort(uint8_t* base, uint32_t c) {
  for (uint32_t i = 1; i < c; ++i) {
    const Rec<R> x = ld_rec<R>(base + (size_t)i * R);
    const Key<K> kx = key_of<R, K>(x);
    int j = (int)i - 1;
    for (; j >= 0; --j) {
      const Rec<R> y = ld_rec<R>(base + (size_t)j * R);
      if (!key_lt(kx, key_of<R, K>(y))) break;
      st_rec<R>(base + (size_t)(j + 1) * R, y);
    }
    st_rec<R>(base + (size_t)(j + 1) * R, x);
  }
}

template <int R, int K> __device__ __forceinline__ Key<K> ld_key(const uint8_t* p);
template <> __device__ __forceinline__ Key<8> ld_key<8, 8>(const uint8_t* p) { return {*reinterpret_cast<const uint64_t*>(p)}; }
template <> __device__ __forceinline__ Key<8> ld_key<16, 8>(const uint8_t* p) { return {*reinterpret_cast<const uint64_t*>(p)}; }
template <> __device__ __forceinline__ Key<8> ld_key<32, 8>(const uint8_t* p) { return {*reinterpret_cast<const uint64_t*>(p)}; }
template <> __device__ __forceinline__ Key<16> ld_key<16, 16>(const uint8_t* p) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  return {u64of(v.x, v.y), u64of(v.z, v.w)};
}
template <> __device__ __forceinline__ Key<16> ld_key<32, 16>(const uint8_t* p) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  return {u64of(v.x, v.y), u64of(v.z, v.w)};
}
template <> __device__ __forceinline__ Key<8> ld_key<24, 8>(const uint8_t* p) { return {*reinterpret_cast<const uint64_t*>(p)}; }
template <> __device__ __forceinline__ Key<16> ld_key<24, 16>(const uint8_t* p) {
  const uint64_t* q = reinterpret_cast<const uint64_t*>(p);
  return {q[0], q[1]};
}
template <> __device__ __forceinline__ Key<16> ld_key<40, 16>(const uint8_t* p) {
  const uint64_t* q = reinterpret_cast<const uint64_t*>(p);
  return {q[0], q[1]};
}
__device__ __forceinline__ bool key_eq(const Key<8>& a, const Key<8>& b) { return a.w0 == b.w0; }
__device__ __forceinline__ bool key_eq(const Key<16>& a, const Key<16>& b) { return (a.w0 == b.w0) & (a.w1 == b.w1); }

// Enumeration-sort rank of record i inside bin [base, base+c) (PAPER.md:102-104
// §2.2 "the final position of each element is determined by comparing it
// against each other ... the number of element moves is only O(n)"; ties by
// index): #{j: key_j < key_i} + #{j < i: key_j == key_i}.
template <int R, int K>
__device__ __forceinline__ uint32_t es_rank(const uint8_t* base, uint32_t c, uint32_t i, const Key<K>& ki) {
  // branch-free accumulation (the paper's SETcc idea), 4 keys in flight
  uint32_t rank = 0, j = 0;
  for (; j + 4 <= c; j += 4) {
    Key<K> kj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) kj[u] = ld_key<R, K>(base + (size_t)(j + u) * R);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      rank += (uint32_t)key_lt(kj[u], ki) | ((uint32_t)(j + u < i) & (uint32_t)key_eq(kj[u], ki));
  }
  for (; j < c; ++j) {
    const Key<K> kj = ld_key<R, K>(base + (size_t)j * R);
    rank += (uint32_t)key_lt(kj, ki) | ((uint32_t)(j < i) & (uint32_t)key_eq(kj, ki));
  }
  return rank;
}

// Enumeration-sort ceiling: bins of 2..ES_MAX records are finished record-
// parallel by es_rank (§3.3: ES for the tiniest bins, and
// for wider records up to 24); larger tiny bins use warp_tail_sort.
template <int R> __host__ __device__ constexpr uint32_t es_max() { return R >= 32 ? 24u : 16u; }

// Per-warp scratch of the tail sorter (shared memory).
template <int K>
struct TailScratch {
  uint32_t cnt[RADIX];      // digit counters, then packed (start << 16 | count)
  Key<K> key[TINY_MAX];     // keys in partitioned order
  uint32_t ltm[TINY_MAX / 32], eqm[TINY_MAX / 32];  // per slot: key < / == its sub-bin's pivot
};

// number of set bits of the TINY_MAX-bit mask m in [a, b)
__device__ __forceinline__ uint32_t popc_range(const uint32_t* m, uint32_t a, uint32_t b) {
  uint32_t s = 0;
#pragma unroll
  for (uint32_t w = 0; w < TINY_MAX / 32; ++w) {
    const uint32_t x0 = max(a, w * 32u), x1 = min(b, w * 32u + 32u);
    if (x0 < x1) {
      const uint32_t len = x1 - x0;
      const uint32_t mk = (len == 32u ? 0xffffffffu : ((1u << len) - 1u)) << (x0 - w * 32u);
      s += __popc(m[w] & mk);
    }
  }
  return s;
}

// Tail sorter for a bin of 2 <= n <= TINY_MAX records, one warp (PAPER.md
// §3.3, GPU form).  One counting pass on digit `depth` with warp-private smem
// counters (sub-bins holding a single record are final and
// never visited again); every record of a sub-bin with c >= 2 records gets its
// place by enumeration sort among those c records only (PAPER.md:102-104 ES:
// n comparisons, one move per record; ties by partition slot).  Works on keys;
// each full record is then moved once, src -> out.  src and out must not alias.
template <int R, int K, int E, bool PV>
__device__ __forceinline__ void warp_tail_sort_e(const uint8_t* src, uint8_t* out, uint32_t n, uint32_t depth, int lane,
                                                 TailScratch<K>& ws) {
  uint4* w4 = reinterpret_cast<uint4*>(ws.cnt);
  w4[lane * 2] = make_uint4(0, 0, 0, 0);
  w4[lane * 2 + 1] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  Key<K> k[E];
  uint32_t pr[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)(e * 32 + lane);
    if (i < n) {
      k[e] = ld_key<R, K>(src + (size_t)i * R);
      pr[e] = atomicAdd(&ws.cnt[digit_of(k[e], depth)], 1u);
    }
  }
  __syncwarp();
  {
    const uint4 c0 = w4[lane * 2], c1 = w4[lane * 2 + 1];
    const uint32_t tot = c0.x + c0.y + c0.z + c0.w + c1.x + c1.y + c1.z + c1.w;
    uint32_t inc = tot;
#pragma unroll
    for (int sft = 1; sft < 32; sft <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, sft);
      if (lane >= sft) inc += y;
    }
    const uint32_t r0 = inc - tot;
    const uint32_t r1 = r0 + c0.x, r2 = r1 + c0.y, r3 = r2 + c0.z, r4 = r3 + c0.w;
    const uint32_t r5 = r4 + c1.x, r6 = r5 + c1.y, r7 = r6 + c1.z;
    __syncwarp();
    w4[lane * 2] = make_uint4((r0 << 16) | c0.x, (r1 << 16) | c0.y, (r2 << 16) | c0.z, (r3 << 16) | c0.w);
    w4[lane * 2 + 1] = make_uint4((r4 << 16) | c1.x, (r5 << 16) | c1.y, (r6 << 16) | c1.z, (r7 << 16) | c1.w);
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)(e * 32 + lane);
    if (i < n) {
      const uint32_t w = ws.cnt[digit_of(k[e], depth)];
      const uint32_t slot = (w >> 16) + pr[e];
      ws.key[slot] = k[e];
      pr[e] = slot | ((w >> 16) << 8) | ((w & 0xffu) << 16);  // slot | start << 8 | count << 16
    }
  }
  __syncwarp();
  // sub-bins whose records all carry the same key need no ordering (PAPER.md:38
  // "bins with all keys equal"): flag (bit 15 of the packed counter) the ones
  // holding a key different from their first record's
  bool big = false;
#pragma unroll
  for (int e = 0; e < E; ++e) big |= ((uint32_t)(e * 32 + lane) < n) && (pr[e] >> 16) > 4u;
  const bool checked = __any_sync(0xffffffffu, big);
  if (checked) {  // only sub-bins of > 4 records are worth the check
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = (uint32_t)(e * 32 + lane);
      if (i < n && (pr[e] >> 16) > 1u && !key_eq(ws.key[(pr[e] >> 8) & 0xffu], k[e]))
        atomicOr(&ws.cnt[digit_of(k[e], depth)], 0x8000u);
    }
    __syncwarp();
  }
  // mixed sub-bins of > HV records (typically many copies of one key and a
  // few others): three-way classification against a pivot key (the sub-bin's
  // middle slot), so that ES runs only among the records below / above it and
  // the pivot's copies are placed by slot order -- O(c * m) instead of O(c^2)
  // for m records different from the pivot
  constexpr uint32_t HV = PV ? 8u : 0xffffu;  // PV = false: no pivot path (callers short of registers)
  auto is_mixed = [&](int e) {
    return (uint32_t)(e * 32 + lane) < n && (pr[e] >> 16) > 1u &&
           (!checked || (ws.cnt[digit_of(k[e], depth)] & 0x8000u) != 0u);
  };
  bool heavy = false;
#pragma unroll
  for (int e = 0; e < E; ++e) heavy |= (uint32_t)(e * 32 + lane) < n && (pr[e] >> 16) > HV;
  heavy = PV && __any_sync(0xffffffffu, heavy);
  if (heavy) {
    if (lane < (int)(TINY_MAX / 32)) { ws.ltm[lane] = 0; ws.eqm[lane] = 0; }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t slot = pr[e] & 0xffu, s0 = (pr[e] >> 8) & 0xffu, c = pr[e] >> 16;
      if (c > HV && is_mixed(e)) {
        const Key<K> pv = ws.key[s0 + c / 2];
        if (key_lt(k[e], pv)) atomicOr(&ws.ltm[slot >> 5], 1u << (slot & 31u));
        else if (key_eq(k[e], pv)) atomicOr(&ws.eqm[slot >> 5], 1u << (slot & 31u));
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)(e * 32 + lane);
    if (i < n) {
      const uint32_t slot = pr[e] & 0xffu, s0 = (pr[e] >> 8) & 0xffu, c = pr[e] >> 16;
      uint32_t fin = slot;
      const bool mixed = !checked || (ws.cnt[digit_of(k[e], depth)] & 0x8000u) != 0u;
      if (heavy && c > HV && mixed) {
        const uint32_t bit = 1u << (slot & 31u);
        const uint32_t nlt = popc_range(ws.ltm, s0, s0 + c);
        if (ws.eqm[slot >> 5] & bit) {
          fin = s0 + nlt + popc_range(ws.eqm, s0, slot);
        } else {  // ES among the records on the same side of the pivot
          const bool lt = (ws.ltm[slot >> 5] & bit) != 0u;
          uint32_t r = lt ? 0u : nlt + popc_range(ws.eqm, s0, s0 + c);
          for (uint32_t w = s0 >> 5; w <= (s0 + c - 1u) >> 5; ++w) {
            uint32_t m = lt ? ws.ltm[w] : ~(ws.ltm[w] | ws.eqm[w]);
            const uint32_t lo = max(s0, w * 32u) - w * 32u, hi = min(s0 + c, w * 32u + 32u) - w * 32u;
            m &= (hi - lo == 32u ? 0xffffffffu : ((1u << (hi - lo)) - 1u) << lo);
            while (m) {
              const uint32_t q = w * 32u + (uint32_t)(__ffs(m) - 1);
              m &= m - 1u;
              const Key<K> kq = ws.key[q];
              r += (uint32_t)key_lt(kq, k[e]) | ((uint32_t)(q < slot) & (uint32_t)key_eq(kq, k[e]));
            }
          }
          fin = s0 + r;
        }
      } else if (c > 1 && mixed) {  // ES among the sub-bin's c records (pairs / triples: predicated, no divergent loop)
        uint32_t r = 0;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          const Key<K> kq = ws.key[min(s0 + q, (uint32_t)TINY_MAX - 1u)];
          r += (uint32_t)(q < c) & ((uint32_t)key_lt(kq, k[e]) | ((uint32_t)(s0 + q < slot) & (uint32_t)key_eq(kq, k[e])));
        }
        for (uint32_t q = s0 + 4; q < s0 + c; ++q) {
          const Key<K> kq = ws.key[q];
          r += (uint32_t)key_lt(kq, k[e]) | ((uint32_t)(q < slot) & (uint32_t)key_eq(kq, k[e]));
        }
        fin = s0 + r;
      }
      st_rec<R>(out + (size_t)fin * R, ld_rec<R>(src + (size_t)i * R));
    }
  }
  __syncwarp();
}

// Dominant-key fast path of the tail sorter (duplicate-heavy bins such as the
// k-mer stream's: ~100 copies of one key plus a few variants).  Pivot = the
// middle record's key; one ballot pass counts the records below / above it.
// If at most 32 records differ from it, the pivot's copies go straight to
// their final slots (order inside an equal-key run is free, R2), the
// others are parked in the scratch and placed by enumeration sort among their
// own side.  Returns false (nothing written) when the bin is not of that kind.
template <int R, int K>
__device__ __forceinline__ bool warp_tail_dominant(const uint8_t* src, uint8_t* out, uint32_t n, int lane,
                                                   TailScratch<K>& ws) {
  static_assert(32 * R <= sizeof(TailScratch<K>), "scratch holds 32 records");
  const Key<K> pv = ld_key<R, K>(src + (size_t)(n / 2) * R);
  uint32_t nlt = 0, ngt = 0;
  for (uint32_t j0 = 0; j0 < n; j0 += 32) {
    const uint32_t j = j0 + (uint32_t)lane;
    bool lt = false, gt = false;
    if (j < n) {
      const Key<K> k = ld_key<R, K>(src + (size_t)j * R);
      lt = key_lt(k, pv);
      gt = key_lt(pv, k);
    }
    nlt += (uint32_t)__popc(__ballot_sync(0xffffffffu, lt));
    ngt += (uint32_t)__popc(__ballot_sync(0xffffffffu, gt));
  }
  const uint32_t m = nlt + ngt, neq = n - m;
  if (m > 32 || neq < m) return false;
  uint8_t* scr = reinterpret_cast<uint8_t*>(&ws);
  const uint32_t below = (1u << lane) - 1u;
  uint32_t plt = 0, pgt = 0, peq = 0;  // records of each class placed so far
  for (uint32_t j0 = 0; j0 < n; j0 += 32) {
    const uint32_t j = j0 + (uint32_t)lane;
    Rec<R> x;
    int cls = 3;
    if (j < n) {
      x = ld_rec<R>(src + (size_t)j * R);
      const Key<K> k = key_of<R, K>(x);
      cls = key_lt(k, pv) ? 0 : (key_lt(pv, k) ? 2 : 1);
    }
    const uint32_t b0 = __ballot_sync(0xffffffffu, cls == 0), b1 = __ballot_sync(0xffffffffu, cls == 1),
                   b2 = __ballot_sync(0xffffffffu, cls == 2);
    if (cls == 0) st_rec<R>(scr + (size_t)(plt + __popc(b0 & below)) * R, x);
    else if (cls == 2) st_rec<R>(scr + (size_t)(nlt + pgt + __popc(b2 & below)) * R, x);
    else if (cls == 1) st_rec<R>(out + (size_t)(nlt + peq + __popc(b1 & below)) * R, x);
    plt += __popc(b0);
    pgt += __popc(b2);
    peq += __popc(b1);
  }
  __syncwarp();
  if ((uint32_t)lane < m) {  // ES among the records on the lane's side of the pivot
    const bool lo = (uint32_t)lane < nlt;
    const uint32_t g0 = lo ? 0u : nlt, gn = lo ? nlt : ngt, i = (uint32_t)lane - g0;
    const Rec<R> x = ld_rec<R>(scr + (size_t)lane * R);
    const uint32_t rk = es_rank<R, K>(scr + (size_t)g0 * R, gn, i, key_of<R, K>(x));
    st_rec<R>(out + (size_t)((lo ? 0u : nlt + neq) + rk) * R, x);
  }
  __syncwarp();
  return true;
}

template <int R, int K, bool PV = true>
__device__ __forceinline__ void warp_tail_sort(const uint8_t* src, uint8_t* out, uint32_t n, uint32_t depth, int lane,
                                               TailScratch<K>& ws) {
  if (PV && n > 32 && warp_tail_dominant<R, K>(src, out, n, lane, ws)) return;
  if (n <= 32) warp_tail_sort_e<R, K, 1, PV>(src, out, n, depth, lane, ws);
  else if (n <= 64) warp_tail_sort_e<R, K, 2, PV>(src, out, n, depth, lane, ws);
  else warp_tail_sort_e<R, K, 4, PV>(src, out, n, depth, lane, ws);
}

}  // namespace radsort
