// k_local2: the two-phase local sort of a bin too large for one CTA's shared
// memory to sort in one step (GPU analog of PAPER.md:130-135 §3.2: "if the bin
// is small enough to fit in a half of L2 ... simple counting and scatter").
//
// One CTA per bin (many bins in flight per SM), the bin's own range of the
// other buffer as scratch (it is dead at this point of the recursion):
//   P1  read the bin's keys: AND/OR (first bit that differs over the bin,
//       PAPER.md:38 constant digits) and the histogram of the G = 2^gb groups
//       given by the gb key bits from there;
//   P2  group starts (exclusive prefix);
//   P3  partition the bin into its groups in the scratch range: TR-record
//       tiles ranked by warp-private counters, staged in shared memory grouped
//       by group, written out as coalesced runs (the paper's buffered scatter,
//       PAPER.md:63-67);
//   P4  each group (<= GCAP records, just written: read back from L2) is
//       sorted in shared memory by one counting pass on the next W4 key bits
//       (W4 = ceil(log2 m) + 1, about half a record per bucket; R3)
//       plus the in-place fix-up of colliding buckets, and
//       written to its final place in `records` with coalesced stores.
// Both reads of the bin and the scratch round trip stay in L2 (the bin is a
// few hundred KB); HBM sees one read and one write of every record.
// Rare cases leave the kernel as bins of the next level: a group larger than
// GCAP (skewed keys) -> Large list; a group in one W4-bucket, or a colliding
// bucket of > ES records holding several keys -> Local list.
#pragma once
#include "passes.cuh"

namespace radsort {

// key bits [s, s + w) counted from the most significant bit (1 <= w <= 32;
// bits past the end of the key read as zero)
__device__ __forceinline__ uint32_t bits_at(const Key<8>& k, uint32_t s, uint32_t w) {
  const uint64_t x = s < 64u ? k.w0 << s : 0ull;
  return (uint32_t)(x >> (64u - w));
}
__device__ __forceinline__ uint32_t bits_at(const Key<16>& k, uint32_t s, uint32_t w) {
  uint64_t x;
  if (s == 0u) x = k.w1;
  else if (s < 64u) x = (k.w1 << s) | (k.w0 >> (64u - s));
  else if (s < 128u) x = k.w0 << (s - 64u);
  else x = 0ull;
  return (uint32_t)(x >> (64u - w));
}

// First key bit (from the most significant) in which the AND and the OR of a
// bin's keys differ; 8K when every key is equal.
template <int K>
__device__ __forceinline__ uint32_t first_diff_bit(const uint64_t* A, const uint64_t* O) {
  if constexpr (K == 8) {
    const uint64_t x = A[0] ^ O[0];
    return x ? (uint32_t)__clzll((long long)x) : 64u;
  } else {
    const uint64_t x1 = A[1] ^ O[1], x0 = A[0] ^ O[0];
    if (x1) return (uint32_t)__clzll((long long)x1);
    return x0 ? 64u + (uint32_t)__clzll((long long)x0) : 128u;
  }
}

// read-only key of a record in global memory
template <int R, int K>
__device__ __forceinline__ Key<K> ldg_key(const uint8_t* p) {
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p);
  Key<K> k;
  k.w0 = __ldg(q);
  if constexpr (K == 16) k.w1 = __ldg(q + 1);
  return k;
}

template <int R> struct L2Cfg;
// LB threads, groups of <= GCAP records, P3 tiles of TR records, MINB CTAs per SM
template <> struct L2Cfg<8> { static constexpr int LB = 256, GCAP = 2048, TR = 2048, MINB = 4; };
template <> struct L2Cfg<16> { static constexpr int LB = 256, GCAP = 2048, TR = 1024, MINB = 4; };
template <> struct L2Cfg<32> { static constexpr int LB = 512, GCAP = 2048, TR = 1024, MINB = 2; };
constexpr uint32_t L2_GBMAX = 6;  // at most 64 groups
constexpr uint32_t L2_GMAX = 1u << L2_GBMAX;

template <int R> __host__ __device__ constexpr uint32_t local2_max() { return 32u * (uint32_t)L2Cfg<R>::GCAP; }
template <int R> __host__ __device__ constexpr size_t local2_stage_bytes() {
  return (size_t)(L2Cfg<R>::GCAP > L2Cfg<R>::TR ? L2Cfg<R>::GCAP : L2Cfg<R>::TR) * R;
}
template <int R> __host__ __device__ constexpr uint32_t local2_wmax() {  // W4 for a full group
  return 32u - (uint32_t)__builtin_clz((unsigned)L2Cfg<R>::GCAP - 1u) + 1u;
}
template <int R> __host__ __device__ constexpr size_t local2_smem() {
  return local2_stage_bytes<R>() + ((size_t)2 << local2_wmax<R>()) + ((size_t)(L2Cfg<R>::GCAP / 2 + 1) * 4 + 15) / 16 * 16;
}

template <int R, int K>
__global__ void __launch_bounds__(L2Cfg<R>::LB, L2Cfg<R>::MINB)
    k_local2(const Seg* __restrict__ list, uint32_t nlist, uint32_t lmin, uint32_t lmax, Seg* local_next, int nxt,
             Seg* large_next, Ctl* ctl, uint8_t* recs, uint8_t* tmp, int discard) {
  constexpr int LB = L2Cfg<R>::LB, GCAP = L2Cfg<R>::GCAP, TR = L2Cfg<R>::TR;
  constexpr int NW = LB / 32, IT = TR / LB, IG = GCAP / LB, KW = K / 8;
  constexpr uint32_t WMAX4 = local2_wmax<R>();
  constexpr uint32_t STAGE = (uint32_t)local2_stage_bytes<R>();
  constexpr uint32_t CNTB = 2u << WMAX4;
  constexpr uint32_t CAP = GCAP / 2 + 1;
  static_assert(TR % LB == 0 && GCAP % LB == 0, "tile shapes");
  extern __shared__ uint4 smem_raw[];
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem_raw);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(stage + STAGE);
  uint32_t* blist = reinterpret_cast<uint32_t*>(stage + STAGE + CNTB);
  const uint16_t* start16 = reinterpret_cast<const uint16_t*>(cnt);
  __shared__ uint32_t wcnt[NW][L2_GMAX];  // warp-private group counters (P1, P3)
  __shared__ uint32_t tst[NW][L2_GMAX];   // P3: start of warp w's records of group g in the staged tile
  __shared__ uint32_t gcnt[L2_GMAX], gst[L2_GMAX + 1], gcur[L2_GMAX], tgs[L2_GMAX];
  __shared__ uint32_t wsum[NW], s_ncol, s_nbig, s_cst;
  __shared__ unsigned long long sna[2], so[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto zero_cnt = [&](uint32_t bytes) {
    uint4* c4 = reinterpret_cast<uint4*>(cnt);
    for (uint32_t i = tid; i < bytes / 16u; i += LB) c4[i] = make_uint4(0, 0, 0, 0);
  };
  auto zero_w = [&]() {
    for (uint32_t i = tid; i < (uint32_t)NW * L2_GMAX; i += LB) (&wcnt[0][0])[i] = 0;
  };
  auto skip = [&](uint32_t b) {
    const uint32_t l = list[b].len;
    return l > lmax || l < lmin;
  };
  uint32_t bi = blockIdx.x;
  while (bi < nlist && skip(bi)) bi += gridDim.x;
  if (bi >= nlist) return;
  zero_cnt(CNTB);
  zero_w();
  if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  if (tid == 0) { s_ncol = 0; s_nbig = 0; s_cst = 0; }
  __syncthreads();
  unsigned long long done = 0;
  // P1 body: AND/OR (optional) and the warp-private group histogram at bit s
  auto count_groups = [&](const uint8_t* sp, uint32_t n, uint32_t s, uint32_t gb, bool andor) {
    uint64_t na[2] = {0, 0}, o[2] = {0, 0};
    constexpr int U = 4;
    for (uint32_t i0 = tid; i0 < n; i0 += LB * U) {
      Key<K> k[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + (uint32_t)u * LB;
        if (i < n) k[u] = ldg_key<R, K>(sp + (size_t)i * R);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + (uint32_t)u * LB;
        if (i < n) {
          if (andor) {
            na[0] |= ~k[u].w0; o[0] |= k[u].w0;
            if constexpr (KW == 2) { na[1] |= ~k[u].w1; o[1] |= k[u].w1; }
          }
          atomicAdd(&wcnt[warp][bits_at(k[u], s, gb)], 1u);
        }
      }
    }
    if (andor) {
#pragma unroll
      for (int w = 0; w < KW; ++w) {
        const uint32_t x0 = __reduce_or_sync(0xffffffffu, (uint32_t)na[w]);
        const uint32_t x1 = __reduce_or_sync(0xffffffffu, (uint32_t)(na[w] >> 32));
        const uint32_t y0 = __reduce_or_sync(0xffffffffu, (uint32_t)o[w]);
        const uint32_t y1 = __reduce_or_sync(0xffffffffu, (uint32_t)(o[w] >> 32));
        if (lane == 0) { atomicOr(&sna[w], u64of(x0, x1)); atomicOr(&so[w], u64of(y0, y1)); }
      }
    }
  };
  for (;;) {
    const Seg sg = list[bi];
    const uint32_t n = sg.len, off = sg.off;
    const uint8_t* sp = buf_of(sg.src, recs, tmp) + (size_t)off * R;
    const uint8_t xid = sg.src == SRC_TMP ? SRC_REC : SRC_TMP;  // scratch: the bin's range of the other buffer
    uint8_t* xp = buf_of(xid, recs, tmp) + (size_t)off * R;
    uint8_t* dp = recs + (size_t)off * R;
    const bool x_is_d = xid == SRC_REC;
    // groups of about GCAP / 2 records
    uint32_t gb = 1;
    while (gb < L2_GBMAX && (n >> gb) > (uint32_t)GCAP / 2u) ++gb;
    const uint32_t G = 1u << gb;
    uint32_t nb = bi + gridDim.x;
    while (nb < nlist && skip(nb)) nb += gridDim.x;
    // ---- P1
    uint32_t s0 = 8u * sg.depth;
    count_groups(sp, n, s0, gb, true);
    __syncthreads();
    uint32_t s1;
    {
      const uint64_t A[2] = {~(uint64_t)sna[0], ~(uint64_t)sna[1]}, O[2] = {so[0], so[1]};
      s1 = first_diff_bit<K>(A, O);
    }
    if (s1 >= 8u * K) {  // every key equal: final; moved to `records` if it sits in tmp
      if (sg.src == SRC_TMP)
        for (uint32_t q = tid; q < n; q += LB) st_rec<R>(dp + (size_t)q * R, ldg_rec<R>(sp + (size_t)q * R));
      done += n;
      __syncthreads();
      zero_w();
      if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
      __syncthreads();
      if (nb >= nlist) break;
      bi = nb;
      continue;
    }
    if (s1 != s0) {  // leading key bits constant over the bin: group by the first bits that differ
      __syncthreads();
      zero_w();
      __syncthreads();
      s0 = s1;
      count_groups(sp, n, s0, gb, false);
      __syncthreads();
    }
    // ---- P2: group totals and starts (one warp; lane l holds groups l and l + 32)
    if (warp == 0) {
      uint32_t c0 = 0, c1 = 0;
      for (int w = 0; w < NW; ++w) {
        c0 += (uint32_t)lane < G ? wcnt[w][lane] : 0u;
        c1 += (uint32_t)lane + 32u < G ? wcnt[w][lane + 32] : 0u;
      }
      uint32_t e0 = c0, e1 = c1;  // inclusive scans over the lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y0 = __shfl_up_sync(0xffffffffu, e0, o), y1 = __shfl_up_sync(0xffffffffu, e1, o);
        if (lane >= o) { e0 += y0; e1 += y1; }
      }
      const uint32_t tot0 = __shfl_sync(0xffffffffu, e0, 31);
      if ((uint32_t)lane < G) { gcnt[lane] = c0; gst[lane] = e0 - c0; gcur[lane] = 0; }
      if ((uint32_t)lane + 32u < G) { gcnt[lane + 32] = c1; gst[lane + 32] = tot0 + e1 - c1; gcur[lane + 32] = 0; }
      if (lane == 0) gst[G] = n;
    }
    __syncthreads();
    zero_w();
    if (tid == 0 && nb < nlist) {  // the next bin streams into L2 while this one is partitioned and sorted
      const Seg g = list[nb];
      const uintptr_t a0 = (uintptr_t)(buf_of(g.src, recs, tmp) + (size_t)g.off * R);
      const uintptr_t a1 = (a0 + 15) & ~(uintptr_t)15, e1 = (a0 + (size_t)g.len * R) & ~(uintptr_t)15;
      if (e1 > a1) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a1), "r"((uint32_t)(e1 - a1)) : "memory");
    }
    __syncthreads();
    // ---- P3: partition into the scratch range, tile by tile
    for (uint32_t t0 = 0; t0 < n; t0 += TR) {
      const uint32_t m = min((uint32_t)TR, n - t0);
      Rec<R> r[IT];
      uint32_t rk[IT];
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const uint32_t idx = (uint32_t)j * LB + tid;
        if (idx < m) r[j] = ldg_wide<R>(sp + (size_t)(t0 + idx) * R);
      }
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const uint32_t idx = (uint32_t)j * LB + tid;
        if (idx < m) rk[j] = atomicAdd(&wcnt[warp][bits_at(key_of<R, K>(r[j]), s0, gb)], 1u);
      }
      __syncthreads();
      // tile starts in (group, warp) order: tst[w][g] = sum over (g' < g, all w') + (g, w' < w)
      if (warp == 0) {
        uint32_t run = 0;
        for (uint32_t g0 = 0; g0 < G; g0 += 32u) {
          // lane l handles group g0 + l (if present): total over warps, exclusive scan over groups
          const uint32_t g = g0 + (uint32_t)lane;
          uint32_t tot = 0;
          if (g < G)
            for (int w = 0; w < NW; ++w) tot += wcnt[w][g];
          uint32_t inc = tot;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
          }
          if (g < G) {
            uint32_t st = run + inc - tot;
            tgs[g] = st;
            for (int w = 0; w < NW; ++w) {
              tst[w][g] = st;
              st += wcnt[w][g];
            }
          }
          run += __shfl_sync(0xffffffffu, inc, 31);
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const uint32_t idx = (uint32_t)j * LB + tid;
        if (idx < m) st_rec<R>(stage + (size_t)(tst[warp][bits_at(key_of<R, K>(r[j]), s0, gb)] + rk[j]) * R, r[j]);
      }
      __syncthreads();
      for (uint32_t q = tid; q < m; q += LB) {
        const Rec<R> x = ld_rec<R>(stage + (size_t)q * R);
        const uint32_t g = bits_at(key_of<R, K>(x), s0, gb);
        stg_rec<R>(xp + (size_t)(gst[g] + gcur[g] + (q - tgs[g])) * R, x);
      }
      __syncthreads();
      for (uint32_t g = tid; g < G; g += LB) {
        uint32_t c = 0;
        for (int w = 0; w < NW; ++w) c += wcnt[w][g];
        gcur[g] += c;
      }
      __syncthreads();
      zero_w();
      __syncthreads();
    }
    // the scratch range is complete and visible to the whole CTA (barrier above)
    // ---- P4: sort each group into its final place
    const uint32_t sb = s0 + gb;  // first key bit below the group bits
    for (uint32_t g = 0; g < G; ++g) {
      const uint32_t m = gcnt[g], goff = gst[g];
      if (m == 0) continue;
      const uint8_t* gx = xp + (size_t)goff * R;
      uint8_t* gd = dp + (size_t)goff * R;
      if (m == 1) {
        if (!x_is_d && tid == 0) stg_rec<R>(gd, ldcg_rec<R>(gx));
        continue;
      }
      if (m > (uint32_t)GCAP) {  // skewed keys: the group becomes a Large bin of the next level
        if (tid == 0) {
          Seg ns = {off + goff, m, (uint8_t)(sb / 8u), xid, MODE_NONE, 0, 0};
          large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
        }
        continue;
      }
      const uint32_t W4 = local_width(m, WMAX4);
      const int lim = (int)m - tid;
      Rec<R> r[IG];
#pragma unroll
      for (int j = 0; j < IG; ++j)
        if (j * LB < lim) r[j] = ldcg_rec<R>(gx + (size_t)(j * LB + tid) * R);
      uint32_t rk[(IG + 1) / 2];
#pragma unroll
      for (int j = 0; j < (IG + 1) / 2; ++j) rk[j] = 0;
      uint32_t ones = 0;
      bool cst = false;
#pragma unroll
      for (int j = 0; j < IG; ++j) {
        if (j * LB < lim) {
          const uint32_t b = bits_at(key_of<R, K>(r[j]), sb, W4);
          const uint32_t sh = 16u * (b & 1u);
          const uint32_t old = (atomicAdd(&cnt[b >> 1], 1u << sh) >> sh) & 0xffffu;
          rk[j >> 1] |= old << (16 * (j & 1));
          ones += (uint32_t)(old == 1u);
          cst |= old == m - 1u;
        }
      }
      if (cst) s_cst = 1u;
      __syncthreads();
      if (s_cst) {  // the whole group in one bucket: a Local bin of the next level (k_local skips constant bits)
        if (tid == 0) {
          Seg ns = {off + goff, m, (uint8_t)(sb / 8u), xid, MODE_NONE, 0, 0};
          local_next[atomicAdd(&ctl->n_local[nxt], 1u)] = ns;
          atomicMax(&ctl->max_local_len[nxt], m);
          if (m <= small_cap<R>()) atomicAdd(&ctl->n_local_small[nxt], 1u);
          else if (m <= med_cap<R>()) atomicAdd(&ctl->n_local_med[nxt], 1u);
        }
        __syncthreads();
        zero_cnt(2u << W4);
        if (tid == 0) s_cst = 0;
        __syncthreads();
        continue;
      }
      local_scan<LB>(cnt, W4, wsum);
      __syncthreads();
      {
        uint32_t inc = ones;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        uint32_t slot = 0;
        if (lane == 31 && inc) slot = atomicAdd(&s_ncol, inc);
        slot = __shfl_sync(0xffffffffu, slot, 31) + inc - ones;
#pragma unroll
        for (int j = 0; j < IG; ++j) {
          if (j * LB < lim) {
            const uint32_t b = bits_at(key_of<R, K>(r[j]), sb, W4);
            const uint32_t rnk = (rk[j >> 1] >> (16 * (j & 1))) & 0xffffu;
            st_rec<R>(stage + (size_t)((uint32_t)start16[b] + rnk) * R, r[j]);
            if (rnk == 1u) blist[slot++] = b;
          }
        }
      }
      if (discard && !x_is_d) {  // the scratch lines of this group are dead: drop them from L2 unwritten
        const uintptr_t a0 = ((uintptr_t)gx + 127) & ~(uintptr_t)127, a1 = ((uintptr_t)gx + (size_t)m * R) & ~(uintptr_t)127;
        for (uintptr_t a = a0 + (uintptr_t)tid * 128; a < a1; a += (uintptr_t)LB * 128)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
      }
      __syncthreads();
      const bool fix = sb + W4 < 8u * K;  // key bits left below the buckets
      local_finish<R, K, LB, NW, false, true>(stage, start16, blist, CAP, m, 1u << W4, 0u, W4, fix ? s_ncol : 0u,
                                              &s_nbig, nullptr, gd, off + goff, local_next, nxt, ctl, false, nullptr,
                                              (int)((sb + W4) / 8u), SRC_REC);
      __syncthreads();
      zero_cnt(2u << W4);
      if (tid == 0) { s_ncol = 0; s_nbig = 0; }
      __syncthreads();
    }
    done += n;
    if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
    __syncthreads();
    if (nb >= nlist) break;
    bi = nb;
  }
  if (tid == 0) atomicAdd(&ctl->rec_local, done);
}

}  // namespace radsort
