// k_local_pipe: the CTA-local sort (k_local, §3.2 / :181-183
// §3.3) for the one-bin-per-SM configuration (512 threads), pipelined across
// bins.  k_local runs each bin as a chain of barrier-separated phases
// (count, scan, stage, fix-up, write-out) with one bin in flight, so every
// phase's latency is exposed.  Here the fix-up of bin i's colliding buckets
// (smem work on bin i's staged records) is issued in the same phase as bin
// i+1's counting atomics (smem work on other addresses), and bin i's
// write-out is one TMA bulk store that drains while bin i+1 is scanned:
//
//   [count i+1 | fix up i] #  [big buckets of i; bulk store i] [scan i+1] #
//   [wait for store i's smem reads] # [stage i+1; load i+2] # ...
//
// The collision list therefore carries each bucket's (start, count) instead
// of its index (bin i's counters are reused by bin i+1), and mixed buckets of
// more than ES_MAX records go to the next Local level (the warp tail sorter's
// scratch would alias the live counters).  Same result as k_local.
#pragma once
#include "passes.cuh"

namespace radsort {

// EF (early finish): bin i's fix-up and bulk store are issued right after it is
// staged, while bin i+1's loads are in flight, instead of beside bin i+1's
// counting atomics (which then wait on those loads)
template <int R, int K, int IL, int LB, bool EF = true>
__global__ void __launch_bounds__(LB, LB <= 256 ? 2 : 1)
    k_local_pipe(const Seg* __restrict__ list, uint32_t nlist, uint32_t wmax, uint32_t stage_bytes,
                 uint32_t cnt_bytes, uint32_t cap, Seg* local_next, int nxt, Ctl* ctl, uint8_t* recs, uint8_t* tmp,
                 uint32_t lmin, uint32_t lmax, int wdelta, uint32_t pfd) {
  extern __shared__ uint4 smem_raw[];
  constexpr int KW = K / 8;
  constexpr int NW = LB / 32;
  constexpr uint32_t ES = es_max<R>();
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem_raw);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(stage + stage_bytes);                // 2^W u16 counters
  uint32_t* blist = reinterpret_cast<uint32_t*>(stage + stage_bytes + cnt_bytes);  // start | count << 16
  __shared__ uint32_t wsum[NW], s_ncol[2], s_nbig[2], s_const;
  __shared__ unsigned long long sna[2], so[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t bi = blockIdx.x;
  auto skip = [&](uint32_t b) {
    const uint32_t l = list[b].len;
    return l > lmax || l < lmin;
  };
  while (bi < nlist && skip(bi)) bi += gridDim.x;
  if (bi >= nlist) return;
  auto zero_cnt = [&](uint32_t bytes) {
    uint4* c4 = reinterpret_cast<uint4*>(cnt);
    for (uint32_t i = tid; i < bytes / 16u; i += LB) c4[i] = make_uint4(0, 0, 0, 0);
  };
  Rec<R> r[IL];
  auto load = [&](const Seg& g) {
    const uint8_t* p = buf_of(g.src, recs, tmp) + ((size_t)g.off + tid) * R;
    const int lim = (int)g.len - tid;
#pragma unroll
    for (int i = 0; i < IL; ++i)
      if (i * LB < lim) r[i] = ldcg_rec<R>(p + (size_t)i * LB * R);  // L2 only (c4 local 16.4 -> 15.6 ms vs ld.global.nc)
  };
  auto prefetch_l2 = [&](uint32_t b) {
    if (tid == 0 && b < nlist) {
      const Seg g = list[b];
      const uintptr_t s0 = (uintptr_t)(buf_of(g.src, recs, tmp) + (size_t)g.off * R);
      const uintptr_t e0 = s0 + (size_t)g.len * R;
      const uintptr_t s1 = (s0 + 15) & ~(uintptr_t)15, e1 = e0 & ~(uintptr_t)15;
      if (e1 > s1)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s1), "r"((uint32_t)(e1 - s1)) : "memory");
    }
  };
  // the staged bin whose fix-up / write-out is still to do
  uint8_t* p_stg = nullptr;
  uint8_t* p_out = nullptr;
  uint32_t p_n = 0, p_ncol = 0, p_off = 0, p_nd = 0, par = 0;
  bool p_live = false, pending = false;
  // fix-up of the previous bin's colliding buckets (thread per bucket); > ES records: listed from the top
  auto fixup = [&]() {
    for (uint32_t e = tid; e < p_ncol; e += LB) {
      const uint32_t en = blist[e];
      const uint32_t s0 = en & 0xffffu, c = en >> 16;
      uint8_t* base = p_stg + (size_t)s0 * R;
      if (c == 2) {
        const Rec<R> x = ld_rec<R>(base), y = ld_rec<R>(base + R);
        if (key_lt(key_of<R, K>(y), key_of<R, K>(x))) { st_rec<R>(base, y); st_rec<R>(base + R, x); }
      } else if (c <= ES) {
        lane_insertion_sort<R, K>(base, c);
      } else {
        blist[cap - 1u - atomicAdd(&s_nbig[par], 1u)] = en;
      }
    }
  };
  // after the fix-up: big buckets (one warp each: one key -> final as staged, several -> next
  // Local level), then the bin's bulk store
  auto finish = [&]() {
    const uint32_t nbig = s_nbig[par];
    for (uint32_t e = warp; e < nbig; e += NW) {
      const uint32_t en = blist[cap - 1u - e];
      const uint32_t s0 = en & 0xffffu, c = en >> 16;
      const Key<K> k0 = ld_key<R, K>(p_stg + (size_t)s0 * R);
      bool diff = false;
      for (uint32_t j = s0 + lane; j < s0 + c; j += 32) diff |= !key_eq(ld_key<R, K>(p_stg + (size_t)j * R), k0);
      if (__any_sync(0xffffffffu, diff) && lane == 0) {
        Seg ns = {p_off + s0, c, (uint8_t)p_nd, SRC_REC, MODE_NONE, 0, 0};
        local_next[atomicAdd(&ctl->n_local[nxt], 1u)] = ns;
        atomicMax(&ctl->max_local_len[nxt], c);
        if (c <= small_cap<R>()) atomicAdd(&ctl->n_local_small[nxt], 1u);
        else if (c <= med_cap<R>()) atomicAdd(&ctl->n_local_med[nxt], 1u);
      }
    }
    // bulk store of the 16-byte-aligned middle; 8-byte words outside it by threads
    const uintptr_t o0 = (uintptr_t)p_out, o1 = o0 + (size_t)p_n * R;
    const uintptr_t a0 = (o0 + 15) & ~(uintptr_t)15, a1 = o1 & ~(uintptr_t)15;
    if (a1 > a0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(p_stg + (a0 - o0));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a0), "r"(sa),
                     "r"((uint32_t)(a1 - a0))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (tid == 0 && a0 > o0) *reinterpret_cast<uint2*>(o0) = *reinterpret_cast<const uint2*>(p_stg);
      if (tid == 1 && o1 > a1) *reinterpret_cast<uint2*>(a1) = *reinterpret_cast<const uint2*>(p_stg + (a1 - o0));
      pending = true;
    } else {
      for (uint32_t q = tid; q < p_n * (uint32_t)R / 8u; q += LB)
        reinterpret_cast<uint2*>(p_out)[q] = reinterpret_cast<const uint2*>(p_stg)[q];
    }
  };
  Seg sg = list[bi];
  load(sg);
  for (uint32_t k = 1; k <= pfd; ++k) prefetch_l2(bi + k * gridDim.x);
  zero_cnt(cnt_bytes);
  if (tid < 2) { sna[tid] = 0; so[tid] = 0; s_ncol[tid] = 0; s_nbig[tid] = 0; }
  if (tid == 0) s_const = 0;
  unsigned long long done = 0;
  constexpr int IP = (IL + 1) / 2;
#ifdef RADSORT_PHASE_PROF
  unsigned long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tA = clock64(), tB = 0;
#define RS_PROF(i) do { if (tid == 0) { tB = clock64(); pf[i] += tB - tA; tA = tB; } } while (0)
#else
#define RS_PROF(i) do { } while (0)
#endif
  for (;;) {
    const uint32_t n = sg.len;
    const int lim = (int)n - tid;
    uint8_t* out = recs + (size_t)sg.off * R;
    uint8_t* stg = stage + ((uintptr_t)out & 15u);
    // key bits the bin's records already share (digits, plus 2 bits below a wide level)
    uint32_t sb = 8u * sg.depth + seg_skip(sg.flags);
    const uint32_t W = (uint32_t)max((int)LOCAL_WMIN, min((int)wmax, (int)local_width(n, wmax) + wdelta));
    const uint32_t nbk = 1u << W;
    uint32_t rk[IP];
    uint32_t ones = 0;
    bool all_equal = false, first = true;
    __syncthreads();  // counters zero; the previous bin staged (stage, collision list)
    if (tid == 0) {
      const uint32_t p1 = bi + gridDim.x, p2 = p1 + gridDim.x;
      if (p1 < nlist) asm volatile("prefetch.global.L1 [%0];" ::"l"(list + p1));
      if (p2 < nlist) asm volatile("prefetch.global.L1 [%0];" ::"l"(list + p2));
      s_ncol[par ^ 1u] = 0;  // this bin's list (the previous bin's is read below)
      s_nbig[par ^ 1u] = 0;
    }
    for (;;) {  // one round unless the composite digit is constant over the bin
#pragma unroll
      for (int i = 0; i < IP; ++i) rk[i] = 0;
      ones = 0;
      bool cst = false;
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if (i * LB < lim) {
          const uint32_t b = key_bits(key_of<R, K>(r[i]), sb, W);
          const uint32_t sh = 16u * (b & 1u);
          const uint32_t old = (atomicAdd(&cnt[b >> 1], 1u << sh) >> sh) & 0xffffu;
          rk[i >> 1] |= old << (16 * (i & 1));
          ones += (uint32_t)(old == 1u);
          cst |= old == n - 1u;
        }
      }
      if (first && p_live) fixup();  // the previous bin, behind the atomics
      if (cst) s_const = 1u;
      __syncthreads();
      RS_PROF(0);
      if (first && p_live) {
        finish();  // big buckets, bulk store (contains a barrier when it stores)
        p_live = false;
      }
      first = false;
      RS_PROF(1);
      if (!s_const) {
        local_scan<LB, R == 8 ? 2 : 1>(cnt, W, wsum);  // (c5 local 6.70 -> 6.51 ms; R >= 16 lose)
        RS_PROF(2);
        if (pending && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        pending = false;
        __syncthreads();  // starts in place; the stage is free
        RS_PROF(3);
        break;
      }
      // every record in one bucket: skip the constant digits
      uint64_t na[2] = {0, 0}, o[2] = {0, 0};
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if (i * LB < lim) {
          const Key<K> k = key_of<R, K>(r[i]);
          na[0] |= ~k.w0; o[0] |= k.w0;
          if constexpr (KW == 2) { na[1] |= ~k.w1; o[1] |= k.w1; }
        }
      }
#pragma unroll
      for (int w = 0; w < KW; ++w) {
        const uint32_t x0 = __reduce_or_sync(0xffffffffu, (uint32_t)na[w]);
        const uint32_t x1 = __reduce_or_sync(0xffffffffu, (uint32_t)(na[w] >> 32));
        const uint32_t y0 = __reduce_or_sync(0xffffffffu, (uint32_t)o[w]);
        const uint32_t y1 = __reduce_or_sync(0xffffffffu, (uint32_t)(o[w] >> 32));
        if (lane == 0) { atomicOr(&sna[w], u64of(x0, x1)); atomicOr(&so[w], u64of(y0, y1)); }
      }
      __syncthreads();
      uint64_t A[2] = {~(uint64_t)sna[0], ~(uint64_t)sna[1]}, O[2] = {so[0], so[1]};
      const uint32_t d2 = first_nonconst_digit<K>(A, O, sb / 8u);
      __syncthreads();
      zero_cnt(2u << W);
      if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
      if (tid == 0) s_const = 0;
      __syncthreads();
      if (d2 >= (uint32_t)K) { all_equal = true; break; }
      sb = 8u * d2;
    }
    const uint32_t q = par ^ 1u;  // this bin's list parity
    const uint16_t* start16 = reinterpret_cast<const uint16_t*>(cnt);
    const bool fix = 8u * K > sb + W;  // key bits left below the composite digit
    if (all_equal) {  // final where it is (copied out of tmp)
      if (sg.src == SRC_TMP) {
#pragma unroll
        for (int i = 0; i < IL; ++i)
          if (i * LB < lim) st_rec<R>(out + (size_t)(i * LB + tid) * R, r[i]);
      }
    } else {
      uint32_t inc = ones;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      uint32_t slot = 0;
      if (lane == 31 && inc && fix) slot = atomicAdd(&s_ncol[q], inc);
      slot = __shfl_sync(0xffffffffu, slot, 31) + inc - ones;
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if (i * LB < lim) {
          const uint32_t b = key_bits(key_of<R, K>(r[i]), sb, W);
          const uint32_t rnk = (rk[i >> 1] >> (16 * (i & 1))) & 0xffffu;
          st_rec<R>(stg + (size_t)(start16[b] + rnk) * R, r[i]);
          if (rnk == 1u && fix) blist[slot++] = b;  // the bucket; turned into start | count below
        }
      }
    }
    RS_PROF(5);
    // registers are free: the next bin's loads overlap this bin's finish
    uint32_t nb = bi + gridDim.x;
    while (nb < nlist && skip(nb)) nb += gridDim.x;
    Seg nsg = sg;
    if (nb < nlist) {
      nsg = list[nb];
      load(nsg);
    }
    if (pfd) prefetch_l2(nb + pfd * gridDim.x);  // the bin pfd ahead of the one being loaded streams into L2
    done += n;
    RS_PROF(4);
    __syncthreads();  // staged
    if (!all_equal) {
      p_live = true;
      p_stg = stg;
      p_out = out;
      p_n = n;
      p_ncol = s_ncol[q];
      p_off = sg.off;
      p_nd = (sb + W) / 8u;  // digits shared by a bucket's keys
      // collision list: bucket -> start | count << 16 (the counters are reused by the next bin)
      for (uint32_t e = tid; e < p_ncol; e += LB) {
        const uint32_t b = blist[e], s0 = start16[b];
        blist[e] = s0 | (((b + 1 < nbk ? (uint32_t)start16[b + 1] : n) - s0) << 16);
      }
      __syncthreads();  // starts consumed
    }
    par = q;
    zero_cnt(2u << W);
    RS_PROF(6);
    if constexpr (EF) {
      if (p_live) {
        fixup();
        __syncthreads();  // fix-ups done; the big-bucket list complete
        RS_PROF(1);
        finish();
        p_live = false;
      }
    }
    RS_PROF(7);
    if (nb >= nlist) break;
    bi = nb;
    sg = nsg;
  }
  if (p_live) {  // the last bin
    __syncthreads();
    fixup();
    __syncthreads();
    finish();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (tid == 0) atomicAdd(&ctl->rec_local, done);
#ifdef RADSORT_PHASE_PROF
  if (tid == 0)
    for (int q = 0; q < 8; ++q) atomicAdd(&ctl->prof[8 + q], pf[q]);
#endif
#undef RS_PROF
}

}  // namespace radsort
