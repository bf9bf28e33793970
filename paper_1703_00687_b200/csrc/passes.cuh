// radsort kernels: one MSD level = sample/hist -> plan -> scatter -> children,
// plus the CTA-local sorter.  See DESIGN.md §3 for the roofline of each.
#pragma once
#include "kernels.cuh"

namespace radsort {

__device__ __forceinline__ uint8_t* buf_of(uint8_t src, uint8_t* recs, uint8_t* tmp) { return src == SRC_TMP ? tmp : recs; }

// Index of the segment owning tile t: largest s with tile_start[s] <= t.
__device__ __forceinline__ uint32_t seg_of_tile(const uint32_t* __restrict__ tile_start, uint32_t nseg, uint32_t t) {
  uint32_t lo = 0, hi = nseg;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(tile_start + mid) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// -------------------------------------------------------------- k_tilemap
// tile -> segment map of the level (one independent binary search per tile,
// all in parallel), so the histogram and scatter passes look a tile's segment
// up with one load instead of a chain of dependent ones.
static __global__ void k_tilemap(const uint32_t* __restrict__ tile_start, uint32_t nseg, const Ctl* __restrict__ ctl,
                                 uint32_t* __restrict__ tile_seg) {
  const uint32_t total = ctl->tiles_total;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x)
    tile_seg[t] = seg_of_tile(tile_start, nseg, t);
}

// Bins of up to small_cap<R>() records are sorted by 64-thread CTAs (<= 256
// bytes of records per thread; Sorter::launch_local).
template <int R>
__host__ __device__ constexpr uint32_t small_cap() {
  return 64u * (256 / R >= 16 ? 16u : (256 / R >= 8 ? 8u : 4u));
}
// ... and bins of up to med_cap<R>() by 256-thread CTAs, two per SM (above it: 512 x 1)
template <int R>
__host__ __device__ constexpr uint32_t med_cap() {
  return 256u * ((local_capacity<R>() + 511u) / 512u);
}

// -------------------------------------------------------------- k_init
// Level-0 set-up: the whole input is one bin.  If it fits the CTA-local
// sorter it goes straight to the Local list, otherwise it becomes the single
// Large segment of level 0 ("parallel processing of the whole
// array according to the first digit").
static __global__ void k_init(Seg* large0, Seg* local0, Ctl* ctl, uint32_t n, uint32_t local_cap) {
  Ctl c = {};
  Seg s = {0u, n, 0, SRC_REC, MODE_NONE, 0, 0};
  if (n <= local_cap) {
    local0[0] = s;
    c.n_local[0] = 1;
    c.max_local_len[0] = n;
  } else {
    large0[0] = s;
  }
  *ctl = c;
}

// -------------------------------------------------------------- k_sample
// Guess the first non-constant digit d0 from a strided sample (AND/OR of the
// sampled keys).  A digit constant over the whole input is constant over any
// sample, so the guess is never below the true d0; k_plan corrects it from
// the full AND/OR if it was too high (one extra histogram read).
template <int R, int K>
__global__ void k_sample(Seg* large0, Ctl* ctl, const uint8_t* __restrict__ recs, uint32_t n) {
  __shared__ unsigned long long sa[2], so[2];
  constexpr int KW = K / 8;
  if (threadIdx.x < 2) { sa[threadIdx.x] = ~0ull; so[threadIdx.x] = 0ull; }
  __syncthreads();
  uint64_t a[2] = {~0ull, ~0ull}, o[2] = {0ull, 0ull};
  const uint32_t S = 4096;
  const uint32_t stride = n > S ? n / S : 1;
  for (uint32_t i = threadIdx.x; i < S && (uint64_t)i * stride < n; i += blockDim.x) {
    Key<K> k = key_of<R, K>(ldg_rec<R>(recs + (size_t)i * stride * R));
    a[0] &= k.w0; o[0] |= k.w0;
    if constexpr (KW == 2) { a[1] &= k.w1; o[1] |= k.w1; }
  }
  for (int w = 0; w < KW; ++w) { atomicAnd(&sa[w], a[w]); atomicOr(&so[w], o[w]); }
  __syncthreads();
  if (threadIdx.x == 0) {  // k_init's Large case, folded in (one launch fewer per sort)
    uint64_t A[2] = {sa[0], sa[1]}, O[2] = {so[0], so[1]};
    uint32_t d = first_nonconst_digit<K>(A, O, 0);
    if (d >= (uint32_t)K) d = 0;
    Ctl c = {};
    c.d0 = d;
    *ctl = c;
    large0[0] = Seg{0u, n, (uint8_t)d, SRC_REC, MODE_NONE, 0, 0};
  }
}

// ------------------------------------------------------------- k_dupest
// Duplicate-key estimate for the wide-level rule of R < 24: S keys
// at evenly spaced positions are hashed to 64 bits and inserted into an
// open-addressing table (zeroed scratch at the head of tmp, 4 S slots); a
// sample that meets an equal hash counts in Ctl::dup_est.  Two records share
// a key with probability p2 ~ dup_est / (S^2 / 2), so a record has ~ p2 n
// equal partners in the input: the 10-bit level leaves bins close to the
// CTA-local capacity, which sort slowly when their keys repeat (kmc), so
// R < 24 takes it only where p2 n is small.
template <int R, int K>
__global__ void __launch_bounds__(256) k_dupest(Ctl* ctl, const uint8_t* __restrict__ recs, uint32_t n, uint32_t S,
                                                unsigned long long* table, uint32_t tmask) {
  const uint32_t i = blockIdx.x * 256u + threadIdx.x;
  if (i >= S) return;
  const uint64_t pos = (uint64_t)i * n / S;
  const Key<K> k = key_of<R, K>(ldg_rec<R>(recs + pos * R));
  uint64_t h = k.w0;
  if constexpr (K == 16) {
    uint64_t g = k.w1 + 0x9E3779B97F4A7C15ull;
    g = (g ^ (g >> 30)) * 0xBF58476D1CE4E5B9ull;
    h ^= g ^ (g >> 31);
  }
  h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
  h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
  h = (h ^ (h >> 31)) | 1ull;  // never the empty slot's 0
  uint32_t slot = (uint32_t)(h >> 32) & tmask;
  for (int p = 0; p < 256; ++p) {
    const unsigned long long old = atomicCAS(&table[slot], 0ull, (unsigned long long)h);
    if (old == 0ull) return;
    if (old == h) {
      atomicAdd(&ctl->dup_est, 1u);
      return;
    }
    slot = (slot + 1) & tmask;
  }
}

// -------------------------------------------------------------- k_prep
// Per level: tiles per Large segment -> exclusive prefix (single CTA), and
// reset of the level's counters.
static __global__ void k_prep(const Seg* __restrict__ segs, uint32_t nseg, uint32_t tile_recs, uint32_t* tile_start,
                       Ctl* ctl, int nxt) {
  __shared__ uint32_t ws[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint32_t per = (nseg + nt - 1) / nt;
  const uint32_t b = tid * per, e = min(nseg, b + per);
  uint32_t sum = 0;
  for (uint32_t s = b; s < e; ++s) sum += (segs[s].len + tile_recs - 1) / tile_recs;
  // block exclusive scan of `sum` (blockDim = 1024)
  const int lane = tid & 31, w = tid >> 5;
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;
  }
  __syncthreads();
  uint32_t run = x - sum + (w > 0 ? ws[w - 1] : 0u);
  for (uint32_t s = b; s < e; ++s) {
    tile_start[s] = run;
    run += (segs[s].len + tile_recs - 1) / tile_recs;
  }
  if (tid == nt - 1) {
    tile_start[nseg] = run;
    ctl->tiles_total = run;
    ctl->scatter_ticket = 0;
    ctl->n_large_next = 0;
    ctl->rec_large_next = 0;
    ctl->n_local[nxt] = 0;
    ctl->n_local_small[nxt] = 0;
    ctl->n_local_med[nxt] = 0;
    ctl->max_local_len[nxt] = 0;
  }
}

// -------------------------------------------------------------- k_cand
// One warp per Large segment: 32 keys sampled evenly across the segment are
// compared with its first key; 12 or more matches flag the segment as
// possibly dominated by that key (FLAG_CAND), and only flagged segments pay
// for counting the exact equal/below counts in k_hist_pre (k_plan decides).
template <int R, int K>
__global__ void k_cand(Seg* segs, uint32_t nseg, const uint8_t* recs, const uint8_t* tmp) {
  const uint32_t s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= nseg) return;
  const Seg sg = segs[s];
  if (sg.flags & (FLAG_EQUAL | FLAG_FILL)) return;
  const uint8_t* b = (sg.src == SRC_TMP ? tmp : recs) + (size_t)sg.off * R;
  const Key<K> k0 = ld_key<R, K>(b);
  const Key<K> kj = ld_key<R, K>(b + (size_t)((uint64_t)sg.len * (uint32_t)lane / 32u) * R);
  const int votes = __popc(__ballot_sync(0xffffffffu, key_eq(kj, k0)));
  if (lane == 0) segs[s].flags = (uint8_t)((sg.flags & ~FLAG_CAND) | (votes >= 12 ? FLAG_CAND : 0));
}

// -------------------------------------------------------------- k_hist
// Per-segment histogram of the segment's digit + AND/OR of its keys, one read
// of the data ("counting sort may be applied per single phase").
// Each CTA owns a contiguous range of tiles and accumulates in shared memory
// (smem atomics: measured ~10/clk/SM on B200, ample for one digit per record)
// until the segment changes, so global atomics are per CTA and segment, not per
// tile.  andor[s] = {OR of ~key words, OR of key words}: all accumulators start
// at zero.
template <int R, int K, uint32_t T>
__global__ void __launch_bounds__(HIST_B) k_hist(const Seg* __restrict__ segs, const uint32_t* __restrict__ tile_start,
                                                 uint32_t nseg, const Ctl* __restrict__ ctl, uint32_t* __restrict__ hist,
                                                 unsigned long long* __restrict__ andor, const uint8_t* recs,
                                                 const uint8_t* tmp) {
  constexpr int KW = K / 8;
  constexpr int U = 8;  // keys in flight per thread
  __shared__ uint32_t h[RADIX];
  __shared__ unsigned long long sna[2], so[2];
  const uint32_t total = ctl->tiles_total;
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * per, t1 = min(total, t0 + per);
  if (t0 >= t1) return;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < RADIX; i += HIST_B) h[i] = 0;
  if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  __syncthreads();
  uint64_t na[2] = {0, 0}, o[2] = {0, 0};
  unsigned long long cnt_recs = 0;
  uint32_t cur = seg_of_tile(tile_start, nseg, t0);
  uint32_t cur_end = tile_start[cur + 1];
  auto flush = [&](uint32_t s) {
#pragma unroll
    for (int w = 0; w < KW; ++w) {
      const uint32_t x0 = __reduce_or_sync(0xffffffffu, (uint32_t)na[w]);
      const uint32_t x1 = __reduce_or_sync(0xffffffffu, (uint32_t)(na[w] >> 32));
      const uint32_t y0 = __reduce_or_sync(0xffffffffu, (uint32_t)o[w]);
      const uint32_t y1 = __reduce_or_sync(0xffffffffu, (uint32_t)(o[w] >> 32));
      if (lane == 0) { atomicOr(&sna[w], u64of(x0, x1)); atomicOr(&so[w], u64of(y0, y1)); }
      na[w] = 0;
      o[w] = 0;
    }
    __syncthreads();
    for (int i = tid; i < RADIX; i += HIST_B) {
      if (h[i]) atomicAdd(&hist[(size_t)s * RADIX + i], h[i]);
      h[i] = 0;
    }
    if (tid < KW) {
      if (sna[tid]) atomicOr(&andor[(size_t)s * 8 + tid], sna[tid]);
      if (so[tid]) atomicOr(&andor[(size_t)s * 8 + 2 + tid], so[tid]);
    }
    __syncthreads();
    if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  };
  for (uint32_t t = t0; t < t1; ++t) {
    if (t >= cur_end) {
      flush(cur);
      cur = seg_of_tile(tile_start, nseg, t);
      cur_end = tile_start[cur + 1];
    }
    const Seg sg = segs[cur];
    if (sg.flags & (FLAG_EQUAL | FLAG_FILL)) continue;
    const uint32_t lt = t - tile_start[cur];
    const uint32_t m = min(T, sg.len - lt * T);
    const uint8_t* src = (sg.src == SRC_TMP ? tmp : recs) + (size_t)(sg.off + lt * T) * R;
    const uint32_t d = sg.depth;
    for (uint32_t i0 = tid; i0 < m; i0 += HIST_B * U) {
      Key<K> k[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + u * HIST_B;
        if (i < m) k[u] = key_of<R, K>(ldg_rec<R>(src + (size_t)i * R));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + u * HIST_B;
        if (i < m) {
          atomicAdd(&h[digit_of(k[u], d)], 1u);
          na[0] |= ~k[u].w0; o[0] |= k[u].w0;
          if constexpr (KW == 2) { na[1] |= ~k[u].w1; o[1] |= k[u].w1; }
        }
      }
    }
    cnt_recs += m;
  }
  flush(cur);
  if (tid == 0 && cnt_recs) atomicAdd((unsigned long long*)&ctl->rec_hist, cnt_recs);
}

// -------------------------------------------------------------- k_hist_pre
// k_hist plus the cross-tile prefix the scatter needs, so the scatter has no
// inter-CTA dependency (reduce-then-scan instead of look-back).  CTA c owns the
// contiguous chunk of tiles [c*per, (c+1)*per).  For every tile it writes
// tile_pre[t][v] = count of digit v in the tiles of the same segment that
// precede t inside the chunk; per chunk it writes its first and last segment
// and ch_tot[c][v] = count of digit v of the chunk's last segment in the chunk
// (k_carry turns these into each chunk's carry-in).
constexpr uint32_t NO_SEG = 0xffffffffu;
template <int R, int K, uint32_t T, int DB = 8>
__global__ void __launch_bounds__(HIST_B, 4) k_hist_pre(const Seg* __restrict__ segs, const uint32_t* __restrict__ tile_start,
                                                     uint32_t nseg, const Ctl* __restrict__ ctl,
                                                     uint32_t* __restrict__ hist, unsigned long long* __restrict__ andor,
                                                     const uint8_t* recs, const uint8_t* tmp, uint32_t* __restrict__ tile_pre,
                                                     uint32_t* __restrict__ ch_first, uint32_t* __restrict__ ch_last,
                                                     uint32_t* __restrict__ ch_tot, const uint32_t* __restrict__ tile_seg) {
  constexpr int KW = K / 8;
  constexpr int DG = 1 << DB;  // digits of the pass (256, or 1024 on a wide level)
  constexpr int U = DB == 10 ? (R <= 8 ? 8 : 4) : (R <= 8 ? 16 : 8);  // keys in flight per thread (wide: registers)
  __shared__ uint32_t h[DG], run[DG];
  __shared__ unsigned long long sna[2], so[2];
  const uint32_t total = ctl->tiles_total;
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t c = blockIdx.x;
  const uint32_t t0 = c * per, t1 = min(total, t0 + per);
  const int tid = threadIdx.x, lane = tid & 31;
  if (t0 >= t1) {
    if (tid == 0) ch_first[c] = ch_last[c] = NO_SEG;
    return;
  }
  for (int i = tid; i < DG; i += HIST_B) h[i] = run[i] = 0;
  if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  __syncthreads();
  uint64_t na[2] = {0, 0}, o[2] = {0, 0};
  uint32_t n_eq = 0, n_lt = 0;  // keys equal to / below the segment's probe key
  unsigned long long cnt_recs = 0;
  uint32_t cur = __ldg(tile_seg + t0);
  uint32_t cur_end = tile_start[cur + 1];
  Key<K> probe{};
  uint32_t probe_seg = NO_SEG;  // the probe (first record's key) is loaded once per segment
  if (tid == 0) ch_first[c] = cur;
  auto flush = [&](uint32_t s) {
    {
      const uint32_t e = __reduce_add_sync(0xffffffffu, n_eq), l = __reduce_add_sync(0xffffffffu, n_lt);
      if (lane == 0 && e) atomicAdd(&andor[(size_t)s * 8 + 4], (unsigned long long)e);
      if (lane == 0 && l) atomicAdd(&andor[(size_t)s * 8 + 5], (unsigned long long)l);
      n_eq = 0;
      n_lt = 0;
    }
#pragma unroll
    for (int w = 0; w < KW; ++w) {
      const uint32_t x0 = __reduce_or_sync(0xffffffffu, (uint32_t)na[w]);
      const uint32_t x1 = __reduce_or_sync(0xffffffffu, (uint32_t)(na[w] >> 32));
      const uint32_t y0 = __reduce_or_sync(0xffffffffu, (uint32_t)o[w]);
      const uint32_t y1 = __reduce_or_sync(0xffffffffu, (uint32_t)(o[w] >> 32));
      if (lane == 0) { atomicOr(&sna[w], u64of(x0, x1)); atomicOr(&so[w], u64of(y0, y1)); }
      na[w] = 0;
      o[w] = 0;
    }
    __syncthreads();
    for (int i = tid; i < DG; i += HIST_B) {
      if (run[i]) atomicAdd(&hist[(size_t)s * DG + i], run[i]);
      run[i] = 0;
    }
    if (tid < KW) {
      if (sna[tid]) atomicOr(&andor[(size_t)s * 8 + tid], sna[tid]);
      if (so[tid]) atomicOr(&andor[(size_t)s * 8 + 2 + tid], so[tid]);
    }
    __syncthreads();
    if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  };
  for (uint32_t t = t0; t < t1; ++t) {
    if (t >= cur_end) {
      flush(cur);
      cur = __ldg(tile_seg + t);
      cur_end = tile_start[cur + 1];
    }
    const Seg sg = segs[cur];
    if (sg.flags & (FLAG_EQUAL | FLAG_FILL)) continue;
    const uint32_t lt = t - tile_start[cur];
    const uint32_t m = min(T, sg.len - lt * T);
    const uint8_t* sbase = (sg.src == SRC_TMP ? tmp : recs) + (size_t)sg.off * R;
    const uint8_t* src = sbase + (size_t)lt * T * R;
    if ((sg.flags & FLAG_CAND) && probe_seg != cur) {
      probe = ld_key<R, K>(sbase);
      probe_seg = cur;
    }
    const uint32_t d = sg.depth;
    if (!(sg.flags & FLAG_CAND)) {
      for (uint32_t i0 = tid; i0 < m; i0 += HIST_B * U) {
        Key<K> k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = i0 + u * HIST_B;
          if (i < m) k[u] = key_of<R, K>(ldg_rec<R>(src + (size_t)i * R));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = i0 + u * HIST_B;
          if (i < m) {
            atomicAdd(&h[digit_w<DB>(k[u], d)], 1u);
            na[0] |= ~k[u].w0; o[0] |= k[u].w0;
            if constexpr (KW == 2) { na[1] |= ~k[u].w1; o[1] |= k[u].w1; }
          }
        }
      }
    } else {  // a candidate for the dominant-key split: also count keys equal to / below the probe
      constexpr int U2 = U / 2;
      for (uint32_t i0 = tid; i0 < m; i0 += HIST_B * U2) {
        Key<K> k[U2];
#pragma unroll
        for (int u = 0; u < U2; ++u) {
          const uint32_t i = i0 + u * HIST_B;
          if (i < m) k[u] = key_of<R, K>(ldg_rec<R>(src + (size_t)i * R));
        }
#pragma unroll
        for (int u = 0; u < U2; ++u) {
          const uint32_t i = i0 + u * HIST_B;
          if (i < m) {
            atomicAdd(&h[digit_w<DB>(k[u], d)], 1u);
            na[0] |= ~k[u].w0; o[0] |= k[u].w0;
            if constexpr (KW == 2) { na[1] |= ~k[u].w1; o[1] |= k[u].w1; }
            n_eq += (uint32_t)key_eq(k[u], probe);
            n_lt += (uint32_t)key_lt(k[u], probe);
          }
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < DG; i += HIST_B) {
      tile_pre[(size_t)t * DG + i] = run[i];
      run[i] += h[i];
      h[i] = 0;
    }
    __syncthreads();
    cnt_recs += m;
  }
  for (int i = tid; i < DG; i += HIST_B) ch_tot[(size_t)c * DG + i] = run[i];
  if (tid == 0) ch_last[c] = cur;
  flush(cur);
  if (tid == 0 && cnt_recs) atomicAdd((unsigned long long*)&ctl->rec_hist, cnt_recs);
}

// -------------------------------------------------------------- k_carry
// Carry of each chunk's first segment from the earlier chunks: a segmented
// scan over the chunks, one thread per digit (single CTA; 32 chunks in flight).
template <int DG = RADIX>
__global__ void __launch_bounds__(DG) k_carry(const uint32_t* __restrict__ ch_first, const uint32_t* __restrict__ ch_last,
                                                 const uint32_t* __restrict__ ch_tot, uint32_t nch,
                                                 uint32_t* __restrict__ carry_in) {
  const int d = threadIdx.x;
  uint32_t carry = 0, prev_last = NO_SEG;
  constexpr int B = DG > 256 ? 16 : 32;  // chunks in flight (1024 threads: 64 registers)
  for (uint32_t c0 = 0; c0 < nch; c0 += B) {
    uint32_t f[B], l[B], tt[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const uint32_t c = c0 + j;
      f[j] = c < nch ? __ldg(ch_first + c) : NO_SEG;
      l[j] = c < nch ? __ldg(ch_last + c) : NO_SEG;
      tt[j] = c < nch ? __ldg(ch_tot + (size_t)c * DG + d) : 0u;
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const uint32_t c = c0 + j;
      if (c >= nch || f[j] == NO_SEG) continue;
      const uint32_t cin = (f[j] == prev_last) ? carry : 0u;
      carry_in[(size_t)c * DG + d] = cin;
      carry = (f[j] == l[j] ? cin : 0u) + tt[j];
      prev_last = l[j];
    }
  }
}

// -------------------------------------------------------------- k_plan
// Per Large segment: constant-digit skip / all-equal detection,
// bin bases = exclusive prefix of the histogram.  A segment in
// which more than half of the records carry its first record's key (a
// dominant key: skewed inputs, PAPER.md:247 Zipf) is split three ways instead
// -- keys below / equal to / above that key -- so the dominant key's records
// are final after one pass rather than being carried through every later
// level with the few other keys of their bin ("bins with all keys
// equal" generalised to "all but a few").  andor[s] holds 8
// words: ~AND (2), OR (2), #keys == probe, #keys < probe (k_hist_pre).
template <int R, int K, int DG = RADIX>
__global__ void __launch_bounds__(DG) k_plan(Seg* segs, uint32_t* __restrict__ hist,
                                                const unsigned long long* __restrict__ andor,
                                                uint32_t* __restrict__ segbase, Seg* large_next, Ctl* ctl,
                                                uint32_t* __restrict__ splitc, int split_ok, int force = 0) {
  __shared__ uint32_t ws[DG / 32];
  __shared__ int sh_const, sh_requeue;
  const uint32_t s = blockIdx.x;
  const int tid = threadIdx.x;
  const Seg sg = segs[s];
  if (sg.flags & (FLAG_EQUAL | FLAG_FILL)) {  // known final bin: copied tmp -> records / filled with its key
    if (tid == 0) {
      segs[s].mode = (sg.flags & FLAG_FILL) ? MODE_FILL : (sg.src == SRC_TMP ? MODE_COPY : MODE_NONE);
      atomicAdd(&ctl->rec_final, (unsigned long long)sg.len);
    }
    return;
  }
  const unsigned long long* ao = andor + (size_t)s * 8;
  if (tid == 0) {
    sh_const = 0;
    sh_requeue = 0;
    // The digit a segment is histogrammed at must be its first non-constant
    // one.  Bins below level 0 share their leading digits by construction; the
    // level-0 depth is a guess from a strided sample (k_sample) that can be too
    // deep when the sample misses a record differing in a higher digit.  The
    // full-pass AND/OR decides: a segment with a non-constant digit above its
    // depth is histogrammed again at that digit (one extra read, rare).
    if (!force) {
      uint64_t A[2], O[2];
      for (int w = 0; w < K / 8; ++w) { A[w] = ~ao[w]; O[w] = ao[2 + w]; }
      const uint32_t dt = first_nonconst_digit<K>(A, O, 0);
      if (dt < (uint32_t)sg.depth) {
        segs[s].mode = MODE_NONE;
        Seg ns = sg;
        ns.depth = (uint8_t)dt;
        ns.mode = MODE_NONE;
        ns.flags = (uint8_t)(sg.flags & ~(FLAG_CAND | FLAG_SKIP_MASK));
        large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
        atomicAdd(&ctl->rec_large_next, (unsigned long long)sg.len);
        atomicMin(&ctl->d0, dt);
        sh_requeue = 1;
      }
    }
  }
  __syncthreads();
  if (sh_requeue) return;
  const uint32_t c = hist[(size_t)s * DG + tid];
  if (c == sg.len && !force) sh_const = 1;
  __syncthreads();
  if (sh_const) {
    if (tid == 0) {
      uint64_t A[2], O[2];
      for (int w = 0; w < K / 8; ++w) { A[w] = ~ao[w]; O[w] = ao[2 + w]; }
      const uint32_t d2 = first_nonconst_digit<K>(A, O, sg.depth);
      if (d2 >= (uint32_t)K) {  // all keys equal: final
        segs[s].mode = sg.src == SRC_TMP ? MODE_COPY : MODE_NONE;
        atomicAdd(&ctl->rec_final, (unsigned long long)sg.len);
      } else {                  // skip constant digits, re-histogram next level
        segs[s].mode = MODE_NONE;
        Seg ns = sg;
        ns.depth = (uint8_t)d2;
        ns.mode = MODE_NONE;
        ns.flags = (uint8_t)(sg.flags & ~FLAG_SKIP_MASK);
        large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
        atomicAdd(&ctl->rec_large_next, (unsigned long long)sg.len);
      }
    }
    return;
  }
  const uint32_t n_eq = (uint32_t)ao[4], n_lt = (uint32_t)ao[5];
  // the equal records become final: written straight to `records` when the
  // segment sits in tmp; when it sits in `records` they can only be skipped
  // and re-filled (records that are all key, R == K)
  if (split_ok && (sg.flags & FLAG_CAND) && 2ull * n_eq > sg.len && (sg.src == SRC_TMP || R == K)) {
    __syncthreads();
    hist[(size_t)s * DG + tid] = tid == 0 ? n_lt : tid == 1 ? n_eq : tid == 2 ? sg.len - n_lt - n_eq : 0u;
    if (tid < 3) segbase[(size_t)s * DG + tid] = sg.off + (tid >= 1 ? n_lt : 0u) + (tid == 2 ? n_eq : 0u);
    if (tid < 4) splitc[(size_t)s * 4 + tid] = 0;
    if (tid == 0) {
      segs[s].mode = MODE_SPLIT;
      atomicAdd(&ctl->bins_split, 1ull);
      atomicAdd(&ctl->rec_split, (unsigned long long)n_eq);
    }
    return;
  }
  const uint32_t ex = block_excl_scan<DG>(c, ws);
  segbase[(size_t)s * DG + tid] = sg.off + ex;
  if (tid == 0) segs[s].mode = MODE_SCATTER;
}

// One tile of a MODE_SPLIT segment (k_plan): three-way split around the
// segment's dominant key -- class 0/1/2 = key below / equal to / above it.
// Ranks by warp ballots + one smem atomic per class and warp; each class's range
// is reserved per tile with one global atomic (order inside a class is free,
// DESIGN.md R2).  The equal class is final: written to `records` (segment in
// tmp), or skipped and filled later (segment in `records`, R == K).  Reads the
// tile twice from L1/L2 (the scatter's register prefetch of the tile warms
// them) and is kept out of line so the digit scatter's register allocation
// does not pay for it.  Every thread calls it.
template <int R, int K, int SB, int DG = RADIX>
__device__ __noinline__ void split_tile(const Seg sg, uint32_t s, uint32_t base, uint32_t m, uint8_t* dst,
                                        uint8_t* recs, uint8_t* tmp, const uint32_t* __restrict__ segbase,
                                        uint32_t* __restrict__ splitc, uint8_t* stage, uint32_t* cnt,
                                        uint32_t* gofs) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint8_t* sb = buf_of(sg.src, recs, tmp);
  const uint8_t* src = sb + (size_t)base * R;
  const Key<K> probe = ld_key<R, K>(sb + (size_t)sg.off * R);
  uint32_t* rkv = reinterpret_cast<uint32_t*>(stage);  // per-record class << 16 | rank (T * 4 <= TB bytes)
  const uint32_t lanelt = (1u << lane) - 1u;
  for (uint32_t q0 = 0; q0 < m; q0 += SB) {
    const uint32_t q = q0 + tid;
    uint32_t cl = 3u;
    if (q < m) {
      const Key<K> kx = ld_key<R, K>(src + (size_t)q * R);
      cl = key_lt(kx, probe) ? 0u : (key_eq(kx, probe) ? 1u : 2u);
    }
    const uint32_t m0 = __ballot_sync(0xffffffffu, cl == 0u), m1 = __ballot_sync(0xffffffffu, cl == 1u),
                   m2 = __ballot_sync(0xffffffffu, cl == 2u);
    uint32_t b = 0;
    if (lane < 3) {
      const uint32_t mm = lane == 0 ? m0 : (lane == 1 ? m1 : m2);
      if (mm) b = atomicAdd(&cnt[lane], (uint32_t)__popc(mm));
    }
    const uint32_t b0 = __shfl_sync(0xffffffffu, b, 0), b1 = __shfl_sync(0xffffffffu, b, 1),
                   b2 = __shfl_sync(0xffffffffu, b, 2);
    const uint32_t mk = cl == 0u ? m0 : (cl == 1u ? m1 : m2);
    if (q < m) rkv[q] = ((cl == 0u ? b0 : (cl == 1u ? b1 : b2)) + (uint32_t)__popc(mk & lanelt)) | (cl << 16);
  }
  __syncthreads();
  if (tid < 3) gofs[tid] = segbase[(size_t)s * DG + tid] + atomicAdd(&splitc[(size_t)s * 4 + tid], cnt[tid]);
  __syncthreads();
  const bool eq_skip = sg.src == SRC_REC;  // R == K: the equal run is filled later
  for (uint32_t q = tid; q < m; q += SB) {
    const uint32_t v = rkv[q], cl = v >> 16;
    if (cl == 1u && eq_skip) continue;
    st_rec<R>((cl == 1u ? recs : dst) + (size_t)(gofs[cl] + (v & 0xffffu)) * R, ldg_rec<R>(src + (size_t)q * R));
  }
}

// -------------------------------------------------------------- k_scatter
// One radix pass over every SCATTER segment of the level (§2.1
// buffered scatter, §3.2): per tile, rank each record inside
// its digit with shared-memory atomics, stage the tile in smem grouped by
// digit, obtain each digit's global offset by single-pass decoupled look-back
// over the segment's tiles, and write every digit run with coalesced stores.
// Tiles come from an atomic ticket so look-back only waits on running CTAs.
constexpr int SCATTER_PAD = 64;  // dynamic smem beyond the TB-byte tile: the pad slot of absent records

// TMA write-out of a record size that is an odd multiple of 8 bytes (8, 24, 40):
// a run is 16-byte aligned in HBM only from an even record position, so each
// digit's run is staged at the parity of its global position (one spare slot
// per digit, DG + 1 more slots); its odd head / tail record leaves as a plain
// store, the even middle as one bulk copy
template <int R, int TB, int SB, int DB, bool TMA_OUT>
__host__ __device__ constexpr bool scatter_parity() { return TMA_OUT && R % 16 != 0; }
template <int R, int TB, int SB, int DB, bool TMA_OUT>
__host__ __device__ constexpr uint32_t scatter_padslot() {
  return scatter_parity<R, TB, SB, DB, TMA_OUT>() ? tile_recs<R, TB, SB>() + (1u << DB) + 1u : tile_recs<R, TB, SB>();
}
template <int R, int TB, int SB, int DB, bool TMA_OUT>
__host__ __device__ constexpr size_t scatter_smem() {
  return scatter_parity<R, TB, SB, DB, TMA_OUT>()
             ? (((size_t)(scatter_padslot<R, TB, SB, DB, TMA_OUT>() + 1u) * R + 15) & ~(size_t)15)
             : (size_t)TB + SCATTER_PAD;
}

template <int R, int K, int TB, int SB, int MINB, bool PRE, bool PEER = false, int DB = 8, bool TMA_OUT = false>
__global__ void __launch_bounds__(SB, MINB) k_scatter(const Seg* __restrict__ segs, const uint32_t* __restrict__ tile_start,
                                                       uint32_t nseg, const uint32_t* __restrict__ segbase,
                                                       unsigned long long* __restrict__ status, uint32_t epoch, Ctl* ctl,
                                                       uint8_t* recs, uint8_t* tmp, const uint32_t* __restrict__ tile_pre,
                                                       const uint32_t* __restrict__ ch_first,
                                                       const uint32_t* __restrict__ carry_in, uint32_t hist_grid,
                                                       uint32_t* __restrict__ splitc,
                                                       const unsigned long long* __restrict__ probes,
                                                       const uint32_t* __restrict__ tile_seg,
                                                       const unsigned long long* __restrict__ seg_dst = nullptr) {
  constexpr uint32_t T = tile_recs<R, TB, SB>();
  constexpr int I = (int)(T / SB);
  constexpr int LBW = 8;  // look-back window: predecessor statuses loaded in parallel
  constexpr int DG = 1 << DB;  // digits of the pass: 256, or 1024 on a wide level
  constexpr int DPT = DG > SB ? DG / SB : 1;  // digits per thread (consecutive: tid * DPT + j)
  static_assert(DB == 8 ? DG <= SB : (PRE && (SB == DG || 2 * SB == DG)),
                "a wide pass: one or two digits per thread, reduce-then-scan offsets");
  // TMA write-out: every digit's staged run leaves as one bulk copy (cp.async.bulk
  // shared -> global, issued by the digit's thread) that drains while the next
  // tile is loaded, ranked and scanned; needs 16-byte aligned runs (R = 16, 32)
  constexpr bool TW = TMA_OUT && PRE && !PEER;
  constexpr bool TWP = TW && scatter_parity<R, TB, SB, DB, TMA_OUT>();  // runs staged at their HBM parity
  constexpr uint32_t PADSLOT = scatter_padslot<R, TB, SB, DB, TW>();     // the stage slot of absent records
  extern __shared__ uint4 smem_raw[];
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem_raw);
  __shared__ uint32_t cnt[DG + 1], start[DG], gofs[DG], ws[(DPT == 1 ? DG : SB) / 32];  // cnt[DG]: absent records
  __shared__ uint32_t sh_t, sh_s;
  const int tid = threadIdx.x;
  const uint32_t total = ctl->tiles_total;
  const uint64_t ep = (uint64_t)epoch << 48;
  unsigned long long moved = 0;
#ifdef RADSORT_PHASE_PROF
  unsigned long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tA = 0, tB = 0;
#define RS_PROF(i) do { if (tid == 0) { tB = clock64(); pf[i] += tB - tA; tA = tB; } } while (0)
#else
#define RS_PROF(i) do { } while (0)
#endif
  // thread 0: take a ticket (the look-back forward-progress order) and find its segment
  auto take = [&]() {
    const uint32_t t = atomicAdd(&ctl->scatter_ticket, 1u);
    sh_t = t;
    sh_s = t < total ? (tile_seg ? __ldg(tile_seg + t) : seg_of_tile(tile_start, nseg, t)) : 0u;
  };
  Rec<R> r[I];
  // reduce-then-scan offsets of the loaded tile (PRE), loaded with its records
  // and summed only when the tile is processed, so no warp waits on them
  uint32_t q_tp[DPT] = {}, q_sb[DPT] = {}, q_cf = 0, q_ci[DPT] = {};
  const bool has_dg = tid * DPT < DG;  // this thread owns digits tid * DPT ..
  const uint32_t per = PRE ? (total + hist_grid - 1) / hist_grid : 1u;
  // issue this tile's loads into r[] (software pipelining: the loads of tile
  // k+1 are in flight while tile k is looked back and written out)
  auto load = [&](uint32_t t, uint32_t s) {
    const Seg sg = segs[s];
    if (sg.mode != MODE_SCATTER && sg.mode != MODE_SPLIT) return;  // split tiles: a cache-warming prefetch
    if constexpr (PRE && R >= 16) {  // (R = 8 measured 0.5 % slower: registers)
      if (sg.mode == MODE_SCATTER && has_dg) {
        const uint32_t ch = t / per;
        q_cf = __ldg(ch_first + ch);
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
          const uint32_t v = (uint32_t)(tid * DPT + j);
          q_tp[j] = __ldg(tile_pre + (size_t)t * DG + v);
          q_sb[j] = __ldg(segbase + (size_t)s * DG + v);
          q_ci[j] = __ldg(carry_in + (size_t)ch * DG + v);
        }
      }
    }
    const uint32_t lt = t - tile_start[s];
    const uint32_t m = min(T, sg.len - lt * T);
    const uint8_t* src = buf_of(sg.src, recs, tmp) + (size_t)(sg.off + lt * T) * R;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t idx = (uint32_t)(i * SB + tid);
      if (idx < m) r[i] = ldg_rec<R>(src + (size_t)idx * R);
    }
  };
  if (tid == 0) take();
#pragma unroll
  for (int j = 0; j < DPT; ++j)
    if (tid * DPT + j < DG) cnt[tid * DPT + j] = 0;
  __syncthreads();
  uint32_t t = sh_t, s = sh_s;
  if (t < total) load(t, s);
  while (t < total) {
#ifdef RADSORT_PHASE_PROF
    if (tid == 0) { tA = clock64(); pf[7]++; }
#endif
    const Seg sg = segs[s];
    const uint32_t lt = t - tile_start[s];
    const uint32_t base = sg.off + lt * T;
    const uint32_t m = min(T, sg.len - lt * T);
    // PEER (multi-GPU fused exchange): segment s is written into the buffer at
    // seg_dst[s] -- another GPU's records, mapped over NVLink -- and segbase
    // holds record offsets in that buffer
    uint8_t* dst = PEER ? reinterpret_cast<uint8_t*>(__ldg(seg_dst + s))
                        : buf_of(sg.src == SRC_TMP ? SRC_REC : SRC_TMP, recs, tmp);
    if (sg.mode == MODE_SCATTER) {
      const uint32_t d = sg.depth;
      uint32_t pre_excl[DPT] = {};
      if constexpr (PRE) {  // reduce-then-scan offsets (k_hist_pre / k_carry) + bin base, loaded with the tile
        if constexpr (R >= 16) {
          if (has_dg) {
#pragma unroll
            for (int j = 0; j < DPT; ++j) pre_excl[j] = q_tp[j] + q_sb[j] + (s == q_cf ? q_ci[j] : 0u);
          }
        } else if (has_dg) {
          const uint32_t ch = t / per;
          const bool first = s == __ldg(ch_first + ch);
#pragma unroll
          for (int j = 0; j < DPT; ++j) {
            const uint32_t v = (uint32_t)(tid * DPT + j);
            pre_excl[j] = __ldg(tile_pre + (size_t)t * DG + v) + __ldg(segbase + (size_t)s * DG + v) +
                          (first ? __ldg(carry_in + (size_t)ch * DG + v) : 0u);
          }
        }
      }
      uint32_t rk[(I + 1) / 2];  // ranks < T <= 2^16: two per register (fewer live registers under the cap)
#pragma unroll
      for (int i = 0; i < (I + 1) / 2; ++i) rk[i] = 0;
      // branch-free: an absent record (ragged last tile) counts in cnt[DG]
      // and is staged in the pad slot T (no divergent branches around the atomics)
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const uint32_t idx = (uint32_t)(i * SB + tid);
        const uint32_t dg = idx < m ? digit_w<DB>(key_of<R, K>(r[i]), d) : (uint32_t)DG;
        rk[i >> 1] |= atomicAdd(&cnt[dg], 1u) << (16 * (i & 1));
      }
      __syncthreads();
      RS_PROF(1);
      uint32_t c[DPT] = {};
      unsigned long long* my = status + (size_t)t * DG + tid;
      if (has_dg) {
#pragma unroll
        for (int j = 0; j < DPT; ++j) c[j] = cnt[tid * DPT + j];
        if constexpr (!PRE) st_relaxed(my, ep | (lt == 0 ? ST_PREFIX : ST_AGG) | c[0]);
      }
      if (tid == 0) take();  // next ticket, ready before the stage barrier
      uint32_t ex[DPT];
      if constexpr (DPT == 1) {
        ex[0] = block_excl_scan<DG>(c[0], ws);
      } else {
        ex[0] = block_excl_scan<SB>(c[0] + c[1], ws);
        ex[1] = ex[0] + c[0];
      }
      if constexpr (TWP) {  // stage slot of the run = ex + digit + parity fix (<= 1): same parity as its HBM slot
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
          const uint32_t e = ex[j] + (uint32_t)(tid * DPT + j);
          ex[j] = e + ((e ^ pre_excl[j]) & 1u);
        }
      }
      if (has_dg) {
#pragma unroll
        for (int j = 0; j < DPT; ++j) start[tid * DPT + j] = ex[j];
      }
      if constexpr (TW) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the stage is free
      __syncthreads();
      RS_PROF(2);
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const uint32_t idx = (uint32_t)(i * SB + tid);
        const uint32_t pos = start[digit_w<DB>(key_of<R, K>(r[i]), d)] + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu);
        st_rec<R>(stage + (size_t)(idx < m ? pos : PADSLOT) * R, r[i]);
      }
      if constexpr (TW) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staged -> visible to TMA
      __syncthreads();  // r[] free, sh_t/sh_s hold the next ticket
      const uint32_t tn = sh_t, sn = sh_s;
#pragma unroll
      for (int j = 0; j < DPT; ++j)
        if (tid * DPT + j < DG) cnt[tid * DPT + j] = 0;
      if (tn < total) load(tn, sn);
      RS_PROF(3);
      if constexpr (TW) {
        if (has_dg) {
          bool any = false;
#pragma unroll
          for (int j = 0; j < DPT; ++j) {
            uint32_t cc = c[j], sp = ex[j], g = pre_excl[j];
            if constexpr (TWP) {  // odd head / tail records: plain stores (16-byte bulk alignment)
              if (cc && (g & 1u)) {
                st_rec<R>(dst + (size_t)g * R, ld_rec<R>(stage + (size_t)sp * R));
                ++g; ++sp; --cc;
              }
              if (cc & 1u) {
                --cc;
                st_rec<R>(dst + (size_t)(g + cc) * R, ld_rec<R>(stage + (size_t)(sp + cc) * R));
              }
            }
            if (cc) {
              const uint32_t sa = (uint32_t)__cvta_generic_to_shared(stage + (size_t)sp * R);
              uint8_t* ga = dst + (size_t)g * R;
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(ga), "r"(sa),
                           "r"(cc * (uint32_t)R)
                           : "memory");
              any = true;
            }
          }
          if (any) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else if constexpr (DPT == 2) {
#pragma unroll
        for (int j = 0; j < DPT; ++j) gofs[tid * DPT + j] = pre_excl[j] - ex[j];
      } else if (has_dg) {
        uint64_t excl = 0;
        if constexpr (PRE) {
          excl = pre_excl[0];  // includes the bin base
        } else if (lt > 0) {
          // windowed decoupled look-back over this segment's earlier tiles
          uint32_t p = t - 1;
          for (;;) {
            unsigned long long w[LBW];
#pragma unroll
            for (int j = 0; j < LBW; ++j)
              w[j] = (p >= (uint32_t)j) ? ld_relaxed(status + (size_t)(p - j) * DG + tid) : 0ull;
            int j = 0;
            bool done = false;
#pragma unroll
            for (int q = 0; q < LBW; ++q) {
              if (done || j != q) continue;
              if ((w[q] & ~((1ull << 48) - 1)) != ep) continue;  // not yet published: reload from here
              excl += w[q] & ST_VAL;
              if (w[q] & ST_PREFIX) done = true;
              else j = q + 1;
            }
            if (done) break;
            p -= (uint32_t)j;
#ifdef RADSORT_PHASE_PROF
            if (tid == 0) pf[6]++;
#endif
          }
          st_relaxed(my, ep | ST_PREFIX | (excl + c[0]));
        }
        gofs[tid] = (PRE ? 0u : segbase[(size_t)s * DG + tid]) + (uint32_t)excl - ex[0];
      }
      if constexpr (!TW) __syncthreads();
      RS_PROF(4);
      if constexpr (TW) {
      } else if constexpr (R == 32) {
        // a lane pair moves one record, 16 bytes each: consecutive 16-byte smem
        // reads (a lane per 32-byte record conflicts 2-way on every read); the
        // key sits in the first half, its digit is passed to the partner lane
        const int lane = tid & 31;
        for (uint32_t h0 = 0; h0 < 2 * m; h0 += SB) {
          const uint32_t h = h0 + (uint32_t)tid;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (h < 2 * m) v = reinterpret_cast<const uint4*>(stage)[h];
          Rec<16> hr;
          hr.a = v;
          uint32_t dg = digit_w<DB>(key_of<16, K>(hr), d);
          dg = __shfl_sync(0xffffffffu, dg, lane & ~1);
          if (h < 2 * m) reinterpret_cast<uint4*>(dst + (size_t)(gofs[dg] + (h >> 1)) * R)[h & 1u] = v;
        }
      } else {
        for (uint32_t q = tid; q < m; q += SB) {
          const Rec<R> x = ld_rec<R>(stage + (size_t)q * R);
          st_rec<R>(dst + (size_t)(gofs[digit_w<DB>(key_of<R, K>(x), d)] + q) * R, x);
        }
      }
      moved += m;
      t = tn;
      s = sn;
    } else if (sg.mode == MODE_SPLIT) {
      // three-way split around the segment's dominant key (k_plan): class
      // 0/1/2 = key below / equal to / above it.  Ranks by warp ballots; each
      // class's range is reserved per tile with one atomic (order inside a
      // class is free, R2); each warp stores its records of a class
      // as one contiguous run, straight from registers.  The equal class is
      // final: written to `records` (segment in tmp), or skipped and filled
      // later (segment in `records`, R == K).
      if (tid == 0) take();  // next ticket (ordered before the barriers inside)
      if constexpr (TW) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
      }
      split_tile<R, K, SB, DG>(sg, s, base, m, dst, recs, tmp, segbase, splitc, stage, cnt, gofs);
      __syncthreads();  // sh_t/sh_s hold the next ticket; cnt / gofs / stage reusable
      const uint32_t tn = sh_t, sn = sh_s;
#pragma unroll
      for (int j = 0; j < DPT; ++j)
        if (tid * DPT + j < DG) cnt[tid * DPT + j] = 0;
      if (tn < total) load(tn, sn);
      moved += m;
      t = tn;
      s = sn;
    } else {
      if (sg.mode == MODE_COPY) {
        const uint8_t* src = buf_of(sg.src, recs, tmp);
        for (uint32_t i = tid; i < m; i += SB)
          st_rec<R>(dst + (size_t)(base + i) * R, ldg_rec<R>(src + (size_t)(base + i) * R));
        moved += m;
      } else if (sg.mode == MODE_FILL) {  // write-only: every record of the bin is its (dominant) key
        if constexpr (R == K) {
          Key<K> kf;
          kf.w0 = probes[(size_t)sg.aux * 2];
          if constexpr (K == 16) kf.w1 = probes[(size_t)sg.aux * 2 + 1];
          const Rec<R> x = rec_of_key<R, K>(kf);
          for (uint32_t i = tid; i < m; i += SB) st_rec<R>(recs + (size_t)(base + i) * R, x);
          moved += m / 2;  // write-only: R bytes per record
        }
      }
      if (tid == 0) take();
      __syncthreads();
      t = sh_t;
      s = sh_s;
      if (t < total) load(t, s);
    }
    __syncthreads();  // stage / gofs / sh_* reuse
    RS_PROF(5);
  }
  if constexpr (PEER) __threadfence_system();  // peer stores performed before the kernel's completion is observed
  if constexpr (TW) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (tid == 0 && moved) atomicAdd(&ctl->rec_scatter, moved);
#ifdef RADSORT_PHASE_PROF
  if (tid == 0) {
    for (int q = 0; q < 8; ++q) atomicAdd(&ctl->prof[q], pf[q]);
  }
#endif
#undef RS_PROF
}

// -------------------------------------------------------------- k_children
// Classify the 256 child bins of every scattered segment (PAPER.md:120-121
// §3.1, §3.2): empty/singleton/all-equal ->
// final (copied to the output buffer if they sit in tmp); 2..ES_MAX records ->
// enumeration sort right here; <= TINY_MAX -> warp small-bin sorter right here
// (§3.3); <= C -> Local list; larger -> next level's Large
// list.  Dynamic smem: one TINY_MAX*R scratch per warp.
template <int R, int K, int DB = 8>
__global__ void __launch_bounds__(CHILD_B, 3) k_children(const Seg* __restrict__ segs, const uint32_t* __restrict__ hist,
                                                      const uint32_t* __restrict__ segbase, Seg* large_next,
                                                      Seg* local_cur, int cur, Ctl* ctl, uint8_t* recs, uint8_t* tmp,
                                                      unsigned long long* __restrict__ probes, uint32_t lmin,
                                                      uint32_t lcap, uint32_t bitonic_max) {
  enum : uint8_t { C_NONE = 0, C_COPY = 1, C_ES = 2, C_TINY = 3 };
  constexpr int DG = 1 << DB;  // children per segment (1024 on a wide level)
  extern __shared__ uint4 smem_raw[];
  __shared__ uint8_t cls[DG];
  __shared__ uint32_t coff[DG], clen[DG];
  __shared__ __align__(16) TailScratch<K> wsc[CHILD_B / 32];
  const uint32_t s = blockIdx.x;
  const Seg sg = segs[s];
  if (sg.mode != MODE_SCATTER && sg.mode != MODE_SPLIT) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* scratch = reinterpret_cast<uint8_t*>(smem_raw) + (size_t)warp * TINY_MAX * R;
  const uint8_t loc = sg.src == SRC_TMP ? SRC_REC : SRC_TMP;  // children live where the scatter wrote
  const bool split = sg.mode == MODE_SPLIT;  // children 0/1/2: below / equal to / above the dominant key
  const uint32_t d1 = split ? sg.depth : sg.depth + 1u;
  constexpr uint32_t C = local_capacity<R>();
  uint8_t* cbuf = buf_of(loc, recs, tmp);
  // children of a wide (10-bit) pass share the two leading bits of digit d1
  const uint8_t cflags = (DB == 10 && !split) ? (uint8_t)(2u << FLAG_SKIP_SHIFT) : (uint8_t)0;
  for (int v = tid; v < DG; v += CHILD_B) {
    const uint32_t len = hist[(size_t)s * DG + v];
    const uint32_t off = segbase[(size_t)s * DG + v];
    uint8_t c = C_NONE;
    if (len == 0) {
    } else if (split && v == 1) {  // the dominant key: final (written to records, or filled below)
      if (sg.src == SRC_REC) {
        const uint32_t pi = atomicAdd(&ctl->n_probe, 1u);
        const Key<K> pk = ld_key<R, K>(recs + (size_t)sg.off * R);  // untouched by the split scatter
        probes[(size_t)pi * 2] = pk.w0;
        if constexpr (K == 16) probes[(size_t)pi * 2 + 1] = pk.w1;
        Seg ns = {off, len, (uint8_t)K, SRC_REC, MODE_NONE, FLAG_FILL, pi};
        large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
      }
      atomicAdd(&ctl->rec_final, (unsigned long long)len);
      atomicAdd(&ctl->bins_final, 1ull);
    } else if (d1 >= (uint32_t)K || len == 1) {  // all digits consumed / singleton: final
      if (loc == SRC_TMP) {
        if (len <= C) c = C_COPY;
        else {
          Seg ns = {off, len, (uint8_t)d1, loc, MODE_NONE, FLAG_EQUAL, 0};
          large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
        }
      }
      if (len <= C || loc != SRC_TMP) {
        atomicAdd(&ctl->rec_final, (unsigned long long)len);
        atomicAdd(&ctl->bins_final, 1ull);
      }
    } else if (len <= es_max<R>()) {
      c = C_ES;
    } else if (len <= TINY_MAX) {
      c = C_TINY;
    } else if (len <= C || (len >= lmin && len <= lcap)) {  // CTA-local sort, or cluster-local sort in [lmin, lcap]
      Seg ns = {off, len, (uint8_t)d1, loc, MODE_NONE, cflags, 0};
      local_cur[atomicAdd(&ctl->n_local[cur], 1u)] = ns;
      if (len <= small_cap<R>()) atomicAdd(&ctl->n_local_small[cur], 1u);
      else if (len <= med_cap<R>()) atomicAdd(&ctl->n_local_med[cur], 1u);
      atomicMax(&ctl->max_local_len[cur], len);
      atomicAdd(&ctl->bins_local, 1ull);
    } else {
      Seg ns = {off, len, (uint8_t)d1, loc, MODE_NONE, cflags, 0};
      large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
      atomicAdd(&ctl->rec_large_next, (unsigned long long)len);
      atomicAdd(&ctl->bins_large, 1ull);
    }
    cls[v] = c;
    coff[v] = off;
    clen[v] = len;
  }
  __syncthreads();
  unsigned long long tiny_recs = 0, tiny_bins = 0;
  for (int v = warp; v < DG; v += CHILD_B / 32) {
    const uint8_t c = cls[v];
    if (c == C_NONE) continue;
    const uint32_t off = coff[v], len = clen[v];
    const uint8_t* src = cbuf + (size_t)off * R;
    uint8_t* out = recs + (size_t)off * R;
    {  // the warp's next bin into L1 while this one is sorted (one 128-byte line per lane)
      const int vn = v + CHILD_B / 32;
      if (vn < DG && (cls[vn] == C_TINY || cls[vn] == C_ES)) {
        const uint8_t* pn = cbuf + (size_t)coff[vn] * R + (size_t)lane * 128;
        if ((uint32_t)lane * 128u < clen[vn] * (uint32_t)R) asm volatile("prefetch.global.L1 [%0];" ::"l"(pn));
      }
    }
    if (c == C_COPY) {
      warp_copy<R>(src, out, len, lane);
    } else if (c == C_ES) {
      Rec<R> x;
      uint32_t rank = 0;
      if ((uint32_t)lane < len) {
        x = ld_rec<R>(src + (size_t)lane * R);
        rank = es_rank<R, K>(src, len, (uint32_t)lane, key_of<R, K>(x));
      }
      __syncwarp();
      if ((uint32_t)lane < len) st_rec<R>(out + (size_t)rank * R, x);
      tiny_recs += len;
      tiny_bins += 1;
    } else if (len <= bitonic_max && d1 >= 1u) {  // the warp bitonic network (measured faster at 17..32, R <= 16)
      warp_tiny_sort<R, K>(src, out, len, d1, lane);   // (gathers before it stores: in place is fine)
      tiny_recs += len;
      tiny_bins += 1;
    } else {
      if (src == out) {  // in place: stage the bin in the warp's smem scratch first
        warp_copy<R>(src, scratch, len, lane);
        __syncwarp();
        src = scratch;
      }
      warp_tail_sort<R, K>(src, out, len, d1, lane, wsc[warp]);
      tiny_recs += len;
      tiny_bins += 1;
    }
  }
  if (lane == 0 && tiny_bins) {
    atomicAdd(&ctl->rec_tiny, tiny_recs);
    atomicAdd(&ctl->bins_tiny, tiny_bins);
  }
}

// -------------------------------------------------------------- k_local
// CTA-local sort of bins of <= C records (the GPU analog of PAPER.md:134
// §3.2 "the bin is small enough to fit in a half of L2 ... simple counting
// and scatter", and of PAPER.md:181-183 §3.3 for what is left inside it).
//
// Per bin, with the bin's records in registers:
//  1. counting pass on a composite digit of W bits -- digit d followed by the
//     leading W-8 bits of digit d+1 (W = ceil(log2(bin)) + 1, 10..16; DESIGN.md §4:
//     one smem counting pass doing the work of up to two MSD levels) -- u16
//     counters, two per word, ranks from smem atomics;
//     The record that finds one earlier record in its bucket lists the bucket
//     (a dense list of the buckets holding >= 2 records).  A bucket holding
//     the whole bin means constant leading digits: the AND/OR of the keys
//     picks the first non-constant digit and the pass is redone
//     there, or the bin is final when all keys are equal;
//  2. exclusive scan of the counters (warp-cooperative, 16-byte accesses);
//  3. every record is stored to smem at its bucket position, and the next
//     bin's loads are issued right away (registers are free again);
//  4. one thread per listed bucket of 2..ES_MAX records sorts it in place in
//     smem (insertion sort on the full key, PAPER.md:94 / PAPER.md:177: the
//     fix-up sorter for a handful of records); a larger bucket is checked by a
//     warp for holding a single key (final as staged);
//  5. the staged bin is written out with coalesced stores;
//  6. larger buckets holding several keys (only duplicated or skewed keys
//     produce them): <= TINY_MAX records by the warp tail sorter, larger ones
//     are queued as Local bins of the next level.
constexpr uint32_t LOCAL_WMIN = 10;  // narrowest composite digit: 2^(W-1) >= 512 counter words

// Bucket of a key at depth d (< K): the top W bits of the key bits below its
// d leading digits (zero bits past the end of the key).
__device__ __forceinline__ uint32_t bucket_of(const Key<8>& k, uint32_t d, uint32_t W) {
  return (uint32_t)((k.w0 << (8u * d)) >> (64u - W));
}
__device__ __forceinline__ uint32_t bucket_of(const Key<16>& k, uint32_t d, uint32_t W) {
  const uint32_t s = 8u * d;
  uint64_t x;
  if (s == 0) x = k.w1;
  else if (s < 64) x = (k.w1 << s) | (k.w0 >> (64u - s));
  else x = k.w0 << (s - 64u);
  return (uint32_t)(x >> (64u - W));
}

__host__ __device__ __forceinline__ uint32_t local_width(uint32_t n, uint32_t wmax) {
  // ceil(log2 n) + 1: about half a record per bucket (measured best)
#ifdef __CUDA_ARCH__
  const uint32_t w = (n > 1 ? 32u - (uint32_t)__clz((int)(n - 1)) : 1u) + 1u;
#else
  uint32_t w = 1;
  while ((1u << w) < n) ++w;
  ++w;
#endif
  return w < LOCAL_WMIN ? LOCAL_WMIN : (w > wmax ? wmax : w);
}

// In-place exclusive scan of the 2^W u16 bucket counters (two per word): one
// contiguous chunk per warp, 16-byte accesses, the two halves of a word summed
// as one 32-bit add (no half overflows: every count and sum is <= n <= 2^14).
// Contains one block barrier; the caller synchronises after it.
// U = 2: two 32-uint4 blocks per step with interleaved shuffle scans (more ILP,
// more live registers: measured a win for k_local_pipe on R = 8 only)
template <int LB, int U = 1>
__device__ __forceinline__ void local_scan(uint32_t* cnt, uint32_t W, uint32_t* wsum) {
  static_assert(U == 1 || U == 2, "one or two blocks per step");
  constexpr int NW = LB / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t pw = (1u << (W - 1)) / NW;  // words per warp, a multiple of 4
  const uint32_t n4 = pw / 4;
  uint4* c4 = reinterpret_cast<uint4*>(cnt + (size_t)warp * pw);
  uint32_t tot = 0;
  for (uint32_t j = lane; j < n4; j += 32) {
    const uint4 v = c4[j];
    tot += v.x + v.y + v.z + v.w;
  }
  tot = __reduce_add_sync(0xffffffffu, (tot & 0xffffu) + (tot >> 16));
  if (lane == 0) wsum[warp] = tot;
  __syncthreads();
  // carry-in of this warp's chunk: exclusive prefix of the warp totals (lane w holds warp w's)
  uint32_t carry = (lane < NW && lane < warp) ? wsum[lane] : 0u;
  carry = __reduce_add_sync(0xffffffffu, carry);
  for (uint32_t j0 = 0; j0 < n4; j0 += 32 * U) {
    uint4 v[U];
    uint32_t t[U], inc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + 32u * u + lane;
      v[u] = j < n4 ? c4[j] : make_uint4(0, 0, 0, 0);
      const uint32_t p = v[u].x + v[u].y + v[u].z + v[u].w;
      t[u] = (p & 0xffffu) + (p >> 16);
      inc[u] = t[u];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc[u], o);
        if (lane >= o) inc[u] += y;
      }
    }
    const uint32_t tot0 = __shfl_sync(0xffffffffu, inc[0], 31);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + 32u * u + lane;
      // word start (both halves) = s | s << 16, then + (lo << 16) for the high half
      uint32_t s = carry + (u ? tot0 : 0u) + inc[u] - t[u];
      uint4 o4;
      o4.x = s * 0x10001u + (v[u].x << 16); s += (v[u].x & 0xffffu) + (v[u].x >> 16);
      o4.y = s * 0x10001u + (v[u].y << 16); s += (v[u].y & 0xffffu) + (v[u].y >> 16);
      o4.z = s * 0x10001u + (v[u].z << 16); s += (v[u].z & 0xffffu) + (v[u].z >> 16);
      o4.w = s * 0x10001u + (v[u].w << 16);
      if (j < n4) c4[j] = o4;
    }
    carry += tot0 + (U > 1 ? __shfl_sync(0xffffffffu, inc[U - 1], 31) : 0u);
  }
}

// Steps 4-6 of the CTA-local sort, for a bin staged in smem in bucket order
// (see k_local).  All threads of the CTA call it (it contains barriers).
// Returns true when the tail sorter used the counter region as scratch.
template <int R, int K, int LB, int NTW, bool PV = true, bool QT = false>
__device__ __forceinline__ bool local_finish(uint8_t* stage, const uint16_t* start16, uint32_t* blist, uint32_t cap,
                                             uint32_t n, uint32_t nbk, uint32_t d, uint32_t W, uint32_t ncol,
                                             uint32_t* s_nbig, TailScratch<K>* tsc, uint8_t* out, uint32_t off,
                                             Seg* local_next, int nxt, Ctl* ctl, bool bulk = false,
                                             unsigned long long* pfx = nullptr, int nd_force = -1,
                                             uint8_t src_big = SRC_REC) {
  constexpr int NW = LB / 32;
  constexpr uint32_t ES = es_max<R>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto start_of = [&](uint32_t b) { return (uint32_t)start16[b]; };
#ifdef RADSORT_PHASE_PROF
  unsigned long long fA = clock64();
#define RS_FPROF(i) do { if (pfx && tid == 0) { const unsigned long long fB = clock64(); pfx[i] += fB - fA; fA = fB; } } while (0)
#else
#define RS_FPROF(i) do { } while (0)
#endif
  uint32_t nbig = 0;
  if (ncol) {
    for (uint32_t e = tid; e < ncol; e += LB) {
      const uint32_t b = blist[e];
      const uint32_t s0 = start_of(b), c = (b + 1 < nbk ? start_of(b + 1) : n) - s0;
      uint8_t* base = stage + (size_t)s0 * R;
      if (c == 2) {  // a pair: one compare-exchange
        const Rec<R> x = ld_rec<R>(base), y = ld_rec<R>(base + R);
        if (key_lt(key_of<R, K>(y), key_of<R, K>(x))) { st_rec<R>(base, y); st_rec<R>(base + R, x); }
      } else if (c <= ES) {  // 3..ES records: insertion sort in place
        lane_insertion_sort<R, K>(base, c);
      } else {  // more: listed from the top as {start | count << 16}
        blist[cap - 1u - atomicAdd(s_nbig, 1u)] = s0 | (c << 16);
      }
    }
    __syncthreads();
    RS_FPROF(0);
    nbig = *s_nbig;
    for (uint32_t e = warp; e < nbig; e += NW) {  // > ES records: one key or several?
      const uint32_t en = blist[cap - 1u - e];
      const uint32_t s0 = en & 0xffffu, c = en >> 16;
      const Key<K> k0 = ld_key<R, K>(stage + (size_t)s0 * R);
      bool diff = false;
      for (uint32_t j = s0 + lane; j < s0 + c; j += 32) diff |= !key_eq(ld_key<R, K>(stage + (size_t)j * R), k0);
      if (__any_sync(0xffffffffu, diff) && lane == 0) blist[cap - 1u - e] = en | 0x80000000u;
    }
    if (nbig) __syncthreads();
  }
  RS_FPROF(1);
  if (bulk) {
    // one TMA bulk store of the 16-byte-aligned middle of the bin (stage and out
    // agree mod 16: the caller shifts the stage); the head / tail words by threads;
    // the caller waits for the bulk read before reusing the stage
    const uintptr_t o0 = (uintptr_t)out, o1 = o0 + (size_t)n * R;
    const uintptr_t a0 = (o0 + 15) & ~(uintptr_t)15, a1 = o1 & ~(uintptr_t)15;
    if (a1 > a0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(stage + (a0 - o0));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a0), "r"(sa),
                     "r"((uint32_t)(a1 - a0))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      // 8-byte words outside [a0, a1): at most one before and one after
      if (tid < 2) {
        const uintptr_t w = tid == 0 ? o0 : a1;
        if ((tid == 0 && a0 > o0) || (tid == 1 && o1 > a1))
          *reinterpret_cast<uint2*>(w) = *reinterpret_cast<const uint2*>(stage + (w - o0));
      }
    } else {  // shorter than one aligned 16-byte chunk
      for (uint32_t q = tid; q < n * (uint32_t)R / 8u; q += LB)
        reinterpret_cast<uint2*>(out)[q] = reinterpret_cast<const uint2*>(stage)[q];
    }
  } else {
    for (uint32_t q = tid; q < n; q += LB) st_rec<R>(out + (size_t)q * R, ld_rec<R>(stage + (size_t)q * R));
  }
#ifdef RADSORT_PHASE_PROF
  __syncthreads();
#endif
  RS_FPROF(2);
#undef RS_FPROF
  if (!nbig) return false;
  if (bulk && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // tails overwrite their part
  __syncthreads();  // written out; counters dead: the tail sorter's scratch aliases them
  // digits shared by a bucket's keys (nd_force: the caller's bucket does not start at a digit boundary)
  const uint32_t nd = nd_force >= 0 ? (uint32_t)nd_force : d + (W >= 16 ? 2u : 1u);
  for (uint32_t e = warp; e < nbig && warp < NTW; e += NTW) {
    const uint32_t en = blist[cap - 1u - e];
    if (!(en >> 31)) continue;
    const uint32_t s0 = en & 0xffffu, c = (en >> 16) & 0x7fffu;
    if (!QT && c <= TINY_MAX) {
      warp_tail_sort<R, K, PV>(stage + (size_t)s0 * R, out + (size_t)s0 * R, c, nd, lane, tsc[warp]);
    } else if (lane == 0) {  // (QT: every mixed bucket; the caller's counters are live)
      Seg ns = {off + s0, c, (uint8_t)nd, src_big, MODE_NONE, 0, 0};
      local_next[atomicAdd(&ctl->n_local[nxt], 1u)] = ns;
      atomicMax(&ctl->max_local_len[nxt], c);
      if (c <= small_cap<R>()) atomicAdd(&ctl->n_local_small[nxt], 1u);
      else if (c <= med_cap<R>()) atomicAdd(&ctl->n_local_med[nxt], 1u);
    }
  }
#ifdef RADSORT_PHASE_PROF
  if (pfx && tid == 0) pfx[3] += clock64() - fA;
#endif
  return true;
}

template <int R, int K, int IL, int LB>
__global__ void __launch_bounds__(LB, LB <= 64 ? 8 : (LB <= 256 ? 2 : 1))
    k_local(const Seg* __restrict__ list, uint32_t nlist, uint32_t wmax, uint32_t stage_bytes, uint32_t cnt_bytes,
            uint32_t cap, Seg* local_next, int nxt, Ctl* ctl, uint8_t* recs, uint8_t* tmp, uint32_t lmin,
            uint32_t lmax) {
  extern __shared__ uint4 smem_raw[];
  constexpr int KW = K / 8;
  constexpr int NW = LB / 32;
  constexpr uint32_t ES = es_max<R>();
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem_raw);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(stage + stage_bytes);                 // 2^W u16 counters
  uint32_t* blist = reinterpret_cast<uint32_t*>(stage + stage_bytes + cnt_bytes);   // buckets of >= 2 records
  __shared__ uint32_t wsum[NW], s_ncol, s_nbig, s_const;
  __shared__ unsigned long long sna[2], so[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t C = local_capacity<R>();  // larger bins of the list belong to k_local_cluster
  uint32_t bi = blockIdx.x;
  auto skip = [&](uint32_t b) {  // bins of another launch: other size class, or k_local_cluster's (> C)
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
      if (i * LB < lim) r[i] = ldg_rec<R>(p + (size_t)i * LB * R);
  };
  auto prefetch_l2 = [&](uint32_t b) {  // TMA bulk prefetch of a whole bin into L2
    if (tid == 0 && b < nlist) {
      const Seg g = list[b];
      const uintptr_t s0 = (uintptr_t)(buf_of(g.src, recs, tmp) + (size_t)g.off * R);
      const uintptr_t e0 = s0 + (size_t)g.len * R;
      const uintptr_t s1 = (s0 + 15) & ~(uintptr_t)15, e1 = e0 & ~(uintptr_t)15;
      if (e1 > s1)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s1), "r"((uint32_t)(e1 - s1)) : "memory");
    }
  };
  Seg sg = list[bi];
  load(sg);
  prefetch_l2(bi + gridDim.x);
  zero_cnt(cnt_bytes);
  if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  if (tid == 0) { s_ncol = 0; s_nbig = 0; s_const = 0; }
  unsigned long long done = 0;
  bool pending = false;  // the previous bin's bulk store may still read the stage
#ifdef RADSORT_PHASE_PROF
  unsigned long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tA = clock64(), tB = 0;
#define RS_PROF(i) do { if (tid == 0) { tB = clock64(); pf[i] += tB - tA; tA = tB; } } while (0)
#else
#define RS_PROF(i) do { } while (0)
#endif
  constexpr int IP = (IL + 1) / 2;  // ranks < 2^16: two per register
#ifdef RADSORT_PHASE_PROF
  unsigned long long pfl[4] = {0, 0, 0, 0};
#endif
  for (;;) {
    const uint32_t n = sg.len;
    const int lim = (int)n - tid;
    uint8_t* out = recs + (size_t)sg.off * R;
    // 512-thread CTAs (one bin per SM): the bin is staged at the same alignment
    // mod 16 as its output, so the write-out is one TMA bulk store (plus at most
    // two 8-byte words) that overlaps the next bin's count and scan (c5 local
    // 7.52 -> 7.08 ms; with several bins per SM the thread stores are faster:
    // c2 1.82 vs 1.86, kmc 12.9 vs 14.3 ms)
    constexpr bool BULK = LB >= 512;
    uint8_t* stg = BULK ? stage + ((uintptr_t)out & 15u) : stage;
    // key bits the bin's records already share (digits, plus 2 bits below a wide level)
    uint32_t sb = 8u * sg.depth + seg_skip(sg.flags);
    const uint32_t W = local_width(n, wmax);
    const uint32_t nbk = 1u << W;
    uint32_t rk[IP];
    uint32_t ones = 0;
    bool all_equal = false;
    __syncthreads();  // counters zero, flags reset
    if (tid == 0) {  // the next bins' descriptors into L1 (read after staging / for the L2 prefetch)
      const uint32_t p1 = bi + gridDim.x, p2 = p1 + gridDim.x;
      if (p1 < nlist) asm volatile("prefetch.global.L1 [%0];" ::"l"(list + p1));
      if (p2 < nlist) asm volatile("prefetch.global.L1 [%0];" ::"l"(list + p2));
    }
    RS_PROF(7);
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
          ones += (uint32_t)(old == 1u);  // the second record of a bucket will list it
          cst |= old == n - 1u;           // the whole bin in one bucket
        }
      }
      if (cst) s_const = 1u;
      __syncthreads();
      RS_PROF(0);
      if (!s_const) {
        local_scan<LB>(cnt, W, wsum);
        if (pending && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        pending = false;
        __syncthreads();  // starts in place; the stage is free
        RS_PROF(1);
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
    const uint16_t* start16 = reinterpret_cast<const uint16_t*>(cnt);
    auto start_of = [&](uint32_t b) { return (uint32_t)start16[b]; };
    if (all_equal) {  // final where it is (copied out of tmp)
      if (sg.src == SRC_TMP) {
#pragma unroll
        for (int i = 0; i < IL; ++i)
          if (i * LB < lim) st_rec<R>(out + (size_t)(i * LB + tid) * R, r[i]);
      }
    } else {
      // slots in the list of buckets holding >= 2 records: warp scan + one atomic per warp
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
      for (int i = 0; i < IL; ++i) {
        if (i * LB < lim) {
          const uint32_t b = key_bits(key_of<R, K>(r[i]), sb, W);
          const uint32_t rnk = (rk[i >> 1] >> (16 * (i & 1))) & 0xffffu;
          st_rec<R>(stg + (size_t)(start_of(b) + rnk) * R, r[i]);
          if (rnk == 1u) blist[slot++] = b;
        }
      }
    }
    // registers are free: the next bin's loads overlap this bin's write-out;
    // the bin after next streams into L2
    uint32_t nb = bi + gridDim.x;
    while (nb < nlist && skip(nb)) nb += gridDim.x;
    Seg nsg = sg;
    if (nb < nlist) {
      nsg = list[nb];
      load(nsg);
    }
    prefetch_l2(nb + gridDim.x);
    bool tail = false;
    if (!all_equal) {
      const bool fix = 8u * K > sb + W;  // key bits left below the composite digit
      RS_PROF(2);
      __syncthreads();  // staged
      RS_PROF(3);
      // the tail sorter's pivot path only in the small-bin configuration (duplicate-heavy
      // streams of small bins live there; the big-bin ones are short of registers)
      tail = local_finish<R, K, LB, NW, LB == 64>(stg, start16, blist, cap, n, nbk, sb / 8u, W, fix ? s_ncol : 0u, &s_nbig,
                                       reinterpret_cast<TailScratch<K>*>(cnt), out, sg.off, local_next, nxt, ctl, BULK,
#ifdef RADSORT_PHASE_PROF
                                       pfl,
#else
                                       nullptr,
#endif
                                       (int)((sb + W) / 8u));
      pending = BULK;
    }
    done += n;
    __syncthreads();
    RS_PROF(5);
    zero_cnt(tail ? cnt_bytes : (2u << W));
    if (tid == 0) { s_ncol = 0; s_nbig = 0; s_const = 0; }
    if (nb >= nlist) break;
    bi = nb;
    sg = nsg;
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (tid == 0) atomicAdd(&ctl->rec_local, done);
#ifdef RADSORT_PHASE_PROF
  if (tid == 0) {
    for (int q = 0; q < 8; ++q) atomicAdd(&ctl->prof[8 + q], pf[q]);
    atomicAdd(&ctl->prof[0], pfl[0]);
    atomicAdd(&ctl->prof[6], pfl[1]);
    atomicAdd(&ctl->prof[7], pfl[2]);
    atomicAdd(&ctl->prof[12], pfl[3]);
  }
#endif
#undef RS_PROF
}

// L2-coherent loads (.cg: the SM's L1 may hold lines of the bin read before
// the cluster's other CTAs wrote them)

template <int R, int K>
__device__ __forceinline__ void cswap_rec(Rec<R>& a, Rec<R>& b) {
  if (key_lt(key_of<R, K>(b), key_of<R, K>(a))) { const Rec<R> t = a; a = b; b = t; }
}

// Fix-up of the colliding buckets of a slice written straight to global memory
// by the direct-write cluster sort (k_local_cluster<.., DW = true>): the
// records of a bucket sit in [start, start + c) in arbitrary order.  Buckets of
// 2..4 records are loaded whole (independent L2 loads), sorted by a
// compare-exchange network and written back (§2.2 sorting
// networks for the tiniest arrays); 5..ES by insertion sort in place
// (the fix-up sorter); larger buckets holding several keys
// become Local bins of the next level.  Every thread of the CTA calls it.
template <int R, int K, int LB>
__device__ __forceinline__ void global_fixup(uint8_t* out, const uint16_t* start16, uint32_t* blist, uint32_t n,
                                             uint32_t nbk, uint32_t d, uint32_t W, uint32_t ncol, uint32_t* s_nbig,
                                             uint32_t off, Seg* local_next, int nxt, Ctl* ctl) {
  constexpr uint32_t ES = es_max<R>();
  constexpr int NW = LB / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!ncol) return;
  for (uint32_t e = tid; e < ncol; e += LB) {
    const uint32_t b = blist[e];
    const uint32_t s0 = start16[b], c = (b + 1 < nbk ? (uint32_t)start16[b + 1] : n) - s0;
    uint8_t* base = out + (size_t)s0 * R;
    if (c <= 4) {
      Rec<R> x0 = ldcg_rec<R>(base), x1 = ldcg_rec<R>(base + R), x2, x3;
      if (c > 2) x2 = ldcg_rec<R>(base + 2 * R);
      if (c > 3) x3 = ldcg_rec<R>(base + 3 * R);
      if (c == 2) {
        if (key_lt(key_of<R, K>(x1), key_of<R, K>(x0))) { stg_rec<R>(base, x1); stg_rec<R>(base + R, x0); }
      } else if (c == 3) {
        cswap_rec<R, K>(x0, x1); cswap_rec<R, K>(x1, x2); cswap_rec<R, K>(x0, x1);
        stg_rec<R>(base, x0); stg_rec<R>(base + R, x1); stg_rec<R>(base + 2 * R, x2);
      } else {
        cswap_rec<R, K>(x0, x1); cswap_rec<R, K>(x2, x3); cswap_rec<R, K>(x0, x2); cswap_rec<R, K>(x1, x3);
        cswap_rec<R, K>(x1, x2);
        stg_rec<R>(base, x0); stg_rec<R>(base + R, x1); stg_rec<R>(base + 2 * R, x2); stg_rec<R>(base + 3 * R, x3);
      }
    } else if (c <= ES) {
      for (uint32_t i = 1; i < c; ++i) {
        const Rec<R> x = ldcg_rec<R>(base + (size_t)i * R);
        const Key<K> kx = key_of<R, K>(x);
        int j = (int)i - 1;
        for (; j >= 0; --j) {
          const Rec<R> y = ldcg_rec<R>(base + (size_t)j * R);
          if (!key_lt(kx, key_of<R, K>(y))) break;
          stg_rec<R>(base + (size_t)(j + 1) * R, y);
        }
        stg_rec<R>(base + (size_t)(j + 1) * R, x);
      }
    } else {
      blist[e] = s0 | (c << 16) | 0x80000000u;  // > ES: checked below
      atomicAdd(s_nbig, 1u);
    }
  }
  __syncthreads();
  if (!*s_nbig) return;
  // > ES records: one warp per bucket checks for a single key (final as it is,
  // PAPER.md:38); several keys -> a Local bin of the next level
  for (uint32_t e = warp; e < ncol; e += NW) {
    const uint32_t en = blist[e];
    if (!(en >> 31)) continue;
    const uint32_t s0 = en & 0xffffu, c = (en >> 16) & 0x7fffu;
    const Key<K> k0 = key_of<R, K>(ldcg_rec<R>(out + (size_t)s0 * R));
    bool diff = false;
    for (uint32_t j = s0 + lane; j < s0 + c; j += 32) diff |= !key_eq(key_of<R, K>(ldcg_rec<R>(out + (size_t)j * R)), k0);
    if (__any_sync(0xffffffffu, diff) && lane == 0) {
      const uint32_t nd = d + (W >= 16 ? 2u : 1u);
      Seg ns = {off + s0, c, (uint8_t)nd, SRC_REC, MODE_NONE, 0, 0};
      local_next[atomicAdd(&ctl->n_local[nxt], 1u)] = ns;
      atomicMax(&ctl->max_local_len[nxt], c);
      if (c <= small_cap<R>()) atomicAdd(&ctl->n_local_small[nxt], 1u);
      else if (c <= med_cap<R>()) atomicAdd(&ctl->n_local_med[nxt], 1u);
    }
  }
}

// -------------------------------------------------------------- k_local_big
// The CTA-local sort (k_local's steps 1-6) for the largest local bins (up to C
// records, one bin per SM: its staging takes most of the shared memory),
// written for occupancy: 1024 threads (32 warps to hide the latency of the
// barrier-separated phases) with IL <= 16 records each, and no per-record
// state kept between the phases besides the records themselves:
//  1. count: one smem atomic per record on the composite-digit bucket; the
//     record that finds one earlier record in its bucket lists it (buckets of
//     >= 2 records are the only ones the fix-up visits);
//  2. exclusive scan of the counters;
//  3. stage: a second atomic per record on the scanned starts gives its slot
//     (order inside a bucket is free: the fix-up sorts every bucket of >= 2
//     records by full key); afterwards counter b holds the END of bucket b,
//     i.e. the start of bucket b + 1, so bucket b spans [E[b-1], E[b]) with
//     E[-1] = 0 (a zero word in front of the counters);
//  4.-6. as k_local (local_finish): fix-up, one TMA bulk store of the bin,
//     mixed buckets of > ES records queued as Local bins of the next level.
// The whole bin landing in one bucket (constant leading digits) is checked
// once per bin (the bucket of record 0 holding n records), not per record.
template <int R, int K, int IL, int LB>
__global__ void __launch_bounds__(LB, 1)
    k_local_big(const Seg* __restrict__ list, uint32_t nlist, uint32_t wmax, uint32_t stage_bytes, uint32_t cnt_bytes,
                uint32_t cap, Seg* local_next, int nxt, Ctl* ctl, uint8_t* recs, uint8_t* tmp, uint32_t lmin,
                uint32_t lmax) {
  extern __shared__ uint4 smem_raw[];
  constexpr int KW = K / 8;
  constexpr int NW = LB / 32;
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem_raw);
  uint32_t* zpad = reinterpret_cast<uint32_t*>(stage + stage_bytes);  // 16 zero bytes: E[-1] = 0
  uint32_t* cnt = zpad + 4;                                             // 2^W u16 counters
  uint32_t* blist = cnt + cnt_bytes / 4u;                               // buckets of >= 2 records
  __shared__ uint32_t wsum[NW], s_ncol, s_nbig, s_const;
  __shared__ unsigned long long sna[2], so[2];
  const int tid = threadIdx.x, lane = tid & 31;
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
      if (i * LB < lim) r[i] = ldg_rec<R>(p + (size_t)i * LB * R);
  };
  auto prefetch_l2 = [&](uint32_t b) {
    if (tid == 0 && b < nlist) {
      const Seg g = list[b];
      const uintptr_t s0 = (uintptr_t)(buf_of(g.src, recs, tmp) + (size_t)g.off * R);
      const uintptr_t s1 = (s0 + 15) & ~(uintptr_t)15, e1 = (s0 + (size_t)g.len * R) & ~(uintptr_t)15;
      if (e1 > s1) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s1), "r"((uint32_t)(e1 - s1)) : "memory");
    }
  };
  Seg sg = list[bi];
  load(sg);
  prefetch_l2(bi + gridDim.x);
  zero_cnt(cnt_bytes);
  if (tid < 4) zpad[tid] = 0;
  if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
  if (tid == 0) { s_ncol = 0; s_nbig = 0; s_const = 0; }
  unsigned long long done = 0;
  bool pending = false;  // a bulk store may still read the stage
  for (;;) {
    const uint32_t n = sg.len;
    const int lim = (int)n - tid;
    uint8_t* out = recs + (size_t)sg.off * R;
    uint32_t d = sg.depth;
    const uint32_t W = local_width(n, wmax);
    bool all_equal = false;
    __syncthreads();  // counters zero, flags reset
    for (;;) {  // one round unless the composite digit is constant over the bin
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if (i * LB < lim) {
          const uint32_t b = bucket_of(key_of<R, K>(r[i]), d, W);
          const uint32_t sh = 16u * (b & 1u);
          const uint32_t old = (atomicAdd(&cnt[b >> 1], 1u << sh) >> sh) & 0xffffu;
          if (old == 1u) blist[atomicAdd(&s_ncol, 1u)] = b;  // the bucket holds >= 2 records: list it once
        }
      }
      __syncthreads();
      if (tid == 0) {  // the whole bin in one bucket?
        const uint32_t b0 = bucket_of(key_of<R, K>(r[0]), d, W);
        s_const = reinterpret_cast<const uint16_t*>(cnt)[b0] == n ? 1u : 0u;
      }
      local_scan<LB>(cnt, W, wsum);  // (its barrier also publishes s_const)
      __syncthreads();
      if (!s_const) break;
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
      const uint32_t d2 = first_nonconst_digit<K>(A, O, d);
      __syncthreads();
      zero_cnt(2u << W);
      if (tid < 2) { sna[tid] = 0; so[tid] = 0; }
      if (tid == 0) { s_const = 0; s_ncol = 0; }
      __syncthreads();
      if (d2 >= (uint32_t)K) { all_equal = true; break; }
      d = d2;
    }
    if (pending && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    pending = false;
    __syncthreads();  // the previous bin's bulk store has read the stage
    if (all_equal) {  // final where it is (copied out of tmp)
      if (sg.src == SRC_TMP) {
#pragma unroll
        for (int i = 0; i < IL; ++i)
          if (i * LB < lim) st_rec<R>(out + (size_t)(i * LB + tid) * R, r[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if (i * LB < lim) {
          const uint32_t b = bucket_of(key_of<R, K>(r[i]), d, W);
          const uint32_t sh = 16u * (b & 1u);
          const uint32_t pos = (atomicAdd(&cnt[b >> 1], 1u << sh) >> sh) & 0xffffu;
          st_rec<R>(stage + (size_t)pos * R, r[i]);
        }
      }
    }
    // registers are free: the next bin's loads overlap this bin's finish
    uint32_t nb = bi + gridDim.x;
    while (nb < nlist && skip(nb)) nb += gridDim.x;
    Seg nsg = sg;
    if (nb < nlist) {
      nsg = list[nb];
      load(nsg);
    }
    prefetch_l2(nb + gridDim.x);
    if (!all_equal) {
      const bool fix = 8 * ((int)K - (int)d) > (int)W;  // key bits left below the composite digit
      __syncthreads();  // staged
      const bool bulk = (((uintptr_t)out | ((uintptr_t)n * R)) & 15u) == 0;
      // counters now hold bucket ends: start of bucket b = E[b - 1] (E[-1] = 0 in the pad)
      local_finish<R, K, LB, NW, false, true>(stage, reinterpret_cast<const uint16_t*>(cnt) - 1, blist, cap, n,
                                              1u << W, d, W, fix ? s_ncol : 0u, &s_nbig, nullptr, out, sg.off,
                                              local_next, nxt, ctl, bulk);
      pending = bulk;
    }
    done += n;
    __syncthreads();
    zero_cnt(2u << W);
    if (tid == 0) { s_ncol = 0; s_nbig = 0; s_const = 0; }
    if (nb >= nlist) break;
    bi = nb;
    sg = nsg;
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (tid == 0) atomicAdd(&ctl->rec_local, done);
}

// -------------------------------------------------------------- k_local_cluster
// The CTA-local sort for bins larger than one CTA's capacity C (up to about
// CS * C): a cluster of CS CTAs sorts one bin (GPU analog of PAPER.md:134, the
// counting scatter of a bin that fits on chip, with the cluster's distributed
// shared memory as the chip).  The composite digit's 2^W buckets are split
// into CS slices; CTA o owns slice o and sorts the records that fall in it.
//   1 each CTA loads 1/CS of the bin and ranks its records in a private
//     counter array over all 2^W buckets (local atomics);
//   2 the owner of each slice sums the CS counter arrays over its slice
//     (coalesced DSMEM reads), scans them into the slice's bucket starts,
//     lists the buckets of >= 2 records, and writes each CTA's base offset
//     per bucket back into that CTA's array (coalesced DSMEM writes);
//   3 every record is stored once into its owner's staging buffer, at
//     base (local read) + rank -- one remote store per record;
//   4 each CTA finishes its slice exactly as k_local does (fix-up of
//     colliding buckets, coalesced write-out).
// A bin whose slice would overflow a CTA's staging buffer, or whose composite
// digit is constant, is handed to the next level as a Large bin (nothing has
// been written yet).  The next bin of each CTA is prefetched into L2 (TMA
// bulk prefetch) while the current one is sorted.
template <int R, int K, int IL, int LB, int CS, bool DW>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(LB, 1)
    k_local_cluster(const Seg* __restrict__ list, uint32_t nlist, uint32_t wmax, uint32_t stage_bytes,
                    uint32_t cnt_bytes, uint32_t cap, Seg* local_next, int nxt, Seg* large_next, Ctl* ctl,
                    uint8_t* recs, uint8_t* tmp) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ uint4 smem_raw[];
  constexpr int NW = LB / 32;
  constexpr uint32_t LCS = CS == 2 ? 1u : (CS == 4 ? 2u : 3u);  // log2 CS
  constexpr uint32_t WMIN = LCS + 3u + 9u;                         // >= one 8-bucket chunk per thread and slice
  constexpr int NTW = (int)((2u << WMIN) / sizeof(TailScratch<K>)) < NW ? (int)((2u << WMIN) / sizeof(TailScratch<K>))
                                                                           : NW;  // tail scratch aliases the counters
  constexpr uint32_t C = local_capacity<R>();
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem_raw);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(stage + stage_bytes);  // 2^W u16: counts, then bases
  uint32_t* sst = cnt + cnt_bytes / 4u;                              // the slice's bucket starts (u16)
  uint32_t* blist = sst + (cnt_bytes >> LCS) / 4u;
  const uint16_t* cnt16 = reinterpret_cast<const uint16_t*>(cnt);
  __shared__ uint32_t wsum[NW], s_ncol, s_nbig, s_tot[CS], s_np, s_n3;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t crank = cl.block_rank();
  const uint32_t ncl = gridDim.x / CS;
  const uint32_t stage_cap = stage_bytes / R;
  auto zero_cnt = [&](uint32_t bytes) {
    uint4* c4 = reinterpret_cast<uint4*>(cnt);
    for (uint32_t i = tid; i < bytes / 16u; i += LB) c4[i] = make_uint4(0, 0, 0, 0);
  };
  auto prefetch_l2 = [&](uint32_t b) {  // this CTA's part of bin b
    if (tid == 0 && b < nlist) {
      const Seg g = list[b];
      if (g.len <= C) return;
      const uint32_t pt = (g.len + CS - 1) / CS, q0 = min(g.len, crank * pt), qn = min(g.len, q0 + pt) - q0;
      const uintptr_t s0 = (uintptr_t)(buf_of(g.src, recs, tmp) + ((size_t)g.off + q0) * R);
      const uintptr_t s1 = (s0 + 15) & ~(uintptr_t)15, e1 = (s0 + (size_t)qn * R) & ~(uintptr_t)15;
      if (e1 > s1)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s1), "r"((uint32_t)(e1 - s1)) : "memory");
    }
  };
  zero_cnt(cnt_bytes);
  if (tid == 0) { s_ncol = 0; s_nbig = 0; s_np = 0; s_n3 = 0; }
  __syncthreads();
  unsigned long long done = 0;
  Rec<R> r[IL];
#ifdef RADSORT_PHASE_PROF
  unsigned long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tA = clock64(), tB = 0;
#define RS_PROF(i) do { if (tid == 0) { tB = clock64(); pf[i] += tB - tA; tA = tB; } } while (0)
#else
#define RS_PROF(i) do { } while (0)
#endif
  auto next_bin = [&](uint32_t b) {  // bins <= C are k_local's
    while (b < nlist && list[b].len <= C) b += ncl;
    return b;
  };
  auto load = [&](const Seg& g) {  // this CTA's part of bin g into registers
    const uint32_t pt = (g.len + CS - 1) / CS, q0 = min(g.len, crank * pt), qn = min(g.len, q0 + pt) - q0;
    const uint8_t* src = buf_of(g.src, recs, tmp) + ((size_t)g.off + q0 + tid) * R;
#pragma unroll
    for (int i = 0; i < IL; ++i)
      if ((uint32_t)(i * LB + tid) < qn) r[i] = ldg_wide<R>(src + (size_t)i * LB * R);
  };
  // private ranks of this CTA's part of bin g (composite digit of width W(g))
  constexpr int IP = (IL + 1) / 2;
  uint32_t rk[IP];
  auto count = [&](const Seg& g) {
    const uint32_t pt = (g.len + CS - 1) / CS, q0 = min(g.len, crank * pt), qn = min(g.len, q0 + pt) - q0;
    const uint32_t Wg = max(local_width(g.len, wmax), WMIN);
#pragma unroll
    for (int i = 0; i < IP; ++i) rk[i] = 0;
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      if ((uint32_t)(i * LB + tid) < qn) {
        const uint32_t b = key_bits(key_of<R, K>(r[i]), 8u * g.depth + seg_skip(g.flags), Wg), sh = 16u * (b & 1u);
        const uint32_t old = (atomicAdd(&cnt[b >> 1], 1u << sh) >> sh) & 0xffffu;
        rk[i >> 1] |= old << (16 * (i & 1));
      }
    }
  };
  // per bin: [owner scan] #B [stage] #C [count the next bin | finish this one] #A
  uint32_t bi = next_bin(blockIdx.x / CS);
  Seg sg;
  if (bi < nlist) {
    sg = list[bi];
    load(sg);
    prefetch_l2(next_bin(bi + ncl));
    count(sg);
  }
  cl.sync();  // #A: every CTA has counted
  bool pending = false;  // a bulk store still reads the stage
  while (bi < nlist) {
    const uint32_t n = sg.len, d = sg.depth, sk = seg_skip(sg.flags);
    const uint32_t part = (n + CS - 1) / CS, p0 = min(n, crank * part), pn = min(n, p0 + part) - p0;
    const uint32_t W = max(local_width(n, wmax), WMIN);
    const uint32_t Wl = W - LCS, slice = 1u << Wl;
    if (tid == 0) {  // the next bins' descriptors into L1
      const uint32_t p1 = bi + ncl, p2 = p1 + ncl;
      if (p1 < nlist) asm volatile("prefetch.global.L1 [%0];" ::"l"(list + p1));
      if (p2 < nlist) asm volatile("prefetch.global.L1 [%0];" ::"l"(list + p2));
    }
    RS_PROF(0);
    // 2. slice owner: totals, starts, collision list, per-CTA bases
    const uint32_t nch = slice / 8u, m = nch / LB, c0 = (uint32_t)tid * m;
    uint4* sst4 = reinterpret_cast<uint4*>(sst);
    uint32_t T = 0, np = 0;
    bool cst = false;
    auto eqn = [&](uint32_t x) { return (x & 0xffffu) == n || (x >> 16) == n; };
    for (uint32_t j = 0; j < m; ++j) {
      const uint32_t ch = crank * nch + c0 + j;
      uint4 t = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < CS; ++k) {
        const uint4 v = reinterpret_cast<const uint4*>(cl.map_shared_rank(cnt, (uint32_t)k))[ch];
        t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
      }
      sst4[c0 + j] = t;
      const uint32_t p = t.x + t.y + t.z + t.w;
      T += (p & 0xffffu) + (p >> 16);
      cst |= eqn(t.x) | eqn(t.y) | eqn(t.z) | eqn(t.w);
      const uint32_t tw[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) np += ((tw[q >> 1] >> (16 * (q & 1))) & 0xffffu) == 2u;
    }
    np = __reduce_add_sync(0xffffffffu, np);  // pairs: listed first, so that the fix-up warps stay uniform
    if (lane == 0 && np) atomicAdd(&s_np, np);
    cst = __syncthreads_or(cst);
    uint32_t inc = T;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t tot = 0, carry = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      carry += w < warp ? wsum[w] : 0u;
      tot += wsum[w];
    }
    uint32_t s = carry + inc - T;
    for (uint32_t j = 0; j < m; ++j) {
      const uint32_t ch = crank * nch + c0 + j;
      const uint4 t = sst4[c0 + j];
      uint4 o4;
      o4.x = s * 0x10001u + (t.x << 16); s += (t.x & 0xffffu) + (t.x >> 16);
      o4.y = s * 0x10001u + (t.y << 16); s += (t.y & 0xffffu) + (t.y >> 16);
      o4.z = s * 0x10001u + (t.z << 16); s += (t.z & 0xffffu) + (t.z >> 16);
      o4.w = s * 0x10001u + (t.w << 16); s += (t.w & 0xffffu) + (t.w >> 16);
      sst4[c0 + j] = o4;
      uint4 v[CS];
#pragma unroll
      for (int k = 0; k < CS; ++k) v[k] = reinterpret_cast<const uint4*>(cl.map_shared_rank(cnt, (uint32_t)k))[ch];
      // buckets of >= 2 records join the collision list (one list append per warp)
      const uint32_t tw[4] = {t.x, t.y, t.z, t.w};
      uint32_t cm2 = 0, cm3 = 0;  // buckets of 2, and of >= 3 records
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t c = (tw[q >> 1] >> (16 * (q & 1))) & 0xffffu;
        cm2 |= (uint32_t)(c == 2u) << q;
        cm3 |= (uint32_t)(c >= 3u) << q;
      }
      const uint32_t cc = __popc(cm2) | __popc(cm3) << 16;  // both counts, one scan
      uint32_t ci = cc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) ci += y;
      }
      uint32_t b2 = 0, b3 = 0;
      if (lane == 31) {
        if (ci & 0xffffu) b2 = atomicAdd(&s_ncol, ci & 0xffffu);
        if (ci >> 16) b3 = s_np + atomicAdd(&s_n3, ci >> 16);
      }
      const uint32_t ex = ci - cc;
      b2 = __shfl_sync(0xffffffffu, b2, 31) + (ex & 0xffffu);
      b3 = __shfl_sync(0xffffffffu, b3, 31) + (ex >> 16);
      while (cm2) {
        const int q = __ffs(cm2) - 1;
        cm2 &= cm2 - 1u;
        if (b2 < cap) blist[b2] = (c0 + j) * 8u + (uint32_t)q;  // (a longer list: the slice overflows
        ++b2;                                                    // its stage, the bin is handed back)
      }
      while (cm3) {
        const int q = __ffs(cm3) - 1;
        cm3 &= cm3 - 1u;
        if (b3 < cap) blist[b3] = (c0 + j) * 8u + (uint32_t)q;
        ++b3;
      }
      uint4 run = o4;  // CTA k's records of a bucket follow those of CTAs < k
#pragma unroll
      for (int k = 0; k < CS; ++k) {
        reinterpret_cast<uint4*>(cl.map_shared_rank(cnt, (uint32_t)k))[ch] = run;
        run.x += v[k].x; run.y += v[k].y; run.z += v[k].z; run.w += v[k].w;
      }
    }
    if (tid < CS) cl.map_shared_rank(s_tot, (uint32_t)tid)[crank] = cst ? 0xffffffffu : tot;
    if (pending && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    pending = false;
    cl.sync();  // bases and slice totals in place; the stage is free
    RS_PROF(1);
    uint32_t off[CS], mine = 0;
    {
      uint32_t run = 0;
      bool over = false;
#pragma unroll
      for (int o = 0; o < CS; ++o) {
        off[o] = run;
        run += s_tot[o];
        over |= DW ? s_tot[o] == 0xffffffffu : s_tot[o] > stage_cap;  // DW: no staging, only a constant digit
      }
      mine = s_tot[crank];
      if (over) {  // skewed slices or a constant composite digit: the next level's Large list takes the bin
        if (crank == 0 && tid == 0) {
          Seg ns = sg;
          ns.mode = MODE_NONE;
          large_next[atomicAdd(&ctl->n_large_next, 1u)] = ns;
          atomicAdd(&ctl->rec_large_next, (unsigned long long)ns.len);
        }
        __syncthreads();
        zero_cnt(2u << W);
        if (tid == 0) { s_ncol = 0; s_nbig = 0; s_np = 0; s_n3 = 0; }
        __syncthreads();
        bi = next_bin(bi + ncl);
        if (bi < nlist) {
          sg = list[bi];
          load(sg);
          prefetch_l2(next_bin(bi + ncl));
          count(sg);
        }
        cl.sync();  // #A
        continue;
      }
    }
    if constexpr (DW) {
      // 3'. every record straight to its place in the output (the whole bin is
      // on chip in the cluster's registers, so writing over the input is safe):
      // a 32-byte record is one full sector, the write needs no staging
      uint8_t* bout = recs + (size_t)sg.off * R;
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if ((uint32_t)(i * LB + tid) < pn) {
          const uint32_t b = key_bits(key_of<R, K>(r[i]), 8u * d + sk, W);
          const uint32_t pos = (uint32_t)cnt16[b] + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu);
          stg_rec<R>(bout + (size_t)(off[b >> Wl] + pos) * R, r[i]);
        }
      }
    } else {
      // 3. one remote store per record
#pragma unroll
      for (int i = 0; i < IL; ++i) {
        if ((uint32_t)(i * LB + tid) < pn) {
          const uint32_t b = key_bits(key_of<R, K>(r[i]), 8u * d + sk, W);
          const uint32_t pos = (uint32_t)cnt16[b] + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu);
          const uint32_t o = b >> Wl;
          st_rec<R>((o == crank ? stage : cl.map_shared_rank(stage, o)) + (size_t)pos * R, r[i]);
        }
      }
    }
    // staged (this CTA's slice complete): split cluster barrier; the next
    // bin's records load between arrive and wait and while this one is finished
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    const uint32_t nb = next_bin(bi + ncl);
    Seg nsg;
    if (nb < nlist) {
      nsg = list[nb];
      load(nsg);
      prefetch_l2(next_bin(nb + ncl));
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // #C
    RS_PROF(2);
    // the bases are consumed: zero the counters (the next bin is counted after this one is finished)
    zero_cnt(2u << W);
    // 4. finish the slice (mixed buckets of > ES records go to the next Local
    // level: the tail sorter's scratch would alias the live counters)
    const bool fix = 8 * ((int)K - (int)d) - (int)sk > (int)W;
    uint8_t* out = recs + ((size_t)sg.off + off[crank]) * R;
    if constexpr (DW) {  // the slice's colliding buckets, in place in global memory (L2-resident)
      global_fixup<R, K, LB>(out, reinterpret_cast<const uint16_t*>(sst), blist, mine, slice, d, W,
                             fix ? s_np + s_n3 : 0u, &s_nbig, sg.off + off[crank], local_next, nxt, ctl);
    } else {
      const bool bulk = mine && (((uintptr_t)out | ((uintptr_t)mine * R)) & 15u) == 0;
      local_finish<R, K, LB, NW, false, true>(stage, reinterpret_cast<const uint16_t*>(sst), blist, cap, mine, slice,
                                              d, W, fix ? s_np + s_n3 : 0u, &s_nbig, nullptr, out,
                                              sg.off + off[crank], local_next, nxt, ctl, bulk,
#ifdef RADSORT_PHASE_PROF
                                              pf + 4,
#else
                                              nullptr,
#endif
                                              (int)(d + (sk + W) / 8u));
      pending = bulk;
    }
    done += mine;
    __syncthreads();  // counters zeroed by every thread
    if (nb < nlist) count(nsg);
    __syncthreads();
    RS_PROF(3);
    if (tid == 0) { s_ncol = 0; s_nbig = 0; s_np = 0; s_n3 = 0; }
    cl.sync();  // #A: every CTA has counted the next bin (and finished this one)
    bi = nb;
    sg = nsg;
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (tid == 0 && done) atomicAdd(&ctl->rec_local, done);
#ifdef RADSORT_PHASE_PROF
  if (tid == 0) {
    for (int q = 0; q < 8; ++q) atomicAdd(&ctl->prof[8 + q], pf[q]);
  }
#endif
#undef RS_PROF
  cl.sync();  // no CTA leaves while peers may still access its shared memory
}

// -------------------------------------------------------------- k_bounds
// Multi-GPU splitter search: for probe m, the number of keys < probe (lt) and
// <= probe (le) inside the SORTED record range [lo[m], hi[m]) of buf (binary
// search; the keys there are sorted by the single-GPU path first).
template <int R, int K>
__global__ void k_bounds(const uint8_t* __restrict__ buf, const uint32_t* __restrict__ lo,
                         const uint32_t* __restrict__ hi, const unsigned long long* __restrict__ probes, uint32_t M,
                         unsigned long long* __restrict__ lt, unsigned long long* __restrict__ le) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  Key<K> x;
  x.w0 = probes[(size_t)m * 2];
  if constexpr (K == 16) x.w1 = probes[(size_t)m * 2 + 1];
  uint32_t a = lo[m], b = hi[m];
  while (a < b) {  // first key >= x
    const uint32_t mid = a + ((b - a) >> 1);
    if (key_lt(ld_key<R, K>(buf + (size_t)mid * R), x)) a = mid + 1; else b = mid;
  }
  const uint32_t l = a;
  b = hi[m];
  while (a < b) {  // first key > x
    const uint32_t mid = a + ((b - a) >> 1);
    if (!key_lt(x, ld_key<R, K>(buf + (size_t)mid * R))) a = mid + 1; else b = mid;
  }
  lt[m] = l - lo[m];
  le[m] = a - lo[m];
}

}  // namespace radsort
