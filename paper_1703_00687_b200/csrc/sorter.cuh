// The MSD level loop for one record layout (instantiated in layout_R_K.cu).
#pragma once
#include "driver.cuh"

namespace radsort {

// -------------------------------------------------------------- the sort
template <int R, int K>
struct Sorter {
  static constexpr uint32_t C = local_capacity<R>();
  static constexpr int CHILD_SCRATCH = (CHILD_B / 32) * (int)TINY_MAX * R;
  static constexpr size_t LOCAL_SMEM_MAX = 227 * 1024 - 1024;  // dynamic smem ceiling per CTA (static smem aside)

  template <int IL, int LB>
  static void launch_local_t(Context* ctx, uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt,
                             Ctl* ctl, uint8_t* recs, uint8_t* tmp, cudaStream_t st, uint32_t lmin = 0,
                             uint32_t lmax = C) {
    const int sms = ctx->sms;
    lmax = std::min(lmax, ctx_local_hi);  // larger bins belong to k_local2
    maxlen = std::min(maxlen, lmax);
    // smem: staged bin | 2^W u16 counters (aliased by the tail sorter's per-warp
    // scratch) | list of the buckets holding >= 2 records
    const size_t stage_bytes = (((size_t)maxlen * R + 15) & ~(size_t)15) + 16;  // + the alignment shift
    const size_t tail_bytes = (LB / 32) * sizeof(TailScratch<K>);
    const uint32_t cap = maxlen / 2 + 1;  // buckets holding >= 2 records
    const size_t big_bytes = ((size_t)cap * 4 + 15) & ~(size_t)15;
    uint32_t wmax = local_width(maxlen, 16);
    auto cnt_of = [&](uint32_t w) { return std::max((size_t)2 << w, tail_bytes); };
    while (wmax > LOCAL_WMIN && stage_bytes + cnt_of(wmax) + big_bytes > LOCAL_SMEM_MAX) --wmax;
    const size_t cnt_bytes = cnt_of(wmax);
    const size_t smem = stage_bytes + cnt_bytes + big_bytes;
    if constexpr (LB == 512 || LB == 256) {
      // one bin per SM (512 threads) or two (256): the bin-pipelined variant (k_local_pipe).
      // Measured and dropped: the same at 1024 threads (c5 local 6.74 -> 6.52 ms but c3 5.06 ->
      // 5.23 ms, 18 B of spills)
      if (pipe_on() && (LB == 512 || pipe256_on())) {
        auto* kfn = early_on() ? k_local_pipe<R, K, IL, LB, true> : k_local_pipe<R, K, IL, LB, false>;
        smem_attr(ctx, kfn, (int)LOCAL_SMEM_MAX);
        int occ = 1;
        if (LB < 512) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, LB, smem);
        const unsigned g = (unsigned)std::min<size_t>(nloc, (size_t)sms * std::max(occ, 1));
        kfn<<<g, LB, smem, st>>>(list, nloc, wmax, (uint32_t)stage_bytes, (uint32_t)cnt_bytes, cap, next, nxt, ctl, recs,
                                 tmp, lmin, lmax, wdelta(), pf_dist());
        return;
      }
    }
    if constexpr (LB <= 512) launch_local_k<IL, LB>(ctx, nloc, list, next, nxt, ctl, recs, tmp, lmin, lmax, wmax,
                                                   stage_bytes, cnt_bytes, cap, smem, st);
  }
  template <int IL, int LB>
  static void launch_local_k(Context* ctx, uint32_t nloc, const Seg* list, Seg* next, int nxt, Ctl* ctl, uint8_t* recs,
                             uint8_t* tmp, uint32_t lmin, uint32_t lmax, uint32_t wmax, size_t stage_bytes,
                             size_t cnt_bytes, uint32_t cap, size_t smem, cudaStream_t st) {
    const int sms = ctx->sms;
    smem_attr(ctx, k_local<R, K, IL, LB>, (int)LOCAL_SMEM_MAX);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_local<R, K, IL, LB>, LB, smem);
    const unsigned g = (unsigned)std::min<size_t>(nloc, (size_t)sms * std::max(occ, 1));
    k_local<R, K, IL, LB><<<g, LB, smem, st>>>(list, nloc, wmax, (uint32_t)stage_bytes, (uint32_t)cnt_bytes, cap, next, nxt,
                                               ctl, recs, tmp, lmin, lmax);
  }

  // RADSORT_LOCAL_PIPE=0: the 512-thread local sort as k_local (round 1) instead of k_local_pipe
  // RADSORT_LOCAL_WDELTA: composite digit width of k_local_pipe relative to ceil(log2 n) + 1 (experiments)
  static int wdelta() {
    const char* e = getenv("RADSORT_LOCAL_WDELTA");
    return e ? atoi(e) : 0;
  }
  // k_local_pipe<EF>: a bin's fix-up and bulk store issued before the next bin's count, while its
  // loads are in flight (default; measured c4 local 16.97 -> 15.26 ms, c5 / c2 unchanged);
  // RADSORT_LOCAL_EARLY=0: beside the next bin's counting atomics.  Measured and dropped: a
  // branch-free count (absent records counted in pad words): c4 15.26 -> 15.57, c5 6.70 -> 9.02 (spills)
  static bool early_on() {
    const char* e = getenv("RADSORT_LOCAL_EARLY");
    return !(e && e[0] == '0');
  }
  // the 256-thread (two CTAs per SM) local sorts pipelined too: default for R >= 16 (measured
  // c2 local 1.81 -> 1.56 ms, kmc unchanged; c3 (R = 8, Zipf) 5.19 -> 5.51 ms: off for R = 8);
  // RADSORT_LOCAL_PIPE256=1 / 0 forces it on / off
  static bool pipe256_on() {
    const char* e = getenv("RADSORT_LOCAL_PIPE256");
    return e ? e[0] == '1' : R >= 16;
  }
  static uint32_t pf_dist() {  // k_local_pipe: how many bins ahead of the loaded one go to L2 (RADSORT_LOCAL_PFD)
    const char* e = getenv("RADSORT_LOCAL_PFD");
    return e ? (uint32_t)std::max(0, atoi(e)) : 1u;
  }
  static bool pipe_on() {
    const char* e = getenv("RADSORT_LOCAL_PIPE");
    return !(e && e[0] == '0');
  }

  // ---- the largest local bins: k_local_big (1024 threads, one bin per SM) with
  // RADSORT_LOCAL_BIG=1; k_local at 512 threads otherwise
  static bool big_on() {  // measured: c5 local 7.52 -> 7.22 ms, c3 5.23 -> 5.68 ms: opt-in
    const char* e = getenv("RADSORT_LOCAL_BIG");
    return e && e[0] == '1';
  }
  static void launch_big(Context* ctx, uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt, Ctl* ctl,
                         uint8_t* recs, uint8_t* tmp, cudaStream_t st, uint32_t lmin, uint32_t lmax) {
    constexpr int LB = 1024, IL = (int)((C + LB - 1) / LB);
    lmax = std::min(lmax, ctx_local_hi);
    maxlen = std::min(maxlen, lmax);
    const size_t stage_bytes = ((size_t)maxlen * R + 15) & ~(size_t)15;
    const uint32_t cap = maxlen / 2 + 1;
    const size_t big_bytes = ((size_t)cap * 4 + 15) & ~(size_t)15;
    uint32_t wmax = local_width(maxlen, 16);
    while (wmax > LOCAL_WMIN && stage_bytes + 16 + ((size_t)2 << wmax) + big_bytes > LOCAL_SMEM_MAX) --wmax;
    const size_t cnt_bytes = (size_t)2 << wmax;
    const size_t smem = stage_bytes + 16 + cnt_bytes + big_bytes;
    auto* kfn = k_local_big<R, K, IL, LB>;
    smem_attr(ctx, kfn, (int)LOCAL_SMEM_MAX);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, LB, smem);
    const unsigned g = (unsigned)std::min<size_t>(nloc, (size_t)ctx->sms * std::max(occ, 1));
    kfn<<<g, LB, smem, st>>>(list, nloc, wmax, (uint32_t)stage_bytes, (uint32_t)cnt_bytes, cap, next, nxt, ctl, recs,
                             tmp, lmin, lmax);
  }

  // ---- two-phase local sort (bins of local2_min() <= n <= local2_max<R>() records, k_local2)
  static constexpr bool L2_BUILT = R == 8 || R == 16 || R == 32;  // off by default (RADSORT_LOCAL2=1): measured slower, DESIGN.md §3
  static inline thread_local uint32_t ctx_local_hi = 0xffffffffu;  // the k_local launches' ceiling (set per launch_local)
  // RADSORT_LOCAL2=0 disables it (the single-CTA and cluster sorts take the bins, as in round 1);
  // RADSORT_LOCAL2_MIN sets the smallest bin it takes (default: 4096 records)
  static uint32_t local2_min() {
    if constexpr (!L2_BUILT) return 0xffffffffu;
    const char* e = getenv("RADSORT_LOCAL2");
    if (!e || e[0] != '1') return 0xffffffffu;
    const char* m = getenv("RADSORT_LOCAL2_MIN");
    return m ? (uint32_t)atoi(m) : 4096u;
  }
  static uint32_t l2_gcap() {  // smallest group k_local2 hands back as a Large bin (+1)
    if constexpr (L2_BUILT) return (uint32_t)L2Cfg<R>::GCAP;
    return C;
  }
  static uint32_t local_max() {  // the largest bin the Local list takes
    if constexpr (L2_BUILT) {
      if (local2_min() != 0xffffffffu) return std::max(C, local2_max<R>());
    }
    return C;
  }
  static void launch_local2(Context* ctx, uint32_t nloc, const Seg* list, Seg* next, int nxt, Seg* large_next,
                            Ctl* ctl, uint8_t* recs, uint8_t* tmp, cudaStream_t st, uint32_t lmin) {
    if constexpr (L2_BUILT) {
      constexpr int LB = L2Cfg<R>::LB;
      const size_t smem = local2_smem<R>();
      smem_attr(ctx, k_local2<R, K>, (int)smem);
      int occ = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_local2<R, K>, LB, smem);
      const char* e = getenv("RADSORT_DISCARD");
      const int discard = e ? atoi(e) : 1;
      const unsigned g = (unsigned)std::min<size_t>(nloc, (size_t)ctx->sms * std::max(occ, 1));
      k_local2<R, K><<<g, LB, smem, st>>>(list, nloc, lmin, local2_max<R>(), next, nxt, large_next, ctl, recs, tmp,
                                          discard);
    }
  }

  // ---- cluster-local sort (bins of CL_MIN <= n <= ccap() records, k_local_cluster)
  // One shape: clusters of 4 CTAs of 512 threads, one per SM (132 SMs: a GPC
  // holds no fifth 4-CTA cluster).  Measured and dropped: 8 CTAs of 256 threads,
  // two per SM (c4 local 32.5 -> 42.5 ms: the same 33 bins in flight -- the
  // register file holds one bin per 4 SMs either way -- with 7/8 instead of
  // 3/4 of the records crossing DSMEM).
  static constexpr uint32_t CL_W = R >= 24 ? 14 : 15;                     // composite digit width cap
  static constexpr int CL_ILMAX = R <= 8 ? 32 : (R <= 16 ? 16 : 8);       // register budget of the record array
  template <int CS_, int LB_, int MINB_>
  struct ClCfg {
    static constexpr int CS = CS_, LB = LB_, MINB = MINB_;
    static constexpr uint32_t LCS = CS == 2 ? 1u : (CS == 4 ? 2u : 3u);
    static constexpr size_t CNT = (size_t)2 << CL_W;                       // 2^W u16 counters / bases
    static constexpr size_t SST = CNT >> LCS;                               // the slice's bucket starts
    static constexpr size_t SMEM = MINB == 1 ? LOCAL_SMEM_MAX : (size_t)228 * 1024 / MINB - 1536;
    // smem: stage | counters | slice starts | collision list
    static constexpr uint32_t STAGE_CAP = (uint32_t)((SMEM - CNT - SST - 2048) / (R + 2));
    // 20 % slack for uneven bucket slices (an overflowing slice hands the bin back to the Large list)
    static constexpr uint32_t CCAP_SMEM = STAGE_CAP / 5 * 4 * CS;
    static constexpr uint32_t CCAP = CCAP_SMEM < (uint32_t)(CL_ILMAX * LB * CS) ? CCAP_SMEM : CL_ILMAX * LB * CS;
  };
  using Cl4 = ClCfg<4, 512, 1>;
  static uint32_t ccap() { return Cl4::CCAP; }
  // smaller bins (C < n < CL_MIN) take a further radix level: below ~2.5 C the
  // cluster's per-bin phases cost more than the pass they save (measured, R = 32)
  static constexpr uint32_t CL_MIN = C * 5 / 2;

  // DW (direct write): records go from the cluster's registers straight to
  // their output slots (no shared-memory staging; a 32-byte record is one full
  // sector, one STG.256), colliding buckets are fixed up in global memory.
  // Measured on c4: direct writes 10.3 K vs DSMEM staging 14.6 K cycles per
  // bin, but the global fix-up costs more than it saves (local 34.3 vs 32.7
  // ms) -- off unless RADSORT_CLUSTER_DW=1 (R >= 24)
  static bool cluster_dw() {
    const char* e = getenv("RADSORT_CLUSTER_DW");
    return R >= 24 && e && e[0] == '1';
  }

  template <int IL, bool DW, class CF>
  static void launch_cluster_t(Context* ctx, uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt,
                               Seg* large_next, Ctl* ctl, uint8_t* recs, uint8_t* tmp, cudaStream_t st) {
    const int sms = ctx->sms;
    const uint32_t wmax = CL_W;
    const size_t stage_bytes = DW ? 0 : ((size_t)CF::STAGE_CAP * R + 15) & ~(size_t)15;
    const uint32_t cap = DW ? CF::CCAP / 2 + 1 : CF::STAGE_CAP / 2 + 1;
    const size_t smem = stage_bytes + CF::CNT + CF::SST + (((size_t)cap * 4 + 15) & ~(size_t)15);
    auto* kfn = k_local_cluster<R, K, IL, CF::LB, CF::CS, DW>;
    smem_attr(ctx, kfn, (int)CF::SMEM);
    int& max_clusters = ctx->max_clusters[(const void*)kfn];  // per device (the context's)
    if (!max_clusters) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CF::CS * sms, 1, 1);
      cfg.blockDim = dim3(CF::LB, 1, 1);
      cfg.dynamicSmemBytes = smem;
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kfn, &cfg) != cudaSuccess || max_clusters <= 0) {
        cudaGetLastError();
        max_clusters = sms * CF::MINB / CF::CS;
      }
      if (getenv("RADSORT_LOG"))
        fprintf(stderr, "[radsort] k_local_cluster %dx%d: %d clusters resident, %zu B smem per CTA\n", CF::CS, CF::LB,
                max_clusters, smem);
    }
    const unsigned clusters = (unsigned)std::max<size_t>(1, std::min<size_t>(nloc, (size_t)max_clusters));
    kfn<<<clusters * CF::CS, CF::LB, smem, st>>>(list, nloc, wmax, (uint32_t)stage_bytes, (uint32_t)CF::CNT, cap, next,
                                                  nxt, large_next, ctl, recs, tmp);
  }

  template <class CF>
  static void launch_cluster_c(Context* ctx, uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt,
                               Seg* large_next, Ctl* ctl, uint8_t* recs, uint8_t* tmp, cudaStream_t st) {
    const uint32_t il = (maxlen + CF::CS * CF::LB - 1) / (CF::CS * CF::LB);  // records per thread
#define RS_CL(IL)                                                                                                  \
  do {                                                                                                             \
    bool dw_ = false;                                                                                              \
    if constexpr (CF::CS == 4) {                                                                                   \
      if ((dw_ = cluster_dw()))                                                                                    \
        launch_cluster_t<IL, true, CF>(ctx, nloc, maxlen, list, next, nxt, large_next, ctl, recs, tmp, st);        \
    }                                                                                                              \
    if (!dw_) launch_cluster_t<IL, false, CF>(ctx, nloc, maxlen, list, next, nxt, large_next, ctl, recs, tmp, st); \
  } while (0)
    if (il <= 2) RS_CL(2);
    else if (il <= 4) RS_CL(4);
    else if constexpr (R <= 32) {
      if (il <= 8) RS_CL(8);
      else if constexpr (R <= 8) {
        if (il <= 16) RS_CL(16);
        else RS_CL(32);
      } else if constexpr (R <= 16) {
        RS_CL(16);
      }
    } else {
      RS_CL(8);
    }
#undef RS_CL
  }
  static void launch_cluster(Context* ctx, uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt,
                             Seg* large_next, Ctl* ctl, uint8_t* recs, uint8_t* tmp, cudaStream_t st) {
    launch_cluster_c<Cl4>(ctx, nloc, maxlen, list, next, nxt, large_next, ctl, recs, tmp, st);
  }

  static void set_attrs(Context* ctx) { smem_attr(ctx, k_children<R, K>, CHILD_SCRATCH); }

  // Local bins of up to `maxlen` records: IL records per thread, at most 256
  // bytes of records per thread; 256-thread CTAs (two per SM) unless the bins
  // need 512 threads.
  // Returns true when a cluster launch may have handed bins to the next level's Large list.
  static bool launch_local(Context* ctx, uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt,
                           Seg* large_next, Ctl* ctl, uint8_t* recs, uint8_t* tmp, cudaStream_t st, uint32_t nsmall,
                           uint32_t nmed, int& nl) {
    const int sms = ctx->sms;
    nl = 1;
    ctx_local_hi = 0xffffffffu;
    bool handed = false;
    {
      const uint32_t t2 = local2_min();
      if (t2 != 0xffffffffu) {
        if (maxlen >= t2) {  // the big bins: two-phase local sort (may hand groups back as Large bins)
          launch_local2(ctx, nloc, list, next, nxt, large_next, ctl, recs, tmp, st, t2);
          handed = true;
          if (nloc == 0) return true;
          ++nl;
        }
        ctx_local_hi = t2 - 1;
        if (maxlen >= t2) maxlen = t2 - 1;
      }
    }
    // small bins (up to 256 B of records per thread at 64 threads): 64-thread
    // CTAs, so that many bins are in flight per SM (the per-bin phases are
    // latency-bound).  A list whose largest bin needs a bigger
    // configuration but which holds at least one small bin per SM (counted by
    // k_children / the tail queue) is split by size: its small bins run first
    // in 64-thread CTAs, the bigger configuration then skips them.
    constexpr int ILS = 256 / R >= 16 ? 16 : (256 / R >= 8 ? 8 : 4);
    constexpr uint32_t SMALL = small_cap<R>();
    static_assert(SMALL == 64u * (uint32_t)ILS, "small_cap");
    uint32_t lo = 0;
    if (maxlen > SMALL && nsmall >= (uint32_t)sms && small_split()) {
      launch_local_t<ILS, 64>(ctx, nloc, SMALL, list, next, nxt, ctl, recs, tmp, st, 0, SMALL);
      lo = SMALL + 1;
      ++nl;
    }
    if (maxlen > C) {  // the list holds cluster-size bins: k_local takes the rest at full capacity
      if (big_on()) launch_big(ctx, nloc, C, list, next, nxt, ctl, recs, tmp, st, lo, C);
      else launch_local_t<(int)((C + 511) / 512), 512>(ctx, nloc, C, list, next, nxt, ctl, recs, tmp, st, lo, C);
      launch_cluster(ctx, nloc, maxlen, list, next, nxt, large_next, ctl, recs, tmp, st);
      ++nl;
      return true;
    }
    if (maxlen <= SMALL) {
      const uint32_t il = (maxlen + 63) / 64;
#define RS_LOCAL_S(IL) launch_local_t<IL, 64>(ctx, nloc, maxlen, list, next, nxt, ctl, recs, tmp, st)
      if (il <= 2) RS_LOCAL_S(2);
      else if (il <= 4) RS_LOCAL_S(4);
      else if constexpr (ILS >= 8) {
        if (il <= 8) RS_LOCAL_S(8);
        else if constexpr (ILS >= 16) RS_LOCAL_S(16);
      }
#undef RS_LOCAL_S
      return handed;
    }
    constexpr int ILMAX = (int)((C + 511) / 512);  // records per thread at 512 threads
    static_assert(med_cap<R>() == 256u * (uint32_t)ILMAX, "med_cap");
    if ((size_t)maxlen > (size_t)256 * ILMAX) {
      if (nmed >= (uint32_t)sms && small_split()) {  // the medium bins in 256-thread CTAs, two per SM
        launch_local_t<ILMAX, 256>(ctx, nloc, med_cap<R>(), list, next, nxt, ctl, recs, tmp, st, lo, med_cap<R>());
        lo = med_cap<R>() + 1;
        ++nl;
      }
      if (big_on()) launch_big(ctx, nloc, maxlen, list, next, nxt, ctl, recs, tmp, st, lo, C);
      else launch_local_t<ILMAX, 512>(ctx, nloc, maxlen, list, next, nxt, ctl, recs, tmp, st, lo, C);
      return handed;
    }
    const uint32_t il = (maxlen + 255) / 256;
#define RS_LOCAL(IL) launch_local_t<IL, 256>(ctx, nloc, maxlen, list, next, nxt, ctl, recs, tmp, st, lo, C)
    if (il <= 1) RS_LOCAL(1);
    else if (il <= 2) RS_LOCAL(2);
    else if (il <= 4) RS_LOCAL(4);
    else if constexpr (ILMAX <= 8) RS_LOCAL(ILMAX);
    else if (il <= 8) RS_LOCAL(8);
    else if constexpr (ILMAX <= 16) RS_LOCAL(ILMAX);
    else if (il <= 16) RS_LOCAL(16);
    else RS_LOCAL(ILMAX);
#undef RS_LOCAL
    return handed;
  }

  // tiny bins of 17..32 records (R <= 16) are sorted by the warp bitonic network
  // in k_children instead of the tail sorter: the tiny-sorter grid
  // (profiles/r01_tinybench.txt) has it fastest there; end to end it is
  // neutral on c3 / kmc.  RADSORT_TINY_BITONIC=n sets the
  // ceiling (0 = tail sorter only; R <= 16, n <= 32)
  static uint32_t bitonic_max() {
    const char* e = getenv("RADSORT_TINY_BITONIC");
    const uint32_t v = e ? (uint32_t)atoi(e) : 32u;
    return R <= 16 ? std::min(v, 32u) : 0u;
  }

  // size-split local launches (RADSORT_LOCAL_SPLIT=0 disables; measured)
  static bool small_split() {
    const char* e = getenv("RADSORT_LOCAL_SPLIT");
    return e ? atoi(e) != 0 : true;
  }

  struct Views {
    Seg* L[2];
    Seg* Lo[2];
    uint32_t *hist, *segbase, *tile_start;
    unsigned long long *andor, *status, *probes;
    uint32_t *splitc, *tile_seg, *tile_pre;
    Ctl* ctl;
    size_t tiles_max;
  };

  // Grow the workspace for n records and tiles of T records.
  // lookback: the decoupled look-back status words (tiles x 256 u64) are
  // needed (RADSORT_LOOKBACK=1, multi-GPU level-0 pass); otherwise the
  // reduce-then-scan tile prefixes (tiles x 256 u32).
  // extra: initial segments of a presegmented input (multi-GPU receive side), any size
  static radsort_status prepare(Context* ctx, uint32_t n, uint32_t T, Views& v, bool lookback = false,
                                uint32_t extra = 0) {
    // Large bins hold > C records, except the skewed groups k_local2 hands back (> its GCAP)
    const size_t capL = (size_t)n / (local2_min() != 0xffffffffu ? l2_gcap() : C) + 4 + extra;
    // Local bins: children of > TINY_MAX records, or mixed buckets of > ES_MAX records queued by
    // the cluster / pipelined local sorts
    const size_t capLoc = (size_t)n / (es_max<R>() + 1) + 4 + extra;
    const size_t tiles_max = (size_t)n / T + capL + 4;
    radsort_status rs;
    if ((rs = ensure(ctx->large[0], capL * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->large[1], capL * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->local[0], capLoc * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->local[1], capLoc * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->hist, capL * RADIX * sizeof(uint32_t)))) return rs;
    if ((rs = ensure(ctx->segbase, capL * RADIX * sizeof(uint32_t)))) return rs;
    if ((rs = ensure(ctx->andor, capL * 8 * sizeof(unsigned long long)))) return rs;
    if ((rs = ensure(ctx->splitc, capL * 4 * sizeof(uint32_t)))) return rs;
    if ((rs = ensure(ctx->probes, capL * 2 * sizeof(unsigned long long)))) return rs;
    if ((rs = ensure(ctx->tile_seg, tiles_max * sizeof(uint32_t)))) return rs;
    if ((rs = ensure(ctx->tile_start, (capL + 1) * sizeof(uint32_t)))) return rs;
    if (lookback) {
      const size_t old_status = ctx->status.bytes;
      if ((rs = ensure(ctx->status, tiles_max * RADIX * sizeof(unsigned long long), true))) return rs;
      if (ctx->status.bytes != old_status) ctx->epoch = 0;
    } else {
      if ((rs = ensure(ctx->tile_pre, tiles_max * RADIX * sizeof(uint32_t)))) return rs;
    }
    if ((rs = ensure(ctx->ctl, sizeof(Ctl)))) return rs;
    if (!ctx->h_ctl) RS_CUDA(cudaMallocHost(&ctx->h_ctl, sizeof(Ctl)));
    v.L[0] = (Seg*)ctx->large[0].p;
    v.L[1] = (Seg*)ctx->large[1].p;
    v.Lo[0] = (Seg*)ctx->local[0].p;
    v.Lo[1] = (Seg*)ctx->local[1].p;
    v.hist = (uint32_t*)ctx->hist.p;
    v.segbase = (uint32_t*)ctx->segbase.p;
    v.andor = (unsigned long long*)ctx->andor.p;
    v.splitc = (uint32_t*)ctx->splitc.p;
    v.probes = (unsigned long long*)ctx->probes.p;
    v.tile_seg = (uint32_t*)ctx->tile_seg.p;
    v.tile_start = (uint32_t*)ctx->tile_start.p;
    v.status = (unsigned long long*)ctx->status.p;
    v.tile_pre = (uint32_t*)ctx->tile_pre.p;
    v.ctl = (Ctl*)ctx->ctl.p;
    v.tiles_max = tiles_max;
    return RADSORT_OK;
  }

  // Scatter/histogram tile configuration: TB bytes per tile, SB threads per
  // scatter CTA, MINB scatter CTAs per SM (RADSORT_SCATTER_CFG selects).
  // Initial bins (multi-GPU receive side): records [off[i], off[i]+len[i]) of
  // `recs` already share their first `depth` digits; nullptr = the whole array.
  struct Init {
    const uint32_t* off;
    const uint32_t* len;
    uint32_t nseg, depth;
  };

  // the scatter's digit runs leave by TMA bulk copies (R = 16, 32; RADSORT_SCATTER_TMA=0: thread stores;
  // c4 level-0 scatter 11.8 -> 10.3 ms, c2 2.39 -> 2.16 ms)
  // Measured and dropped (c4, ms per pass): runs shorter than 2 / 4 records stored by the digit's
  // thread instead of a bulk copy (whose issue costs ~12 warp instructions: the operands go to
  // uniform registers lane by lane): wide level 13.57 -> 14.65 / 18.29, 8-bit level 10.2 -> 10.2 / 12.2;
  // the wide level's plain write-out (RADSORT_SCATTER_TMA=3): 14.55
  static bool scatter_tma(int db) {
    const char* e = getenv("RADSORT_SCATTER_TMA");
    if (e && e[0] == '3') return db == 8;  // (experiment: 8-bit levels only)
    // 1 (default): every R but 8; 2: every R; 0: plain coalesced write-out everywhere.  R = 8, 24, 40
    // stage their runs at the parity of their HBM slot; measured (ms per sort, 2 vs 0): (24,8) 900 M
    // 44.7 / 48.7, (24,16) 48.7 / 49.5, (40,16) 500 M 52.4 / 53.0, but c5 (8,8) 17.0 / 16.5
    const int mode = e ? atoi(e) : 1;
    return mode == 2 || (mode == 1 && R != 8);
  }

  // One Large level: tile map, histogram + cross-tile prefix, plan, scatter,
  // children.  DB = 8 (256 digits) or 10 (a wide level, 1024 digits; reduce-then-scan only).
  template <uint32_t T_, int TB_, int SB_, int MINB_, int DB>
  static radsort_status level_pass(Context* ctx, const Views& v, uint32_t n, uint32_t n_large, int cur, int nxt, uint8_t* recs,
                         uint8_t* tmp, cudaStream_t st, Timer& tm, radsort_stats& stats, unsigned hist_grid, int occ_s,
                         uint32_t* ch_first, uint32_t* ch_last, uint32_t* ch_tot, uint32_t* carry_in, bool cluster_ok,
                         bool pre = true, int occ_h = 1) {
    constexpr int DG = 1 << DB;
    Seg* const* L = v.L;
    Seg* const* Lo = v.Lo;
    RS_CUDA(cudaMemsetAsync(v.hist, 0, (size_t)n_large * DG * sizeof(uint32_t), st));
    RS_CUDA(cudaMemsetAsync(v.andor, 0, (size_t)n_large * 8 * sizeof(unsigned long long), st));
    tm.begin(RADSORT_K_PLAN);
    k_prep<<<1, 1024, 0, st>>>(L[cur], n_large, T_, v.tile_start, v.ctl, nxt);
    const size_t tiles_ub = std::min(v.tiles_max, (size_t)n / T_ + n_large + 1);
    k_tilemap<<<(unsigned)std::min<size_t>((tiles_ub + 255) / 256, (size_t)ctx->sms * 16), 256, 0, st>>>(
        v.tile_start, n_large, v.ctl, v.tile_seg);
    tm.end();
    tm.begin(RADSORT_K_HIST);
    if (pre) {
      k_cand<R, K><<<(n_large + 7) / 8, 256, 0, st>>>(L[cur], n_large, recs, tmp);
      k_hist_pre<R, K, T_, DB><<<hist_grid, HIST_B, 0, st>>>(L[cur], v.tile_start, n_large, v.ctl, v.hist, v.andor, recs,
                                                            tmp, v.tile_pre, ch_first, ch_last, ch_tot, v.tile_seg);
      k_carry<DG><<<1, DG, 0, st>>>(ch_first, ch_last, ch_tot, hist_grid, carry_in);
    } else {
      if constexpr (DB == 8) {
        const unsigned gh = (unsigned)std::min(tiles_ub, (size_t)ctx->sms * occ_h);
        k_hist<R, K, T_><<<gh, HIST_B, 0, st>>>(L[cur], v.tile_start, n_large, v.ctl, v.hist, v.andor, recs, tmp);
      }
    }
    tm.end();
    tm.begin(RADSORT_K_PLAN);
    k_plan<R, K, DG><<<n_large, DG, 0, st>>>(L[cur], v.hist, v.andor, v.segbase, L[nxt], v.ctl, v.splitc, pre ? 1 : 0);
    tm.end();
    if (!pre && ++ctx->epoch >= 65536) {  // look-back status words are epoch-tagged, never cleared
      RS_CUDA(cudaMemsetAsync(v.status, 0, ctx->status.bytes, st));
      ctx->epoch = 1;
    }
    const unsigned gs = (unsigned)std::min(tiles_ub, (size_t)ctx->sms * occ_s);
    tm.begin(RADSORT_K_SCATTER);
    // (the parity-staged stage of R = 40 on a wide level would cost a CTA per SM: plain write-out there)
    constexpr size_t sm_tw = scatter_smem<R, TB_, SB_, DB, true>();
    auto* kfn_tw = k_scatter<R, K, TB_, SB_, MINB_, true, false, DB, true>;
    const bool tw = pre && scatter_tma(DB) && (((uintptr_t)recs | (uintptr_t)tmp) & 15u) == 0;  // bulk copies: 16-byte aligned
    if (tw) smem_attr(ctx, kfn_tw, sm_tw);
    if (tw && occupancy(ctx, kfn_tw, SB_, sm_tw) >= MINB_) {
      kfn_tw<<<gs, SB_, sm_tw, st>>>(L[cur], v.tile_start, n_large, v.segbase, v.status, ctx->epoch, v.ctl, recs, tmp,
                                     v.tile_pre, ch_first, carry_in, hist_grid, v.splitc, v.probes, v.tile_seg, nullptr);
    } else if (pre)
      k_scatter<R, K, TB_, SB_, MINB_, true, false, DB><<<gs, SB_, TB_ + SCATTER_PAD, st>>>(
          L[cur], v.tile_start, n_large, v.segbase, v.status, ctx->epoch, v.ctl, recs, tmp, v.tile_pre, ch_first,
          carry_in, hist_grid, v.splitc, v.probes, v.tile_seg);
    else if constexpr (DB == 8)
      k_scatter<R, K, TB_, SB_, MINB_, false><<<gs, SB_, TB_ + SCATTER_PAD, st>>>(
          L[cur], v.tile_start, n_large, v.segbase, v.status, ctx->epoch, v.ctl, recs, tmp, nullptr, nullptr, nullptr, 0,
          v.splitc, v.probes, v.tile_seg);
    tm.end();
    tm.begin(RADSORT_K_CHILDREN);
    k_children<R, K, DB><<<n_large, CHILD_B, CHILD_SCRATCH, st>>>(
        L[cur], v.hist, v.segbase, L[nxt], Lo[cur], cur, v.ctl, recs, tmp, v.probes,
        local_max() > C ? C + 1 : CL_MIN, local_max() > C ? local_max() : (cluster_ok ? ccap() : C), bitonic_max());
    tm.end();
    stats.kernel_launches[RADSORT_K_PLAN] += 2;
    stats.kernel_launches[RADSORT_K_HIST] += pre ? 2 : 1;  // k_hist_pre + k_carry
    stats.kernel_launches[RADSORT_K_SCATTER]++;
    stats.kernel_launches[RADSORT_K_CHILDREN]++;
    stats.scatter_passes++;
    return RADSORT_OK;
  }

  static radsort_status run(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, cudaStream_t st,
                            radsort_stats& stats, const Init* init = nullptr) {
    const char* e = getenv("RADSORT_SCATTER_CFG");
    const int cfg = e ? atoi(e) : 1;
    switch (cfg) {
      case 0: return run_cfg<65536, 512, 2>(ctx, recs, tmp, n, st, stats, init);
      case 2: return run_cfg<32768, 512, 2>(ctx, recs, tmp, n, st, stats, init);
      case 3: return run_cfg<16384, 256, 4>(ctx, recs, tmp, n, st, stats, init);
      case 4: return run_cfg<49152, 384, 3>(ctx, recs, tmp, n, st, stats, init);
      default: return run_cfg<32768, 256, 4>(ctx, recs, tmp, n, st, stats, init);  // measured best
    }
  }

  template <int TB, int SB, int MINB>
  static radsort_status run_cfg(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, cudaStream_t st,
                                radsort_stats& stats, const Init* init) {
    constexpr uint32_t T = tile_recs<R, TB, SB>();
    set_attrs(ctx);
    smem_attr(ctx, k_scatter<R, K, TB, SB, MINB, false>, TB + SCATTER_PAD);
    smem_attr(ctx, k_scatter<R, K, TB, SB, MINB, true>, TB + SCATTER_PAD);
    const bool pre = !(getenv("RADSORT_LOOKBACK") && getenv("RADSORT_LOOKBACK")[0] == '1');
    Views v;
    radsort_status rs = prepare(ctx, n, T, v, !pre, init ? init->nseg : 0u);
    if (rs) return rs;
    Seg** L = v.L;
    Seg** Lo = v.Lo;
    uint32_t* hist = v.hist;
    uint32_t* segbase = v.segbase;
    unsigned long long* andor = v.andor;
    uint32_t* tile_start = v.tile_start;
    unsigned long long* status = v.status;
    Ctl* ctl = v.ctl;
    const size_t tiles_max = v.tiles_max;

    // cluster-local sorting of bins of CL_MIN..ccap() records: on for R = 32, the
    // one layout where it beats a further radix level (measured);
    // RADSORT_CLUSTER=1 forces it on for every layout, =0 off
    const char* cl_env = getenv("RADSORT_CLUSTER");
    const bool cluster_ok = cl_env ? cl_env[0] == '1' : R == 32;
    int occ_s = 0, occ_h = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_scatter<R, K, TB, SB, MINB, false>, SB, TB + SCATTER_PAD);
    const char* hg = getenv("RADSORT_HIST_CTAS_PER_SM");
    const unsigned hist_grid = (unsigned)ctx->sms * (hg ? atoi(hg) : 4);  // chunks of the reduce-then-scan prefix
    uint32_t* tile_pre = v.tile_pre;                      // tiles x 256 u32 (its own buffer: never a stale status word)
    uint32_t* ch_first = (uint32_t*)ctx->mlo.p;
    uint32_t* ch_last = (uint32_t*)ctx->mhi.p;
    uint32_t* ch_tot = (uint32_t*)ctx->mlt.p;
    uint32_t* carry_in = (uint32_t*)ctx->mle.p;
    {
      radsort_status rs2;
      if ((rs2 = ensure(ctx->mlo, hist_grid * 4)) || (rs2 = ensure(ctx->mhi, hist_grid * 4)) ||
          (rs2 = ensure(ctx->mlt, (size_t)hist_grid * RADIX * 4)) || (rs2 = ensure(ctx->mle, (size_t)hist_grid * RADIX * 4)))
        return rs2;
      ch_first = (uint32_t*)ctx->mlo.p;
      ch_last = (uint32_t*)ctx->mhi.p;
      ch_tot = (uint32_t*)ctx->mlt.p;
      carry_in = (uint32_t*)ctx->mle.p;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_h, k_hist<R, K, T>, HIST_B, 0);
    occ_s = std::max(occ_s, 1);
    occ_h = std::max(occ_h, 1);
    // wide levels (10-bit digit): 4x the tile (128 KiB), one 1024-thread CTA per SM, a thread per digit.
    // RADSORT_WIDE=0 off, 1 the default rule, 2 forced wherever segments average >= 2 K records, 3 forced on
    // every level (consecutive wide levels: segments sharing 2 bits of their digit; tests only)
    // (built for the default 32 KiB x 256 tile configuration only)
    constexpr bool WIDE_BUILT = TB == 32768 && SB == 256;
    constexpr int TBW = 4 * TB, SBW = 1024;  // RADSORT_WIDE_CFG=1: one 1024-thread CTA per SM, a digit per thread
    constexpr int TBW2 = 2 * TB, SBW2 = 512;  // (default) two 512-thread CTAs per SM, two digits per thread
    constexpr uint32_t TW = tile_recs<R, TBW, SBW>(), TW2 = tile_recs<R, TBW2, SBW2>();
    const char* wc = getenv("RADSORT_WIDE_CFG");
    // measured: c4 (R = 32) wide scatter 13.75 (1) vs 13.13 ms (2); (16,8) 1 G 25.8 (1) vs 27.4 ms per sort (2: that
    // instance spills at its 64 registers), (16,16) 26.7 vs 28.4, (8,8) 2 G 36.0 vs 36.3
    const int wide_cfg = wc ? atoi(wc) : (R < 24 ? 1 : 2);
    const char* we = getenv("RADSORT_WIDE");
    const int wide_mode = WIDE_BUILT ? (we ? atoi(we) : 1) : 0;
    // The default rule applies to R >= 24, and to R < 24 where the sampled keys hardly repeat
    // (k_dupest; measured: (16,8) 1 G uniform 45.6 -> 27.2 ms, (8,8) 2 G 54.0 -> 35.6, but kmc
    // 27.7 -> 55.5 with ~100 copies per key).  RADSORT_WIDE_MIN_R=r: R >= r, no estimate.
    const char* wr = getenv("RADSORT_WIDE_MIN_R");
    const int wide_min_r = wr ? atoi(wr) : 24;
    constexpr uint32_t DUP_S = 1u << 18, DUP_SLOTS = 4 * DUP_S;
    const bool dup_run = !init && !wr && R < 24 && pre && wide_mode == 1 && (double)n > 256.0 * C &&
                         (size_t)n * R >= (size_t)DUP_SLOTS * 8 && ((uintptr_t)tmp & 7u) == 0;
    bool wide_small_ok = false;
    // p2 n < 1/4 (at least 4 hits: the estimate's noise floor)
    auto dup_few = [n](uint32_t hits) { return (double)hits <= std::max(4.0, (double)DUP_S * DUP_S / (8.0 * n)); };
    int occ_w = 1;
    if constexpr (WIDE_BUILT) if (pre && wide_mode) {
      smem_attr(ctx, k_scatter<R, K, TBW, SBW, 1, true, false, 10>, TBW + SCATTER_PAD);
      smem_attr(ctx, k_scatter<R, K, TBW2, SBW2, 2, true, false, 10>, TBW2 + SCATTER_PAD);
      smem_attr(ctx, k_children<R, K, 10>, CHILD_SCRATCH);
      radsort_status rs2;
      if ((rs2 = ensure(ctx->mlt, (size_t)hist_grid * 1024 * 4)) || (rs2 = ensure(ctx->mle, (size_t)hist_grid * 1024 * 4)))
        return rs2;
      ch_tot = (uint32_t*)ctx->mlt.p;
      carry_in = (uint32_t*)ctx->mle.p;
    }
    bool prev_wide = false;
    uint64_t level_recs = n;  // records of the level's Large list (the wide-level rule)

    Timer tm(ctx, st);
    const bool log = getenv("RADSORT_LOG") && getenv("RADSORT_LOG")[0] == '1';

    uint32_t n_large;
    if (init) {  // presegmented input: the bins go straight to the Large / Local lists
      std::vector<Seg> lg, lc;
      Ctl c0 = {};
      for (uint32_t i = 0; i < init->nseg && init->depth < (uint32_t)K; ++i) {
        if (init->len[i] < 2) continue;
        const Seg sg = {init->off[i], init->len[i], (uint8_t)init->depth, SRC_REC, MODE_NONE, 0, 0};
        if (init->len[i] > local_max()) {
          lg.push_back(sg);
        } else {
          lc.push_back(sg);
          c0.max_local_len[0] = std::max(c0.max_local_len[0], init->len[i]);
        }
      }
      c0.n_local[0] = (uint32_t)lc.size();
      c0.d0 = init->depth;
      if (!lg.empty()) RS_CUDA(cudaMemcpyAsync(L[0], lg.data(), lg.size() * sizeof(Seg), cudaMemcpyHostToDevice, st));
      if (!lc.empty()) RS_CUDA(cudaMemcpyAsync(Lo[0], lc.data(), lc.size() * sizeof(Seg), cudaMemcpyHostToDevice, st));
      RS_CUDA(cudaMemcpyAsync(ctl, &c0, sizeof(Ctl), cudaMemcpyHostToDevice, st));
      RS_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
      n_large = (uint32_t)lg.size();
      level_recs = 0;
      for (const Seg& g : lg) level_recs += g.len;
    } else {
      n_large = n > C ? 1u : 0u;
      if (n_large) {  // k_sample also writes the control block and the level-0 segment (k_init's Large case)
        tm.begin(RADSORT_K_SAMPLE);
        k_sample<R, K><<<1, 256, 0, st>>>(L[0], ctl, recs, n);
        if (dup_run) {  // after k_sample (it resets the control block); tmp is free until the level-0 scatter
          RS_CUDA(cudaMemsetAsync(tmp, 0, (size_t)DUP_SLOTS * 8, st));
          k_dupest<R, K><<<DUP_S / 256, 256, 0, st>>>(ctl, recs, n, DUP_S, (unsigned long long*)tmp, DUP_SLOTS - 1);
          stats.kernel_launches[RADSORT_K_SAMPLE]++;
        }
        tm.end();
        if (dup_run && (double)n <= 0.95 * 1024.0 * C) {
          // level 0 itself is in the rule's window (one 10-bit pass + the local sort instead of
          // two 8-bit passes): the estimate is needed now, at the price of one more host sync
          RS_CUDA(cudaMemcpyAsync(ctx->h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
          RS_CUDA(cudaStreamSynchronize(st));
          wide_small_ok = dup_few(ctx->h_ctl->dup_est);
        }
        stats.kernel_launches[RADSORT_K_SAMPLE]++;
      } else {
        k_init<<<1, 1, 0, st>>>(L[0], Lo[0], ctl, n, C);
      }
    }
    int cur = 0;
    bool ctl_fresh = false;  // h_ctl equals the device control block (no kernel since its read)
    const int max_levels = 2 * K + 4;
    static const char* level_names[] = {"radsort level 0", "radsort level 1", "radsort level 2", "radsort level 3",
                                        "radsort level 4", "radsort level 5", "radsort level 6", "radsort level 7",
                                        "radsort level 8+"};
    for (int level = 0;; ++level) {
      NvtxRange nvtx_level(level_names[level < 8 ? level : 8]);
      if (level > max_levels) {
        set_detail("MSD level loop did not terminate (%d levels)", level);
        return RADSORT_ERR_CUDA;
      }
      const int nxt = cur ^ 1;
      if (n_large) {
        // wide level: one 10-bit pass instead of an 8-bit one where
        // the 8-bit children would be too big for the CTA-local sort but the
        // 10-bit ones fit it (saves a radix level / the cluster sort).  Default for
        // R >= 24 only: for R = 8 / 16 the 10-bit pass costs more than it saves
        // (c5 16.6 -> 17.5, c2 5.3 -> 5.9 ms) and duplicate-heavy bins near C make
        // the local sort slow (kmc 27.8 -> 55.6 ms; measured)
        bool wide = false;
        if (pre && wide_mode && (!prev_wide || wide_mode == 3)) {
          const double avg = (double)level_recs / n_large;
          wide = wide_mode == 3 ? avg >= 64.0
                                : (wide_mode == 2 ? avg >= 2048.0
                                                  : ((R >= wide_min_r || wide_small_ok) && avg > 256.0 * C && avg <= 0.95 * 1024.0 * C));
        }
        if (wide) {  // the workspace is sized for 8-bit levels: grow it where a wide level needs more
          // (between levels: the previous level's histograms, bases and tile prefixes are dead)
          radsort_status rs2;
          if ((rs2 = ensure(ctx->hist, (size_t)n_large * 1024 * 4)) || (rs2 = ensure(ctx->segbase, (size_t)n_large * 1024 * 4)) ||
              (rs2 = ensure(ctx->tile_pre, ((size_t)n / std::min(TW, TW2) + n_large + 1) * 1024 * 4)))
            return rs2;
          v.hist = (uint32_t*)ctx->hist.p;
          v.segbase = (uint32_t*)ctx->segbase.p;
          v.tile_pre = (uint32_t*)ctx->tile_pre.p;
        }
        radsort_status lrs = RADSORT_OK;
        if constexpr (WIDE_BUILT) {
          if (wide && wide_cfg == 2)
            lrs = level_pass<TW2, TBW2, SBW2, 2, 10>(ctx, v, n, n_large, cur, nxt, recs, tmp, st, tm, stats, hist_grid,
                                                     2, ch_first, ch_last, ch_tot, carry_in, cluster_ok);
          else if (wide)
            lrs = level_pass<TW, TBW, SBW, 1, 10>(ctx, v, n, n_large, cur, nxt, recs, tmp, st, tm, stats, hist_grid,
                                                  occ_w, ch_first, ch_last, ch_tot, carry_in, cluster_ok);
        }
        if (!wide)
          lrs = level_pass<T, TB, SB, MINB, 8>(ctx, v, n, n_large, cur, nxt, recs, tmp, st, tm, stats, hist_grid, occ_s,
                                               ch_first, ch_last, ch_tot, carry_in, cluster_ok, pre, occ_h);
        if (lrs) return lrs;
        prev_wide = wide;
        stats.wide_levels += wide ? 1 : 0;
      } else {
        k_prep<<<1, 1024, 0, st>>>(L[cur], 0, T, tile_start, ctl, nxt);
        stats.kernel_launches[RADSORT_K_PLAN]++;
      }
      RS_CUDA(cudaGetLastError());
      if (ctl_fresh && !n_large && level > 0) {
        // nothing but this k_prep ran since the last control-block read (the previous
        // level had Large segments only): mirror k_prep's reset on the host copy
        // instead of a D2H + host sync (one sync less per sort: c1 is sync-bound)
        Ctl& h = *ctx->h_ctl;
        h.tiles_total = h.scatter_ticket = h.n_large_next = 0;
        h.rec_large_next = 0;
        h.n_local[nxt] = h.n_local_small[nxt] = h.n_local_med[nxt] = h.max_local_len[nxt] = 0;
      } else {
        RS_CUDA(cudaMemcpyAsync(ctx->h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaStreamSynchronize(st));
      }
      Ctl c = *ctx->h_ctl;
      if (level == 0) stats.first_digit = c.d0;
      if (level == 0 && dup_run) {
        wide_small_ok = dup_few(c.dup_est);
        if (log) fprintf(stderr, "[radsort] duplicate estimate: %u of %u sampled keys repeat: wide levels %s\n",
                         c.dup_est, DUP_S, wide_small_ok ? "on" : "off");
      }
      const uint32_t nloc = c.n_local[cur];
      if (log)
        fprintf(stderr, "[radsort] level %d%s: large=%u tiles=%u -> large_next=%u local=%u (max %u)\n", level,
                prev_wide && n_large ? " (wide)" : "", n_large, c.tiles_total, c.n_large_next, nloc,
                c.max_local_len[cur]);
      if (nloc) {
        tm.begin(RADSORT_K_LOCAL);
        int nl = 1;
        const bool cl = launch_local(ctx, nloc, c.max_local_len[cur], Lo[cur], Lo[nxt], nxt, L[nxt], ctl, recs, tmp,
                                     st, c.n_local_small[cur], c.n_local_med[cur], nl);
        tm.end();
        stats.kernel_launches[RADSORT_K_LOCAL] += nl;
        RS_CUDA(cudaGetLastError());
        if (cl) {  // the cluster sort may have handed bins back as Large bins of the next level
          RS_CUDA(cudaMemcpyAsync(ctx->h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
          RS_CUDA(cudaStreamSynchronize(st));
          c.n_large_next = ctx->h_ctl->n_large_next;
          c.rec_large_next = ctx->h_ctl->rec_large_next;
        }
      }
      stats.levels = level + 1;
      if (log && tm.on) {  // per-level kernel times (radsort_set_timing(1) + RADSORT_LOG=1)
        float before[RADSORT_K_COUNT];
        for (int q = 0; q < RADSORT_K_COUNT; ++q) before[q] = stats.kernel_ms[q];
        tm.flush(stats);
        fprintf(stderr, "[radsort] level %d ms: hist %.3f scatter %.3f children %.3f local %.3f\n", level,
                stats.kernel_ms[RADSORT_K_HIST] - before[RADSORT_K_HIST],
                stats.kernel_ms[RADSORT_K_SCATTER] - before[RADSORT_K_SCATTER],
                stats.kernel_ms[RADSORT_K_CHILDREN] - before[RADSORT_K_CHILDREN],
                stats.kernel_ms[RADSORT_K_LOCAL] - before[RADSORT_K_LOCAL]);
      }
      tm.flush(stats);
      if (c.n_large_next == 0 && nloc == 0 && n_large == 0) break;
      ctl_fresh = nloc == 0;  // no kernel launched since h_ctl was read
      n_large = c.n_large_next;
      level_recs = c.rec_large_next;
      cur = nxt;
    }
    // final statistics: the loop leaves only after a control-block read with no
    // kernel launched since (nloc == 0 at the last level), so h_ctl is current
    // (saves a D2H + host sync per sort: c1 is sync-bound)
    const Ctl c = *ctx->h_ctl;
#ifdef RADSORT_PHASE_PROF
    if (log) {
      for (int q = 0; q < 16; ++q) fprintf(stderr, "[radsort prof] %s%d %llu\n", q < 8 ? "scatter" : "local", q & 7, (unsigned long long)c.prof[q]);
    }
#endif
    stats.records_scattered = c.rec_scatter;
    stats.records_hist = c.rec_hist;
    stats.records_local = c.rec_local;
    stats.records_tiny = c.rec_tiny;
    stats.records_copied = c.rec_copy;
    stats.bins_large = c.bins_large;
    stats.bins_local = c.bins_local;
    stats.bins_tiny = c.bins_tiny;
    stats.bins_final = c.bins_final;
    stats.bins_split = c.bins_split;
    stats.records_split = c.rec_split;
    stats.kernel_bytes[RADSORT_K_HIST] = c.rec_hist * R;
    stats.kernel_bytes[RADSORT_K_SCATTER] = 2ull * c.rec_scatter * R;
    stats.kernel_bytes[RADSORT_K_LOCAL] = 2ull * c.rec_local * R;
    stats.kernel_bytes[RADSORT_K_CHILDREN] = 2ull * c.rec_tiny * R;
    return RADSORT_OK;
  }
};


// ---------------------------------------------- NEXT-1: key + index sort
// For records much wider than their key (PAPER.md:166-169
// §3.3: with long records the record moves dominate, so move them once): sort
// (key, 32-bit index) records of KI = 16 (K = 8) or 24 (K = 16) bytes with the
// same MSD radix sort, then move every full record once, by a gather.
//   k_ki_build : records -> a copy in tmp, and (key, i) into the workspace
//   radix sort of the (key, index) records (layout (KI, K), tmp half as scratch)
//   k_ki_gather: records[j] = copy[index of the j-th sorted pair]
// The workspace holds 2 n KI bytes (the pairs and the radix sort's scratch).
template <int R, int K, int KI>
__global__ void __launch_bounds__(256) k_ki_build(const uint8_t* __restrict__ recs, uint8_t* __restrict__ copy,
                                                  uint8_t* __restrict__ ki, uint32_t n) {
  constexpr int U = 4;  // records in flight per thread
  const uint32_t stride = gridDim.x * 256u * U;
  for (uint32_t b = blockIdx.x * 256u * U; b < n; b += stride) {
    Rec<R> r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = b + u * 256u + threadIdx.x;
      if (i < n) r[u] = ldg_wide<R>(recs + (size_t)i * R);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = b + u * 256u + threadIdx.x;
      if (i < n) {
        stg_rec<R>(copy + (size_t)i * R, r[u]);
        const Key<K> k = key_of<R, K>(r[u]);
        uint8_t* q = ki + (size_t)i * KI;
        if constexpr (KI == 16) {
          *reinterpret_cast<uint4*>(q) = make_uint4((uint32_t)k.w0, (uint32_t)(k.w0 >> 32), i, 0u);
        } else {
          uint2* q2 = reinterpret_cast<uint2*>(q);
          q2[0] = make_uint2((uint32_t)k.w0, (uint32_t)(k.w0 >> 32));
          q2[1] = make_uint2((uint32_t)k.w1, (uint32_t)(k.w1 >> 32));
          q2[2] = make_uint2(i, 0u);
        }
      }
    }
  }
}

template <int R, int K, int KI>
__global__ void __launch_bounds__(256) k_ki_gather(const uint8_t* __restrict__ ki, const uint8_t* __restrict__ copy,
                                                   uint8_t* __restrict__ recs, uint32_t n) {
  constexpr int U = 8;  // independent random reads in flight per thread
  const uint32_t stride = gridDim.x * 256u * U;
  for (uint32_t b = blockIdx.x * 256u * U; b < n; b += stride) {
    uint32_t src[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = b + u * 256u + threadIdx.x;
      src[u] = j < n ? __ldg(reinterpret_cast<const uint32_t*>(ki + (size_t)j * KI + K)) : 0u;
    }
    Rec<R> r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = b + u * 256u + threadIdx.x;
      if (j < n) r[u] = ldg_wide<R>(copy + (size_t)src[u] * R);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = b + u * 256u + threadIdx.x;
      if (j < n) stg_rec<R>(recs + (size_t)j * R, r[u]);
    }
  }
}

template <int R, int K>
struct KeyIndex {
  static constexpr bool BUILT = (R == 32 && K == 8) || (R == 40 && K == 16);
  static constexpr int KI = K == 8 ? 16 : 24;
  // RADSORT_KEY_INDEX=1/0 forces it on/off; default: on where it was measured faster
  static bool on() {
    if constexpr (!BUILT) return false;
    const char* e = getenv("RADSORT_KEY_INDEX");
    return e ? e[0] == '1' : KI_DEFAULT;
  }
  // measured slower on B200 (profiles/r02_key_index_bench.jsonl: (32,8) 1 G 91.4 vs 67.0 ms,
  // (40,16) 500 M 76.3 vs 69.5 ms -- the random 32/40-byte gather runs at a fraction of the
  // sequential HBM rate): opt-in
  static constexpr bool KI_DEFAULT = false;
  static radsort_status run(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, cudaStream_t st,
                            radsort_stats& s) {
    if constexpr (BUILT) {
      radsort_status rs;
      if ((rs = ensure(ctx->kiw, (size_t)2 * n * KI))) return rs;
      uint8_t* ki = (uint8_t*)ctx->kiw.p;
      const unsigned g = (unsigned)std::max<size_t>(1, std::min<size_t>(((size_t)n + 1023) / 1024, (size_t)ctx->sms * 8));
      Timer tm(ctx, st);
      tm.begin(RADSORT_K_GATHER);
      k_ki_build<R, K, KI><<<g, 256, 0, st>>>(recs, tmp, ki, n);
      tm.end();
      RS_CUDA(cudaGetLastError());
      tm.flush(s);
      if ((rs = run_layout<KI, K>(ctx, ki, ki + (size_t)n * KI, n, st, s))) return rs;
      const unsigned gg = (unsigned)std::max<size_t>(1, std::min<size_t>(((size_t)n + 2047) / 2048, (size_t)ctx->sms * 8));
      tm.begin(RADSORT_K_GATHER);
      k_ki_gather<R, K, KI><<<gg, 256, 0, st>>>(ki, tmp, recs, n);
      tm.end();
      RS_CUDA(cudaGetLastError());
      tm.flush(s);
      s.kernel_launches[RADSORT_K_GATHER] += 2;
      s.kernel_bytes[RADSORT_K_GATHER] += (uint64_t)n * (2 * R + KI) + (uint64_t)n * (KI + 2 * R);
      s.key_index = 1;
      s.rec_size = R;
    }
    return RADSORT_OK;
  }
};

template <int R, int K>
radsort_status run_layout(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, cudaStream_t st, radsort_stats& s) {
  if constexpr (KeyIndex<R, K>::BUILT) {
    if (KeyIndex<R, K>::on() && n > Sorter<R, K>::C) return KeyIndex<R, K>::run(ctx, recs, tmp, n, st, s);
  }
  workspace_acquire(ctx, st);
  const radsort_status rs = Sorter<R, K>::run(ctx, recs, tmp, n, st, s);
  workspace_release(ctx, st);
  return rs;
}

// The same sort started from bins that already share their first `depth`
// digits (the multi-GPU receive side: data arrives grouped by its top digit).
template <int R, int K>
radsort_status run_layout_segs(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, const uint32_t* off,
                               const uint32_t* len, uint32_t nseg, uint32_t depth, cudaStream_t st, radsort_stats& s) {
  workspace_acquire(ctx, st);
  const typename Sorter<R, K>::Init init = {off, len, nseg, depth};
  const radsort_status rs = Sorter<R, K>::run(ctx, recs, tmp, n, st, s, &init);
  workspace_release(ctx, st);
  return rs;
}

// ------------------------------------------------ multi-GPU building blocks
constexpr int MULTI_TB = 65536, MULTI_SB = 512, MULTI_MINB = 2;

template <int R, int K>
radsort_status multi_hist(Context* ctx, const uint8_t* recs, uint32_t n, uint32_t digit, cudaStream_t st,
                          uint64_t* h256, uint64_t* andor4) {
  using S = Sorter<R, K>;
  constexpr uint32_t T = tile_recs<R, MULTI_TB, MULTI_SB>();
  workspace_acquire(ctx, st);
  typename S::Views v;
  radsort_status rs = S::prepare(ctx, n > 0 ? n : 1, T, v);
  if (rs) return rs;
  const Seg sg = {0u, n, (uint8_t)digit, SRC_REC, MODE_NONE, 0, 0};
  RS_CUDA(cudaMemcpyAsync(v.L[0], &sg, sizeof(Seg), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemsetAsync(v.hist, 0, RADIX * sizeof(uint32_t), st));
  RS_CUDA(cudaMemsetAsync(v.andor, 0, 4 * sizeof(unsigned long long), st));
  RS_CUDA(cudaMemsetAsync(v.ctl, 0, sizeof(Ctl), st));
  k_prep<<<1, 1024, 0, st>>>(v.L[0], 1, T, v.tile_start, v.ctl, 1);
  int occ_h = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_h, k_hist<R, K, T>, HIST_B, 0);
  const unsigned gh = (unsigned)std::max<size_t>(1, std::min<size_t>((size_t)n / T + 1, (size_t)ctx->sms * occ_h));
  k_hist<R, K, T><<<gh, HIST_B, 0, st>>>(v.L[0], v.tile_start, 1, v.ctl, v.hist, v.andor, (const uint8_t*)recs,
                                                 (const uint8_t*)recs);
  uint32_t h32[RADIX];
  RS_CUDA(cudaMemcpyAsync(h32, v.hist, sizeof h32, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaMemcpyAsync(andor4, v.andor, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < RADIX; ++b) h256[b] = h32[b];
  workspace_release(ctx, st);
  return RADSORT_OK;
}

template <int R, int K>
radsort_status multi_scatter(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, uint32_t digit, const uint64_t* h256,
                             cudaStream_t st) {
  using S = Sorter<R, K>;
  constexpr uint32_t T = tile_recs<R, MULTI_TB, MULTI_SB>();
  if (n == 0) return RADSORT_OK;
  workspace_acquire(ctx, st);
  typename S::Views v;
  radsort_status rs = S::prepare(ctx, n, T, v, true);
  if (rs) return rs;
  smem_attr(ctx, k_scatter<R, K, MULTI_TB, MULTI_SB, MULTI_MINB, false>, MULTI_TB + SCATTER_PAD);
  const Seg sg = {0u, n, (uint8_t)digit, SRC_REC, MODE_NONE, 0, 0};
  uint32_t h32[RADIX];
  for (int b = 0; b < RADIX; ++b) h32[b] = (uint32_t)h256[b];
  RS_CUDA(cudaMemcpyAsync(v.L[0], &sg, sizeof(Seg), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(v.hist, h32, sizeof h32, cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemsetAsync(v.ctl, 0, sizeof(Ctl), st));
  k_prep<<<1, 1024, 0, st>>>(v.L[0], 1, T, v.tile_start, v.ctl, 1);
  k_plan<R, K><<<1, RADIX, 0, st>>>(v.L[0], v.hist, v.andor, v.segbase, v.L[1], v.ctl, v.splitc, 0, 1);
  if (++ctx->epoch >= 65536) {
    RS_CUDA(cudaMemsetAsync(v.status, 0, ctx->status.bytes, st));
    ctx->epoch = 1;
  }
  int occ_s = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_scatter<R, K, MULTI_TB, MULTI_SB, MULTI_MINB, false>,
                                                MULTI_SB, MULTI_TB + SCATTER_PAD);
  const unsigned gs = (unsigned)std::max<size_t>(1, std::min<size_t>((size_t)n / T + 1, (size_t)ctx->sms * occ_s));
  k_scatter<R, K, MULTI_TB, MULTI_SB, MULTI_MINB, false><<<gs, MULTI_SB, MULTI_TB + SCATTER_PAD, st>>>(
      v.L[0], v.tile_start, 1, v.segbase, v.status, ctx->epoch, v.ctl, recs, tmp, nullptr, nullptr, nullptr, 0,
      v.splitc, v.probes, nullptr);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaStreamSynchronize(st));
  workspace_release(ctx, st);
  return RADSORT_OK;
}

// Fused exchange (multi-GPU, SURVEY.md §8(e) k_merge_scatter + §8(f) NEXT-3):
// the sender's level-0 buckets, cut into pieces by destination rank, are
// histogrammed by the next digit (multi_piece_hist) and then scattered by that
// digit straight into the destination ranks' record buffers (multi_piece_scatter,
// k_scatter<PEER>: remote stores over NVLink), at offsets the host derives
// from every rank's piece histograms.  The per-call workspace keeps the
// reduce-then-scan tile prefixes between the two calls, so other users of the
// context (loopback ranks sharing the device) cannot clobber them.
constexpr int PIECE_TB = 32768, PIECE_SB = 256, PIECE_MINB = 4;

template <int R, int K>
radsort_status multi_piece_hist(Context* ctx, PieceWs& w, const uint8_t* src, const uint32_t* off,
                                const uint32_t* len, uint32_t np, uint32_t digit, cudaStream_t st, uint32_t* h_hist) {
  constexpr uint32_t T = tile_recs<R, PIECE_TB, PIECE_SB>();
  w.np = np;
  if (np == 0) return RADSORT_OK;
  size_t tiles = 0;
  std::vector<Seg> segs(np);
  for (uint32_t i = 0; i < np; ++i) {
    segs[i] = {off[i], len[i], (uint8_t)digit, SRC_TMP, MODE_SCATTER, 0, 0};
    tiles += (len[i] + T - 1) / T;
  }
  w.hist_grid = (uint32_t)ctx->sms * 4;
  w.tiles = tiles;
  radsort_status rs;
  if ((rs = ensure(w.segs, np * sizeof(Seg))) || (rs = ensure(w.tile_start, (np + 1) * 4)) ||
      (rs = ensure(w.tile_seg, (tiles + 1) * 4)) || (rs = ensure(w.hist, (size_t)np * RADIX * 4)) ||
      (rs = ensure(w.andor, (size_t)np * 8 * 8)) || (rs = ensure(w.tile_pre, (tiles + 1) * RADIX * 4)) ||
      (rs = ensure(w.ch_first, w.hist_grid * 4)) || (rs = ensure(w.ch_last, w.hist_grid * 4)) ||
      (rs = ensure(w.ch_tot, (size_t)w.hist_grid * RADIX * 4)) ||
      (rs = ensure(w.carry_in, (size_t)w.hist_grid * RADIX * 4)) || (rs = ensure(w.ctl, sizeof(Ctl))) ||
      (rs = ensure(w.segbase, (size_t)np * RADIX * 4)) || (rs = ensure(w.dst, (size_t)np * 8)))
    return rs;
  Seg* dsegs = (Seg*)w.segs.p;
  Ctl* ctl = (Ctl*)w.ctl.p;
  RS_CUDA(cudaMemcpyAsync(dsegs, segs.data(), np * sizeof(Seg), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
  RS_CUDA(cudaMemsetAsync(w.hist.p, 0, (size_t)np * RADIX * 4, st));
  RS_CUDA(cudaMemsetAsync(w.andor.p, 0, (size_t)np * 8 * 8, st));
  k_prep<<<1, 1024, 0, st>>>(dsegs, np, T, (uint32_t*)w.tile_start.p, ctl, 1);
  k_tilemap<<<(unsigned)std::max<size_t>(1, std::min<size_t>((tiles + 255) / 256, (size_t)ctx->sms * 16)), 256, 0, st>>>(
      (const uint32_t*)w.tile_start.p, np, ctl, (uint32_t*)w.tile_seg.p);
  k_hist_pre<R, K, T><<<w.hist_grid, HIST_B, 0, st>>>(
      dsegs, (const uint32_t*)w.tile_start.p, np, ctl, (uint32_t*)w.hist.p, (unsigned long long*)w.andor.p, src, src,
      (uint32_t*)w.tile_pre.p, (uint32_t*)w.ch_first.p, (uint32_t*)w.ch_last.p, (uint32_t*)w.ch_tot.p,
      (const uint32_t*)w.tile_seg.p);
  k_carry<RADIX><<<1, RADIX, 0, st>>>((const uint32_t*)w.ch_first.p, (const uint32_t*)w.ch_last.p,
                               (const uint32_t*)w.ch_tot.p, w.hist_grid, (uint32_t*)w.carry_in.p);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpyAsync(h_hist, w.hist.p, (size_t)np * RADIX * 4, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  return RADSORT_OK;
}

// h_base[i * 256 + v]: record offset, in the buffer at h_dst[i], of the first
// record of piece i with digit v (this sender's share of that bin).
template <int R, int K>
radsort_status multi_piece_scatter(Context* ctx, PieceWs& w, const uint8_t* src, const uint32_t* h_base,
                                   const uint64_t* h_dst, cudaStream_t st) {
  const uint32_t np = w.np;
  if (np == 0) return RADSORT_OK;
  auto* kfn = k_scatter<R, K, PIECE_TB, PIECE_SB, PIECE_MINB, true, true>;
  smem_attr(ctx, kfn, PIECE_TB + SCATTER_PAD);
  RS_CUDA(cudaMemcpyAsync(w.segbase.p, h_base, (size_t)np * RADIX * 4, cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(w.dst.p, h_dst, (size_t)np * 8, cudaMemcpyHostToDevice, st));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, PIECE_SB, PIECE_TB + SCATTER_PAD);
  const unsigned gs = (unsigned)std::max<size_t>(1, std::min(w.tiles, (size_t)ctx->sms * std::max(occ, 1)));
  kfn<<<gs, PIECE_SB, PIECE_TB + SCATTER_PAD, st>>>(
      (const Seg*)w.segs.p, (const uint32_t*)w.tile_start.p, np, (const uint32_t*)w.segbase.p, nullptr, 0,
      (Ctl*)w.ctl.p, const_cast<uint8_t*>(src), const_cast<uint8_t*>(src), (const uint32_t*)w.tile_pre.p,
      (const uint32_t*)w.ch_first.p, (const uint32_t*)w.carry_in.p, w.hist_grid, nullptr, nullptr,
      (const uint32_t*)w.tile_seg.p, (const unsigned long long*)w.dst.p);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaStreamSynchronize(st));
  return RADSORT_OK;
}

template <int R, int K>
radsort_status multi_bounds(Context* ctx, const uint8_t* buf, const uint32_t* lo, const uint32_t* hi,
                            const uint64_t* probes, uint32_t M, cudaStream_t st, uint64_t* lt, uint64_t* le) {
  if (M == 0) return RADSORT_OK;
  radsort_status rs;
  if ((rs = ensure(ctx->mprobe, (size_t)M * 16))) return rs;
  if ((rs = ensure(ctx->mlo, (size_t)M * 4))) return rs;
  if ((rs = ensure(ctx->mhi, (size_t)M * 4))) return rs;
  if ((rs = ensure(ctx->mlt, (size_t)M * 8))) return rs;
  if ((rs = ensure(ctx->mle, (size_t)M * 8))) return rs;
  RS_CUDA(cudaMemcpyAsync(ctx->mprobe.p, probes, (size_t)M * 16, cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(ctx->mlo.p, lo, (size_t)M * 4, cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(ctx->mhi.p, hi, (size_t)M * 4, cudaMemcpyHostToDevice, st));
  k_bounds<R, K><<<(M + 255) / 256, 256, 0, st>>>(buf, (const uint32_t*)ctx->mlo.p, (const uint32_t*)ctx->mhi.p,
                                                  (const unsigned long long*)ctx->mprobe.p, M,
                                                  (unsigned long long*)ctx->mlt.p, (unsigned long long*)ctx->mle.p);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpyAsync(lt, ctx->mlt.p, (size_t)M * 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaMemcpyAsync(le, ctx->mle.p, (size_t)M * 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  return RADSORT_OK;
}

}  // namespace radsort
