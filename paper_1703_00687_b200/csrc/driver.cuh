// radsort host-side shared declarations (context, workspace, timing, errors).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (ranges show in nsys / ncu when a tool is attached)

#include "../../include/radsort.h"
#include "passes.cuh"
#include "local2.cuh"
#include "local_pipe.cuh"

namespace radsort {

void set_detail(const char* fmt, ...);
extern bool g_timing;

#define RS_CUDA(x)                                                                 \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      ::radsort::set_detail("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return RADSORT_ERR_CUDA;                                                     \
    }                                                                              \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Context {
  int device = -1;
  int sms = 148;
  std::mutex mu;
  // workspace
  DevBuf large[2], local[2], hist, andor, segbase, tile_start, status, ctl, host_io[2];
  DevBuf splitc, probes;  // dominant-key split: per-segment class cursors; keys of the bins to fill
  DevBuf tile_seg;        // tile -> segment map of the current level
  DevBuf tile_pre;        // reduce-then-scan per-tile digit prefixes (never aliases `status`)
  // per-device launch state: kernels whose dynamic-smem attribute is set on this
  // device, and the max active clusters of each cluster kernel on this device
  std::set<const void*> smem_attr_set;
  std::map<const void*, int> max_clusters;
  std::map<const void*, int> occupancy;  // resident CTAs per SM of a kernel at its launch shape
  Ctl* h_ctl = nullptr;  // pinned
  uint32_t epoch = 0;
  cudaEvent_t ev[2 * 64] = {};
  bool ev_init = false;
  cudaEvent_t done_ev = nullptr;  // workspace free once this event (last sort's stream) completes
  bool done_valid = false;
  DevBuf mprobe, mlo, mhi, mlt, mle;  // multi-GPU splitter search scratch
  std::map<std::string, void*> ipc_open;  // peer buffers opened by CUDA IPC (handle bytes -> mapped base)
  DevBuf kiw;                             // key + index sort: the (key, index) records and their scratch
};

// Order `st` after the previous user of the workspace (another stream may still
// be running the tail of the last sort), and mark the end of this use.
inline void workspace_acquire(Context* ctx, cudaStream_t st) {
  if (ctx->done_valid) cudaStreamWaitEvent(st, ctx->done_ev, 0);
}
inline void workspace_release(Context* ctx, cudaStream_t st) {
  cudaEventRecord(ctx->done_ev, st);
  ctx->done_valid = true;
}

radsort_status ensure(DevBuf& b, size_t bytes, bool zero = false);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device
// (the attribute is per device; the context is per device and its mutex is
// held by every sort).
template <class F>
inline void smem_attr(Context* ctx, F* f, int bytes) {
  if (ctx->smem_attr_set.insert((const void*)f).second)
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// resident CTAs per SM of kernel f at (threads, dynamic smem), cached per device
template <class F>
inline int occupancy(Context* ctx, F* f, int threads, size_t smem) {
  auto it = ctx->occupancy.find((const void*)f);
  if (it != ctx->occupancy.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, threads, smem) != cudaSuccess) occ = 0;
  ctx->occupancy[(const void*)f] = occ;
  return occ;
}

// NVTX range for the host-side phases (the MSD level, the multi-GPU steps)
struct NvtxRange {
  explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
inline const char* kernel_class_name(int k) {
  static const char* names[RADSORT_K_COUNT] = {"radsort sample", "radsort hist",  "radsort plan",   "radsort scatter",
                                               "radsort children", "radsort local", "radsort multi", "radsort gather"};
  return (k >= 0 && k < RADSORT_K_COUNT) ? names[k] : "radsort";
}

// per-kernel-class CUDA-event timing on the sort's stream (radsort_set_timing),
// and an NVTX range per kernel class
struct Timer {
  Context* ctx;
  cudaStream_t st;
  int n = 0;
  int cls[64];
  bool on;
  Timer(Context* c, cudaStream_t s) : ctx(c), st(s), on(g_timing) {}
  void begin(int k) {
    nvtxRangePushA(kernel_class_name(k));
    if (!on || n >= 64) return;
    cls[n] = k;
    cudaEventRecord(ctx->ev[2 * n], st);
  }
  void end() {
    nvtxRangePop();
    if (!on || n >= 64) return;
    cudaEventRecord(ctx->ev[2 * n + 1], st);
    ++n;
  }
  void flush(radsort_stats& s) {
    if (!on || n == 0) return;
    cudaStreamSynchronize(st);
    for (int i = 0; i < n; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ctx->ev[2 * i], ctx->ev[2 * i + 1]);
      s.kernel_ms[cls[i]] += ms;
    }
    n = 0;
  }
};

// One instantiation per built record layout (layout_R_K.cu).
template <int R, int K>
radsort_status run_layout(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, cudaStream_t st, radsort_stats& s);

// Multi-GPU building blocks (same instantiation units).  All are synchronous
// on `st` (they return host results) and use the context workspace.
// multi_hist: histogram of `digit` over recs[0,n) (h256) and the AND/OR of all
//   keys (andor4 = {~AND w0, ~AND w1, OR w0, OR w1}).
// multi_scatter: one counting-scatter pass of recs[0,n) by `digit` into tmp;
//   bucket b lands at [sum_{u<b} h[u], ...); h256 = multi_hist's histogram.
// multi_bounds: for M probes, #keys < probe and <= probe in sorted [lo, hi).
template <int R, int K>
radsort_status multi_hist(Context* ctx, const uint8_t* recs, uint32_t n, uint32_t digit, cudaStream_t st,
                          uint64_t* h256, uint64_t* andor4);
template <int R, int K>
radsort_status multi_scatter(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, uint32_t digit, const uint64_t* h256,
                             cudaStream_t st);
template <int R, int K>
radsort_status multi_bounds(Context* ctx, const uint8_t* buf, const uint32_t* lo, const uint32_t* hi,
                            const uint64_t* probes, uint32_t M, cudaStream_t st, uint64_t* lt, uint64_t* le);

// Per-call workspace of the fused exchange (multi_piece_hist -> multi_piece_scatter).
struct PieceWs {
  DevBuf segs, tile_start, tile_seg, hist, andor, tile_pre, ch_first, ch_last, ch_tot, carry_in, ctl, segbase, dst;
  uint32_t np = 0, hist_grid = 0;
  size_t tiles = 0;
  ~PieceWs() {
    DevBuf* b[] = {&segs, &tile_start, &tile_seg, &hist, &andor, &tile_pre, &ch_first,
                   &ch_last, &ch_tot, &carry_in, &ctl, &segbase, &dst};
    for (DevBuf* x : b)
      if (x->p) cudaFree(x->p);
  }
};
template <int R, int K>
radsort_status multi_piece_hist(Context* ctx, PieceWs& w, const uint8_t* src, const uint32_t* off,
                                const uint32_t* len, uint32_t np, uint32_t digit, cudaStream_t st, uint32_t* h_hist);
template <int R, int K>
radsort_status multi_piece_scatter(Context* ctx, PieceWs& w, const uint8_t* src, const uint32_t* h_base,
                                   const uint64_t* h_dst, cudaStream_t st);

template <int R, int K>
radsort_status run_layout_segs(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, const uint32_t* off,
                               const uint32_t* len, uint32_t nseg, uint32_t depth, cudaStream_t st, radsort_stats& s);

struct LayoutOps {
  radsort_status (*sort)(Context*, uint8_t*, uint8_t*, uint32_t, cudaStream_t, radsort_stats&);
  radsort_status (*sort_segs)(Context*, uint8_t*, uint8_t*, uint32_t, const uint32_t*, const uint32_t*, uint32_t,
                              uint32_t, cudaStream_t, radsort_stats&);
  radsort_status (*hist)(Context*, const uint8_t*, uint32_t, uint32_t, cudaStream_t, uint64_t*, uint64_t*);
  radsort_status (*scatter)(Context*, uint8_t*, uint8_t*, uint32_t, uint32_t, const uint64_t*, cudaStream_t);
  radsort_status (*bounds)(Context*, const uint8_t*, const uint32_t*, const uint32_t*, const uint64_t*, uint32_t,
                           cudaStream_t, uint64_t*, uint64_t*);
  radsort_status (*piece_hist)(Context*, PieceWs&, const uint8_t*, const uint32_t*, const uint32_t*, uint32_t, uint32_t,
                               cudaStream_t, uint32_t*);
  radsort_status (*piece_scatter)(Context*, PieceWs&, const uint8_t*, const uint32_t*, const uint64_t*, cudaStream_t);
};
// nullptr for layouts that are not built
const LayoutOps* layout_ops(uint32_t R, uint32_t K);
Context* get_or_create_ctx(int device);

}  // namespace radsort
