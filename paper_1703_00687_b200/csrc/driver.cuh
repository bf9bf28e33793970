// radsort host-side shared declarations (context, workspace, timing, errors).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/radsort.h"
#include "passes.cuh"

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
  Ctl* h_ctl = nullptr;  // pinned
  uint32_t epoch = 0;
  cudaEvent_t ev[2 * 64] = {};
  bool ev_init = false;
};

radsort_status ensure(DevBuf& b, size_t bytes, bool zero = false);

// per-kernel-class CUDA-event timing on the sort's stream (radsort_set_timing)
struct Timer {
  Context* ctx;
  cudaStream_t st;
  int n = 0;
  int cls[64];
  bool on;
  Timer(Context* c, cudaStream_t s) : ctx(c), st(s), on(g_timing) {}
  void begin(int k) {
    if (!on || n >= 64) return;
    cls[n] = k;
    cudaEventRecord(ctx->ev[2 * n], st);
  }
  void end() {
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

}  // namespace radsort
