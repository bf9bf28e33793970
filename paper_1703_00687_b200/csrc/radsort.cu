// radsort: host driver (MSD level loop) and the C ABI declared in
// include/radsort.h.  All data movement and arithmetic of the sort happens in
// the kernels of passes.cuh; this file only sizes workspace, launches, and
// reads one small control block per MSD level.
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

static thread_local std::string g_detail;
static thread_local radsort_stats g_stats;
static bool g_timing = false;

static void set_detail(const char* fmt, ...) {
  char b[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(b, sizeof b, fmt, ap);
  va_end(ap);
  g_detail = b;
}

#define RS_CUDA(x)                                                                 \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      set_detail("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
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

static std::mutex g_ctx_mu;
static std::vector<Context*> g_ctx;

static Context* get_ctx(int dev) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (auto* c : g_ctx)
    if (c->device == dev) return c;
  return nullptr;
}

static radsort_status ensure(DevBuf& b, size_t bytes, bool zero = false) {
  if (b.bytes >= bytes) return RADSORT_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  size_t want = std::max(bytes, (size_t)256);
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_detail("cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
    return RADSORT_ERR_OOM;
  }
  b.bytes = want;
  if (zero) RS_CUDA(cudaMemset(b.p, 0, want));
  return RADSORT_OK;
}

// ------------------------------------------------------------------ timing
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

// -------------------------------------------------------------- the sort
template <int R, int K>
struct Sorter {
  static constexpr uint32_t T = tile_records<R>();
  static constexpr uint32_t C = local_capacity<R>();

  static void set_attrs() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_scatter<R, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_BYTES);
    cudaFuncSetAttribute(k_local<R, K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL_SMEM_BYTES);
    cudaFuncSetAttribute(k_local<R, K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL_SMEM_BYTES);
    cudaFuncSetAttribute(k_local<R, K, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL_SMEM_BYTES);
    cudaFuncSetAttribute(k_local<R, K, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL_SMEM_BYTES);
    if constexpr (R <= 16)
      cudaFuncSetAttribute(k_local<R, K, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL_SMEM_BYTES);
    if constexpr (R <= 8)
      cudaFuncSetAttribute(k_local<R, K, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL_SMEM_BYTES);
    done = true;
  }

  static void launch_local(uint32_t nloc, uint32_t maxlen, const Seg* list, Seg* next, int nxt, Ctl* ctl,
                           uint8_t* recs, uint8_t* tmp, cudaStream_t st) {
    const uint32_t il = (maxlen + LOCAL_B - 1) / LOCAL_B;
    const size_t smem = (size_t)maxlen * R;
#define RS_LOCAL(IL) k_local<R, K, IL><<<nloc, LOCAL_B, smem, st>>>(list, next, nxt, ctl, recs, tmp)
    if (il <= 1) RS_LOCAL(1);
    else if (il <= 2) RS_LOCAL(2);
    else if (il <= 4) RS_LOCAL(4);
    else if (il <= 8) RS_LOCAL(8);
    else if constexpr (R <= 16) {
      if (il <= 16) RS_LOCAL(16);
      else if constexpr (R <= 8) RS_LOCAL(32);
    }
#undef RS_LOCAL
  }

  static radsort_status run(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, cudaStream_t st,
                            radsort_stats& stats) {
    set_attrs();
    // ---- workspace
    const size_t capL = (size_t)n / C + 4;
    const size_t capLoc = (size_t)n / (TINY_MAX + 1) + 4;
    const size_t tiles_max = (size_t)n / T + capL + 4;
    radsort_status rs;
    if ((rs = ensure(ctx->large[0], capL * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->large[1], capL * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->local[0], capLoc * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->local[1], capLoc * sizeof(Seg)))) return rs;
    if ((rs = ensure(ctx->hist, capL * RADIX * sizeof(uint32_t)))) return rs;
    if ((rs = ensure(ctx->segbase, capL * RADIX * sizeof(uint32_t)))) return rs;
    if ((rs = ensure(ctx->andor, capL * 4 * sizeof(unsigned long long)))) return rs;
    if ((rs = ensure(ctx->tile_start, (capL + 1) * sizeof(uint32_t)))) return rs;
    const size_t old_status = ctx->status.bytes;
    if ((rs = ensure(ctx->status, tiles_max * RADIX * sizeof(unsigned long long), true))) return rs;
    if (ctx->status.bytes != old_status) ctx->epoch = 0;
    if ((rs = ensure(ctx->ctl, sizeof(Ctl)))) return rs;
    if (!ctx->h_ctl) RS_CUDA(cudaMallocHost(&ctx->h_ctl, sizeof(Ctl)));

    Seg* L[2] = {(Seg*)ctx->large[0].p, (Seg*)ctx->large[1].p};
    Seg* Lo[2] = {(Seg*)ctx->local[0].p, (Seg*)ctx->local[1].p};
    uint32_t* hist = (uint32_t*)ctx->hist.p;
    uint32_t* segbase = (uint32_t*)ctx->segbase.p;
    unsigned long long* andor = (unsigned long long*)ctx->andor.p;
    uint32_t* tile_start = (uint32_t*)ctx->tile_start.p;
    unsigned long long* status = (unsigned long long*)ctx->status.p;
    Ctl* ctl = (Ctl*)ctx->ctl.p;

    int occ_s = 0, occ_h = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_scatter<R, K>, SCAT_B, TILE_BYTES);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_h, k_hist<R, K>, HIST_B, 0);
    occ_s = std::max(occ_s, 1);
    occ_h = std::max(occ_h, 1);

    Timer tm(ctx, st);
    const bool log = getenv("RADSORT_LOG") && getenv("RADSORT_LOG")[0] == '1';

    k_init<<<1, 1, 0, st>>>(L[0], Lo[0], ctl, n, C);
    uint32_t n_large = n > C ? 1u : 0u;
    if (n_large) {
      tm.begin(RADSORT_K_SAMPLE);
      k_sample<R, K><<<1, 256, 0, st>>>(L[0], ctl, recs, n);
      tm.end();
      stats.kernel_launches[RADSORT_K_SAMPLE]++;
    }
    int cur = 0;
    const int max_levels = 2 * K + 4;
    for (int level = 0;; ++level) {
      if (level > max_levels) {
        set_detail("MSD level loop did not terminate (%d levels)", level);
        return RADSORT_ERR_CUDA;
      }
      const int nxt = cur ^ 1;
      if (n_large) {
        RS_CUDA(cudaMemsetAsync(hist, 0, (size_t)n_large * RADIX * sizeof(uint32_t), st));
        RS_CUDA(cudaMemsetAsync(andor, 0, (size_t)n_large * 4 * sizeof(unsigned long long), st));
        tm.begin(RADSORT_K_PLAN);
        k_prep<<<1, 1024, 0, st>>>(L[cur], n_large, T, tile_start, ctl, nxt);
        tm.end();
        const size_t tiles_ub = std::min(tiles_max, (size_t)n / T + n_large + 1);
        const unsigned gh = (unsigned)std::min(tiles_ub, (size_t)ctx->sms * occ_h);
        tm.begin(RADSORT_K_HIST);
        k_hist<R, K><<<gh, HIST_B, 0, st>>>(L[cur], tile_start, n_large, ctl, hist, andor, recs, tmp);
        tm.end();
        tm.begin(RADSORT_K_PLAN);
        k_plan<K><<<n_large, RADIX, 0, st>>>(L[cur], hist, andor, segbase, L[nxt], ctl);
        tm.end();
        if (++ctx->epoch >= 65536) {
          RS_CUDA(cudaMemsetAsync(status, 0, ctx->status.bytes, st));
          ctx->epoch = 1;
        }
        const unsigned gs = (unsigned)std::min(tiles_ub, (size_t)ctx->sms * occ_s);
        tm.begin(RADSORT_K_SCATTER);
        k_scatter<R, K><<<gs, SCAT_B, TILE_BYTES, st>>>(L[cur], tile_start, n_large, segbase, status, ctx->epoch, ctl,
                                                        recs, tmp);
        tm.end();
        tm.begin(RADSORT_K_CHILDREN);
        k_children<R, K><<<n_large, CHILD_B, 0, st>>>(L[cur], hist, segbase, L[nxt], Lo[cur], cur, ctl, recs, tmp);
        tm.end();
        stats.kernel_launches[RADSORT_K_PLAN] += 2;
        stats.kernel_launches[RADSORT_K_HIST]++;
        stats.kernel_launches[RADSORT_K_SCATTER]++;
        stats.kernel_launches[RADSORT_K_CHILDREN]++;
        stats.scatter_passes++;
      } else {
        k_prep<<<1, 1024, 0, st>>>(L[cur], 0, T, tile_start, ctl, nxt);
        stats.kernel_launches[RADSORT_K_PLAN]++;
      }
      RS_CUDA(cudaGetLastError());
      RS_CUDA(cudaMemcpyAsync(ctx->h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaStreamSynchronize(st));
      const Ctl c = *ctx->h_ctl;
      if (level == 0) stats.first_digit = c.d0;
      const uint32_t nloc = c.n_local[cur];
      if (log)
        fprintf(stderr, "[radsort] level %d: large=%u tiles=%u -> large_next=%u local=%u (max %u)\n", level, n_large,
                c.tiles_total, c.n_large_next, nloc, c.max_local_len[cur]);
      if (nloc) {
        tm.begin(RADSORT_K_LOCAL);
        launch_local(nloc, c.max_local_len[cur], Lo[cur], Lo[nxt], nxt, ctl, recs, tmp, st);
        tm.end();
        stats.kernel_launches[RADSORT_K_LOCAL]++;
        RS_CUDA(cudaGetLastError());
      }
      stats.levels = level + 1;
      tm.flush(stats);
      if (c.n_large_next == 0 && nloc == 0 && n_large == 0) break;
      n_large = c.n_large_next;
      cur = nxt;
    }
    // final statistics (one more small read; the sort's last kernels are ordered before it)
    RS_CUDA(cudaMemcpyAsync(ctx->h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    const Ctl c = *ctx->h_ctl;
    stats.records_scattered = c.rec_scatter;
    stats.records_hist = c.rec_hist;
    stats.records_local = c.rec_local;
    stats.records_tiny = c.rec_tiny;
    stats.records_copied = c.rec_copy;
    stats.bins_large = c.bins_large;
    stats.bins_local = c.bins_local;
    stats.bins_tiny = c.bins_tiny;
    stats.bins_final = c.bins_final;
    stats.kernel_bytes[RADSORT_K_HIST] = c.rec_hist * R;
    stats.kernel_bytes[RADSORT_K_SCATTER] = 2ull * c.rec_scatter * R;
    stats.kernel_bytes[RADSORT_K_LOCAL] = 2ull * c.rec_local * R;
    stats.kernel_bytes[RADSORT_K_CHILDREN] = 2ull * c.rec_tiny * R;
    return RADSORT_OK;
  }
};

static radsort_status dispatch(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, uint32_t R, uint32_t K,
                               cudaStream_t st, radsort_stats& s) {
  if (R == 8 && K == 8) return Sorter<8, 8>::run(ctx, recs, tmp, n, st, s);
  if (R == 16 && K == 8) return Sorter<16, 8>::run(ctx, recs, tmp, n, st, s);
  if (R == 16 && K == 16) return Sorter<16, 16>::run(ctx, recs, tmp, n, st, s);
  if (R == 32 && K == 8) return Sorter<32, 8>::run(ctx, recs, tmp, n, st, s);
  if (R == 32 && K == 16) return Sorter<32, 16>::run(ctx, recs, tmp, n, st, s);
  set_detail("rec_size=%u key_size=%u not built", R, K);
  return RADSORT_ERR_UNSUPPORTED;
}

static radsort_status check_layout(uint32_t R, uint32_t K) {
  if (K != 8 && K != 16) {
    set_detail("key_size must be 8 or 16 (got %u)", K);
    return RADSORT_ERR_INVALID_ARG;
  }
  if (R < K || R > 64 || R % 8) {
    set_detail("rec_size must be a multiple of 8 in [key_size, 64] (got %u)", R);
    return RADSORT_ERR_INVALID_ARG;
  }
  if (!((R == 8 && K == 8) || R == 16 || R == 32)) {
    set_detail("rec_size=%u key_size=%u is not built", R, K);
    return RADSORT_ERR_UNSUPPORTED;
  }
  return RADSORT_OK;
}

}  // namespace radsort

using namespace radsort;

extern "C" {

radsort_status radsort_init(int device) {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || device < 0 || device >= cnt) {
    cudaGetLastError();
    set_detail("radsort_init: device %d unavailable (%s)", device, e == cudaSuccess ? "out of range" : cudaGetErrorString(e));
    return e == cudaSuccess ? RADSORT_ERR_INVALID_ARG : RADSORT_ERR_CUDA;
  }
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (auto* c : g_ctx)
    if (c->device == device) return RADSORT_OK;
  Context* c = new Context();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  cudaSetDevice(prev);
  c->ev_init = true;
  g_ctx.push_back(c);
  return RADSORT_OK;
}

radsort_status radsort_sort(void* dev_records, void* dev_tmp, uint64_t n, uint32_t rec_size, uint32_t key_size,
                            void* stream) {
  g_detail.clear();
  radsort_status rs = check_layout(rec_size, key_size);
  if (rs) return rs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    set_detail("no CUDA device");
    return RADSORT_ERR_CUDA;
  }
  Context* ctx = get_ctx(dev);
  if (!ctx) {
    set_detail("radsort_init(%d) was not called", dev);
    return RADSORT_ERR_NOT_INITIALIZED;
  }
  radsort_stats s = {};
  s.n = n;
  s.rec_size = rec_size;
  s.key_size = key_size;
  if (n <= 1) {
    g_stats = s;
    return RADSORT_OK;
  }
  if (!dev_records || !dev_tmp) {
    set_detail("NULL buffer with n=%llu", (unsigned long long)n);
    return RADSORT_ERR_INVALID_ARG;
  }
  if (n >= (1ull << 32)) {
    set_detail("n=%llu >= 2^32 records is not supported", (unsigned long long)n);
    return RADSORT_ERR_UNSUPPORTED;
  }
  if (((uintptr_t)dev_records | (uintptr_t)dev_tmp) & 15) {
    set_detail("buffers must be 16-byte aligned");
    return RADSORT_ERR_INVALID_ARG;
  }
  const uint64_t bytes = n * rec_size;
  const uintptr_t a = (uintptr_t)dev_records, b = (uintptr_t)dev_tmp;
  if (a < b + bytes && b < a + bytes) {
    set_detail("dev_records and dev_tmp overlap");
    return RADSORT_ERR_INVALID_ARG;
  }
  std::lock_guard<std::mutex> g(ctx->mu);
  rs = dispatch(ctx, (uint8_t*)dev_records, (uint8_t*)dev_tmp, (uint32_t)n, rec_size, key_size, (cudaStream_t)stream, s);
  g_stats = s;
  return rs;
}

radsort_status radsort_sort_host(void* host_records, uint64_t n, uint32_t rec_size, uint32_t key_size, void* stream) {
  g_detail.clear();
  radsort_status rs = check_layout(rec_size, key_size);
  if (rs) return rs;
  if (n <= 1) return RADSORT_OK;
  if (!host_records) {
    set_detail("NULL host buffer");
    return RADSORT_ERR_INVALID_ARG;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return RADSORT_ERR_CUDA; }
  Context* ctx = get_ctx(dev);
  if (!ctx) return RADSORT_ERR_NOT_INITIALIZED;
  const size_t bytes = (size_t)n * rec_size;
  {
    std::lock_guard<std::mutex> g(ctx->mu);
    if ((rs = ensure(ctx->host_io[0], bytes))) return rs;
    if ((rs = ensure(ctx->host_io[1], bytes))) return rs;
  }
  cudaStream_t st = (cudaStream_t)stream;
  RS_CUDA(cudaMemcpyAsync(ctx->host_io[0].p, host_records, bytes, cudaMemcpyHostToDevice, st));
  rs = radsort_sort(ctx->host_io[0].p, ctx->host_io[1].p, n, rec_size, key_size, stream);
  if (rs) return rs;
  RS_CUDA(cudaMemcpyAsync(host_records, ctx->host_io[0].p, bytes, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  return RADSORT_OK;
}

radsort_status radsort_locate_bucket(const uint64_t* hist256, uint64_t q, uint32_t* bucket, uint64_t* before) {
  if (!hist256 || !bucket || !before) return RADSORT_ERR_INVALID_ARG;
  uint64_t acc = 0;
  for (uint32_t v = 0; v < 256; ++v) {
    if (q < acc + hist256[v]) {
      *bucket = v;
      *before = acc;
      return RADSORT_OK;
    }
    acc += hist256[v];
  }
  return RADSORT_ERR_INVALID_ARG;
}

radsort_status radsort_set_timing(int enable) {
  g_timing = enable != 0;
  return RADSORT_OK;
}

radsort_status radsort_last_stats(radsort_stats* out) {
  if (!out) return RADSORT_ERR_INVALID_ARG;
  *out = g_stats;
  return RADSORT_OK;
}

const char* radsort_error_string(radsort_status s) {
  static thread_local std::string msg;
  const char* base = "unknown status";
  switch (s) {
    case RADSORT_OK: base = "ok"; break;
    case RADSORT_ERR_INVALID_ARG: base = "invalid argument"; break;
    case RADSORT_ERR_UNSUPPORTED: base = "unsupported record layout or size"; break;
    case RADSORT_ERR_NOT_INITIALIZED: base = "radsort_init not called for this device"; break;
    case RADSORT_ERR_CUDA: base = "CUDA error"; break;
    case RADSORT_ERR_NCCL: base = "NCCL error"; break;
    case RADSORT_ERR_OOM: base = "out of device memory"; break;
    case RADSORT_ERR_CAPACITY: base = "output shard exceeds capacity"; break;
  }
  msg = base;
  if (s != RADSORT_OK && !g_detail.empty()) msg += ": " + g_detail;
  return msg.c_str();
}

void radsort_finalize(void) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (auto* c : g_ctx) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    DevBuf* bufs[] = {&c->large[0], &c->large[1], &c->local[0], &c->local[1], &c->hist, &c->andor, &c->segbase,
                      &c->tile_start, &c->status, &c->ctl, &c->host_io[0], &c->host_io[1]};
    for (auto* b : bufs)
      if (b->p) cudaFree(b->p);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    for (auto& ev : c->ev)
      if (ev) cudaEventDestroy(ev);
    cudaSetDevice(prev);
    delete c;
  }
  g_ctx.clear();
}

const char* radsort_version(void) { return "radsort 0.1 sm_100a"; }

}  // extern "C"
