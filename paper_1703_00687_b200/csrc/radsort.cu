// radsort: host driver entry points and the C ABI declared in
// include/radsort.h.  All data movement and arithmetic of the sort happens in
// the kernels of passes.cuh (instantiated per record layout in layout_R_K.cu);
// this file validates arguments, owns the per-device contexts and dispatches.
#include "driver.cuh"

namespace radsort {

static thread_local std::string g_detail;
static thread_local radsort_stats g_stats;
bool g_timing = false;

void set_detail(const char* fmt, ...) {
  char b[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(b, sizeof b, fmt, ap);
  va_end(ap);
  g_detail = b;
}

void set_last_stats(const radsort_stats& s) { g_stats = s; }

static std::mutex g_ctx_mu;
static std::vector<Context*> g_ctx;

static Context* get_ctx(int dev) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (auto* c : g_ctx)
    if (c->device == dev) return c;
  return nullptr;
}

Context* get_or_create_ctx(int dev) {
  Context* c = get_ctx(dev);
  if (!c && radsort_init(dev) == RADSORT_OK) c = get_ctx(dev);
  return c;
}

const LayoutOps* layout_ops(uint32_t R, uint32_t K) {
#define RS_OPS(r, k) \
  static const LayoutOps ops_##r##_##k = {run_layout<r, k>, run_layout_segs<r, k>, multi_hist<r, k>, \
                                          multi_scatter<r, k>, multi_bounds<r, k>, multi_piece_hist<r, k>, \
                                          multi_piece_scatter<r, k>}
  RS_OPS(8, 8);
  RS_OPS(16, 8);
  RS_OPS(16, 16);
  RS_OPS(32, 8);
  RS_OPS(32, 16);
  RS_OPS(24, 8);
  RS_OPS(24, 16);
  RS_OPS(40, 16);
#undef RS_OPS
  if (R == 8 && K == 8) return &ops_8_8;
  if (R == 16 && K == 8) return &ops_16_8;
  if (R == 16 && K == 16) return &ops_16_16;
  if (R == 32 && K == 8) return &ops_32_8;
  if (R == 32 && K == 16) return &ops_32_16;
  if (R == 24 && K == 8) return &ops_24_8;
  if (R == 24 && K == 16) return &ops_24_16;
  if (R == 40 && K == 16) return &ops_40_16;
  return nullptr;
}

radsort_status ensure(DevBuf& b, size_t bytes, bool zero) {
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

static radsort_status dispatch(Context* ctx, uint8_t* recs, uint8_t* tmp, uint32_t n, uint32_t R, uint32_t K,
                               cudaStream_t st, radsort_stats& s) {
  if (R == 8 && K == 8) return run_layout<8, 8>(ctx, recs, tmp, n, st, s);
  if (R == 16 && K == 8) return run_layout<16, 8>(ctx, recs, tmp, n, st, s);
  if (R == 16 && K == 16) return run_layout<16, 16>(ctx, recs, tmp, n, st, s);
  if (R == 32 && K == 8) return run_layout<32, 8>(ctx, recs, tmp, n, st, s);
  if (R == 32 && K == 16) return run_layout<32, 16>(ctx, recs, tmp, n, st, s);
  if (R == 24 && K == 8) return run_layout<24, 8>(ctx, recs, tmp, n, st, s);
  if (R == 24 && K == 16) return run_layout<24, 16>(ctx, recs, tmp, n, st, s);
  if (R == 40 && K == 16) return run_layout<40, 16>(ctx, recs, tmp, n, st, s);
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
  if (!((R == 8 && K == 8) || R == 16 || R == 32 || R == 24 || (R == 40 && K == 16))) {
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
  cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming);
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

radsort_status radsort_sort_host_stream(void* const* host_in, void* const* host_out, uint32_t nbatch, uint64_t n,
                                        uint32_t rec_size, uint32_t key_size, void* const* dev_bufs, uint32_t nbuf,
                                        void* dev_tmp, void* stream) {
  g_detail.clear();
  radsort_status rs = check_layout(rec_size, key_size);
  if (rs) return rs;
  if (nbatch == 0) return RADSORT_OK;
  if (!host_in || !host_out || !dev_bufs || !dev_tmp || nbuf < 2) {
    set_detail("NULL pointer array or nbuf < 2");
    return RADSORT_ERR_INVALID_ARG;
  }
  for (uint32_t k = 0; k < nbatch; ++k)
    if (!host_in[k] || !host_out[k]) {
      set_detail("NULL host buffer of batch %u", k);
      return RADSORT_ERR_INVALID_ARG;
    }
  for (uint32_t b = 0; b < nbuf; ++b)
    if (!dev_bufs[b]) {
      set_detail("NULL device buffer %u", b);
      return RADSORT_ERR_INVALID_ARG;
    }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return RADSORT_ERR_CUDA; }
  if (!get_ctx(dev)) return RADSORT_ERR_NOT_INITIALIZED;
  const size_t bytes = (size_t)n * rec_size;
  if (n <= 1) {
    for (uint32_t k = 0; k < nbatch; ++k)
      if (host_out[k] != host_in[k]) memcpy(host_out[k], host_in[k], bytes);
    return RADSORT_OK;
  }
  cudaStream_t st = (cudaStream_t)stream, cin = nullptr, cout = nullptr;
  std::vector<cudaEvent_t> ev_in(nbatch, nullptr), ev_sorted(nbatch, nullptr), ev_out(nbatch, nullptr);
  auto cleanup = [&]() {
    for (auto* v : {&ev_in, &ev_sorted, &ev_out})
      for (cudaEvent_t e : *v)
        if (e) cudaEventDestroy(e);
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
  };
  auto fail = [&](cudaError_t e, const char* what) {
    set_detail("%s: %s", what, cudaGetErrorString(e));
    cudaGetLastError();
    if (cin) cudaStreamSynchronize(cin);
    if (cout) cudaStreamSynchronize(cout);
    if (st) cudaStreamSynchronize(st);
    cleanup();
    return RADSORT_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking)) ||
      (e = cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking)))
    return fail(e, "stream create");
  for (uint32_t k = 0; k < nbatch; ++k)
    if ((e = cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming)) ||
        (e = cudaEventCreateWithFlags(&ev_sorted[k], cudaEventDisableTiming)) ||
        (e = cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming)))
      return fail(e, "event create");
  // copy-in of batch k into dev_bufs[k % nbuf], once the copy-out of batch k - nbuf has read it
  auto copy_in = [&](uint32_t k) -> cudaError_t {
    cudaError_t r;
    if (k >= nbuf && (r = cudaStreamWaitEvent(cin, ev_out[k - nbuf], 0))) return r;
    if ((r = cudaMemcpyAsync(dev_bufs[k % nbuf], host_in[k], bytes, cudaMemcpyHostToDevice, cin))) return r;
    return cudaEventRecord(ev_in[k], cin);
  };
  if ((e = copy_in(0))) return fail(e, "copy-in");
  for (uint32_t k = 0; k < nbatch; ++k) {
    // the next batch's copy-in is enqueued before this batch's sort: radsort_sort
    // waits on its stream between MSD levels, so what must overlap it goes first
    if (k + 1 < nbatch && (e = copy_in(k + 1))) return fail(e, "copy-in");
    if ((e = cudaStreamWaitEvent(st, ev_in[k], 0))) return fail(e, "wait copy-in");
    rs = radsort_sort(dev_bufs[k % nbuf], dev_tmp, n, rec_size, key_size, stream);
    if (rs) {
      const std::string d = g_detail;
      cudaStreamSynchronize(cin);
      cudaStreamSynchronize(cout);
      cleanup();
      g_detail = d;
      return rs;
    }
    if ((e = cudaEventRecord(ev_sorted[k], st)) || (e = cudaStreamWaitEvent(cout, ev_sorted[k], 0)) ||
        (e = cudaMemcpyAsync(host_out[k], dev_bufs[k % nbuf], bytes, cudaMemcpyDeviceToHost, cout)) ||
        (e = cudaEventRecord(ev_out[k], cout)))
      return fail(e, "copy-out");
  }
  if ((e = cudaStreamSynchronize(cout)) || (e = cudaStreamSynchronize(cin)) || (e = cudaStreamSynchronize(st)))
    return fail(e, "synchronize");
  cleanup();
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
    DevBuf* bufs[] = {&c->large[0], &c->large[1], &c->local[0], &c->local[1], &c->hist,     &c->andor,
                      &c->segbase,  &c->tile_start, &c->status, &c->ctl,   &c->host_io[0], &c->host_io[1],
                      &c->mprobe,   &c->mlo,      &c->mhi,      &c->mlt,   &c->mle,       &c->splitc,
                      &c->probes,   &c->tile_seg, &c->tile_pre, &c->kiw};
    for (auto* b : bufs)
      if (b->p) cudaFree(b->p);
    for (auto& kv : c->ipc_open) cudaIpcCloseMemHandle(kv.second);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    for (auto& ev : c->ev)
      if (ev) cudaEventDestroy(ev);
    if (c->done_ev) cudaEventDestroy(c->done_ev);
    cudaSetDevice(prev);
    delete c;
  }
  g_ctx.clear();
}

const char* radsort_version(void) { return "radsort 0.1 sm_100a"; }

}  // extern "C"
