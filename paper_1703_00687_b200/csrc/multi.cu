// radsort multi-GPU path: key-range sharding with one exchange step
// (the paper's phase-1 "parallel processing of the whole
// array according to the first digit", §3.1, carried across
// GPUs).  One process (or, for tests, one host thread) per GPU rank:
//
//  1. agree on the layout and N = sum of n_local (allreduce min/max/sum);
//     exact-balance quotas q_r = floor(N/G) + (r < N mod G)   (R11)
//  2. local AND/OR of the keys -> allgather -> global first non-constant
//     digit d0; local 256-bin histogram of d0 -> allreduce -> global H
//  3. local counting-scatter by d0 (records -> tmp), the level-0 pass
//  4. each boundary Q_g = q_0 + .. + q_{g-1} falls in global bucket b_g; every
//     rank sorts its (small) bucket b_g locally, then the Q_g-th key k_g is
//     found digit by digit: 256 probes per boundary, #keys < probe by binary
//     search on the sorted bucket, allreduce, keep the largest digit whose
//     count stays <= Q_g
//  5. records equal to k_g are split across ranks by source-rank order so the
//     quotas hold exactly (any order inside an equal-key run is correct, R2)
//  6. send ranges are contiguous slices of tmp, grouped by d0; they travel as
//     one message per (destination, d0 bucket) in grouped ncclSend/ncclRecv
//     (NVLink / NVSwitch), so that each receiver lands its records bucket by
//     bucket (bucket b from every sender contiguous in dev_records)
//  7. the received shard is sorted by the single-GPU path, starting from those
//     buckets at digit d0 + 1: the receiver never re-partitions by d0.
//
// The algorithm is written against a small Transport interface with two
// implementations: NCCL (the product) and an in-process loopback with host
// threads as ranks (tests, since the pool gives one GPU per box).
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <numeric>
#include <thread>

#include <unistd.h>

#include "driver.cuh"

namespace radsort {

// --------------------------------------------------------------- planner
// Pure host functions (exported for tests through the C ABI).
static void plan_quotas(uint64_t N, int G, uint64_t* q) {
  for (int r = 0; r < G; ++r) q[r] = N / (uint64_t)G + ((uint64_t)r < N % (uint64_t)G ? 1 : 0);
}
// largest digit v with count_lt[v] <= q (count_lt non-decreasing, count_lt[0] <= q)
static uint32_t plan_digit(const uint64_t* count_lt, uint64_t q) {
  uint32_t v = 0;
  for (uint32_t u = 1; u < 256; ++u)
    if (count_lt[u] <= q) v = u;
  return v;
}
// records equal to the boundary key that rank r keeps below the boundary:
// the first (Q - L) equal records in source-rank order go below.
static void plan_equal_split(const uint64_t* e, int G, uint64_t L, uint64_t Q, uint64_t* below) {
  uint64_t need = Q > L ? Q - L : 0;
  for (int r = 0; r < G; ++r) {
    const uint64_t take = std::min(need, e[r]);
    below[r] = take;
    need -= take;
  }
}

// Fused exchange plan (step 6' below).  all[((src * G + r) * 256 + b) * 256 + v]
// = records of sender src's piece for receiver r in d0 bucket b with digit
// d0+1 = v (every rank's dense table, allgathered).  Receiver r lays its
// (b, v) bins out in (b, v) order, senders in rank order inside a bin.
// Outputs: base[i * 256 + v] = offset in receiver pdst[i]'s buffer of this
// rank's share of bin (pbkt[i], v); recv_off[0..65536] = the bin offsets of
// rank `me` (recv_off[65536] = its record count).  Returns false if a
// receiver's total does not fit in 32 bits.
static bool plan_fused(const uint32_t* all, int G, int me, uint32_t np, const uint32_t* pdst, const uint32_t* pbkt,
                       uint32_t* base, uint64_t* recv_off, std::vector<uint64_t>* totals = nullptr) {
  auto cnt = [&](int src, int r, size_t bv) { return all[((size_t)src * G + r) * 65536 + bv]; };
  std::vector<char> need(G, 0);
  for (uint32_t i = 0; i < np; ++i) need[pdst[i]] = 1;
  need[me] = 1;
  std::vector<std::vector<uint64_t>> roff(G);
  for (int r = 0; r < G; ++r) {
    if (!need[r]) continue;
    roff[r].resize(65537);
    uint64_t run = 0;
    for (size_t bv = 0; bv < 65536; ++bv) {
      roff[r][bv] = run;
      for (int p = 0; p < G; ++p) run += cnt(p, r, bv);
    }
    roff[r][65536] = run;
    if (run >> 32) return false;
    if (totals) (*totals)[r] = run;
  }
  for (uint32_t i = 0; i < np; ++i) {
    const int r = (int)pdst[i];
    for (int v = 0; v < 256; ++v) {
      const size_t bv = (size_t)pbkt[i] * 256 + v;
      uint64_t o = roff[r][bv];
      for (int p = 0; p < me; ++p) o += cnt(p, r, bv);
      base[(size_t)i * 256 + v] = (uint32_t)o;
    }
  }
  std::copy(roff[me].begin(), roff[me].end(), recv_off);
  return true;
}

// -------------------------------------------------------------- transport
enum class ROp { Sum, Min, Max };

// one point-to-point message of the exchange: `bytes` bytes at byte offset
// `off` of the send (or receive) buffer, to (or from) rank `peer`; messages
// between one pair of ranks match in the order they are listed
struct Msg {
  int peer;
  uint64_t off, bytes;
};

struct Transport {
  virtual ~Transport() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // host in -> host out (small control data)
  virtual radsort_status allreduce(const uint64_t* in, uint64_t* out, size_t cnt, ROp op, cudaStream_t st) = 0;
  virtual radsort_status allgather(const uint64_t* in, uint64_t* out, size_t cnt, cudaStream_t st) = 0;
  // device data: every message of `sends` from `send`, every one of `recvs` into `recv`
  virtual radsort_status exchange(const uint8_t* send, const std::vector<Msg>& sends, uint8_t* recv,
                                  const std::vector<Msg>& recvs, cudaStream_t st) = 0;
  // Peer access for the fused exchange: out[p] = rank p's `mine` (its record
  // buffer) mapped into this process.  Collective; every rank gets the same
  // answer: RADSORT_OK everywhere, or RADSORT_ERR_UNSUPPORTED everywhere (the
  // caller then takes the send/recv exchange).
  virtual radsort_status peer_bases(uint8_t* mine, std::vector<uint8_t*>& out, Context* ctx, cudaStream_t st) = 0;
  radsort_status barrier(cudaStream_t st) {
    const uint64_t one = 1;
    uint64_t sum = 0;
    return allreduce(&one, &sum, 1, ROp::Sum, st);
  }
};

#define RS_NCCL(x)                                                                             \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess) {                                                                   \
      set_detail("%s failed: %s (%s:%d)", #x, ncclGetErrorString(r_), __FILE__, __LINE__);    \
      return RADSORT_ERR_NCCL;                                                                 \
    }                                                                                          \
  } while (0)

struct NcclTransport : Transport {
  ncclComm_t comm;
  int r = 0, g = 1;
  DevBuf buf;
  explicit NcclTransport(ncclComm_t c) : comm(c) {
    ncclCommUserRank(comm, &r);
    ncclCommCount(comm, &g);
  }
  ~NcclTransport() override {
    if (buf.p) cudaFree(buf.p);
  }
  int rank() const override { return r; }
  int size() const override { return g; }
  // Wait for the stream's work without blocking inside the driver: a dead peer
  // would leave an NCCL kernel spinning forever, so poll the stream and the
  // communicator's asynchronous error state; give up after
  // RADSORT_NCCL_TIMEOUT_S seconds (default 600).  On an error or a timeout the
  // communicator is unusable: the caller aborts it (ncclCommAbort / torch).
  radsort_status check(cudaStream_t st) {
    const char* e = getenv("RADSORT_NCCL_TIMEOUT_S");
    const double limit = e ? atof(e) : 600.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; ++spin) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) {
        set_detail("stream error during NCCL collective: %s", cudaGetErrorString(q));
        return RADSORT_ERR_CUDA;
      }
      ncclResult_t ar = ncclSuccess;
      if (ncclCommGetAsyncError(comm, &ar) != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
        set_detail("NCCL async error: %s", ncclGetErrorString(ar));
        return RADSORT_ERR_NCCL;
      }
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
        set_detail("NCCL collective did not complete within %.0f s (peer lost?)", limit);
        return RADSORT_ERR_NCCL;
      }
      if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(comm, &ar);
    if (ar != ncclSuccess) {
      set_detail("NCCL async error: %s", ncclGetErrorString(ar));
      return RADSORT_ERR_NCCL;
    }
    return RADSORT_OK;
  }
  radsort_status allreduce(const uint64_t* in, uint64_t* out, size_t cnt, ROp op, cudaStream_t st) override {
    radsort_status rs;
    if ((rs = ensure(buf, 2 * cnt * 8))) return rs;
    uint64_t* d = (uint64_t*)buf.p;
    RS_CUDA(cudaMemcpyAsync(d, in, cnt * 8, cudaMemcpyHostToDevice, st));
    const ncclRedOp_t o = op == ROp::Sum ? ncclSum : (op == ROp::Min ? ncclMin : ncclMax);
    RS_NCCL(ncclAllReduce(d, d + cnt, cnt, ncclUint64, o, comm, st));
    RS_CUDA(cudaMemcpyAsync(out, d + cnt, cnt * 8, cudaMemcpyDeviceToHost, st));
    return check(st);
  }
  radsort_status allgather(const uint64_t* in, uint64_t* out, size_t cnt, cudaStream_t st) override {
    radsort_status rs;
    if ((rs = ensure(buf, (1 + (size_t)g) * cnt * 8))) return rs;
    uint64_t* d = (uint64_t*)buf.p;
    RS_CUDA(cudaMemcpyAsync(d, in, cnt * 8, cudaMemcpyHostToDevice, st));
    RS_NCCL(ncclAllGather(d, d + cnt, cnt, ncclUint64, comm, st));
    RS_CUDA(cudaMemcpyAsync(out, d + cnt, (size_t)g * cnt * 8, cudaMemcpyDeviceToHost, st));
    return check(st);
  }
  radsort_status exchange(const uint8_t* send, const std::vector<Msg>& sends, uint8_t* recv,
                          const std::vector<Msg>& recvs, cudaStream_t st) override {
    RS_NCCL(ncclGroupStart());
    ncclResult_t r = ncclSuccess;  // the group is always closed, also when an enqueue fails
    for (size_t i = 0; i < sends.size() && r == ncclSuccess; ++i)
      r = ncclSend(send + sends[i].off, sends[i].bytes, ncclUint8, sends[i].peer, comm, st);
    for (size_t i = 0; i < recvs.size() && r == ncclSuccess; ++i)
      r = ncclRecv(recv + recvs[i].off, recvs[i].bytes, ncclUint8, recvs[i].peer, comm, st);
    const ncclResult_t re = ncclGroupEnd();
    RS_NCCL(r);
    RS_NCCL(re);
    return check(st);
  }
  // CUDA IPC: every rank exports the allocation holding its record buffer
  // (cudaIpcGetMemHandle of the allocation base, found with the driver's
  // cuMemGetAddressRange) and opens its peers' handles once per context (the
  // mappings are cached until radsort_finalize).  Allocations IPC cannot export
  // (e.g. VMM / expandable segments) make every rank fall back.
  radsort_status peer_bases(uint8_t* mine, std::vector<uint8_t*>& out, Context* ctx, cudaStream_t st) override {
    typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
    static GetRange get_range = nullptr;
    if (!get_range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        get_range = (GetRange)fn;
      cudaGetLastError();
    }
    int dev = 0;
    cudaGetDevice(&dev);
    uint64_t pay[13] = {};
    unsigned long long base = 0;
    size_t size = 0;
    cudaIpcMemHandle_t h;
    bool ok = mine && get_range && get_range(&base, &size, (unsigned long long)(uintptr_t)mine) == 0 &&
              cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base) == cudaSuccess;
    cudaGetLastError();
    if (ok) memcpy(pay, &h, sizeof h);
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
    pay[8] = ok ? (uint64_t)(uintptr_t)mine - base : 0;
    pay[9] = (uint64_t)getpid();
    pay[10] = (uint64_t)dev;
    pay[11] = ok ? 1 : 0;
    pay[12] = (uint64_t)(uintptr_t)mine;
    std::vector<uint64_t> all(13 * (size_t)g);
    radsort_status rs;
    if ((rs = allgather(pay, all.data(), 13, st))) return rs;
    uint64_t okall = 1;
    for (int p = 0; p < g; ++p) okall &= all[13 * (size_t)p + 11];
    out.assign(g, nullptr);
    uint64_t opened = okall;
    std::unique_lock<std::mutex> lk(ctx->mu);  // the context's cache of opened handles
    for (int p = 0; p < g && opened; ++p) {
      const uint64_t* q = &all[13 * (size_t)p];
      if (p == r) {
        out[p] = mine;
      } else if (q[9] == (uint64_t)getpid()) {  // same process (another device): the pointer itself
        int can = 0;
        cudaDeviceCanAccessPeer(&can, dev, (int)q[10]);
        if (!can || ((cudaDeviceEnablePeerAccess((int)q[10], 0) != cudaSuccess) &&
                     cudaGetLastError() != cudaErrorPeerAccessAlreadyEnabled))
          opened = 0;
        cudaGetLastError();
        out[p] = (uint8_t*)(uintptr_t)q[12];
      } else {
        const std::string key((const char*)q, 64);
        auto it = ctx->ipc_open.find(key);
        void* ptr = nullptr;
        if (it != ctx->ipc_open.end()) {
          ptr = it->second;
        } else {
          cudaIpcMemHandle_t ph;
          memcpy(&ph, q, sizeof ph);
          if (cudaIpcOpenMemHandle(&ptr, ph, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
            ctx->ipc_open[key] = ptr;
          } else {
            cudaGetLastError();
            ptr = nullptr;
            opened = 0;
          }
        }
        out[p] = ptr ? (uint8_t*)ptr + q[8] : nullptr;
      }
    }
    lk.unlock();
    uint64_t all_opened = 0;  // every rank mapped every peer, or everyone falls back
    if ((rs = allreduce(&opened, &all_opened, 1, ROp::Min, st))) return rs;
    if (!all_opened) {
      set_detail("peer buffers not mappable (CUDA IPC); send/recv exchange used");
      return RADSORT_ERR_UNSUPPORTED;
    }
    return RADSORT_OK;
  }
};

// In-process loopback group: G host threads act as ranks on one device.
struct LoopGroup {
  int G;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<std::vector<uint64_t>> slot;
  std::vector<const uint8_t*> sbase;
  std::vector<std::vector<Msg>> sends;
  std::vector<uint8_t*> rbase;
  explicit LoopGroup(int g) : G(g), slot(g), sbase(g), sends(g), rbase(g) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
  }
};

struct LoopTransport : Transport {
  LoopGroup* grp;
  int r;
  LoopTransport(LoopGroup* g, int rk) : grp(g), r(rk) {}
  int rank() const override { return r; }
  int size() const override { return grp->G; }
  radsort_status allreduce(const uint64_t* in, uint64_t* out, size_t cnt, ROp op, cudaStream_t) override {
    grp->slot[r].assign(in, in + cnt);
    grp->barrier();
    for (size_t i = 0; i < cnt; ++i) {
      uint64_t a = grp->slot[0][i];
      for (int p = 1; p < grp->G; ++p) {
        const uint64_t b = grp->slot[p][i];
        a = op == ROp::Sum ? a + b : (op == ROp::Min ? std::min(a, b) : std::max(a, b));
      }
      out[i] = a;
    }
    grp->barrier();
    return RADSORT_OK;
  }
  radsort_status allgather(const uint64_t* in, uint64_t* out, size_t cnt, cudaStream_t) override {
    grp->slot[r].assign(in, in + cnt);
    grp->barrier();
    for (int p = 0; p < grp->G; ++p) std::copy(grp->slot[p].begin(), grp->slot[p].end(), out + (size_t)p * cnt);
    grp->barrier();
    return RADSORT_OK;
  }
  radsort_status exchange(const uint8_t* send, const std::vector<Msg>& sends, uint8_t* recv,
                          const std::vector<Msg>& recvs, cudaStream_t st) override {
    grp->sbase[r] = send;
    grp->sends[r] = sends;
    RS_CUDA(cudaStreamSynchronize(st));  // every rank's send data is complete before peers read it
    grp->barrier();
    // the k-th message from p to r pairs with the k-th receive r lists from p
    std::vector<size_t> cursor(grp->G, 0);
    radsort_status rs = RADSORT_OK;
    for (const Msg& m : recvs) {
      const std::vector<Msg>& ps = grp->sends[m.peer];
      size_t& k = cursor[m.peer];
      while (k < ps.size() && ps[k].peer != r) ++k;
      if (k == ps.size() || ps[k].bytes != m.bytes) {
        set_detail("loopback: rank %d expects a %llu-byte message from %d that was not sent", r,
                   (unsigned long long)m.bytes, m.peer);
        rs = RADSORT_ERR_INVALID_ARG;
        break;
      }
      if (m.bytes)
        if (cudaMemcpyAsync(recv + m.off, grp->sbase[m.peer] + ps[k].off, m.bytes, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess) {
          set_detail("loopback: cudaMemcpyAsync failed");
          rs = RADSORT_ERR_CUDA;
          break;
        }
      ++k;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && rs == RADSORT_OK) rs = RADSORT_ERR_CUDA;
    grp->barrier();
    return rs;
  }
  // every rank's buffer lives on this device in this process
  radsort_status peer_bases(uint8_t* mine, std::vector<uint8_t*>& out, Context*, cudaStream_t) override {
    grp->rbase[r] = mine;
    grp->barrier();
    out = grp->rbase;
    grp->barrier();
    return RADSORT_OK;
  }
};

// ------------------------------------------------------------- algorithm
static void set_digit(uint64_t* key, uint32_t K, uint32_t d, uint32_t v) {
  const uint32_t bi = K - 1 - d;
  const uint32_t w = bi >> 3, sh = 8 * (bi & 7);
  key[w] = (key[w] & ~(0xffull << sh)) | ((uint64_t)v << sh);
}

// Fused exchange + receive-side level (SURVEY.md §8(e) k_merge_scatter, §8(f)
// NEXT-3).  After the level-0 pass and the boundary search, each rank's send
// range to rank p is a run of d0 buckets in tmp ("pieces": the whole bucket,
// or the part of a straddling bucket on p's side of the cut).  Instead of
// sending the pieces and re-reading them on the receiver, every sender
//   a. histograms its pieces by the next digit d0+1 (one local read),
//   b. allgathers the piece histograms: every rank then knows, for every
//      receiver r, the size of each (d0, d0+1) bin from every sender, hence
//      where its own share of each bin lands in r's buffer (bins in (b, v)
//      order, senders in rank order inside a bin),
//   c. scatters its pieces by digit d0+1 straight into the receivers' record
//      buffers (k_scatter<PEER>: the radix pass's coalesced run stores go over
//      NVLink to the peer's HBM, so the transfer overlaps the pass tile by
//      tile and no separate copy or receive-side pass over the data remains).
// The receiver then sorts its (d0, d0+1) bins from digit d0+2 on: the whole
// multi-GPU sort moves each record through HBM as often as the 1-GPU sort does.
static radsort_status fused_exchange(Transport& tr, Context* ctx, const LayoutOps* ops, uint8_t* recs, uint8_t* tmp,
                                     uint64_t n_local, const std::vector<uint64_t>& cut, const uint64_t* lbase,
                                     const std::vector<uint64_t>& q, uint32_t d0, uint32_t R, uint32_t K,
                                     const std::vector<uint8_t*>& peer, cudaStream_t st, radsort_stats& stats,
                                     uint64_t* n_out) {
  const int G = tr.size(), me = tr.rank();
  radsort_status rs;
  std::vector<uint32_t> poff, plen, pdst;  // piece = (destination rank, bucket)
  std::vector<uint32_t> pbkt;
  for (int p = 0; p < G; ++p)
    for (int b = 0; b < 256; ++b) {
      const uint64_t lo = std::max(cut[p], lbase[b]), hi = std::min(cut[p + 1], lbase[b + 1]);
      if (hi > lo) {
        poff.push_back((uint32_t)lo);
        plen.push_back((uint32_t)(hi - lo));
        pdst.push_back((uint32_t)p);
        pbkt.push_back((uint32_t)b);
      }
    }
  const uint32_t np = (uint32_t)poff.size();
  NvtxRange nvtx_fx("radsort multi: fused exchange");
  PieceWs w;
  std::vector<uint32_t> ph((size_t)np * 256);
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if ((rs = ops->piece_hist(ctx, w, tmp, poff.data(), plen.data(), np, d0 + 1, st, ph.data()))) return rs;
  }
  // dense table of this sender: cnt[(r * 256 + b) * 256 + v], u32 packed in u64 pairs
  const size_t E = (size_t)G * 65536;
  std::vector<uint32_t> tab(E, 0);
  for (uint32_t i = 0; i < np; ++i)
    for (int v = 0; v < 256; ++v) tab[((size_t)pdst[i] * 256 + pbkt[i]) * 256 + v] = ph[(size_t)i * 256 + v];
  std::vector<uint32_t> all(E * (size_t)G);
  if ((rs = tr.allgather(reinterpret_cast<const uint64_t*>(tab.data()), reinterpret_cast<uint64_t*>(all.data()),
                         E / 2, st)))
    return rs;
  std::vector<uint32_t> hbase((size_t)np * 256);
  std::vector<uint64_t> hdst(np), recv(65537), tot(G, 0);
  if (!plan_fused(all.data(), G, me, np, pdst.data(), pbkt.data(), hbase.data(), recv.data(), &tot)) {
    set_detail("fused exchange: a receiver's record count exceeds 2^32");
    return RADSORT_ERR_CAPACITY;
  }
  for (int r = 0; r < G; ++r) {
    if (tot[r] && tot[r] != q[r]) {
      set_detail("fused exchange: rank %d would receive %llu records, quota %llu", r, (unsigned long long)tot[r],
                 (unsigned long long)q[r]);
      return RADSORT_ERR_CUDA;
    }
  }
  if (recv[65536] != q[me]) {
    set_detail("fused exchange: %llu records received, quota %llu", (unsigned long long)recv[65536],
               (unsigned long long)q[me]);
    return RADSORT_ERR_CUDA;
  }
  uint64_t sent = 0;
  for (uint32_t i = 0; i < np; ++i) {
    hdst[i] = (uint64_t)(uintptr_t)peer[pdst[i]];
    if ((int)pdst[i] != me) sent += plen[i];
  }
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if ((rs = ops->piece_scatter(ctx, w, tmp, hbase.data(), hdst.data(), st))) return rs;
  }
  if ((rs = tr.barrier(st))) return rs;  // every sender's stores into this rank's buffer are complete
  // receive side: the (d0, d0+1) bins, sorted from digit d0+2 on
  std::vector<uint32_t> seg_off, seg_len;
  uint64_t recv_other = 0;
  for (size_t bv = 0; bv < 65536; ++bv) {
    const uint64_t len = recv[bv + 1] - recv[bv];
    if (len) {
      seg_off.push_back((uint32_t)recv[bv]);
      seg_len.push_back((uint32_t)len);
    }
    recv_other += len - all[((size_t)me * G + me) * 65536 + bv];
  }
  const uint64_t got = recv[65536];
  stats.nvlink_bytes_sent = sent * R;
  stats.nvlink_bytes_recv = recv_other * R;
  radsort_stats sub = {};
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if ((rs = ops->sort_segs(ctx, recs, tmp, (uint32_t)got, seg_off.data(), seg_len.data(), (uint32_t)seg_off.size(),
                             d0 + 2, st, sub)))
      return rs;
  }
  stats.levels = sub.levels;
  stats.scatter_passes = sub.scatter_passes + 2;
  stats.records_scattered = sub.records_scattered + 2 * n_local;
  stats.records_hist = sub.records_hist + 2 * n_local;
  stats.records_local = sub.records_local;
  stats.records_tiny = sub.records_tiny;
  for (int k = 0; k < RADSORT_K_COUNT; ++k) {
    stats.kernel_launches[k] += sub.kernel_launches[k];
    stats.kernel_ms[k] += sub.kernel_ms[k];
    stats.kernel_bytes[k] += sub.kernel_bytes[k];
  }
  stats.kernel_launches[RADSORT_K_HIST] += 2;
  stats.kernel_launches[RADSORT_K_SCATTER] += 1;
  stats.kernel_launches[RADSORT_K_PLAN] += 2;
  stats.exchange = 2;
  stats.n = got;
  *n_out = got;
  return RADSORT_OK;
}

static radsort_status sort_multi_impl(Transport& tr, uint8_t* recs, uint8_t* tmp, uint64_t n_local, uint64_t capacity,
                                      uint64_t* n_out, uint32_t R, uint32_t K, cudaStream_t st, radsort_stats& stats) {
  const int G = tr.size(), me = tr.rank();
  int dev = 0;
  RS_CUDA(cudaGetDevice(&dev));
  Context* ctx = get_or_create_ctx(dev);
  if (!ctx) return RADSORT_ERR_NOT_INITIALIZED;
  const LayoutOps* ops = layout_ops(R, K);
  radsort_status rs;

  // 1. consistent arguments (every rank fails the same way instead of hanging)
  const uint64_t mine[5] = {R, K, ops ? 1ull : 0ull, n_local < (1ull << 32) ? 1ull : 0ull,
                            (recs && tmp) || n_local == 0 ? 1ull : 0ull};
  uint64_t mn[5], mx[5];
  if ((rs = tr.allreduce(mine, mn, 5, ROp::Min, st))) return rs;
  if ((rs = tr.allreduce(mine, mx, 5, ROp::Max, st))) return rs;
  if (mn[0] != mx[0] || mn[1] != mx[1]) {
    set_detail("ranks disagree on rec_size/key_size");
    return RADSORT_ERR_INVALID_ARG;
  }
  if (!mn[2]) {
    set_detail("rec_size=%u key_size=%u not built", R, K);
    return RADSORT_ERR_UNSUPPORTED;
  }
  if (!mn[3] || !mn[4]) {
    set_detail("a rank has n_local >= 2^32 or NULL buffers");
    return RADSORT_ERR_INVALID_ARG;
  }
  uint64_t N = 0;
  if ((rs = tr.allreduce(&n_local, &N, 1, ROp::Sum, st))) return rs;
  std::vector<uint64_t> q(G), Qb(G + 1, 0);
  plan_quotas(N, G, q.data());
  for (int g = 0; g < G; ++g) Qb[g + 1] = Qb[g] + q[g];
  const uint64_t cap_ok = (capacity >= q[me] && capacity >= n_local && q[me] < (1ull << 32)) ? 1 : 0;
  uint64_t all_ok = 0;
  if ((rs = tr.allreduce(&cap_ok, &all_ok, 1, ROp::Min, st))) return rs;
  if (!all_ok) {
    set_detail("capacity %llu < quota %llu or n_local on some rank", (unsigned long long)capacity,
               (unsigned long long)q[me]);
    return RADSORT_ERR_CAPACITY;
  }
  const uint32_t n = (uint32_t)n_local;

  // 2. global first non-constant digit and its histogram
  NvtxRange nvtx_plan("radsort multi: histogram + splitters");
  uint64_t h[256], ao[4];
  auto hist_op = [&](uint32_t digit) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    return ops->hist(ctx, recs, n, digit, st, h, ao);
  };
  if ((rs = hist_op(0))) return rs;
  std::vector<uint64_t> aog(4 * (size_t)G);
  if ((rs = tr.allgather(ao, aog.data(), 4, st))) return rs;
  uint64_t AND[2] = {~0ull, ~0ull}, OR[2] = {0, 0};
  for (int p = 0; p < G; ++p)
    for (int w = 0; w < 2; ++w) {
      AND[w] &= ~aog[4 * p + w];
      OR[w] |= aog[4 * p + 2 + w];
    }
  uint32_t d0 = 0;
  for (; d0 < K; ++d0) {
    const uint32_t bi = K - 1 - d0;
    if (((AND[bi >> 3] ^ OR[bi >> 3]) >> (8 * (bi & 7))) & 255) break;
  }
  if (d0 >= K) d0 = 0;  // every key equal: one bucket, split by quotas
  if (d0 != 0 && (rs = hist_op(d0))) return rs;
  uint64_t H[256];
  if ((rs = tr.allreduce(h, H, 256, ROp::Sum, st))) return rs;
  stats.first_digit = d0;

  // 3. level-0 pass: records -> tmp grouped by d0
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if ((rs = ops->scatter(ctx, recs, tmp, n, d0, h, st))) return rs;
  }
  uint64_t lbase[257];
  lbase[0] = 0;
  for (int b = 0; b < 256; ++b) lbase[b + 1] = lbase[b] + h[b];
  uint64_t Hbase[257];
  Hbase[0] = 0;
  for (int b = 0; b < 256; ++b) Hbase[b + 1] = Hbase[b] + H[b];

  // 4. boundaries: bucket, local sort of each distinct straddling bucket
  const int NB = G - 1;
  std::vector<uint32_t> bk(NB, 0);
  std::vector<char> active(NB, 0);
  for (int g = 1; g < G; ++g) {
    const uint64_t Qg = Qb[g];
    if (Qg >= N) continue;
    uint32_t b = 0;
    while (Qg >= Hbase[b + 1]) ++b;
    bk[g - 1] = b;
    active[g - 1] = 1;
  }
  {
    std::vector<uint32_t> done;
    for (int i = 0; i < NB; ++i) {
      if (!active[i] || std::find(done.begin(), done.end(), bk[i]) != done.end()) continue;
      done.push_back(bk[i]);
      const uint64_t off = lbase[bk[i]], len = h[bk[i]];
      if (len > 1) {
        radsort_stats sub = {};
        std::lock_guard<std::mutex> lk(ctx->mu);
        if ((rs = ops->sort(ctx, tmp + off * R, recs + off * R, (uint32_t)len, st, sub))) return rs;
      }
    }
    RS_CUDA(cudaStreamSynchronize(st));
  }
  // digit-by-digit selection of the boundary keys k_g
  std::vector<uint64_t> key(2 * (size_t)NB, 0);
  for (int i = 0; i < NB; ++i) {
    key[2 * i] = AND[0];  // digits constant over all keys are fixed by the global AND (== OR there)
    key[2 * i + 1] = K == 16 ? AND[1] : 0;
    if (active[i]) set_digit(&key[2 * i], K, d0, bk[i]);
  }
  std::vector<uint32_t> lo(256 * (size_t)NB), hi(256 * (size_t)NB);
  std::vector<uint64_t> probes(512 * (size_t)NB), lt(256 * (size_t)NB), le(256 * (size_t)NB), glt(256 * (size_t)NB);
  for (int i = 0; i < NB; ++i)
    for (int v = 0; v < 256; ++v) {
      lo[256 * i + v] = (uint32_t)lbase[bk[i]];
      hi[256 * i + v] = (uint32_t)(lbase[bk[i]] + (active[i] ? h[bk[i]] : 0));
    }
  for (uint32_t d = d0 + 1; d < K && NB > 0; ++d) {
    const uint32_t bi = K - 1 - d;
    if (!(((AND[bi >> 3] ^ OR[bi >> 3]) >> (8 * (bi & 7))) & 255)) continue;  // globally constant digit
    for (int i = 0; i < NB; ++i)
      for (uint32_t v = 0; v < 256; ++v) {
        uint64_t* pk = &probes[2 * (256 * (size_t)i + v)];
        pk[0] = key[2 * i];
        pk[1] = key[2 * i + 1];
        set_digit(pk, K, d, v);
        for (uint32_t dd = d + 1; dd < K; ++dd) set_digit(pk, K, dd, 0);
      }
    {
      std::lock_guard<std::mutex> lk(ctx->mu);
      if ((rs = ops->bounds(ctx, tmp, lo.data(), hi.data(), probes.data(), 256 * NB, st, lt.data(), le.data())))
        return rs;
    }
    if ((rs = tr.allreduce(lt.data(), glt.data(), 256 * (size_t)NB, ROp::Sum, st))) return rs;
    for (int i = 0; i < NB; ++i) {
      if (!active[i]) continue;
      const uint64_t target = Qb[i + 1] - Hbase[bk[i]];  // position of k_g inside bucket b_g
      set_digit(&key[2 * i], K, d, plan_digit(&glt[256 * (size_t)i], target));
    }
  }
  // 5. exact cut points: keys < k_g, then the equal run split by source rank
  for (int i = 0; i < NB; ++i) {
    probes[2 * i] = key[2 * i];
    probes[2 * i + 1] = key[2 * i + 1];
    lo[i] = (uint32_t)lbase[bk[i]];
    hi[i] = (uint32_t)(lbase[bk[i]] + (active[i] ? h[bk[i]] : 0));
  }
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if ((rs = ops->bounds(ctx, tmp, lo.data(), hi.data(), probes.data(), NB, st, lt.data(), le.data()))) return rs;
  }
  std::vector<uint64_t> mine2(2 * (size_t)NB), all2(2 * (size_t)NB * G);
  for (int i = 0; i < NB; ++i) {
    mine2[2 * i] = lt[i];
    mine2[2 * i + 1] = le[i] - lt[i];
  }
  if (NB > 0 && (rs = tr.allgather(mine2.data(), all2.data(), 2 * (size_t)NB, st))) return rs;
  std::vector<uint64_t> cut(G + 1, 0);
  cut[G] = n_local;
  for (int g = 1; g < G; ++g) {
    const int i = g - 1;
    if (!active[i]) {
      cut[g] = n_local;
      continue;
    }
    uint64_t L = Hbase[bk[i]];
    std::vector<uint64_t> e(G), below(G);
    for (int p = 0; p < G; ++p) {
      L += all2[(size_t)p * 2 * NB + 2 * i];
      e[p] = all2[(size_t)p * 2 * NB + 2 * i + 1];
    }
    plan_equal_split(e.data(), G, L, Qb[g], below.data());
    cut[g] = lbase[bk[i]] + lt[i] + below[me];
  }
  for (int g = 1; g <= G; ++g) cut[g] = std::max(cut[g], cut[g - 1]);

  // 6'. fused exchange (the product path when every rank can map its peers'
  // record buffers: NVLink P2P through CUDA IPC, or one device for the
  // loopback ranks).  Otherwise the send/recv exchange below.
  {
    const char* fe = getenv("RADSORT_MULTI_FUSED");
    const bool want = !(fe && fe[0] == '0') && d0 + 1 < K && ops->piece_hist && ops->piece_scatter;
    uint64_t want_all = 0, mine_w = want ? 1 : 0;
    if ((rs = tr.allreduce(&mine_w, &want_all, 1, ROp::Min, st))) return rs;
    if (want_all) {
      std::vector<uint8_t*> peer;
      rs = tr.peer_bases(recs, peer, ctx, st);
      if (rs == RADSORT_OK)
        return fused_exchange(tr, ctx, ops, recs, tmp, n_local, cut, lbase, q, d0, R, K, peer, st, stats, n_out);
      if (rs != RADSORT_ERR_UNSUPPORTED) return rs;
    }
  }

  // 6. exchange.  Each destination's records are contiguous in tmp and grouped
  // by their top digit d0 (step 3); they go out as one message per bucket so
  // that every receiver lands its records bucket by bucket (bucket b from all
  // senders contiguous) and can start its MSD at digit d0 + 1 (step 7).
  std::vector<uint64_t> sc(G), S((size_t)G * G);
  for (int g = 0; g < G; ++g) sc[g] = cut[g + 1] - cut[g];
  if ((rs = tr.allgather(sc.data(), S.data(), G, st))) return rs;
  std::vector<uint64_t> allh((size_t)G * 256), allcut((size_t)G * (G + 1));
  if ((rs = tr.allgather(h, allh.data(), 256, st))) return rs;
  if ((rs = tr.allgather(cut.data(), allcut.data(), (size_t)G + 1, st))) return rs;
  std::vector<Msg> sends, recvs;
  for (int p = 0; p < G; ++p)
    for (int b = 0; b < 256; ++b) {
      const uint64_t lo = std::max(cut[p], lbase[b]), hi = std::min(cut[p + 1], lbase[b + 1]);
      if (hi > lo) sends.push_back({p, lo * R, (hi - lo) * R});
    }
  std::vector<uint32_t> seg_off, seg_len;
  uint64_t got = 0;
  for (int b = 0; b < 256; ++b) {
    const uint64_t b0 = got;
    for (int r = 0; r < G; ++r) {
      const uint64_t* hr = &allh[(size_t)r * 256];
      uint64_t rb = 0;  // start of bucket b on rank r
      for (int u = 0; u < b; ++u) rb += hr[u];
      const uint64_t* cr = &allcut[(size_t)r * (G + 1)];
      const uint64_t lo = std::max(cr[me], rb), hi = std::min(cr[me + 1], rb + hr[b]);
      if (hi > lo) {
        recvs.push_back({r, got * R, (hi - lo) * R});
        got += hi - lo;
      }
    }
    if (got > b0) {
      seg_off.push_back((uint32_t)b0);
      seg_len.push_back((uint32_t)(got - b0));
    }
  }
  if (got != q[me]) {
    set_detail("exchange plan gives %llu records, quota %llu", (unsigned long long)got, (unsigned long long)q[me]);
    return RADSORT_ERR_CUDA;
  }
  if ((rs = tr.exchange(tmp, sends, recs, recvs, st))) return rs;
  stats.exchange = 1;
  stats.nvlink_bytes_sent = (n_local - sc[me]) * R;
  stats.nvlink_bytes_recv = (got - S[(size_t)me * G + me]) * R;

  // 7. local sort of the received key range, from its top-digit buckets on
  radsort_stats sub = {};
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if ((rs = ops->sort_segs(ctx, recs, tmp, (uint32_t)got, seg_off.data(), seg_len.data(), (uint32_t)seg_off.size(),
                             d0 + 1, st, sub)))
      return rs;
  }
  stats.levels = sub.levels;
  stats.scatter_passes = sub.scatter_passes + 1;
  stats.records_scattered = sub.records_scattered + n_local;
  stats.records_hist = sub.records_hist + n_local;
  stats.records_local = sub.records_local;
  stats.records_tiny = sub.records_tiny;
  for (int k = 0; k < RADSORT_K_COUNT; ++k) {
    stats.kernel_launches[k] += sub.kernel_launches[k];
    stats.kernel_ms[k] += sub.kernel_ms[k];
    stats.kernel_bytes[k] += sub.kernel_bytes[k];
  }
  stats.n = got;
  *n_out = got;
  return RADSORT_OK;
}

void set_last_stats(const radsort_stats& s);

}  // namespace radsort

using namespace radsort;

extern "C" {

radsort_status radsort_sort_multi(void* dev_records, void* dev_tmp, uint64_t n_local, uint64_t capacity,
                                  uint64_t* n_out, uint32_t rec_size, uint32_t key_size, void* nccl_comm,
                                  void* stream) {
  if (!nccl_comm || !n_out) {
    set_detail("NULL nccl_comm or n_out");
    return RADSORT_ERR_INVALID_ARG;
  }
  NcclTransport tr((ncclComm_t)nccl_comm);
  radsort_stats s = {};
  s.rec_size = rec_size;
  s.key_size = key_size;
  const radsort_status rs = sort_multi_impl(tr, (uint8_t*)dev_records, (uint8_t*)dev_tmp, n_local, capacity, n_out,
                                            rec_size, key_size, (cudaStream_t)stream, s);
  set_last_stats(s);
  return rs;
}

radsort_status radsort_comm_get_unique_id(void* id_out) {
  if (!id_out) return RADSORT_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  RS_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof id);
  return RADSORT_OK;
}

radsort_status radsort_comm_init(const void* unique_id, int nranks, int rank, int max_ctas, void** comm) {
  if (!unique_id || !comm || nranks < 1 || rank < 0 || rank >= nranks || max_ctas < 0) {
    set_detail("radsort_comm_init: bad arguments");
    return RADSORT_ERR_INVALID_ARG;
  }
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof id);
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  if (max_ctas > 0) {
    cfg.maxCTAs = max_ctas;
    cfg.minCTAs = std::min(cfg.minCTAs > 0 ? cfg.minCTAs : 1, max_ctas);
  }
  ncclComm_t c = nullptr;
  RS_NCCL(ncclCommInitRankConfig(&c, nranks, id, rank, &cfg));
  *comm = c;
  return RADSORT_OK;
}

radsort_status radsort_comm_destroy(void* comm) {
  if (!comm) return RADSORT_ERR_INVALID_ARG;
  RS_NCCL(ncclCommDestroy((ncclComm_t)comm));
  return RADSORT_OK;
}

radsort_status radsort_loopback_create(int nranks, void** group) {
  if (nranks < 1 || !group) return RADSORT_ERR_INVALID_ARG;
  *group = new LoopGroup(nranks);
  return RADSORT_OK;
}

radsort_status radsort_loopback_destroy(void* group) {
  delete static_cast<LoopGroup*>(group);
  return RADSORT_OK;
}

radsort_status radsort_sort_multi_loopback(void* group, int rank, void* dev_records, void* dev_tmp, uint64_t n_local,
                                           uint64_t capacity, uint64_t* n_out, uint32_t rec_size, uint32_t key_size,
                                           void* stream) {
  LoopGroup* g = static_cast<LoopGroup*>(group);
  if (!g || rank < 0 || rank >= g->G || !n_out) return RADSORT_ERR_INVALID_ARG;
  LoopTransport tr(g, rank);
  radsort_stats s = {};
  s.rec_size = rec_size;
  s.key_size = key_size;
  const radsort_status rs = sort_multi_impl(tr, (uint8_t*)dev_records, (uint8_t*)dev_tmp, n_local, capacity, n_out,
                                            rec_size, key_size, (cudaStream_t)stream, s);
  set_last_stats(s);
  return rs;
}

radsort_status radsort_plan_quotas(uint64_t N, int G, uint64_t* quotas) {
  if (G < 1 || !quotas) return RADSORT_ERR_INVALID_ARG;
  plan_quotas(N, G, quotas);
  return RADSORT_OK;
}

radsort_status radsort_plan_digit(const uint64_t* count_lt256, uint64_t q, uint32_t* digit) {
  if (!count_lt256 || !digit || count_lt256[0] > q) return RADSORT_ERR_INVALID_ARG;
  *digit = plan_digit(count_lt256, q);
  return RADSORT_OK;
}

radsort_status radsort_plan_fused(const uint32_t* all_tables, int G, int me, uint32_t npieces, const uint32_t* piece_dst,
                                  const uint32_t* piece_bucket, uint32_t* piece_base, uint64_t* recv_off) {
  if (!all_tables || G < 1 || me < 0 || me >= G || (npieces && (!piece_dst || !piece_bucket || !piece_base)) ||
      !recv_off)
    return RADSORT_ERR_INVALID_ARG;
  for (uint32_t i = 0; i < npieces; ++i)
    if ((int)piece_dst[i] >= G || piece_bucket[i] > 255) return RADSORT_ERR_INVALID_ARG;
  return plan_fused(all_tables, G, me, npieces, piece_dst, piece_bucket, piece_base, recv_off) ? RADSORT_OK
                                                                                                 : RADSORT_ERR_CAPACITY;
}

radsort_status radsort_plan_equal_split(const uint64_t* e, int G, uint64_t L, uint64_t Q, uint64_t* below) {
  if (!e || !below || G < 1) return RADSORT_ERR_INVALID_ARG;
  plan_equal_split(e, G, L, Q, below);
  return RADSORT_OK;
}

}  // extern "C"
