/* radsort.h -- C ABI of radsort, a B200-native MSD radix sort of fixed-size
 * records (the hot path of RADULS2, arXiv 1703.00687).
 *
 * Problem statement (§1): radix sort "works in k phases, each
 * phase is related to sorting keys according to the current digit ... MSD ...
 * starts sorting the data according to the most significant digit. This
 * results in partitioning data into bins that may be further processed
 * independently in the recursive manner."  PAPER.md:116 §3.1: "MSD radix sort
 * with 1 B digits".  Records are fixed-size: a key plus an opaque data field
 * (§4.2 "16 B records (8 B key and 8 B data)"
 * §3.3 record layouts).
 *
 * Record model (reading R1): record i occupies bytes
 * [i*rec_size, (i+1)*rec_size).  Its key is bytes [0, key_size) read as a
 * key_size-byte LITTLE-ENDIAN unsigned integer (key_size = 16: low 8-byte
 * word at +0, high word at +8).  Digit d (d = 0 most significant) is byte
 * key_size-1-d.  Order: unsigned, i.e. lexicographic on digits 0..key_size-1.
 * Bytes [key_size, rec_size) are payload and travel with the key.  The sort is
 * NOT stable: inside an equal-key run any order is a correct result
 * (reading R2).
 *
 * Every function returns a radsort_status; no C++ exception crosses the ABI.
 * All pointers named dev_* are device pointers on the current CUDA device.
 */
#ifndef RADSORT_H_
#define RADSORT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RADSORT_OK = 0,
  RADSORT_ERR_INVALID_ARG = 1,     /* NULL pointer with n > 0, overlap, misalignment, size overflow */
  RADSORT_ERR_UNSUPPORTED = 2,     /* rec_size / key_size combination not built */
  RADSORT_ERR_NOT_INITIALIZED = 3, /* radsort_init not called for the current device */
  RADSORT_ERR_CUDA = 4,            /* a CUDA call failed; detail in radsort_error_string */
  RADSORT_ERR_NCCL = 5,            /* an NCCL call failed (multi-GPU path) */
  RADSORT_ERR_OOM = 6,             /* workspace allocation failed */
  RADSORT_ERR_CAPACITY = 7         /* multi-GPU: output shard would exceed `capacity` */
} radsort_status;

/* Per-call statistics of the last radsort_sort / radsort_sort_multi on the
 * calling thread's device.  Kernel times are filled only when timing is
 * enabled (radsort_set_timing(1)); they are CUDA-event times on the sort's
 * stream, summed over launches of that kernel class. */
enum {
  RADSORT_K_SAMPLE = 0, /* strided sample -> first non-constant digit guess           */
  RADSORT_K_HIST = 1,   /* per-segment digit histogram + key AND/OR (one read)          */
  RADSORT_K_PLAN = 2,   /* constant-digit skip, bin bases, tile map (per segment)       */
  RADSORT_K_SCATTER = 3,/* decoupled-look-back scatter pass (one read + one write)      */
  RADSORT_K_CHILDREN = 4,/* classify child bins; sort tiny ones; copy final ones        */
  RADSORT_K_LOCAL = 5,  /* CTA-local shared-memory sort of a bin <= C records           */
  RADSORT_K_MULTI = 6,  /* multi-GPU exchange-side kernels                               */
  RADSORT_K_GATHER = 7, /* key + index sort: build the (key, index) records, gather the
                           full records in sorted order (wide records, NEXT-1)          */
  RADSORT_K_COUNT = 8
};

typedef struct {
  uint64_t n;                 /* records sorted on this device                          */
  uint32_t rec_size, key_size;
  uint32_t levels;            /* MSD levels executed (host loop iterations)             */
  uint32_t scatter_passes;    /* data-moving segmented scatter launches                 */
  uint32_t constant_digits_skipped; /* leading digits constant over the whole input     */
  uint32_t first_digit;       /* d0: first digit the level-0 scatter used               */
  uint64_t records_scattered; /* sum over scatter launches of records moved             */
  uint64_t records_hist;      /* sum over histogram launches of records read            */
  uint64_t records_local;     /* records finished by the CTA-local sorter               */
  uint64_t records_tiny;      /* records finished by the warp tiny sorter (in CHILDREN) */
  uint64_t records_copied;    /* records of final bins copied tmp -> records            */
  uint64_t bins_large, bins_local, bins_tiny, bins_final; /* children per class         */
  uint64_t nvlink_bytes_sent, nvlink_bytes_recv;          /* multi-GPU exchange         */
  uint32_t kernel_launches[RADSORT_K_COUNT];
  float kernel_ms[RADSORT_K_COUNT];
  uint64_t kernel_bytes[RADSORT_K_COUNT]; /* algorithmic HBM bytes (read + write)      */
  uint64_t bins_split;        /* segments split three ways around a dominant key        */
  uint64_t records_split;     /* records of those dominant keys (final after the split) */
  uint32_t exchange;          /* multi-GPU: 1 = send/recv exchange, 2 = fused exchange
                                 (next-digit scatter straight into the peers' buffers) */
  uint32_t key_index;         /* 1: sorted as (key, index) records + one payload gather */
  uint32_t wide_levels;       /* levels that scattered by a 10-bit digit (digit d plus the
                                 two leading bits of digit d+1; DESIGN.md §3 "wide level") */
} radsort_stats;

/* Create the per-(process, device) context for `device` (cudaSetDevice is the
 * caller's business; this only records the device and queries its
 * attributes).  Idempotent.  The context holds the sort's workspace: the bin
 * lists of the recursion (§1 "bins that may be further processed
 * independently in the recursive manner"; §3.1, the
 * whole-array pass, then small bins, then tiny bins), the per-bin digit
 * histograms and bin bases of each pass, and a small control block.
 *   device   CUDA ordinal, 0 <= device < cudaGetDeviceCount(); else
 *            RADSORT_ERR_INVALID_ARG (RADSORT_ERR_CUDA if CUDA is unusable).
 * Ownership: the library owns the context until radsort_finalize.
 * Environment overrides (read per sort): RADSORT_LOG=1 prints a per-level
 * summary to stderr. */
radsort_status radsort_init(int device);

/* Sort n records in place in dev_records (§3.1 general scheme:
 * whole-array pass by the first digit, then bins by further digits, tiny bins
 * by a comparison sorter).
 *   dev_records  n*rec_size bytes, 16-byte aligned; output = same buffer,
 *                permuted so keys are non-decreasing.
 *   dev_tmp      scratch of >= n*rec_size bytes, 16-byte aligned, must not
 *                overlap dev_records; contents undefined afterwards.
 *   rec_size     8, 16, 24, 32 or 40; built (rec_size, key_size) layouts:
 *                (8,8) (16,8) (16,16) (24,8) (24,16) (32,8) (32,16) (40,16) --
 *                SPEC.md:28-30's five paper layouts (8,0) (8,8) (8,16) (8,24)
 *                (16,0) as (key+data, key) plus the 16-byte-key ones; other
 *                multiples of 8 up to 64 -> RADSORT_ERR_UNSUPPORTED.
 *   key_size     8 or 16, key_size <= rec_size.
 *   stream       cudaStream_t (NULL = legacy default stream) on which all
 *                work is ordered.  The call blocks the host once per MSD level
 *                for a <= 64-byte summary read and returns with the last
 *                kernels possibly still running on `stream`.
 * n = 0 or 1 is a no-op returning RADSORT_OK.  Ownership: the caller owns
 * both buffers; the library owns only its workspace (grown on demand, freed in
 * radsort_finalize).  n must be < 2^32.  Concurrent calls on one device are
 * serialised by an internal mutex. */
radsort_status radsort_sort(void* dev_records, void* dev_tmp, uint64_t n, uint32_t rec_size,
                            uint32_t key_size, void* stream);

/* End-to-end variant on HOST memory: copies host_records (n*rec_size bytes,
 * ideally pinned) to the device, sorts it with radsort_sort, and copies the
 * sorted records back into host_records.  Device buffers come from the
 * library workspace.  Synchronous: returns after the result is in host memory. */
radsort_status radsort_sort_host(void* host_records, uint64_t n, uint32_t rec_size,
                                 uint32_t key_size, void* stream);

/* Streaming end-to-end sort of `nbatch` independent batches on HOST memory
 * (a sequence of sorting problems as stated at PAPER.md:35 §1, each sorted as
 * by radsort_sort): batch k is host_in[k] (n*rec_size bytes, pinned for
 * overlap), its sorted records land in host_out[k] (may equal host_in[k];
 * batches may share one host_out buffer, the copies-out run in batch order).
 * The host<->device copies are pipelined: the copy-in of batch k+1 and the
 * copy-out of batch k-1 run on two internal streams while batch k is sorted
 * on `stream`, so the sustained rate is bounded by the slower copy direction
 * rather than by copy-in + sort + copy-out.  dev_bufs: nbuf >= 2 device record
 * buffers of n*rec_size bytes (batch k is staged in dev_bufs[k % nbuf]; 3
 * overlap the sort too), dev_tmp: one scratch buffer of n*rec_size bytes; all
 * 16-byte aligned and non-overlapping, caller-owned, contents undefined on
 * return.  Synchronous: returns after the last batch is in host memory.
 * Errors as radsort_sort (plus RADSORT_ERR_INVALID_ARG for nbuf < 2 or a NULL
 * pointer); on error, batches already copied out are complete, later ones are
 * undefined. */
radsort_status radsort_sort_host_stream(void* const* host_in, void* const* host_out, uint32_t nbatch,
                                        uint64_t n, uint32_t rec_size, uint32_t key_size,
                                        void* const* dev_bufs, uint32_t nbuf, void* dev_tmp, void* stream);

/* Multi-GPU collective sort (one process per GPU; every rank of nccl_comm
 * calls it with the same rec_size/key_size).  The paper's phase 1 -- "parallel
 * processing of the whole array according to the first digit" (PAPER.md:119
 * §3.1) -- carried across GPUs: the global top-digit histogram (allreduce)
 * gives key-range splitters balanced by record count, one exchange sends every
 * record to the rank owning its key range, and each rank then sorts its bins
 * "independently in the recursive manner" (§1).
 * Input: dev_records[0..n_local).
 * Output: dev_records[0..*n_out) holds this rank's key range; concatenating
 * the ranks' outputs in rank order equals radsort_sort of the concatenated
 * inputs (up to order inside equal-key runs).  Exact-balance quotas:
 * *n_out = floor(N/G) + (rank < N mod G), N = sum of n_local.  Both buffers
 * must hold >= capacity records and capacity >= *n_out, else every rank
 * returns RADSORT_ERR_CAPACITY.  nccl_comm is an ncclComm_t created from the
 * same libnccl this library links (torch's ProcessGroupNCCL._comm_ptr()). */
radsort_status radsort_sort_multi(void* dev_records, void* dev_tmp, uint64_t n_local,
                                  uint64_t capacity, uint64_t* n_out, uint32_t rec_size,
                                  uint32_t key_size, void* nccl_comm, void* stream);

/* Communicator created by the library itself (instead of torch's
 * ProcessGroupNCCL), so that the number of CTAs NCCL occupies during the
 * exchange can be capped and the sort kernels keep the SMs.
 *   radsort_comm_get_unique_id  rank 0 creates the 128-byte id (an
 *                               ncclUniqueId) into id_out; the caller ships
 *                               it to every rank (e.g. a torch broadcast).
 *   radsort_comm_init           collective over nranks ranks; rank in
 *                               [0, nranks); max_ctas = NCCL's maxCTAs
 *                               (0 = NCCL's default).  *comm receives an
 *                               ncclComm_t usable as radsort_sort_multi's
 *                               nccl_comm, on the current device.
 *   radsort_comm_destroy        frees it (after all work on it completed).
 * Errors: NULL pointers / bad rank -> RADSORT_ERR_INVALID_ARG; NCCL failures
 * -> RADSORT_ERR_NCCL with detail. */
radsort_status radsort_comm_get_unique_id(void* id_out);
radsort_status radsort_comm_init(const void* unique_id, int nranks, int rank, int max_ctas, void** comm);
radsort_status radsort_comm_destroy(void* comm);

/* In-process loopback transport for radsort_sort_multi (tests and emulation:
 * the build pool has one GPU per box).  G host threads act as the G ranks on
 * the current device; each calls radsort_sort_multi_loopback with its rank
 * and its own stream and buffers.  Collectives are host barriers; the
 * exchange is device-to-device copies.  Same algorithm as the NCCL path. */
radsort_status radsort_loopback_create(int nranks, void** group);
radsort_status radsort_loopback_destroy(void* group);
radsort_status radsort_sort_multi_loopback(void* group, int rank, void* dev_records, void* dev_tmp, uint64_t n_local,
                                           uint64_t capacity, uint64_t* n_out, uint32_t rec_size, uint32_t key_size,
                                           void* stream);

/* Host planner steps of radsort_sort_multi (pure functions; exposed so the
 * multi-rank host logic can be tested on CPU):
 *   quotas      q_r = floor(N/G) + (r < N mod G)                 (R11)
 *   digit       largest v with count_lt[v] <= q (splitter refinement round)
 *   equal split the first (Q - L) records equal to a boundary key, in
 *               source-rank order, stay below the boundary; below[r] per rank */
radsort_status radsort_plan_quotas(uint64_t N, int G, uint64_t* quotas);
radsort_status radsort_plan_digit(const uint64_t* count_lt256, uint64_t q, uint32_t* digit);
radsort_status radsort_plan_equal_split(const uint64_t* e, int G, uint64_t L, uint64_t Q, uint64_t* below);
/* Fused-exchange plan (SURVEY.md §8(e) k_merge_scatter, §8(f) NEXT-3;
 * PAPER.md:119-121 §3.1, the bins of the first digit processed independently):
 *   all_tables   host, G*G*256*256 uint32: [sender][receiver][d0 bucket][digit
 *                d0+1] = records of that sender's piece for that receiver with
 *                those two digits (every rank's table, allgathered)
 *   me           this rank; npieces, piece_dst[i] (receiver), piece_bucket[i]
 *                (d0 bucket) describe this rank's pieces
 *   piece_base   out, npieces*256 uint32: offset, in receiver piece_dst[i]'s
 *                record buffer, of this rank's share of bin (piece_bucket[i], v);
 *                receivers lay bins out in (d0, d0+1) order, senders in rank
 *                order inside a bin
 *   recv_off     out, 65537 uint64: offsets of rank me's 65536 bins; [65536] =
 *                its record count
 * INVALID_ARG on NULL / out-of-range arguments, CAPACITY when a receiver's
 * count does not fit 32 bits.  Pure host function; the caller owns every buffer. */
radsort_status radsort_plan_fused(const uint32_t* all_tables, int G, int me, uint32_t npieces, const uint32_t* piece_dst,
                                  const uint32_t* piece_bucket, uint32_t* piece_base, uint64_t* recv_off);

/* Splitter planning used by radsort_sort_multi (pure host function, exposed
 * for testing).  Given the GLOBAL (allreduced) 256-bin histogram `hist` of
 * the current digit over a bucket range, per-rank quotas and the global rank
 * q of a boundary already located inside that bucket range, returns the
 * bucket b containing global position q and the count of records in buckets
 * < b (before).  Returns RADSORT_ERR_INVALID_ARG if q >= sum(hist). */
radsort_status radsort_locate_bucket(const uint64_t* hist256, uint64_t q, uint32_t* bucket,
                                     uint64_t* before);

/* Enable (1) / disable (0) per-kernel CUDA-event timing in radsort_stats. */
radsort_status radsort_set_timing(int enable);

/* Statistics of the last sort call on this thread's current device. */
radsort_status radsort_last_stats(radsort_stats* out);

/* Static description of a status plus, for the last failing call on this
 * thread, a detail string (e.g. the CUDA error). */
const char* radsort_error_string(radsort_status s);

/* Free every device's workspace and context.  Safe to call repeatedly. */
void radsort_finalize(void);

/* Library version, e.g. "radsort 0.1 sm_100a". */
const char* radsort_version(void);

/* Run-length "unique key + count" over records sorted by radsort_sort (the
 * k-mer counting step the paper's sorter serves in KMC3).
 * dev_sorted: n records of rec_size bytes, non-decreasing keys (any built
 * layout), n < 2^32.  Output, on the device: dev_keys_out[u] = the u-th
 * distinct key (key_size bytes, same little-endian layout as in a record) and
 * dev_counts_out[u] = its number of records, for u < *n_unique (host).  Both
 * output buffers must hold n entries (the worst case).  Work is ordered on
 * `stream` (a cudaStream_t passed as void*, NULL = legacy default stream); the
 * call returns after synchronizing it (to report *n_unique). */
radsort_status radsort_unique_count(const void* dev_sorted, uint64_t n, uint32_t rec_size, uint32_t key_size,
                                    void* dev_keys_out, uint32_t* dev_counts_out, uint64_t* n_unique,
                                    void* stream);

/* Tiny-sorter benchmark (the GPU analog of PAPER.md:193-232 §4.1, Fig. 1;
 * benchmark infrastructure, not on the sort path): `bins` arrays of n
 * records (rec_size, key_size in {(8,8), (16,8), (16,16), (32,8), (32,16)}),
 * keys sharing their top digit, are sorted in device memory by algorithm
 * `algo` -- 0 enumeration sort (n <= 32), 1 warp bitonic network, 2 warp
 * tail sorter (counting pass + ES among colliders), 3 insertion sort, one
 * thread per array -- for 2 <= n <= 128.  *ns_per_record = best of 3 timed
 * runs (CUDA events) / (bins * n).  The output is checked on the device
 * (RADSORT_ERR_CUDA with detail if any array is out of order).  Allocates
 * and frees its own device memory on the current device. */
radsort_status radsort_tinybench(uint32_t rec_size, uint32_t key_size, uint32_t n, uint32_t algo,
                                 uint64_t bins, double* ns_per_record);

/* One tiny sorter of radsort_tinybench on caller-provided device arrays (test
 * infrastructure for the sorters of PAPER.md:94-104 §2.2 / :159-183 §3.3):
 * dev_in holds `bins` consecutive arrays of n records (2 <= n <= 128; algo 0:
 * n <= 32), the keys of each array sharing their most significant byte (as
 * every bin below the top level does); dev_out (same size, not overlapping)
 * receives each array sorted by key.  Layouts as radsort_tinybench.  Ordered
 * on `stream` (cudaStream_t as void*); returns after enqueueing. */
radsort_status radsort_tinysort(uint32_t rec_size, uint32_t key_size, uint32_t n, uint32_t algo,
                                const void* dev_in, void* dev_out, uint64_t bins, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RADSORT_H_ */
