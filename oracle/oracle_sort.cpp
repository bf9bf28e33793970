// CPU ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may call it; the product
// path never does).  Plain, slow, obviously correct.  Shares no code with the
// CUDA path (paper_1703_00687_b200/csrc) or the input generator (datagen/).
//
// What it computes (§1 "radix sort ... MSD ... starts sorting the
// data according to the most significant digit"; §3.1 "MSD radix
// sort with 1 B digits"; SPEC.md:57 key_compare "unsigned lexicographic
// comparison of key bytes from most significant to least significant;
// equivalently unsigned integer comparison of the full-width key"):
// the input records permuted so that keys are non-decreasing.  The method
// reaches exactly that result (the order inside an equal-key run is
// unspecified, reading R2), so the oracle is that plain
// definition written out: a stable comparison sort on the key (std::stable_sort,
// a library primitive), which makes its own output deterministic.
//
// Record layout (reading R1): bytes [0,K) of a record hold the key
// as a K-byte little-endian unsigned integer; byte K-1 is the most
// significant byte, i.e. digit 0 (SPEC.md:51-53 examples); bytes [K,R) are
// opaque payload carried with the key.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

// Key word w (0 = least significant 8 bytes) of record r.
inline uint64_t key_word(const uint8_t* rec, uint32_t w) {
  uint64_t v;
  std::memcpy(&v, rec + 8 * w, 8);  // little-endian host (x86-64 / aarch64)
  return v;
}

// a < b as unsigned K-byte integers: compare words K/8-1 down to 0
// (for K = 16 "compare high word, then low word", BASELINE.json C4).
inline bool key_less(const uint8_t* a, const uint8_t* b, uint32_t K) {
  for (int w = (int)(K / 8) - 1; w >= 0; --w) {
    uint64_t x = key_word(a, (uint32_t)w), y = key_word(b, (uint32_t)w);
    if (x != y) return x < y;
  }
  return false;
}

inline bool key_equal(const uint8_t* a, const uint8_t* b, uint32_t K) {
  return std::memcmp(a, b, K) == 0;
}

}  // namespace

extern "C" {

// Sorted copy of `in` (n records of R bytes, key = first K bytes) into `out`.
// Returns 0, or -1 on invalid arguments (K, R not multiples of 8, K > R).
int oracle_sort(const uint8_t* in, uint8_t* out, uint64_t n, uint32_t R, uint32_t K) {
  if (R == 0 || K == 0 || R % 8 || K % 8 || K > R) return -1;
  std::vector<uint64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
    return key_less(in + a * R, in + b * R, K);
  });
  for (uint64_t i = 0; i < n; ++i) std::memcpy(out + i * R, in + idx[i] * R, R);
  return 0;
}

// The same stable sort on `threads` host cores (BASELINE.md §4 "all-cores
// variant": the CPU baseline of the benchmark, not a parity reference): T
// contiguous chunks are sorted by std::stable_sort in parallel, then merged in
// ceil(log2 T) rounds of pairwise std::merge (parallel within a round).
// std::merge takes from the left (earlier) range on ties, so the result is the
// stable sort: byte-identical to oracle_sort.  Returns 0, or -1 on bad args.
int oracle_sort_parallel(const uint8_t* in, uint8_t* out, uint64_t n, uint32_t R, uint32_t K, uint32_t threads) {
  if (R == 0 || K == 0 || R % 8 || K % 8 || K > R || threads == 0) return -1;
  const uint64_t T = std::max<uint64_t>(1, std::min<uint64_t>(threads, n / 1024 + 1));
  auto less = [&](uint64_t a, uint64_t b) { return key_less(in + a * R, in + b * R, K); };
  std::vector<uint64_t> idx(n), tmp(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::vector<uint64_t> bound(T + 1);
  for (uint64_t t = 0; t <= T; ++t) bound[t] = n * t / T;
  {
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < T; ++t)
      th.emplace_back([&, t] { std::stable_sort(idx.begin() + bound[t], idx.begin() + bound[t + 1], less); });
    for (auto& x : th) x.join();
  }
  for (uint64_t width = 1; width < T; width *= 2) {  // runs of `width` chunks -> runs of 2*width
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < T; t += 2 * width) {
      const uint64_t a = bound[t], m = bound[std::min(T, t + width)], e = bound[std::min(T, t + 2 * width)];
      th.emplace_back([&, a, m, e] {
        std::merge(idx.begin() + a, idx.begin() + m, idx.begin() + m, idx.begin() + e, tmp.begin() + a, less);
      });
    }
    for (auto& x : th) x.join();
    idx.swap(tmp);
  }
  const uint64_t per = (n + T - 1) / T;
  std::vector<std::thread> th;
  for (uint64_t t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (uint64_t i = t * per; i < std::min(n, (t + 1) * per); ++i) std::memcpy(out + i * R, in + idx[i] * R, R);
    });
  for (auto& x : th) x.join();
  return 0;
}

// Digit d of record rec ("1 B digits"; SPEC.md:45-53 digit_at:
// depth 0 is the most significant byte) = byte K-1-d of the little-endian key.
int oracle_digit(const uint8_t* rec, uint32_t K, uint32_t d) {
  if (d >= K) return -1;
  return rec[K - 1 - d];
}

// Histogram of digit d over n records ("counting sort may be
// applied per single phase"): counts[v] = #{i : digit_d(i) == v}.
int oracle_digit_hist(const uint8_t* in, uint64_t n, uint32_t R, uint32_t K, uint32_t d,
                      uint64_t* counts) {
  if (d >= K || K > R) return -1;
  for (int v = 0; v < 256; ++v) counts[v] = 0;
  for (uint64_t i = 0; i < n; ++i) counts[oracle_digit(in + i * R, K, d)]++;
  return 0;
}

// Rank bounds of one key value in an unsorted array (plain definition of the
// sorted position): in any correct sort, the record at output position i has
// a key k with lt(k) <= i < le(k), lt = #{j: key_j < k}, le = #{j: key_j <= k}.
// Lets full-size results be checked at sampled positions one by one.
int oracle_rank_bounds(const uint8_t* in, uint64_t n, uint32_t R, uint32_t K, const uint8_t* key_rec,
                       uint64_t* lt, uint64_t* le) {
  if (K > R) return -1;
  uint64_t a = 0, b = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint8_t* r = in + i * R;
    if (key_less(r, key_rec, K)) ++a;
    else if (key_equal(r, key_rec, K)) ++b;
  }
  *lt = a;
  *le = a + b;
  return 0;
}

// Three-way key comparison of two single records: -1, 0, +1.
int oracle_key_compare(const uint8_t* a, const uint8_t* b, uint32_t K) {
  if (key_less(a, b, K)) return -1;
  if (key_less(b, a, K)) return 1;
  return 0;
}

// Canonical comparison of a candidate sort result `got` against the oracle
// output `want`: (1) identical key sequence; (2) inside
// every maximal equal-key run of `want`, identical multisets of full records
// (MSD radix sort is not stable).  Returns -1 when equal,
// otherwise the first record index at which they differ (for a multiset
// mismatch: the start of the offending run).
int64_t oracle_compare(const uint8_t* got, const uint8_t* want, uint64_t n, uint32_t R, uint32_t K) {
  for (uint64_t i = 0; i < n; ++i)
    if (!key_equal(got + i * R, want + i * R, K)) return (int64_t)i;
  if (R == K) return -1;
  uint64_t a = 0;
  while (a < n) {
    uint64_t b = a + 1;
    while (b < n && key_equal(want + a * R, want + b * R, K)) ++b;
    if (b - a == 1) {
      if (std::memcmp(got + a * R, want + a * R, R) != 0) return (int64_t)a;
    } else {
      std::vector<std::vector<uint8_t>> x, y;
      for (uint64_t i = a; i < b; ++i) {
        x.emplace_back(got + i * R, got + (i + 1) * R);
        y.emplace_back(want + i * R, want + (i + 1) * R);
      }
      std::sort(x.begin(), x.end());
      std::sort(y.begin(), y.end());
      if (x != y) return (int64_t)a;
    }
    a = b;
  }
  return -1;
}

}
