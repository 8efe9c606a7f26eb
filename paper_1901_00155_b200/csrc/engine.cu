// Host driver and C ABI of the B200 discord-search engine (include/tsdd_cuda.h).
//
// Replaces, for the CUDA engine, the body of tsdd::run_discovery
// (/root/reference/proj/src/pipeline.cpp:53-93): check_config, the preparation
// stage (pipeline.cpp:60-69) and phidd_discord (discovery.cpp:360-373).  All
// arithmetic of the path runs in the kernels of prep_kernels.cu and
// search_kernels.cu; this file owns device memory, launch order, the batched
// HOTSAX outer loop, the top-k passes and the best-so-far exchange between
// ranks.  There is no CPU fallback.

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "tsdd_cuda.h"

namespace {

using namespace tsdd_b200;

struct Failure {
  int code;
  std::string message;
};

[[noreturn]] void fail(int code, const std::string& message) { throw Failure{code, message}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TSDD_ERR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_OK(expr) cuda_check((expr), #expr)

thread_local std::string g_create_error;

template <typename T>
struct DeviceArray {
  T* ptr = nullptr;
  size_t count = 0;
  // grow-only: a context that is prepared again with the same shape allocates nothing
  void alloc(size_t n) {
    if (n == 0) n = 1;
    if (ptr && count >= n) return;
    release();
    CUDA_OK(cudaMalloc(reinterpret_cast<void**>(&ptr), n * sizeof(T)));
    count = n;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    count = 0;
  }
  ~DeviceArray() { release(); }
  DeviceArray() = default;
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
};

inline uint32_t round_up_u32(uint32_t v, uint32_t to) { return (v + to - 1) / to * to; }

inline float float_from_bits(uint32_t bits) {
  float f;
  std::memcpy(&f, &bits, sizeof(f));
  return f;
}

int bits_for(uint64_t max_value) {
  int bits = 1;
  while (bits < 64 && (max_value >> bits) != 0) ++bits;
  return bits;
}

// ---- NCCL, loaded at run time (the torch-bundled libnccl.so.2 when the
// caller is a Python process that imported torch, else the system one) -------
struct NcclApi {
  typedef struct { char internal[128]; } UniqueId;
  typedef void* Comm;
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*CommCount)(Comm, int*) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  void* handle = nullptr;
  static constexpr int kUint8 = 1;   // ncclUint8
  static constexpr int kUint64 = 5;  // ncclUint64
  static constexpr int kMax = 2;     // ncclMax
  static constexpr int kMin = 3;     // ncclMin

  void load() {
    if (handle) return;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* name : names) {
      handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (handle) break;
    }
    if (!handle) fail(TSDD_ERR_RUNTIME, std::string("cannot load libnccl.so.2: ") + dlerror());
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(dlsym(handle, "ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(dlsym(handle, "ncclCommInitRank"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(dlsym(handle, "ncclAllReduce"));
    AllGather = reinterpret_cast<decltype(AllGather)>(dlsym(handle, "ncclAllGather"));
    CommCount = reinterpret_cast<decltype(CommCount)>(dlsym(handle, "ncclCommCount"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(handle, "ncclCommDestroy"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(dlsym(handle, "ncclGetErrorString"));
    if (!GetUniqueId || !CommInitRank || !AllReduce || !AllGather || !CommCount || !CommDestroy || !GetErrorString)
      fail(TSDD_ERR_RUNTIME, "libnccl.so.2 lacks an expected symbol");
  }
  void check(int rc, const char* what) const {
    if (rc != 0) fail(TSDD_ERR_RUNTIME, std::string(what) + ": " + GetErrorString(rc));
  }
};
NcclApi g_nccl;

// Several contexts of ONE process working as ranks (tsdd_cuda_group_create): one host thread
// per context.  The ranks meet in a host barrier; what they exchange stays on the devices — a
// rank reads its peers' arrays straight from their memory (NVLink P2P, or same-device pointers
// when several ranks share a GPU), staged through cudaMemcpyPeer where P2P is unavailable.
struct PeerGroup {
  explicit PeerGroup(int world_) : world(world_), members(static_cast<size_t>(world_), nullptr), slots(static_cast<size_t>(world_)) {}
  const int world;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<tsdd_cuda_ctx*> members;        // by rank; nullptr once a member is destroyed
  std::vector<std::vector<uint64_t>> slots;   // keys of the running max-reduction
  std::vector<uint64_t> merged;
  int arrived = 0;
  uint64_t round = 0;
  bool failed = false;
  bool peer_access = true;                     // every pair of distinct devices can map the other's memory

  // Barrier + element-wise max of `count` keys (count 0: barrier only).  False once any rank has failed.
  bool reduce_max(int rank, uint64_t* keys, size_t count) {
    std::unique_lock<std::mutex> lock(mu);
    if (failed) return false;
    slots[static_cast<size_t>(rank)].assign(keys, keys + count);
    const uint64_t my_round = round;
    if (++arrived == world) {
      merged.assign(count, 0);
      for (const auto& slot : slots)
        for (size_t i = 0; i < count && i < slot.size(); ++i) merged[i] = std::max(merged[i], slot[i]);
      arrived = 0;
      ++round;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return round != my_round || failed; });
      if (round == my_round) return false;  // released by a failure
    }
    for (size_t i = 0; i < count; ++i) keys[i] = merged[i];
    return true;
  }
  void abort() {
    std::lock_guard<std::mutex> lock(mu);
    failed = true;
    cv.notify_all();
  }
};

}  // namespace

struct tsdd_cuda_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  cudaEvent_t ev_prep[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // encode | build rows | summaries+index | end
  std::string error;

  // tunables (tsdd_cuda_set_option)
  uint32_t opt_batch = 1048576;     // (capped by batch_limit(): the batch's dense copy of its rows stays under 2 GB)
  uint32_t opt_first_batch = 128;
  uint32_t opt_batch_growth = 12;
  int opt_rounds = 64;            // upper limit on neighbour ranges per batch
  uint32_t opt_first_range = 8192;  // rows in the first range
  double opt_growth = 2.0;          // each range is this much larger than the one before (dot form: opt_dot_growth)
  int opt_window_rounds = 2;        // same-word-neighbourhood rounds before the covering scan
  uint32_t opt_window_first = 1024; // slots in the first of them
  double opt_window_growth = 3.0;
  bool opt_rotate = true;           // each batch starts its covering scan at a different row
  int opt_mates = 8;
  int opt_mates_form = -1;          // -1: by the input (k_bucket_mates_runs / _f32 / float64); 0 float64, 1 float32, 2 along runs
  int opt_propagate = 8;            // time-topology tries per candidate and call (0 = off)
  int opt_propagate_every = 2;      // ... called again after every this-many-th compaction of a batch (0: only at its start)
  bool opt_rescore = true;
  double opt_margin_delta = -1.0;  // < 0: derive from n (see discard_margin)
  double opt_margin_q = -1.0;      // < 0: derive from n (see quantisation_margin)
  uint32_t opt_finalist_cap = 64;  // finalists the first collection has room for (more: collected again, all settled)
  bool opt_symmetric = true;
  bool opt_packed = true;
  bool opt_wide_tile = false;
  int opt_kernel = 0;
  bool opt_time_kernels = true;
  bool opt_share_bounds = true;
  bool opt_lower_bound = true;      // tile filter by segment-mean lower bounds in the covering scan
  double opt_encode_tol_scale = 1.0;  // k_window_encode4<aligned>: x its tolerance around the breakpoints (0: the exact path only)
  uint32_t opt_seed_rows = 4096;    // rows whose lower bounds seed the best-so-far of the first pass (0 = none)
  // the lower-bound filter on the ws kernel's producer warpgroup (needs tensor_map).  Correct, and
  // faster per term, but its 128-row neighbour tiles rule out and abandon less than k_scan_tiles'
  // 64-row ones: 25 % more terms, 3-5 % slower on workloads 3 and 4 — off by default
  bool opt_lb_in_ws = false;
  bool opt_tile16 = true;           // dot form: 256-candidate tiles, 16 x 8 pairs per thread (k_scan_tiles_ws16)
  bool opt_tensor_map = true;       // covering scans of the ws kernel load tiles as TMA boxes
  int opt_dot = 1;
  double opt_dot_growth = 1.3;      // ... range growth of a dot-form batch: no abandoning inside tiles, so dead
                                    // candidates cost full price until the next compaction — compact more often
  double opt_dot_window_growth = 1.6;
  // ... and of a dot-form batch on the tensor cores: ranges, window rounds and their growth
  double opt_tc_growth = 2.0, opt_tc_window_growth = 2.5;
  int opt_tc_window_rounds = 5;
  int opt_dot_window_rounds = 8;    // ... of a batch in the dot-product form whose window tiles load as tensor-map boxes                  // dot-product form of the ws kernel: 0 never, 1 when it pays, 2 always

  // prepared series
  bool prepared = false;
  size_t m = 0, n = 0, word_len = 0, alphabet = 0;
  uint32_t rows = 0, stride = 0, rows_padded = 0;
  DeviceArray<float> series_f32;
  DeviceArray<double> series, mean, inv_sigma;
  DeviceArray<float> matrix, lb_means, lb_boxes, row_norms, matrix_sorted;
  // tensor-core experiment: the matrix, its hash-sorted copy and the batch split into tf32 parts
  DeviceArray<float> matrix_hi, matrix_lo, sorted_hi, sorted_lo, batch_hi, batch_lo;
  bool split_ready = false, sorted_split_ready = false;
  uint32_t run_pairs = 0;     // slots whose successor in the hash-sorted order is the same word's next row
  // the dot-product form runs on the tensor cores (csrc/tc_kernels.cu) with fp16 hi / lo parts: dot_form 5, the default
  bool opt_tensor_cores = true;
  bool opt_tc_half = true;    // the split parts are fp16 (dot_form 5 / 6) instead of tf32 (3 / 4)
  bool series_is_f32 = false; // series_f32 holds the prepared series' float32 originals (series = the same values, widened)
  bool norms_ready = false;   // row_norms holds the norms of the prepared matrix
  bool sorted_ready = false;  // matrix_sorted holds the prepared matrix in the hash-sorted order
  DeviceArray<uint32_t> hash0, freq, offsets, slot_bucket, scalars, slot_of_row, first_bad;
  DeviceArray<uint32_t> sort_buf[4], order_buf[4];
  uint32_t *sorted_hash = nullptr, *sorted_row = nullptr, *order = nullptr, *sorted_freq = nullptr;
  DeviceArray<uint32_t> scan_scratch, radix_hist;

  // search state
  DeviceArray<uint64_t> nn, best, xchg;
  DeviceArray<uint8_t> exact, excluded;
  DeviceArray<DeviceCounters> counters;
  DeviceArray<uint32_t> flags, batch_rows, batch_alt, batch_slots, batch_slots_alt, sel;
  DeviceArray<float> batch_matrix;
  DeviceArray<double> zrow;
  DeviceArray<uint32_t> finalists, seed_lb, tc_work;
  DeviceArray<uint64_t> finalist_keys;
  DeviceArray<unsigned long long> nn_bits;
  uint32_t batch_capacity = 0;
  bool lb_active = true;    // the lower-bound filter is still worth its (small) cost in this search
  bool lb_decided = false;
  // Dot-product form (k_scan_tiles_ws<.., kDot>): wanted once tiles turn out not to be abandoned
  // anyway; used (and the discard band widened by margin_abs, for the rest of the search) from the
  // first batch on whose best-so-far dwarfs the error bound; dot_now: this batch launches it.
  bool dot_wanted = false, dot_used = false, dot_now = false;
  // tail_now: this batch's covering scans of FEW candidates run on the tensor cores although the search is not in
  // the dot form (the candidates that reach a covering scan of a search whose tiles are abandoned and ruled out are
  // those that must meet every row — the rows around a discord: dense work); the band is widened like for dot_used
  bool tail_now = false;
  int sm_count = 148;
  // The FIRST batch of a search has no best-so-far to size the band against, yet its candidates are the ones that scan
  // every row: it may use the tails on trust (tail_unproven).  The best-so-far it ends with settles it: if that does
  // not dwarf the band after all and tensor-core bounds are out (tail_used), the search starts over without
  // (restart_wanted -> tail_blocked); if none are, the band is simply taken back.
  bool tail_unproven = false, tail_used = false, tail_blocked = false, restart_wanted = false;
  bool opt_tc_tail_first = true;
  bool opt_tc_convert = true;   // tails without split copies: the kernel converts the float32 neighbour rows itself
  bool opt_tc_tail_force = false;
  uint32_t opt_tc_tail_evidence = 64;   // neighbour tiles a CUDA-core segment must have had to count as evidence
  uint64_t lb_launches = 0;  // launches of the kernel with the lower-bound filter in this search (evidence for lb_decided)
  bool opt_tc_tail = true;
  uint32_t opt_tc_tail_most = 1024;  // ... while at most so many candidates are left
  uint32_t* h_sel = nullptr;      // pinned, 4 words + a ring of 4 x 4 words for lagged counts
  cudaEvent_t ev_ring[4] = {nullptr, nullptr, nullptr, nullptr};
  uint64_t* h_keys = nullptr;     // pinned, 4 keys
  double* h_double = nullptr;     // pinned, 1 value
  std::vector<cudaEvent_t> event_pool;
  size_t events_used = 0;
  // TSDD_TRACE=1: one line per tile-kernel launch on stderr after the search (development aid)
  struct LaunchNote {
    int pass;
    uint64_t batch;
    bool window;
    uint32_t k_begin, k_end, count;
    ScanChoice choice;
  };
  std::vector<LaunchNote> trace;
  int cur_pass = 0;

  // ranks
  int world = 1, rank = 0;
  tsdd_exchange_fn exchange_fn = nullptr;
  void* exchange_user = nullptr;
  NcclApi::Comm comm = nullptr;
  std::shared_ptr<PeerGroup> group;  // in-process ranks (tsdd_cuda_group_create)
  DeviceArray<uint64_t> peer_stage;  // staging for peers' bounds where P2P mapping is unavailable
  bool several() const { return world > 1 || comm != nullptr || group != nullptr; }
  uint32_t shard_rows = 0;           // > 0: window statistics / hashes are computed in per-rank slices of this many rows
  bool opt_shard_prep = true;

  tsdd_cuda_stats stats{};

  // Safety factor of the discard test (common.cuh: dead_bound): a float32 distance of n
  // terms is within about n * 2^-24 (relative) of its float64 value; twice that, and at
  // least 4e-6, keeps every row that float32 noise could mis-rank alive until the float64
  // decision.
  float discard_margin() const {
    const double delta = opt_margin_delta >= 0.0 ? opt_margin_delta : std::max(4e-6, 1.2e-7 * static_cast<double>(n));
    return static_cast<float>(1.0 + delta);
  }

  // Rounding the z-normalised rows to float32 moves a squared distance d^2 by up to
  // d sqrt(n) 2^-22 (two rows of norm sqrt(n), relative element error 2^-24, Cauchy-Schwarz);
  // the bound and the best-so-far both carry it: 2 x, and a quarter more for second-order terms.
  // The discard band is widened by this times sqrt(best-so-far) (common.cuh: dead_bound).
  float quantisation_margin() const {
    if (opt_margin_q >= 0.0) return static_cast<float>(opt_margin_q);
    return static_cast<float>(1.25 * std::sqrt(static_cast<double>(n)) * 4.76837158203125e-07);
  }

  // Dot-form distances |a|^2 + |b|^2 - 2 a.b: two FFMA chains of n/2 products of magnitude
  // <= |a||b| <= n, the two norms and three more roundings — within (n + 32) n 2^-24 of the
  // float32 rows' true distance.  The band covers the error of a bound and of the best-so-far.
  double dot_error() const {
    // (x 3 on the tensor cores: the tf32 split drops products below 3 x 2^-20 |a||b| <= 2.9e-6 n, and
    // the float32 accumulation in tensor memory may truncate where the CUDA cores round)
    // (+ n 2^-22: the row norms are those of the float64 rows, k_build_rows; each float32 row's is within 2^-23 of it)
    return (opt_tensor_cores ? 3.0 : 1.0) * (static_cast<double>(n) + 32.0) * static_cast<double>(n) * 5.9604644775390625e-08 +
           static_cast<double>(n) * 2.384185791015625e-07;
  }
  // candidates per batch: the option, with the dense copy of the batch's rows (and its two split twins) kept under 2 GB each
  uint32_t batch_limit() const {
    const uint64_t by_memory = std::max<uint64_t>(4096, (uint64_t{1} << 29) / std::max<uint32_t>(stride, 1u));
    return static_cast<uint32_t>(std::min<uint64_t>(opt_batch, by_memory));
  }
  bool dot_eligible(uint64_t best_key_now) const {
    if (opt_dot == 2) return true;
    const double best_d2 = static_cast<double>(float_from_bits(key_bits(best_key_now)));
    return best_d2 >= 1000.0 * dot_error();  // the band is then below 0.2 % of the best-so-far
  }

  ScanConfig scan_config() const {
    ScanConfig c;
    c.packed = opt_packed;
    c.wide_tile = opt_wide_tile;
    c.variant = opt_packed ? opt_kernel : 1;
    c.tensor_map = opt_tensor_map;
    c.filter_in_ws = opt_lb_in_ws;
    c.tile16 = opt_tile16;
    c.tensor_cores = opt_tensor_cores && split_ready;
    return c;
  }

  SearchState state() {
    SearchState s;
    s.rows = matrix.ptr;
    s.n_rows = rows;
    s.n = static_cast<uint32_t>(n);
    s.stride = stride;
    s.nn = nn.ptr;
    s.exact = exact.ptr;
    s.excluded = excluded.ptr;
    s.best = best.ptr;
    s.counters = counters.ptr;
    s.margin = discard_margin();
    s.margin_abs = dot_used ? static_cast<float>(2.0 * dot_error()) : 0.f;
    s.margin_q = quantisation_margin();
    s.row_norms = norms_ready ? row_norms.ptr : nullptr;
    s.rows_sorted = sorted_ready ? matrix_sorted.ptr : nullptr;
    s.lb_means = (opt_lower_bound && lb_active) ? lb_means.ptr : nullptr;
    s.lb_boxes = lb_boxes.ptr;
    s.lb_scale = static_cast<float>(stride / kLbSegments);
    s.lb_q = 4e-6f * std::sqrt(s.lb_scale);
    return s;
  }
};

namespace {

void bind_device(tsdd_cuda_ctx* ctx) { CUDA_OK(cudaSetDevice(ctx->device)); }

void sync_stream(tsdd_cuda_ctx* ctx) {
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  CUDA_OK(cudaGetLastError());
}

// ------------------------------------------------------------------ validation
// check_config (pipeline.cpp:21-49) with the reference's order and messages:
// series first (series.cpp:10-19), then n, word_len, alphabet, dictionary, and
// feasibility last.  The dictionary guard is 2^32 here (sax.hpp:80 has 2^24).
template <typename T>
void check_series(const T* series, size_t m) {
  if (m == 0 || series == nullptr) fail(TSDD_ERR_VALIDATION, "series is empty");
  for (size_t i = 0; i < m; ++i) {
    if (!std::isfinite(static_cast<double>(series[i])))
      fail(TSDD_ERR_VALIDATION, "non-finite value at index " + std::to_string(i + 1));
  }
}

void check_shape(size_t m, size_t n, size_t word_len, size_t alphabet) {
  if (n < 1 || n > m)
    fail(TSDD_ERR_PARAMETER, "n=" + std::to_string(n) + " must satisfy 1 <= n <= m=" + std::to_string(m));
  if (word_len < 1 || word_len > n)
    fail(TSDD_ERR_PARAMETER,
         "word_len=" + std::to_string(word_len) + " must satisfy 1 <= word_len <= n=" + std::to_string(n));
  if (alphabet < 2 || alphabet > 10)
    fail(TSDD_ERR_PARAMETER, "alphabet cardinality " + std::to_string(alphabet) + " is outside the built-in range 2..10");
  // |A|^w <= 2^32, checked without overflow
  long double dict = 1.0L;
  for (size_t j = 0; j < word_len; ++j) {
    dict *= static_cast<long double>(alphabet);
    if (dict > 4294967296.0L)
      fail(TSDD_ERR_PARAMETER, "dictionary of " + std::to_string(alphabet) + "^" + std::to_string(word_len) +
                                   " words exceeds the 2^32 guard of the device index");
  }
  const size_t rows = m - n + 1;
  if (rows < n + 1)
    fail(TSDD_ERR_INFEASIBLE, "no subsequence has a non-self match: N=" + std::to_string(rows) +
                                  " <= n=" + std::to_string(n) + " (need m >= 2n)");
  if (m > 0xFFFFFF00ull) fail(TSDD_ERR_PARAMETER, "series longer than 2^32 - 256 samples is not supported");
}

uint64_t dict_size_of(size_t word_len, size_t alphabet) {
  uint64_t d = 1;
  for (size_t j = 0; j < word_len; ++j) d *= alphabet;  // <= 2^32 after check_shape
  return d;
}

// ------------------------------------------------------------------ preparation
// All-gather of the per-rank slices of mean / 1/sigma / hash0 (slice s of every array belongs
// to rank s; arrays hold world x slice entries).
void gather_slices(tsdd_cuda_ctx* ctx, uint32_t slice) {
  cudaStream_t st = ctx->stream;
  const size_t at = static_cast<size_t>(slice) * ctx->rank;
  if (ctx->comm) {  // in place: send buffer = receive buffer + rank x count
    g_nccl.check(g_nccl.AllGather(ctx->mean.ptr + at, ctx->mean.ptr, slice * sizeof(double), NcclApi::kUint8, ctx->comm, st),
                 "ncclAllGather(mean)");
    g_nccl.check(g_nccl.AllGather(ctx->inv_sigma.ptr + at, ctx->inv_sigma.ptr, slice * sizeof(double), NcclApi::kUint8,
                                  ctx->comm, st),
                 "ncclAllGather(inv_sigma)");
    g_nccl.check(g_nccl.AllGather(ctx->hash0.ptr + at, ctx->hash0.ptr, slice * sizeof(uint32_t), NcclApi::kUint8,
                                  ctx->comm, st),
                 "ncclAllGather(hash)");
    return;
  }
  PeerGroup& g = *ctx->group;
  sync_stream(ctx);  // this rank's slice is complete ...
  if (!g.reduce_max(ctx->rank, nullptr, 0)) fail(TSDD_ERR_RUNTIME, "another rank of the group failed");  // ... so is everyone's
  for (int r = 0; r < g.world; ++r) {
    if (r == ctx->rank) continue;
    const tsdd_cuda_ctx* other = g.members[static_cast<size_t>(r)];
    if (!other || other->shard_rows != slice || other->rows != ctx->rows)
      fail(TSDD_ERR_RUNTIME, "the ranks of a group must prepare the same series with the same parameters");
    const size_t from = static_cast<size_t>(slice) * r;
    CUDA_OK(cudaMemcpyPeerAsync(ctx->mean.ptr + from, ctx->device, other->mean.ptr + from, other->device,
                                slice * sizeof(double), st));
    CUDA_OK(cudaMemcpyPeerAsync(ctx->inv_sigma.ptr + from, ctx->device, other->inv_sigma.ptr + from, other->device,
                                slice * sizeof(double), st));
    CUDA_OK(cudaMemcpyPeerAsync(ctx->hash0.ptr + from, ctx->device, other->hash0.ptr + from, other->device,
                                slice * sizeof(uint32_t), st));
  }
}

// The SAX-word bucket / frequency / rarity index of the hashes in ctx->hash0 (index.cpp:12-109):
// stable radix sort of (hash, row) -> runs are the buckets; run-length histogram -> frequencies;
// stable sort of (frequency, row) -> rarity order.  Returns the kernels launched.
uint64_t build_index(tsdd_cuda_ctx* ctx) {
  cudaStream_t st = ctx->stream;
  const uint32_t rows = ctx->rows;
  const size_t word_len = ctx->word_len, alphabet = ctx->alphabet;
  uint64_t launches = 0;
  // bucket index: stable sort of (hash, row) -> runs are the buckets
  const size_t longest_scan = std::max<size_t>(rows, radix_sort_scratch_words(rows));
  ctx->scan_scratch.alloc(scan_scratch_words(static_cast<uint32_t>(longest_scan)) + 1024);
  ctx->radix_hist.alloc(radix_sort_scratch_words(rows));
  for (auto& b : ctx->sort_buf) b.alloc(rows);
  for (auto& b : ctx->order_buf) b.alloc(rows);
  CUDA_OK(cudaMemcpyAsync(ctx->sort_buf[0].ptr, ctx->hash0.ptr, rows * sizeof(uint32_t),
                          cudaMemcpyDeviceToDevice, st));
  launches += launch_iota(ctx->sort_buf[1].ptr, rows, st);
  uint32_t *k0 = ctx->sort_buf[0].ptr, *v0 = ctx->sort_buf[1].ptr, *k1 = ctx->sort_buf[2].ptr,
           *v1 = ctx->sort_buf[3].ptr;
  const int hash_bits = bits_for(dict_size_of(word_len, alphabet) - 1);
  launches += launch_radix_sort_pairs(&k0, &v0, &k1, &v1, rows, hash_bits, ctx->radix_hist.ptr,
                                      ctx->scan_scratch.ptr, st);
  ctx->sorted_hash = k0;
  ctx->sorted_row = v0;
  ctx->slot_of_row.alloc(rows);
  launches += launch_invert_order(ctx->sorted_row, rows, ctx->slot_of_row.ptr, st);

  ctx->slot_bucket.alloc(rows);
  ctx->offsets.alloc(static_cast<size_t>(rows) + 1);
  ctx->freq.alloc(rows);
  ctx->scalars.alloc(4);
  CUDA_OK(cudaMemsetAsync(ctx->scalars.ptr, 0, 4 * sizeof(uint32_t), st));
  launches += launch_bucket_index(ctx->sorted_hash, ctx->sorted_row, rows, /*heads=*/k1, ctx->slot_bucket.ptr,
                                  ctx->offsets.ptr, ctx->freq.ptr, ctx->scalars.ptr, ctx->scan_scratch.ptr, st);

  // rarity order: stable sort of (freq, row): rarest words first, ties by position
  CUDA_OK(cudaMemcpyAsync(ctx->order_buf[0].ptr, ctx->freq.ptr, rows * sizeof(uint32_t),
                          cudaMemcpyDeviceToDevice, st));
  launches += launch_iota(ctx->order_buf[1].ptr, rows, st);
  uint32_t *f0 = ctx->order_buf[0].ptr, *o0 = ctx->order_buf[1].ptr, *f1 = ctx->order_buf[2].ptr,
           *o1 = ctx->order_buf[3].ptr;
  launches += launch_radix_sort_pairs(&f0, &o0, &f1, &o1, rows, bits_for(rows), ctx->radix_hist.ptr,
                                      ctx->scan_scratch.ptr, st);
  ctx->sorted_freq = f0;
  ctx->order = o0;
  launches += launch_count_min_freq(ctx->sorted_freq, rows, ctx->scalars.ptr, st);
  launches += launch_count_runs(ctx->sorted_hash, ctx->sorted_row, rows, ctx->scalars.ptr, st);

  return launches;
}

void prepare_on_device(tsdd_cuda_ctx* ctx, size_t m, size_t n, size_t word_len, size_t alphabet) {
  // ctx->series_f32 or ctx->series already holds the samples; `have_f64` says which
  cudaStream_t st = ctx->stream;
  const uint32_t rows = static_cast<uint32_t>(m - n + 1);
  ctx->m = m;
  ctx->n = n;
  ctx->word_len = word_len;
  ctx->alphabet = alphabet;
  ctx->rows = rows;
  ctx->stride = round_up_u32(static_cast<uint32_t>(n), kRowAlign);
  ctx->rows_padded = round_up_u32(rows + 1, kTileRows);  // at least one all-zero row after the last
  uint64_t launches = 0;

  const size_t matrix_floats = static_cast<size_t>(ctx->rows_padded) * ctx->stride;
  if (matrix_floats > ctx->matrix.count) {  // only when the matrix has to grow (cudaMemGetInfo is slow)
    // The float32 matrix dominates the footprint; fail with a clear message instead of a
    // bare cudaMalloc error when the series does not fit this GPU (no CPU fallback).
    size_t free_bytes = 0, total_bytes = 0;
    CUDA_OK(cudaMemGetInfo(&free_bytes, &total_bytes));
    const size_t held = ctx->matrix.count * sizeof(float);  // reused when large enough
    const size_t need = matrix_floats * sizeof(float) + static_cast<size_t>(rows) * 160 + (512u << 20);
    if (need > free_bytes + held)
      fail(TSDD_ERR_RUNTIME, "the subsequence matrix needs " + std::to_string(need >> 20) + " MiB of device memory (N=" +
                                 std::to_string(rows) + " rows x " + std::to_string(ctx->stride) + " floats), " +
                                 std::to_string((free_bytes + held) >> 20) + " MiB are free on device " +
                                 std::to_string(ctx->device));
  }
  // Window statistics and hashes: replicated on one rank; with several ranks that can move device
  // memory between them (NCCL communicator or in-process group) each rank encodes ONE slice of
  // the rows and the slices are all-gathered — 20 bytes a row instead of the float64 arithmetic
  // of every window on every rank (the matrix itself stays replicated: every rank scans all rows).
  const uint32_t world = static_cast<uint32_t>(ctx->world);
  const bool shard = ctx->opt_shard_prep && world > 1 && (ctx->comm || ctx->group);
  const uint32_t slice = shard ? round_up_u32((rows + world - 1) / world, 1024) : rows;
  ctx->shard_rows = shard ? slice : 0;
  const size_t padded_rows = shard ? static_cast<size_t>(slice) * world : rows;
  ctx->mean.alloc(padded_rows);
  ctx->inv_sigma.alloc(padded_rows);
  ctx->hash0.alloc(padded_rows);
  ctx->matrix.alloc(matrix_floats);
  CUDA_OK(cudaEventRecord(ctx->ev_prep[0], st));
  {
    const uint32_t row0 = shard ? std::min<uint64_t>(static_cast<uint64_t>(slice) * ctx->rank, rows) : 0;
    const uint32_t count = shard ? std::min(slice, rows - row0) : rows;
    if (count > 0)
      launches += launch_window_encode(ctx->series.ptr + row0, count, static_cast<uint32_t>(n),
                                       static_cast<uint32_t>(word_len), static_cast<uint32_t>(alphabet),
                                       ctx->mean.ptr + row0, ctx->inv_sigma.ptr + row0, ctx->hash0.ptr + row0, nullptr,
                                       nullptr, st, ctx->opt_encode_tol_scale);
  }
  if (shard) gather_slices(ctx, slice);

  CUDA_OK(cudaEventRecord(ctx->ev_prep[1], st));
  if (ctx->rows_padded > rows)
    CUDA_OK(cudaMemsetAsync(ctx->matrix.ptr + static_cast<size_t>(rows) * ctx->stride, 0,
                            static_cast<size_t>(ctx->rows_padded - rows) * ctx->stride * sizeof(float), st));
  ctx->lb_means.alloc(static_cast<size_t>(rows) * kLbSegments);
  ctx->lb_boxes.alloc(static_cast<size_t>((rows + kLbBoxRows - 1) / kLbBoxRows) * 2 * kLbSegments);
  ctx->row_norms.alloc(static_cast<size_t>(rows) + 1);  // (a by-product of the matrix: the dot-product forms need them)
  launches += launch_build_rows(ctx->series.ptr, ctx->mean.ptr, ctx->inv_sigma.ptr, rows,
                                static_cast<uint32_t>(n), ctx->stride, ctx->matrix.ptr, ctx->lb_means.ptr, st,
                                ctx->row_norms.ptr);
  ctx->norms_ready = true;

  CUDA_OK(cudaEventRecord(ctx->ev_prep[2], st));
  launches += launch_segment_boxes(ctx->lb_means.ptr, rows, ctx->lb_boxes.ptr, st);
  launches += build_index(ctx);
  CUDA_OK(cudaEventRecord(ctx->ev_prep[3], st));

  // search-state storage
  ctx->nn.alloc(rows);
  ctx->best.alloc(1);
  ctx->xchg.alloc(4);
  ctx->exact.alloc(rows);
  ctx->excluded.alloc(rows);
  ctx->counters.alloc(1);
  ctx->flags.alloc(2 * static_cast<size_t>(rows));
  ctx->sel.alloc(4);
  ctx->zrow.alloc(4 * n);   // (up to four finalists are settled per launch)
  ctx->nn_bits.alloc(4);
  ctx->batch_capacity = 0;
  ctx->stats.kernel_launches = launches;
}

void finish_prepare(tsdd_cuda_ctx* ctx) {
  uint32_t scalars[4] = {0, 0, 0, 0};
  CUDA_OK(cudaMemcpyAsync(scalars, ctx->scalars.ptr, sizeof(scalars), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaEventRecord(ctx->ev_b, ctx->stream));
  sync_stream(ctx);
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
  ctx->stats.prep_ms = ms;
  CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_prep[0], ctx->ev_prep[1]));
  ctx->stats.encode_ms = ms;
  CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_prep[1], ctx->ev_prep[2]));
  ctx->stats.build_rows_ms = ms;
  CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_prep[2], ctx->ev_prep[3]));
  ctx->stats.index_ms = ms;
  ctx->stats.rows = ctx->rows;
  ctx->stats.buckets = scalars[0];
  ctx->stats.min_freq_candidates = scalars[1];
  ctx->run_pairs = scalars[2];
  ctx->prepared = true;
  // (a rank of a group must not start another prepare while a peer still copies from its slices)
  if (ctx->group && ctx->shard_rows && !ctx->group->reduce_max(ctx->rank, nullptr, 0))
    fail(TSDD_ERR_RUNTIME, "another rank of the group failed");
}

void reset_stats(tsdd_cuda_ctx* ctx) {
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  ctx->prepared = false;
  ctx->norms_ready = false;
  ctx->series_is_f32 = false;
  ctx->sorted_ready = false;
  ctx->split_ready = false;
  ctx->sorted_split_ready = false;
}

template <typename T>
void prepare_host(tsdd_cuda_ctx* ctx, const T* series, size_t m, size_t n, size_t word_len, size_t alphabet) {
  check_series(series, m);
  check_shape(m, n, word_len, alphabet);
  bind_device(ctx);
  reset_stats(ctx);
  cudaStream_t st = ctx->stream;
  cudaEvent_t ev_h0, ev_h1;
  CUDA_OK(cudaEventCreate(&ev_h0));
  CUDA_OK(cudaEventCreate(&ev_h1));
  ctx->series.alloc(m);
  CUDA_OK(cudaEventRecord(ev_h0, st));
  uint64_t extra = 0;
  if constexpr (sizeof(T) == sizeof(float)) {
    ctx->series_f32.alloc(m);
    CUDA_OK(cudaMemcpyAsync(ctx->series_f32.ptr, series, m * sizeof(float), cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaEventRecord(ev_h1, st));
    CUDA_OK(cudaEventRecord(ctx->ev_a, st));
    extra += launch_widen_series(ctx->series_f32.ptr, ctx->series.ptr, m, nullptr, st);  // (check_series ran on the host)
    ctx->series_is_f32 = true;
  } else {
    CUDA_OK(cudaMemcpyAsync(ctx->series.ptr, series, m * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaEventRecord(ev_h1, st));
    CUDA_OK(cudaEventRecord(ctx->ev_a, st));
  }
  prepare_on_device(ctx, m, n, word_len, alphabet);
  ctx->stats.kernel_launches += extra;
  finish_prepare(ctx);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev_h0, ev_h1);
  ctx->stats.h2d_ms = ms;
  cudaEventDestroy(ev_h0);
  cudaEventDestroy(ev_h1);
}

// ------------------------------------------------------------------ exchange
// In place, element-wise max of `count` (<= 4) keys over all ranks.
void exchange_keys(tsdd_cuda_ctx* ctx, uint64_t* keys, size_t count) {
  if (!ctx->several()) return;
  if (ctx->comm) {
    CUDA_OK(cudaMemcpyAsync(ctx->xchg.ptr, keys, count * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    g_nccl.check(g_nccl.AllReduce(ctx->xchg.ptr, ctx->xchg.ptr, count, NcclApi::kUint64, NcclApi::kMax,
                                  ctx->comm, ctx->stream),
                 "ncclAllReduce");
    CUDA_OK(cudaMemcpyAsync(keys, ctx->xchg.ptr, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync_stream(ctx);
    return;
  }
  if (ctx->group) {
    if (!ctx->group->reduce_max(ctx->rank, keys, count)) fail(TSDD_ERR_RUNTIME, "another rank of the group failed");
    return;
  }
  if (!ctx->exchange_fn) fail(TSDD_ERR_RUNTIME, "world > 1 but no exchange is configured");
  if (ctx->exchange_fn(ctx->exchange_user, keys, count) != 0)
    fail(TSDD_ERR_RUNTIME, "the best-so-far exchange hook reported a failure");
}

// Element-wise MIN of the nn bounds over all ranks.  Every rank scans its own share of the
// candidates, but every scan lowers the bounds of the rows it meets (d(i,j) = d(j,i)); sharing
// them lets each rank discard candidates another rank has already undercut, which keeps the
// pruning of the sharded search at the level of the single-GPU one.  One
// ncclAllReduce(ncclMin, ncclUint64, N) over NVLink per batch: 8 MB at N = 1 M.
void exchange_bounds(tsdd_cuda_ctx* ctx) {
  if (!ctx->opt_share_bounds || !ctx->several()) return;
  if (ctx->comm) {
    g_nccl.check(g_nccl.AllReduce(ctx->nn.ptr, ctx->nn.ptr, ctx->rows, NcclApi::kUint64, NcclApi::kMin, ctx->comm,
                                  ctx->stream),
                 "ncclAllReduce(min)");
    return;
  }
  if (ctx->group) {
    // Device-side min over the peers' arrays.  Every rank first finishes its own batch, then all
    // meet; from then on a peer's nn only ever DEcreases (its next batch's atomicMin), so whatever
    // a read races with is still a valid upper bound.  Each rank's reads complete before it
    // reaches the next barrier (it synchronises its stream there), so nothing is reset under them.
    PeerGroup& g = *ctx->group;
    sync_stream(ctx);
    if (!g.reduce_max(ctx->rank, nullptr, 0)) fail(TSDD_ERR_RUNTIME, "another rank of the group failed");
    PeerPointers peers{};
    for (int r = 0; r < g.world; ++r) {
      if (r == ctx->rank) continue;
      const tsdd_cuda_ctx* other = g.members[static_cast<size_t>(r)];
      if (!other || other->rows != ctx->rows) fail(TSDD_ERR_RUNTIME, "the ranks of a group must prepare the same series");
      if (g.peer_access || other->device == ctx->device) {
        peers.ptr[peers.count++] = other->nn.ptr;
      } else {  // no P2P mapping between the two devices: stage the peer's bounds, then fold them in
        ctx->peer_stage.alloc(ctx->rows);
        CUDA_OK(cudaMemcpyPeerAsync(ctx->peer_stage.ptr, ctx->device, other->nn.ptr, other->device,
                                    static_cast<size_t>(ctx->rows) * sizeof(uint64_t), ctx->stream));
        PeerPointers one{};
        one.ptr[one.count++] = ctx->peer_stage.ptr;
        ctx->stats.kernel_launches += launch_min_from_peers(ctx->nn.ptr, one, ctx->rows, ctx->stream);
      }
    }
    if (peers.count) ctx->stats.kernel_launches += launch_min_from_peers(ctx->nn.ptr, peers, ctx->rows, ctx->stream);
    return;
  }
  // host hook: it only knows max; keys stay below 2^63, so max of (2^63 - 1 - key) is min of key
  constexpr uint64_t kFlip = 0x7FFFFFFFFFFFFFFFull;
  std::vector<uint64_t> keys(ctx->rows);
  CUDA_OK(cudaMemcpyAsync(keys.data(), ctx->nn.ptr, keys.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync_stream(ctx);
  for (uint64_t& key : keys) key = kFlip - key;
  if (ctx->exchange_fn(ctx->exchange_user, keys.data(), keys.size()) != 0)
    fail(TSDD_ERR_RUNTIME, "the bound exchange hook reported a failure");
  for (uint64_t& key : keys) key = kFlip - key;
  CUDA_OK(cudaMemcpyAsync(ctx->nn.ptr, keys.data(), keys.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  sync_stream(ctx);
}

// ------------------------------------------------------------------ search
cudaEvent_t next_event(tsdd_cuda_ctx* ctx) {
  if (ctx->events_used == ctx->event_pool.size()) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreate(&e));
    ctx->event_pool.push_back(e);
  }
  return ctx->event_pool[ctx->events_used++];
}

void ensure_batch_capacity(tsdd_cuda_ctx* ctx, uint32_t batch) {
  const uint32_t padded = round_up_u32(batch, 2 * kTileRows);  // (the 16 x 8 kernel works on 256-candidate tiles)
  if (padded <= ctx->batch_capacity) return;
  ctx->batch_rows.alloc(padded);
  ctx->batch_alt.alloc(padded);
  ctx->batch_slots.alloc(padded);
  ctx->batch_slots_alt.alloc(padded);
  ctx->batch_matrix.alloc(static_cast<size_t>(padded) * ctx->stride);
  if (ctx->opt_tensor_cores && ctx->split_ready) {
    ctx->batch_hi.alloc(static_cast<size_t>(padded) * ctx->stride);
    ctx->batch_lo.alloc(static_cast<size_t>(padded) * ctx->stride);
  } else if (ctx->opt_tensor_cores && ctx->opt_tc_tail) {  // (a tail's candidates: at most opt_tc_tail_most of them)
    const size_t tail_rows = round_up_u32(std::min(padded, ctx->opt_tc_tail_most + 2 * kTileRows), 2 * kTileRows);
    ctx->batch_hi.alloc(tail_rows * ctx->stride);
    ctx->batch_lo.alloc(tail_rows * ctx->stride);
  }
  ctx->batch_capacity = padded;
}

uint32_t read_sel(tsdd_cuda_ctx* ctx) {
  CUDA_OK(cudaMemcpyAsync(ctx->h_sel, ctx->sel.ptr, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  sync_stream(ctx);
  return ctx->h_sel[0];
}

// Neighbour ranges of one batch: `first` rows, then each range `growth` times the one
// before it, at most `rounds` of them (the last takes the rest); boundaries on tile
// multiples.  Dead candidates are dropped between ranges, so a candidate costs at most
// `growth` times the rows it needed to meet a neighbour closer than the best-so-far.
std::vector<uint32_t> range_bounds(uint32_t rows, int rounds, uint32_t first, double growth, bool pruning) {
  std::vector<uint32_t> bounds{0};
  if (pruning) {
    double size = std::max<double>(first, kTileRows);
    uint64_t at = 0;
    for (int r = 1; r < rounds; ++r) {
      at += static_cast<uint64_t>(size) / kTileRows * kTileRows;
      if (at >= rows) break;
      bounds.push_back(static_cast<uint32_t>(at));
      size *= growth;
    }
  }
  bounds.push_back(rows);
  return bounds;
}

inline bool tail_on_possible(const tsdd_cuda_ctx* ctx) { return ctx->split_ready || ctx->opt_tc_convert; }

// The tensor-core form's operands: fp16 (or tf32) hi / lo parts of the matrix and, where it exists, of its
// hash-sorted copy; skipped when memory is short.
void build_split_copies(tsdd_cuda_ctx* ctx, uint32_t batch_now) {
  cudaStream_t st = ctx->stream;
  const size_t floats = static_cast<size_t>(ctx->rows_padded) * ctx->stride;
  const size_t words = ctx->opt_tc_half ? (floats + 1) / 2 : floats;  // (the arrays are float-typed; fp16 parts take half)
  const bool want_main = !ctx->split_ready, want_sorted = ctx->sorted_ready && !ctx->sorted_split_ready;
  if (!want_main && !want_sorted) return;
  size_t free_b = 0, total_b = 0;
  const bool have = (!want_main || ctx->matrix_hi.count >= words) && (!want_sorted || ctx->sorted_hi.count >= words);
  if (!have) CUDA_OK(cudaMemGetInfo(&free_b, &total_b));  // (slow: only when the copies have to grow)
  const size_t need = words * sizeof(float) * ((want_main ? 2 : 0) + (want_sorted ? 2 : 0));
  if (!have && free_b <= need + (size_t{2} << 30)) return;
  if (want_main) {
    ctx->matrix_hi.alloc(words);
    ctx->matrix_lo.alloc(words);
    if (!ctx->norms_ready) {  // one pass over the matrix for both
      ctx->row_norms.alloc(static_cast<size_t>(ctx->rows) + 1);
      ctx->stats.kernel_launches += launch_split_rows_norms(ctx->matrix.ptr, ctx->rows_padded, ctx->stride, ctx->opt_tc_half,
                                                            ctx->matrix_hi.ptr, ctx->matrix_lo.ptr, ctx->row_norms.ptr, ctx->rows + 1, st);
      ctx->norms_ready = true;
    } else {
      ctx->stats.kernel_launches += launch_split_rows(ctx->matrix.ptr, floats, ctx->opt_tc_half, ctx->matrix_hi.ptr, ctx->matrix_lo.ptr, st);
    }
  }
  if (want_sorted) {  // (the hash-sorted copy may come later than the matrix's own split: a tail came first)
    ctx->sorted_hi.alloc(words);
    ctx->sorted_lo.alloc(words);
    ctx->stats.kernel_launches +=
        launch_split_rows(ctx->matrix_sorted.ptr, floats, ctx->opt_tc_half, ctx->sorted_hi.ptr, ctx->sorted_lo.ptr, st);
    ctx->sorted_split_ready = true;
  }
  ctx->split_ready = true;
  const uint32_t capacity = ctx->batch_capacity;
  ctx->batch_capacity = 0;  // (the batch buffers grow their split twins)
  ensure_batch_capacity(ctx, std::max(capacity, batch_now));
}

struct Segment {
  bool window;              // same-word neighbourhood (bounds only) or covering scan
  uint32_t k_begin, k_end;  // neighbour tile numbers
};

// The neighbour tiles one batch visits, in order; dead candidates are dropped between
// segments.  First the window rounds around each candidate tile's own SAX word (the
// HOTSAX inner heuristic), then the covering scan of all rows in growing ranges.
std::vector<Segment> plan_segments(const tsdd_cuda_ctx* ctx, bool pruning) {
  std::vector<Segment> plan;
  const uint32_t tile = kTileRows;  // planning unit: 128 neighbour rows
  const uint32_t slot_tiles = (ctx->rows + tile - 1) / tile;
  if (pruning) {
    // the windows only lower bounds (their rows are met again by the covering scan):
    // keep them to an eighth of the rows
    const uint32_t window_limit = slot_tiles / 8;
    double size = std::max<double>(ctx->opt_window_first, kTileRows);
    uint32_t at = 0;
    // Window tiles of a dot-form batch stream at the full rate of the covering scan (tensor-map
    // boxes from the hash-sorted copy of the matrix), and on the noise-like inputs that run in
    // the dot form more rounds pay; the direct form feeds them with per-row copies.  They also
    // grow more gently there: nothing is abandoned inside a dot-form tile, so a candidate that
    // dies costs full price until the round ends (the widest round of a 3x schedule ran with a
    // quarter of its candidate slots dead).
    const bool dot_windows = ctx->dot_now && ctx->sorted_ready;
    // (on the tensor cores a dead candidate's slot costs a fifth of what it does on the CUDA cores, and a launch with
    // its compaction, gather and time-topology step as much as ever: fewer, wider rounds — cfg 5: 27.0 -> 24.7 ms)
    const bool tc_windows = dot_windows && ctx->opt_tensor_cores && ctx->sorted_split_ready;
    const int window_rounds = tc_windows ? ctx->opt_tc_window_rounds
                              : dot_windows ? std::max(ctx->opt_window_rounds, ctx->opt_dot_window_rounds) : ctx->opt_window_rounds;
    const double window_growth = tc_windows ? ctx->opt_tc_window_growth
                                 : dot_windows ? std::min(ctx->opt_window_growth, ctx->opt_dot_window_growth) : ctx->opt_window_growth;
    for (int r = 0; r < window_rounds && at < window_limit; ++r) {
      const uint32_t upto = std::min<uint64_t>(window_limit, at + static_cast<uint64_t>(size) / tile);
      plan.push_back({true, at, upto});
      at = upto;
      size *= window_growth;
    }
  }
  const std::vector<uint32_t> bounds =
      range_bounds(ctx->rows, ctx->opt_rounds, ctx->opt_first_range,
                   (ctx->dot_now && ctx->opt_tensor_cores && ctx->split_ready) ? ctx->opt_tc_growth
                   : ctx->dot_now ? std::min(ctx->opt_growth, ctx->opt_dot_growth) : ctx->opt_growth, pruning);
  for (size_t r = 0; r + 1 < bounds.size(); ++r)
    plan.push_back({false, bounds[r] / tile, (bounds[r + 1] + tile - 1) / tile});
  return plan;
}

void scan_batch(tsdd_cuda_ctx* ctx, uint32_t count, bool pruning) {
  cudaStream_t st = ctx->stream;
  SearchState s = ctx->state();
  uint64_t launches = 0;

  // word-coherent candidate tiles: sort the batch by slot in the hash-sorted order
  uint32_t *list = ctx->batch_rows.ptr, *list_alt = ctx->batch_alt.ptr;
  uint32_t *slots = ctx->batch_slots.ptr, *slots_alt = ctx->batch_slots_alt.ptr;
  const bool use_windows = pruning && ctx->opt_window_rounds > 0;
  if (use_windows) {
    launches += launch_batch_slots(list, ctx->sel.ptr, ctx->slot_of_row.ptr, count, slots, st);
    launches += launch_radix_sort_pairs(&slots, &list, &slots_alt, &list_alt, count, bits_for(ctx->rows),
                                        ctx->radix_hist.ptr, ctx->scan_scratch.ptr, st);
  }

  // Every batch starts its covering scan somewhere else (golden-ratio steps around the
  // ring of tiles), so that the rows whose bounds drop as a by-product (d(i,j) = d(j,i))
  // are spread over the whole series instead of always being the first ones.
  const uint32_t slot_tiles = (ctx->rows + kTileRows - 1) / kTileRows;
  // (the tensor-core kernel walks 256-row tiles in place: its launches are given the rotated ranges, below)
  const uint32_t rotation =
      (pruning && ctx->opt_rotate)
          ? static_cast<uint32_t>((ctx->stats.batches * 0.6180339887498949 - std::floor(ctx->stats.batches * 0.6180339887498949)) * slot_tiles) % slot_tiles
          : 0u;
  // The live count after each compaction is read back ONE segment late: segment r's grid is
  // sized with the count after compaction r - 1 (an upper bound, candidates only die; surplus
  // CTAs exit at once), so the host never waits for the segment the GPU is working on and
  // the GPU never waits for the host.
  const std::vector<Segment> plan = plan_segments(ctx, pruning);
  struct SegEvent {
    size_t r;
    bool window, tc;
    uint32_t tiles;
    cudaEvent_t e0, e1;
  };
  std::vector<SegEvent> seg_events;  // this batch's tile launches (for the tensor-core tail's decision)
  bool tail_on = false;
  // time topology: before anything else, and again once the window rounds are over
  if (pruning) launches += launch_propagate(s, list, ctx->sel.ptr, count, ctx->opt_propagate, st);
  for (size_t r = 0; r < plan.size(); ++r) {
    if (r > 0 && pruning) {
      launches += launch_compact_batch(s, list, slots, list_alt, slots_alt, pruning, ctx->sel.ptr, count,
                                       ctx->flags.ptr, st);
      std::swap(list, list_alt);
      std::swap(slots, slots_alt);
      // time topology again: the rows around a survivor keep learning (symmetric updates)
      if (ctx->opt_propagate_every > 0 && (r % static_cast<size_t>(ctx->opt_propagate_every) == 0 ||
                                           (plan[r - 1].window && !plan[r].window))) {
        launches += launch_propagate(s, list, ctx->sel.ptr, count, ctx->opt_propagate, st);
        launches += launch_compact_batch(s, list, slots, list_alt, slots_alt, pruning, ctx->sel.ptr, count,
                                         ctx->flags.ptr, st);
        std::swap(list, list_alt);
        std::swap(slots, slots_alt);
      }
      uint32_t* slot_now = ctx->h_sel + 4 + 4 * (r & 3);
      CUDA_OK(cudaMemcpyAsync(slot_now, ctx->sel.ptr, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaEventRecord(ctx->ev_ring[r & 3], st));
      if (r >= 2) {
        CUDA_OK(cudaEventSynchronize(ctx->ev_ring[(r - 1) & 3]));
        count = ctx->h_sel[4 + 4 * ((r - 1) & 3)];
        if (count == 0) break;
      }
    }
    const ScanChoice choice = choose_scan_kernel(ctx->scan_config(), s, count, plan[r].window, pruning, ctx->dot_now);
    ScanChoice choice_now = choice;
    if (choice_now.tc && plan[r].window && !ctx->sorted_split_ready) choice_now.tc = false;  // (no split copy of the sorted matrix)
    if (choice.tc && !choice_now.tc) choice_now.tile16 = ctx->opt_tile16 && count > 192;
    // Tensor-core tail (tail_now): the covering scan of a search that is NOT in the dot form goes on on the tensor
    // cores once that is the cheaper way for what is left of it.  Evidence: the time the latest FINISHED covering
    // segment of this batch took per neighbour tile on the CUDA cores (filter, abandoning and all) against what the
    // tensor cores need for the same tiles — every pair of the tile, about 40 % of their MMA rate — plus, the first
    // time, the price of the split copies of the matrix.  (The early segments are small and cost next to nothing
    // either way; the decision is taken again at every segment until it falls.)
    if (ctx->tail_now && !plan[r].window && !choice_now.tc && !tail_on && count <= ctx->opt_tc_tail_most && ctx->opt_time_kernels) {
      double cuda_ms_per_tile = -1.0;
      for (size_t q = seg_events.size(); q-- > 0;) {  // the latest covering segment whose events have completed
        const SegEvent& ev = seg_events[q];
        if (ev.window || ev.tc || (ev.tiles < ctx->opt_tc_tail_evidence && !ctx->opt_tc_tail_force) || ev.r + 2 > r) continue;  // (a small segment is mostly launch overhead)
        float ms = 0.f;
        if (cudaEventQuery(ev.e1) == cudaSuccess && cudaEventElapsedTime(&ms, ev.e0, ev.e1) == cudaSuccess)
          cuda_ms_per_tile = ms / ev.tiles;
        else
          (void)cudaGetLastError();  // (not finished yet: no evidence this time)
        break;
      }
      if (cuda_ms_per_tile > 0.0) {
        uint64_t tiles_left = 0;
        for (size_t q = r; q < plan.size(); ++q) tiles_left += plan[q].window ? 0 : plan[q].k_end - plan[q].k_begin;
        const double cuda_ms = cuda_ms_per_tile * static_cast<double>(tiles_left);
        const double cand_tiles = std::ceil(count / 128.0);
        // one 128 x 256 tile: 3 MMAs per 16 columns, 128 cycles each at 1.9 GHz, over the SMs, at 40 % of that rate
        const double tile_ms = 3.0 * (ctx->stride / 16.0) * 128.0 / 1.9e6 / ctx->sm_count / (ctx->split_ready ? 0.4 : 0.3);  // (converting: 0.3)
        const double tc_ms = cand_tiles * (tiles_left / 2.0) * tile_ms;
        const double matrix_bytes = static_cast<double>(ctx->rows_padded) * ctx->stride * sizeof(float);
        const double split_ms = (ctx->split_ready || ctx->opt_tc_convert) ? 0.0 : 2.0 * matrix_bytes / 6.0e9;  // (read once, written once, ~6 TB/s)
        if (const char* env = std::getenv("TSDD_TRACE"); env && env[0] == '1')
          std::fprintf(stderr, "tail? batch %llu segment %zu live<=%u: cuda %.3f ms for %llu tiles, tensor cores %.3f ms + split %.3f ms\n",
                       static_cast<unsigned long long>(ctx->stats.batches), r, count, cuda_ms,
                       static_cast<unsigned long long>(tiles_left), tc_ms, split_ms);
        const bool force = ctx->opt_tc_tail_force;  // (tests: switch at the first chance, whatever the estimate says)
        if (force || cuda_ms > ((ctx->split_ready || ctx->opt_tc_convert) ? 1.5 : 2.5) * (tc_ms + split_ms)) {
          if (!ctx->split_ready && !ctx->opt_tc_convert) build_split_copies(ctx, count);
          if (tail_on_possible(ctx) && !ctx->norms_ready) {
            ctx->row_norms.alloc(static_cast<size_t>(ctx->rows) + 1);
            ctx->stats.kernel_launches += launch_row_norms(ctx->matrix.ptr, ctx->rows + 1, ctx->stride, ctx->row_norms.ptr, st);
            ctx->norms_ready = true;
          }
          tail_on = ctx->split_ready || ctx->opt_tc_convert;
          if (tail_on) ctx->tail_used = true;
          s = ctx->state();
        }
      }
    }
    if (tail_on && !plan[r].window && !choice_now.tc && count <= ctx->opt_tc_tail_most) {
      choice_now = ScanChoice{};  // the tensor-core kernel: dot form, tensor-map boxes, no filter, no abandoning
      choice_now.packed = choice.packed;
      choice_now.ws = choice_now.dot = choice_now.tma = choice_now.tc = true;
    }
    const uint32_t padded = round_up_u32(count, choice_now.tile16 ? 2 * kTileRows : kTileRows);
    if (choice_now.tc)
      launches += launch_gather_rows_split(s, list, ctx->sel.ptr, padded, (tail_on && !ctx->split_ready) ? true : ctx->opt_tc_half,
                                           ctx->batch_hi.ptr, ctx->batch_lo.ptr, st);
    else
      launches += launch_gather_rows(s, list, ctx->sel.ptr, padded, choice_now.tile16 ? 2 : choice_now.tma ? 1 : 0,
                                     ctx->batch_matrix.ptr, st);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->opt_time_kernels) {
      e0 = next_event(ctx);
      e1 = next_event(ctx);
      CUDA_OK(cudaEventRecord(e0, st));
    }
    const char* launch_error = nullptr;
    int launched = 0;
    if (choice_now.tc) {
      ctx->tc_work.alloc(1);
      // (a tail of a search without split copies: the kernel makes the neighbours' fp16 parts itself)
      const bool convert = tail_on && !ctx->split_ready && !plan[r].window;
      const TcOperands op{ctx->batch_hi.ptr, ctx->batch_lo.ptr, ctx->matrix_hi.ptr, ctx->matrix_lo.ptr,
                          ctx->sorted_hi.ptr, ctx->sorted_lo.ptr, ctx->rows_padded, convert ? true : ctx->opt_tc_half,
                          ctx->tc_work.ptr, ctx->tail_now && !ctx->dot_now, convert};
      if (plan[r].window || rotation == 0) {
        launched = launch_scan_tiles_tc(s, op, list, slots, ctx->sel.ptr, count, plan[r].window ? ctx->sorted_row : nullptr,
                                        plan[r].k_begin, plan[r].k_end, pruning, ctx->opt_symmetric, st, &launch_error);
      } else {
        // the rows the other kernels reach as units (k + rotation) mod T: one range of the ring, or two where it wraps
        const uint32_t from = (plan[r].k_begin + rotation) % slot_tiles, len = plan[r].k_end - plan[r].k_begin;
        const uint32_t upto = std::min(from + len, slot_tiles);
        launched = launch_scan_tiles_tc(s, op, list, slots, ctx->sel.ptr, count, nullptr, from, upto, pruning,
                                        ctx->opt_symmetric, st, &launch_error);
        if (from + len > slot_tiles && !launch_error)
          launched += launch_scan_tiles_tc(s, op, list, slots, ctx->sel.ptr, count, nullptr, 0, from + len - slot_tiles, pruning,
                                           ctx->opt_symmetric, st, &launch_error);
      }
      if (launched) ctx->stats.scan_kernel_tc_launches += launched;
    } else {
      launched = launch_scan_tiles(choice_now, s, ctx->batch_matrix.ptr, list, slots, ctx->sel.ptr, count,
                                   plan[r].window ? ctx->sorted_row : nullptr, plan[r].k_begin, plan[r].k_end, rotation,
                                   pruning, ctx->opt_symmetric, st, &launch_error);
    }
    if (ctx->opt_time_kernels) CUDA_OK(cudaEventRecord(e1, st));
    if (ctx->opt_time_kernels && launched) seg_events.push_back({r, plan[r].window, choice_now.tc, plan[r].k_end - plan[r].k_begin, e0, e1});
    if (launch_error) fail(TSDD_ERR_RUNTIME, launch_error);
    if (ctx->opt_time_kernels) ctx->trace.push_back({ctx->cur_pass, ctx->stats.batches, plan[r].window, plan[r].k_begin, plan[r].k_end, count, choice_now});
    launches += launched;
    ctx->stats.scan_kernel_launches += launched;
    if (launched && choice_now.lb) ctx->lb_launches += launched;
    if (launched && choice_now.ws) ctx->stats.scan_kernel_ws_launches += launched;
    if (launched && choice_now.dot) ctx->stats.scan_kernel_dot_launches += launched;
  }
  launches += launch_finalize_batch(s, list, ctx->sel.ptr, ctx->batch_capacity, pruning, st);
  ctx->stats.kernel_launches += launches;
  ctx->stats.batches += 1;
}

// Whether early abandoning inside tiles has been worth anything so far in this search
// (< 5 % of the started pair distances were cut short): then the dot-product form, which
// cannot abandon inside a tile but needs half the FP32 instructions, is the better kernel.
// Only asked once the lower-bound filter has been found useless on this input as well (or is
// switched off): where the filter rules tiles out, covering scans stay with it and the dot
// form would only reach the window rounds.
bool few_abandoned(tsdd_cuda_ctx* ctx) {
  if (ctx->opt_lower_bound && !(ctx->lb_decided && !ctx->lb_active)) return false;
  DeviceCounters c{};
  CUDA_OK(cudaMemcpyAsync(&c, ctx->counters.ptr, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
  sync_stream(ctx);
  const unsigned long long calls = c.calls - c.tail_calls;  // (tensor-core tails never abandon: no evidence either way)
  if (ctx->stats.batches < 2) return calls > 0 && c.abandoned == 0;  // after one batch: only if nothing at all
  return calls > 0 && c.abandoned * 20 < calls;
}

// The first batch used the tensor-core tails before there was a best-so-far to size the band against.  `proven`:
// the best-so-far does dwarf the band now.  Returns false when the search has to start over without tails.
bool settle_tail_trust(tsdd_cuda_ctx* ctx, bool proven) {
  ctx->tail_unproven = false;
  if (proven) return true;
  if (!ctx->tail_used) {  // no tensor-core bound is out: take the band back and go on
    ctx->dot_used = false;
    ctx->tail_blocked = true;
    return true;
  }
  ctx->restart_wanted = true;
  return false;
}

// One exact arg-max pass over this rank's share of the rarity order.
uint64_t run_pass(tsdd_cuda_ctx* ctx, bool pruning, int pass) {
  cudaStream_t st = ctx->stream;
  SearchState s = ctx->state();
  uint32_t cursor = 0;
  // Small batches first: the best-so-far rises fastest over the rarest words, and every
  // later candidate is cheaper for it.  Later top-k passes start from a best-so-far that is
  // already seeded with exact rows, so they use full batches at once — every batch leaves a
  // few long-lived survivors that scan the whole series in a part-filled tile, and fewer
  // batches mean fewer such tiles.
  const uint32_t batch_most = ctx->batch_limit();
  uint32_t batch_now = pass == 0 ? std::min(ctx->opt_first_batch, batch_most) : batch_most;
  for (;;) {
    if (cursor < ctx->rows) {
      ensure_batch_capacity(ctx, batch_now);
      ctx->stats.kernel_launches +=
          launch_select_batch(s, ctx->order, cursor, batch_now, static_cast<uint32_t>(ctx->world),
                              static_cast<uint32_t>(ctx->rank), pruning, ctx->flags.ptr, ctx->scan_scratch.ptr,
                              ctx->batch_rows.ptr, ctx->sel.ptr, st);
      const uint32_t count = read_sel(ctx);
      cursor = count == 0 ? ctx->rows : ctx->h_sel[1];
      if (count > 0) {
        // After two batches, see what the lower-bound filter has ruled out so far; on inputs
        // where it finds nothing (noise), the rest of the search runs the kernel without it.
        // (After ONE batch only on the plainest evidence: not a single pair ruled out.  Anything
        // less than that waits for the second batch — cfg 4 looks harmless after its first.)
        if (pruning && ctx->opt_lower_bound && !ctx->lb_decided && ctx->stats.batches >= 1 && ctx->lb_launches > 0) {
          DeviceCounters c{};
          CUDA_OK(cudaMemcpyAsync(&c, ctx->counters.ptr, sizeof(c), cudaMemcpyDeviceToHost, st));
          sync_stream(ctx);
          if (ctx->stats.batches >= 2 || (c.lb_skipped == 0 && c.tile_live > 0)) {
            ctx->lb_active = c.lb_skipped * 20 >= c.lb_skipped + c.tile_live;  // >= 5 % of (candidate, tile) pairs
            ctx->lb_decided = true;
            s = ctx->state();
          }
        }
        if ((pruning && ctx->opt_dot) || ctx->opt_dot == 2) {
          // Dot form or not, for this batch.  One rank decides from its own counters; several
          // agree on `wanted` / `used` in the per-batch exchange below (the band must widen
          // on every rank before dot-form bounds travel between them).
          const bool alone = !ctx->several();
          CUDA_OK(cudaMemcpyAsync(ctx->h_keys + 3, ctx->best.ptr, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
          if (alone && !ctx->dot_wanted && ctx->stats.batches >= 1) ctx->dot_wanted = few_abandoned(ctx);
          sync_stream(ctx);
          const uint64_t best_now = ctx->h_keys[3];
          if (alone && ctx->dot_wanted && ctx->dot_eligible(best_now)) ctx->dot_used = true;
          ctx->dot_now = ctx->dot_wanted && ctx->dot_used && ctx->dot_eligible(best_now);
          // (the same on every rank: the option, and the best-so-far after the exchange)
          const bool proven = key_bits(best_now) != 0 && ctx->dot_eligible(best_now);  // (a seeded bound counts: the final best is no smaller)
          if (ctx->tail_unproven && ctx->stats.batches >= 1) {  // the first batch ran its tails on trust: was it right to?
            if (!settle_tail_trust(ctx, proven)) return 0;
          }
          const bool tails = pruning && ctx->opt_tc_tail && ctx->opt_tensor_cores && !ctx->dot_now && ctx->opt_tensor_map &&
                             !ctx->tail_blocked;
          // (one rank only: whether a tail really ran is each rank's own, timing-dependent decision, and ranks that
          // disagreed on starting over would part ways)
          const bool on_trust = tails && ctx->opt_tc_tail_first && pass == 0 && ctx->stats.batches == 0 && !ctx->dot_used &&
                                !ctx->several();
          ctx->tail_now = tails && ((key_bits(best_now) != 0 && ctx->dot_eligible(best_now)) || on_trust);
          if (on_trust && !proven) ctx->tail_unproven = true;
          if (ctx->tail_now) ctx->dot_used = true;  // the band stays widened from here on
          if (ctx->dot_now && !ctx->norms_ready) {
            ctx->row_norms.alloc(static_cast<size_t>(ctx->rows) + 1);
            ctx->stats.kernel_launches += launch_row_norms(ctx->matrix.ptr, ctx->rows + 1, ctx->stride, ctx->row_norms.ptr, st);
            ctx->norms_ready = true;
          }
          if (ctx->dot_now && !ctx->sorted_ready && ctx->opt_tensor_map && ctx->opt_window_rounds > 0 &&
              ctx->opt_dot_window_rounds > 0) {
            // a second copy of the matrix, in the hash-sorted order, so that window tiles are
            // consecutive rows too (tensor-map loads); skipped when memory is short
            const size_t floats = static_cast<size_t>(ctx->rows_padded) * ctx->stride;
            size_t free_b = 0, total_b = 0;
            if (ctx->matrix_sorted.count < floats) CUDA_OK(cudaMemGetInfo(&free_b, &total_b));  // (slow: only when it has to grow)
            if (ctx->matrix_sorted.count >= floats || free_b > floats * sizeof(float) + (size_t{2} << 30)) {
              ctx->matrix_sorted.alloc(floats);
              ctx->stats.kernel_launches += launch_permute_rows(ctx->matrix.ptr, ctx->sorted_row, ctx->rows,
                                                                ctx->rows_padded, ctx->stride, ctx->matrix_sorted.ptr, st);
              ctx->sorted_ready = true;
            }
          }
          if (ctx->dot_now && ctx->opt_tensor_cores) build_split_copies(ctx, batch_now);  // (whatever of them is missing)
          s = ctx->state();
        }
        ctx->stats.scanned_candidates += count;
        scan_batch(ctx, count, pruning);
      }
      batch_now = static_cast<uint32_t>(std::min<uint64_t>(static_cast<uint64_t>(batch_now) * ctx->opt_batch_growth, batch_most));
    }
    if (ctx->several()) {  // a 1-rank communicator still runs the exchange
      CUDA_OK(cudaMemcpyAsync(ctx->h_keys, ctx->best.ptr, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      sync_stream(ctx);
      ctx->h_keys[1] = cursor < ctx->rows ? 1 : 0;
      ctx->h_keys[2] = 0;
      if (pruning && ctx->opt_dot && !ctx->dot_wanted && ctx->stats.batches >= 1) ctx->h_keys[2] = few_abandoned(ctx) ? 1 : 0;
      exchange_keys(ctx, ctx->h_keys, 3);
      CUDA_OK(cudaMemcpyAsync(ctx->best.ptr, ctx->h_keys, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
      if (ctx->h_keys[2]) ctx->dot_wanted = true;  // the same on every rank, like the best-so-far
      if (pruning && ctx->opt_dot && ctx->dot_wanted && ctx->dot_eligible(ctx->h_keys[0])) ctx->dot_used = true;
      const bool finished = ctx->h_keys[1] == 0;
      if (!finished) exchange_bounds(ctx);
      if (finished) break;
    } else if (cursor >= ctx->rows) {
      break;
    }
  }
  CUDA_OK(cudaMemcpyAsync(ctx->h_keys, ctx->best.ptr, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  sync_stream(ctx);
  if (ctx->tail_unproven) {  // (a pass of one batch)
    const uint64_t best_now = ctx->h_keys[0];
    const bool proven = key_bits(best_now) != 0 && ctx->dot_eligible(best_now);
    if (!settle_tail_trust(ctx, proven)) return 0;
  }
  return ctx->h_keys[0];
}

void collect_search_stats(tsdd_cuda_ctx* ctx) {
  DeviceCounters c{};
  CUDA_OK(cudaMemcpy(&c, ctx->counters.ptr, sizeof(c), cudaMemcpyDeviceToHost));
  ctx->stats.calls = c.calls;
  ctx->stats.abandoned = c.abandoned;
  ctx->stats.terms = c.terms;
  ctx->stats.scan_kernel_terms = c.tile_terms;
  ctx->stats.tiles = c.tiles;
  ctx->stats.tile_live_candidates = c.tile_live;
  ctx->stats.lb_skipped = c.lb_skipped;
  ctx->stats.scan_kernel_dot_terms = c.dot_terms;
  ctx->stats.useful_terms = c.useful_terms;
  ctx->stats.propagated = c.propagated;
  ctx->stats.scan_kernel_tc_terms = c.tc_terms;
  double total = 0.0, total_tc = 0.0;
  for (size_t e = 0; e + 1 < ctx->events_used; e += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->event_pool[e], ctx->event_pool[e + 1]) == cudaSuccess) {
      total += ms;
      if (e / 2 < ctx->trace.size() && ctx->trace[e / 2].choice.tc) total_tc += ms;
    }
  }
  ctx->stats.scan_kernel_ms = total;
  ctx->stats.scan_kernel_tc_ms = total_tc;
  if (const char* env = std::getenv("TSDD_TRACE"); env && env[0] == '1') {
    for (size_t t = 0; t < ctx->trace.size() && 2 * t + 1 < ctx->events_used; ++t) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->event_pool[2 * t], ctx->event_pool[2 * t + 1]);
      const auto& n = ctx->trace[t];
      std::fprintf(stderr, "trace pass %d batch %llu %s tiles %u..%u live<=%u kernel %s%s%s%s%s  %.3f ms\n", n.pass,
                   static_cast<unsigned long long>(n.batch), n.window ? "window" : "cover ", n.k_begin, n.k_end, n.count,
                   n.choice.ws ? "ws" : "cp", n.choice.lb ? "+lb" : "", n.choice.tma ? "+tma" : "",
                   n.choice.dot ? "+dot" : "", n.choice.tc ? "+tc" : n.choice.tile16 ? "+16" : "", ms);
    }
  }
}

void search(tsdd_cuda_ctx* ctx, int k, unsigned flags, uint64_t* positions, double* distances) {
  if (!ctx->prepared) fail(TSDD_ERR_PARAMETER, "tsdd_cuda_search needs a prepared context");
  if (k < 1) fail(TSDD_ERR_PARAMETER, "k must be >= 1, got " + std::to_string(k));
  if (!positions || !distances) fail(TSDD_ERR_PARAMETER, "positions and distances must not be null");
  bind_device(ctx);
  const bool pruning = (flags & TSDD_SEARCH_DISABLE_PRUNING) == 0;
  cudaStream_t st = ctx->stream;
  SearchState s = ctx->state();
  const uint64_t prep_launches = ctx->stats.kernel_launches;
  (void)prep_launches;
  ctx->stats.batches = 0;
  ctx->lb_active = true;
  ctx->lb_decided = false;
  ctx->dot_wanted = ctx->dot_used = ctx->opt_dot == 2;
  ctx->dot_now = false;
  ctx->tail_now = false;
  ctx->tail_unproven = ctx->tail_used = ctx->tail_blocked = ctx->restart_wanted = false;
  ctx->lb_launches = 0;
  ctx->stats.tail_restarts = 0;
  s = ctx->state();
  ctx->stats.scan_kernel_dot_launches = 0;
  ctx->stats.scan_kernel_tc_launches = 0;
  ctx->stats.finalists = 0;
  ctx->stats.exact_reruns = 0;
  ctx->stats.scanned_candidates = 0;
  ctx->stats.scan_kernel_launches = 0;
  ctx->stats.scan_kernel_ws_launches = 0;
  ctx->events_used = 0;
  ctx->trace.clear();

  CUDA_OK(cudaEventRecord(ctx->ev_a, st));
  bool seeded = false;
  auto begin_search = [&] {  // (again when the first batch's trust in the tensor-core tails was misplaced)
    s = ctx->state();
    ctx->stats.kernel_launches += launch_reset_search(s, st);
    if (pruning && ctx->opt_lower_bound && ctx->opt_seed_rows > 0 && s.lb_means != nullptr) {
      // (the seed costs seed_rows x N / 16 box tests: keep it at 1/64 of the rows on small inputs)
      const uint32_t seed_rows = std::min(ctx->opt_seed_rows, std::max(256u, ctx->rows / 64));
      ctx->seed_lb.alloc(2 * static_cast<size_t>(seed_rows));  // (the two-pass seed keeps its selection there)
      ctx->stats.kernel_launches += launch_seed_lower_bound(s, ctx->order, seed_rows, ctx->seed_lb.ptr, st);
      seeded = true;
    }
    if (pruning) {  // (after the seed: a row whose first mates already put it below the seed stops there)
      // Ranks that share their bounds split this stage too (slot p, or 32-slot chunk p, belongs to rank p mod world)
      // and merge the results with the same min-exchange that follows every batch.
      const bool split = ctx->several() && ctx->opt_share_bounds && ctx->opt_mates > 0;
      ctx->stats.kernel_launches += launch_bucket_mates(
          s, ctx->series.ptr, ctx->series_is_f32 ? ctx->series_f32.ptr : nullptr, ctx->mean.ptr, ctx->inv_sigma.ptr, ctx->sorted_row, ctx->slot_bucket.ptr, ctx->offsets.ptr,
          ctx->opt_mates, ctx->run_pairs, split ? static_cast<uint32_t>(ctx->world) : 1u, split ? static_cast<uint32_t>(ctx->rank) : 0u, st,
        ctx->opt_mates_form);
      if (split) exchange_bounds(ctx);
    }

};
  begin_search();

  for (int pass = 0; pass < k; ++pass) {
    ctx->cur_pass = pass;
    if (pass > 0) {
      CUDA_OK(cudaMemsetAsync(ctx->best.ptr, 0, sizeof(uint64_t), st));
      ctx->stats.kernel_launches += launch_seed_best(ctx->state(), st);
    }
    uint64_t key = run_pass(ctx, pruning, pass);
    if (ctx->restart_wanted) {  // the first batch's best-so-far does not dwarf the band of its tensor-core tails: start over without
      ctx->restart_wanted = false;
      ctx->tail_blocked = true;
      ctx->tail_now = ctx->tail_used = ctx->tail_unproven = false;
      ctx->dot_wanted = ctx->dot_used = ctx->opt_dot == 2;
      ctx->dot_now = false;
      ctx->lb_active = true;
      ctx->lb_decided = false;
      ctx->lb_launches = 0;
      ctx->stats.batches = 0;
      ctx->stats.tail_restarts += 1;
      begin_search();
      pass = -1;
      continue;
    }
    if (pass == 0 && seeded && key != 0 && best_key_row(key) == 0xFFFFFFFFu) {
      // no candidate rose above the seeded bound (it can only happen through float32 rounding at
      // an exact tie): drop the seed and let the pass finish on its own best-so-far
      CUDA_OK(cudaMemsetAsync(ctx->best.ptr, 0, sizeof(uint64_t), st));
      ctx->stats.kernel_launches += launch_seed_best(ctx->state(), st);
      key = run_pass(ctx, pruning, pass);
    }
    if (key == 0 || key_bits(key) == 0) {  // nothing beat 0: the reference's fallback (discovery.cpp:90-93)
      positions[pass] = 1;
      distances[pass] = 0.0;
      continue;
    }
    uint32_t row = best_key_row(key);
    double d2 = static_cast<double>(float_from_bits(key_bits(key)));
    if (ctx->opt_rescore) {
      // Decide the pass in float64: every exact row whose float32 nn lies within the safety
      // band of the best-so-far gets its exact nn over all non-self rows, straight from the
      // series; greatest distance wins, ties go to the smaller position.  However many there
      // are, ALL of them are settled (in descending order of their float32 value, so that most
      // of a long list is ruled out by the float64 leader before it costs a kernel).
      s = ctx->state();  // (the band may have widened during the pass: dot form)
      uint32_t cap = std::max<uint32_t>(ctx->opt_finalist_cap, 1);
      uint32_t n_final = 0;
      for (int attempt = 0; attempt < 2; ++attempt) {
        ctx->finalists.alloc(static_cast<size_t>(cap) + 1);
        ctx->finalist_keys.alloc(cap);
        uint32_t* d_count = ctx->finalists.ptr + cap;
        ctx->stats.kernel_launches += launch_collect_finalists(s, ctx->finalists.ptr, cap, d_count, st);
        CUDA_OK(cudaMemcpyAsync(&n_final, d_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        sync_stream(ctx);
        if (n_final <= cap) break;
        cap = n_final;  // collected again with room for all (nothing changes nn / exact / best in between)
      }
      ctx->stats.finalists += n_final;
      std::vector<uint32_t> mine(n_final);
      std::vector<uint64_t> mine_keys(n_final);
      if (n_final > 0) {
        ctx->stats.kernel_launches += launch_gather_keys(s, ctx->finalists.ptr, n_final, ctx->finalist_keys.ptr, st);
        CUDA_OK(cudaMemcpyAsync(mine.data(), ctx->finalists.ptr, n_final * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaMemcpyAsync(mine_keys.data(), ctx->finalist_keys.ptr, n_final * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, st));
        sync_stream(ctx);
      }
      std::vector<uint32_t> by_value(n_final);
      for (uint32_t f = 0; f < n_final; ++f) by_value[f] = f;
      std::sort(by_value.begin(), by_value.end(), [&](uint32_t a, uint32_t b) {
        const uint32_t ka = key_bits(mine_keys[a]), kb = key_bits(mine_keys[b]);
        return ka != kb ? ka > kb : mine[a] < mine[b];
      });
      const double inf64 = std::numeric_limits<double>::infinity();
      auto exact_nn_from = [&](uint32_t cand, double start) -> double {
        unsigned long long bits, start_bits;
        std::memcpy(&start_bits, &start, sizeof(start_bits));
        CUDA_OK(cudaMemcpyAsync(ctx->nn_bits.ptr, &start_bits, sizeof(start_bits), cudaMemcpyHostToDevice, st));
        ctx->stats.kernel_launches +=
            launch_exact_nn(ctx->series.ptr, ctx->mean.ptr, ctx->inv_sigma.ptr, ctx->rows, static_cast<uint32_t>(ctx->n),
                            cand, ctx->zrow.ptr, ctx->opt_lower_bound ? ctx->lb_means.ptr : nullptr, s.lb_scale, s.lb_q,
                            ctx->nn_bits.ptr, st);
        CUDA_OK(cudaMemcpyAsync(&bits, ctx->nn_bits.ptr, sizeof(bits), cudaMemcpyDeviceToHost, st));
        sync_stream(ctx);
        if (bits == start_bits) return inf64;  // no neighbour came in under the start bound
        double exact;
        std::memcpy(&exact, &bits, sizeof(exact));
        return exact;
      };
      double best64 = -1.0;
      uint32_t best_row = 0xFFFFFFFFu;
      // an upper bound of the float64 nn just above the float32 value (relative rounding, the
      // dot form's absolute error, the rows' quantisation), so that most rows abandon early
      auto start_of = [&](uint32_t f) {
        const double nn32 = static_cast<double>(float_from_bits(key_bits(mine_keys[f])));
        return nn32 * static_cast<double>(s.margin) * static_cast<double>(s.margin) + 2.0 * static_cast<double>(s.margin_abs) +
               2.0 * static_cast<double>(s.margin_q) * std::sqrt(nn32);
      };
      auto settle = [&](uint32_t cand, double exact) {
        // the start bound was not one after all (float32 rows further off than the band allows
        // for): measure from +inf rather than report the bound itself
        if (exact == inf64) {
          ctx->stats.exact_reruns += 1;
          exact = exact_nn_from(cand, inf64);
        }
        if (exact == inf64) return;
        if (exact > best64 || (exact == best64 && cand < best_row)) {
          best64 = exact;
          best_row = cand;
        }
      };
      // in descending order of the float32 values, up to four per launch (a group's members cannot rule one
      // another out, the leader of an earlier group can)
      for (size_t at = 0; at < by_value.size();) {
        uint32_t rows_now[4];
        uint32_t idx_now[4];
        double start_now[4];
        uint32_t count_now = 0;
        while (at < by_value.size() && count_now < 4) {
          const uint32_t f = by_value[at++];
          const double start = start_of(f);
          if (start < best64) continue;  // cannot reach the float64 leader
          rows_now[count_now] = mine[f];
          idx_now[count_now] = f;
          start_now[count_now] = start;
          ++count_now;
        }
        if (count_now == 0) break;
        if (count_now == 1) {
          settle(rows_now[0], exact_nn_from(rows_now[0], start_now[0]));
          continue;
        }
        unsigned long long bits[4], start_bits[4];
        std::memcpy(start_bits, start_now, sizeof(double) * count_now);
        CUDA_OK(cudaMemcpyAsync(ctx->nn_bits.ptr, start_bits, sizeof(unsigned long long) * count_now, cudaMemcpyHostToDevice, st));
        ctx->stats.kernel_launches += launch_exact_nn_group(
            ctx->series.ptr, ctx->mean.ptr, ctx->inv_sigma.ptr, ctx->rows, static_cast<uint32_t>(ctx->n), rows_now, count_now,
            ctx->zrow.ptr, ctx->opt_lower_bound ? ctx->lb_means.ptr : nullptr, s.lb_scale, s.lb_q, ctx->nn_bits.ptr, st);
        CUDA_OK(cudaMemcpyAsync(bits, ctx->nn_bits.ptr, sizeof(unsigned long long) * count_now, cudaMemcpyDeviceToHost, st));
        sync_stream(ctx);
        for (uint32_t g = 0; g < count_now; ++g) {
          (void)idx_now[g];
          double exact = inf64;
          if (bits[g] != start_bits[g]) std::memcpy(&exact, &bits[g], sizeof(exact));
          settle(rows_now[g], exact);
        }
      }
      if (ctx->several()) {
        // the finalists are spread over the ranks: greatest float64 distance, then smallest row
        uint64_t value_bits = 0;
        if (best_row != 0xFFFFFFFFu) std::memcpy(&value_bits, &best64, sizeof(value_bits));
        ctx->h_keys[0] = value_bits;
        exchange_keys(ctx, ctx->h_keys, 1);
        const uint64_t global_bits = ctx->h_keys[0];
        ctx->h_keys[0] = (best_row != 0xFFFFFFFFu && value_bits == global_bits) ? 0xFFFFFFFFull - best_row : 0ull;
        exchange_keys(ctx, ctx->h_keys, 1);
        if (global_bits != 0 || ctx->h_keys[0] != 0) {
          std::memcpy(&best64, &global_bits, sizeof(best64));
          best_row = static_cast<uint32_t>(0xFFFFFFFFull - ctx->h_keys[0]);
        }
      }
      if (best_row != 0xFFFFFFFFu) {
        row = best_row;
        d2 = best64;
      }
    }
    positions[pass] = static_cast<uint64_t>(row) + 1;
    distances[pass] = std::sqrt(d2);
    if (pass + 1 < k) ctx->stats.kernel_launches += launch_exclude_zone(ctx->state(), row, st);
  }
  CUDA_OK(cudaEventRecord(ctx->ev_b, st));
  sync_stream(ctx);
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
  ctx->stats.search_ms = ms;
  collect_search_stats(ctx);
}

template <typename Fn>
int guarded(tsdd_cuda_ctx* ctx, Fn&& fn) {
  try {
    fn();
    return TSDD_OK;
  } catch (const Failure& f) {
    if (ctx) ctx->error = f.message;
    else g_create_error = f.message;
    if (ctx && ctx->group) ctx->group->abort();  // release the ranks waiting for this one
    return f.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->error = e.what();
    else g_create_error = e.what();
    if (ctx && ctx->group) ctx->group->abort();
    return TSDD_ERR_RUNTIME;
  }
}

void leave_group(tsdd_cuda_ctx* ctx) {
  if (!ctx->group) return;
  {
    std::lock_guard<std::mutex> lock(ctx->group->mu);
    for (auto& member : ctx->group->members)
      if (member == ctx) member = nullptr;
  }
  ctx->group.reset();
}

template <typename Src, typename Dst>
void fetch_converted(tsdd_cuda_ctx* ctx, const Src* d_src, size_t count, Dst add, void* dst) {
  std::vector<Src> host(count);
  CUDA_OK(cudaMemcpy(host.data(), d_src, count * sizeof(Src), cudaMemcpyDeviceToHost));
  Dst* out = static_cast<Dst*>(dst);
  for (size_t i = 0; i < count; ++i) out[i] = static_cast<Dst>(host[i]) + add;
  (void)ctx;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int tsdd_cuda_create(tsdd_cuda_ctx** out, int device) {
  if (!out) {
    g_create_error = "out must not be null";
    return TSDD_ERR_PARAMETER;
  }
  *out = nullptr;
  tsdd_cuda_ctx* ctx = nullptr;
  const int rc = guarded(nullptr, [&] {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      fail(TSDD_ERR_RUNTIME, std::string("no CUDA device: the engine has no CPU fallback (") +
                                 (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") + ")");
    if (device < 0 || device >= count)
      fail(TSDD_ERR_PARAMETER, "device " + std::to_string(device) + " is outside 0.." + std::to_string(count - 1));
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(TSDD_ERR_RUNTIME, std::string("device '") + prop.name + "' is sm_" + std::to_string(prop.major) +
                                 std::to_string(prop.minor) + "; this library holds sm_100a code only");
    ctx = new tsdd_cuda_ctx();
    ctx->device = device;
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    CUDA_OK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    for (auto& e : ctx->ev_prep) CUDA_OK(cudaEventCreate(&e));
    CUDA_OK(cudaEventCreate(&ctx->ev_a));
    CUDA_OK(cudaEventCreate(&ctx->ev_b));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_sel), 20 * sizeof(uint32_t)));
    for (auto& e : ctx->ev_ring) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_keys), 4 * sizeof(uint64_t)));
    CUDA_OK(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_double), sizeof(double)));
  });
  if (rc != TSDD_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return TSDD_OK;
}

void tsdd_cuda_destroy(tsdd_cuda_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  leave_group(ctx);
  if (ctx->comm) g_nccl.CommDestroy(ctx->comm);
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_prep)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_ring)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  if (ctx->h_sel) cudaFreeHost(ctx->h_sel);
  if (ctx->h_keys) cudaFreeHost(ctx->h_keys);
  if (ctx->h_double) cudaFreeHost(ctx->h_double);
  cudaStream_t st = ctx->own_stream;
  delete ctx;  // frees the device arrays
  if (st) cudaStreamDestroy(st);
}

const char* tsdd_cuda_last_error(const tsdd_cuda_ctx* ctx) {
  return ctx ? ctx->error.c_str() : g_create_error.c_str();
}

int tsdd_cuda_set_stream(tsdd_cuda_ctx* ctx, void* cuda_stream) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    bind_device(ctx);
    sync_stream(ctx);
    ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
  });
}

int tsdd_cuda_set_option(tsdd_cuda_ctx* ctx, const char* name, double value) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    const std::string key = name ? name : "";
    if (key == "batch") {
      if (value < 1 || value > 1048576) fail(TSDD_ERR_PARAMETER, "batch must be in 1..1048576");
      ctx->opt_batch = static_cast<uint32_t>(value);
    } else if (key == "first_batch") {
      if (value < 1 || value > 1048576) fail(TSDD_ERR_PARAMETER, "first_batch must be in 1..1048576");
      ctx->opt_first_batch = static_cast<uint32_t>(value);
    } else if (key == "batch_growth") {
      if (value < 1 || value > 1024) fail(TSDD_ERR_PARAMETER, "batch_growth must be in 1..1024");
      ctx->opt_batch_growth = static_cast<uint32_t>(value);
    } else if (key == "rounds") {
      if (value < 1 || value > 4096) fail(TSDD_ERR_PARAMETER, "rounds must be in 1..4096");
      ctx->opt_rounds = static_cast<int>(value);
    } else if (key == "first_range") {
      if (value < 128 || value > 1e9) fail(TSDD_ERR_PARAMETER, "first_range must be in 128..1e9");
      ctx->opt_first_range = static_cast<uint32_t>(value);
    } else if (key == "window_rounds") {
      if (value < 0 || value > 64) fail(TSDD_ERR_PARAMETER, "window_rounds must be in 0..64");
      ctx->opt_window_rounds = static_cast<int>(value);
    } else if (key == "window_first") {
      if (value < 128 || value > 1e9) fail(TSDD_ERR_PARAMETER, "window_first must be in 128..1e9");
      ctx->opt_window_first = static_cast<uint32_t>(value);
    } else if (key == "window_growth") {
      if (value < 1.0 || value > 16.0) fail(TSDD_ERR_PARAMETER, "window_growth must be in 1..16");
      ctx->opt_window_growth = value;
    } else if (key == "rotate") {
      ctx->opt_rotate = value != 0;
    } else if (key == "growth") {
      if (value < 1.0 || value > 16.0) fail(TSDD_ERR_PARAMETER, "growth must be in 1..16");
      ctx->opt_growth = value;
    } else if (key == "bucket_mates") {
      if (value < 0 || value > 1024) fail(TSDD_ERR_PARAMETER, "bucket_mates must be in 0..1024");
      ctx->opt_mates = static_cast<int>(value);
    } else if (key == "mates_form") {
      if (value != -1 && value != 0 && value != 1 && value != 2) fail(TSDD_ERR_PARAMETER, "mates_form must be -1, 0, 1 or 2");
      ctx->opt_mates_form = static_cast<int>(value);
    } else if (key == "propagate") {
      if (value < 0 || value > 32) fail(TSDD_ERR_PARAMETER, "propagate must be in 0..32");
      ctx->opt_propagate = static_cast<int>(value);
    } else if (key == "propagate_every") {
      if (value < 0 || value > 64) fail(TSDD_ERR_PARAMETER, "propagate_every must be in 0..64");
      ctx->opt_propagate_every = static_cast<int>(value);
    } else if (key == "rescore") {
      ctx->opt_rescore = value != 0;
    } else if (key == "margin_delta") {
      if (value > 0.5) fail(TSDD_ERR_PARAMETER, "margin_delta must be below 0.5 (negative = derive from n)");
      ctx->opt_margin_delta = value;
    } else if (key == "margin_q") {
      if (value > 1.0) fail(TSDD_ERR_PARAMETER, "margin_q must be below 1 (negative = derive from n)");
      ctx->opt_margin_q = value;
    } else if (key == "finalist_cap") {
      if (value < 1 || value > 1048576) fail(TSDD_ERR_PARAMETER, "finalist_cap must be in 1..1048576");
      ctx->opt_finalist_cap = static_cast<uint32_t>(value);
    } else if (key == "symmetric") {
      ctx->opt_symmetric = value != 0;
    } else if (key == "packed") {
      ctx->opt_packed = value != 0;
    } else if (key == "kernel") {
      if (value != 0 && value != 1 && value != 2) fail(TSDD_ERR_PARAMETER, "kernel must be 0, 1 or 2");
      ctx->opt_kernel = static_cast<int>(value);
    } else if (key == "wide_tile") {
      ctx->opt_wide_tile = value != 0;
    } else if (key == "lower_bound") {
      ctx->opt_lower_bound = value != 0;
    } else if (key == "tc_convert") {
      ctx->opt_tc_convert = value != 0;
    } else if (key == "tc_tail_evidence") {
      if (value < 1 || value > 1048576) fail(TSDD_ERR_PARAMETER, "tc_tail_evidence must be in 1..1048576");
      ctx->opt_tc_tail_evidence = static_cast<uint32_t>(value);
    } else if (key == "tc_tail_force") {
      ctx->opt_tc_tail_force = value != 0;
    } else if (key == "tc_tail_first") {
      ctx->opt_tc_tail_first = value != 0;
    } else if (key == "tc_tail") {
      if (value < 0 || value > 1048576) fail(TSDD_ERR_PARAMETER, "tc_tail must be in 0..1048576");
      ctx->opt_tc_tail = value != 0;
      if (value > 1) ctx->opt_tc_tail_most = static_cast<uint32_t>(value);
    } else if (key == "encode_tol_scale") {
      if (value < 0) fail(TSDD_ERR_PARAMETER, "encode_tol_scale must be >= 0");
      ctx->opt_encode_tol_scale = value;
    } else if (key == "seed_rows") {
      if (value < 0 || value > 1048576) fail(TSDD_ERR_PARAMETER, "seed_rows must be in 0..1048576");
      ctx->opt_seed_rows = static_cast<uint32_t>(value);
    } else if (key == "tc_growth") {
      if (value < 1.0 || value > 16.0) fail(TSDD_ERR_PARAMETER, "tc_growth must be in 1..16");
      ctx->opt_tc_growth = value;
    } else if (key == "tc_window_growth") {
      if (value < 1.0 || value > 16.0) fail(TSDD_ERR_PARAMETER, "tc_window_growth must be in 1..16");
      ctx->opt_tc_window_growth = value;
    } else if (key == "tc_window_rounds") {
      if (value < 0 || value > 64) fail(TSDD_ERR_PARAMETER, "tc_window_rounds must be in 0..64");
      ctx->opt_tc_window_rounds = static_cast<int>(value);
    } else if (key == "dot_growth") {
      if (value < 1.0 || value > 16.0) fail(TSDD_ERR_PARAMETER, "dot_growth must be in 1..16");
      ctx->opt_dot_growth = value;
    } else if (key == "dot_window_growth") {
      if (value < 1.0 || value > 16.0) fail(TSDD_ERR_PARAMETER, "dot_window_growth must be in 1..16");
      ctx->opt_dot_window_growth = value;
    } else if (key == "dot_window_rounds") {
      if (value < 0 || value > 64) fail(TSDD_ERR_PARAMETER, "dot_window_rounds must be in 0..64");
      ctx->opt_dot_window_rounds = static_cast<int>(value);
    } else if (key == "dot_tile16") {
      ctx->opt_tile16 = value != 0;
    } else if (key == "filter_in_ws") {
      ctx->opt_lb_in_ws = value != 0;
    } else if (key == "tensor_map") {
      ctx->opt_tensor_map = value != 0;
    } else if (key == "dot_form") {
      if (value != std::floor(value) || value < 0 || value > 6) fail(TSDD_ERR_PARAMETER, "dot_form must be 0 .. 6");
      const int form = static_cast<int>(value);
      ctx->opt_dot = form >= 5 ? form - 4 : form >= 3 ? form - 2 : form;  // 3 / 4 and 5 / 6: as 1 / 2 ...
      ctx->opt_tensor_cores = form >= 3;                                  // ... on the tensor cores,
      if (ctx->opt_tc_half != (form >= 5)) ctx->split_ready = ctx->sorted_split_ready = false;  // (copies in the other format)
      ctx->opt_tc_half = form >= 5;                                       // ... with tf32 (3 / 4) or fp16 (5 / 6) parts
    } else if (key == "shard_prep") {
      ctx->opt_shard_prep = value != 0;
    } else if (key == "share_bounds") {
      ctx->opt_share_bounds = value != 0;
    } else if (key == "time_kernels") {
      ctx->opt_time_kernels = value != 0;
    } else {
      fail(TSDD_ERR_PARAMETER, "unknown option '" + key + "'");
    }
  });
}

int tsdd_cuda_check_config_f32(const float* series, size_t m, size_t n, size_t word_len, size_t alphabet,
                               char* message, size_t message_bytes) {
  try {
    check_series(series, m);
    check_shape(m, n, word_len, alphabet);
  } catch (const Failure& f) {
    if (message && message_bytes) std::snprintf(message, message_bytes, "%s", f.message.c_str());
    return f.code;
  }
  if (message && message_bytes) message[0] = '\0';
  return TSDD_OK;
}

int tsdd_cuda_check_config_f64(const double* series, size_t m, size_t n, size_t word_len, size_t alphabet,
                               char* message, size_t message_bytes) {
  try {
    check_series(series, m);
    check_shape(m, n, word_len, alphabet);
  } catch (const Failure& f) {
    if (message && message_bytes) std::snprintf(message, message_bytes, "%s", f.message.c_str());
    return f.code;
  }
  if (message && message_bytes) message[0] = '\0';
  return TSDD_OK;
}

int tsdd_cuda_prepare_f32(tsdd_cuda_ctx* ctx, const float* series, size_t m, size_t n, size_t word_len,
                          size_t alphabet) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] { prepare_host(ctx, series, m, n, word_len, alphabet); });
}

int tsdd_cuda_prepare_f64(tsdd_cuda_ctx* ctx, const double* series, size_t m, size_t n, size_t word_len,
                          size_t alphabet) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] { prepare_host(ctx, series, m, n, word_len, alphabet); });
}

int tsdd_cuda_prepare_device_f32(tsdd_cuda_ctx* ctx, const float* d_series, size_t m, size_t n,
                                 size_t word_len, size_t alphabet) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (!d_series || m == 0) fail(TSDD_ERR_VALIDATION, "series is empty");
    check_shape(m, n, word_len, alphabet);
    bind_device(ctx);
    reset_stats(ctx);
    ctx->series.alloc(m);
    // unless the caller handed over its stream (tsdd_cuda_set_stream), its work is
    // unordered with ours: wait for everything already queued on the device
    if (ctx->stream == ctx->own_stream) CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaEventRecord(ctx->ev_a, ctx->stream));
    // validate_series (series.cpp:10-19) on the device: the samples never passed through the host
    ctx->first_bad.alloc(1);
    // (a copy of the caller's float32 samples: the caller's buffer is only borrowed for this call)
    ctx->series_f32.alloc(m);
    CUDA_OK(cudaMemcpyAsync(ctx->series_f32.ptr, d_series, m * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->series_is_f32 = true;
    const uint64_t extra = launch_widen_series(d_series, ctx->series.ptr, m, ctx->first_bad.ptr, ctx->stream);
    prepare_on_device(ctx, m, n, word_len, alphabet);
    ctx->stats.kernel_launches += extra;
    uint32_t bad = 0xFFFFFFFFu;
    CUDA_OK(cudaMemcpyAsync(&bad, ctx->first_bad.ptr, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
    finish_prepare(ctx);  // (synchronises the stream)
    if (bad != 0xFFFFFFFFu) {
      ctx->prepared = false;
      fail(TSDD_ERR_VALIDATION, "non-finite value at index " + std::to_string(static_cast<uint64_t>(bad) + 1));
    }
  });
}

int tsdd_cuda_reindex(tsdd_cuda_ctx* ctx, size_t word_len, size_t alphabet) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (!ctx->prepared) fail(TSDD_ERR_PARAMETER, "tsdd_cuda_reindex needs a prepared context");
    check_shape(ctx->m, ctx->n, word_len, alphabet);
    bind_device(ctx);
    cudaStream_t st = ctx->stream;
    ctx->word_len = word_len;
    ctx->alphabet = alphabet;
    ctx->sorted_ready = false;  // (the hash-sorted copy of the matrix follows the OLD order)
    ctx->sorted_split_ready = false;
    ctx->split_ready = false;   // (both split copies are rebuilt together at the next switch to the dot form)
    CUDA_OK(cudaEventRecord(ctx->ev_a, st));
    uint64_t launches = launch_window_encode(ctx->series.ptr, ctx->rows, static_cast<uint32_t>(ctx->n),
                                             static_cast<uint32_t>(word_len), static_cast<uint32_t>(alphabet),
                                             ctx->mean.ptr, ctx->inv_sigma.ptr, ctx->hash0.ptr, nullptr, nullptr, st,
                                             ctx->opt_encode_tol_scale);
    launches += build_index(ctx);
    uint32_t scalars[4] = {0, 0, 0, 0};
    CUDA_OK(cudaMemcpyAsync(scalars, ctx->scalars.ptr, sizeof(scalars), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaEventRecord(ctx->ev_b, st));
    sync_stream(ctx);
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
    ctx->stats.index_ms = ms;
    ctx->stats.prep_ms += ms;
    ctx->stats.kernel_launches += launches;
    ctx->stats.buckets = scalars[0];
    ctx->stats.min_freq_candidates = scalars[1];
    ctx->run_pairs = scalars[2];
  });
}

int tsdd_cuda_fetch_rows(tsdd_cuda_ctx* ctx, size_t first_row, size_t n_rows, float* dst) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (!ctx->prepared) fail(TSDD_ERR_PARAMETER, "tsdd_cuda_fetch_rows needs a prepared context");
    if (!dst) fail(TSDD_ERR_PARAMETER, "dst must not be null");
    if (first_row > ctx->rows || n_rows > ctx->rows - first_row)
      fail(TSDD_ERR_PARAMETER, "rows " + std::to_string(first_row) + " .. " + std::to_string(first_row + n_rows) +
                                   " are outside 0 .. " + std::to_string(ctx->rows));
    bind_device(ctx);
    sync_stream(ctx);
    CUDA_OK(cudaMemcpy(dst, ctx->matrix.ptr + first_row * ctx->stride, n_rows * ctx->stride * sizeof(float),
                       cudaMemcpyDeviceToHost));
  });
}

int tsdd_cuda_search(tsdd_cuda_ctx* ctx, int k, unsigned flags, uint64_t* positions, double* distances) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] { search(ctx, k, flags, positions, distances); });
}

int tsdd_cuda_get_stats(const tsdd_cuda_ctx* ctx, tsdd_cuda_stats* out) {
  if (!ctx || !out) return TSDD_ERR_PARAMETER;
  *out = ctx->stats;
  return TSDD_OK;
}

size_t tsdd_cuda_row_stride(const tsdd_cuda_ctx* ctx) { return ctx ? ctx->stride : 0; }

int tsdd_cuda_fetch(tsdd_cuda_ctx* ctx, int what, void* dst, size_t bytes) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (!ctx->prepared) fail(TSDD_ERR_PARAMETER, "tsdd_cuda_fetch needs a prepared context");
    if (!dst) fail(TSDD_ERR_PARAMETER, "dst must not be null");
    bind_device(ctx);
    sync_stream(ctx);
    const size_t N = ctx->rows, w = ctx->word_len;
    auto expect = [&](size_t want) {
      if (bytes != want)
        fail(TSDD_ERR_PARAMETER, "fetch " + std::to_string(what) + " needs exactly " + std::to_string(want) +
                                     " bytes, got " + std::to_string(bytes));
    };
    switch (what) {
      case TSDD_FETCH_ROWS:
        expect(N * ctx->stride * sizeof(float));
        CUDA_OK(cudaMemcpy(dst, ctx->matrix.ptr, bytes, cudaMemcpyDeviceToHost));
        break;
      case TSDD_FETCH_MEAN:
        expect(N * sizeof(double));
        CUDA_OK(cudaMemcpy(dst, ctx->mean.ptr, bytes, cudaMemcpyDeviceToHost));
        break;
      case TSDD_FETCH_INV_SIGMA:
        expect(N * sizeof(double));
        CUDA_OK(cudaMemcpy(dst, ctx->inv_sigma.ptr, bytes, cudaMemcpyDeviceToHost));
        break;
      case TSDD_FETCH_PAA:
      case TSDD_FETCH_SAX: {
        // not kept resident: re-run the encoder with the optional outputs switched on
        expect(what == TSDD_FETCH_PAA ? N * w * sizeof(double) : N * w * sizeof(uint32_t));
        DeviceArray<double> paa, mean, inv;
        DeviceArray<uint32_t> sax, hash;
        paa.alloc(N * w);
        sax.alloc(N * w);
        mean.alloc(N);
        inv.alloc(N);
        hash.alloc(N);
        launch_window_encode(ctx->series.ptr, ctx->rows, static_cast<uint32_t>(ctx->n), static_cast<uint32_t>(w),
                             static_cast<uint32_t>(ctx->alphabet), mean.ptr, inv.ptr, hash.ptr, paa.ptr, sax.ptr,
                             ctx->stream);
        sync_stream(ctx);
        CUDA_OK(cudaMemcpy(dst, what == TSDD_FETCH_PAA ? static_cast<void*>(paa.ptr) : static_cast<void*>(sax.ptr),
                           bytes, cudaMemcpyDeviceToHost));
        break;
      }
      case TSDD_FETCH_HASH:
        expect(N * sizeof(uint64_t));
        fetch_converted<uint32_t, uint64_t>(ctx, ctx->hash0.ptr, N, 1, dst);
        break;
      case TSDD_FETCH_FREQ:
        expect(N * sizeof(uint32_t));
        CUDA_OK(cudaMemcpy(dst, ctx->freq.ptr, bytes, cudaMemcpyDeviceToHost));
        break;
      case TSDD_FETCH_BUCKETS:
        expect(N * sizeof(uint64_t));
        fetch_converted<uint32_t, uint64_t>(ctx, ctx->sorted_row, N, 1, dst);
        break;
      case TSDD_FETCH_ORDER:
        expect(N * sizeof(uint64_t));
        fetch_converted<uint32_t, uint64_t>(ctx, ctx->order, N, 1, dst);
        break;
      case TSDD_FETCH_CANDIDATES:
        expect(ctx->stats.min_freq_candidates * sizeof(uint64_t));
        fetch_converted<uint32_t, uint64_t>(ctx, ctx->order, ctx->stats.min_freq_candidates, 1, dst);
        break;
      case TSDD_FETCH_NN_SQ: {
        expect(N * sizeof(float));
        std::vector<uint64_t> keys(N);
        CUDA_OK(cudaMemcpy(keys.data(), ctx->nn.ptr, N * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        float* out = static_cast<float*>(dst);
        for (size_t i = 0; i < N; ++i) out[i] = float_from_bits(key_bits(keys[i]));
        break;
      }
      case TSDD_FETCH_NN_EXACT:
        expect(N);
        CUDA_OK(cudaMemcpy(dst, ctx->exact.ptr, N, cudaMemcpyDeviceToHost));
        break;
      default:
        fail(TSDD_ERR_PARAMETER, "unknown fetch selector " + std::to_string(what));
    }
  });
}

int tsdd_cuda_comm_unique_id(char id[128]) {
  return guarded(nullptr, [&] {
    g_nccl.load();
    NcclApi::UniqueId uid;
    g_nccl.check(g_nccl.GetUniqueId(&uid), "ncclGetUniqueId");
    std::memcpy(id, uid.internal, 128);
  });
}

int tsdd_cuda_comm_init(tsdd_cuda_ctx* ctx, const char id[128], int world, int rank) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world) fail(TSDD_ERR_PARAMETER, "need 0 <= rank < world");
    bind_device(ctx);
    g_nccl.load();
    if (ctx->comm) {
      g_nccl.CommDestroy(ctx->comm);
      ctx->comm = nullptr;
    }
    NcclApi::UniqueId uid;
    std::memcpy(uid.internal, id, 128);
    g_nccl.check(g_nccl.CommInitRank(&ctx->comm, world, uid, rank), "ncclCommInitRank");
    leave_group(ctx);
    ctx->world = world;
    ctx->rank = rank;
    ctx->exchange_fn = nullptr;
  });
}

int tsdd_cuda_comm_size(const tsdd_cuda_ctx* ctx, int* nranks) {
  if (!ctx || !nranks) return TSDD_ERR_PARAMETER;
  *nranks = ctx->world;
  if (ctx->comm) {  // what NCCL itself says about the communicator
    int count = 0;
    if (g_nccl.CommCount(ctx->comm, &count) != 0) return TSDD_ERR_RUNTIME;
    *nranks = count;
  }
  return TSDD_OK;
}

int tsdd_cuda_group_create(tsdd_cuda_ctx** ctxs, int world) {
  if (!ctxs || world < 1 || world > kMaxPeers + 1) return TSDD_ERR_PARAMETER;
  for (int r = 0; r < world; ++r)
    if (!ctxs[r]) return TSDD_ERR_PARAMETER;
  return guarded(ctxs[0], [&] {
    auto group = std::make_shared<PeerGroup>(world);
    for (int r = 0; r < world; ++r) {
      for (int q = 0; q < r; ++q)
        if (ctxs[q] == ctxs[r]) fail(TSDD_ERR_PARAMETER, "a context can be only one rank of a group");
      group->members[static_cast<size_t>(r)] = ctxs[r];
    }
    // map every other device's memory where the hardware can (NVLink / NVSwitch, or PCIe P2P)
    for (int r = 0; r < world; ++r) {
      for (int q = 0; q < world; ++q) {
        const int a = ctxs[r]->device, b = ctxs[q]->device;
        if (a == b) continue;
        int can = 0;
        CUDA_OK(cudaDeviceCanAccessPeer(&can, a, b));
        if (!can) {
          group->peer_access = false;
          continue;
        }
        CUDA_OK(cudaSetDevice(a));
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
        (void)cudaGetLastError();
      }
    }
    for (int r = 0; r < world; ++r) {
      tsdd_cuda_ctx* ctx = ctxs[r];
      leave_group(ctx);
      if (ctx->comm) {
        g_nccl.CommDestroy(ctx->comm);
        ctx->comm = nullptr;
      }
      ctx->exchange_fn = nullptr;
      ctx->world = world;
      ctx->rank = r;
      ctx->group = world > 1 ? group : nullptr;
    }
  });
}

int tsdd_cuda_set_exchange(tsdd_cuda_ctx* ctx, tsdd_exchange_fn fn, void* user, int world, int rank) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world) fail(TSDD_ERR_PARAMETER, "need 0 <= rank < world");
    if (world > 1 && !fn) fail(TSDD_ERR_PARAMETER, "world > 1 needs an exchange function");
    if (ctx->comm) {
      g_nccl.CommDestroy(ctx->comm);
      ctx->comm = nullptr;
    }
    leave_group(ctx);
    ctx->exchange_fn = fn;
    ctx->exchange_user = user;
    ctx->world = world;
    ctx->rank = rank;
  });
}

int tsdd_cuda_fp32_probe(tsdd_cuda_ctx* ctx, int which, double* ops_per_s, double* ms_out) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (which >= 16 && which <= 19) {  // packed + scalar mixes (see probe_kernels.cu)
      bind_device(ctx);
      const int blocks = 148 * 8, iters = 4096;
      DeviceArray<float> sink;
      sink.alloc(static_cast<size_t>(blocks) * 256);
      launch_fp32_probe(which, sink.ptr, blocks, 64, ctx->stream);
      float best_ms = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        CUDA_OK(cudaEventRecord(ctx->ev_a, ctx->stream));
        launch_fp32_probe(which, sink.ptr, blocks, iters, ctx->stream);
        CUDA_OK(cudaEventRecord(ctx->ev_b, ctx->stream));
        sync_stream(ctx);
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
        best_ms = std::min(best_ms, ms);
      }
      if (ops_per_s) *ops_per_s = fp32_probe_ops(which, blocks, iters) / (best_ms * 1e-3);
      if (ms_out) *ms_out = best_ms;
      return;
    }
    if (which < 0 || which > 11) fail(TSDD_ERR_PARAMETER, "probe selector must be 0..11 or 16..19");
    bind_device(ctx);
    // 0..3: 64 warps per SM; 4..7: the same mixes at 8 warps per SM (the 128 x 128 tile
    // kernel's occupancy); 8..11: at 16 warps per SM (the 128 x 64 tile kernel's)
    const int blocks = which < 4 ? 148 * 8 : which < 8 ? 148 : 148 * 2;
    const int iters = 4096;
    which &= 3;
    DeviceArray<float> sink;
    sink.alloc(static_cast<size_t>(blocks) * 256);
    launch_fp32_probe(which, sink.ptr, blocks, 64, ctx->stream);  // warm-up
    float best_ms = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CUDA_OK(cudaEventRecord(ctx->ev_a, ctx->stream));
      launch_fp32_probe(which, sink.ptr, blocks, iters, ctx->stream);
      CUDA_OK(cudaEventRecord(ctx->ev_b, ctx->stream));
      sync_stream(ctx);
      float ms = 0.f;
      CUDA_OK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
      best_ms = std::min(best_ms, ms);
    }
    if (ops_per_s) *ops_per_s = fp32_probe_ops(which, blocks, iters) / (best_ms * 1e-3);
    if (ms_out) *ms_out = best_ms;
  });
}

int tsdd_cuda_nn_profile(tsdd_cuda_ctx* ctx, float* nn_sq_host) {
  if (!ctx) return TSDD_ERR_PARAMETER;
  return guarded(ctx, [&] {
    if (!nn_sq_host) fail(TSDD_ERR_PARAMETER, "nn_sq_host must not be null");
    uint64_t pos = 0;
    double dist = 0.0;
    search(ctx, 1, TSDD_SEARCH_DISABLE_PRUNING, &pos, &dist);
    std::vector<uint64_t> keys(ctx->rows);
    CUDA_OK(cudaMemcpy(keys.data(), ctx->nn.ptr, keys.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < keys.size(); ++i) nn_sq_host[i] = float_from_bits(key_bits(keys[i]));
  });
}

}  // extern "C"
