// tsdd/cuda_engine.hpp — C++ host side of the B200 discord-search engine.
//
// Header-only binding of the C ABI (tsdd_cuda.h) to the reference's own
// interface for this path: the same type names, fields, 1-based positions and
// exception contract as /root/reference/proj/include/tsdd/
//     pipeline.hpp:15-37   DiscoveryConfig, RunOutcome, run_discovery
//     discovery.hpp:16-32  Engine, DiscordResult, DiscoveryOptions
//     discovery.hpp:86-88  phidd_discord(matrix, indexes, options)
//     series.hpp:38-66     SubsequenceMatrix          (device-backed mirror: tsdd::cuda::SubsequenceMatrix)
//     index.hpp:14-64      FrequencyIndex, CandidateIndex, WordIndex, DiscordIndexes (tsdd::cuda::DiscordIndexes)
//     series.hpp:14-19     TimeSeries
//     errors.hpp:10-25     ParameterError, ValidationError, InfeasibleInputError
//
// Two ways to use it:
//   * inside the reference tree: define TSDD_CUDA_WITH_REFERENCE_HEADERS, the
//     reference's headers supply the types and tsdd::cuda::run_discovery is the
//     body of one more case of the engine switch (pipeline.cpp:78-88); see
//     INTEGRATION.md;
//   * standalone (default): the small mirror types below are defined here.
//
// No exception crosses the C ABI: return codes are turned back into the
// reference's exception types here.
#ifndef TSDD_CUDA_ENGINE_HPP
#define TSDD_CUDA_ENGINE_HPP

#include <cstddef>
#include <memory>
#include <utility>
#include <cstdint>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

#include "tsdd_cuda.h"

#ifdef TSDD_CUDA_WITH_REFERENCE_HEADERS
#include "tsdd/errors.hpp"
#include "tsdd/pipeline.hpp"
#else
namespace tsdd {

struct ParameterError : std::invalid_argument {  // CLI exit code 2
  using std::invalid_argument::invalid_argument;
};
struct ValidationError : std::runtime_error {  // CLI exit code 3
  using std::runtime_error::runtime_error;
};
struct InfeasibleInputError : ParameterError {  // no non-self match at this n
  using ParameterError::ParameterError;
};

struct TimeSeries {
  std::vector<double> values;
  std::size_t length() const { return values.size(); }
};

enum class Engine { brute, hotsax, phidd, cuda };

struct DiscordResult {
  std::size_t position = 0;     // 1-based start of the discord
  double distance = 0.0;        // Euclidean, square root taken once
  std::uint64_t calls = 0;      // distance evaluations started
  std::uint64_t abandoned = 0;  // of which cut short
  Engine engine = Engine::cuda;
};

struct DiscoveryOptions {  // discovery.hpp:28-32
  int threads = 1;
  int chunk = 1;
  bool disable_pruning = false;
};

struct FrequencyIndex {  // index.hpp:14-16: freq[i] = rows whose SAX word equals row i's
  std::vector<std::uint32_t> freq;
};

struct CandidateIndex {  // index.hpp:20-22: 1-based positions of minimal word frequency, ascending
  std::vector<std::size_t> positions;
};

struct DiscoveryConfig {
  std::size_t n = 0;
  std::size_t word_len = 4;
  std::size_t alphabet = 4;
  std::size_t vec_width = 8;  // validated (>= 1); the device row stride is fixed at 32 floats
  Engine engine = Engine::cuda;
  int threads = 1;  // validated (>= 1); no meaning on the device
  int chunk = 1;    // validated (>= 1); no meaning on the device
  bool disable_pruning = false;
};

struct RunOutcome {
  DiscordResult result;
  std::size_t m = 0;
  double prep_time_s = 0.0;
  double search_time_s = 0.0;
};

}  // namespace tsdd
#endif  // TSDD_CUDA_WITH_REFERENCE_HEADERS

namespace tsdd::cuda {

// Thrown for TSDD_ERR_RUNTIME: CUDA / NCCL failure or no usable device.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void raise_for(int code, const std::string& message) {
  switch (code) {
    case TSDD_OK: return;
    case TSDD_ERR_PARAMETER: throw ParameterError(message);
    case TSDD_ERR_VALIDATION: throw ValidationError(message);
    case TSDD_ERR_INFEASIBLE: throw InfeasibleInputError(message);
    default: throw DeviceError(message);
  }
}

// One engine instance on one GPU.  Externally synchronised, like every
// instance in the reference.
class Session {
 public:
  explicit Session(int device = 0) {
    const int rc = tsdd_cuda_create(&ctx_, device);
    if (rc != TSDD_OK) raise_for(rc, tsdd_cuda_last_error(nullptr));
  }
  ~Session() { tsdd_cuda_destroy(ctx_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  tsdd_cuda_ctx* handle() const { return ctx_; }

  void set_option(const char* name, double value) { check(tsdd_cuda_set_option(ctx_, name, value)); }

  // Preparation stage (pipeline.cpp:60-69) on the device.
  void prepare(const TimeSeries& series, std::size_t n, std::size_t word_len, std::size_t alphabet) {
    check(tsdd_cuda_prepare_f64(ctx_, series.values.data(), series.values.size(), n, word_len, alphabet));
  }
  void prepare(const std::vector<float>& series, std::size_t n, std::size_t word_len, std::size_t alphabet) {
    check(tsdd_cuda_prepare_f32(ctx_, series.data(), series.size(), n, word_len, alphabet));
  }

  // Search stage (phidd_discord, discovery.cpp:360-373); k > 1 adds the
  // exclusion-zone top-k of tsdd_cuda.h.
  std::vector<DiscordResult> search(int k = 1, bool disable_pruning = false) {
    std::vector<std::uint64_t> pos(static_cast<std::size_t>(k > 0 ? k : 1));
    std::vector<double> dist(pos.size());
    check(tsdd_cuda_search(ctx_, k, disable_pruning ? TSDD_SEARCH_DISABLE_PRUNING : 0u, pos.data(), dist.data()));
    const tsdd_cuda_stats st = stats();
    std::vector<DiscordResult> out(pos.size());
    for (std::size_t r = 0; r < out.size(); ++r) {
      out[r].position = static_cast<std::size_t>(pos[r]);
      out[r].distance = dist[r];
      out[r].calls = st.calls;
      out[r].abandoned = st.abandoned;
      out[r].engine = Engine::cuda;
    }
    return out;
  }

  tsdd_cuda_stats stats() const {
    tsdd_cuda_stats st{};
    tsdd_cuda_get_stats(ctx_, &st);
    return st;
  }

 private:
  void check(int rc) const {
    if (rc != TSDD_OK) raise_for(rc, tsdd_cuda_last_error(ctx_));
  }
  tsdd_cuda_ctx* ctx_ = nullptr;
};

// ---- the reference's two-step preparation and its search entry point ---------
//
//   reference (pipeline.cpp:60-87)                       this header
//   SubsequenceMatrix::build(series, n, vec_width)   ->  cuda::SubsequenceMatrix::build(series, n[, vec_width, device])
//   paa -> sax -> DiscordIndexes::build(sax, alpha)  ->  cuda::DiscordIndexes::build(matrix, word_len, alphabet)
//   phidd_discord(matrix, indexes, options)          ->  cuda::phidd_discord(matrix, indexes, options)
//
// The reference's SubsequenceMatrix has a private constructor (series.hpp:59) and its WordIndex
// private storage with one friend (index.hpp:36-40), so device-built data cannot be poured into
// them; these are mirrors with the same accessors.  The matrix lives in device memory (float32,
// row stride a multiple of 64); the index arrays are public host vectors, as in the reference.

// series.hpp:38-66.  Immutable after construction; copies share one device-resident matrix.
class SubsequenceMatrix {
 public:
  // Requires 1 <= n <= series length and vec_width >= 1 (ParameterError otherwise,
  // series.cpp:48-56); rejects empty / non-finite series (ValidationError).
  static SubsequenceMatrix build(const TimeSeries& series, std::size_t n, std::size_t vec_width = 8,
                                 int device = 0) {
    // the reference's order (series.cpp:46-56): series, then n, then vec_width
    const std::size_t m = series.values.size();
    char message[256];
    const int rc = tsdd_cuda_check_config_f64(series.values.data(), m, 1, 1, 2, message, sizeof(message));
    if (rc == TSDD_ERR_VALIDATION) raise_for(rc, message);
    if (n < 1 || n > m)
      throw ParameterError("subsequence length n=" + std::to_string(n) + " must satisfy 1 <= n <= m=" +
                           std::to_string(m));
    if (vec_width < 1) throw ParameterError("vec_width must be >= 1");
    SubsequenceMatrix matrix;
    matrix.rows_ = m - n + 1;
    matrix.n_ = n;
    matrix.vec_width_ = vec_width;
    matrix.session_ = std::make_shared<Session>(device);
    // N <= n: no row has a non-self match.  The reference still builds such a matrix and only
    // its engines refuse it (discovery.cpp:114-121); the device has nothing to prepare for.
    matrix.infeasible_ = matrix.rows_ < n + 1;
    if (!matrix.infeasible_) {
      // The C ABI prepares matrix and index in one call: the index is built here for the smallest
      // legal SAX shape and rebuilt by DiscordIndexes::build (tsdd_cuda_reindex keeps the matrix).
      matrix.session_->prepare(series, n, 1, 2);
      matrix.stride_ = tsdd_cuda_row_stride(matrix.session_->handle());
    } else {
      matrix.stride_ = (n + 63) / 64 * 64;
    }
    return matrix;
  }

  std::size_t rows() const { return rows_; }  // N = m - n + 1
  std::size_t subsequence_length() const { return n_; }
  std::size_t stride() const { return stride_; }  // floats per device row: n rounded up to a multiple of 64
  std::size_t pad() const { return stride_ - n_; }
  std::size_t vec_width() const { return vec_width_; }  // (validated; the device stride does not depend on it)

  // Full padded row i (0-based), copied from the device: `stride()` float32 values, padding 0.
  std::vector<float> row(std::size_t i) const {
    require_device();
    std::vector<float> out(stride_);
    const int rc = tsdd_cuda_fetch_rows(session_->handle(), i, 1, out.data());
    if (rc != TSDD_OK) raise_for(rc, tsdd_cuda_last_error(session_->handle()));
    return out;
  }

  Session& session() const { return *session_; }
  bool infeasible() const { return infeasible_; }  // N <= n: the engines must refuse (discovery.cpp:114-121)

 private:
  SubsequenceMatrix() = default;
  void require_device() const {
    if (infeasible_) throw InfeasibleInputError("the matrix of an infeasible input is not kept on the device");
  }
  friend struct DiscordIndexes;

  std::shared_ptr<Session> session_;
  bool infeasible_ = false;
  std::size_t rows_ = 0, n_ = 0, stride_ = 0, vec_width_ = 1;
};

// index.hpp:27-41: bucket(h) lists, ascending, the 1-based positions whose SAX word hashes to h.
// Sort-based instead of an |A|^w + 1 offset table (4^16 words do not fit one): the distinct
// hashes present, ascending, with one offset each.
class WordIndex {
 public:
  struct Bucket {  // (std::span in the reference; this header stays C++17)
    const std::size_t* first = nullptr;
    std::size_t count = 0;
    const std::size_t* begin() const { return first; }
    const std::size_t* end() const { return first + count; }
    std::size_t size() const { return count; }
    bool empty() const { return count == 0; }
    std::size_t operator[](std::size_t k) const { return first[k]; }
  };
  Bucket bucket(std::uint64_t hash) const {
    const auto it = std::lower_bound(hashes_.begin(), hashes_.end(), hash);
    if (it == hashes_.end() || *it != hash) return {};
    const std::size_t b = static_cast<std::size_t>(it - hashes_.begin());
    return {positions_.data() + offsets_[b], offsets_[b + 1] - offsets_[b]};
  }
  std::uint64_t bucket_count() const { return dict_size_; }  // |A|^w, as in the reference
  std::uint64_t occupied_buckets() const { return hashes_.size(); }
  std::size_t total_positions() const { return positions_.size(); }

 private:
  friend struct DiscordIndexes;
  std::vector<std::uint64_t> hashes_;   // distinct 1-based hashes present, ascending
  std::vector<std::size_t> offsets_;    // hashes_.size() + 1
  std::vector<std::size_t> positions_;  // N entries, bucket after bucket
  std::uint64_t dict_size_ = 0;
};

// index.hpp:57-64: the three indexes plus the per-position hashes — public fields, like the
// reference's.  Built on the device (radix sort + run-length histogram) and mirrored on the host.
struct DiscordIndexes {
  FrequencyIndex freq;
  CandidateIndex candidates;
  WordIndex words;
  std::vector<std::uint64_t> hashes;

  // The reference's DiscordIndexes::build(sax(paa(matrix, word_len), alphabet), alphabet)
  // (pipeline.cpp:64-67) in one step: PAA, SAX and hashing happen on the device.
  static DiscordIndexes build(const SubsequenceMatrix& matrix, std::size_t word_len, std::size_t alphabet) {
    DiscordIndexes out;
    out.session_ = matrix.session_;
    out.word_len_ = word_len;
    out.alphabet_ = alphabet;
    if (matrix.infeasible_) {  // parameters are still validated; nothing to index on the device
      if (word_len < 1 || word_len > matrix.n_)
        throw ParameterError("word_len=" + std::to_string(word_len) + " must satisfy 1 <= word_len <= n=" +
                             std::to_string(matrix.n_));
      if (alphabet < 2 || alphabet > 10)
        throw ParameterError("alphabet cardinality " + std::to_string(alphabet) + " is outside the built-in range 2..10");
      return out;
    }
    tsdd_cuda_ctx* ctx = matrix.session_->handle();
    auto check = [&](int rc) {
      if (rc != TSDD_OK) raise_for(rc, tsdd_cuda_last_error(ctx));
    };
    check(tsdd_cuda_reindex(ctx, word_len, alphabet));
    const std::size_t rows = matrix.rows_;
    out.hashes.resize(rows);
    check(tsdd_cuda_fetch(ctx, TSDD_FETCH_HASH, out.hashes.data(), rows * sizeof(std::uint64_t)));
    out.freq.freq.resize(rows);
    check(tsdd_cuda_fetch(ctx, TSDD_FETCH_FREQ, out.freq.freq.data(), rows * sizeof(std::uint32_t)));
    const tsdd_cuda_stats st = matrix.session_->stats();
    std::vector<std::uint64_t> wide(static_cast<std::size_t>(st.min_freq_candidates));
    check(tsdd_cuda_fetch(ctx, TSDD_FETCH_CANDIDATES, wide.data(), wide.size() * sizeof(std::uint64_t)));
    out.candidates.positions.assign(wide.begin(), wide.end());
    wide.resize(rows);
    check(tsdd_cuda_fetch(ctx, TSDD_FETCH_BUCKETS, wide.data(), rows * sizeof(std::uint64_t)));
    out.words.positions_.assign(wide.begin(), wide.end());
    for (std::size_t p = 0; p < rows; ++p) {  // runs of equal hashes in bucket order
      const std::uint64_t h = out.hashes[out.words.positions_[p] - 1];
      if (out.words.hashes_.empty() || out.words.hashes_.back() != h) {
        out.words.hashes_.push_back(h);
        out.words.offsets_.push_back(p);
      }
    }
    out.words.offsets_.push_back(rows);
    out.words.dict_size_ = 1;
    for (std::size_t j = 0; j < word_len; ++j) out.words.dict_size_ *= alphabet;
    return out;
  }

  bool built_from(const SubsequenceMatrix& matrix) const { return session_ == matrix.session_; }
  std::size_t word_len() const { return word_len_; }
  std::size_t alphabet() const { return alphabet_; }

 private:
  std::shared_ptr<Session> session_;
  std::size_t word_len_ = 0, alphabet_ = 0;
};

// discovery.hpp:86-88, for the CUDA engine: feasibility (discovery.cpp:114-121) and options
// (discovery.cpp:22-29) checked first, then both PhiDD stages on the device.  `indexes` must
// have been built from `matrix` (they share one device context).  `all`, when given, receives
// the k discords.
inline DiscordResult phidd_discord(const SubsequenceMatrix& matrix, const DiscordIndexes& indexes,
                                   const DiscoveryOptions& options = {}, int k = 1,
                                   std::vector<DiscordResult>* all = nullptr) {
  if (options.threads < 1) throw ParameterError("threads must be >= 1, got " + std::to_string(options.threads));
  if (options.chunk < 1) throw ParameterError("chunk must be >= 1, got " + std::to_string(options.chunk));
  if (matrix.infeasible())  // require_feasible, discovery.cpp:114-121 (after check_options, as there)
    throw InfeasibleInputError("no subsequence has a non-self match: N=" + std::to_string(matrix.rows()) + " <= n=" +
                               std::to_string(matrix.subsequence_length()) + " (need series length m >= 2n)");
  if (k < 1) throw ParameterError("k must be >= 1, got " + std::to_string(k));
  if (!indexes.built_from(matrix))
    throw ParameterError("the indexes were not built from this matrix (they must share one device context)");
  std::vector<DiscordResult> found = matrix.session().search(k, options.disable_pruning);
  DiscordResult first = found.front();
  if (all) *all = std::move(found);
  return first;
}

// The host-only part of check_config that the C ABI does not see
// (pipeline.cpp:33-41), placed where the reference places it: after the
// series / n / word_len checks and before alphabet, dictionary, feasibility.
inline void check_host_fields(const TimeSeries& series, const DiscoveryConfig& config) {
  char message[512];
  const int rc = tsdd_cuda_check_config_f64(series.values.data(), series.values.size(), config.n,
                                            config.word_len, config.alphabet, message, sizeof(message));
  const std::string text = message;
  const bool early = rc == TSDD_ERR_VALIDATION ||
                     (rc == TSDD_ERR_PARAMETER && (text.rfind("n=", 0) == 0 || text.rfind("word_len=", 0) == 0));
  if (early) raise_for(rc, text);
  if (config.vec_width < 1) throw ParameterError("vec_width must be >= 1");
  if (config.threads < 1) throw ParameterError("threads must be >= 1, got " + std::to_string(config.threads));
  if (config.chunk < 1) throw ParameterError("chunk must be >= 1, got " + std::to_string(config.chunk));
  raise_for(rc, text);
}

// tsdd::run_discovery for Engine::cuda: validate everything, then the two
// timed stages.  `all`, when given, receives the k discords (best first).
// Counters and device timings of the last run_discovery on this thread, one entry per rank
// (tsdd_cuda_stats: terms, tile-kernel time, ... — what the bench harness reports beside the
// reference's columns).
inline std::vector<tsdd_cuda_stats>& last_run_stats() {
  thread_local std::vector<tsdd_cuda_stats> stats;
  return stats;
}

inline RunOutcome run_discovery(const TimeSeries& series, const DiscoveryConfig& config, int k = 1,
                                std::vector<DiscordResult>* all = nullptr, int device = 0) {
  check_host_fields(series, config);
  if (k < 1) throw ParameterError("k must be >= 1, got " + std::to_string(k));
  Session session(device);
  session.prepare(series, config.n, config.word_len, config.alphabet);
  std::vector<DiscordResult> found = session.search(k, config.disable_pruning);
  const tsdd_cuda_stats st = session.stats();
  last_run_stats().assign(1, st);
  RunOutcome outcome;
  outcome.result = found.front();
  outcome.m = series.length();
  outcome.prep_time_s = (st.prep_ms + st.h2d_ms) * 1e-3;
  outcome.search_time_s = st.search_ms * 1e-3;
  if (all) *all = std::move(found);
  return outcome;
}

// ---- several GPUs from one process ------------------------------------------
// One host thread and one Session per device, linked into a group of ranks
// (tsdd_cuda_group_create): the rarity-ordered candidates are dealt round-robin, the ranks
// meet in a host barrier after every batch and exchange ON THE DEVICES — each rank
// min-reduces its peers' nn bounds straight from their memory (NVLink P2P) and the window
// statistics are computed in per-rank slices and gathered.  The kernels of different devices
// never wait on one another — only the host threads meet.  (One process per GPU with NCCL is
// the other way: tsdd_cuda_comm_init.)  The same device may be listed twice, which is how
// the tests exercise the path on a single GPU.
inline RunOutcome run_discovery(const TimeSeries& series, const DiscoveryConfig& config, int k,
                                std::vector<DiscordResult>* all, const std::vector<int>& devices) {
  if (devices.size() <= 1) return run_discovery(series, config, k, all, devices.empty() ? 0 : devices[0]);
  check_host_fields(series, config);
  if (k < 1) throw ParameterError("k must be >= 1, got " + std::to_string(k));
  const int world = static_cast<int>(devices.size());
  std::vector<std::unique_ptr<Session>> sessions;
  std::vector<tsdd_cuda_ctx*> handles;
  for (const int device : devices) {
    sessions.push_back(std::make_unique<Session>(device));
    handles.push_back(sessions.back()->handle());
  }
  const int rc = tsdd_cuda_group_create(handles.data(), world);
  if (rc != TSDD_OK) raise_for(rc, tsdd_cuda_last_error(handles[0]));
  std::vector<std::vector<DiscordResult>> found(devices.size());
  std::vector<tsdd_cuda_stats> stats(devices.size());
  std::vector<std::exception_ptr> errors(devices.size());
  std::vector<std::thread> workers;
  for (int rank = 0; rank < world; ++rank) {
    workers.emplace_back([&, rank] {
      const std::size_t r = static_cast<std::size_t>(rank);
      try {  // (a failure inside the library releases the other ranks from the group's barrier)
        sessions[r]->prepare(series, config.n, config.word_len, config.alphabet);
        found[r] = sessions[r]->search(k, config.disable_pruning);
        stats[r] = sessions[r]->stats();
      } catch (...) {
        errors[r] = std::current_exception();
      }
    });
  }
  for (std::thread& t : workers) t.join();
  // the rank that failed first carries the cause; the others only report that a peer failed
  for (const std::exception_ptr& e : errors) {
    if (!e) continue;
    try {
      std::rethrow_exception(e);
    } catch (const DeviceError& d) {
      if (std::string(d.what()).find("another rank of the group failed") == std::string::npos) throw;
    }
  }
  for (const std::exception_ptr& e : errors)
    if (e) std::rethrow_exception(e);
  last_run_stats() = stats;
  RunOutcome outcome;
  outcome.result = found[0].front();
  outcome.m = series.length();
  std::uint64_t calls = 0, abandoned = 0;
  for (const tsdd_cuda_stats& st : stats) {
    calls += st.calls;
    abandoned += st.abandoned;
    outcome.prep_time_s = std::max(outcome.prep_time_s, (st.prep_ms + st.h2d_ms) * 1e-3);
    outcome.search_time_s = std::max(outcome.search_time_s, st.search_ms * 1e-3);
  }
  for (DiscordResult& d : found[0]) {
    d.calls = calls;
    d.abandoned = abandoned;
  }
  outcome.result = found[0].front();
  if (all) *all = std::move(found[0]);
  return outcome;
}

}  // namespace tsdd::cuda

#endif  // TSDD_CUDA_ENGINE_HPP
