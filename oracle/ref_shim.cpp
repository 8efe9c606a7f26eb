// TEST INFRASTRUCTURE — C shim over the UNMODIFIED reference library.
//
// This file contains no algorithm of its own: it only calls the public API
// declared in /root/reference/proj/include/tsdd/*.hpp and copies the results
// out through a C ABI so that tests (ctypes) and bench.py's reference arm
// can drive the real reference.  It is compiled together with the reference
// sources where they lie (see oracle/Makefile); outputs go to oracle/_ref/.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  The product never does.
//
// Error mapping mirrors tools/tsdd.cpp:212-223 (2 parameter, 3 validation),
// with InfeasibleInputError split out as 4.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "tsdd/discovery.hpp"
#include "tsdd/errors.hpp"
#include "tsdd/generate.hpp"
#include "tsdd/index.hpp"
#include "tsdd/pipeline.hpp"
#include "tsdd/sax.hpp"
#include "tsdd/series.hpp"

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const tsdd::InfeasibleInputError& e) {
    g_error = e.what();
    return 4;
  } catch (const tsdd::ParameterError& e) {
    g_error = e.what();
    return 2;
  } catch (const tsdd::ValidationError& e) {
    g_error = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

tsdd::TimeSeries as_series(const double* v, std::uint64_t m) {
  tsdd::TimeSeries s;
  s.values.assign(v, v + m);
  return s;
}

tsdd::Engine engine_from(int e) {
  return e == 0 ? tsdd::Engine::brute : e == 1 ? tsdd::Engine::hotsax : tsdd::Engine::phidd;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// tsdd::run_discovery (pipeline.hpp:37).  engine: 0 brute, 1 hotsax, 2 phidd.
int ref_run_discovery(const double* series, std::uint64_t m, std::uint64_t n,
                      std::uint64_t word_len, std::uint64_t alphabet, int engine, int threads,
                      int chunk, int disable_pruning, std::uint64_t* position, double* distance,
                      std::uint64_t* calls, std::uint64_t* abandoned, double* prep_s,
                      double* search_s) {
  return guarded([&] {
    tsdd::DiscoveryConfig cfg;
    cfg.n = n;
    cfg.word_len = word_len;
    cfg.alphabet = alphabet;
    cfg.engine = engine_from(engine);
    cfg.threads = threads;
    cfg.chunk = chunk;
    cfg.disable_pruning = disable_pruning != 0;
    const tsdd::RunOutcome out = tsdd::run_discovery(as_series(series, m), cfg);
    if (position) *position = out.result.position;
    if (distance) *distance = out.result.distance;
    if (calls) *calls = out.result.calls;
    if (abandoned) *abandoned = out.result.abandoned;
    if (prep_s) *prep_s = out.prep_time_s;
    if (search_s) *search_s = out.search_time_s;
  });
}

// Every preparation-stage array through the reference's public accessors
// (series.hpp:53, sax.hpp:37,47, index.hpp:29,57-61).  Any out pointer may be
// null.  rows: N*n (padding dropped), paa: N*w, sax: N*w, hashes/freq: N,
// candidates: up to N (count in *n_candidates), bucket_positions: the N
// 1-based positions listed bucket after bucket in ascending hash order,
// bucket_sizes_by_row: size of row i's own bucket.
int ref_prepare(const double* series, std::uint64_t m, std::uint64_t n, std::uint64_t word_len,
                std::uint64_t alphabet, double* rows, double* paa, std::uint32_t* sax,
                std::uint64_t* hashes, std::uint32_t* freq, std::uint64_t* candidates,
                std::uint64_t* n_candidates, std::uint64_t* bucket_positions) {
  return guarded([&] {
    const tsdd::TimeSeries ts = as_series(series, m);
    const tsdd::Alphabet alpha(alphabet);
    const tsdd::SubsequenceMatrix mat = tsdd::SubsequenceMatrix::build(ts, n);
    const std::size_t N = mat.rows();
    if (rows) {
      for (std::size_t i = 0; i < N; ++i) std::memcpy(rows + i * n, mat.row_ptr(i), n * sizeof(double));
    }
    const tsdd::PaaMatrix P = tsdd::paa(mat, word_len);
    if (paa) std::memcpy(paa, P.data.data(), P.data.size() * sizeof(double));
    const tsdd::SaxMatrix S = tsdd::sax(P, alpha);
    if (sax) std::memcpy(sax, S.data.data(), S.data.size() * sizeof(std::uint32_t));
    const tsdd::DiscordIndexes idx = tsdd::DiscordIndexes::build(S, alpha);
    if (hashes) std::memcpy(hashes, idx.hashes.data(), N * sizeof(std::uint64_t));
    if (freq) std::memcpy(freq, idx.freq.freq.data(), N * sizeof(std::uint32_t));
    if (n_candidates) *n_candidates = idx.candidates.positions.size();
    if (candidates) {
      for (std::size_t c = 0; c < idx.candidates.positions.size(); ++c) candidates[c] = idx.candidates.positions[c];
    }
    if (bucket_positions) {
      std::size_t at = 0;
      for (std::uint64_t h = 1; h <= idx.words.bucket_count(); ++h) {
        for (const std::size_t p : idx.words.bucket(h)) bucket_positions[at++] = p;
      }
    }
  });
}

// squared_distance_early_abandon (series.hpp:117-146).  Returns 0 and sets
// *abandoned_flag; *value is only meaningful when not abandoned.
int ref_distance(const double* a, const double* b, std::uint64_t len, double threshold,
                 std::uint64_t block, double* value, int* abandoned_flag) {
  return guarded([&] {
    tsdd::DistanceBudget budget;
    budget.best_so_far_sq = threshold;
    const auto d = tsdd::squared_distance_early_abandon({a, len}, {b, len}, budget, block);
    *abandoned_flag = d ? 0 : 1;
    *value = d ? *d : 0.0;
  });
}

int ref_paa_row(const double* values, std::uint64_t n, double* out, std::uint64_t w) {
  return guarded([&] { tsdd::paa_row({values, n}, {out, w}); });
}

int ref_symbol_for(std::uint64_t alphabet, double value, std::uint32_t* symbol) {
  return guarded([&] { *symbol = tsdd::Alphabet(alphabet).symbol_for(value); });
}

int ref_word_hash(const std::uint32_t* word, std::uint64_t w, std::uint64_t alphabet,
                  std::uint64_t* hash) {
  return guarded([&] { *hash = tsdd::word_hash({word, w}, tsdd::Alphabet(alphabet)); });
}

int ref_z_normalize(double* data, std::uint64_t n) {
  return guarded([&] { tsdd::z_normalize_range(data, n); });
}

// Top-k discords with the exclusion-zone definition of SURVEY.md §8(c)
// (discord r = arg-max nn distance over positions at least n away from every
// earlier discord; neighbour sets unrestricted), computed with the reference's
// unmodified public stages:
//   stage 1 = potential_discord_stage over the min-frequency candidates that
//             are still allowed (discovery.cpp:209-287);
//   stage 2 = refine_discord_stage over every other allowed position
//             (discovery.cpp:289-358) — excluded rows are hidden from it by
//             listing them in the public candidates.positions field
//             (index.hpp:20-22,58), which is exactly the mask it skips.
// For k = 1 this is phidd_discord (discovery.cpp:360-373) verbatim.
int ref_topk(const double* series, std::uint64_t m, std::uint64_t n, std::uint64_t word_len,
             std::uint64_t alphabet, int k, int threads, int chunk, std::uint64_t* positions,
             double* distances, std::uint64_t* calls, std::uint64_t* abandoned, double* prep_s,
             double* search_s) {
  return guarded([&] {
    const tsdd::TimeSeries ts = as_series(series, m);
    // same validation the pipeline performs (pipeline.cpp:21-49)
    tsdd::validate_series(ts);
    if (k < 1) throw tsdd::ParameterError("k must be >= 1");
    const auto t_prep = std::chrono::steady_clock::now();
    const tsdd::Alphabet alpha(alphabet);
    tsdd::dict_size(alpha, word_len);
    const tsdd::SubsequenceMatrix mat = tsdd::SubsequenceMatrix::build(ts, n);
    tsdd::require_feasible(mat);
    const tsdd::PaaMatrix P = tsdd::paa(mat, word_len);
    const tsdd::SaxMatrix S = tsdd::sax(P, alpha);
    const tsdd::DiscordIndexes base = tsdd::DiscordIndexes::build(S, alpha);
    if (prep_s) *prep_s = seconds_since(t_prep);

    tsdd::DiscoveryOptions opt;
    opt.threads = threads;
    opt.chunk = chunk;
    const std::size_t N = mat.rows();
    std::vector<char> excluded(N, 0);
    std::uint64_t total_calls = 0, total_abandoned = 0;
    const auto t_search = std::chrono::steady_clock::now();
    for (int r = 0; r < k; ++r) {
      tsdd::DiscordIndexes stage1 = base;
      stage1.candidates.positions.clear();
      for (const std::size_t p : base.candidates.positions) {
        if (!excluded[p - 1]) stage1.candidates.positions.push_back(p);
      }
      tsdd::SharedBest shared;
      const tsdd::StageCounters c1 = tsdd::potential_discord_stage(mat, stage1, shared, opt);

      tsdd::DiscordIndexes stage2 = base;
      std::vector<char> hidden = excluded;
      for (const std::size_t p : stage1.candidates.positions) hidden[p - 1] = 1;
      stage2.candidates.positions.clear();
      for (std::size_t i = 0; i < N; ++i) {
        if (hidden[i]) stage2.candidates.positions.push_back(i + 1);
      }
      const tsdd::DiscordResult res = tsdd::refine_discord_stage(mat, stage2, shared, opt);
      total_calls += c1.calls + res.calls;
      total_abandoned += c1.abandoned + res.abandoned;
      positions[r] = res.position;
      distances[r] = res.distance;
      // exclusion zone: every start within n of the discord just found
      const std::size_t p0 = res.position - 1;
      const std::size_t lo = p0 >= n - 1 ? p0 - (n - 1) : 0;
      const std::size_t hi = std::min<std::size_t>(N - 1, p0 + (n - 1));
      for (std::size_t i = lo; i <= hi; ++i) excluded[i] = 1;
    }
    if (search_s) *search_s = seconds_since(t_search);
    if (calls) *calls = total_calls;
    if (abandoned) *abandoned = total_abandoned;
  });
}

// Full nearest-neighbour profile by exhaustive search, using the reference's
// squared_distance (series.hpp:150-164) over the reference's matrix — the
// body of brute_force_discord (discovery.cpp:123-173) with the profile kept.
// nn_sq[i] = +inf where row i has no non-self match.
int ref_nn_profile(const double* series, std::uint64_t m, std::uint64_t n, int threads,
                   double* nn_sq) {
  return guarded([&] {
    const tsdd::TimeSeries ts = as_series(series, m);
    const tsdd::SubsequenceMatrix mat = tsdd::SubsequenceMatrix::build(ts, n);
    const std::ptrdiff_t N = static_cast<std::ptrdiff_t>(mat.rows());
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
    for (std::ptrdiff_t i = 0; i < N; ++i) {
      tsdd::DistanceBudget budget;
      double best = std::numeric_limits<double>::infinity();
      for (std::ptrdiff_t j = 0; j < N; ++j) {
        const std::ptrdiff_t gap = i > j ? i - j : j - i;
        if (gap < static_cast<std::ptrdiff_t>(n)) continue;
        const double d = tsdd::squared_distance(mat.row(i), mat.row(j), budget);
        if (d < best) best = d;
      }
      nn_sq[i] = best;
    }
  });
}

// generate_series (generate.cpp:19-59); anomaly by name as on the reference's command line
int ref_generate_series(std::uint64_t m, const char* anomaly, std::uint64_t anomaly_pos, std::uint64_t anomaly_len,
                        std::uint64_t seed, double* out) {
  return guarded([&] {
    tsdd::GeneratorSpec spec;
    spec.length = m;
    spec.anomaly = tsdd::parse_anomaly_kind(anomaly);
    spec.anomaly_pos = anomaly_pos;
    spec.anomaly_len = anomaly_len;
    spec.seed = seed;
    const tsdd::TimeSeries series = tsdd::generate_series(spec);
    std::copy(series.values.begin(), series.values.end(), out);
  });
}

}  // extern "C"
