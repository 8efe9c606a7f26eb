// Seeded synthetic series for the five BASELINE.json workloads.
//
// These ARE the benchmark inputs: BASELINE.json describes five synthetic
// series (no public dataset is involved; the paper's SCD-1M/10M sets are
// proprietary).  BASELINE.json leaves the RNG family and the "seed-chosen"
// anomaly offsets open; this file fixes them once (SURVEY.md gap G6):
//   * bits        : std::mt19937_64(seed)           (portable by the C++ standard)
//   * uniform     : (bits >> 11) * 2^-53  in [0,1)
//   * normal      : Box-Muller on two uniforms (cos branch only, no caching)
//   * offsets     : drawn FIRST from the stream, rejection-sampled so that
//                   every anomaly lies >= 2*len from both ends and the
//                   anomalies are >= 4*len apart (so top-k discords are distinct)
// Values are generated in double and rounded once to float32 at the end; the
// oracle receives the same float32 values widened losslessly to double.
//
// Host-only code (no CUDA): used by tests/, bench.py and the host tools.
// The reference's own generator family (proj/src/generate.cpp:19-59: uniform-step walk
// with an optional spike or shape anomaly) is restated at the end of this file
// (tsdd_generate_series) for the CLI's `generate --m ...` form.

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

namespace {

struct Stream {
  std::mt19937_64 bits;
  explicit Stream(std::uint64_t seed) : bits(seed) {}
  double uniform() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }
  double normal() {
    double u1 = uniform();
    const double u2 = uniform();
    if (u1 < 0x1.0p-53) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925 * u2);
  }
  std::uint64_t below(std::uint64_t bound) { return bits() % bound; }
};

// `count` window starts, each `len` long, >= 2*len from the ends and
// >= 4*len apart from one another; returned in draw order.
std::vector<std::size_t> draw_offsets(Stream& rng, std::size_t m, std::size_t len,
                                      int count, std::size_t align = 1) {
  std::vector<std::size_t> out;
  const std::size_t lo = 2 * len;
  const std::size_t hi = m - 3 * len;  // exclusive upper bound for a start
  while (static_cast<int>(out.size()) < count) {
    std::size_t s = lo + rng.below(hi - lo);
    s -= s % align;
    bool ok = s >= lo;
    for (const std::size_t t : out) {
      const std::size_t gap = s > t ? s - t : t - s;
      if (gap < 4 * len) ok = false;
    }
    if (ok) out.push_back(s);
  }
  return out;
}

void window_mean_std(const std::vector<double>& x, std::size_t s, std::size_t len,
                     double* mean, double* sd) {
  double sum = 0, sq = 0;
  for (std::size_t t = 0; t < len; ++t) sum += x[s + t];
  const double mu = sum / static_cast<double>(len);
  for (std::size_t t = 0; t < len; ++t) sq += (x[s + t] - mu) * (x[s + t] - mu);
  *mean = mu;
  *sd = std::sqrt(sq / static_cast<double>(len));
}

struct Workload {
  std::size_t m, n, word_len, alphabet;
  int k;
  std::uint64_t seed;
  int anomalies;
  std::size_t anomaly_len;
};

// BASELINE.json configs[0..4]
constexpr Workload kWorkloads[5] = {
    {65536, 128, 4, 4, 1, 0, 1, 128},
    {262144, 256, 8, 4, 4, 1, 4, 256},
    {1000000, 512, 8, 6, 3, 2, 3, 250},
    {4000000, 1024, 16, 4, 5, 3, 5, 1024},
    {1000000, 256, 8, 4, 1, 4, 0, 0},
};

// cfg 1 and 2: Gaussian random walk, t0 = 0.
void random_walk(Stream& rng, std::vector<double>& x) {
  double level = 0.0;
  x[0] = 0.0;
  for (std::size_t i = 1; i < x.size(); ++i) {
    level += rng.normal();
    x[i] = level;
  }
}

void make_cfg1(const Workload& w, std::vector<double>& x, std::vector<std::size_t>& at) {
  Stream rng(w.seed);
  at = draw_offsets(rng, w.m, w.anomaly_len, w.anomalies);
  random_walk(rng, x);
  for (const std::size_t s : at) {
    double mu, sd;
    window_mean_std(x, s, w.anomaly_len, &mu, &sd);
    for (std::size_t t = 0; t < w.anomaly_len; ++t) {
      x[s + t] = mu + 3.0 * sd * std::sin(6.283185307179586476925 * static_cast<double>(t) / 32.0);
    }
  }
}

void make_cfg2(const Workload& w, std::vector<double>& x, std::vector<std::size_t>& at) {
  Stream rng(w.seed);
  at = draw_offsets(rng, w.m, w.anomaly_len, w.anomalies);
  random_walk(rng, x);
  for (const std::size_t s : at) {
    // local step std over the window's own increments
    double sum = 0, sq = 0;
    for (std::size_t t = 0; t < w.anomaly_len; ++t) {
      const double d = x[s + t] - x[s + t - 1];
      sum += d;
      sq += d * d;
    }
    const double L = static_cast<double>(w.anomaly_len);
    const double var = sq / L - (sum / L) * (sum / L);
    const double step_sd = var > 0 ? std::sqrt(var) : 1.0;
    double mu, sd;
    window_mean_std(x, s, w.anomaly_len, &mu, &sd);
    for (std::size_t t = 0; t < w.anomaly_len; ++t) x[s + t] = mu + 4.0 * step_sd * rng.normal();
  }
}

void make_cfg3(const Workload& w, std::vector<double>& x, std::vector<std::size_t>& at) {
  Stream rng(w.seed);
  const std::size_t beat = 250;
  // altered beats: starts aligned to the beat grid
  at = draw_offsets(rng, w.m, 2 * beat, w.anomalies, beat);
  const double centre[3] = {60, 100, 140};
  const double width[3] = {5, 3, 8};
  const double amp[3] = {0.2, 1.0, 0.3};
  for (std::size_t i = 0; i < w.m; ++i) {
    const std::size_t b0 = i - i % beat;
    double gain = 1.0, widen = 1.0;
    if (b0 == at[0]) gain = 0.0;        // omitted beat
    else if (b0 == at[1]) widen = 2.0;  // pulses twice as wide
    else if (b0 == at[2]) gain = 0.5;   // half amplitude
    const double t = static_cast<double>(i % beat);
    double v = 0.0;
    for (int p = 0; p < 3; ++p) {
      const double z = (t - centre[p]) / (width[p] * widen);
      v += amp[p] * std::exp(-0.5 * z * z);
    }
    x[i] = gain * v + 0.05 * rng.normal();
  }
}

void make_cfg4(const Workload& w, std::vector<double>& x, std::vector<std::size_t>& at) {
  Stream rng(w.seed);
  at = draw_offsets(rng, w.m, w.anomaly_len, w.anomalies);
  const double period[3] = {1000, 3700, 11000};
  const double amp[3] = {1.0, 0.5, 0.25};
  double ar = 0.0;
  double sum = 0, sq = 0;
  for (std::size_t i = 0; i < w.m; ++i) {
    ar = 0.9 * ar + 0.1 * rng.normal();
    double v = ar;
    for (int p = 0; p < 3; ++p) {
      v += amp[p] * std::sin(6.283185307179586476925 * static_cast<double>(i) / period[p]);
    }
    x[i] = v;
    sum += v;
    sq += v * v;
  }
  const double M = static_cast<double>(w.m);
  const double var = sq / M - (sum / M) * (sum / M);
  const double sd = var > 0 ? std::sqrt(var) : 1.0;
  for (const std::size_t s : at) {
    for (std::size_t t = 0; t < w.anomaly_len; ++t) x[s + t] += 2.0 * sd;
  }
}

void make_cfg5(const Workload& w, std::vector<double>& x, std::vector<std::size_t>& at) {
  Stream rng(w.seed);
  at.clear();
  for (std::size_t i = 0; i < w.m; ++i) x[i] = rng.uniform();
}

}  // namespace

extern "C" {

// cfg is 1..5 (BASELINE.json configs[cfg-1]).  Any out pointer may be null.
int tsdd_workload_info(int cfg, std::uint64_t* m, std::uint64_t* n, std::uint64_t* word_len,
                       std::uint64_t* alphabet, int* k, std::uint64_t* seed, int* anomalies,
                       std::uint64_t* anomaly_len) {
  if (cfg < 1 || cfg > 5) return 2;
  const Workload& w = kWorkloads[cfg - 1];
  if (m) *m = w.m;
  if (n) *n = w.n;
  if (word_len) *word_len = w.word_len;
  if (alphabet) *alphabet = w.alphabet;
  if (k) *k = w.k;
  if (seed) *seed = w.seed;
  if (anomalies) *anomalies = w.anomalies;
  if (anomaly_len) *anomaly_len = w.anomaly_len;
  return 0;
}

// Fills out[0..m) with the float32 series of workload cfg and anomaly_at
// (capacity >= 8, may be null) with the 0-based starts of the planted windows.
int tsdd_workload_series(int cfg, float* out, std::uint64_t capacity, std::uint64_t* anomaly_at) {
  if (cfg < 1 || cfg > 5 || !out) return 2;
  const Workload& w = kWorkloads[cfg - 1];
  if (capacity < w.m) return 2;
  std::vector<double> x(w.m);
  std::vector<std::size_t> at;
  switch (cfg) {
    case 1: make_cfg1(w, x, at); break;
    case 2: make_cfg2(w, x, at); break;
    case 3: make_cfg3(w, x, at); break;
    case 4: make_cfg4(w, x, at); break;
    default: make_cfg5(w, x, at); break;
  }
  for (std::size_t i = 0; i < w.m; ++i) out[i] = static_cast<float>(x[i]);
  if (anomaly_at) {
    for (std::size_t i = 0; i < at.size(); ++i) anomaly_at[i] = at[i];
  }
  return 0;
}

// Generic seeded Gaussian random walk (float32), for the SPEC-style
// acceptance sweeps (many small random walks).
int tsdd_random_walk(std::uint64_t seed, float* out, std::uint64_t m) {
  if (!out || m == 0) return 2;
  Stream rng(seed);
  double level = 0.0;
  out[0] = 0.0f;
  for (std::uint64_t i = 1; i < m; ++i) {
    level += rng.normal();
    out[i] = static_cast<float>(level);
  }
  return 0;
}

// The reference's generator (generate.cpp:19-59, generate.hpp:16-28), restated: a walk of
// m uniform[-1, 1) steps from std::mt19937_64(seed) through std::uniform_real_distribution
// (the same library calls, so the same values); anomaly 0 none, 1 spike (+100 at one sample),
// 2 shape (anomaly_len samples from anomaly_pos on replaced by base + 12 sin(6 pi t / (len-1))).
// anomaly_pos is 1-based.  Returns 0, or 2 with the reference's ParameterError text in `message`.
int tsdd_generate_series(std::uint64_t m, int anomaly, std::uint64_t anomaly_pos, std::uint64_t anomaly_len,
                         std::uint64_t seed, double* out, char* message, std::uint64_t message_bytes) {
  auto reject = [&](const std::string& text) {
    if (message && message_bytes) std::snprintf(message, message_bytes, "%s", text.c_str());
    return 2;
  };
  if (m < 1) return reject("generator length must be >= 1");
  if (anomaly < 0 || anomaly > 2) return reject("unknown anomaly kind (expected none, spike or shape)");
  const std::uint64_t extent = anomaly == 2 ? anomaly_len : 1;
  if (anomaly != 0) {
    if (anomaly_pos < 1 || anomaly_pos - 1 + extent > m)
      return reject("anomaly at position " + std::to_string(anomaly_pos) + " with extent " + std::to_string(extent) +
                    " does not fit in series of length " + std::to_string(m));
    if (anomaly == 2 && anomaly_len < 2) return reject("shape anomaly length must be >= 2");
  }
  if (!out) return reject("output buffer is null");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> step(-1.0, 1.0);
  double level = 0.0;
  for (std::uint64_t i = 0; i < m; ++i) {
    level += step(rng);
    out[i] = level;
  }
  if (anomaly == 1) {
    out[anomaly_pos - 1] += 100.0;
  } else if (anomaly == 2) {
    const std::uint64_t start = anomaly_pos - 1;
    const double base = out[start];
    for (std::uint64_t t = 0; t < anomaly_len; ++t) {
      const double phase = 6.0 * M_PI * static_cast<double>(t) / static_cast<double>(anomaly_len - 1);
      // (one rounding: the reference's build, -O3 -march=native, contracts this into an fma)
      out[start + t] = std::fma(12.0, std::sin(phase), base);
    }
  }
  return 0;
}

}  // extern "C"
