// tsdd_cuda — command-line front end of the CUDA discord-search engine.
//
// The analogue of the reference's `tsdd` tool (tools/tsdd.cpp:116-223) for Engine::cuda,
// written against include/tsdd/cuda_engine.hpp: the same sub-commands and flag names
// where they apply, the same JSON / CSV result fields (tools/tsdd.cpp:84-110), the same
// bench CSV header plus GPU columns (src/bench.cpp:76-87), and the same exit codes
// (tools/tsdd.cpp:212-223: 2 parameter error, 3 input error, 1 anything else).  The flag
// parser and the series readers are this repo's own (the reference's CLI11 / nlohmann
// headers are not shipped); the readers keep the reference's formats and the wording of
// its input errors (src/io.cpp:23-91) and add `f32le`, the workloads' native precision.
//
//   tsdd_cuda find     --input FILE [--format csv|f64le|f32le] --n N [--word-len W] [--alphabet A]
//                      [--k K] [--gpus 0,1,...] [--disable-pruning] [--output json|csv]
//   tsdd_cuda bench    --input FILE [--format ...] --n N1,N2,... [--gpus 1,2,4,8] [--repeats R]
//                      [--word-len W] [--alphabet A] [--k K] [--output FILE]
//   tsdd_cuda generate --m M [--anomaly none|spike|shape] [--anomaly-pos P] [--anomaly-len L] [--seed S]
//                      --output FILE [--format csv|f64le|f32le]        the reference's generator (tools/tsdd.cpp:140-153)
//   tsdd_cuda generate --workload 1..5 --output FILE [--format f32le|f64le|csv]     the BASELINE.json workloads
//                                                                       (both need libtsdd_gen.so beside the tool)
//
// `--threads`, `--chunk`, `--vec-width` are accepted and validated like the reference's and
// have no effect on the device.  `--gpus` lists CUDA devices (find) or device COUNTS to sweep
// (bench; devices 0..c-1, one host thread each).  TSDD_CUDA_SAME_DEVICE=1 maps every rank to
// device 0 (how the tests exercise several ranks on a single GPU).
#include <dlfcn.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "tsdd/cuda_engine.hpp"

namespace {

using tsdd::ParameterError;
using tsdd::ValidationError;

// ------------------------------------------------------------------ flags
struct Flags {
  std::string command;
  std::map<std::string, std::string> values;
  bool has(const std::string& name) const { return values.count(name) != 0; }
  std::string get(const std::string& name, const std::string& fallback = "") const {
    const auto it = values.find(name);
    return it == values.end() ? fallback : it->second;
  }
};

Flags parse_flags(int argc, char** argv, const std::vector<std::string>& known, const std::vector<std::string>& switches) {
  Flags flags;
  if (argc < 2) throw ParameterError("a sub-command is required: find, bench or generate");
  flags.command = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string arg = argv[i];
    if (arg.rfind("--", 0) != 0) throw ParameterError("unexpected argument '" + arg + "'");
    std::string name = arg.substr(2), value;
    const std::size_t eq = name.find('=');
    const bool inline_value = eq != std::string::npos;
    if (inline_value) {
      value = name.substr(eq + 1);
      name = name.substr(0, eq);
    }
    if (std::find(switches.begin(), switches.end(), name) != switches.end()) {
      flags.values[name] = "1";
      continue;
    }
    if (std::find(known.begin(), known.end(), name) == known.end())
      throw ParameterError("unknown option '--" + name + "'");
    if (!inline_value) {
      if (i + 1 >= argc) throw ParameterError("option '--" + name + "' needs a value");
      value = argv[++i];
    }
    flags.values[name] = value;
  }
  return flags;
}

std::size_t to_size(const std::string& text, const std::string& what) {
  errno = 0;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(text.c_str(), &end, 10);
  if (text.empty() || *end != '\0' || errno == ERANGE || text[0] == '-')
    throw ParameterError("'" + text + "' is not a valid value for --" + what);
  return static_cast<std::size_t>(v);
}

std::vector<std::size_t> to_size_list(const std::string& text, const std::string& what) {
  std::vector<std::size_t> out;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) out.push_back(to_size(item, what));
  if (out.empty()) throw ParameterError("--" + what + " needs at least one value");
  return out;
}

// ------------------------------------------------------------------ series files
enum class Format { csv, f64le, f32le };

Format parse_format(const std::string& name) {
  if (name == "csv") return Format::csv;
  if (name == "f64le") return Format::f64le;
  if (name == "f32le") return Format::f32le;
  throw ParameterError("unknown series format '" + name + "' (expected csv, f64le or f32le)");
}

std::string trimmed(const std::string& line) {
  std::size_t a = 0, b = line.size();
  while (b > a && (line[b - 1] == '\r' || line[b - 1] == ' ' || line[b - 1] == '\t')) --b;
  while (a < b && (line[a] == ' ' || line[a] == '\t')) ++a;
  return line.substr(a, b - a);
}

tsdd::TimeSeries read_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open '" + path + "' for reading");
  tsdd::TimeSeries series;
  std::string raw;
  for (std::size_t line_no = 1; std::getline(in, raw); ++line_no) {
    const std::string line = trimmed(raw);
    if (line.empty()) continue;
    errno = 0;
    char* end = nullptr;
    const double value = std::strtod(line.c_str(), &end);
    const bool parsed = end != line.c_str() && *end == '\0' && errno != ERANGE;
    if (!parsed) {
      if (line_no == 1 && series.values.empty()) continue;  // one non-numeric header line is allowed
      throw ValidationError("cannot parse '" + line + "' at " + path + ":" + std::to_string(line_no));
    }
    if (!std::isfinite(value)) throw ValidationError("non-finite value at " + path + ":" + std::to_string(line_no));
    series.values.push_back(value);
  }
  if (series.values.empty()) throw ValidationError("no values found in '" + path + "'");
  return series;
}

template <typename T>
tsdd::TimeSeries read_raw(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw ValidationError("cannot open '" + path + "' for reading");
  const std::streamoff size = in.tellg();
  in.seekg(0);
  if (size <= 0) throw ValidationError("no values found in '" + path + "'");
  const std::streamoff width = static_cast<std::streamoff>(sizeof(T));
  if (size % width != 0)
    throw ValidationError("file size " + std::to_string(size) + " of '" + path + "' is not a multiple of " +
                          std::to_string(width) + " (truncated at byte offset " +
                          std::to_string((size / width) * width) + ")");
  std::vector<T> raw(static_cast<std::size_t>(size / width));
  in.read(reinterpret_cast<char*>(raw.data()), size);
  if (!in) throw ValidationError("short read from '" + path + "'");
  tsdd::TimeSeries series;
  series.values.assign(raw.begin(), raw.end());
  for (std::size_t i = 0; i < series.values.size(); ++i)
    if (!std::isfinite(series.values[i]))
      throw ValidationError("non-finite value at index " + std::to_string(i + 1) + " of '" + path + "'");
  return series;
}

tsdd::TimeSeries read_series(const std::string& path, Format format) {
  switch (format) {
    case Format::csv: return read_csv(path);
    case Format::f64le: return read_raw<double>(path);
    default: return read_raw<float>(path);
  }
}

void write_series(const std::vector<float>& values, const std::string& path, Format format) {
  std::ofstream out(path, format == Format::csv ? std::ios::out : std::ios::binary);
  if (!out) throw ValidationError("cannot open '" + path + "' for writing");
  if (format == Format::csv) {
    char buf[64];
    for (const float v : values) {
      std::snprintf(buf, sizeof(buf), "%.9g\n", static_cast<double>(v));  // 9 digits round-trip a float
      out << buf;
    }
  } else if (format == Format::f32le) {
    out.write(reinterpret_cast<const char*>(values.data()), static_cast<std::streamsize>(values.size() * sizeof(float)));
  } else {
    const std::vector<double> wide(values.begin(), values.end());
    out.write(reinterpret_cast<const char*>(wide.data()), static_cast<std::streamsize>(wide.size() * sizeof(double)));
  }
  if (!out) throw ValidationError("write to '" + path + "' failed");
}

tsdd::TimeSeries acquire_series(const Flags& flags) {
  if (!flags.has("input")) throw ParameterError("--input is required");
  return read_series(flags.get("input"), parse_format(flags.get("format", "csv")));
}

void print_series_summary(const tsdd::TimeSeries& series) {
  const auto [lo, hi] = std::minmax_element(series.values.begin(), series.values.end());
  std::cerr << "series: " << series.length() << " values, min " << *lo << ", max " << *hi << "\n";
}

tsdd::DiscoveryConfig config_from(const Flags& flags) {
  tsdd::DiscoveryConfig config;
  config.engine = tsdd::Engine::cuda;
  if (flags.has("word-len")) config.word_len = to_size(flags.get("word-len"), "word-len");
  if (flags.has("alphabet")) config.alphabet = to_size(flags.get("alphabet"), "alphabet");
  if (flags.has("vec-width")) config.vec_width = to_size(flags.get("vec-width"), "vec-width");
  if (flags.has("threads")) config.threads = std::atoi(flags.get("threads").c_str());
  if (flags.has("chunk")) config.chunk = std::atoi(flags.get("chunk").c_str());
  config.disable_pruning = flags.has("disable-pruning");
  const std::string engine = flags.get("engine", "cuda");
  if (engine != "cuda") throw ParameterError("unknown engine '" + engine + "' (this tool runs 'cuda')");
  return config;
}

std::vector<int> devices_for(std::size_t count) {
  const char* same = std::getenv("TSDD_CUDA_SAME_DEVICE");
  std::vector<int> devices(count);
  for (std::size_t r = 0; r < count; ++r) devices[r] = (same && same[0] == '1') ? 0 : static_cast<int>(r);
  return devices;
}

// ------------------------------------------------------------------ find
int run_find(const Flags& flags) {
  if (!flags.has("n")) throw ParameterError("--n is required");
  tsdd::DiscoveryConfig config = config_from(flags);
  config.n = to_size(flags.get("n"), "n");
  const int k = flags.has("k") ? static_cast<int>(to_size(flags.get("k"), "k")) : 1;
  std::vector<int> devices{0};
  if (flags.has("gpus")) {
    devices.clear();
    for (const std::size_t d : to_size_list(flags.get("gpus"), "gpus")) devices.push_back(static_cast<int>(d));
  }
  const std::string output = flags.get("output", "json");
  if (output != "json" && output != "csv") throw ParameterError("unknown output format '" + output + "' (expected json or csv)");

  const tsdd::TimeSeries series = acquire_series(flags);
  print_series_summary(series);
  std::vector<tsdd::DiscordResult> all;
  const tsdd::RunOutcome outcome = tsdd::cuda::run_discovery(series, config, k, &all, devices);

  if (output == "json") {
    std::printf("{\n  \"engine\": \"cuda\",\n  \"m\": %zu,\n  \"n\": %zu,\n  \"word_len\": %zu,\n  \"alphabet\": %zu,\n"
                "  \"threads\": %d,\n  \"gpus\": %zu,\n  \"pos\": %zu,\n  \"dist\": %.17g,\n  \"calls\": %llu,\n"
                "  \"prep_time_s\": %.9f,\n  \"search_time_s\": %.9f,\n  \"discords\": [",
                outcome.m, config.n, config.word_len, config.alphabet, config.threads, devices.size(),
                outcome.result.position, outcome.result.distance,
                static_cast<unsigned long long>(outcome.result.calls), outcome.prep_time_s, outcome.search_time_s);
    for (std::size_t r = 0; r < all.size(); ++r)
      std::printf("%s{\"pos\": %zu, \"dist\": %.17g}", r ? ", " : "", all[r].position, all[r].distance);
    std::printf("]\n}\n");
  } else {
    std::printf("engine,m,n,word_len,alphabet,threads,pos,dist,calls,prep_time_s,search_time_s\n");
    for (const tsdd::DiscordResult& d : all)
      std::printf("cuda,%zu,%zu,%zu,%zu,%d,%zu,%.17g,%llu,%.9f,%.9f\n", outcome.m, config.n, config.word_len,
                  config.alphabet, config.threads, d.position, d.distance, static_cast<unsigned long long>(d.calls),
                  outcome.prep_time_s, outcome.search_time_s);
  }
  return 0;
}

// ------------------------------------------------------------------ bench (run_bench, src/bench.cpp:21-74)
double median_of(std::vector<double> values) {
  std::sort(values.begin(), values.end());
  const std::size_t c = values.size();
  return c % 2 ? values[c / 2] : 0.5 * (values[c / 2 - 1] + values[c / 2]);
}

int run_bench(const Flags& flags) {
  if (!flags.has("n")) throw ParameterError("--n is required");
  const std::vector<std::size_t> n_values = to_size_list(flags.get("n"), "n");
  const std::vector<std::size_t> gpu_counts = to_size_list(flags.get("gpus", "1"), "gpus");
  const int repeats = flags.has("repeats") ? static_cast<int>(to_size(flags.get("repeats"), "repeats")) : 3;
  const int k = flags.has("k") ? static_cast<int>(to_size(flags.get("k"), "k")) : 1;
  if (repeats < 1) throw ParameterError("repeats must be >= 1");
  if (std::find(gpu_counts.begin(), gpu_counts.end(), 1u) == gpu_counts.end())
    throw ParameterError("GPU sweep must include 1, the speedup baseline");
  for (const std::size_t c : gpu_counts)
    if (c < 1) throw ParameterError("GPU counts must be >= 1");
  tsdd::DiscoveryConfig config = config_from(flags);
  const tsdd::TimeSeries series = acquire_series(flags);

  std::ostringstream csv;
  // FP32 lane-operations per second of one device (FFMA-only probe): the denominator of fma_pipe_util
  double lane_ops_per_s = 0.0;
  {
    tsdd::cuda::Session probe(0);
    double ms = 0.0;
    if (tsdd_cuda_fp32_probe(probe.handle(), 0, &lane_ops_per_s, &ms) != TSDD_OK) lane_ops_per_s = 0.0;
  }
  csv << "engine,m,n,threads,wall_time_s,calls,pos,dist,speedup,efficiency,gpus,prep_time_s,search_time_s,terms,"
         "fma_pipe_util\n";
  for (const std::size_t n : n_values) {
    config.n = n;
    struct Row {
      std::size_t gpus;
      double wall, prep, search;
      tsdd::DiscordResult result;
      unsigned long long terms;  // distance terms accumulated by the tile kernels, all ranks
      double fma_pipe_util;      // their FP32-pipe lane operations / (tile-kernel time x measured lane rate), per GPU
    };
    std::vector<Row> rows;
    double t1 = 0.0;
    for (const std::size_t gpus : gpu_counts) {
      std::vector<double> times, preps, searches;
      tsdd::RunOutcome last;
      for (int r = 0; r < repeats; ++r) {
        last = tsdd::cuda::run_discovery(series, config, k, nullptr, devices_for(gpus));
        times.push_back(last.prep_time_s + last.search_time_s);
        preps.push_back(last.prep_time_s);
        searches.push_back(last.search_time_s);
      }
      unsigned long long terms = 0;
      double lane_ops = 0.0, kernel_s = 0.0;
      for (const tsdd_cuda_stats& st : tsdd::cuda::last_run_stats()) {
        terms += st.scan_kernel_terms;
        // a term is FADD + FFMA in the direct form, one FFMA in the dot-product form
        lane_ops += 2.0 * static_cast<double>(st.scan_kernel_terms - st.scan_kernel_dot_terms) +
                    static_cast<double>(st.scan_kernel_dot_terms);
        kernel_s += st.scan_kernel_ms * 1e-3;
      }
      const double util = (kernel_s > 0.0 && lane_ops_per_s > 0.0) ? lane_ops / (kernel_s * lane_ops_per_s) : 0.0;
      rows.push_back({gpus, median_of(times), median_of(preps), median_of(searches), last.result, terms, util});
      if (gpus == 1) t1 = rows.back().wall;
    }
    for (const Row& row : rows) {
      const double speedup = t1 / row.wall;
      char line[512];
      std::snprintf(line, sizeof(line), "cuda,%zu,%zu,%d,%.9f,%llu,%zu,%.17g,%.6f,%.6f,%zu,%.9f,%.9f,%llu,%.4f\n",
                    series.length(), n, config.threads, row.wall, static_cast<unsigned long long>(row.result.calls),
                    row.result.position, row.result.distance, speedup, speedup / static_cast<double>(row.gpus),
                    row.gpus, row.prep, row.search, row.terms, row.fma_pipe_util);
      csv << line;
    }
  }
  if (flags.has("output")) {
    std::ofstream out(flags.get("output"));
    if (!out) throw ValidationError("cannot open '" + flags.get("output") + "' for writing");
    out << csv.str();
  } else {
    std::cout << csv.str();
  }
  return 0;
}

// ------------------------------------------------------------------ generate
void write_series(const std::vector<double>& values, const std::string& path, Format format) {
  // (the reference's write_series, src/io.cpp:101-127: "%.17g" per line, or raw little-endian doubles)
  std::ofstream out(path, format == Format::csv ? std::ios::out : std::ios::binary);
  if (!out) throw ValidationError("cannot open '" + path + "' for writing");
  if (format == Format::csv) {
    char buf[64];
    for (const double v : values) {
      std::snprintf(buf, sizeof(buf), "%.17g\n", v);
      out << buf;
    }
  } else if (format == Format::f64le) {
    out.write(reinterpret_cast<const char*>(values.data()), static_cast<std::streamsize>(values.size() * sizeof(double)));
  } else {
    const std::vector<float> narrow(values.begin(), values.end());
    out.write(reinterpret_cast<const char*>(narrow.data()), static_cast<std::streamsize>(narrow.size() * sizeof(float)));
  }
  if (!out) throw ValidationError("write to '" + path + "' failed");
}

void* open_generators(const char* argv0) {
  std::string dir = argv0;
  dir = dir.find('/') == std::string::npos ? "." : dir.substr(0, dir.rfind('/'));
  const std::string lib = dir + "/libtsdd_gen.so";
  void* handle = dlopen(lib.c_str(), RTLD_NOW);
  if (!handle) throw ValidationError("cannot load " + lib + ": " + dlerror());
  return handle;
}

// `generate --m ...`: the reference's own generator family and flags (tools/tsdd.cpp:140-153,
// src/generate.cpp:19-59): uniform-step walk, optional spike / shape anomaly, default format csv.
int run_generate_walk(const Flags& flags, const char* argv0) {
  if (!flags.has("m") || !flags.has("output")) throw ParameterError("--m and --output are required");
  const std::string kind = flags.get("anomaly", "none");
  int anomaly = 0;
  if (kind == "none") anomaly = 0;
  else if (kind == "spike") anomaly = 1;
  else if (kind == "shape") anomaly = 2;
  else throw ParameterError("unknown anomaly kind '" + kind + "' (expected none, spike or shape)");
  const std::size_t m = to_size(flags.get("m"), "m");
  const std::size_t pos = flags.has("anomaly-pos") ? to_size(flags.get("anomaly-pos"), "anomaly-pos") : 0;
  const std::size_t len = flags.has("anomaly-len") ? to_size(flags.get("anomaly-len"), "anomaly-len") : 64;
  const std::size_t seed = flags.has("seed") ? to_size(flags.get("seed"), "seed") : 0;
  const Format format = parse_format(flags.get("format", "csv"));
  using GenFn = int (*)(std::uint64_t, int, std::uint64_t, std::uint64_t, std::uint64_t, double*, char*, std::uint64_t);
  auto generate = reinterpret_cast<GenFn>(dlsym(open_generators(argv0), "tsdd_generate_series"));
  if (!generate) throw ValidationError("libtsdd_gen.so lacks tsdd_generate_series");
  tsdd::TimeSeries series;
  series.values.resize(m);
  char message[256] = {0};
  if (generate(m, anomaly, pos, len, seed, series.values.data(), message, sizeof(message)) != 0)
    throw ParameterError(message);
  write_series(series.values, flags.get("output"), format);
  print_series_summary(series);
  return 0;
}

// `generate --workload c`: the five BASELINE.json workloads (float32; csrc/series_gen.cpp)
int run_generate(const Flags& flags, const char* argv0) {
  if (!flags.has("workload")) return run_generate_walk(flags, argv0);
  if (!flags.has("output")) throw ParameterError("--workload and --output are required");
  const int cfg = static_cast<int>(to_size(flags.get("workload"), "workload"));
  void* handle = open_generators(argv0);
  using InfoFn = int (*)(int, std::uint64_t*, std::uint64_t*, std::uint64_t*, std::uint64_t*, int*, std::uint64_t*,
                         int*, std::uint64_t*);
  using SeriesFn = int (*)(int, float*, std::uint64_t, std::uint64_t*);
  auto info = reinterpret_cast<InfoFn>(dlsym(handle, "tsdd_workload_info"));
  auto fill = reinterpret_cast<SeriesFn>(dlsym(handle, "tsdd_workload_series"));
  if (!info || !fill) throw ValidationError("libtsdd_gen.so lacks the workload generators");
  std::uint64_t m = 0, n = 0, w = 0, a = 0, seed = 0, alen = 0, at[8] = {0};
  int k = 0, anomalies = 0;
  if (info(cfg, &m, &n, &w, &a, &k, &seed, &anomalies, &alen) != 0)
    throw ParameterError("no such workload: " + std::to_string(cfg) + " (expected 1..5)");
  std::vector<float> values(m);
  if (fill(cfg, values.data(), m, at) != 0) throw ValidationError("the workload generator failed");
  write_series(values, flags.get("output"), parse_format(flags.get("format", "f32le")));
  std::cerr << "workload " << cfg << ": m=" << m << " n=" << n << " word_len=" << w << " alphabet=" << a << " k=" << k
            << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::vector<std::string> known = {"input", "format", "n", "word-len", "alphabet", "vec-width", "engine",
                                            "threads", "chunk", "output", "k", "gpus", "repeats", "workload", "m", "anomaly",
                                            "anomaly-pos", "anomaly-len", "seed"};
    const Flags flags = parse_flags(argc, argv, known, {"disable-pruning"});
    if (flags.command == "find") return run_find(flags);
    if (flags.command == "bench") return run_bench(flags);
    if (flags.command == "generate") return run_generate(flags, argv[0]);
    throw ParameterError("unknown sub-command '" + flags.command + "' (expected find, bench or generate)");
  } catch (const ParameterError& e) {
    std::cerr << "parameter error: " << e.what() << "\n";
    return 2;
  } catch (const ValidationError& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
