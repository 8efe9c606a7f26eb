// tsdd_cuda_find — minimal C++ caller of the CUDA engine through the reference-shaped
// interface (include/tsdd/cuda_engine.hpp).  It stands where `tsdd find` stands in the
// reference (tools/tsdd.cpp:78-110): read a series, run_discovery, print the result, map
// exceptions to the reference's exit codes (tools/tsdd.cpp:212-223: 2 parameter, 3 input,
// 1 anything else).  The reference's full CLI (CLI11 + nlohmann/json, not shipped) is out
// of scope; this tool exists so the C++ host layer is exercised end to end by the tests.
//
//   tsdd_cuda_find <series.f64le|series.f32le> <n> <word_len> <alphabet> [k] [--disable-pruning]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>

#include "tsdd/cuda_engine.hpp"

namespace {

tsdd::TimeSeries read_raw(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw tsdd::ValidationError("cannot open '" + path + "'");
  const std::streamsize bytes = in.tellg();
  in.seekg(0);
  tsdd::TimeSeries series;
  const bool f32 = path.size() > 6 && path.compare(path.size() - 6, 6, ".f32le") == 0;
  if (f32) {
    std::vector<float> raw(static_cast<std::size_t>(bytes) / sizeof(float));
    in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size() * sizeof(float)));
    series.values.assign(raw.begin(), raw.end());
  } else {
    series.values.resize(static_cast<std::size_t>(bytes) / sizeof(double));
    in.read(reinterpret_cast<char*>(series.values.data()),
            static_cast<std::streamsize>(series.values.size() * sizeof(double)));
  }
  return series;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 5) throw tsdd::ParameterError("usage: tsdd_cuda_find <series> <n> <word_len> <alphabet> [k] [--disable-pruning]");
    tsdd::DiscoveryConfig config;
    config.n = std::strtoull(argv[2], nullptr, 10);
    config.word_len = std::strtoull(argv[3], nullptr, 10);
    config.alphabet = std::strtoull(argv[4], nullptr, 10);
    config.engine = tsdd::Engine::cuda;
    int k = 1;
    for (int a = 5; a < argc; ++a) {
      if (std::strcmp(argv[a], "--disable-pruning") == 0) config.disable_pruning = true;
      else k = std::atoi(argv[a]);
    }
    const tsdd::TimeSeries series = read_raw(argv[1]);
    std::vector<tsdd::DiscordResult> all;
    const tsdd::RunOutcome outcome = tsdd::cuda::run_discovery(series, config, k, &all);
    std::printf("{\"engine\": \"cuda\", \"m\": %zu, \"n\": %zu, \"word_len\": %zu, \"alphabet\": %zu, \"pos\": %zu, "
                "\"dist\": %.17g, \"calls\": %llu, \"prep_time_s\": %.9f, \"search_time_s\": %.9f, \"discords\": [",
                outcome.m, config.n, config.word_len, config.alphabet, outcome.result.position,
                outcome.result.distance, static_cast<unsigned long long>(outcome.result.calls), outcome.prep_time_s,
                outcome.search_time_s);
    for (std::size_t r = 0; r < all.size(); ++r)
      std::printf("%s{\"pos\": %zu, \"dist\": %.17g}", r ? ", " : "", all[r].position, all[r].distance);
    std::printf("]}\n");
    return 0;
  } catch (const tsdd::ParameterError& e) {
    std::cerr << "parameter error: " << e.what() << "\n";
    return 2;
  } catch (const tsdd::ValidationError& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
