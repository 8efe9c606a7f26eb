// TEST INFRASTRUCTURE — a minimal front end over the PATCHED reference library
// (tools/patch_reference.py applied to a copy of /root/reference/proj):
// it calls the reference's own tsdd::parse_engine and tsdd::run_discovery, so that
// `--engine cuda` goes through the reference's entry point into libtsdd_cuda.so and
// `--engine phidd|hotsax|brute` runs the reference's CPU engines from the same binary.
// (The reference's own tool needs CLI11 / nlohmann headers that are not shipped.)
//
//   tsdd_patched SERIES.f64le ENGINE N WORD_LEN ALPHABET [THREADS]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "tsdd/errors.hpp"
#include "tsdd/pipeline.hpp"

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: tsdd_patched SERIES.f64le ENGINE N WORD_LEN ALPHABET [THREADS]\n");
    return 2;
  }
  try {
    std::ifstream in(argv[1], std::ios::binary | std::ios::ate);
    if (!in) throw tsdd::ValidationError(std::string("cannot open '") + argv[1] + "' for reading");
    const std::streamoff bytes = in.tellg();
    in.seekg(0);
    tsdd::TimeSeries series;
    series.values.resize(static_cast<std::size_t>(bytes) / sizeof(double));
    in.read(reinterpret_cast<char*>(series.values.data()), bytes);
    tsdd::DiscoveryConfig config;
    config.engine = tsdd::parse_engine(argv[2]);
    config.n = std::strtoull(argv[3], nullptr, 10);
    config.word_len = std::strtoull(argv[4], nullptr, 10);
    config.alphabet = std::strtoull(argv[5], nullptr, 10);
    config.threads = argc > 6 ? std::atoi(argv[6]) : 1;
    const tsdd::RunOutcome outcome = tsdd::run_discovery(series, config);
    std::printf("{\"engine\": \"%s\", \"m\": %zu, \"pos\": %zu, \"dist\": %.17g, \"calls\": %llu, "
                "\"prep_time_s\": %.9f, \"search_time_s\": %.9f}\n",
                std::string(tsdd::engine_name(outcome.result.engine)).c_str(), outcome.m, outcome.result.position,
                outcome.result.distance, static_cast<unsigned long long>(outcome.result.calls), outcome.prep_time_s,
                outcome.search_time_s);
    return 0;
  } catch (const tsdd::ParameterError& e) {  // tools/tsdd.cpp:212-223
    std::fprintf(stderr, "parameter error: %s\n", e.what());
    return 2;
  } catch (const tsdd::ValidationError& e) {
    std::fprintf(stderr, "input error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
