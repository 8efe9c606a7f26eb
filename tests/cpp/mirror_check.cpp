// Test program for the reference-shaped C++ entry points of include/tsdd/cuda_engine.hpp:
// SubsequenceMatrix::build -> DiscordIndexes::build -> phidd_discord, the way
// /root/reference/proj/src/pipeline.cpp:60-87 chains the reference's own.  Prints everything
// the mirrors expose as JSON; tests/test_gpu_parity.py compares it with the CPU oracle.
//
//   mirror_check SERIES.f64le N WORD_LEN ALPHABET [K] [rows: i,j,...]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "tsdd/cuda_engine.hpp"

namespace {

template <typename T>
void print_list(const char* name, const T* values, std::size_t count, const char* fmt, bool last = false) {
  std::printf("  \"%s\": [", name);
  for (std::size_t i = 0; i < count; ++i) {
    if (i) std::printf(", ");
    std::printf(fmt, values[i]);
  }
  std::printf("]%s\n", last ? "" : ",");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: mirror_check SERIES.f64le N WORD_LEN ALPHABET [K] [ROWS]\n");
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
    const std::size_t n = std::strtoull(argv[2], nullptr, 10), word_len = std::strtoull(argv[3], nullptr, 10),
                      alphabet = std::strtoull(argv[4], nullptr, 10);
    const int k = argc > 5 ? std::atoi(argv[5]) : 1;
    std::vector<std::size_t> want_rows;
    if (argc > 6) {
      std::stringstream ss(argv[6]);
      std::string item;
      while (std::getline(ss, item, ',')) want_rows.push_back(std::strtoull(item.c_str(), nullptr, 10));
    }

    // the reference's preparation stage, step by step (pipeline.cpp:60-67)
    const tsdd::cuda::SubsequenceMatrix matrix = tsdd::cuda::SubsequenceMatrix::build(series, n);
    const tsdd::cuda::DiscordIndexes indexes = tsdd::cuda::DiscordIndexes::build(matrix, word_len, alphabet);
    // ... and its search stage (pipeline.cpp:85-87)
    tsdd::DiscoveryOptions options;
    options.threads = 3;  // validated, otherwise without meaning on the device
    options.chunk = 2;
    std::vector<tsdd::DiscordResult> all;
    const tsdd::DiscordResult result = tsdd::cuda::phidd_discord(matrix, indexes, options, k, &all);

    std::printf("{\n  \"rows\": %zu, \"n\": %zu, \"stride\": %zu, \"pad\": %zu, \"vec_width\": %zu,\n", matrix.rows(),
                matrix.subsequence_length(), matrix.stride(), matrix.pad(), matrix.vec_width());
    std::printf("  \"pos\": %zu, \"dist\": %.17g, \"calls\": %llu, \"abandoned\": %llu,\n", result.position,
                result.distance, static_cast<unsigned long long>(result.calls),
                static_cast<unsigned long long>(result.abandoned));
    std::vector<std::size_t> positions;
    std::vector<double> distances;
    for (const tsdd::DiscordResult& d : all) positions.push_back(d.position), distances.push_back(d.distance);
    print_list("positions", positions.data(), positions.size(), "%zu");
    print_list("distances", distances.data(), distances.size(), "%.17g");
    print_list("hashes", indexes.hashes.data(), indexes.hashes.size(), "%llu");
    print_list("freq", indexes.freq.freq.data(), indexes.freq.freq.size(), "%u");
    print_list("candidates", indexes.candidates.positions.data(), indexes.candidates.positions.size(), "%zu");
    std::printf("  \"bucket_count\": %llu, \"total_positions\": %zu,\n",
                static_cast<unsigned long long>(indexes.words.bucket_count()), indexes.words.total_positions());
    // every bucket of the dictionary when it is small, else the occupied ones via the hashes
    std::printf("  \"buckets\": {");
    bool first = true;
    const std::uint64_t dict = indexes.words.bucket_count();
    for (std::uint64_t h = 1; h <= dict && dict <= 4096; ++h) {
      const tsdd::cuda::WordIndex::Bucket b = indexes.words.bucket(h);
      if (b.empty()) continue;
      std::printf("%s\"%llu\": [", first ? "" : ", ", static_cast<unsigned long long>(h));
      for (std::size_t q = 0; q < b.size(); ++q) std::printf("%s%zu", q ? ", " : "", b[q]);
      std::printf("]");
      first = false;
    }
    std::printf("},\n  \"row_values\": {");
    for (std::size_t r = 0; r < want_rows.size(); ++r) {
      const std::vector<float> row = matrix.row(want_rows[r]);
      std::printf("%s\"%zu\": [", r ? ", " : "", want_rows[r]);
      for (std::size_t c = 0; c < row.size(); ++c) std::printf("%s%.9g", c ? ", " : "", static_cast<double>(row[c]));
      std::printf("]");
    }
    std::printf("}\n}\n");
    return 0;
  } catch (const tsdd::InfeasibleInputError& e) {
    std::fprintf(stderr, "infeasible: %s\n", e.what());
    return 4;
  } catch (const tsdd::ParameterError& e) {
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
