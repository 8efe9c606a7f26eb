// Preparation stage on the device (replaces src/pipeline.cpp:60-69 of the
// reference): per-window statistics and SAX encoding, the float32
// z-normalised subsequence matrix, and the SAX-word bucket / frequency /
// rarity index built with a radix sort and a run-length histogram.
//
// Everything here is HBM-bound integer / streaming work; kernels are laid
// out for coalesced 128-byte accesses and sized in whole waves of the SMs.

#include "kernels.hpp"

#include <cstdlib>

namespace tsdd_b200 {

namespace {

// Equiprobable N(0,1) breakpoints for |A| = 2..10, lower half mirrored onto
// the upper half; row a-2 holds the a-1 finite thresholds.  Regenerated with
// scipy norm.ppf (tools/gen_sax_breakpoints.py, checked by tests/test_host.py); same values as the
// reference's table (sax.cpp:14-46).
__constant__ double c_breaks[9][9] = {
    {0},
    {-0.43072729929545756, 0.43072729929545756},
    {-0.67448975019608171, 0, 0.67448975019608171},
    {-0.84162123357291418, -0.25334710313579972, 0.25334710313579972, 0.84162123357291418},
    {-0.96742156610170105, -0.43072729929545756, 0, 0.43072729929545756, 0.96742156610170105},
    {-1.0675705238781414, -0.56594882193286311, -0.1800123697927051, 0.1800123697927051,
     0.56594882193286311, 1.0675705238781414},
    {-1.1503493803760079, -0.67448975019608171, -0.31863936396437514, 0, 0.31863936396437514,
     0.67448975019608171, 1.1503493803760079},
    {-1.2206403488473501, -0.7647096737863871, -0.43072729929545756, -0.13971029888186212,
     0.13971029888186212, 0.43072729929545756, 0.7647096737863871, 1.2206403488473501},
    {-1.2815515655446004, -0.84162123357291418, -0.52440051270804089, -0.25334710313579972, 0,
     0.25334710313579972, 0.52440051270804089, 0.84162123357291418, 1.2815515655446004},
};

inline unsigned blocks_for(size_t items, unsigned per_block) {
  return static_cast<unsigned>((items + per_block - 1) / per_block);
}

// ------------------------------------------------------------------ series
// Also validate_series (series.cpp:10-19) for a series that never passed through the host:
// *first_bad receives the smallest index of a non-finite sample (preset to ~0 = none).
__global__ void k_widen_series(const float* __restrict__ in, double* __restrict__ out, size_t m,
                               uint32_t* __restrict__ first_bad) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const float v = in[i];
  out[i] = static_cast<double>(v);
  if (first_bad != nullptr && !isfinite(v)) atomicMin(first_bad, static_cast<uint32_t>(i));
}

// One thread per window.  Adjacent threads read adjacent samples, so every
// step of the loops below is one coalesced 256-byte request per warp, served
// from L1/L2 (the whole series is a few tens of MB).
//
//   mean, sigma : series.cpp:21-37 — sum and sum of squares in sequence order,
//                 population variance sum_sq/n - mu^2, sigma < 1e-12 -> flat
//   PAA         : sax.cpp:63-80   — n*w unit grid, weighted sum / n
//   symbol      : sax.cpp:53-57   — 1 + #{breakpoints <= value}
//   hash        : sax.cpp:121-132 — big-endian base |A|; stored 0-based so that
//                 4^16 words still fit 32 bits
__global__ void __launch_bounds__(256)
k_window_encode(const double* __restrict__ x, uint32_t rows, uint32_t n, uint32_t word_len,
                uint32_t alphabet, double* __restrict__ mean, double* __restrict__ inv_sigma,
                uint32_t* __restrict__ hash0, double* __restrict__ paa_out,
                uint32_t* __restrict__ sax_out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double* p = x + i;
  double sum = 0.0, sum_sq = 0.0;
  for (uint32_t t = 0; t < n; ++t) {
    const double v = p[t];
    sum += v;
    sum_sq += v * v;
  }
  const double dn = static_cast<double>(n);
  const double mu = sum / dn;
  const double var = sum_sq / dn - mu * mu;
  const double sigma = var > 0.0 ? sqrt(var) : 0.0;
  const bool flat = sigma < 1e-12;
  const double inv = flat ? 0.0 : 1.0 / sigma;
  mean[i] = mu;
  inv_sigma[i] = inv;

  const double* bp = c_breaks[alphabet - 2];
  uint64_t h = 0;
  for (uint32_t k = 0; k < word_len; ++k) {
    const uint64_t lo = static_cast<uint64_t>(k) * n;
    const uint64_t hi = lo + n;
    const uint32_t t_first = static_cast<uint32_t>(lo / word_len);
    const uint32_t t_last = static_cast<uint32_t>((hi - 1) / word_len);
    double acc = 0.0;
    for (uint32_t t = t_first; t <= t_last; ++t) {
      const uint64_t el = static_cast<uint64_t>(t) * word_len;
      const uint64_t eh = el + word_len;
      const uint64_t units = (eh < hi ? eh : hi) - (el > lo ? el : lo);
      const double v = flat ? 0.0 : (p[t] - mu) * inv;
      acc += static_cast<double>(units) * v;
    }
    const double seg = acc / dn;
    uint32_t sym = 1;
    for (uint32_t b = 0; b + 1 < alphabet; ++b) sym += (bp[b] <= seg) ? 1u : 0u;
    if (paa_out) paa_out[static_cast<size_t>(i) * word_len + k] = seg;
    if (sax_out) sax_out[static_cast<size_t>(i) * word_len + k] = sym;
    h = h * alphabet + (sym - 1);
  }
  hash0[i] = static_cast<uint32_t>(h);
}

// The same, four consecutive windows per thread.  k_window_encode is bound by the L1 data path
// (every window reads its n samples twice, 8 bytes each); here a block stages the samples of
// its 1,024 windows in shared memory once, interleaved by four (sample j at quarter j & 3,
// index j >> 2) so that the threads of a warp — whose windows start four samples apart — still
// read consecutive words, and a thread slides a four-sample register window along: one
// LDS.64 per step feeds four windows.  Every window's sums run in the same sequence order as
// before (bit-identical mean, sigma, PAA, symbols: the parity tests compare every array).
constexpr int kEncWindows = 4;
constexpr int kEncThreads = 256;
constexpr size_t encode4_smem_bytes(uint32_t n, bool with_prefix = false) {
  // samples (interleaved by four, with slack) + in the aligned form their prefix sums and the block-scan scratch
  const size_t samples = static_cast<size_t>(kEncThreads) * kEncWindows + n + 16;
  return (samples + (with_prefix ? samples + 2 * kEncThreads : 0)) * sizeof(double);
}

// kAligned (word_len divides n, and nobody asked for the PAA values): every sample lies wholly in one
// segment, so a segment's sum over the NORMALISED samples is ((P[end] - P[start]) - len * mu) / sigma with P the
// prefix sums of the block's staged samples — two loads a segment instead of four float64 operations a sample
// (60 % of the kernel's arithmetic; workload 4: 3.4 -> ... ms).  That value differs from the reference's
// sample-by-sample sum by rounding only, which can matter to a SYMBOL only within `tol` of a breakpoint (tol: a
// rigorous bound of both roundings from the block's sum of |x|); a window with a segment that close is encoded
// the reference's way.  Means, 1/sigma (their sums stay in sequence order), symbols and hashes remain
// bit-identical to the reference's.
template <bool kAligned>
__global__ void __launch_bounds__(kEncThreads)
k_window_encode4(const double* __restrict__ x, uint32_t rows, uint32_t n, uint32_t word_len,
                 uint32_t alphabet, double* __restrict__ mean, double* __restrict__ inv_sigma,
                 uint32_t* __restrict__ hash0, double* __restrict__ paa_out,
                 uint32_t* __restrict__ sax_out, double tol_scale) {
  extern __shared__ double s_x[];
  const uint32_t w0 = blockIdx.x * (kEncThreads * kEncWindows);  // first window of the block
  const uint32_t span = kEncThreads * kEncWindows + n + 4;       // samples any of its threads touches
  const uint32_t quarter = (span + 3) / 4 + 1;
  const size_t m = static_cast<size_t>(rows) + n - 1;
  for (uint32_t j = threadIdx.x; j < span; j += kEncThreads) {
    const size_t at = static_cast<size_t>(w0) + j;
    s_x[(j & 3u) * quarter + (j >> 2)] = at < m ? x[at] : 0.0;
  }
  __syncthreads();
  const uint32_t base = kEncWindows * threadIdx.x;  // this thread's first window, relative to w0
  auto sample = [&](uint32_t j) -> double { return s_x[(j & 3u) * quarter + (j >> 2)]; };
  double* s_p = s_x + 4 * quarter;          // kAligned: s_p[j] = sum of the staged samples before j
  double abs_total = 0.0;                   // ... and the sum of their magnitudes
  if constexpr (kAligned) {
    double* s_part = s_p + span + 1;        // block-scan scratch: kEncThreads sums, kEncThreads sums of magnitudes
    const uint32_t per = (span + kEncThreads - 1) / kEncThreads;
    const uint32_t j0 = min(threadIdx.x * per, span), j1 = min(j0 + per, span);
    double part = 0.0, part_abs = 0.0;
    for (uint32_t j = j0; j < j1; ++j) {
      const double v = sample(j);
      part += v;
      part_abs += fabs(v);
    }
    s_part[threadIdx.x] = part;
    s_part[kEncThreads + threadIdx.x] = part_abs;
    __syncthreads();
    double before = 0.0;
    for (uint32_t t = 0; t < kEncThreads; ++t) {  // (256 broadcast loads; the block's own arithmetic is 4 x n per thread)
      before += t < threadIdx.x ? s_part[t] : 0.0;
      abs_total += s_part[kEncThreads + t];
    }
    for (uint32_t j = j0; j < j1; ++j) {
      s_p[j] = before;
      before += sample(j);
    }
    if (j1 == span && j0 < span) s_p[span] = before;
    __syncthreads();
  }

  // ---- mean, sigma (series.cpp:21-37)
  double w[kEncWindows], sum[kEncWindows], sum_sq[kEncWindows];
#pragma unroll
  for (int r = 0; r < kEncWindows; ++r) w[r] = sample(base + r), sum[r] = 0.0, sum_sq[r] = 0.0;
  for (uint32_t t = 0; t < n; ++t) {
#pragma unroll
    for (int r = 0; r < kEncWindows; ++r) {
      const double v = w[r];
      sum[r] += v;
      sum_sq[r] += v * v;
    }
#pragma unroll
    for (int r = 0; r + 1 < kEncWindows; ++r) w[r] = w[r + 1];
    w[kEncWindows - 1] = sample(base + t + kEncWindows);
  }
  const double dn = static_cast<double>(n);
  double mu[kEncWindows], inv[kEncWindows];
  bool flat[kEncWindows];
#pragma unroll
  for (int r = 0; r < kEncWindows; ++r) {
    mu[r] = sum[r] / dn;
    const double var = sum_sq[r] / dn - mu[r] * mu[r];
    const double sigma = var > 0.0 ? sqrt(var) : 0.0;
    flat[r] = sigma < 1e-12;
    inv[r] = flat[r] ? 0.0 : 1.0 / sigma;
    const uint32_t i = w0 + base + r;
    if (i < rows) {
      mean[i] = mu[r];
      inv_sigma[i] = inv[r];
    }
  }

  // ---- PAA, symbols, hash (sax.cpp:53-80,121-132)
  const double* bp = c_breaks[alphabet - 2];
  uint64_t h[kEncWindows];
  if constexpr (kAligned) {
    const uint32_t len = n / word_len;
    const double scale = static_cast<double>(word_len) / dn, dlen = static_cast<double>(len);
    // both roundings: prefix sums (<= span additions each), len * mu, and the reference's own sum (<= 4 n 2^-53 |seg|)
    const double eps_sum = 3.0 * static_cast<double>(span) * 2.220446049250313e-16 * abs_total * scale;
    bool close = false;
#pragma unroll
    for (int r = 0; r < kEncWindows; ++r) {
      h[r] = 0;
      const double tol = (eps_sum * inv[r] + 1e-11) * tol_scale;
      for (uint32_t k = 0; k < word_len; ++k) {
        const double sum_k = s_p[base + r + (k + 1) * len] - s_p[base + r + k * len];
        const double seg = flat[r] ? 0.0 : (sum_k - dlen * mu[r]) * inv[r] * scale;
        uint32_t sym = 1;
        for (uint32_t b = 0; b + 1 < alphabet; ++b) {
          sym += (bp[b] <= seg) ? 1u : 0u;
          close |= !flat[r] && fabs(seg - bp[b]) <= tol;
        }
        h[r] = h[r] * alphabet + (sym - 1);
      }
    }
    if (!close) {
#pragma unroll
      for (int r = 0; r < kEncWindows; ++r) {
        const uint32_t i = w0 + base + r;
        if (i < rows) hash0[i] = static_cast<uint32_t>(h[r]);
      }
      return;
    }
  }
#pragma unroll
  for (int r = 0; r < kEncWindows; ++r) w[r] = sample(base + r), h[r] = 0;
  uint32_t cur = 0;  // w[r] holds local sample cur of window r
  const double full_units = static_cast<double>(word_len);
  for (uint32_t k = 0; k < word_len; ++k) {
    const uint64_t lo = static_cast<uint64_t>(k) * n;
    const uint64_t hi = lo + n;
    const uint32_t t_first = static_cast<uint32_t>(lo / word_len);
    const uint32_t t_last = static_cast<uint32_t>((hi - 1) / word_len);
    double acc[kEncWindows];
#pragma unroll
    for (int r = 0; r < kEncWindows; ++r) acc[r] = 0.0;
    for (uint32_t t = t_first; t <= t_last; ++t) {
      while (cur < t) {  // (segments meet in at most one shared sample: the window only moves forward)
#pragma unroll
        for (int r = 0; r + 1 < kEncWindows; ++r) w[r] = w[r + 1];
        w[kEncWindows - 1] = sample(base + cur + kEncWindows);
        ++cur;
      }
      // a sample strictly inside the segment counts word_len units of the n*w grid; only the
      // first and the last can be cut by the segment's ends
      double units_d = full_units;
      if (t == t_first || t == t_last) {
        const uint64_t el = static_cast<uint64_t>(t) * word_len;
        const uint64_t eh = el + word_len;
        units_d = static_cast<double>((eh < hi ? eh : hi) - (el > lo ? el : lo));
      }
#pragma unroll
      for (int r = 0; r < kEncWindows; ++r) {
        const double v = flat[r] ? 0.0 : (w[r] - mu[r]) * inv[r];
        acc[r] += units_d * v;
      }
    }
#pragma unroll
    for (int r = 0; r < kEncWindows; ++r) {
      const double seg = acc[r] / dn;
      uint32_t sym = 1;
      for (uint32_t b = 0; b + 1 < alphabet; ++b) sym += (bp[b] <= seg) ? 1u : 0u;
      const uint32_t i = w0 + base + r;
      if (i < rows) {
        if (paa_out) paa_out[static_cast<size_t>(i) * word_len + k] = seg;
        if (sax_out) sax_out[static_cast<size_t>(i) * word_len + k] = sym;
      }
      h[r] = h[r] * alphabet + (sym - 1);
    }
  }
#pragma unroll
  for (int r = 0; r < kEncWindows; ++r) {
    const uint32_t i = w0 + base + r;
    if (i < rows) hash0[i] = static_cast<uint32_t>(h[r]);
  }
}

// Subsequence matrix (series.cpp:46-74), float32: element (i, t) is the
// float64 value (x[i+t] - mu_i) * (1/sigma_i) rounded once.  HBM write-bound:
// a block owns kBuildRows consecutive rows x kBuildCols columns, whose samples
// x[i0 + t0 .. i0 + t0 + kBuildRows + kBuildCols) it stages in shared memory
// ONCE (each sample is needed by up to kBuildRows rows).  Thread j produces
// columns j, j + 256, ... of every row: consecutive lanes read consecutive
// doubles (conflict-free) and write consecutive floats (one full 128-byte line
// per warp and store).
constexpr int kBuildRows = 32;
constexpr int kBuildCols = 1024;
constexpr int kBuildThreads = 256;

//
// The same staged samples also give the 16 segment means of every row (the lower-bound
// summaries of the search): with P the prefix sums of the staged samples, the sum of row r
// over columns [c0, c1) is ((P[r + c1] - P[r + c0]) - (c1 - c0) mu_r) / sigma_r.  A segment
// that lies inside the block's columns is stored directly; one that straddles column blocks
// (stride > 1024) is accumulated with atomicAdd into the pre-zeroed array.
__global__ void __launch_bounds__(kBuildThreads)
k_build_rows(const double* __restrict__ x, const double* __restrict__ mean,
             const double* __restrict__ inv_sigma, uint32_t rows, uint32_t n, uint32_t stride,
             float* __restrict__ out, float* __restrict__ seg_means, float* __restrict__ norms) {
  __shared__ double s_x[kBuildRows + kBuildCols];
  __shared__ double s_p2[kBuildRows + kBuildCols + 1];  // prefix sums of (sample - mean of the block's first row)^2: the row norms
  __shared__ double s_p[kBuildRows + kBuildCols + 1];
  __shared__ double s_mu[kBuildRows], s_inv[kBuildRows];
  const uint32_t i0 = blockIdx.x * kBuildRows;
  const uint32_t t0 = blockIdx.y * kBuildCols;
  const uint32_t n_rows = min(static_cast<uint32_t>(kBuildRows), rows - i0);
  const uint32_t n_cols = min(static_cast<uint32_t>(kBuildCols), stride - t0);
  // samples x[i0 + t0 + e], e < n_rows + n_cols - 1, clipped to the window columns that exist (t < n)
  const uint32_t last_sample = i0 + n_rows - 1 + n;  // exclusive end of what these rows may touch
  for (uint32_t e = threadIdx.x; e < n_rows + n_cols; e += kBuildThreads) {
    const uint32_t at = i0 + t0 + e;
    s_x[e] = at < last_sample ? x[at] : 0.0;
  }
  if (threadIdx.x < n_rows) {
    s_mu[threadIdx.x] = mean[i0 + threadIdx.x];
    s_inv[threadIdx.x] = inv_sigma[i0 + threadIdx.x];
  }
  __syncthreads();
  if ((seg_means != nullptr || norms != nullptr) && threadIdx.x < 32) {  // one warp: prefix sums of the staged samples
    const uint32_t total = n_rows + n_cols, per_lane = (total + 31) / 32;
    const uint32_t lo = min(threadIdx.x * per_lane, total), hi = min(lo + per_lane, total);
    double mine = 0.0;
    for (uint32_t e = lo; e < hi; ++e) mine += s_x[e];
    double incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double up = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (threadIdx.x >= static_cast<uint32_t>(d)) incl += up;
    }
    double run = incl - mine;
    for (uint32_t e = lo; e < hi; ++e) {
      s_p[e] = run;
      run += s_x[e];
    }
    if (threadIdx.x == 31) s_p[total] = run;  // lane 31's range ends at `total` (or is empty: run = grand total)
  } else if (norms != nullptr && threadIdx.x >= 32 && threadIdx.x < 64) {  // a second warp: prefix sums of the shifted squares
    const uint32_t lane = threadIdx.x - 32;
    const uint32_t total = n_rows + n_cols, per_lane = (total + 31) / 32;
    const uint32_t lo = min(lane * per_lane, total), hi = min(lo + per_lane, total);
    const double shift = s_mu[0];
    double mine = 0.0;
    for (uint32_t e = lo; e < hi; ++e) {
      const double v = s_x[e] - shift;
      mine = fma(v, v, mine);
    }
    double incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double up = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= static_cast<uint32_t>(d)) incl += up;
    }
    double run = incl - mine;
    for (uint32_t e = lo; e < hi; ++e) {
      s_p2[e] = run;
      const double v = s_x[e] - shift;
      run = fma(v, v, run);
    }
    if (lane == 31) s_p2[total] = run;
  }
  for (uint32_t r = 0; r < n_rows; ++r) {
    const double mu = s_mu[r], inv = s_inv[r];
    float* dst = out + static_cast<size_t>(i0 + r) * stride + t0;
#pragma unroll
    for (int q = 0; q < kBuildCols / kBuildThreads; ++q) {
      const uint32_t c = threadIdx.x + q * kBuildThreads;
      if (c < n_cols) dst[c] = (t0 + c < n) ? static_cast<float>((s_x[r + c] - mu) * inv) : 0.f;
    }
  }
  if (seg_means == nullptr && norms == nullptr) return;
  __syncthreads();  // s_p and s_p2 complete
  // Squared norms of the rows (the dot-product forms of the search), from the same staged samples: with
  // c the block's first row mean, sum (x - mu_r)^2 = S2 - 2 (mu_r - c) S1 + cnt (mu_r - c)^2 over the shifted
  // samples x - c (S1, S2 from the prefix sums; c keeps every term of the size of the windows' variance).
  // This is the norm of the float64 row; the float32 row's differs by at most 2^-23 of it (every element is
  // rounded once), which the dot forms' error bound carries (engine.cu: dot_error).
  if (norms != nullptr && threadIdx.x < n_rows) {
    const uint32_t r = threadIdx.x;
    const uint32_t c0 = t0, c1 = min(t0 + n_cols, n);
    if (c1 > c0) {
      const double cnt = static_cast<double>(c1 - c0), shift = s_mu[0], d = s_mu[r] - shift;
      const double s1 = (s_p[r + c1 - t0] - s_p[r + c0 - t0]) - cnt * shift;
      const double s2 = s_p2[r + c1 - t0] - s_p2[r + c0 - t0];
      const double part = fmax((s2 - 2.0 * d * s1 + cnt * d * d) * s_inv[r] * s_inv[r], 0.0);
      if (gridDim.y == 1) norms[i0 + r] = static_cast<float>(part);
      else atomicAdd(norms + i0 + r, static_cast<float>(part));  // (rows wider than one column block: pre-zeroed)
    }
  }
  if (seg_means == nullptr) return;
  const uint32_t seg_cols = stride / kLbSegments;
  for (uint32_t item = threadIdx.x; item < n_rows * kLbSegments; item += kBuildThreads) {
    const uint32_t r = item / kLbSegments, seg = item % kLbSegments;
    // columns of the segment that lie in this block and inside the window (t < n)
    const uint32_t c0 = max(seg * seg_cols, t0), c1 = min(min((seg + 1) * seg_cols, t0 + n_cols), n);
    if (c1 <= c0) {
      if (seg * seg_cols >= t0 && (seg + 1) * seg_cols <= t0 + n_cols)  // wholly padding: mean 0
        seg_means[static_cast<size_t>(i0 + r) * kLbSegments + seg] = 0.f;
      continue;
    }
    const double sum = ((s_p[r + c1 - t0] - s_p[r + c0 - t0]) - static_cast<double>(c1 - c0) * s_mu[r]) * s_inv[r];
    const float part = static_cast<float>(sum / static_cast<double>(seg_cols));
    float* dst = seg_means + static_cast<size_t>(i0 + r) * kLbSegments + seg;
    if (seg * seg_cols >= t0 && (seg + 1) * seg_cols <= t0 + n_cols) *dst = part;  // the block holds the whole segment
    else atomicAdd(dst, part);
  }
}

// ------------------------------------------------------------------ lower-bound summaries
// For the covering scan's tile filter (search_kernels.cu): kLbSegments segment means of
// every matrix row (over the padded stride, so every segment has stride / 16 columns;
// produced by k_build_rows), and, per kLbBoxRows consecutive rows, the per-segment minimum
// and maximum (k_segment_boxes).
// For two rows a, b:  sum_t (a_t - b_t)^2  >=  (stride / 16) * sum_k (A_k - B_k)^2
// (Cauchy-Schwarz per segment), and replacing B_k by the nearest point of a box
// [lo_k, hi_k] that contains it can only lower the right-hand side further.
// boxes[unit][0..15] = min, boxes[unit][16..31] = max over the unit's rows; one thread per (unit, segment)
__global__ void k_segment_boxes(const float* __restrict__ means, uint32_t n_rows, float* __restrict__ boxes) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t unit = idx / kLbSegments, k = idx % kLbSegments;
  const uint32_t units = (n_rows + kLbBoxRows - 1) / kLbBoxRows;
  if (unit >= units) return;
  float lo = 3.0e38f, hi = -3.0e38f;
  for (uint32_t r = unit * kLbBoxRows; r < min(n_rows, (unit + 1) * kLbBoxRows); ++r) {
    const float v = means[static_cast<size_t>(r) * kLbSegments + k];
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  boxes[static_cast<size_t>(unit) * 2 * kLbSegments + k] = lo;
  boxes[static_cast<size_t>(unit) * 2 * kLbSegments + kLbSegments + k] = hi;
}

// ------------------------------------------------------------------ scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t value, uint32_t* total) {
  __shared__ uint32_t warp_sums[kScanThreads / 32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = value;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= static_cast<uint32_t>(d)) incl += up;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  uint32_t warp_base = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    const uint32_t s = warp_sums[w];
    if (static_cast<uint32_t>(w) < warp) warp_base += s;
    all += s;
  }
  __syncthreads();
  *total = all;
  return warp_base + incl - value;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_tile(const uint32_t* in, uint32_t* out, uint32_t count, uint32_t* tile_sums) {
  const uint32_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < count) ? in[base + k] : 0u;
    mine += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(mine, &total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < count) out[base + k] = run;
    run += v[k];
  }
  if (tile_sums && threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_add(uint32_t* out, uint32_t count, const uint32_t* tile_offsets) {
  const uint32_t add = tile_offsets[blockIdx.x];
  const uint32_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < count) out[base + k] += add;
}

inline size_t round_up64(size_t v) { return (v + 63) / 64 * 64; }

int scan_recursive(const uint32_t* in, uint32_t* out, uint32_t count, uint32_t* scratch,
                   cudaStream_t stream) {
  const uint32_t tiles = (count + kScanTile - 1) / kScanTile;
  if (tiles <= 1) {
    k_scan_tile<<<1, kScanThreads, 0, stream>>>(in, out, count, nullptr);
    return 1;
  }
  k_scan_tile<<<tiles, kScanThreads, 0, stream>>>(in, out, count, scratch);
  const int deeper = scan_recursive(scratch, scratch, tiles, scratch + round_up64(tiles), stream);
  k_scan_add<<<tiles, kScanThreads, 0, stream>>>(out, count, scratch);
  return 2 + deeper;
}

__global__ void k_iota(uint32_t* out, uint32_t count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = i;
}

// ------------------------------------------------------------------ radix sort
// LSD, 8-bit digits.  A block owns a tile of 4096 consecutive pairs; warp w
// owns the w-th 512 of them and walks them 32 at a time, so the order
// (block, warp, round, lane) is the input order and the sort is stable —
// which is what keeps every bucket ascending by position (index.cpp:92-97).
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;

__global__ void __launch_bounds__(kSortThreads)
k_radix_histogram(const uint32_t* __restrict__ keys, uint32_t count, int shift,
                  uint32_t* __restrict__ hist, uint32_t tiles) {
  __shared__ uint32_t local[256];
  local[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * kSortTile;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t idx = base + k * kSortThreads + threadIdx.x;
    if (idx < count) atomicAdd(&local[(keys[idx] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * tiles + blockIdx.x] = local[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t count,
                int shift, const uint32_t* __restrict__ scanned_hist, uint32_t tiles) {
  __shared__ uint32_t cnt[kSortThreads / 32][256];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int w = 0; w < kSortThreads / 32; ++w) cnt[w][threadIdx.x] = 0;
  __syncthreads();

  const uint32_t base = blockIdx.x * kSortTile + warp * (32 * kSortItems);
  uint32_t key[kSortItems], val[kSortItems], rank[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const uint32_t idx = base + r * 32 + lane;
    const bool valid = idx < count;
    key[r] = valid ? keys_in[idx] : 0u;
    val[r] = valid ? vals_in[idx] : 0u;
    const uint32_t digit = valid ? ((key[r] >> shift) & 255u) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, digit);
    const uint32_t lower = __popc(peers & ((1u << lane) - 1u));
    const uint32_t prior = valid ? cnt[warp][digit] : 0u;
    __syncwarp();
    if (valid && lower == 0) cnt[warp][digit] = prior + __popc(peers);
    __syncwarp();
    rank[r] = prior + lower;
  }
  __syncthreads();
  {
    const uint32_t digit = threadIdx.x;
    uint32_t running = scanned_hist[digit * tiles + blockIdx.x];
    for (int w = 0; w < kSortThreads / 32; ++w) {
      const uint32_t c = cnt[w][digit];
      cnt[w][digit] = running;
      running += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const uint32_t idx = base + r * 32 + lane;
    if (idx < count) {
      const uint32_t dst = cnt[warp][(key[r] >> shift) & 255u] + rank[r];
      TSDD_BOUND(dst, count);
      keys_out[dst] = key[r];
      vals_out[dst] = val[r];
    }
  }
}

// ------------------------------------------------------------------ bucket index
__global__ void k_mark_heads(const uint32_t* __restrict__ sorted_hash, uint32_t rows,
                             uint32_t* __restrict__ heads) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < rows) heads[s] = (s == 0 || sorted_hash[s] != sorted_hash[s - 1]) ? 1u : 0u;
}

// heads[s] = 1 at the first slot of a bucket; slot_bucket[s] holds the
// exclusive scan of heads on entry and the bucket id on exit.
__global__ void k_bucket_offsets(const uint32_t* __restrict__ heads, uint32_t* slot_bucket,
                                 uint32_t rows, uint32_t* __restrict__ offsets,
                                 uint32_t* __restrict__ scalars) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= rows) return;
  const uint32_t head = heads[s];
  const uint32_t id = slot_bucket[s] + head - 1u;
  TSDD_BOUND(id, rows);
  slot_bucket[s] = id;
  if (head) offsets[id] = s;
  if (s == rows - 1) {
    offsets[id + 1] = rows;
    scalars[0] = id + 1;
  }
}

// freq[i] = size of row i's bucket (index.cpp:51-64)
__global__ void k_bucket_freq(const uint32_t* __restrict__ sorted_row,
                              const uint32_t* __restrict__ slot_bucket,
                              const uint32_t* __restrict__ offsets, uint32_t rows,
                              uint32_t* __restrict__ freq) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= rows) return;
  const uint32_t id = slot_bucket[s];
  TSDD_BOUND(id + 1, rows + 1);
  TSDD_BOUND(sorted_row[s], rows);
  freq[sorted_row[s]] = offsets[id + 1] - offsets[id];
}

__global__ void k_count_min_freq(const uint32_t* __restrict__ sorted_freq, uint32_t rows,
                                 uint32_t* __restrict__ scalars) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= rows) return;
  const uint32_t lowest = sorted_freq[0];
  if (sorted_freq[s] == lowest && (s + 1 == rows || sorted_freq[s + 1] != lowest)) scalars[1] = s + 1;
}

__global__ void __launch_bounds__(256)
k_count_runs(const uint32_t* __restrict__ sorted_hash, const uint32_t* __restrict__ sorted_row, uint32_t rows,
             uint32_t* __restrict__ scalars) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const bool run = p + 1 < rows && sorted_hash[p + 1] == sorted_hash[p] && sorted_row[p + 1] == sorted_row[p] + 1;
  const uint32_t n = __popc(__ballot_sync(0xFFFFFFFFu, run));
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(scalars + 2, n);
}

}  // namespace

// ------------------------------------------------------------------ launchers
int launch_widen_series(const float* d_in, double* d_out, size_t m, uint32_t* d_first_bad, cudaStream_t stream) {
  if (d_first_bad != nullptr) cudaMemsetAsync(d_first_bad, 0xFF, sizeof(uint32_t), stream);
  k_widen_series<<<blocks_for(m, 256), 256, 0, stream>>>(d_in, d_out, m, d_first_bad);
  return 1;
}

int launch_window_encode(const double* d_series, uint32_t rows, uint32_t n, uint32_t word_len,
                         uint32_t alphabet, double* d_mean, double* d_inv_sigma, uint32_t* d_hash0,
                         double* d_paa, uint32_t* d_sax, cudaStream_t stream, double tol_scale) {
  const bool aligned = n % word_len == 0 && d_paa == nullptr && d_sax == nullptr && tol_scale > 0.0;
  const size_t smem = encode4_smem_bytes(n, aligned);
  if (smem <= 200 * 1024) {  // (longer windows than ~24,000 samples: the one-window-per-thread kernel)
    auto kernel = aligned ? k_window_encode4<true> : k_window_encode4<false>;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kernel<<<blocks_for(rows, kEncThreads * kEncWindows), kEncThreads, smem, stream>>>(
        d_series, rows, n, word_len, alphabet, d_mean, d_inv_sigma, d_hash0, d_paa, d_sax, tol_scale);
    return 1;
  }
  k_window_encode<<<blocks_for(rows, 256), 256, 0, stream>>>(d_series, rows, n, word_len, alphabet,
                                                             d_mean, d_inv_sigma, d_hash0, d_paa,
                                                             d_sax);
  return 1;
}

int launch_build_rows(const double* d_series, const double* d_mean, const double* d_inv_sigma,
                      uint32_t rows, uint32_t n, uint32_t stride, float* d_rows, float* d_seg_means,
                      cudaStream_t stream, float* d_norms) {
  dim3 grid(blocks_for(rows, kBuildRows), blocks_for(stride, kBuildCols));
  if (d_norms != nullptr)  // (row `rows`, the zero row, has norm 0; wider rows are accumulated)
    cudaMemsetAsync(d_norms, 0, (static_cast<size_t>(rows) + 1) * sizeof(float), stream);
  if (d_seg_means != nullptr && grid.y > 1)  // segments straddle column blocks: they are accumulated
    cudaMemsetAsync(d_seg_means, 0, static_cast<size_t>(rows) * kLbSegments * sizeof(float), stream);
  k_build_rows<<<grid, kBuildThreads, 0, stream>>>(d_series, d_mean, d_inv_sigma, rows, n, stride, d_rows,
                                                   d_seg_means, d_norms);
  return 1;
}

int launch_segment_boxes(const float* d_means, uint32_t rows, float* d_boxes, cudaStream_t stream) {
  const size_t cells = static_cast<size_t>((rows + kLbBoxRows - 1) / kLbBoxRows) * kLbSegments;
  k_segment_boxes<<<blocks_for(cells, 256), 256, 0, stream>>>(d_means, rows, d_boxes);
  return 1;
}

size_t scan_scratch_words(uint32_t count) {
  size_t words = 64;
  size_t level = count;
  while (level > static_cast<size_t>(kScanTile)) {
    level = (level + kScanTile - 1) / kScanTile;
    words += round_up64(level);
  }
  return words;
}

int launch_exclusive_scan(const uint32_t* d_in, uint32_t* d_out, uint32_t count,
                          uint32_t* d_scratch, cudaStream_t stream) {
  if (count == 0) return 0;
  return scan_recursive(d_in, d_out, count, d_scratch, stream);
}

int launch_iota(uint32_t* d_out, uint32_t count, cudaStream_t stream) {
  k_iota<<<blocks_for(count, 256), 256, 0, stream>>>(d_out, count);
  return 1;
}

size_t radix_sort_scratch_words(uint32_t count) {
  const size_t tiles = (static_cast<size_t>(count) + kSortTile - 1) / kSortTile;
  return 256 * tiles;
}

int launch_radix_sort_pairs(uint32_t** keys, uint32_t** vals, uint32_t** keys_alt,
                            uint32_t** vals_alt, uint32_t count, int key_bits, uint32_t* d_hist,
                            uint32_t* d_scan_scratch, cudaStream_t stream) {
  if (count == 0) return 0;
  const uint32_t tiles = (count + kSortTile - 1) / kSortTile;
  int passes = (key_bits + 7) / 8;
  if (passes < 1) passes = 1;
  if (passes > 4) passes = 4;
  int launches = 0;
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = pass * 8;
    k_radix_histogram<<<tiles, kSortThreads, 0, stream>>>(*keys, count, shift, d_hist, tiles);
    launches += 1 + launch_exclusive_scan(d_hist, d_hist, 256 * tiles, d_scan_scratch, stream);
    k_radix_scatter<<<tiles, kSortThreads, 0, stream>>>(*keys, *vals, *keys_alt, *vals_alt, count,
                                                        shift, d_hist, tiles);
    launches += 1;
    uint32_t* t = *keys;
    *keys = *keys_alt;
    *keys_alt = t;
    t = *vals;
    *vals = *vals_alt;
    *vals_alt = t;
  }
  return launches;
}

int launch_bucket_index(const uint32_t* d_sorted_hash, const uint32_t* d_sorted_row, uint32_t rows,
                        uint32_t* d_head_scan, uint32_t* d_slot_bucket, uint32_t* d_offsets,
                        uint32_t* d_freq, uint32_t* d_scalars, uint32_t* d_scan_scratch,
                        cudaStream_t stream) {
  const unsigned blocks = blocks_for(rows, 256);
  k_mark_heads<<<blocks, 256, 0, stream>>>(d_sorted_hash, rows, d_head_scan);
  int launches = 1 + launch_exclusive_scan(d_head_scan, d_slot_bucket, rows, d_scan_scratch, stream);
  k_bucket_offsets<<<blocks, 256, 0, stream>>>(d_head_scan, d_slot_bucket, rows, d_offsets, d_scalars);
  k_bucket_freq<<<blocks, 256, 0, stream>>>(d_sorted_row, d_slot_bucket, d_offsets, rows, d_freq);
  return launches + 2;
}

int launch_count_runs(const uint32_t* d_sorted_hash, const uint32_t* d_sorted_row, uint32_t rows, uint32_t* d_scalars,
                      cudaStream_t stream) {
  k_count_runs<<<blocks_for(rows, 256), 256, 0, stream>>>(d_sorted_hash, d_sorted_row, rows, d_scalars);
  return 1;
}

int launch_count_min_freq(const uint32_t* d_sorted_freq, uint32_t rows, uint32_t* d_scalars,
                          cudaStream_t stream) {
  k_count_min_freq<<<blocks_for(rows, 256), 256, 0, stream>>>(d_sorted_freq, rows, d_scalars);
  return 1;
}

}  // namespace tsdd_b200
