// Search stage on the device (replaces phidd_discord, src/discovery.cpp:209-373).
//
// State per row i (SearchState): nn[i] — a packed (distance^2, neighbour) key
// that only ever decreases (integer atomicMin), so its distance is always an
// upper bound of row i's nearest-neighbour distance; exact[i] once a complete
// scan of every non-self neighbour has finished; and one packed best-so-far
// key that only ever increases (atomicMax).  A row whose upper bound cannot
// beat the best-so-far is dead — the HOTSAX discard (discovery.cpp:58,70).
//
// Exactness rests on the reference's own invariants (discovery.cpp:36-40):
//  * the in-row abandon threshold is the row's running minimum, never the
//    best-so-far (discovery.cpp:55,67): an abandoned pair is strictly above it
//    and can change neither the minimum nor the discard decision;
//  * a stale (smaller) best-so-far prunes less, never more (discovery.hpp:34-36);
//  * all comparisons are strict.

#include "kernels.hpp"

#include <cuda.h>

#include <cstdlib>
#include <cudaTypedefs.h>

#include <type_traits>


namespace tsdd_b200 {

namespace {

inline unsigned blocks_for(size_t items, unsigned per_block) {
  return static_cast<unsigned>((items + per_block - 1) / per_block);
}

__device__ __forceinline__ uint32_t gap_u32(uint32_t a, uint32_t b) { return a > b ? a - b : b - a; }

__device__ __forceinline__ uint64_t load_key(const uint64_t* p) {
  // nn keys are raced on by design (atomicMin from other CTAs); read through L2.
  return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}

// ------------------------------------------------------------------ reset / bookkeeping
__global__ void k_reset_search(SearchState s) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.n_rows) {
    s.nn[i] = kNnUnset;
    s.exact[i] = 0;
    s.excluded[i] = 0;
  }
  if (i == 0) {
    *s.best = 0;
    *s.counters = DeviceCounters{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  }
}

// Two keys per thread (one 16-byte access per array): each array is streamed once, coalesced.
__global__ void __launch_bounds__(256)
k_min_from_peers(uint64_t* __restrict__ nn, PeerPointers peers, uint32_t rows) {
  const uint32_t i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < rows) {
    ulonglong2 mine = *reinterpret_cast<const ulonglong2*>(nn + i);
    for (int p = 0; p < peers.count; ++p) {
      const ulonglong2 other = __ldcg(reinterpret_cast<const ulonglong2*>(peers.ptr[p] + i));
      mine.x = other.x < mine.x ? other.x : mine.x;
      mine.y = other.y < mine.y ? other.y : mine.y;
    }
    *reinterpret_cast<ulonglong2*>(nn + i) = mine;
  } else if (i < rows) {
    uint64_t mine = nn[i];
    for (int p = 0; p < peers.count; ++p) {
      const uint64_t other = load_key(peers.ptr[p] + i);
      mine = other < mine ? other : mine;
    }
    nn[i] = mine;
  }
}

__global__ void k_exclude_zone(SearchState s, uint32_t row) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // 0 .. 2n-2
  const uint32_t lo = row >= s.n - 1 ? row - (s.n - 1) : 0;
  const uint32_t i = lo + t;
  if (i < s.n_rows && i <= row + (s.n - 1)) s.excluded[i] = 1;
}

// best = max over rows that are exact, allowed and have a finite nn.
__global__ void __launch_bounds__(256) k_seed_best(SearchState s) {
  uint64_t mine = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n_rows; i += gridDim.x * blockDim.x) {
    if (s.exact[i] && !s.excluded[i]) {
      const uint32_t bits = key_bits(s.nn[i]);
      if (bits != kInfBits) {
        const uint64_t k = best_key(bits, i);
        mine = k > mine ? k : mine;
      }
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, mine, d);
    mine = other > mine ? other : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine) atomicMax(as_ull(s.best), static_cast<unsigned long long>(mine));
}

// ------------------------------------------------------------------ a best-so-far before the first scan
// The first batch of a search has no best-so-far to discard with until one of its candidates
// has met every row.  The lower-bound summaries give one for free: for a row i,
//   L(i) = min over 16-row boxes u that hold at least one non-self match of i of
//          (stride / 16) * sum_k dist(mean_k(i), [lo_k(u), hi_k(u)])^2
// is a lower bound of i's nearest-neighbour distance (prep_kernels.cu: Cauchy-Schwarz per
// segment), and the discord's distance is >= nn(i) >= L(i) for EVERY i — so max_i L(i) over
// any set of rows (here the first entries of the rarity order) is a valid, if stale,
// best-so-far (discovery.hpp:34-36: a smaller best-so-far prunes less, never more).
// It is installed with the row field of the key empty: any real candidate wins a tie.
constexpr int kSeedUnits = 128;  // boxes staged per block
__global__ void __launch_bounds__(256)
k_seed_lower_bound(SearchState s, const uint32_t* __restrict__ order, uint32_t seed_rows,
                   uint32_t* __restrict__ seed_lb, uint32_t box_step) {
  // (box_step > 1: only every box_step-th box — an UPPER bound of L(i), used to pick the rows worth the full pass)
  __shared__ float4 s_box[kSeedUnits * 2 * kLbSegments / 4];
  const uint32_t units = ((s.n_rows + kLbBoxRows - 1) / kLbBoxRows + box_step - 1) / box_step;  // boxes this launch looks at
  const uint32_t unit0 = blockIdx.x * kSeedUnits;
  const uint32_t n_units = min(static_cast<uint32_t>(kSeedUnits), units - unit0);
  constexpr uint32_t kBoxQuads = 2 * kLbSegments / 4;
  for (uint32_t t = threadIdx.x; t < n_units * kBoxQuads; t += blockDim.x) {
    const size_t box = static_cast<size_t>(unit0 + t / kBoxQuads) * box_step;
    s_box[t] = __ldg(reinterpret_cast<const float4*>(s.lb_boxes + box * 2 * kLbSegments) + t % kBoxQuads);
  }
  __syncthreads();
  const uint32_t e = blockIdx.y * blockDim.x + threadIdx.x;  // one seed row per thread
  if (e < seed_rows) {
    const uint32_t row = order[e];
    float mine[kLbSegments];
    const float4* pm = reinterpret_cast<const float4*>(s.lb_means + static_cast<size_t>(row) * kLbSegments);
#pragma unroll
    for (int q = 0; q < kLbSegments / 4; ++q) {
      const float4 v = __ldg(pm + q);
      mine[4 * q] = v.x, mine[4 * q + 1] = v.y, mine[4 * q + 2] = v.z, mine[4 * q + 3] = v.w;
    }
    float best = __uint_as_float(kInfBits);
    for (uint32_t u = 0; u < n_units; ++u) {
      // a box all of whose rows are self matches of `row` holds no neighbour of it
      const uint32_t r0 = (unit0 + u) * box_step * kLbBoxRows, r1 = min(r0 + kLbBoxRows, s.n_rows) - 1;
      if (gap_u32(row, r0) < s.n && gap_u32(row, r1) < s.n) continue;
      const float4* pb = s_box + u * (2 * kLbSegments / 4);
      float lb = 0.f;
#pragma unroll
      for (int q = 0; q < kLbSegments / 4; ++q) {
        const float4 lo = pb[q], hi = pb[kLbSegments / 4 + q];
        float g;
        g = fmaxf(fmaxf(lo.x - mine[4 * q], mine[4 * q] - hi.x), 0.f), lb = fmaf(g, g, lb);
        g = fmaxf(fmaxf(lo.y - mine[4 * q + 1], mine[4 * q + 1] - hi.y), 0.f), lb = fmaf(g, g, lb);
        g = fmaxf(fmaxf(lo.z - mine[4 * q + 2], mine[4 * q + 2] - hi.z), 0.f), lb = fmaf(g, g, lb);
        g = fmaxf(fmaxf(lo.w - mine[4 * q + 3], mine[4 * q + 3] - hi.w), 0.f), lb = fmaf(g, g, lb);
      }
      best = fminf(best, lb);
    }
    if (best != __uint_as_float(kInfBits)) atomicMin(seed_lb + e, __float_as_uint(best));  // >= 0: bits order like floats
  }
}

__global__ void __launch_bounds__(256)
k_install_seed(SearchState s, const uint32_t* __restrict__ seed_lb, uint32_t seed_rows) {
  __shared__ float s_max[8];
  float mine = 0.f;
  for (uint32_t e = threadIdx.x; e < seed_rows; e += blockDim.x) {
    const uint32_t bits = seed_lb[e];
    if (bits < 0x7F000000u) mine = fmaxf(mine, __uint_as_float(bits));  // (unset slots hold 0x7F7F7F7F)
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mine = fmaxf(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, d));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mine = fmaxf(mine, s_max[w]);
    // 0.5 % below the bound: the means and boxes are float32 (the tile filter allows 0.1 %)
    float seed = mine * s.lb_scale * 0.995f;
    seed -= fmaf(s.lb_q, sqrtf(fmaxf(seed, 0.f)), s.lb_q * s.lb_q);  // absolute part of the means' rounding
    if (seed > 0.f)
      atomicMax(as_ull(s.best), static_cast<unsigned long long>(best_key(__float_as_uint(seed), 0xFFFFFFFFu)));
  }
}

// The `keep` seed rows with the greatest values (ties: the earlier entry): every block stages all the values in
// shared memory and each of its threads ranks ONE entry against them (one block for all of it took 0.47 ms).
constexpr int kSeedSelectMax = 8192;
__global__ void __launch_bounds__(256)
k_seed_select(const uint32_t* __restrict__ order, const uint32_t* __restrict__ upper, uint32_t seed_rows, uint32_t keep,
              uint32_t* __restrict__ kept_rows) {
  __shared__ uint32_t s_val[kSeedSelectMax];
  for (uint32_t e = threadIdx.x; e < seed_rows; e += blockDim.x) s_val[e] = upper[e];
  __syncthreads();
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= seed_rows) return;
  const uint32_t mine = s_val[e];
  uint32_t rank = 0;
  for (uint32_t o = 0; o < seed_rows; ++o) {
    const uint32_t other = s_val[o];
    rank += (other > mine || (other == mine && o < e)) ? 1u : 0u;
  }
  if (rank < keep) kept_rows[rank] = order[e];
}

// ------------------------------------------------------------------ same-word neighbours
// One warp per slot of the hash-sorted order.  The row is measured against up
// to `mates` rows spread evenly over its own bucket (positions at least n
// apart); every completed distance lowers the bound of BOTH rows, d(i,j) =
// d(j,i).  The rows are taken from the SERIES (float64 samples, window mean and 1/sigma), not
// from the matrix: consecutive slots of a bucket are consecutive positions in time, so the
// windows of neighbouring warps overlap almost entirely and come from L1 / L2, where the
// matrix rows (16 GB at workload 4, each read once) had to come from HBM.  Lanes stride over
// the window (256 contiguous bytes per warp per step); the sum is folded with warp shuffles.
// (kSample: float when the series arrived as float32 — the float64 copy holds exactly those values,
// so reading the 4-byte originals and widening in registers gives bit-identical distances for
// half the L1 / L2 traffic, which is what bounds this kernel.)
template <typename kSample>
__global__ void __launch_bounds__(256)
k_bucket_mates(SearchState s, const kSample* __restrict__ x, const double* __restrict__ mean,
               const double* __restrict__ inv_sigma, const uint32_t* __restrict__ sorted_row,
               const uint32_t* __restrict__ slot_bucket, const uint32_t* __restrict__ offsets,
               int mates, uint32_t world, uint32_t rank) {
  const uint32_t lane = threadIdx.x & 31;
  // several ranks that share their bounds afterwards (engine: exchange_bounds) split the slots
  const uint32_t slot = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * world + rank;
  if (slot >= s.n_rows) return;
  const uint32_t bucket = slot_bucket[slot];
  const uint32_t b0 = offsets[bucket], b1 = offsets[bucket + 1];
  const uint32_t len = b1 - b0;
  if (len < 2) return;
  const uint32_t row_i = sorted_row[slot];
  TSDD_BOUND(bucket + 1, s.n_rows + 1);
  TSDD_BOUND(row_i, s.n_rows);
  TSDD_BOUND(b1 - 1, s.n_rows);
  const kSample* pi = x + row_i;
  const double mu_i = mean[row_i], inv_i = inv_sigma[row_i];
  uint32_t tries = static_cast<uint32_t>(mates);
  uint32_t step = len / (tries + 1);
  if (step == 0) {
    step = 1;
    tries = len - 1;
  }
  unsigned long long calls = 0, terms = 0;
  // With a best-so-far already in place (k_install_seed), a row stops as soon as one of its
  // mates has pushed its bound below it: it is dead, more mates would change nothing.
  const uint64_t best = *s.best;
  float bound_i = __uint_as_float(kInfBits);
  for (uint32_t q = 1; q <= tries; ++q) {
    if (dead_bound(bound_i, best, s.margin, s.margin_abs, s.margin_q)) break;
    const uint32_t other = b0 + (slot - b0 + q * step) % len;
    TSDD_BOUND(other, s.n_rows);
    const uint32_t row_j = sorted_row[other];
    TSDD_BOUND(row_j, s.n_rows);
    if (gap_u32(row_i, row_j) < s.n) continue;
    const kSample* pj = x + row_j;
    const double mu_j = mean[row_j], inv_j = inv_sigma[row_j];
    // eight loads in flight per lane before the first use (the kernel is bound by load latency,
    // not arithmetic: ncu long_scoreboard), two accumulators; the order of the additions is not
    // the reference's, nor does it have to be: this is an upper bound, settled later in float64
    double sum_a = 0.0, sum_b = 0.0;
    uint32_t t = lane;
    for (; t + 96 < s.n; t += 128) {
      const double a0 = static_cast<double>(pi[t]), a1 = static_cast<double>(pi[t + 32]), a2 = static_cast<double>(pi[t + 64]),
                   a3 = static_cast<double>(pi[t + 96]);
      const double b0 = static_cast<double>(__ldg(pj + t)), b1 = static_cast<double>(__ldg(pj + t + 32)),
                   b2 = static_cast<double>(__ldg(pj + t + 64)), b3 = static_cast<double>(__ldg(pj + t + 96));
      const double d0 = (a0 - mu_i) * inv_i - (b0 - mu_j) * inv_j, d1 = (a1 - mu_i) * inv_i - (b1 - mu_j) * inv_j;
      const double d2 = (a2 - mu_i) * inv_i - (b2 - mu_j) * inv_j, d3 = (a3 - mu_i) * inv_i - (b3 - mu_j) * inv_j;
      sum_a = fma(d0, d0, sum_a), sum_b = fma(d1, d1, sum_b), sum_a = fma(d2, d2, sum_a), sum_b = fma(d3, d3, sum_b);
    }
    for (; t < s.n; t += 32) {
      const double d = (static_cast<double>(pi[t]) - mu_i) * inv_i - (static_cast<double>(__ldg(pj + t)) - mu_j) * inv_j;
      sum_a = fma(d, d, sum_a);
    }
    double sum64 = sum_a + sum_b;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum64 += __shfl_xor_sync(0xFFFFFFFFu, sum64, d);
    const float sum = static_cast<float>(sum64);
    bound_i = fminf(bound_i, sum);
    if (lane == 0) {
      const uint32_t bits = __float_as_uint(sum);
      atomicMin(as_ull(s.nn + row_i), static_cast<unsigned long long>(nn_key(bits, row_j)));
      atomicMin(as_ull(s.nn + row_j), static_cast<unsigned long long>(nn_key(bits, row_i)));
      calls += 1;
      terms += s.n;
    }
  }
  if (lane == 0 && calls) {
    atomicAdd(&s.counters->calls, calls);
    atomicAdd(&s.counters->terms, terms);
  }
}

// The same step for a float32 series and windows of up to 1,024 samples, in float32 and with every
// load of a pair in flight at once (the float64 version above is bound by load latency: ncu
// long_scoreboard 25 per issue at workload 4, and by its float64 <-> float32 conversions).  The row's own
// window is z-normalised once and kept in registers (kPerLane values a lane); the mates' rows, means
// and 1/sigma are fetched by one lane each, side by side, before the first pair; a pair is then
// kPerLane independent loads followed by five float32 operations a term.  z = ((x - mu_hi) - mu_lo) *
// inv with mu = mu_hi + mu_lo split into two floats: three roundings of 2^-24 relative to |z| besides
// that of 1/sigma, against one for a row of the matrix — so the sum is INFLATED by a bound of its own
// error (relative 1.2e-7 n for the accumulation, absolute 1e-6 sqrt(n d^2) for the four roundings of
// the 2 sqrt(n)-long difference): what is published is an upper bound of the exact distance, which is
// all a bound has to be.  Identical windows still give exactly 0.
template <int kPerLane>
__global__ void __launch_bounds__(256)
k_bucket_mates_f32(SearchState s, const float* __restrict__ x, const double* __restrict__ mean,
                   const double* __restrict__ inv_sigma, const uint32_t* __restrict__ sorted_row,
                   const uint32_t* __restrict__ slot_bucket, const uint32_t* __restrict__ offsets, int mates,
                   uint32_t world, uint32_t rank) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t slot = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * world + rank;
  if (slot >= s.n_rows) return;
  const uint32_t bucket = slot_bucket[slot];
  const uint32_t b0 = offsets[bucket], b1 = offsets[bucket + 1];
  const uint32_t len = b1 - b0;
  if (len < 2) return;
  const uint32_t row_i = sorted_row[slot];
  TSDD_BOUND(bucket + 1, s.n_rows + 1);
  TSDD_BOUND(row_i, s.n_rows);
  TSDD_BOUND(b1 - 1, s.n_rows);
  uint32_t tries = min(static_cast<uint32_t>(mates), 31u);
  uint32_t step = len / (tries + 1);
  if (step == 0) {
    step = 1;
    tries = min(len - 1, 31u);
  }
  // lane q fetches what is needed of mate q (q = 1 .. tries)
  uint32_t my_row = 0xFFFFFFFFu;
  float my_hi = 0.f, my_lo = 0.f, my_inv = 0.f;
  if (lane >= 1 && lane <= tries) {
    const uint32_t other = b0 + (slot - b0 + lane * step) % len;
    TSDD_BOUND(other, s.n_rows);
    const uint32_t r = sorted_row[other];
    TSDD_BOUND(r, s.n_rows);
    if (gap_u32(row_i, r) >= s.n) {
      my_row = r;
      const double mu = mean[r];
      my_hi = static_cast<float>(mu);
      my_lo = static_cast<float>(mu - static_cast<double>(my_hi));
      my_inv = static_cast<float>(inv_sigma[r]);
    }
  }
  float za[kPerLane];
  {
    const double mu = mean[row_i];
    const float hi = static_cast<float>(mu), lo = static_cast<float>(mu - static_cast<double>(hi));
    const float inv = static_cast<float>(inv_sigma[row_i]);
    const float* pi = x + row_i;
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const uint32_t t = lane + 32 * k;
      za[k] = t < s.n ? ((pi[t] - hi) - lo) * inv : 0.f;
    }
  }
  unsigned long long calls = 0, terms = 0;
  const uint64_t best = *s.best;
  const float grow = 1.f + fmaxf(4e-6f, 1.2e-7f * static_cast<float>(s.n)), root_n = sqrtf(static_cast<float>(s.n));
  float bound_i = __uint_as_float(kInfBits);
  for (uint32_t q = 1; q <= tries; ++q) {
    if (dead_bound(bound_i, best, s.margin, s.margin_abs, s.margin_q)) break;
    const uint32_t row_j = __shfl_sync(0xFFFFFFFFu, my_row, q);
    const float hi = __shfl_sync(0xFFFFFFFFu, my_hi, q), lo = __shfl_sync(0xFFFFFFFFu, my_lo, q);
    const float inv = __shfl_sync(0xFFFFFFFFu, my_inv, q);
    if (row_j == 0xFFFFFFFFu) continue;
    const float* pj = x + row_j;
    float b[kPerLane];
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const uint32_t t = lane + 32 * k;
      b[k] = t < s.n ? __ldg(pj + t) : 0.f;
    }
    float sum_a = 0.f, sum_b = 0.f;
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const uint32_t t = lane + 32 * k;
      const float zb = t < s.n ? ((b[k] - hi) - lo) * inv : 0.f;
      const float d = za[k] - zb;
      if (k & 1) sum_b = fmaf(d, d, sum_b);
      else sum_a = fmaf(d, d, sum_a);
    }
    float sum = sum_a + sum_b;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, d);
    sum = fmaf(sum, grow, 1e-6f * root_n * sqrtf(sum));  // an upper bound of the exact distance (see above)
    bound_i = fminf(bound_i, sum);
    if (lane == 0) {
      const uint32_t bits = __float_as_uint(sum);
      atomicMin(as_ull(s.nn + row_i), static_cast<unsigned long long>(nn_key(bits, row_j)));
      atomicMin(as_ull(s.nn + row_j), static_cast<unsigned long long>(nn_key(bits, row_i)));
      calls += 1;
      terms += s.n;
    }
  }
  if (lane == 0 && calls) {
    atomicAdd(&s.counters->calls, calls);
    atomicAdd(&s.counters->terms, terms);
  }
}

// ------------------------------------------------------------------ same-word neighbours along runs of consecutive rows
// Consecutive slots of a bucket are, for the most part, consecutive positions in time (a smooth
// series keeps its word for a while), and so are their mates: the pairs (i, j), (i+1, j+1), ... of
// one warp's 32 slots lie on a diagonal, along which the three sums a pair distance is made of,
//   P = sum (x[i+t]-a)(x[j+t]-b),  SA = sum (x[i+t]-a)^2,  SB = sum (x[j+t]-b)^2      (t < n),
// move by ONE product each per step:  P(i+1, j+1) = P(i, j) - (x[i]-a)(x[j]-b) + (x[i+n]-a)(x[j+n]-b).
// So the warp evaluates the full sums only at the HEADS of its chains (the first lane, and every
// lane whose row or mate does not continue its left neighbour's), all 32 lanes striding over the
// window, and reaches the other lanes with a segmented prefix sum over their one-product deltas: a
// pair costs about 50 instructions instead of 5 n / 32 — workload 4: 5.9 -> ... ms.  Float64
// throughout, with the head's two window means as the shifts a, b: every product is of the size of
// the windows' variance, the sums carry ~n 2^-53 of n sigma_i sigma_j, and the distance
//   d^2 = SSi / sigma_i^2 + SSj / sigma_j^2 - 2 C / (sigma_i sigma_j),  SSi = SA - n (mu_i - a)^2, ...
// — no use of sum z^2 = n, which holds only as far as sigma itself is exact — comes out to ~1e-9
// absolute; it is inflated by 1e-6 relative + 1e-8 n absolute and rounded UP to float32: an upper bound.
// A pair that comes out (almost) at zero is measured again directly, so that exact twins still
// give exactly 0 (a bound of 0 is dead at once).
template <typename kSample>
__global__ void __launch_bounds__(256)
k_bucket_mates_runs(SearchState s, const kSample* __restrict__ x, const double* __restrict__ mean,
                    const double* __restrict__ inv_sigma, const uint32_t* __restrict__ sorted_row,
                    const uint32_t* __restrict__ slot_bucket, const uint32_t* __restrict__ offsets, int mates,
                    uint32_t world, uint32_t rank) {
  const uint32_t lane = threadIdx.x & 31;
  // several ranks that share their bounds afterwards split the 32-slot chunks
  const uint32_t chunk = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * world + rank;
  if (static_cast<uint64_t>(chunk) * 32 >= s.n_rows) return;
  const uint32_t slot = chunk * 32 + lane;
  const bool valid = slot < s.n_rows;
  uint32_t b0 = 0, len = 0, row_i = 0xFFFFFFFFu;
  double mu_i = 0.0, inv_i = 0.0;
  if (valid) {
    const uint32_t bucket = slot_bucket[slot];
    TSDD_BOUND(bucket + 1, s.n_rows + 1);
    b0 = offsets[bucket];
    len = offsets[bucket + 1] - b0;
    row_i = sorted_row[slot];
    TSDD_BOUND(row_i, s.n_rows);
    mu_i = mean[row_i];
    inv_i = inv_sigma[row_i];
  }
  uint32_t tries = min(static_cast<uint32_t>(mates), 31u), step = len / (tries + 1);
  if (step == 0) {
    step = 1;
    tries = len > 0 ? min(len - 1, 31u) : 0u;
  }
  if (!valid || len < 2) tries = 0;
  uint32_t most = tries;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) most = max(most, __shfl_xor_sync(0xFFFFFFFFu, most, d));
  const uint64_t best = *s.best;
  const double dn = static_cast<double>(s.n);
  float bound_i = __uint_as_float(kInfBits);
  unsigned long long calls = 0, terms = 0;
  for (uint32_t q = 1; q <= most; ++q) {
    bool active = q <= tries && !dead_bound(bound_i, best, s.margin, s.margin_abs, s.margin_q);
    uint32_t row_j = 0xFFFFFFFFu;
    double mu_j = 0.0, inv_j = 0.0;
    if (active) {
      const uint32_t other = b0 + (slot - b0 + q * step) % len;
      TSDD_BOUND(other, s.n_rows);
      row_j = sorted_row[other];
      TSDD_BOUND(row_j, s.n_rows);
      if (gap_u32(row_i, row_j) < s.n) {
        active = false;
      } else {
        mu_j = mean[row_j];
        inv_j = inv_sigma[row_j];
      }
    }
    const uint32_t act = __ballot_sync(0xFFFFFFFFu, active);
    if (act == 0) {
      if (__ballot_sync(0xFFFFFFFFu, q < tries && !dead_bound(bound_i, best, s.margin, s.margin_abs, s.margin_q)) == 0) break;
      continue;
    }
    // chains: lane k continues lane k-1 when both its row and its mate are the next position
    const uint32_t pi = __shfl_up_sync(0xFFFFFFFFu, row_i, 1), pj = __shfl_up_sync(0xFFFFFFFFu, row_j, 1);
    const bool prev_active = lane > 0 && ((act >> (lane - 1)) & 1u);
    const bool follows = active && prev_active && row_i == pi + 1 && row_j == pj + 1;
    const bool head = active && !follows;
    const uint32_t heads = __ballot_sync(0xFFFFFFFFu, head);
    const uint32_t my_head = active ? 31u - __clz(heads & (0xFFFFFFFFu >> (31 - lane))) : lane;
    const double a = __shfl_sync(0xFFFFFFFFu, mu_i, my_head), b = __shfl_sync(0xFFFFFFFFu, mu_j, my_head);
    double P = 0.0, SA = 0.0, SB = 0.0;
    if (follows) {  // one step along the diagonal: the window loses sample -1 and gains sample n-1
      const double uo = static_cast<double>(x[row_i - 1]) - a, vo = static_cast<double>(x[row_j - 1]) - b;
      const double un = static_cast<double>(x[row_i + s.n - 1]) - a, vn = static_cast<double>(x[row_j + s.n - 1]) - b;
      P = un * vn - uo * vo;
      SA = un * un - uo * uo;
      SB = vn * vn - vo * vo;
    }
    for (uint32_t todo = heads; todo != 0; todo &= todo - 1) {  // the full sums of every chain's first pair
      const int h = __ffs(todo) - 1;
      const uint32_t ri = __shfl_sync(0xFFFFFFFFu, row_i, h), rj = __shfl_sync(0xFFFFFFFFu, row_j, h);
      const double ha = __shfl_sync(0xFFFFFFFFu, mu_i, h), hb = __shfl_sync(0xFFFFFFFFu, mu_j, h);
      const kSample* qi = x + ri;
      const kSample* qj = x + rj;
      double p0 = 0.0, p1 = 0.0, sa0 = 0.0, sa1 = 0.0, sb0 = 0.0, sb1 = 0.0;
      uint32_t t = lane;
      for (; t + 32 < s.n; t += 64) {
        const kSample x0 = qi[t], x1 = qi[t + 32], y0 = __ldg(qj + t), y1 = __ldg(qj + t + 32);
        const double u0 = static_cast<double>(x0) - ha, u1 = static_cast<double>(x1) - ha;
        const double v0 = static_cast<double>(y0) - hb, v1 = static_cast<double>(y1) - hb;
        p0 = fma(u0, v0, p0), p1 = fma(u1, v1, p1);
        sa0 = fma(u0, u0, sa0), sa1 = fma(u1, u1, sa1);
        sb0 = fma(v0, v0, sb0), sb1 = fma(v1, v1, sb1);
      }
      if (t < s.n) {
        const double u0 = static_cast<double>(qi[t]) - ha, v0 = static_cast<double>(__ldg(qj + t)) - hb;
        p0 = fma(u0, v0, p0), sa0 = fma(u0, u0, sa0), sb0 = fma(v0, v0, sb0);
      }
      double p = p0 + p1, sa = sa0 + sa1, sb = sb0 + sb1;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        p += __shfl_xor_sync(0xFFFFFFFFu, p, d);
        sa += __shfl_xor_sync(0xFFFFFFFFu, sa, d);
        sb += __shfl_xor_sync(0xFFFFFFFFu, sb, d);
      }
      if (static_cast<int>(lane) == h) P = p, SA = sa, SB = sb;
    }
    // segmented inclusive prefix sums: a head holds its chain's full sums, a follower its delta
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double tp = __shfl_up_sync(0xFFFFFFFFu, P, d), ta = __shfl_up_sync(0xFFFFFFFFu, SA, d),
                   tb = __shfl_up_sync(0xFFFFFFFFu, SB, d);
      if (active && lane >= my_head + d) P += tp, SA += ta, SB += tb;
    }
    float sum = __uint_as_float(kInfBits);
    bool again = false;
    if (active) {
      const double da = mu_i - a, db = mu_j - b;
      const double ssi = SA - dn * da * da, ssj = SB - dn * db * db, cov = P - dn * da * db;
      double d2 = inv_i * inv_i * ssi + inv_j * inv_j * ssj - 2.0 * inv_i * inv_j * cov;
      d2 = fmax(d2, 0.0);
      again = d2 < 1e-6 * dn;  // (almost) a twin: settled by the direct sum below
      sum = __double2float_ru(fma(d2, 1.0 + 1e-6, 1e-8 * dn));
    }
    for (uint32_t todo = __ballot_sync(0xFFFFFFFFu, again); todo != 0; todo &= todo - 1) {
      const int h = __ffs(todo) - 1;
      const uint32_t ri = __shfl_sync(0xFFFFFFFFu, row_i, h), rj = __shfl_sync(0xFFFFFFFFu, row_j, h);
      const double ma = __shfl_sync(0xFFFFFFFFu, mu_i, h), mb = __shfl_sync(0xFFFFFFFFu, mu_j, h);
      const double ia = __shfl_sync(0xFFFFFFFFu, inv_i, h), ib = __shfl_sync(0xFFFFFFFFu, inv_j, h);
      double acc = 0.0;
      for (uint32_t t = lane; t < s.n; t += 32) {
        const double d = (static_cast<double>(x[ri + t]) - ma) * ia - (static_cast<double>(__ldg(x + rj + t)) - mb) * ib;
        acc = fma(d, d, acc);
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
      if (static_cast<int>(lane) == h) sum = __double2float_ru(acc);
    }
    if (active) {
      bound_i = fminf(bound_i, sum);
      const uint32_t bits = __float_as_uint(sum);
      atomicMin(as_ull(s.nn + row_i), static_cast<unsigned long long>(nn_key(bits, row_j)));
      atomicMin(as_ull(s.nn + row_j), static_cast<unsigned long long>(nn_key(bits, row_i)));
      calls += 1;
      terms += head || again ? s.n : 2u;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    calls += __shfl_xor_sync(0xFFFFFFFFu, calls, d);
    terms += __shfl_xor_sync(0xFFFFFFFFu, terms, d);
  }
  if (lane == 0 && calls) {
    atomicAdd(&s.counters->calls, calls);
    atomicAdd(&s.counters->terms, terms);
  }
}

// ------------------------------------------------------------------ time topology
// Overlapping windows have overlapping matches.  If row a = c + delta has found a neighbour j at
// distance d, then rows c and j - delta are those same two windows, both shifted by delta
// samples: all but |delta| of their columns were part of d(a, j), so d(c, j - delta) is usually
// close to d.  One warp per batch candidate: each lane looks at one row a within kReach
// positions of c and proposes j - delta; the proposals backed by the smallest bounds are
// measured (up to `tries` of them, full float32 distance from the matrix), and each result
// lowers the bound of BOTH rows.  In time series whose anomalies are short, almost every row
// has a neighbour in time that already knows a good match — from the bucket mates, the window
// rounds, or the symmetric updates of earlier scans — and is discarded here, for the price of
// one or two pair distances, before it ever enters a tile.  (Only real pair distances lower
// bounds, so exactness is untouched; the reference has no such step — it is the "time
// topology" heuristic of later HOTSAX variants.)
constexpr int kReach = 16;
__global__ void __launch_bounds__(256)
k_propagate(SearchState s, const uint32_t* __restrict__ batch_rows, const uint32_t* __restrict__ sel, int tries) {
  const uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (idx >= sel[0]) return;
  const uint32_t c = batch_rows[idx];
  const uint64_t best = *s.best;
  uint64_t key_c = load_key(s.nn + c);
  if (is_dead(key_c, best, s.margin, s.margin_abs, s.margin_q)) return;
  const int delta = lane < kReach ? -static_cast<int>(lane + 1) : static_cast<int>(lane) - (kReach - 1);
  const long long a = static_cast<long long>(c) + delta;
  uint64_t proposal = ~0ull;  // (anchor's bound bits << 32) | lane; ~0 = none
  uint32_t jj = 0xFFFFFFFFu;
  if (a >= 0 && a < static_cast<long long>(s.n_rows)) {
    const uint64_t key_a = load_key(s.nn + a);
    const uint32_t j = static_cast<uint32_t>(key_a);
    const long long shifted = static_cast<long long>(j) - delta;
    if (j != 0xFFFFFFFFu && shifted >= 0 && shifted < static_cast<long long>(s.n_rows) &&
        gap_u32(c, static_cast<uint32_t>(shifted)) >= s.n && static_cast<uint32_t>(shifted) != static_cast<uint32_t>(key_c)) {
      jj = static_cast<uint32_t>(shifted);
      proposal = (static_cast<uint64_t>(key_bits(key_a)) << 32) | lane;
    }
  }
  const float4* pc = reinterpret_cast<const float4*>(s.rows + static_cast<size_t>(c) * s.stride);
  unsigned long long calls = 0;
  for (int t = 0; t < tries; ++t) {
    uint64_t winner = proposal;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, winner, d);
      winner = other < winner ? other : winner;
    }
    if (winner == ~0ull) break;
    const uint32_t j_now = __shfl_sync(0xFFFFFFFFu, jj, static_cast<int>(winner & 31u));
    TSDD_BOUND(c, s.n_rows);
    TSDD_BOUND(j_now, s.n_rows);
    if (jj == j_now) proposal = ~0ull;  // (this proposal, and every other lane's copy of it)
    const float4* pj = reinterpret_cast<const float4*>(s.rows + static_cast<size_t>(j_now) * s.stride);
    float sum = 0.f;
    for (uint32_t q = lane; q < s.stride / 4; q += 32) {
      const float4 x = __ldg(pc + q), y = __ldg(pj + q);
      const float d0 = x.x - y.x, d1 = x.y - y.y, d2 = x.z - y.z, d3 = x.w - y.w;
      sum = fmaf(d0, d0, sum), sum = fmaf(d1, d1, sum), sum = fmaf(d2, d2, sum), sum = fmaf(d3, d3, sum);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, d);
    calls += 1;
    if (lane == 0) {
      const uint32_t bits = __float_as_uint(sum);
      atomicMin(as_ull(s.nn + c), static_cast<unsigned long long>(nn_key(bits, j_now)));
      atomicMin(as_ull(s.nn + j_now), static_cast<unsigned long long>(nn_key(bits, c)));
    }
    if (dead_bound(sum, best, s.margin, s.margin_abs, s.margin_q)) break;  // (warp-uniform)
  }
  if (lane == 0 && calls) {
    atomicAdd(&s.counters->calls, calls);
    atomicAdd(&s.counters->terms, calls * s.n);
    atomicAdd(&s.counters->propagated, calls);
  }
}

// ------------------------------------------------------------------ batch selection
// flags[e - cursor] = 1 when entry e of the rarity order is this rank's and
// its row can still beat the best-so-far.
__global__ void k_flag_live(SearchState s, const uint32_t* __restrict__ order, uint32_t cursor,
                            uint32_t world, uint32_t rank, int pruning, uint32_t* __restrict__ flags) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t e = cursor + t;
  if (e >= s.n_rows) return;
  const uint32_t row = order[e];
  TSDD_BOUND(row, s.n_rows);
  bool live = (e % world == rank) && !s.excluded[row] && !s.exact[row];
  if (live && pruning) live = !is_dead(s.nn[row], *s.best, s.margin, s.margin_abs, s.margin_q);
  flags[t] = live ? 1u : 0u;
}

// ranks[] is the exclusive scan of flags[].  The first `batch` live entries
// become the batch; sel[0] = batch size, sel[1] = cursor after the last one taken.
__global__ void k_take_batch(const uint32_t* __restrict__ order, const uint32_t* __restrict__ flags,
                             const uint32_t* __restrict__ ranks, uint32_t cursor, uint32_t n_rows,
                             uint32_t batch, uint32_t* __restrict__ batch_rows,
                             uint32_t* __restrict__ sel) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t e = cursor + t;
  if (e >= n_rows) return;
  const uint32_t f = flags[t], r = ranks[t];
  if (f && r < batch) {
    TSDD_BOUND(order[e], n_rows);
    batch_rows[r] = order[e];
    if (r == batch - 1) sel[1] = e + 1;
  }
  if (e == n_rows - 1) {
    const uint32_t live = r + f;
    sel[0] = live < batch ? live : batch;
    if (live < batch) sel[1] = n_rows;
  }
}

// Stable compaction of the batch list (a single block; a batch is a few
// thousand rows): rows and their hash-order slots move together.  sel[0] is
// read and rewritten.
__global__ void __launch_bounds__(1024)
k_compact_batch(SearchState s, const uint32_t* __restrict__ in, const uint32_t* __restrict__ in_slots,
                uint32_t* __restrict__ out, uint32_t* __restrict__ out_slots, int pruning, uint32_t* sel) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry;
  const uint32_t count = sel[0];
  const uint64_t best = *s.best;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < count; base += blockDim.x) {
    const uint32_t idx = base + threadIdx.x;
    uint32_t row = 0, slot = 0;
    bool keep = false;
    if (idx < count) {
      row = in[idx];
      slot = in_slots[idx];
      TSDD_BOUND(row, s.n_rows);
      keep = !pruning || !is_dead(load_key(s.nn + row), best, s.margin, s.margin_abs, s.margin_q);
    }
    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, keep);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_sums[warp] = __popc(ballot);
    __syncthreads();
    uint32_t before = carry, total = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      const uint32_t c = warp_sums[w];
      if (w < warp) before += c;
      total += c;
    }
    if (keep) {
      const uint32_t at = before + __popc(ballot & ((1u << lane) - 1u));
      TSDD_BOUND(at, count);
      out[at] = row;
      out_slots[at] = slot;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) sel[0] = carry;
}

// The same compaction over many blocks, for batches worth it: k_compact_flag marks the entries
// that stay and counts them per block of 1,024; k_compact_scatter places each block after the
// ones before it (stable), the last block stores the new size.  Both read the size from sel[0];
// nothing else runs on the stream in between, so the marks are the ones the counts were made of.
__global__ void __launch_bounds__(1024)
k_compact_flag(SearchState s, const uint32_t* __restrict__ in, int pruning, const uint32_t* __restrict__ sel,
               uint32_t* __restrict__ keep_flags, uint32_t* __restrict__ block_counts) {
  const uint32_t count = sel[0];
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  if (idx < count) TSDD_BOUND(in[idx], s.n_rows);
  if (idx < count) keep = !pruning || !is_dead(load_key(s.nn + in[idx]), *s.best, s.margin, s.margin_abs, s.margin_q);
  if (idx < count) keep_flags[idx] = keep ? 1u : 0u;
  const int kept = __syncthreads_count(keep);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = static_cast<uint32_t>(kept);
}

__global__ void __launch_bounds__(1024)
k_compact_scatter(const uint32_t* __restrict__ in, const uint32_t* __restrict__ in_slots,
                  uint32_t* __restrict__ out, uint32_t* __restrict__ out_slots,
                  const uint32_t* __restrict__ keep_flags, const uint32_t* __restrict__ block_counts,
                  uint32_t* sel) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t s_base;
  const uint32_t count = sel[0];
  const uint32_t blocks_used = (count + blockDim.x - 1) / blockDim.x;
  if (blockIdx.x >= blocks_used && !(blockIdx.x == 0 && count == 0)) return;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {  // entries kept by the blocks before this one (at most a few hundred counts)
    uint32_t before = 0;
    for (uint32_t b = lane; b < blockIdx.x; b += 32) before += block_counts[b];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) before += __shfl_xor_sync(0xFFFFFFFFu, before, d);
    if (lane == 0) s_base = before;
  }
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const bool keep = idx < count && keep_flags[idx] != 0;
  const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, keep);
  if (lane == 0) warp_sums[warp] = __popc(ballot);
  __syncthreads();
  uint32_t before = s_base;
  for (uint32_t w = 0; w < warp; ++w) before += warp_sums[w];
  if (keep) {
    const uint32_t at = before + __popc(ballot & ((1u << lane) - 1u));
    TSDD_BOUND(at, count);
    out[at] = in[idx];
    out_slots[at] = in_slots[idx];
  }
  __syncthreads();
  if (blockIdx.x + 1 == max(blocks_used, 1u) && threadIdx.x == 0) {
    uint32_t total = s_base;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) total += warp_sums[w];
    sel[2] = total;  // parked: other blocks may still be reading sel[0]; k_compact_publish moves it there
  }
}

__global__ void k_compact_publish(uint32_t* sel) { sel[0] = sel[2]; }

// slot_of_row[sorted_row[s]] = s: where each row sits in the hash-sorted order.
__global__ void k_invert_order(const uint32_t* __restrict__ sorted_row, uint32_t rows,
                               uint32_t* __restrict__ slot_of_row) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < rows) {
    TSDD_BOUND(sorted_row[s], rows);
    slot_of_row[sorted_row[s]] = s;
  }
}

// keys[i] = hash-order slot of batch row i (the sort key that makes tiles word-coherent)
__global__ void k_batch_slots(const uint32_t* __restrict__ batch_rows, const uint32_t* __restrict__ sel,
                              const uint32_t* __restrict__ slot_of_row, uint32_t* __restrict__ keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < sel[0]) keys[i] = slot_of_row[batch_rows[i]];  // (batch rows are checked where they are selected)
}

// Dense copy of the batch's rows, NEGATED, so that the tile kernel forms
// x - y as one add (and, packed, one add.f32x2).  Rows past the batch size
// are zero.  One warp per row.
//
// The tensor-map variant of the warp-specialised kernel receives a candidate tile as TMA boxes
// with the hardware's 128-byte swizzle (16-byte piece p of row r lands at piece p ^ (r & 7)).  Its
// thread row ty reads 8 rows that share r & 7, so that the XOR is one per-thread constant:
// rows (ty & 7) + 64 (ty >> 3) + 8 u.  For a warp (thread rows 2w, 2w + 1) to still own 16
// CONSECUTIVE candidates of the word-sorted batch, candidate L = 16 w + 2 u + b of a tile is
// stored at row 2 (w & 3) + b + 8 u + 64 (w >> 2).
__host__ __device__ __forceinline__ uint32_t tma_row_of_candidate(uint32_t l) {
  const uint32_t w = l >> 4, u = (l >> 1) & 7u, b = l & 1u;
  return 2u * (w & 3u) + b + 8u * u + 64u * (w >> 2);
}
// The 16 x 8 variant (k_scan_tiles_ws16): tiles of 256 candidates stored as 128 row PAIRS, the two
// rows of a pair interleaved column by column.  Candidate L = 16 ty + 2 i + h of a tile is half h
// of pair (ty & 7) + 8 i + 64 (ty >> 3).
__host__ __device__ __forceinline__ uint32_t tma16_pair_of_candidate(uint32_t l) {
  const uint32_t ty = l >> 4, i = (l >> 1) & 7u;
  return (ty & 7u) + 8u * i + 64u * (ty >> 3);
}
__global__ void __launch_bounds__(256)
k_gather_rows(SearchState s, const uint32_t* __restrict__ batch_rows, const uint32_t* __restrict__ sel,
              uint32_t capacity_padded, int tma_layout, float* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= capacity_padded) return;
  const uint32_t count = sel[0];
  // only the tiles the scan will touch need refreshing
  const uint32_t tile_rows = tma_layout == 2 ? 256u : static_cast<uint32_t>(kTileRows);
  if (r >= (count + tile_rows - 1) / tile_rows * tile_rows) return;
  const uint32_t quads = s.stride / 4;
  if (tma_layout == 2) {  // pairwise interleaved (k_scan_tiles_ws16)
    const uint32_t l = r & 255u, pair = (r >> 8) * 128u + tma16_pair_of_candidate(l);
    float2* dst2 = reinterpret_cast<float2*>(out + static_cast<size_t>(pair) * 2 * s.stride);
    float* dst1 = reinterpret_cast<float*>(dst2) + (l & 1u);
    if (r < count) {
      TSDD_BOUND(batch_rows[r], s.n_rows);
      const float4* src = reinterpret_cast<const float4*>(s.rows + static_cast<size_t>(batch_rows[r]) * s.stride);
      for (uint32_t c = lane; c < quads; c += 32) {
        const float4 v = __ldg(src + c);
        dst1[8 * c] = -v.x, dst1[8 * c + 2] = -v.y, dst1[8 * c + 4] = -v.z, dst1[8 * c + 6] = -v.w;
      }
    } else {
      for (uint32_t c = lane; c < quads; c += 32)
        dst1[8 * c] = 0.f, dst1[8 * c + 2] = 0.f, dst1[8 * c + 4] = 0.f, dst1[8 * c + 6] = 0.f;
    }
    return;
  }
  // tma_layout 1: candidate L of a tile sits at row tma_row_of_candidate(L) of the tile
  const uint32_t at = tma_layout ? (r & ~(kTileRows - 1u)) + tma_row_of_candidate(r & (kTileRows - 1u)) : r;
  float4* dst = reinterpret_cast<float4*>(out + static_cast<size_t>(at) * s.stride);
  if (r < count) {
    TSDD_BOUND(batch_rows[r], s.n_rows);
    const float4* src =
        reinterpret_cast<const float4*>(s.rows + static_cast<size_t>(batch_rows[r]) * s.stride);
    for (uint32_t c = lane; c < quads; c += 32) {
      const float4 v = __ldg(src + c);
      dst[c] = make_float4(-v.x, -v.y, -v.z, -v.w);
    }
  } else {
    for (uint32_t c = lane; c < quads; c += 32) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Rows of the batch that are still live after every neighbour range has been
// scanned have met all their non-self neighbours: nn is exact.  Each raises
// the best-so-far (warp-shuffle max, then one atomicMax per warp).
__global__ void __launch_bounds__(256)
k_finalize_batch(SearchState s, const uint32_t* __restrict__ batch_rows,
                 const uint32_t* __restrict__ sel, int pruning) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t count = sel[0];
  const uint64_t best = *s.best;  // constant for the whole batch: only this kernel raises it
  uint64_t mine = 0;
  if (idx < count) {
    const uint32_t row = batch_rows[idx];
    TSDD_BOUND(row, s.n_rows);
    const uint64_t key = s.nn[row];
    if (!pruning || !is_dead(key, best, s.margin, s.margin_abs, s.margin_q)) {
      s.exact[row] = 1;
      if (key_bits(key) != kInfBits) mine = best_key(key_bits(key), row);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, mine, d);
    mine = other > mine ? other : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine > best)
    atomicMax(as_ull(s.best), static_cast<unsigned long long>(mine));
}

// ------------------------------------------------------------------ the tiled distance kernel
//
// CTA = 256 threads = a tile of 128 candidates x kNbr neighbour rows (64 by
// default, two CTAs per SM; 128 with "wide_tile"); thread (ty, tx) of a 16 x 16
// grid owns the pairs {ty + 16u} x {tx + 16w}.  Columns stream through shared
// memory kChunk (64) at a time in a kStages-deep cp.async ring — a 64-column
// stage is ~16k cycles of arithmetic per CTA, many times the L2/HBM latency,
// so two stages suffice and leave room for the second CTA.  The 16-byte
// pieces of a row are XOR-swizzled with the row number so that the LDS.128 of
// the rows of a quarter-warp are conflict-free.  Candidate rows arrive negated
// (k_gather_rows), so a term is one add and one fma — packed two columns at a
// time as add.f32x2 / fma.rn.f32x2 (FADD2 / FFMA2) in the kPacked variant.
//
// Early abandoning (series.hpp:117-146 on a tile): after every chunk a thread
// checks whether all of its partial sums already exceed their candidates'
// running minimum; a warp whose pairs have all abandoned stops computing, and
// the CTA leaves the tile when every warp has.  Dead candidates carry the
// threshold -1 and never hold a tile open.
constexpr int kStages = TSDD_SCAN_STAGES;
constexpr int kRowBytes = kChunk * 4;   // bytes of one row inside a stage
constexpr int kPieces = kChunk / 4;     // 16-byte pieces per row and stage
constexpr int kScanThreads = 256;
constexpr size_t scan_smem_bytes(int cand_rows, int nbr_rows) {
  return static_cast<size_t>(kStages) * (cand_rows + nbr_rows) * kChunk * 4 + 7 * kTileRows * 4;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int kPending>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(kPending));
}

// Issues this thread's share of one stage (1024 + 1024 pieces of 16 bytes per
// CTA).  The neighbour rows are addressed through s_brow (row numbers in shared
// memory), so a tile may hold any 128 rows: every piece is still one 16-byte
// part of a full 128-byte line.
// s_map (may be null): slot r of the stage holds candidate s_map[r] of the tile for r < n_mapped —
// the candidates that take part, packed to the front (k_scan_tiles, kLb); the slots behind them are
// filled with the first of those rows (finite values; nobody looks at their sums).
template <int kCand, int kNbr>
__device__ __forceinline__ void issue_stage(unsigned char* stage, const float* a_tile,
                                            const float* rows, const uint32_t* s_brow,
                                            uint32_t stride, uint32_t col0, const uint32_t* s_map = nullptr,
                                            uint32_t n_mapped = 0) {
#pragma unroll
  for (int q = 0; q < kCand * kPieces / kScanThreads; ++q) {  // candidate rows
    const uint32_t piece = threadIdx.x + q * kScanThreads;
    const uint32_t r = piece / kPieces, kc = piece % kPieces;
    const uint32_t from = s_map ? s_map[r < n_mapped ? r : 0u] : r;
    // candidate rows are swizzled by (r >> 3): a thread's 8 rows 8 ty .. 8 ty + 7 then share one
    // slot pattern, and the two thread rows of a warp (ty, ty + 1) get different ones
    cp_async16(stage + r * kRowBytes + ((kc ^ ((r >> 3) & 7)) << 4),
               a_tile + static_cast<size_t>(from) * stride + col0 + kc * 4);
  }
#pragma unroll
  for (int q = 0; q < kNbr * kPieces / kScanThreads; ++q) {  // neighbour rows
    const uint32_t piece = threadIdx.x + q * kScanThreads;
    const uint32_t r = piece / kPieces, kc = piece % kPieces;
    cp_async16(stage + kCand * kRowBytes + r * kRowBytes + ((kc ^ (r & 7)) << 4),
               rows + static_cast<size_t>(s_brow[r]) * stride + col0 + kc * 4);  // (s_brow is checked where it is written)
  }
}

// Per-thread accumulators of a kU x kW block of pairs.  Packed: two partial
// sums per pair (even / odd columns) in one 64-bit register pair, updated with
// add.f32x2 / fma.rn.f32x2.
template <bool kPacked, int kU, int kW>
struct Acc;
template <int kU, int kW>
struct Acc<false, kU, kW> {
  float v[kU][kW];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int w = 0; w < kW; ++w) v[u][w] = 0.f;
  }
  __device__ __forceinline__ float get(int u, int w) const { return v[u][w]; }
  __device__ __forceinline__ void add(int u, int w, const float4& na, const float4& b) {
    float d = b.x + na.x;
    v[u][w] = fmaf(d, d, v[u][w]);
    d = b.y + na.y;
    v[u][w] = fmaf(d, d, v[u][w]);
    d = b.z + na.z;
    v[u][w] = fmaf(d, d, v[u][w]);
    d = b.w + na.w;
    v[u][w] = fmaf(d, d, v[u][w]);
  }
};
template <int kU, int kW>
struct Acc<true, kU, kW> {
  float2 v[kU][kW];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int w = 0; w < kW; ++w) v[u][w] = make_float2(0.f, 0.f);
  }
  __device__ __forceinline__ float get(int u, int w) const { return v[u][w].x + v[u][w].y; }
  __device__ __forceinline__ void add(int u, int w, const float4& na, const float4& b) {
    float2 d = __fadd2_rn(make_float2(b.x, b.y), make_float2(na.x, na.y));
    v[u][w] = __ffma2_rn(d, d, v[u][w]);
    d = __fadd2_rn(make_float2(b.z, b.w), make_float2(na.z, na.w));
    v[u][w] = __ffma2_rn(d, d, v[u][w]);
  }
  // dot-product form: one FFMA2 per two columns; the candidate rows are stored negated, so
  // this accumulates -(a . b)
  __device__ __forceinline__ void dot(int u, int w, const float4& na, const float4& b) {
    v[u][w] = __ffma2_rn(make_float2(b.x, b.y), make_float2(na.x, na.y), v[u][w]);
    v[u][w] = __ffma2_rn(make_float2(b.z, b.w), make_float2(na.z, na.w), v[u][w]);
  }
};

// Which neighbour rows (kNbr = 64 or 128 of them) tile number k of a scan holds.
//   global mode (nbr_index == nullptr): rows [kNbr t, kNbr t + kNbr), t = (k + rotation)
//     mod T — every row exactly once over k = 0 .. T-1 whatever the rotation; this
//     is the scan that makes a survivor exact.
//   window mode: slots of the hash-sorted order around the candidate tile's own
//     bucket, alternating outwards (own tile, +1, -1, +2, ...), wrapping at the
//     ends — the HOTSAX "same word first" heuristic (discovery.cpp:51-63)
//     widened to neighbouring words.  It only lowers bounds; coverage is not
//     counted, so re-centring after a compaction is harmless.
struct ScanArgs {
  const float* batch;          // dense, negated candidate rows
  const uint32_t* batch_rows;  // candidate row numbers
  const uint32_t* batch_slots; // their slots in the hash-sorted order (window mode)
  const uint32_t* sel;         // sel[0] = live batch size
  const uint32_t* nbr_index;   // hash-sorted row list (window mode) or nullptr
  uint32_t k_begin, k_end;     // tile numbers of this launch
  uint32_t rotation;           // global mode: tile k holds rows of tile (k + rotation) mod T
  int tiles_per_cta;
  int pruning;
};

// CTA = 256 threads = kTy x kTx; thread (ty, tx) owns the pairs {ty + kTy u} x {tx + kTx w},
// u < 8, w < kW.  Three shapes (candidates x neighbours per tile):
//   kTy 16, kW 4: 128 x 64   <= 128 registers, 98 KB: TWO CTAs share an SM and one computes
//                            while the other sits in a barrier, threshold refresh or refill
//                            (with one CTA per SM all warps leave the FMA pipe idle together);
//   kTy  8, kW 4:  64 x 128  same resources; for batches that have shrunk to <= 64 live
//                            candidates (the long-lived survivors that scan the whole series):
//                            half the padding rows of a 128-row candidate tile;
//   kTy 16, kW 8: 128 x 128  255 registers, one CTA per SM ("wide_tile", measured 7 % slower).
// Tile numbers k (ScanArgs) always count 128 neighbour rows; a shape with 64-row
// neighbour tiles walks the two halves of each.
// kLb compiles the lower-bound tile filter in; the plain variant carries none of its code.
template <bool kPacked, bool kSymmetric, int kTy, int kW, bool kLb>
__global__ void __launch_bounds__(kScanThreads, kW == 4 ? 2 : 1)
k_scan_tiles(SearchState s, ScanArgs a) {
  constexpr int kU = 8;
  constexpr int kTx = kScanThreads / kTy;
  constexpr int kCand = kTy * kU;                             // candidate rows per tile
  constexpr int kNbr = kTx * kW;                              // neighbour rows per tile
  constexpr int kSub = kTileRows / kNbr;                      // neighbour tiles per 128-row unit
  constexpr int kCandBytes = kCand * kRowBytes;
  constexpr int kStageBytes = (kCand + kNbr) * kRowBytes;
  static_assert(kCand <= kTileRows && kNbr <= kTileRows && kTileRows % kNbr == 0, "tile shape");
  // Candidate row (inside the tile) of pair-row u of thread row ty: 8 ty + u.  A warp holds
  // one ty (kTy = 8) or two (kTy = 16), so its candidates are CONTIGUOUS rows of the
  // word-sorted batch (16 w .. 16 w + 15 for warp w): a warp's candidates want, and abandon,
  // the same neighbour tiles.
  auto cand_of = [](uint32_t ty_, int u) -> uint32_t { return ty_ * kU + u; };
  extern __shared__ __align__(1024) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem + kStages * kStageBytes);  // candidate thresholds
  uint32_t* s_cand = reinterpret_cast<uint32_t*>(s_thr + kTileRows);      // candidate rows
  float* s_nub = reinterpret_cast<float*>(s_cand + kTileRows);            // neighbours' own bounds
  uint32_t* s_jrow = reinterpret_cast<uint32_t*>(s_nub + kTileRows);      // neighbour rows, ~0 = none
  uint32_t* s_brow = s_jrow + kTileRows;                                  // rows to load (none -> zero row)
  float* s_loc = reinterpret_cast<float*>(s_brow + kTileRows);            // bounds this CTA found itself
  uint32_t* s_map = reinterpret_cast<uint32_t*>(s_loc + kTileRows);       // kLb: the candidates taking part in a tile, packed
  __shared__ uint32_t s_wcount[kScanThreads / 32];
  __shared__ unsigned long long s_calls, s_abandoned, s_terms, s_tiles, s_tile_live, s_lb_skipped, s_useful;

  const uint32_t count = a.sel[0];
  const uint32_t cand0 = blockIdx.y * kCand;
  if (cand0 >= count) return;

  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t tx = tid % kTx, ty = tid / kTx;
  if (tid < kCand) s_cand[tid] = (cand0 + tid < count) ? a.batch_rows[cand0 + tid] : 0xFFFFFFFFu;
  if (tid == 0) {
    s_calls = 0;
    s_abandoned = 0;
    s_terms = 0;
    s_tiles = 0;
    s_tile_live = 0;
    s_lb_skipped = 0;
    s_useful = 0;
  }
  const bool window = a.nbr_index != nullptr;
  const uint32_t slot_tiles = (s.n_rows + kTileRows - 1) / kTileRows;
  const uint32_t centre = window ? a.batch_slots[min(cand0 + kCand / 2, count - 1)] / kTileRows : 0u;
  const uint64_t best = a.pruning ? *s.best : 0ull;
  const uint32_t chunks = s.stride / kChunk;
  const float* a_tile = a.batch + static_cast<size_t>(cand0) * s.stride;
  const float inf = __uint_as_float(kInfBits);

  // first slot of sub-tile h: unit h / kSub of the launch, half h % kSub of it
  auto slot0_of = [&](uint32_t h) -> uint32_t {
    const uint32_t k = h / kSub;
    uint32_t unit;
    if (!window) {
      unit = (k + a.rotation) % slot_tiles;
    } else {
      const uint32_t step = (k + 1) >> 1;  // 0, 1, 1, 2, 2, ...
      unit = (k & 1) ? (centre + step) % slot_tiles : (centre + slot_tiles - step % slot_tiles) % slot_tiles;
    }
    return unit * kTileRows + (h % kSub) * kNbr;
  };
  // The bounds a tile starts from are fetched one tile ahead (two dependent global
  // loads in window mode), so their latency hides behind the previous tile's
  // arithmetic.  A bound that is one tile stale is larger, never smaller: it
  // abandons less, and s_loc folds in what this CTA itself has found meanwhile.
  uint64_t pf_key = 0;
  uint32_t pf_j = 0xFFFFFFFFu;
  auto prefetch = [&](uint32_t h) {
    if (tid < kCand) {
      const uint32_t row = s_cand[tid];
      if (row != 0xFFFFFFFFu) TSDD_BOUND(row, s.n_rows);
      pf_key = (row != 0xFFFFFFFFu && a.pruning) ? load_key(s.nn + row) : 0ull;
    } else if (tid < kCand + kNbr) {
      const uint32_t slot = slot0_of(h) + (tid - kCand);
      pf_j = 0xFFFFFFFFu;
      if (slot < s.n_rows) pf_j = window ? a.nbr_index[slot] : slot;
      pf_key = pf_j != 0xFFFFFFFFu ? load_key(s.nn + pf_j) : 0ull;
    }
  };
  if (tid < kCand) s_loc[tid] = inf;
  __syncthreads();  // s_cand visible
  const uint32_t h_first = a.k_begin * kSub + blockIdx.x * a.tiles_per_cta, h_end = a.k_end * kSub;
  if (h_first < h_end) prefetch(h_first);

  for (int tt = 0; tt < a.tiles_per_cta; ++tt) {
    const uint32_t k = h_first + tt;  // sub-tile number
    if (k >= h_end) break;
    const uint32_t slot0 = slot0_of(k);
    __syncthreads();  // everyone is done with the previous tile's shared arrays

    // ---- thresholds and neighbour rows of this tile, from the prefetched registers
    bool live = false;
    if (tid < kCand) {
      const uint32_t row = s_cand[tid];
      float thr = -1.f;
      if (row != 0xFFFFFFFFu) {
        if (!a.pruning) {
          thr = inf;
          live = true;
        } else {
          const float bound = fminf(__uint_as_float(key_bits(pf_key)), s_loc[tid]);
          if (!dead_bound(bound, best, s.margin, s.margin_abs, s.margin_q)) {
            thr = bound;
            live = true;
          }
        }
      }
      s_thr[tid] = thr;
    } else if (tid < kCand + kNbr) {
      const uint32_t t = tid - kCand;
      s_jrow[t] = pf_j;
      s_brow[t] = pf_j != 0xFFFFFFFFu ? pf_j : s.n_rows;  // row n_rows is zero padding
      TSDD_BOUND(s_brow[t], s.n_rows + 1);
      s_nub[t] = pf_j != 0xFFFFFFFFu ? __uint_as_float(key_bits(pf_key)) : -1.f;
    }
    const int n_live = __syncthreads_count(live);
    if (n_live == 0) break;  // every candidate of this tile is dead: nothing left to do
    uint32_t n_mapped = 0;   // > 0: the tile's candidates are packed through s_map (kLb)
    // ---- lower-bound filter (covering scan only): a candidate whose segment means lie
    // further from every 16-row box of this tile than its threshold cannot find a
    // neighbour below it here; it sits this tile out (threshold -1 for this tile).
    if (kLb && !window && a.pruning && s.lb_means != nullptr) {
      bool needed = live;
      if (live && slot0 < s.n_rows) {
        const uint32_t row = s_cand[tid];
        const float limit = s_thr[tid];  // (lb_rules_out adds the rounding slack of the float32 means)
        float mine[kLbSegments];
        const float4* pm = reinterpret_cast<const float4*>(s.lb_means + static_cast<size_t>(row) * kLbSegments);
#pragma unroll
        for (int q = 0; q < kLbSegments / 4; ++q) {
          const float4 v = __ldg(pm + q);
          mine[4 * q] = v.x, mine[4 * q + 1] = v.y, mine[4 * q + 2] = v.z, mine[4 * q + 3] = v.w;
        }
        const uint32_t first_unit = slot0 / kLbBoxRows;
        const uint32_t last_unit = (min(slot0 + kNbr, s.n_rows) - 1) / kLbBoxRows;
        needed = false;
        for (uint32_t unit = first_unit; unit <= last_unit && !needed; ++unit) {
          const float4* pb = reinterpret_cast<const float4*>(s.lb_boxes + static_cast<size_t>(unit) * 2 * kLbSegments);
          float lb = 0.f;
#pragma unroll
          for (int q = 0; q < kLbSegments / 4; ++q) {
            const float4 lo = __ldg(pb + q), hi = __ldg(pb + kLbSegments / 4 + q);
            float g;
            g = fmaxf(fmaxf(lo.x - mine[4 * q], mine[4 * q] - hi.x), 0.f), lb = fmaf(g, g, lb);
            g = fmaxf(fmaxf(lo.y - mine[4 * q + 1], mine[4 * q + 1] - hi.y), 0.f), lb = fmaf(g, g, lb);
            g = fmaxf(fmaxf(lo.z - mine[4 * q + 2], mine[4 * q + 2] - hi.z), 0.f), lb = fmaf(g, g, lb);
            g = fmaxf(fmaxf(lo.w - mine[4 * q + 3], mine[4 * q + 3] - hi.w), 0.f), lb = fmaf(g, g, lb);
          }
          needed = !lb_rules_out(lb * s.lb_scale, limit, s.lb_q);
        }
        if (!needed) {
          s_thr[tid] = -1.f;
          live = false;
        }
      }
      // The candidates that take part are PACKED to the front of the tile (s_map: slot -> candidate),
      // so that they fill as few warps as possible: the filter leaves a started tile about one-sixth
      // full on strongly pruned inputs, and a warp computes for all of its 8 slots or for none.
      const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, needed && tid < kCand);
      if (lane == 0) s_wcount[tid >> 5] = __popc(ballot);
      const int n_needed = __syncthreads_count(needed);  // also publishes the lowered thresholds and the counts
      if (tid == 0) s_lb_skipped += static_cast<unsigned long long>(n_live - n_needed);
      if (n_needed == 0) {  // nobody needs this tile: no loads, no arithmetic
        if (tt + 1 < a.tiles_per_cta && k + 1 < h_end) prefetch(k + 1);
        continue;
      }
      if (needed && tid < kCand) {
        uint32_t at = __popc(ballot & ((1u << lane) - 1u));
        for (uint32_t w = 0; w < (tid >> 5); ++w) at += s_wcount[w];
        s_map[at] = tid;
      }
      n_mapped = static_cast<uint32_t>(n_needed);
      __syncthreads();  // s_map complete
    }
    if (tid == 0) {
      s_tiles += 1;
      s_tile_live += n_live;
    }
    if (tt + 1 < a.tiles_per_cta && k + 1 < h_end) prefetch(k + 1);

    unsigned long long my_calls = 0;
    if (live) {
      const uint32_t row = s_cand[tid];
      const uint32_t valid = slot0 < s.n_rows ? min(static_cast<uint32_t>(kNbr), s.n_rows - slot0) : 0u;
      uint32_t overlap = 0;
      if (!window) {
        // contiguous rows [slot0, slot0 + valid): the self-match zone is an interval
        const uint32_t z0 = row >= s.n - 1 ? row - (s.n - 1) : 0;
        const uint32_t z1 = row + s.n;  // exclusive
        const uint32_t o0 = max(slot0, z0), o1 = min(slot0 + valid, z1);
        overlap = o1 > o0 ? o1 - o0 : 0;
      } else {
        const uint4* jr = reinterpret_cast<const uint4*>(s_jrow);  // empty entries are ~0: far away
#pragma unroll 4
        for (int q = 0; q < kNbr / 4; ++q) {
          const uint4 v = jr[q];
          overlap += (gap_u32(row, v.x) < s.n ? 1u : 0u) + (gap_u32(row, v.y) < s.n ? 1u : 0u) +
                     (gap_u32(row, v.z) < s.n ? 1u : 0u) + (gap_u32(row, v.w) < s.n ? 1u : 0u);
        }
      }
      my_calls = valid - overlap;
    }

    // candidate (index inside the tile) of this thread's pair-row u: slot 8 ty + u, through the packing if there is one
    uint32_t cidx[kU];
    float thr[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t slot = cand_of(ty, u);
      cidx[u] = n_mapped ? (slot < n_mapped ? s_map[slot] : 0xFFFFFFFFu) : slot;
      thr[u] = cidx[u] != 0xFFFFFFFFu ? s_thr[cidx[u]] : -1.f;
    }
    const uint32_t* stage_map = n_mapped ? s_map : nullptr;

    Acc<kPacked, kU, kW> acc;
    acc.zero();

#pragma unroll
    for (int st = 0; st < kStages - 1; ++st) {
      if (static_cast<uint32_t>(st) < chunks)
        issue_stage<kCand, kNbr>(smem + st * kStageBytes, a_tile, s.rows, s_brow, s.stride, st * kChunk, stage_map, n_mapped);
      cp_async_commit();
    }

    // a thread none of whose candidates takes part in this tile (dead, or ruled out by the
    // lower bound) has abandoned before it starts; so has a warp of such threads
    bool mine_abandoned = true;
#pragma unroll
    for (int u = 0; u < kU; ++u) mine_abandoned = mine_abandoned && thr[u] < 0.f;
    bool warp_done = __all_sync(0xFFFFFFFFu, mine_abandoned), cta_abandoned = false;
    uint32_t warp_chunks = 0;
    for (uint32_t c = 0; c < chunks; ++c) {
      cp_async_wait<kStages - 2>();
      if (__syncthreads_and(mine_abandoned)) {
        cta_abandoned = true;
        break;
      }
      if (c + kStages - 1 < chunks)
        issue_stage<kCand, kNbr>(smem + ((c + kStages - 1) % kStages) * kStageBytes, a_tile, s.rows, s_brow,
                          s.stride, (c + kStages - 1) * kChunk, stage_map, n_mapped);
      cp_async_commit();
      if (!warp_done) {
        const unsigned char* a_s = smem + (c % kStages) * kStageBytes + cand_of(ty, 0) * kRowBytes;
        const unsigned char* b_s = smem + (c % kStages) * kStageBytes + kCandBytes + tx * kRowBytes;  // rows tx + kTx*w
#pragma unroll 2
        for (int kc = 0; kc < kPieces; ++kc) {
          const uint32_t off_a = (kc ^ (ty & 7)) << 4, off_b = (kc ^ (tx & 7)) << 4;
          if constexpr (kW == 8) {
            float4 na[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) na[u] = *reinterpret_cast<const float4*>(a_s + u * kRowBytes + off_a);
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              const float4 b = *reinterpret_cast<const float4*>(b_s + w * (kTx * kRowBytes) + off_b);
#pragma unroll
              for (int u = 0; u < kU; ++u) acc.add(u, w, na[u], b);
            }
          } else {
            // hold the neighbours, stream the candidates (a warp shares one candidate
            // row per u: its LDS.128 is a broadcast)
            float4 b[kW];
#pragma unroll
            for (int w = 0; w < kW; ++w) b[w] = *reinterpret_cast<const float4*>(b_s + w * (kTx * kRowBytes) + off_b);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const float4 na = *reinterpret_cast<const float4*>(a_s + u * kRowBytes + off_a);
#pragma unroll
              for (int w = 0; w < kW; ++w) acc.add(u, w, na, b[w]);
            }
          }
        }
        ++warp_chunks;
        bool all_over = true;
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int w = 0; w < kW; ++w) all_over = all_over && (acc.get(u, w) > thr[u]);
        mine_abandoned = all_over;
        warp_done = __all_sync(0xFFFFFFFFu, all_over);
      }
    }
    cp_async_wait<0>();

    // ---- accounting (per warp: the terms its lanes really accumulated, and how many of them
    // belonged to a live candidate, an existing neighbour row and a real column)
    {
      uint32_t taking_part = 0;
#pragma unroll
      for (int u = 0; u < kU; ++u) taking_part += thr[u] >= 0.f ? 1u : 0u;
      // a warp holds 32 / kTx thread rows; lane 0 of each carries that row's count
      uint32_t warp_live = __shfl_sync(0xFFFFFFFFu, taking_part, 0);
      if (kTx < 32) warp_live += __shfl_sync(0xFFFFFFFFu, taking_part, kTx % 32);
      if (lane == 0 && warp_chunks) {
        const uint32_t rows_here = slot0 < s.n_rows ? min(static_cast<uint32_t>(kNbr), s.n_rows - slot0) : 0u;
        atomicAdd(&s_terms, static_cast<unsigned long long>(warp_chunks) * kChunk * 32 * kU * kW);
        atomicAdd(&s_useful, static_cast<unsigned long long>(min(warp_chunks * kChunk, s.n)) * warp_live * rows_here);
      }
    }
    if (my_calls) {
      atomicAdd(&s_calls, my_calls);
      if (cta_abandoned) atomicAdd(&s_abandoned, my_calls);
    }
    if (cta_abandoned) continue;
    // ---- completed tile: lower the candidates' bounds (and, symmetric, the neighbours')
    // Fast test first: in a pruned scan almost no pair of a tile ends below its
    // candidate's (or its neighbour's) bound, and then nothing else is looked at.
    const bool complete = (warp_chunks == chunks);
    float nub[kW];
#pragma unroll
    for (int w = 0; w < kW; ++w) nub[w] = (kSymmetric && complete) ? s_nub[tx + kTx * w] : -1.f;
    bool hit = false;
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        const float d = acc.get(u, w);
        hit = hit || d <= thr[u] || d < nub[w];
      }
    if (!__any_sync(0xFFFFFFFFu, hit)) continue;

    uint32_t jrow[kW];
#pragma unroll
    for (int w = 0; w < kW; ++w) jrow[w] = s_jrow[tx + kTx * w];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t row = cidx[u] != 0xFFFFFFFFu ? s_cand[cidx[u]] : 0xFFFFFFFFu;
      uint32_t d_min = 0xFFFFFFFFu, j_min = 0xFFFFFFFFu;  // this thread's best (distance bits, neighbour)
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        const uint32_t j = jrow[w];
        const float d = acc.get(u, w);
        const bool pair_ok = row != 0xFFFFFFFFu && j != 0xFFFFFFFFu && gap_u32(row, j) >= s.n;
        if (pair_ok && d <= thr[u]) {
          const uint32_t bits = __float_as_uint(d);
          if (bits < d_min || (bits == d_min && j < j_min)) {
            d_min = bits;
            j_min = j;
          }
        }
        if (pair_ok && d < nub[w]) {
          TSDD_BOUND(j, s.n_rows);
          atomicMin(as_ull(s.nn + j), static_cast<unsigned long long>(nn_key(__float_as_uint(d), row)));
        }
      }
      // min over the kTx lanes that share candidate u: distance first, then neighbour
      uint32_t g_min = d_min;
#pragma unroll
      for (int d = kTx / 2; d > 0; d >>= 1) g_min = min(g_min, __shfl_xor_sync(0xFFFFFFFFu, g_min, d));
      uint32_t g_j = d_min == g_min ? j_min : 0xFFFFFFFFu;
#pragma unroll
      for (int d = kTx / 2; d > 0; d >>= 1) g_j = min(g_j, __shfl_xor_sync(0xFFFFFFFFu, g_j, d));
      if (tx == 0 && g_j != 0xFFFFFFFFu) {
        TSDD_BOUND(row, s.n_rows);
        atomicMin(as_ull(s.nn + row), static_cast<unsigned long long>(nn_key(g_min, g_j)));
        s_loc[cidx[u]] = fminf(s_loc[cidx[u]], __uint_as_float(g_min));
      }
    }
  }

  __syncthreads();
  if (tid == 0) {
    if (s_calls) atomicAdd(&s.counters->calls, s_calls);
    if (s_abandoned) atomicAdd(&s.counters->abandoned, s_abandoned);
    if (s_terms) {
      atomicAdd(&s.counters->terms, s_terms);
      atomicAdd(&s.counters->tile_terms, s_terms);
      atomicAdd(&s.counters->useful_terms, s_useful);
    }
    if (s_tiles) {
      atomicAdd(&s.counters->tiles, s_tiles);
      atomicAdd(&s.counters->tile_live, s_tile_live);
    }
    if (s_lb_skipped) atomicAdd(&s.counters->lb_skipped, s_lb_skipped);
  }
}

// ------------------------------------------------------------------ warp-specialised tile kernel
//
// Same arithmetic as k_scan_tiles on a 128 x 128 tile (8 x 8 pairs per thread), different
// plumbing.  CTA = two consumer warpgroups (8 warps, the 16 x 16 thread grid) + one producer
// warpgroup (one active warp); one CTA per SM, launched at 168 registers per thread and
// rebalanced with setmaxnreg: 232 per consumer thread, 40 per producer thread
// (256 x 232 + 128 x 40 = 64,512 = 384 x 168).  The producer streams 64-column stages — one
// 256-byte cp.async.bulk per row (UBLKCP), completing on an mbarrier — through a 3-stage
// ring that runs ACROSS tile boundaries, so the first stages of the next tile land while the
// consumers are still in the last chunk and epilogue of the current one.  It also prepares
// each tile's thresholds / neighbour rows one tile ahead (two metadata slots).  Consumers
// never meet in a CTA-wide barrier: each warp waits for a stage (full mbarrier), reads the
// stage's tag (tile, chunk), computes, and releases the stage (empty mbarrier).  A tile is
// abandoned when all 8 warps have voted (shared counter); the producer then stops feeding
// it and moves on.  Rows sit in shared memory at a 272-byte pitch (256 + 16), which makes
// the LDS.128 of the 8 rows of a quarter-warp conflict-free without a swizzle.
//
// No lower-bound filter here: the producer shares a scheduler with two consumer warps, and
// every instruction it issues is taken from them and, through the stage barriers, from every
// warp (a producer that also ran the filter cost 9 % on cfg 5).  The launcher therefore uses
// this kernel where the filter has nothing to offer — window rounds, and covering scans of
// searches on which it has been switched off — and k_scan_tiles elsewhere.
namespace ws {

#ifndef TSDD_WS_LANES48
#define TSDD_WS_LANES48 1
#endif

constexpr int kStagesWs = 3;
constexpr int kNbrWs = 128;
constexpr int kPitch = kChunk * 4 + 16;
constexpr int kRowsPerStage = kTileRows + kNbrWs;
constexpr int kStageBytesWs = kRowsPerStage * kPitch;
constexpr int kConsumerWarps = 8;
constexpr int kThreadsWs = (kConsumerWarps + 4) * 32;  // + one producer warpgroup
constexpr uint32_t kTagDone = 0xFFFFFFFFu;

struct alignas(16) TileMeta {  // (jrow is read as uint4)
  float thr[kTileRows];      // candidate thresholds, -1 = dead / none
  float nub[kNbrWs];         // neighbours' own bounds, -1 = none
  uint32_t jrow[kNbrWs];     // neighbour rows, ~0 = none
  uint32_t brow[kNbrWs];     // rows to load (none -> the zero row)
  float nnorm[kNbrWs];       // dot form: squared norms of the neighbour rows
  unsigned long long calls;  // pair distances this tile starts
  uint32_t done;             // consumer warps that have abandoned the tile
  uint32_t valid;            // neighbour slots of the tile that hold a row (the first `valid` of them)
};

// Tensor-map variant: a stage is four TMA boxes of 128 rows x 32 columns (128 bytes a row,
// 128-byte swizzle): candidates columns 0-31, 32-63, then neighbours likewise.
constexpr int kBoxCols = 32;
constexpr int kBoxBytes = kTileRows * kBoxCols * 4;
constexpr int kStageBytesTma = 4 * kBoxBytes;
static_assert(kChunk == 2 * kBoxCols, "a chunk is two boxes wide");

// What the four warps of the producer warpgroup need for the lower-bound tile filter (kLb).
struct LbPart {
  uint32_t live, needed;     // this warp's candidates: alive / taking part in the tile
  unsigned long long calls;  // pair distances they start in it
};
template <bool kLb>
struct LbShared {};
template <>
struct LbShared<true> {
  float cmeans[kLbSegments][kTileRows];  // segment means of the CTA's candidates, transposed (conflict-free per lane)
  float4 boxes[4][kTileRows / kLbBoxRows * 2 * kLbSegments / 4];  // per warp: the neighbour tile's 8 boxes
  LbPart part[2][4];                     // per tile parity, per warp
};

template <bool kTma, bool kLb = false>
struct SharedWsT {
  unsigned char stages[kStagesWs][kTma ? kStageBytesTma : kStageBytesWs];
  LbShared<kLb> lb;
  TileMeta meta[2];
  uint32_t cand[kTileRows];
  float loc[kTileRows];
  float cnorm[kTileRows];  // dot form: squared norms of the candidate rows
  uint32_t tag_tile[kStagesWs + 1];
  uint32_t tag_chunk[kStagesWs + 1];
  unsigned long long full[kStagesWs], empty[kStagesWs], meta_full[2], meta_empty[2];  // mbarriers
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @p bra DONE_%=;\n"
      " bra WAIT_%=;\n DONE_%=:\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_box(void* smem_dst, const CUtensorMap* map, uint32_t col, uint32_t row,
                                             unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_addr(smem_dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(col), "r"(row), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_copy_row(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                              unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// kDot: the distance as |a|^2 + |b|^2 - 2 a.b — ONE FFMA per term instead of FADD + FFMA, at
// the price of (1) an absolute rounding error (n + 32) n 2^-24 instead of a relative one, which
// the discard band absorbs (SearchState::margin_abs) and the float64 decision settles, and
// (2) no early abandoning inside a tile (partial dot products are not monotone).  The engine
// picks it for searches whose tiles are not being abandoned anyway (noise-like data) once
// the best-so-far dwarfs the error bound.
//
// kTma (covering scans: the neighbour rows of a tile are consecutive matrix rows): a stage is
// filled by FOUR cp.async.bulk.tensor instructions (two 128 x 32 boxes of the candidate tile,
// two of the neighbour tile, hardware-swizzled) instead of 256 row copies.  The producer warp
// shares a scheduler with two consumer warps, and the per-row copies (one elect / R2UR /
// UBLKCP round per row: ~2,500 instructions per chunk) held that scheduler's consumers back.
// Window launches gather scattered rows and keep the per-row copies.
//
// kLb (covering scans of the direct form, tensor-map loads): the lower-bound tile filter of
// k_scan_tiles, run by ALL FOUR warps of the producer warpgroup — 32 candidates each, one per
// lane — now that tensor maps have left them idle.  Per neighbour tile a lane tests its
// candidate's 16 segment means against the tile's 8 boxes; a candidate the boxes rule out
// gets threshold -1 for this tile, a tile nobody needs is never streamed (the consumers do
// not even hear of it: tiles are announced under a running number), and the consumers, who
// meet no CTA-wide barrier, never wait for a warp that has nothing to do.  The four warps
// meet once per tile in a named barrier (bar.sync 1, 128) to add up their counts.
template <bool kSymmetric, bool kDot, bool kTma, bool kLb = false>
__global__ void __launch_bounds__(kThreadsWs, 1)
k_scan_tiles_ws(SearchState s, ScanArgs a, const __grid_constant__ CUtensorMap map_a,
                const __grid_constant__ CUtensorMap map_b) {
  static_assert(!kLb || (kTma && !kDot), "the filter variant is the direct form fed by tensor maps");
  constexpr int kU = 8, kW = 8, kTx = 16;
  using SharedWs = SharedWsT<kTma, kLb>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  SharedWs& sh = *reinterpret_cast<SharedWs*>(smem_raw);

  const uint32_t count = a.sel[0];
  const uint32_t cand0 = blockIdx.y * kTileRows;
  if (cand0 >= count) return;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float inf = __uint_as_float(kInfBits);
  if (tid < kTileRows) {
    const uint32_t row = (cand0 + tid < count) ? a.batch_rows[cand0 + tid] : 0xFFFFFFFFu;
    sh.cand[tid] = row;
    sh.loc[tid] = inf;
    if constexpr (kDot) sh.cnorm[tid] = row != 0xFFFFFFFFu ? s.row_norms[row] : 0.f;
    if constexpr (kLb) {
      const float4* pm = reinterpret_cast<const float4*>(s.lb_means + static_cast<size_t>(row) * kLbSegments);
#pragma unroll
      for (int q = 0; q < kLbSegments / 4; ++q) {
        const float4 v = row != 0xFFFFFFFFu ? __ldg(pm + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        sh.lb.cmeans[4 * q][tid] = v.x, sh.lb.cmeans[4 * q + 1][tid] = v.y;
        sh.lb.cmeans[4 * q + 2][tid] = v.z, sh.lb.cmeans[4 * q + 3][tid] = v.w;
      }
    }
  }
  if (tid == 0) {
    for (int i = 0; i < kStagesWs; ++i) {
      mbar_init(&sh.full[i], 1);
      mbar_init(&sh.empty[i], kConsumerWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sh.meta_full[i], 1);
      mbar_init(&sh.meta_empty[i], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // the only CTA-wide barrier

  const bool window = a.nbr_index != nullptr;
  constexpr uint32_t kSub = kTileRows / kNbrWs;  // ScanArgs counts 128-row units; this kernel walks their halves
  const uint32_t slot_tiles = (s.n_rows + kTileRows - 1) / kTileRows;
  const uint32_t chunks = s.stride / kChunk;
  const uint32_t k_first = a.k_begin * kSub + blockIdx.x * a.tiles_per_cta, k_end = a.k_end * kSub;
  const uint32_t n_tiles = k_first < k_end ? min(static_cast<uint32_t>(a.tiles_per_cta), k_end - k_first) : 0u;

  if (warp >= kConsumerWarps) {
    // ================================================================ producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if constexpr (kLb) {
      // ============================================================ producer warpgroup, with the filter
      const uint32_t pw = warp - kConsumerWarps;      // 0..3
      const uint32_t c = 32 * pw + lane;              // this lane's candidate
      const uint32_t row = sh.cand[c];
      const uint64_t best = *s.best;
      const uint32_t units_total = (s.n_rows + kLbBoxRows - 1) / kLbBoxRows;
      constexpr uint32_t kUnits = kTileRows / kLbBoxRows;          // 8 boxes per neighbour tile
      constexpr uint32_t kBoxQuads = 2 * kLbSegments / 4;          // float4 per box
      float4* my_boxes = sh.lb.boxes[pw];
      uint32_t seq = 0, sti = 0;  // stages issued; tiles announced to the consumers
      unsigned long long calls_total = 0, tiles_total = 0, live_total = 0, skipped_total = 0;
#pragma unroll 1
      for (uint32_t ti = 0; ti < n_tiles; ++ti) {
        const uint32_t k = k_first + ti, m = sti & 1, use = sti >> 1;
        TileMeta& meta = sh.meta[m];
        if (use >= 1) mbar_wait(&sh.meta_empty[m], (use - 1) & 1);  // every consumer has left announced tile sti - 2
        const uint32_t slot0 = ((k + a.rotation) % slot_tiles) * kTileRows;
        const uint32_t unit0 = slot0 / kLbBoxRows;
        // ---- loads first: the candidate's bound, the tile's boxes (this warp's own copy), the neighbours' bounds
        const uint32_t cand_ub = row != 0xFFFFFFFFu ? key_bits(load_key(s.nn + row)) : 0u;
        {
          const float4* src = reinterpret_cast<const float4*>(s.lb_boxes + static_cast<size_t>(unit0) * 2 * kLbSegments);
#pragma unroll
          for (int q = 0; q < static_cast<int>(kUnits * kBoxQuads) / 32; ++q) {
            const uint32_t at = lane + 32 * q;  // float4 index inside the tile's boxes; box = at / kBoxQuads
            my_boxes[at] = unit0 + at / kBoxQuads < units_total ? __ldg(src + at) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        uint32_t nbr_j = 0xFFFFFFFFu, nbr_ub = 0u;
        {
          const uint32_t slot = slot0 + c;  // the four warps share the 128 neighbours as well
          if (slot < s.n_rows) {
            nbr_j = slot;
            nbr_ub = key_bits(load_key(s.nn + slot));
          }
        }
        __syncwarp();
        // ---- this candidate: dead, ruled out by the boxes, or taking part
        float thr = -1.f;
        bool live = false, needed = false;
        if (row != 0xFFFFFFFFu) {
          const float bound = fminf(__uint_as_float(cand_ub), sh.loc[c]);
          live = !dead_bound(bound, best, s.margin, s.margin_abs, s.margin_q);
          if (live) {
            const float limit = bound;  // (lb_rules_out adds the rounding slack of the float32 means)
            const uint32_t n_units = min(kUnits, units_total - unit0);
            float lb[kUnits];
#pragma unroll
            for (int u = 0; u < static_cast<int>(kUnits); ++u) lb[u] = 0.f;
#pragma unroll
            for (int q = 0; q < kLbSegments / 4; ++q) {
              const float m0 = sh.lb.cmeans[4 * q][c], m1 = sh.lb.cmeans[4 * q + 1][c];
              const float m2 = sh.lb.cmeans[4 * q + 2][c], m3 = sh.lb.cmeans[4 * q + 3][c];
#pragma unroll
              for (int u = 0; u < static_cast<int>(kUnits); ++u) {
                const float4 lo = my_boxes[u * kBoxQuads + q], hi = my_boxes[u * kBoxQuads + kLbSegments / 4 + q];
                float g;
                g = fmaxf(fmaxf(lo.x - m0, m0 - hi.x), 0.f), lb[u] = fmaf(g, g, lb[u]);
                g = fmaxf(fmaxf(lo.y - m1, m1 - hi.y), 0.f), lb[u] = fmaf(g, g, lb[u]);
                g = fmaxf(fmaxf(lo.z - m2, m2 - hi.z), 0.f), lb[u] = fmaf(g, g, lb[u]);
                g = fmaxf(fmaxf(lo.w - m3, m3 - hi.w), 0.f), lb[u] = fmaf(g, g, lb[u]);
              }
            }
            float lb_min = __uint_as_float(kInfBits);
#pragma unroll
            for (int u = 0; u < static_cast<int>(kUnits); ++u)
              if (static_cast<uint32_t>(u) < n_units) lb_min = fminf(lb_min, lb[u]);
            needed = !lb_rules_out(lb_min * s.lb_scale, limit, s.lb_q);
            if (needed) thr = bound;
          }
        }
        meta.thr[c] = thr;
        meta.jrow[c] = nbr_j;
        meta.nub[c] = nbr_j != 0xFFFFFFFFu ? __uint_as_float(nbr_ub) : -1.f;
        // pair distances this candidate starts in the tile (series.hpp:120): neighbours at least n away
        const uint32_t valid = slot0 < s.n_rows ? min(static_cast<uint32_t>(kNbrWs), s.n_rows - slot0) : 0u;
        unsigned long long calls = 0;
        if (needed) {
          const uint32_t z0 = row >= s.n - 1 ? row - (s.n - 1) : 0, z1 = row + s.n;
          const uint32_t o0 = max(slot0, z0), o1 = min(slot0 + valid, z1);
          calls = valid - (o1 > o0 ? o1 - o0 : 0);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) calls += __shfl_xor_sync(0xFFFFFFFFu, calls, d);
        const uint32_t n_live = __popc(__ballot_sync(0xFFFFFFFFu, live));
        const uint32_t n_needed = __popc(__ballot_sync(0xFFFFFFFFu, needed));
        LbPart* part = sh.lb.part[ti & 1];
        if (lane == 0) part[pw] = LbPart{n_live, n_needed, calls};
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the four warps; also publishes thr / jrow / nub
        uint32_t all_live = 0, all_needed = 0;
        unsigned long long all_calls = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          all_live += part[w].live;
          all_needed += part[w].needed;
          all_calls += part[w].calls;
        }
        if (all_live == 0) break;  // candidates only ever die: nothing is left for this CTA
        skipped_total += all_live - all_needed;
        if (all_needed == 0) continue;  // nobody needs this tile: not streamed, not announced
        live_total += all_live;
        calls_total += all_calls;
        tiles_total += 1;
        if (pw == 0) {
          if (lane == 0) {
            meta.calls = all_calls;
            meta.done = 0;
            meta.valid = valid;
            mbar_arrive(&sh.meta_full[m]);
          }
          // ---- stream the tile's chunks; stop as soon as every consumer warp has abandoned it
#pragma unroll 1
          for (uint32_t ch = 0; ch < chunks; ++ch) {
            if (*reinterpret_cast<volatile uint32_t*>(&meta.done) == kConsumerWarps) break;
            const uint32_t st = seq % kStagesWs, round = seq / kStagesWs;
            if (round >= 1) mbar_wait(&sh.empty[st], (round - 1) & 1);
            if (lane == 0) {
              sh.tag_tile[st] = sti;
              sh.tag_chunk[st] = ch;
              mbar_arrive_expect_tx(&sh.full[st], kRowsPerStage * kChunk * 4);
              unsigned char* dst = sh.stages[st];
              const uint32_t col = ch * kChunk;
              tma_load_box(dst, &map_a, col, cand0, &sh.full[st]);
              tma_load_box(dst + kBoxBytes, &map_a, col + kBoxCols, cand0, &sh.full[st]);
              tma_load_box(dst + 2 * kBoxBytes, &map_b, col, slot0, &sh.full[st]);
              tma_load_box(dst + 3 * kBoxBytes, &map_b, col + kBoxCols, slot0, &sh.full[st]);
            }
            ++seq;
          }
        }
        ++sti;
      }
      if (pw == 0) {
        {  // the end-of-work tag
          const uint32_t st = seq % kStagesWs, round = seq / kStagesWs;
          if (round >= 1) mbar_wait(&sh.empty[st], (round - 1) & 1);
          if (lane == 0) {
            sh.tag_tile[st] = kTagDone;
            mbar_arrive(&sh.full[st]);
          }
        }
        if (lane == 0) {
          if (calls_total) atomicAdd(&s.counters->calls, calls_total);
          if (tiles_total) atomicAdd(&s.counters->tiles, tiles_total);
          if (live_total) atomicAdd(&s.counters->tile_live, live_total);
          if (skipped_total) atomicAdd(&s.counters->lb_skipped, skipped_total);
        }
      }
      return;
    }
    if (warp != kConsumerWarps) return;  // one warp does the work; the other three only round the CTA to 12 warps
    const uint32_t centre = window ? a.batch_slots[min(cand0 + kTileRows / 2, count - 1)] / kTileRows : 0u;
    const uint64_t best = a.pruning ? *s.best : 0ull;
    const float* a_tile = a.batch + static_cast<size_t>(cand0) * s.stride;
    auto slot0_of = [&](uint32_t h) -> uint32_t {
      const uint32_t k = h / kSub;
      uint32_t unit;
      if (!window) {
        unit = (k + a.rotation) % slot_tiles;
      } else {
        const uint32_t step = (k + 1) >> 1;
        unit = (k & 1) ? (centre + step) % slot_tiles : (centre + slot_tiles - step % slot_tiles) % slot_tiles;
      }
      return unit * kTileRows + (h % kSub) * kNbrWs;
    };
    // bounds of the next tile, fetched while the current one streams
    uint32_t cand_ub[4], nbr_ub[4];  // float bits of the nn upper bounds
    uint32_t nbr_j[4];
    float nbr_norm[kDot ? 4 : 1];
    auto fetch_bounds = [&](uint32_t k) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t row = sh.cand[lane + 32 * q];
        cand_ub[q] = (row != 0xFFFFFFFFu && a.pruning) ? key_bits(load_key(s.nn + row)) : 0u;
      }
      const uint32_t slot0 = slot0_of(k);
#pragma unroll
      for (int q = 0; q < kNbrWs / 32; ++q) {
        const uint32_t slot = slot0 + lane + 32 * q;
        nbr_j[q] = 0xFFFFFFFFu;
        if (slot < s.n_rows) nbr_j[q] = window ? a.nbr_index[slot] : slot;
        if (nbr_j[q] != 0xFFFFFFFFu) TSDD_BOUND(nbr_j[q], s.n_rows);
        nbr_ub[q] = nbr_j[q] != 0xFFFFFFFFu ? key_bits(load_key(s.nn + nbr_j[q])) : 0u;
        if constexpr (kDot) nbr_norm[q] = nbr_j[q] != 0xFFFFFFFFu ? s.row_norms[nbr_j[q]] : 0.f;
      }
    };
    if (n_tiles) fetch_bounds(k_first);

    // The producer shares a scheduler with two consumer warps; it is kept lean (row pointers of
    // the tile in registers, nothing recomputed per stage).
    uint32_t seq = 0;
    unsigned long long calls_total = 0, tiles_total = 0, live_total = 0;
#pragma unroll 1
    for (uint32_t ti = 0; ti < n_tiles; ++ti) {
      const uint32_t k = k_first + ti, m = ti & 1, use = ti >> 1;
      TileMeta& meta = sh.meta[m];
      if (use >= 1) mbar_wait(&sh.meta_empty[m], (use - 1) & 1);  // every consumer has left tile ti - 2

      // ---- metadata of tile ti from the prefetched bounds
      bool live[4];
      bool any_live = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t r = lane + 32 * q, row = sh.cand[r];
        float thr = -1.f;
        live[q] = false;
        if (row != 0xFFFFFFFFu) {
          if (!a.pruning) {
            thr = inf;
            live[q] = true;
          } else {
            const float bound = fminf(__uint_as_float(cand_ub[q]), sh.loc[r]);
            if (!dead_bound(bound, best, s.margin, s.margin_abs, s.margin_q)) {
              thr = bound;
              live[q] = true;
            }
          }
        }
        meta.thr[r] = thr;
        any_live = any_live || live[q];
        live_total += live[q] ? 1u : 0u;
      }
#pragma unroll
      for (int q = 0; q < kNbrWs / 32; ++q) {
        const uint32_t e = lane + 32 * q, j = nbr_j[q];
        meta.jrow[e] = j;
        meta.brow[e] = j != 0xFFFFFFFFu ? j : s.n_rows;  // row n_rows is zero padding
        TSDD_BOUND(meta.brow[e], s.n_rows + 1);
        meta.nub[e] = j != 0xFFFFFFFFu ? __uint_as_float(nbr_ub[q]) : -1.f;
        if constexpr (kDot) meta.nnorm[e] = nbr_norm[q];
      }
      any_live = __any_sync(0xFFFFFFFFu, any_live);
      __syncwarp();
      // pair distances this tile starts (series.hpp:120): live candidates x neighbours at least n away
      const uint32_t slot0 = slot0_of(k);
      const uint32_t valid = slot0 < s.n_rows ? min(static_cast<uint32_t>(kNbrWs), s.n_rows - slot0) : 0u;
      unsigned long long calls = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!live[q]) continue;
        const uint32_t row = sh.cand[lane + 32 * q];
        uint32_t overlap = 0;
        if (!window) {
          const uint32_t z0 = row >= s.n - 1 ? row - (s.n - 1) : 0, z1 = row + s.n;
          const uint32_t o0 = max(slot0, z0), o1 = min(slot0 + valid, z1);
          overlap = o1 > o0 ? o1 - o0 : 0;
        } else if constexpr (kTma && kDot) {
          // the consumers count the self-match pairs of a window tile in their epilogue (the dot
          // form completes every tile it starts) and take them off the counter at the end
        } else {
          const uint4* jr = reinterpret_cast<const uint4*>(meta.jrow);
#pragma unroll 4
          for (int e = 0; e < kNbrWs / 4; ++e) {
            const uint4 v = jr[e];
            overlap += (gap_u32(row, v.x) < s.n ? 1u : 0u) + (gap_u32(row, v.y) < s.n ? 1u : 0u) +
                       (gap_u32(row, v.z) < s.n ? 1u : 0u) + (gap_u32(row, v.w) < s.n ? 1u : 0u);
          }
        }
        calls += valid - overlap;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) calls += __shfl_xor_sync(0xFFFFFFFFu, calls, d);
      if (lane == 0) {
        meta.calls = calls;
        meta.done = 0;
        meta.valid = valid;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.meta_full[m]);
      if (!any_live) break;  // candidates only ever die: nothing is left for this CTA
      calls_total += calls;
      tiles_total += 1;

      const float* src[kTma ? 1 : kRowsPerStage / 32];
      if constexpr (!kTma) {
#pragma unroll
        for (int q = 0; q < 4; ++q) src[q] = a_tile + static_cast<size_t>(lane + 32 * q) * s.stride;
#pragma unroll
        for (int q = 0; q < kNbrWs / 32; ++q)
          src[4 + q] = s.rows + static_cast<size_t>(meta.brow[lane + 32 * q]) * s.stride;
      }
      if (ti + 1 < n_tiles) fetch_bounds(k + 1);

      // ---- stream the tile's chunks; stop as soon as every consumer warp has abandoned it
#pragma unroll 1
      for (uint32_t c = 0; c < chunks; ++c) {
        if (a.pruning && *reinterpret_cast<volatile uint32_t*>(&meta.done) == kConsumerWarps) break;
        const uint32_t st = seq % kStagesWs, round = seq / kStagesWs;
        if (round >= 1) mbar_wait(&sh.empty[st], (round - 1) & 1);
        if (lane == 0) {
          sh.tag_tile[st] = ti;
          sh.tag_chunk[st] = c;
          mbar_arrive_expect_tx(&sh.full[st], kRowsPerStage * kChunk * 4);
        }
        unsigned char* dst = sh.stages[st];
        if constexpr (kTma) {
          if (lane == 0) {
            const uint32_t col = c * kChunk;
            tma_load_box(dst, &map_a, col, cand0, &sh.full[st]);
            tma_load_box(dst + kBoxBytes, &map_a, col + kBoxCols, cand0, &sh.full[st]);
            tma_load_box(dst + 2 * kBoxBytes, &map_b, col, slot0, &sh.full[st]);
            tma_load_box(dst + 3 * kBoxBytes, &map_b, col + kBoxCols, slot0, &sh.full[st]);
          }
        } else {
          __syncwarp();
#pragma unroll
          for (int q = 0; q < kRowsPerStage / 32; ++q)
            bulk_copy_row(dst + (lane + 32 * q) * kPitch, src[q] + c * kChunk, kChunk * 4, &sh.full[st]);
        }
        ++seq;
      }
    }
    {  // the end-of-work tag
      const uint32_t st = seq % kStagesWs, round = seq / kStagesWs;
      if (round >= 1) mbar_wait(&sh.empty[st], (round - 1) & 1);
      if (lane == 0) {
        sh.tag_tile[st] = kTagDone;
        mbar_arrive(&sh.full[st]);
      }
    }
    if (lane == 0) {
      if (calls_total) atomicAdd(&s.counters->calls, calls_total);
      if (tiles_total) atomicAdd(&s.counters->tiles, tiles_total);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) live_total += __shfl_xor_sync(0xFFFFFFFFu, live_total, d);
    if (lane == 0 && live_total) atomicAdd(&s.counters->tile_live, live_total);
    return;
  }

  // ================================================================== consumer warpgroups
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
#if TSDD_WS_LANES48
  // A warp is 4 thread rows x 8 thread columns: the 16 lanes of a half-warp then read only 8
  // distinct neighbour rows (128 bytes, one shared-memory wavefront) per LDS.128 instead of 16.
  const uint32_t tx = (lane & 7u) | ((warp & 1u) << 3), ty = (lane >> 3) | ((warp >> 1) << 2);
  constexpr int kTxLanes = 8;  // thread columns inside one warp
#else
  const uint32_t tx = tid % kTx, ty = tid / kTx;
  constexpr int kTxLanes = kTx;
#endif
  // Candidate row of pair-row u of thread row ty: warp w (thread rows 2w, 2w + 1) owns the 16
  // CONTIGUOUS rows 16w .. 16w + 15 of the word-sorted batch (they want, and abandon, the same
  // tiles); the two rows a warp reads at once are adjacent, i.e. in different bank groups at
  // the 272-byte pitch.
  const uint32_t cand0_of_thread = (ty >> 1) * 16 + (ty & 1);  // + 2 u
  constexpr uint32_t kCandStep = 2;
  // per-thread constants of the shared-memory addressing, pinned in registers (opaque to the
  // optimiser, which otherwise rematerialises them from the thread id inside the hot loop)
  uint32_t xa = (ty & 7u) << 4, xb = (tx & 7u) << 4;  // kTma: the 128-byte swizzle terms
  uint32_t a_row_off = kTma ? ((ty & 7u) + 64u * (ty >> 3)) * 128u : cand0_of_thread * kPitch;
  uint32_t b_row_off = kTma ? 2 * kBoxBytes + tx * 128u : kTileRows * kPitch + tx * kPitch;
  // (an identity shuffle: ptxas cannot see through it, an empty asm it can)
  xa = __shfl_sync(0xFFFFFFFFu, xa, lane), xb = __shfl_sync(0xFFFFFFFFu, xb, lane);
  a_row_off = __shfl_sync(0xFFFFFFFFu, a_row_off, lane), b_row_off = __shfl_sync(0xFFFFFFFFu, b_row_off, lane);
  Acc<true, kU, kW> acc;
  float thr[kU];
  uint32_t seq = 0, cur = kTagDone, m = 0, chunks_done = 0;
  bool released = true, warp_done = false;
  unsigned long long chunks_total = 0, abandoned_total = 0;
  uint32_t overlap_total = 0, pairs_w = 0, useful_units = 0;
#pragma unroll 1
  for (;;) {
    const uint32_t st = seq % kStagesWs, round = seq / kStagesWs;
    mbar_wait(&sh.full[st], round & 1);
    const uint32_t tile = *reinterpret_cast<volatile uint32_t*>(&sh.tag_tile[st]);
    if (tile == kTagDone) break;
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(&sh.tag_chunk[st]);
    if (tile != cur) {
      if (!released) {  // the previous tile was cut short by the producer
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.meta_empty[m]);
      }
      cur = tile;
      m = tile & 1;
      mbar_wait(&sh.meta_full[m], (tile >> 1) & 1);
#pragma unroll
      for (int u = 0; u < kU; ++u) thr[u] = sh.meta[m].thr[cand0_of_thread + kCandStep * u];
      acc.zero();
      bool none = true;
#pragma unroll
      for (int u = 0; u < kU; ++u) none = none && thr[u] < 0.f;
      warp_done = __all_sync(0xFFFFFFFFu, none);  // none of this warp's candidates takes part in the tile
      if (warp_done && lane == 0 && chunks > 1) {
        if (atomicAdd(&sh.meta[m].done, 1u) == kConsumerWarps - 1) abandoned_total += sh.meta[m].calls;
      }
      {  // (live candidates) x (existing neighbour rows) among this warp's pairs: the useful share of its terms
        uint32_t cc = 0, cn = 0;
        const uint32_t valid = sh.meta[m].valid;
#pragma unroll
        for (int u = 0; u < kU; ++u) cc += thr[u] >= 0.f ? 1u : 0u;
#pragma unroll
        for (int w = 0; w < kW; ++w) cn += tx + kTx * w < valid ? 1u : 0u;
        uint32_t live_w = 0;
#pragma unroll
        for (int g = 0; g < 32; g += kTxLanes) live_w += __shfl_sync(0xFFFFFFFFu, cc, g);
#pragma unroll
        for (int d = kTxLanes / 2; d > 0; d >>= 1) cn += __shfl_xor_sync(0xFFFFFFFFu, cn, d);
        pairs_w = live_w * cn;
      }
      released = false;
      chunks_done = 0;
    }
    TileMeta& meta = sh.meta[m];
    if (!warp_done) {
      // kTma: rows of 128 bytes, 16-byte piece p of row r at piece p ^ (r & 7); this thread's
      // candidate rows (ty & 7) + 64 (ty >> 3) + 8 u and neighbour rows tx + 16 w keep r & 7
      constexpr int kAStep = kTma ? 8 * 128 : kCandStep * kPitch;
      constexpr int kBStep = kTma ? kTx * 128 : kTx * kPitch;
      const unsigned char* a_s = sh.stages[st] + a_row_off;
      const unsigned char* b_s = sh.stages[st] + b_row_off;
      // (two steps per iteration: unrolled further, the loop body outgrows the instruction cache
      // — all 16 steps at once ran 25 % slower)
#pragma unroll 2
      for (int kc = 0; kc < kPieces; ++kc) {
        const uint32_t a_off = kTma ? (kc >> 3) * kBoxBytes + (((kc & 7u) << 4) ^ xa) : kc * 16u;
        const uint32_t b_off = kTma ? (kc >> 3) * kBoxBytes + (((kc & 7u) << 4) ^ xb) : kc * 16u;
        float4 na[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) na[u] = *reinterpret_cast<const float4*>(a_s + u * kAStep + a_off);
#pragma unroll
        for (int w = 0; w < kW; ++w) {
          const float4 b = *reinterpret_cast<const float4*>(b_s + w * kBStep + b_off);
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if constexpr (kDot) acc.dot(u, w, na[u], b);
            else acc.add(u, w, na[u], b);
          }
        }
      }
      ++chunks_done;
      ++chunks_total;
      useful_units += pairs_w * min(static_cast<uint32_t>(kChunk), s.n - min(s.n, c * kChunk));  // (< 2^32 per CTA)
      if constexpr (!kDot) {
        bool all_over = true;
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int w = 0; w < kW; ++w) all_over = all_over && (acc.get(u, w) > thr[u]);
        warp_done = __all_sync(0xFFFFFFFFu, all_over);
        if (warp_done && c + 1 < chunks && lane == 0) {
          if (atomicAdd(&meta.done, 1u) == kConsumerWarps - 1) abandoned_total += meta.calls;  // the last vote
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[st]);  // this warp is done reading the stage

    if (c + 1 == chunks) {
      if (chunks_done == chunks) {
        // ---- completed tile: same epilogue as k_scan_tiles
        float nub[kW];
#pragma unroll
        for (int w = 0; w < kW; ++w) nub[w] = kSymmetric ? meta.nub[tx + kTx * w] : -1.f;
        if constexpr (kDot) {  // not used between the tile's first stage and here: not kept in registers
#pragma unroll
          for (int u = 0; u < kU; ++u) thr[u] = meta.thr[cand0_of_thread + kCandStep * u];
        }
        // dot form: d^2 = |a|^2 + |b|^2 + 2 acc (acc = -(a . b)), never below the error bound
        float cn[kDot ? kU : 1], bn[kDot ? kW : 1];
        if constexpr (kDot) {
#pragma unroll
          for (int u = 0; u < kU; ++u) cn[u] = sh.cnorm[cand0_of_thread + kCandStep * u];
#pragma unroll
          for (int w = 0; w < kW; ++w) bn[w] = meta.nnorm[tx + kTx * w];
        }
        if constexpr (kTma && kDot) {
          if (window) {  // self-match pairs among this thread's 8 x 8 (see the producer's `calls`)
            uint32_t jr[kW];
#pragma unroll
            for (int w = 0; w < kW; ++w) jr[w] = meta.jrow[tx + kTx * w];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              if (thr[u] < 0.f) continue;
              const uint32_t row = sh.cand[cand0_of_thread + kCandStep * u];
#pragma unroll
              for (int w = 0; w < kW; ++w) overlap_total += gap_u32(row, jr[w]) < s.n ? 1u : 0u;
            }
          }
        }
        const float d_floor = 0.5f * s.margin_abs;
        auto dist = [&](int u, int w) -> float {
          if constexpr (kDot) return fmaxf(fmaf(2.f, acc.get(u, w), cn[u] + bn[w]), d_floor);
          else return acc.get(u, w);
        };
        bool hit = false;
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int w = 0; w < kW; ++w) {
            const float d = dist(u, w);
            hit = hit || d <= thr[u] || d < nub[w];
          }
        if (__any_sync(0xFFFFFFFFu, hit)) {
          uint32_t jrow[kW];
#pragma unroll
          for (int w = 0; w < kW; ++w) jrow[w] = meta.jrow[tx + kTx * w];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const uint32_t row = sh.cand[cand0_of_thread + kCandStep * u];
            uint32_t d_min = 0xFFFFFFFFu, j_min = 0xFFFFFFFFu;
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              const uint32_t j = jrow[w];
              const float d = dist(u, w);
              const bool pair_ok = row != 0xFFFFFFFFu && j != 0xFFFFFFFFu && gap_u32(row, j) >= s.n;
              if (pair_ok && d <= thr[u]) {
                const uint32_t bits = __float_as_uint(d);
                if (bits < d_min || (bits == d_min && j < j_min)) {
                  d_min = bits;
                  j_min = j;
                }
              }
              if (pair_ok && d < nub[w]) {
                TSDD_BOUND(j, s.n_rows);
                atomicMin(as_ull(s.nn + j), static_cast<unsigned long long>(nn_key(__float_as_uint(d), row)));
              }
            }
            uint32_t g_min = d_min;
#pragma unroll
            for (int d = kTxLanes / 2; d > 0; d >>= 1) g_min = min(g_min, __shfl_xor_sync(0xFFFFFFFFu, g_min, d));
            uint32_t g_j = d_min == g_min ? j_min : 0xFFFFFFFFu;
#pragma unroll
            for (int d = kTxLanes / 2; d > 0; d >>= 1) g_j = min(g_j, __shfl_xor_sync(0xFFFFFFFFu, g_j, d));
            if ((tx & (kTxLanes - 1)) == 0 && g_j != 0xFFFFFFFFu) {
              TSDD_BOUND(row, s.n_rows);
              atomicMin(as_ull(s.nn + row), static_cast<unsigned long long>(nn_key(g_min, g_j)));
              // (squared distances are >= 0: their bits order like the floats; two warps may share a candidate)
              atomicMin(reinterpret_cast<uint32_t*>(&sh.loc[cand0_of_thread + kCandStep * u]), g_min);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.meta_empty[m]);  // this warp is done with the tile's metadata
      released = true;
    }
    ++seq;
  }
  if (lane == 0) {
    const unsigned long long terms = chunks_total * kChunk * 32ull * kU * kW;
    if (terms) {
      atomicAdd(&s.counters->terms, terms);
      atomicAdd(&s.counters->tile_terms, terms);
      atomicAdd(&s.counters->useful_terms, static_cast<unsigned long long>(useful_units));
      if constexpr (kDot) atomicAdd(&s.counters->dot_terms, terms);
    }
    if (abandoned_total) atomicAdd(&s.counters->abandoned, abandoned_total);
  }
  if constexpr (kTma && kDot) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) overlap_total += __shfl_xor_sync(0xFFFFFFFFu, overlap_total, d);
    if (lane == 0 && overlap_total)  // calls -= overlap (the producer counted live x valid)
      atomicAdd(&s.counters->calls, ~static_cast<unsigned long long>(overlap_total) + 1ull);
  }
}


// ------------------------------------------------------------------ 16 x 8 pairs per thread (dot form)
// What bounds k_scan_tiles_ws in the dot form is not the FMA pipe but its shared-memory loads: 16
// LDS.128 per 64 FFMA2 with 8 x 8 pairs per thread, each LDS.128 costing the scheduler about four
// issue cycles.  This variant doubles the candidates per thread — 16 x 8 pairs, 24
// LDS.128 per 256 FFMA2 — and still fits 232 registers because a pair needs ONE accumulator
// instead of an even / odd couple: an FFMA2 serves two CANDIDATES at once,
//     (acc[2p][w], acc[2p+1][w]) += (a[2p][k], a[2p+1][k]) * (b[w][k], b[w][k]),
// the neighbour value broadcast to both halves (ptxas folds the duplicate into the FFMA2's scalar
// .F32 operand form: no extra instruction).  For the left operand to arrive as a register pair,
// k_gather_rows stores the candidate rows pairwise interleaved (its layout is ours): row pair p of
// a tile is [a(2p,0), a(2p+1,0), a(2p,1), a(2p+1,1), ...].  A probe of exactly this loop runs at
// 0.97 of the FFMA peak with two warps per scheduler.
//   tile: 256 candidates x 128 neighbours; stage: 32 columns = two candidate boxes (128 row
//   pairs x 16 columns x 2) + one neighbour box (128 rows x 32 columns), 48 KB, four stages;
//   thread (ty, tx): row pairs (ty & 7) + 64 (ty >> 3) + 8 i, i < 8 (so that the 128-byte swizzle
//   term is one constant per thread), neighbours tx + 16 w, w < 8; candidate 16 ty + 2 i + h of
//   the tile sits in half h of that pair (tma16_pair_of_candidate).
constexpr int kCand16 = 256;
#ifndef TSDD_WS16_COLS
#define TSDD_WS16_COLS 32
#endif
#ifndef TSDD_WS16_STAGES
#define TSDD_WS16_STAGES 4
#endif

constexpr int kCols16 = TSDD_WS16_COLS;             // columns per stage
constexpr int kStages16 = TSDD_WS16_STAGES;
constexpr int kBox16 = 128 * 128;                   // bytes of one box: 128 rows of 128 bytes
constexpr int kABoxes16 = kCols16 / 16;             // candidate boxes per stage: 16 columns x 2 rows of a pair each
constexpr int kBBoxes16 = kCols16 / 32;             // neighbour boxes per stage: 32 columns each
constexpr int kStageBytes16 = (kABoxes16 + kBBoxes16) * kBox16;

struct alignas(16) TileMeta16 {
  float thr[kCand16];
  float nub[kNbrWs];
  uint32_t jrow[kNbrWs];
  float nnorm[kNbrWs];
  unsigned long long calls;
  uint32_t done;
  uint32_t valid;  // neighbour slots of the tile that hold a row
};

struct Shared16 {
  unsigned char stages[kStages16][kStageBytes16];
  TileMeta16 meta[2];
  uint32_t cand[kCand16];
  float loc[kCand16];
  float cnorm[kCand16];
  uint32_t tag_tile[kStages16 + 1];
  uint32_t tag_chunk[kStages16 + 1];
  unsigned long long full[kStages16], empty[kStages16], meta_full[2], meta_empty[2];  // mbarriers
};

template <bool kSymmetric>
__global__ void __launch_bounds__(kThreadsWs, 1)
k_scan_tiles_ws16(SearchState s, ScanArgs a, const __grid_constant__ CUtensorMap map_a,
                  const __grid_constant__ CUtensorMap map_b) {
  constexpr int kP = 8, kW = 8, kTx = 16;  // row pairs and neighbours per thread
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Shared16& sh = *reinterpret_cast<Shared16*>(smem_raw);

  const uint32_t count = a.sel[0];
  const uint32_t cand0 = blockIdx.y * kCand16;
  if (cand0 >= count) return;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float inf = __uint_as_float(kInfBits);
  if (tid < kCand16) {
    const uint32_t row = (cand0 + tid < count) ? a.batch_rows[cand0 + tid] : 0xFFFFFFFFu;
    sh.cand[tid] = row;
    sh.loc[tid] = inf;
    sh.cnorm[tid] = row != 0xFFFFFFFFu ? s.row_norms[row] : 0.f;
  }
  if (tid == 0) {
    for (int i = 0; i < kStages16; ++i) {
      mbar_init(&sh.full[i], 1);
      mbar_init(&sh.empty[i], kConsumerWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sh.meta_full[i], 1);
      mbar_init(&sh.meta_empty[i], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const bool window = a.nbr_index != nullptr;
  const uint32_t slot_tiles = (s.n_rows + kTileRows - 1) / kTileRows;
  const uint32_t chunks = s.stride / kCols16;
  const uint32_t k_first = a.k_begin + blockIdx.x * a.tiles_per_cta, k_end = a.k_end;
  const uint32_t n_tiles = k_first < k_end ? min(static_cast<uint32_t>(a.tiles_per_cta), k_end - k_first) : 0u;

  if (warp >= kConsumerWarps) {
    // ================================================================ producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp != kConsumerWarps) return;
    const uint32_t centre = window ? a.batch_slots[min(cand0 + kCand16 / 2, count - 1)] / kTileRows : 0u;
    const uint64_t best = a.pruning ? *s.best : 0ull;
    auto slot0_of = [&](uint32_t k) -> uint32_t {
      uint32_t unit;
      if (!window) {
        unit = (k + a.rotation) % slot_tiles;
      } else {
        const uint32_t step = (k + 1) >> 1;
        unit = (k & 1) ? (centre + step) % slot_tiles : (centre + slot_tiles - step % slot_tiles) % slot_tiles;
      }
      return unit * kTileRows;
    };
    uint32_t seq = 0;
    unsigned long long calls_total = 0, tiles_total = 0, live_total = 0;
#pragma unroll 1
    for (uint32_t ti = 0; ti < n_tiles; ++ti) {
      const uint32_t k = k_first + ti, m = ti & 1, use = ti >> 1;
      TileMeta16& meta = sh.meta[m];
      if (use >= 1) mbar_wait(&sh.meta_empty[m], (use - 1) & 1);
      const uint32_t slot0 = slot0_of(k);
      const uint32_t valid = slot0 < s.n_rows ? min(static_cast<uint32_t>(kNbrWs), s.n_rows - slot0) : 0u;
      // ---- candidates: thresholds, and the pair distances they start in this tile
      bool any_live = false;
      unsigned long long calls = 0;
#pragma unroll
      for (int q = 0; q < kCand16 / 32; ++q) {
        const uint32_t r = lane + 32 * q, row = sh.cand[r];
        float thr = -1.f;
        if (row != 0xFFFFFFFFu) {
          if (!a.pruning) {
            thr = inf;
          } else {
            const float bound = fminf(__uint_as_float(key_bits(load_key(s.nn + row))), sh.loc[r]);
            if (!dead_bound(bound, best, s.margin, s.margin_abs, s.margin_q)) thr = bound;
          }
        }
        meta.thr[r] = thr;
        if (thr >= 0.f) {
          any_live = true;
          live_total += 1;
          uint32_t overlap = 0;
          if (!window) {  // (window tiles: the consumers count the self-match pairs)
            const uint32_t z0 = row >= s.n - 1 ? row - (s.n - 1) : 0, z1 = row + s.n;
            const uint32_t o0 = max(slot0, z0), o1 = min(slot0 + valid, z1);
            overlap = o1 > o0 ? o1 - o0 : 0;
          }
          calls += valid - overlap;
        }
      }
      // ---- neighbours
#pragma unroll
      for (int q = 0; q < kNbrWs / 32; ++q) {
        const uint32_t e = lane + 32 * q, slot = slot0 + e;
        uint32_t j = 0xFFFFFFFFu;
        if (slot < s.n_rows) j = window ? a.nbr_index[slot] : slot;
        if (j != 0xFFFFFFFFu) TSDD_BOUND(j, s.n_rows);
        meta.jrow[e] = j;
        meta.nub[e] = j != 0xFFFFFFFFu ? __uint_as_float(key_bits(load_key(s.nn + j))) : -1.f;
        meta.nnorm[e] = j != 0xFFFFFFFFu ? s.row_norms[j] : 0.f;
      }
      any_live = __any_sync(0xFFFFFFFFu, any_live);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) calls += __shfl_xor_sync(0xFFFFFFFFu, calls, d);
      if (lane == 0) {
        meta.calls = calls;
        meta.done = 0;
        meta.valid = valid;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.meta_full[m]);
      if (!any_live) break;
      calls_total += calls;
      tiles_total += 1;
#pragma unroll 1
      for (uint32_t c = 0; c < chunks; ++c) {
        if (a.pruning && *reinterpret_cast<volatile uint32_t*>(&meta.done) == kConsumerWarps) break;
        const uint32_t st = seq % kStages16, round = seq / kStages16;
        if (round >= 1) mbar_wait(&sh.empty[st], (round - 1) & 1);
        if (lane == 0) {
          sh.tag_tile[st] = ti;
          sh.tag_chunk[st] = c;
          mbar_arrive_expect_tx(&sh.full[st], kStageBytes16);
          unsigned char* dst = sh.stages[st];
          // candidate boxes: the interleaved matrix has 2 floats per column; row coordinate = row pair
#pragma unroll
          for (int q = 0; q < kABoxes16; ++q)
            tma_load_box(dst + q * kBox16, &map_a, 2 * c * kCols16 + 32 * q, cand0 / 2, &sh.full[st]);
#pragma unroll
          for (int q = 0; q < kBBoxes16; ++q)
            tma_load_box(dst + (kABoxes16 + q) * kBox16, &map_b, c * kCols16 + 32 * q, slot0, &sh.full[st]);
        }
        ++seq;
      }
    }
    {  // the end-of-work tag
      const uint32_t st = seq % kStages16, round = seq / kStages16;
      if (round >= 1) mbar_wait(&sh.empty[st], (round - 1) & 1);
      if (lane == 0) {
        sh.tag_tile[st] = kTagDone;
        mbar_arrive(&sh.full[st]);
      }
    }
    if (lane == 0) {
      if (calls_total) atomicAdd(&s.counters->calls, calls_total);
      if (tiles_total) atomicAdd(&s.counters->tiles, tiles_total);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) live_total += __shfl_xor_sync(0xFFFFFFFFu, live_total, d);
    if (lane == 0 && live_total) atomicAdd(&s.counters->tile_live, live_total);
    return;
  }

  // ================================================================== consumer warpgroups
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
  const uint32_t tx = (lane & 7u) | ((warp & 1u) << 3), ty = (lane >> 3) | ((warp >> 1) << 2);
  constexpr int kTxLanes = 8;
  const uint32_t cand_of_thread = 16u * ty;  // + 2 i + h
  uint32_t xa = (ty & 7u) << 4, xb = (tx & 7u) << 4;
  uint32_t a_row_off = ((ty & 7u) + 64u * (ty >> 3)) * 128u, b_row_off = kABoxes16 * kBox16 + tx * 128u;
  xa = __shfl_sync(0xFFFFFFFFu, xa, lane), xb = __shfl_sync(0xFFFFFFFFu, xb, lane);
  a_row_off = __shfl_sync(0xFFFFFFFFu, a_row_off, lane), b_row_off = __shfl_sync(0xFFFFFFFFu, b_row_off, lane);
  float2 acc[kP][kW];
  uint32_t seq = 0, cur = kTagDone, m = 0, chunks_done = 0;
  bool released = true, warp_done = false;
  unsigned long long chunks_total = 0;
  uint32_t overlap_total = 0, pairs_w = 0, useful_units = 0;
#pragma unroll 1
  for (;;) {
    const uint32_t st = seq % kStages16, round = seq / kStages16;
    mbar_wait(&sh.full[st], round & 1);
    const uint32_t tile = *reinterpret_cast<volatile uint32_t*>(&sh.tag_tile[st]);
    if (tile == kTagDone) break;
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(&sh.tag_chunk[st]);
    if (tile != cur) {
      if (!released) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.meta_empty[m]);
      }
      cur = tile;
      m = tile & 1;
      mbar_wait(&sh.meta_full[m], (tile >> 1) & 1);
      uint32_t cc = 0, cn = 0;
#pragma unroll
      for (int q = 0; q < 2 * kP; ++q) cc += sh.meta[m].thr[cand_of_thread + q] >= 0.f ? 1u : 0u;
      warp_done = __all_sync(0xFFFFFFFFu, cc == 0);
      if (warp_done && lane == 0 && chunks > 1) atomicAdd(&sh.meta[m].done, 1u);
      {  // (live candidates) x (existing neighbour rows) among this warp's pairs: the useful share of its terms
        const uint32_t valid = sh.meta[m].valid;
#pragma unroll
        for (int w = 0; w < kW; ++w) cn += tx + kTx * w < valid ? 1u : 0u;
        uint32_t live_w = 0;
#pragma unroll
        for (int g = 0; g < 32; g += kTxLanes) live_w += __shfl_sync(0xFFFFFFFFu, cc, g);
#pragma unroll
        for (int d = kTxLanes / 2; d > 0; d >>= 1) cn += __shfl_xor_sync(0xFFFFFFFFu, cn, d);
        pairs_w = live_w * cn;
      }
#pragma unroll
      for (int i = 0; i < kP; ++i)
#pragma unroll
        for (int w = 0; w < kW; ++w) acc[i][w] = make_float2(0.f, 0.f);
      released = false;
      chunks_done = 0;
    }
    TileMeta16& meta = sh.meta[m];
    if (!warp_done) {
      const unsigned char* a_s = sh.stages[st] + a_row_off;
      const unsigned char* b_s = sh.stages[st] + b_row_off;
#pragma unroll 2
      for (int kc = 0; kc < kCols16 / 4; ++kc) {
        // columns 4 kc .. 4 kc + 3: candidate box kc >> 2, its 16-byte pieces 2 (kc & 3) and + 1
        // (a piece = two columns of a row pair); neighbour piece kc
        const uint32_t a_off0 = (kc >> 2) * kBox16 + ((((kc & 3u) * 2u) << 4) ^ xa);
        const uint32_t a_off1 = (kc >> 2) * kBox16 + ((((kc & 3u) * 2u + 1u) << 4) ^ xa);
        const uint32_t b_off = (kc >> 3) * kBox16 + (((static_cast<uint32_t>(kc) & 7u) << 4) ^ xb);
        float4 b[kW];
#pragma unroll
        for (int w = 0; w < kW; ++w) b[w] = *reinterpret_cast<const float4*>(b_s + w * (kTx * 128) + b_off);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4 a01[kP / 2], a23[kP / 2];
#pragma unroll
          for (int p = 0; p < kP / 2; ++p) {
            a01[p] = *reinterpret_cast<const float4*>(a_s + (h * (kP / 2) + p) * (8 * 128) + a_off0);
            a23[p] = *reinterpret_cast<const float4*>(a_s + (h * (kP / 2) + p) * (8 * 128) + a_off1);
          }
#pragma unroll
          for (int p = 0; p < kP / 2; ++p)
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              float2& v = acc[h * (kP / 2) + p][w];
              v = __ffma2_rn(make_float2(a01[p].x, a01[p].y), make_float2(b[w].x, b[w].x), v);
              v = __ffma2_rn(make_float2(a01[p].z, a01[p].w), make_float2(b[w].y, b[w].y), v);
              v = __ffma2_rn(make_float2(a23[p].x, a23[p].y), make_float2(b[w].z, b[w].z), v);
              v = __ffma2_rn(make_float2(a23[p].z, a23[p].w), make_float2(b[w].w, b[w].w), v);
            }
        }
      }
      ++chunks_done;
      ++chunks_total;
      useful_units += pairs_w * min(static_cast<uint32_t>(kCols16), s.n - min(s.n, c * kCols16));  // (< 2^32 per CTA)
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[st]);

    if (c + 1 == chunks) {
      if (chunks_done == chunks) {
        // ---- completed tile: d^2 = |a|^2 + |b|^2 + 2 acc (acc = -(a . b)), never below the error bound
        float nub[kW], bn[kW];
        uint32_t jrow[kW];
#pragma unroll
        for (int w = 0; w < kW; ++w) {
          nub[w] = kSymmetric ? meta.nub[tx + kTx * w] : -1.f;
          bn[w] = meta.nnorm[tx + kTx * w];
          jrow[w] = meta.jrow[tx + kTx * w];
        }
        const float d_floor = 0.5f * s.margin_abs;
        // Which of this thread's 16 candidates can have a pair under their own or a neighbour's
        // bound?  A cheap sufficient test per candidate: its smallest accumulator against ONE limit,
        // max(thr, greatest neighbour bound) - |a|^2 - smallest |b|^2 (no floor: a distance below
        // it can only add a false alarm).  Flagged candidates are then measured pair by pair.
        float nub_max = nub[0], bn_min = bn[0];
#pragma unroll
        for (int w = 1; w < kW; ++w) nub_max = fmaxf(nub_max, nub[w]), bn_min = fminf(bn_min, bn[w]);
        uint32_t hits = 0;
#pragma unroll
        for (int i = 0; i < kP; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t l = cand_of_thread + 2 * i + h;
            const float thr = meta.thr[l], cn = sh.cnorm[l];
            if (window && thr >= 0.f) {  // self-match pairs of a window tile (see the producer's `calls`)
              const uint32_t row = sh.cand[l];
#pragma unroll
              for (int w = 0; w < kW; ++w) overlap_total += gap_u32(row, jrow[w]) < s.n ? 1u : 0u;
            }
            float a_min = h ? acc[i][0].y : acc[i][0].x;
#pragma unroll
            for (int w = 1; w < kW; ++w) a_min = fminf(a_min, h ? acc[i][w].y : acc[i][w].x);
            const bool hit = fmaf(2.f, a_min, cn + bn_min) <= fmaxf(thr, nub_max);
            hits |= (hit ? 1u : 0u) << (2 * i + h);
          }
        // the candidates of a thread row are shared by the 8 lanes of its thread columns
        uint32_t row_hits = hits;
#pragma unroll
        for (int d = kTxLanes / 2; d > 0; d >>= 1) row_hits |= __shfl_xor_sync(0xFFFFFFFFu, row_hits, d);
        if (__any_sync(0xFFFFFFFFu, row_hits != 0)) {
#pragma unroll
          for (int i = 0; i < kP; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (!__any_sync(0xFFFFFFFFu, (row_hits >> (2 * i + h)) & 1u)) continue;  // (warp-uniform)
              const uint32_t l = cand_of_thread + 2 * i + h;
              const uint32_t row = sh.cand[l];
              const float thr = meta.thr[l], cn = sh.cnorm[l];
              uint32_t d_min = 0xFFFFFFFFu, j_min = 0xFFFFFFFFu;
#pragma unroll
              for (int w = 0; w < kW; ++w) {
                const uint32_t j = jrow[w];
                const float d = fmaxf(fmaf(2.f, h ? acc[i][w].y : acc[i][w].x, cn + bn[w]), d_floor);
                const bool pair_ok = row != 0xFFFFFFFFu && j != 0xFFFFFFFFu && gap_u32(row, j) >= s.n;
                if (pair_ok && d <= thr) {
                  const uint32_t bits = __float_as_uint(d);
                  if (bits < d_min || (bits == d_min && j < j_min)) {
                    d_min = bits;
                    j_min = j;
                  }
                }
                if (pair_ok && d < nub[w]) {
                  TSDD_BOUND(j, s.n_rows);
                  atomicMin(as_ull(s.nn + j), static_cast<unsigned long long>(nn_key(__float_as_uint(d), row)));
                }
              }
              // smallest distance among the 8 thread columns; the lane(s) holding it publish it (the
              // 64-bit atomicMin settles a tie towards the smaller neighbour row)
              uint32_t g_min = d_min;
#pragma unroll
              for (int d = kTxLanes / 2; d > 0; d >>= 1) g_min = min(g_min, __shfl_xor_sync(0xFFFFFFFFu, g_min, d));
              if (d_min == g_min && j_min != 0xFFFFFFFFu) {
                TSDD_BOUND(row, s.n_rows);
                atomicMin(as_ull(s.nn + row), static_cast<unsigned long long>(nn_key(d_min, j_min)));
                atomicMin(reinterpret_cast<uint32_t*>(&sh.loc[l]), d_min);
              }
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.meta_empty[m]);
      released = true;
    }
    ++seq;
  }
  if (lane == 0) {
    const unsigned long long terms = chunks_total * kCols16 * 32ull * (2 * kP) * kW;
    if (terms) {
      atomicAdd(&s.counters->terms, terms);
      atomicAdd(&s.counters->tile_terms, terms);
      atomicAdd(&s.counters->dot_terms, terms);
      atomicAdd(&s.counters->useful_terms, static_cast<unsigned long long>(useful_units));
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) overlap_total += __shfl_xor_sync(0xFFFFFFFFu, overlap_total, d);
  if (lane == 0 && overlap_total)
    atomicAdd(&s.counters->calls, ~static_cast<unsigned long long>(overlap_total) + 1ull);
}

}  // namespace ws

// Squared norm of every float32 row (padding columns are zero): one warp per row.
__global__ void __launch_bounds__(256)
k_row_norms(const float* __restrict__ rows, uint32_t n_rows, uint32_t stride, float* __restrict__ norms) {
  const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const float4* p = reinterpret_cast<const float4*>(rows + static_cast<size_t>(row) * stride);
  float acc = 0.f;
  for (uint32_t c = lane; c < stride / 4; c += 32) {
    const float4 v = p[c];
    acc += (v.x * v.x + v.y * v.y) + (v.z * v.z + v.w * v.w);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
  if (lane == 0) norms[row] = acc;
}

// ------------------------------------------------------------------ finalists, decided in float64
__global__ void __launch_bounds__(256)
k_collect_finalists(SearchState s, uint32_t* __restrict__ list, uint32_t cap, uint32_t* __restrict__ count) {
  const uint64_t best = *s.best;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n_rows; i += gridDim.x * blockDim.x) {
    if (!s.exact[i] || s.excluded[i]) continue;
    const uint64_t key = s.nn[i];
    if (key_bits(key) == kInfBits || is_dead(key, best, s.margin, s.margin_abs, s.margin_q)) continue;
    const uint32_t at = atomicAdd(count, 1u);
    if (at < cap) list[at] = i;  // (guarded: the host collects again with room for all)
  }
}

__global__ void k_gather_keys(const uint64_t* __restrict__ nn, const uint32_t* __restrict__ list, uint32_t count,
                              uint64_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = nn[list[i]];  // (list entries are row numbers written by k_collect_finalists)
}

// z-normalised float64 values of one row (series.cpp:21-37), kept in global memory
// so that every thread of k_exact_nn reads them as a broadcast.
__global__ void k_zrow(const double* __restrict__ x, const double* __restrict__ mean,
                       const double* __restrict__ inv_sigma, uint32_t n, uint32_t row, double* __restrict__ z) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) z[t] = __dmul_rn(x[row + t] - mean[row], inv_sigma[row]);  // same rounding as in k_exact_nn
}

// One thread per neighbour j (adjacent threads read adjacent samples: coalesced),
// float64 throughout, early abandoning against the running minimum.  A neighbour whose
// segment means already put it further away than that minimum (the lower bound of
// prep_kernels.cu, with the tile filter's 0.1 % slack for the float32 means) is not measured.
__global__ void __launch_bounds__(256)
k_exact_nn(const double* __restrict__ x, const double* __restrict__ mean, const double* __restrict__ inv_sigma,
           uint32_t n_rows, uint32_t n, uint32_t row, const double* __restrict__ z,
           const float* __restrict__ lb_means, float lb_scale, float lb_q, unsigned long long* out_bits) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  double mine = __longlong_as_double(0x7FF0000000000000ll);  // +inf
  bool wanted = j < n_rows && gap_u32(row, j) >= n;
  const double bound = __longlong_as_double(static_cast<long long>(
      __ldcg(reinterpret_cast<const unsigned long long*>(out_bits))));
  if (wanted && lb_means != nullptr) {
    const float4* pi = reinterpret_cast<const float4*>(lb_means + static_cast<size_t>(row) * kLbSegments);
    const float4* pj = reinterpret_cast<const float4*>(lb_means + static_cast<size_t>(j) * kLbSegments);
    float lb = 0.f;
#pragma unroll
    for (int q = 0; q < kLbSegments / 4; ++q) {
      const float4 a = __ldg(pi + q), b = __ldg(pj + q);
      const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, dw = a.w - b.w;
      lb = fmaf(dx, dx, lb), lb = fmaf(dy, dy, lb), lb = fmaf(dz, dz, lb), lb = fmaf(dw, dw, lb);
    }
    wanted = !(static_cast<double>(lb * lb_scale) >
               bound * 1.001 + static_cast<double>(lb_q) * sqrt(bound) + static_cast<double>(lb_q * lb_q));
  }
  if (wanted) {
    const double mu = mean[j], inv = inv_sigma[j];
    const double* p = x + j;
    double sum = 0.0;
    uint32_t t = 0;
    for (; t < n; ++t) {
      // both rows rounded the same way (no fma contraction), so that d(i, j) == d(j, i) to the
      // last bit and mutual nearest neighbours tie exactly, as they do in the reference
      const double d = z[t] - __dmul_rn(p[t] - mu, inv);
      sum = fma(d, d, sum);
      if ((t & 31) == 31 && sum > bound) break;
    }
    if (t >= n) mine = sum;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mine = fmin(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, d));
  if ((threadIdx.x & 31) == 0 && mine < __longlong_as_double(0x7FF0000000000000ll))
    atomicMin(out_bits, static_cast<unsigned long long>(__double_as_longlong(mine)));  // doubles >= 0 order like their bits
}

// Several finalists at once (blockIdx.y): the same arithmetic per pair as k_exact_nn — the float64 results are
// bit-identical — with one launch and one read-back for the group instead of one per finalist.
constexpr int kExactGroup = 4;
struct ExactGroup {
  uint32_t row[kExactGroup];
};
__global__ void k_zrow_group(const double* __restrict__ x, const double* __restrict__ mean,
                             const double* __restrict__ inv_sigma, uint32_t n, ExactGroup g, double* __restrict__ z) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, row = g.row[blockIdx.y];
  if (t < n) z[static_cast<size_t>(blockIdx.y) * n + t] = __dmul_rn(x[row + t] - mean[row], inv_sigma[row]);
}
__global__ void __launch_bounds__(256)
k_exact_nn_group(const double* __restrict__ x, const double* __restrict__ mean, const double* __restrict__ inv_sigma,
                 uint32_t n_rows, uint32_t n, ExactGroup g, const double* __restrict__ z_all,
                 const float* __restrict__ lb_means, float lb_scale, float lb_q, unsigned long long* out_bits_all) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x, row = g.row[blockIdx.y];
  const double* z = z_all + static_cast<size_t>(blockIdx.y) * n;
  unsigned long long* out_bits = out_bits_all + blockIdx.y;
  double mine = __longlong_as_double(0x7FF0000000000000ll);  // +inf
  bool wanted = j < n_rows && gap_u32(row, j) >= n;
  const double bound = __longlong_as_double(static_cast<long long>(
      __ldcg(reinterpret_cast<const unsigned long long*>(out_bits))));
  if (wanted && lb_means != nullptr) {
    const float4* pi = reinterpret_cast<const float4*>(lb_means + static_cast<size_t>(row) * kLbSegments);
    const float4* pj = reinterpret_cast<const float4*>(lb_means + static_cast<size_t>(j) * kLbSegments);
    float lb = 0.f;
#pragma unroll
    for (int q = 0; q < kLbSegments / 4; ++q) {
      const float4 a = __ldg(pi + q), b = __ldg(pj + q);
      const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, dw = a.w - b.w;
      lb = fmaf(dx, dx, lb), lb = fmaf(dy, dy, lb), lb = fmaf(dz, dz, lb), lb = fmaf(dw, dw, lb);
    }
    wanted = !(static_cast<double>(lb * lb_scale) >
               bound * 1.001 + static_cast<double>(lb_q) * sqrt(bound) + static_cast<double>(lb_q * lb_q));
  }
  if (wanted) {
    const double mu = mean[j], inv = inv_sigma[j];
    const double* p = x + j;
    double sum = 0.0;
    uint32_t t = 0;
    for (; t < n; ++t) {
      const double d = z[t] - __dmul_rn(p[t] - mu, inv);  // (both rows rounded the same way: see k_exact_nn)
      sum = fma(d, d, sum);
      if ((t & 31) == 31 && sum > bound) break;
    }
    if (t >= n) mine = sum;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mine = fmin(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, d));
  if ((threadIdx.x & 31) == 0 && mine < __longlong_as_double(0x7FF0000000000000ll))
    atomicMin(out_bits, static_cast<unsigned long long>(__double_as_longlong(mine)));
}

inline uint32_t slot_tiles_of(uint32_t rows) { return (rows + kTileRows - 1) / kTileRows; }

}  // namespace

// ------------------------------------------------------------------ launchers
int launch_reset_search(SearchState s, cudaStream_t stream) {
  k_reset_search<<<blocks_for(s.n_rows, 256), 256, 0, stream>>>(s);
  return 1;
}

int launch_min_from_peers(uint64_t* d_nn, PeerPointers peers, uint32_t rows, cudaStream_t stream) {
  if (peers.count == 0 || rows == 0) return 0;
  k_min_from_peers<<<blocks_for((static_cast<size_t>(rows) + 1) / 2, 256), 256, 0, stream>>>(d_nn, peers, rows);
  return 1;
}

int launch_bucket_mates(SearchState s, const double* d_series, const float* d_series_f32, const double* d_mean,
                        const double* d_inv_sigma, const uint32_t* d_sorted_row, const uint32_t* d_slot_bucket,
                        const uint32_t* d_offsets, int mates, uint32_t run_pairs, uint32_t world, uint32_t rank,
                        cudaStream_t stream, int form) {
  if (mates <= 0) return 0;
  const size_t slots = (static_cast<size_t>(s.n_rows) + world - 1) / world;
  const bool old_form = form == 0;
  // buckets that are mostly runs of consecutive rows: chains along the diagonals (k_bucket_mates_runs)
  if (form == 2 || (form < 0 && static_cast<uint64_t>(run_pairs) * 2 >= s.n_rows)) {
    const size_t chunks = ((static_cast<size_t>(s.n_rows) + 31) / 32 + world - 1) / world;
    if (d_series_f32 != nullptr)
      k_bucket_mates_runs<float><<<blocks_for(chunks * 32, 256), 256, 0, stream>>>(
          s, d_series_f32, d_mean, d_inv_sigma, d_sorted_row, d_slot_bucket, d_offsets, mates, world, rank);
    else
      k_bucket_mates_runs<double><<<blocks_for(chunks * 32, 256), 256, 0, stream>>>(
          s, d_series, d_mean, d_inv_sigma, d_sorted_row, d_slot_bucket, d_offsets, mates, world, rank);
    return 1;
  }
  if (d_series_f32 != nullptr && s.n <= 1024 && !old_form) {
    const unsigned blocks = blocks_for(slots * 32, 256);
    auto go = [&](auto kernel) {
      kernel<<<blocks, 256, 0, stream>>>(s, d_series_f32, d_mean, d_inv_sigma, d_sorted_row, d_slot_bucket, d_offsets, mates, world,
                                         rank);
    };
    if (s.n <= 64) go(k_bucket_mates_f32<2>);
    else if (s.n <= 128) go(k_bucket_mates_f32<4>);
    else if (s.n <= 256) go(k_bucket_mates_f32<8>);
    else if (s.n <= 512) go(k_bucket_mates_f32<16>);
    else go(k_bucket_mates_f32<32>);
  } else if (d_series_f32 != nullptr)
    k_bucket_mates<float><<<blocks_for(slots * 32, 256), 256, 0, stream>>>(
        s, d_series_f32, d_mean, d_inv_sigma, d_sorted_row, d_slot_bucket, d_offsets, mates, world, rank);
  else
    k_bucket_mates<double><<<blocks_for(slots * 32, 256), 256, 0, stream>>>(
        s, d_series, d_mean, d_inv_sigma, d_sorted_row, d_slot_bucket, d_offsets, mates, world, rank);
  return 1;
}

int launch_propagate(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel, uint32_t live_upper_bound,
                     int tries, cudaStream_t stream) {
  if (tries <= 0 || live_upper_bound == 0) return 0;
  k_propagate<<<blocks_for(static_cast<size_t>(live_upper_bound) * 32, 256), 256, 0, stream>>>(s, d_batch_rows, d_sel, tries);
  return 1;
}

int launch_select_batch(SearchState s, const uint32_t* d_order, uint32_t cursor, uint32_t batch,
                        uint32_t world, uint32_t rank, bool pruning, uint32_t* d_flags,
                        uint32_t* d_scan_scratch, uint32_t* d_batch_rows, uint32_t* d_sel,
                        cudaStream_t stream) {
  const uint32_t span = s.n_rows - cursor;
  const unsigned blocks = blocks_for(span, 256);
  k_flag_live<<<blocks, 256, 0, stream>>>(s, d_order, cursor, world, rank, pruning ? 1 : 0, d_flags);
  // ranks live right behind the flags
  uint32_t* d_ranks = d_flags + s.n_rows;
  int launches = 1 + launch_exclusive_scan(d_flags, d_ranks, span, d_scan_scratch, stream);
  k_take_batch<<<blocks, 256, 0, stream>>>(d_order, d_flags, d_ranks, cursor, s.n_rows, batch,
                                           d_batch_rows, d_sel);
  return launches + 1;
}

int launch_compact_batch(SearchState s, uint32_t* d_batch_rows, uint32_t* d_batch_slots, uint32_t* d_rows_alt,
                         uint32_t* d_slots_alt, bool pruning, uint32_t* d_sel, uint32_t live_upper_bound,
                         uint32_t* d_scratch, cudaStream_t stream) {
  if (live_upper_bound > 4096 && d_scratch != nullptr) {  // many blocks: flags, per-block counts, scatter, publish
    const unsigned blocks = (live_upper_bound + 1023) / 1024;
    uint32_t* d_flags = d_scratch;
    uint32_t* d_counts = d_scratch + static_cast<size_t>(blocks) * 1024;
    k_compact_flag<<<blocks, 1024, 0, stream>>>(s, d_batch_rows, pruning ? 1 : 0, d_sel, d_flags, d_counts);
    k_compact_scatter<<<blocks, 1024, 0, stream>>>(d_batch_rows, d_batch_slots, d_rows_alt, d_slots_alt, d_flags,
                                                   d_counts, d_sel);
    k_compact_publish<<<1, 1, 0, stream>>>(d_sel);
    return 3;
  }
  k_compact_batch<<<1, 1024, 0, stream>>>(s, d_batch_rows, d_batch_slots, d_rows_alt, d_slots_alt,
                                          pruning ? 1 : 0, d_sel);
  return 1;
}

int launch_invert_order(const uint32_t* d_sorted_row, uint32_t rows, uint32_t* d_slot_of_row,
                        cudaStream_t stream) {
  k_invert_order<<<blocks_for(rows, 256), 256, 0, stream>>>(d_sorted_row, rows, d_slot_of_row);
  return 1;
}

int launch_batch_slots(const uint32_t* d_batch_rows, const uint32_t* d_sel, const uint32_t* d_slot_of_row,
                       uint32_t capacity, uint32_t* d_keys, cudaStream_t stream) {
  k_batch_slots<<<blocks_for(capacity, 256), 256, 0, stream>>>(d_batch_rows, d_sel, d_slot_of_row, d_keys);
  return 1;
}

int launch_gather_rows(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel,
                       uint32_t capacity_padded, int tma_layout, float* d_batch_matrix, cudaStream_t stream) {
  k_gather_rows<<<blocks_for(static_cast<size_t>(capacity_padded) * 32, 256), 256, 0, stream>>>(
      s, d_batch_rows, d_sel, capacity_padded, tma_layout, d_batch_matrix);
  return 1;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda).
PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult status = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &status) != cudaSuccess ||
        status != cudaDriverEntryPointSuccess)
      p = nullptr;
    (void)cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}

// float32 matrix [n_rows x stride], boxes of 128 rows x 32 columns, 128-byte swizzle
bool make_row_map(CUtensorMap* map, const float* base, uint64_t n_rows, uint64_t stride) {
  PFN_cuTensorMapEncodeTiled encode = tensor_map_encoder();
  if (!encode) return false;
  const cuuint64_t dims[2] = {stride, n_rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(stride) * sizeof(float)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(ws::kBoxCols), static_cast<cuuint32_t>(kTileRows)};
  const cuuint32_t elem[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, elem,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_row_map_boxed(void* map, const void* base, uint64_t n_rows, uint64_t stride, uint32_t box_cols, uint32_t box_rows,
                        uint32_t elem_bytes) {
  PFN_cuTensorMapEncodeTiled encode = tensor_map_encoder();
  if (!encode) return false;
  const cuuint64_t dims[2] = {stride, n_rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(stride) * elem_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t elem[2] = {1, 1};
  const CUtensorMapSwizzle swizzle = box_cols * elem_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  const CUtensorMapDataType type = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return encode(static_cast<CUtensorMap*>(map), type, 2, const_cast<void*>(base), dims, strides, box, elem,
                CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

ScanChoice choose_scan_kernel(const ScanConfig& cfg, const SearchState& s, uint32_t live_upper_bound, bool window,
                              bool pruning, bool dot_form) {
  ScanChoice c{};
  c.packed = cfg.packed;
  c.wide = cfg.wide_tile;
  c.lb = pruning && !window && s.lb_means != nullptr && cfg.variant != 2;
  // variant 0 (automatic): the warp-specialised kernel wherever the lower-bound filter has
  // nothing to offer (window rounds; covering scans of searches on which it is switched off)
  // and the batch still fills 128-candidate tiles; k_scan_tiles otherwise
  const bool tma_ok = cfg.tensor_map && tensor_map_encoder() != nullptr;
  // ... or, with tensor-map loads, where the filter runs on the producer warpgroup (kLb)
  const bool lb_in_ws = c.lb && tma_ok && cfg.filter_in_ws;
  // (not for the window rounds of a search in the direct form: their launches are a few tiles per candidate tile, and
  // 128 x 64 tiles on two CTAs per SM spread them over twice the SMs — cfg 4: 2.5 -> 1.5 ms, cfg 3: 1.25 -> 0.8 ms)
  c.ws = cfg.variant == 2 || (cfg.variant == 0 && cfg.packed && !cfg.wide_tile && (!c.lb || lb_in_ws) &&
                              live_upper_bound > 64 && !(window && !dot_form));
  c.dot = c.ws && !c.lb && dot_form && s.row_norms != nullptr;
  // window launches read scattered rows unless the engine keeps a copy of the matrix in the
  // hash-sorted order (it does once a search runs in the dot form)
  c.tma = c.ws && tma_ok && (!window || (c.dot && s.rows_sorted != nullptr));
  // the dot form on 256-candidate tiles, 16 x 8 pairs per thread, while the batch fills them
  c.tile16 = c.dot && c.tma && cfg.tile16 && live_upper_bound > 192;
  // ... or on the tensor cores, while it fills 128-candidate tiles (the engine keeps the split operands then)
  c.tc = c.dot && c.tma && cfg.tensor_cores && live_upper_bound > 96;
  if (c.tc) c.tile16 = false;
  return c;
}

int launch_scan_tiles(const ScanChoice& choice, SearchState s, const float* d_batch_matrix,
                      const uint32_t* d_batch_rows, const uint32_t* d_batch_slots, const uint32_t* d_sel,
                      uint32_t live_upper_bound, const uint32_t* d_nbr_index, uint32_t k_begin, uint32_t k_end,
                      uint32_t rotation, bool pruning, bool symmetric, cudaStream_t stream, const char** error) {
  if (error) *error = nullptr;
  if (k_end <= k_begin || live_upper_bound == 0) return 0;
  const bool lb = choice.lb, use_ws = choice.ws;
  const bool wide = choice.wide, use_packed = choice.packed;
  // tile shape: 64-candidate tiles once the batch has shrunk to that, else 128
  const bool narrow = !wide && !use_ws && live_upper_bound <= 64;
  const uint32_t cand_rows = choice.tile16 ? 256 : narrow ? 64 : 128;
  const uint32_t nbr_rows = use_ws ? 128 : wide ? 128 : narrow ? 128 : 64;
  const uint32_t cand_tiles = (live_upper_bound + cand_rows - 1) / cand_rows;
  const uint64_t sub_tiles = static_cast<uint64_t>(k_end - k_begin) * (kTileRows / nbr_rows);
  // a few tiles per CTA (thresholds are refreshed per tile), several waves of CTAs per launch
  const uint64_t resident = 148ull * ((wide || use_ws) ? 1 : 2);
  const uint64_t want = sub_tiles * cand_tiles / (resident * 8ull);
  const int tiles_per_cta = static_cast<int>(want < 1 ? 1 : want > 16 ? 16 : want);
  dim3 grid(static_cast<unsigned>((sub_tiles + tiles_per_cta - 1) / tiles_per_cta), cand_tiles);
  ScanArgs a{d_batch_matrix, d_batch_rows, d_batch_slots, d_sel, d_nbr_index, k_begin, k_end, rotation,
             tiles_per_cta, pruning ? 1 : 0};
  if (use_ws) {
    CUtensorMap map_a{}, map_b{};
    bool tma = choice.tma;
    if (tma)
      tma = (choice.tile16  // row pairs, two floats per column
                 ? make_row_map(&map_a, d_batch_matrix, static_cast<uint64_t>(cand_tiles) * 128, 2ull * s.stride)
                 : make_row_map(&map_a, d_batch_matrix, static_cast<uint64_t>(cand_tiles) * kTileRows, s.stride)) &&
            make_row_map(&map_b, d_nbr_index != nullptr ? s.rows_sorted : s.rows,
                         static_cast<uint64_t>(slot_tiles_of(s.n_rows + 1)) * kTileRows, s.stride);
    if (choice.tma && !tma) {  // the gather already used the tensor-map row order: no way back
      if (error) *error = "cuTensorMapEncodeTiled failed";
      return 0;
    }
    auto launch_ws = [&](auto kernel, size_t smem_bytes) {
      const int smem = static_cast<int>(smem_bytes);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kernel<<<grid, ws::kThreadsWs, smem, stream>>>(s, a, map_a, map_b);
    };
    auto pick_ws = [&](auto sym) {
      constexpr bool kS = decltype(sym)::value;
      if (choice.tile16) launch_ws(ws::k_scan_tiles_ws16<kS>, sizeof(ws::Shared16));
      else if (tma && lb) launch_ws(ws::k_scan_tiles_ws<kS, false, true, true>, sizeof(ws::SharedWsT<true, true>));
      else if (tma && choice.dot) launch_ws(ws::k_scan_tiles_ws<kS, true, true>, sizeof(ws::SharedWsT<true>));
      else if (tma) launch_ws(ws::k_scan_tiles_ws<kS, false, true>, sizeof(ws::SharedWsT<true>));
      else if (choice.dot) launch_ws(ws::k_scan_tiles_ws<kS, true, false>, sizeof(ws::SharedWsT<false>));
      else launch_ws(ws::k_scan_tiles_ws<kS, false, false>, sizeof(ws::SharedWsT<false>));
    };
    if (symmetric) pick_ws(std::true_type{});
    else pick_ws(std::false_type{});
    return 1;
  }
  auto launch = [&](auto kernel) {
    const int smem = static_cast<int>(scan_smem_bytes(cand_rows, nbr_rows));
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kernel<<<grid, kScanThreads, smem, stream>>>(s, a);
  };
  const int shape = (wide ? 2 : narrow ? 1 : 0);
  auto pick = [&](auto packed, auto sym, auto with_lb) {
    constexpr bool kP = decltype(packed)::value, kS = decltype(sym)::value, kL = decltype(with_lb)::value;
    if (shape == 2) launch(k_scan_tiles<kP, kS, 16, 8, kL>);
    else if (shape == 1) launch(k_scan_tiles<kP, kS, 8, 4, kL>);
    else launch(k_scan_tiles<kP, kS, 16, 4, kL>);
  };
  auto pick_lb = [&](auto packed, auto sym) {
    if (lb) pick(packed, sym, std::true_type{});
    else pick(packed, sym, std::false_type{});
  };
  if (use_packed) {
    if (symmetric) pick_lb(std::true_type{}, std::true_type{});
    else pick_lb(std::true_type{}, std::false_type{});
  } else {
    if (symmetric) pick_lb(std::false_type{}, std::true_type{});
    else pick_lb(std::false_type{}, std::false_type{});
  }
  return 1;
}

// The matrix in the hash-sorted order: slot p holds row sorted_row[p]; slots from n_rows on are zero.
__global__ void __launch_bounds__(256)
k_permute_rows(const float* __restrict__ rows, const uint32_t* __restrict__ sorted_row, uint32_t n_rows,
               uint32_t rows_padded, uint32_t stride, float* __restrict__ out) {
  const uint32_t slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (slot >= rows_padded) return;
  float4* dst = reinterpret_cast<float4*>(out + static_cast<size_t>(slot) * stride);
  if (slot < n_rows) {
    TSDD_BOUND(sorted_row[slot], n_rows);
    const float4* src = reinterpret_cast<const float4*>(rows + static_cast<size_t>(sorted_row[slot]) * stride);
    for (uint32_t c = lane; c < stride / 4; c += 32) dst[c] = __ldg(src + c);
  } else {
    for (uint32_t c = lane; c < stride / 4; c += 32) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

int launch_permute_rows(const float* d_rows, const uint32_t* d_sorted_row, uint32_t n_rows, uint32_t rows_padded,
                        uint32_t stride, float* d_out, cudaStream_t stream) {
  k_permute_rows<<<blocks_for(static_cast<size_t>(rows_padded) * 32, 256), 256, 0, stream>>>(
      d_rows, d_sorted_row, n_rows, rows_padded, stride, d_out);
  return 1;
}

int launch_row_norms(const float* d_rows, uint32_t n_rows_plus_one, uint32_t stride, float* d_norms,
                     cudaStream_t stream) {
  k_row_norms<<<blocks_for(static_cast<size_t>(n_rows_plus_one) * 32, 256), 256, 0, stream>>>(d_rows, n_rows_plus_one,
                                                                                            stride, d_norms);
  return 1;
}

int launch_finalize_batch(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel,
                          uint32_t capacity, bool pruning, cudaStream_t stream) {
  k_finalize_batch<<<blocks_for(capacity, 256), 256, 0, stream>>>(s, d_batch_rows, d_sel, pruning ? 1 : 0);
  return 1;
}

int launch_seed_lower_bound(SearchState s, const uint32_t* d_order, uint32_t seed_rows, uint32_t* d_seed_lb,
                            cudaStream_t stream) {
  if (s.lb_means == nullptr || seed_rows == 0) return 0;
  seed_rows = seed_rows < s.n_rows ? seed_rows : s.n_rows;
  const uint32_t units = (s.n_rows + kLbBoxRows - 1) / kLbBoxRows;
  // Two passes on large inputs (d_seed_lb holds 2 x seed_rows words): every 16th box gives an upper bound U(i) >= L(i)
  // for all seed rows at a sixteenth of the price; the exact L(i) is then computed for the eighth of the rows with the
  // greatest U(i) only — the maximum of ANY rows' L(i) is a valid best-so-far, and the greatest L(i) sits among the
  // greatest U(i).  workload 4: 3.0 -> 0.6 ms, the same seed.
  constexpr uint32_t kCoarse = 16;
  if (seed_rows >= 1024 && seed_rows <= kSeedSelectMax && units >= kCoarse * 1024) {
    const uint32_t keep = seed_rows / 8;
    uint32_t* d_rows = d_seed_lb + seed_rows;   // the rows kept
    uint32_t* d_exact = d_rows + keep;          // their exact bounds
    cudaMemsetAsync(d_seed_lb, 0x7F, (seed_rows + 2 * keep) * sizeof(uint32_t), stream);  // 0x7F7F7F7F: above every bound
    const uint32_t coarse_units = (units + kCoarse - 1) / kCoarse;
    k_seed_lower_bound<<<dim3((coarse_units + kSeedUnits - 1) / kSeedUnits, (seed_rows + 255) / 256), 256, 0, stream>>>(
        s, d_order, seed_rows, d_seed_lb, kCoarse);
    k_seed_select<<<(seed_rows + 255) / 256, 256, 0, stream>>>(d_order, d_seed_lb, seed_rows, keep, d_rows);
    k_seed_lower_bound<<<dim3((units + kSeedUnits - 1) / kSeedUnits, (keep + 255) / 256), 256, 0, stream>>>(s, d_rows, keep, d_exact, 1);
    k_install_seed<<<1, 256, 0, stream>>>(s, d_exact, keep);
    return 4;
  }
  cudaMemsetAsync(d_seed_lb, 0x7F, seed_rows * sizeof(uint32_t), stream);  // 0x7F7F7F7F: above every bound
  const dim3 grid((units + kSeedUnits - 1) / kSeedUnits, (seed_rows + 255) / 256);
  k_seed_lower_bound<<<grid, 256, 0, stream>>>(s, d_order, seed_rows, d_seed_lb, 1);
  k_install_seed<<<1, 256, 0, stream>>>(s, d_seed_lb, seed_rows);
  return 2;
}

int launch_seed_best(SearchState s, cudaStream_t stream) {
  k_seed_best<<<296, 256, 0, stream>>>(s);
  return 1;
}

int launch_exclude_zone(SearchState s, uint32_t row, cudaStream_t stream) {
  k_exclude_zone<<<blocks_for(2 * static_cast<size_t>(s.n), 256), 256, 0, stream>>>(s, row);
  return 1;
}

int launch_collect_finalists(SearchState s, uint32_t* d_list, uint32_t cap, uint32_t* d_count,
                             cudaStream_t stream) {
  cudaMemsetAsync(d_count, 0, sizeof(uint32_t), stream);
  k_collect_finalists<<<296, 256, 0, stream>>>(s, d_list, cap, d_count);
  return 1;
}

int launch_gather_keys(SearchState s, const uint32_t* d_list, uint32_t count, uint64_t* d_keys, cudaStream_t stream) {
  if (count == 0) return 0;
  k_gather_keys<<<blocks_for(count, 256), 256, 0, stream>>>(s.nn, d_list, count, d_keys);
  return 1;
}

int launch_exact_nn(const double* d_series, const double* d_mean, const double* d_inv_sigma,
                    uint32_t n_rows, uint32_t n, uint32_t row, double* d_zrow, const float* d_lb_means,
                    float lb_scale, float lb_q, unsigned long long* d_out_bits, cudaStream_t stream) {
  k_zrow<<<blocks_for(n, 256), 256, 0, stream>>>(d_series, d_mean, d_inv_sigma, n, row, d_zrow);
  k_exact_nn<<<blocks_for(n_rows, 256), 256, 0, stream>>>(d_series, d_mean, d_inv_sigma, n_rows, n, row,
                                                         d_zrow, d_lb_means, lb_scale, lb_q, d_out_bits);
  return 2;
}

// `count` <= 4 finalists in one launch: d_zrow holds count x n doubles, d_out_bits count start bounds (in) / results (out)
int launch_exact_nn_group(const double* d_series, const double* d_mean, const double* d_inv_sigma, uint32_t n_rows,
                          uint32_t n, const uint32_t* rows, uint32_t count, double* d_zrow, const float* d_lb_means,
                          float lb_scale, float lb_q, unsigned long long* d_out_bits, cudaStream_t stream) {
  ExactGroup g{};
  for (uint32_t f = 0; f < count && f < static_cast<uint32_t>(kExactGroup); ++f) g.row[f] = rows[f];
  k_zrow_group<<<dim3(blocks_for(n, 256), count), 256, 0, stream>>>(d_series, d_mean, d_inv_sigma, n, g, d_zrow);
  k_exact_nn_group<<<dim3(blocks_for(n_rows, 256), count), 256, 0, stream>>>(d_series, d_mean, d_inv_sigma, n_rows, n, g, d_zrow,
                                                                             d_lb_means, lb_scale, lb_q, d_out_bits);
  return 2;
}

}  // namespace tsdd_b200
