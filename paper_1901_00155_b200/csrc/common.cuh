// Shared device helpers of the B200 discord-search engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include <cstdio>

// -DTSDD_DEBUG_BOUNDS: every index that reaches global memory through a data-dependent path is
// checked in the kernel itself; a violation prints where and traps (the launch fails with
// cudaErrorAssert / an illegal instruction, which the engine reports).  compute-sanitizer is not
// available on the GPU pool this was developed on; the checked build (libtsdd_cuda_dbg.so) runs
// the randomised edge-shape tests in its place.  The release build compiles the checks out.
#ifdef TSDD_DEBUG_BOUNDS
#define TSDD_BOUND(index, limit)                                                                         \
  do {                                                                                                   \
    if (!(static_cast<unsigned long long>(index) < static_cast<unsigned long long>(limit))) {            \
      printf("TSDD_DEBUG_BOUNDS: %s:%d: %s = %llu is not below %s = %llu (block %u,%u thread %u)\n",    \
             __FILE__, __LINE__, #index, static_cast<unsigned long long>(index), #limit,                 \
             static_cast<unsigned long long>(limit), blockIdx.x, blockIdx.y, threadIdx.x);               \
      __trap();                                                                                          \
    }                                                                                                    \
  } while (0)
#else
#define TSDD_BOUND(index, limit) do { } while (0)
#endif

namespace tsdd_b200 {

constexpr uint32_t kInfBits = 0x7F800000u;  // +inf as float bits
// nn slot of a row nobody has measured yet: (+inf, no neighbour)
constexpr uint64_t kNnUnset = (static_cast<uint64_t>(kInfBits) << 32) | 0xFFFFFFFFull;

// Squared distances are >= 0, so their float bits order like the floats.
//
// nn key  : (bits(d^2) << 32) | neighbour row   -> integer MIN = (smaller distance, then smaller row)
// best key: (bits(d^2) << 32) | ~candidate row  -> integer MAX = (greater distance, then smaller row)
//           the rule of the reference's deterministic merges (discovery.cpp:158-165, 328-340).
__host__ __device__ __forceinline__ uint64_t nn_key(uint32_t d2_bits, uint32_t row) {
  return (static_cast<uint64_t>(d2_bits) << 32) | row;
}
__host__ __device__ __forceinline__ uint64_t best_key(uint32_t d2_bits, uint32_t row) {
  return (static_cast<uint64_t>(d2_bits) << 32) | (0xFFFFFFFFu - row);
}
__host__ __device__ __forceinline__ uint32_t key_bits(uint64_t key) {
  return static_cast<uint32_t>(key >> 32);
}
__host__ __device__ __forceinline__ uint32_t best_key_row(uint64_t key) {
  return 0xFFFFFFFFu - static_cast<uint32_t>(key & 0xFFFFFFFFull);
}

// A row whose nn upper bound cannot beat the best-so-far any more is dead: the
// HOTSAX discard `d < bsf` (discovery.cpp:58,70).  The kernels compute in
// float32 and the reference in float64, so the test keeps a safety factor
// (`margin` = 1 + delta, delta a bound of the float32 rounding of a distance):
// a row is discarded only if its bound is below the best-so-far even after the
// factor.  Rows inside the band stay alive, finish their scan, and the winner
// among them is decided in float64 (k_exact_nn): float32 noise can then cost
// work, never the answer.  A bound of exactly 0 is dead at once: nothing beats
// the initial best-so-far 0 with it (discovery.cpp:90-93, hpp:45 `sq > best`).
// `margin_abs` is 0 until a search has used the dot-product form of the distance
// (search_kernels.cu: k_scan_tiles_ws<.., kDot>), whose rounding error is absolute
// (cancellation in |a|^2 + |b|^2 - 2 a.b), not relative; from then on the band is
// widened by twice that error bound.
// `margin_q` covers what neither of the two does: the float32 QUANTISATION of the z-normalised
// rows themselves.  Rounding every element of two rows of norm sqrt(n) to float32 moves their
// squared distance d^2 by up to d * sqrt(n) * 2^-22 — an error whose relative size grows as 1 / d,
// so on clean periodic data (d^2 ~ 1e-5) it exceeds any fixed relative band.  Both the bound
// and the best-so-far carry it and the bound is below the best-so-far when the test matters, so
// the band is widened by margin_q * sqrt(best), margin_q = 1.25 * sqrt(n) * 2^-21 (engine.cu).
__device__ __forceinline__ bool dead_bound(float d2, uint64_t best, float margin, float margin_abs, float margin_q) {
  const float b = __uint_as_float(key_bits(best));
  return d2 == 0.f || fmaf(d2, margin, fmaf(margin_q, sqrtf(b), margin_abs)) < b;
}
__device__ __forceinline__ bool is_dead(uint64_t nn, uint64_t best, float margin, float margin_abs, float margin_q) {
  return dead_bound(__uint_as_float(key_bits(nn)), best, margin, margin_abs, margin_q);
}

// Whether a segment-mean lower bound (already scaled to a squared distance) rules a threshold
// out.  The means are float32 roundings of float64 values of magnitude <= 4, so the bound is off
// by up to lb_q * sqrt(thr) + lb_q^2 with lb_q = 4e-6 * sqrt(columns per segment) (engine.cu) —
// again an error that a relative slack (0.1 %) alone does not cover when thr is tiny.
__device__ __forceinline__ bool lb_rules_out(float lb_scaled, float thr, float lb_q) {
  return lb_scaled > fmaf(thr, 1.001f, fmaf(lb_q, sqrtf(fmaxf(thr, 0.f)), lb_q * lb_q));
}

__device__ __forceinline__ unsigned long long* as_ull(uint64_t* p) {
  return reinterpret_cast<unsigned long long*>(p);
}

// Search-stage counters, one instance in device memory per context.
struct DeviceCounters {
  unsigned long long calls;      // pair distances started for live candidates
  unsigned long long abandoned;  // of those, cut short by an abandoned tile
  unsigned long long terms;      // (x-y)^2 terms accumulated by any scan kernel
  unsigned long long tile_terms; // ... by the tiled kernel only
  unsigned long long dot_terms;  // of tile_terms, those computed as one FFMA (dot-product form)
  unsigned long long tiles;      // candidate-tile x neighbour-tile pairs started by the tiled kernel
  unsigned long long tile_live;  // live candidates summed over those tiles (128 per tile = dense)
  unsigned long long lb_skipped; // (candidate, neighbour tile) pairs the lower-bound filter ruled out
  // of tile_terms, the terms of pairs (live candidate, existing neighbour row) in real columns
  // (t < n): what is left after taking out the dead or empty candidate slots of a tile, the slots
  // past the last row, and the zero padding of the row stride.  (Self-match pairs inside a tile,
  // at most (2n - 1) / N of all pairs, are not taken out.)
  unsigned long long useful_terms;
  unsigned long long propagated;  // pair distances measured by the time-topology step (k_propagate)
  unsigned long long tc_terms;    // of dot_terms, those computed on the tensor cores (tc_kernels.cu: 3 MMA multiply-adds a term)
  // of calls, those of covering scans that ran on the tensor cores in a search that is NOT in the dot form
  // (engine.cu: tail_now) — they never abandon and say nothing about whether abandoning pays
  unsigned long long tail_calls;
};

}  // namespace tsdd_b200
