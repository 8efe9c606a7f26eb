// Host-callable launchers of the sm_100a kernels (prep_kernels.cu,
// search_kernels.cu, probe_kernels.cu).  Every launcher enqueues on `stream`
// and returns the number of kernels it launched; errors surface through
// cudaGetLastError() in the engine.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace tsdd_b200 {

constexpr int kLbSegments = 16;    // segment means per row for the lower-bound tile filter
constexpr uint32_t kLbBoxRows = 16; // rows per bounding box of segment means
constexpr int kTileRows = 128;     // candidates per tile == neighbours per tile
#ifndef TSDD_SCAN_CHUNK
#define TSDD_SCAN_CHUNK 64
#endif
#ifndef TSDD_SCAN_STAGES
#define TSDD_SCAN_STAGES 2
#endif
constexpr int kChunk = TSDD_SCAN_CHUNK;  // columns per pipeline stage (kChunk*4 bytes of every row)
constexpr uint32_t kRowAlign = kChunk;   // row stride is a multiple of this many floats

// ------------------------------------------------------------------ preparation
// d_first_bad (may be null): receives the smallest index of a non-finite sample, ~0 if none.
int launch_widen_series(const float* d_in, double* d_out, size_t m, uint32_t* d_first_bad, cudaStream_t stream);

// Per-window mean / 1/sigma (float64), PAA -> SAX -> 0-based word hash.
// paa_out / sax_out may be null (kept only for parity tests).  tol_scale: the aligned form's distance-to-breakpoint
// tolerance is multiplied by it (tests inflate it to force the exact path; 0 = exact path only).
int launch_window_encode(const double* d_series, uint32_t rows, uint32_t n, uint32_t word_len,
                         uint32_t alphabet, double* d_mean, double* d_inv_sigma, uint32_t* d_hash0,
                         double* d_paa, uint32_t* d_sax, cudaStream_t stream, double tol_scale = 1.0);

// float32 z-normalised matrix, rows x stride, padding columns zero; and, when d_seg_means is
// given, the kLbSegments segment means of every row (from the same staged samples).
int launch_build_rows(const double* d_series, const double* d_mean, const double* d_inv_sigma,
                      uint32_t rows, uint32_t n, uint32_t stride, float* d_rows, float* d_seg_means,
                      cudaStream_t stream, float* d_norms = nullptr);  // d_norms: rows + 1 squared norms of the float32 rows

// Bounding boxes of the rows' segment means per kLbBoxRows rows:
// [ceil(rows / kLbBoxRows) x 2 x kLbSegments] (minimum then maximum per segment).
int launch_segment_boxes(const float* d_means, uint32_t rows, float* d_boxes, cudaStream_t stream);

// Stable LSD radix sort of (key, value) pairs on bits [0, key_bits).  Result is
// left in (*keys, *vals); the alt buffers are scratch.  `hist` needs
// radix_sort_scratch_words(count) uint32 words.
size_t radix_sort_scratch_words(uint32_t count);
int launch_radix_sort_pairs(uint32_t** keys, uint32_t** vals, uint32_t** keys_alt,
                            uint32_t** vals_alt, uint32_t count, int key_bits, uint32_t* d_hist,
                            uint32_t* d_scan_scratch, cudaStream_t stream);

// Exclusive prefix sum of uint32; d_out may alias d_in.  Scratch needs
// scan_scratch_words(count) words.
size_t scan_scratch_words(uint32_t count);
int launch_exclusive_scan(const uint32_t* d_in, uint32_t* d_out, uint32_t count,
                          uint32_t* d_scratch, cudaStream_t stream);

int launch_iota(uint32_t* d_out, uint32_t count, cudaStream_t stream);

// Run-length histogram of the sorted hashes: bucket offsets, per-slot bucket
// id, per-row frequency.  d_scalars[0] = number of buckets.
int launch_bucket_index(const uint32_t* d_sorted_hash, const uint32_t* d_sorted_row, uint32_t rows,
                        uint32_t* d_head_scan, uint32_t* d_slot_bucket, uint32_t* d_offsets,
                        uint32_t* d_freq, uint32_t* d_scalars, uint32_t* d_scan_scratch,
                        cudaStream_t stream);

// d_scalars[1] = number of leading entries of the sorted frequencies equal to the minimum.
// scalars[2] += slots whose successor in the hash-sorted order is the same word's next row (runs of consecutive rows)
int launch_count_runs(const uint32_t* d_sorted_hash, const uint32_t* d_sorted_row, uint32_t rows, uint32_t* d_scalars,
                      cudaStream_t stream);
int launch_count_min_freq(const uint32_t* d_sorted_freq, uint32_t rows, uint32_t* d_scalars,
                          cudaStream_t stream);

// ------------------------------------------------------------------ search
struct SearchState {
  const float* rows;        // rows_padded x stride
  uint32_t n_rows;          // N
  uint32_t n;               // subsequence length
  uint32_t stride;          // floats per row
  uint64_t* nn;             // N nn keys (bits(d^2) << 32 | neighbour)
  uint8_t* exact;           // N
  uint8_t* excluded;        // N
  uint64_t* best;           // 1 best key
  DeviceCounters* counters;
  float margin;             // 1 + delta of the discard test (common.cuh: dead_bound)
  float margin_abs;         // 0, or twice the absolute error bound of dot-form distances once a search uses them
  float margin_q;           // x sqrt(best-so-far): the float32 quantisation of the rows (common.cuh: dead_bound)
  const float* row_norms;   // N + 1 squared norms of the float32 rows (dot form), or nullptr
  const float* rows_sorted; // the matrix in the hash-sorted order (tensor-map loads of window tiles), or nullptr
  const float* lb_means;    // N x kLbSegments segment means, or nullptr: no tile filter
  const float* lb_boxes;    // their bounding boxes per kLbBoxRows rows
  float lb_scale;           // columns per segment (stride / kLbSegments)
  float lb_q;               // absolute rounding slack of the float32 segment means (common.cuh: lb_rules_out)
};

int launch_reset_search(SearchState s, cudaStream_t stream);

// nn[i] = min(nn[i], peer[0][i], peer[1][i], ...): the per-batch min-reduction of the bounds
// between the ranks of one process, read straight from the peers' device memory (NVLink P2P).
constexpr int kMaxPeers = 15;
struct PeerPointers {
  const uint64_t* ptr[kMaxPeers];
  int count;
};
int launch_min_from_peers(uint64_t* d_nn, PeerPointers peers, uint32_t rows, cudaStream_t stream);

// Same-word neighbours first (the HOTSAX inner heuristic, discovery.cpp:51-63):
// every row is measured against up to `mates` rows of its own bucket.
// d_series_f32: the float32 originals when the series arrived in that type (else nullptr): same values, half the bytes.
int launch_bucket_mates(SearchState s, const double* d_series, const float* d_series_f32, const double* d_mean,
                        const double* d_inv_sigma, const uint32_t* d_sorted_row, const uint32_t* d_slot_bucket,
                        const uint32_t* d_offsets, int mates, uint32_t run_pairs, uint32_t world, uint32_t rank,
                        cudaStream_t stream, int form = -1);  // run_pairs: launch_count_runs; form: -1 by the input (runs / float32 / float64), 0 float64, 1 float32, 2 runs

// Time topology: every live batch candidate c tries the matches of its neighbours in time,
// shifted along (row c + delta knows neighbour j  ->  measure (c, j - delta)); up to `tries`
// pair distances per candidate, each lowering the bounds of both rows.
int launch_propagate(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel, uint32_t live_upper_bound,
                     int tries, cudaStream_t stream);

// Outer-loop batch selection: the next `batch` live entries of the rarity
// order at or after `cursor` that belong to this rank.  d_sel[0] = count,
// d_sel[1] = next cursor.
int launch_select_batch(SearchState s, const uint32_t* d_order, uint32_t cursor, uint32_t batch,
                        uint32_t world, uint32_t rank, bool pruning, uint32_t* d_flags,
                        uint32_t* d_scan_scratch, uint32_t* d_batch_rows, uint32_t* d_sel,
                        cudaStream_t stream);

// Drops dead candidates from the batch list (stable); rows and hash-order slots move
// together; count lives in d_sel[0].
int launch_compact_batch(SearchState s, uint32_t* d_batch_rows, uint32_t* d_batch_slots, uint32_t* d_rows_alt,
                         uint32_t* d_slots_alt, bool pruning, uint32_t* d_sel, uint32_t live_upper_bound,
                         uint32_t* d_scratch, cudaStream_t stream);

// slot_of_row = inverse permutation of the hash-sorted row list.
int launch_invert_order(const uint32_t* d_sorted_row, uint32_t rows, uint32_t* d_slot_of_row,
                        cudaStream_t stream);
// keys[i] = slot_of_row[batch_rows[i]] for i < sel[0].
int launch_batch_slots(const uint32_t* d_batch_rows, const uint32_t* d_sel, const uint32_t* d_slot_of_row,
                       uint32_t capacity, uint32_t* d_keys, cudaStream_t stream);

// Copies the batch's matrix rows into a dense [capacity_padded x stride] buffer.
// tma_layout 1: the row order inside each 128-row tile that the tensor-map variant of the
// warp-specialised kernel reads (search_kernels.cu: tma_row_of_candidate); 2: 256-row tiles of
// pairwise interleaved rows for its 16 x 8 variant (tma16_pair_of_candidate); capacity_padded is
// then a multiple of 256.
int launch_gather_rows(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel,
                       uint32_t capacity_padded, int tma_layout, float* d_batch_matrix, cudaStream_t stream);

// Kernel-selection options of one context (tsdd_cuda_set_option); per-context state, so that
// contexts on concurrent host threads never see one another's choices.
struct ScanConfig {
  bool packed = true;        // f32x2 arithmetic
  bool wide_tile = false;    // 128 x 128 tiles, one CTA per SM, instead of 128 x 64, two
  int variant = 0;           // 0: per launch; 1: k_scan_tiles everywhere; 2: k_scan_tiles_ws everywhere
  bool tensor_map = true;    // the warp-specialised kernel loads tiles as TMA boxes where it can
  bool filter_in_ws = false; // covering scans with the lower-bound filter on the ws kernel's producer warpgroup
  bool tile16 = true;        // dot form on 256-candidate tiles (k_scan_tiles_ws16)
  bool tensor_cores = false; // dot form on the tensor cores (k_scan_tiles_tc) while a batch fills 128-candidate tiles
};

// Which kernel a launch uses.  Computed ONCE per segment (choose_scan_kernel) and handed to both
// k_gather_rows (the candidate layout depends on `tma` / `tile16`) and launch_scan_tiles.
struct ScanChoice {
  bool lb;   // k_scan_tiles with the lower-bound tile filter
  bool ws;   // the warp-specialised kernel
  bool tma;  // ... fed by tensor-map box loads (covering scans)
  bool dot;  // ... in the dot-product form
  bool tile16;  // ... on 256-candidate tiles, 16 x 8 pairs per thread (k_scan_tiles_ws16)
  bool tc;      // ... on the tensor cores (tc_kernels.cu: k_scan_tiles_tc)
  bool packed, wide;  // copied from the ScanConfig
};
ScanChoice choose_scan_kernel(const ScanConfig& cfg, const SearchState& s, uint32_t live_upper_bound, bool window,
                              bool pruning, bool dot_form);

// The tiled early-abandoning distance kernel: batch candidates x neighbour units
// [k_begin, k_end), one unit = 128 rows.  d_nbr_index == nullptr: unit k holds the rows of
// unit (k + rotation) mod T of the matrix (the covering scan).  Otherwise (window mode)
// unit k holds 128 slots of d_nbr_index (the hash-sorted row list) around the candidate
// tile's own slot, alternating outwards.  live_upper_bound >= the live batch size in
// d_sel[0]; it sizes the grid and picks the tile shape.  *error receives the message of a
// launch that could not be made (else nullptr).
int launch_scan_tiles(const ScanChoice& choice, SearchState s, const float* d_batch_matrix,
                      const uint32_t* d_batch_rows, const uint32_t* d_batch_slots, const uint32_t* d_sel,
                      uint32_t live_upper_bound, const uint32_t* d_nbr_index, uint32_t k_begin, uint32_t k_end,
                      uint32_t rotation, bool pruning, bool symmetric, cudaStream_t stream, const char** error);

// ---- tensor-core tile kernel (tc_kernels.cu; experiment behind the option "tensor_cores")
struct TcOperands {
  const float *batch_hi, *batch_lo;    // the batch's rows split into tf32 parts (launch_gather_rows_split)
  const float *rows_hi, *rows_lo;      // the matrix, split (launch_split_tf32)
  const float *sorted_hi, *sorted_lo;  // its hash-sorted copy, split (window tiles)
  uint64_t rows_padded;                // rows of each of the four neighbour arrays
  bool half;                           // the parts are fp16 (kind::f16, 22 bits between them) instead of tf32 (kind::tf32, 21 bits)
  uint32_t* work;                      // one word of device memory: the launch's work-item counter
  bool tail;                           // a covering scan of a search that is not in the dot form (counters only)
  bool convert;                        // no split copy of the matrix: the kernel makes the neighbours' fp16 parts from SearchState::rows
};
int launch_split_rows(const float* d_in, size_t floats, bool half, float* d_hi, float* d_lo, cudaStream_t stream);
// ... row by row, with the rows' squared norms (the first n_norms of them) as a by-product
int launch_split_rows_norms(const float* d_in, uint32_t n_rows, uint32_t stride, bool half, float* d_hi, float* d_lo,
                            float* d_norms, uint32_t n_norms, cudaStream_t stream);
int launch_gather_rows_split(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel, uint32_t capacity_padded,
                             bool half, float* d_hi, float* d_lo, cudaStream_t stream);
int launch_scan_tiles_tc(SearchState s, const TcOperands& op, const uint32_t* d_batch_rows, const uint32_t* d_batch_slots,
                         const uint32_t* d_sel, uint32_t live_upper_bound, const uint32_t* d_nbr_index, uint32_t k_begin,
                         uint32_t k_end, bool pruning, bool symmetric, cudaStream_t stream, const char** error);
// float32 (elem_bytes 4) or fp16 (2) matrix [n_rows x stride elements] as a tensor map with boxes of box_rows x box_cols, 128-byte swizzle
// (box_cols * 4 = 128) or the 64-byte one (box_cols * 4 = 64); false when the driver lacks cuTensorMapEncodeTiled.  `map` is a CUtensorMap.
bool make_row_map_boxed(void* map, const void* base, uint64_t n_rows, uint64_t stride, uint32_t box_cols, uint32_t box_rows,
                        uint32_t elem_bytes = 4);

// Squared norms of the float32 rows (rows 0 .. n_rows; row n_rows is the zero row), for the
// dot-product form d^2 = |a|^2 + |b|^2 - 2 a.b of the warp-specialised tile kernel.
int launch_permute_rows(const float* d_rows, const uint32_t* d_sorted_row, uint32_t n_rows, uint32_t rows_padded,
                        uint32_t stride, float* d_out, cudaStream_t stream);
int launch_row_norms(const float* d_rows, uint32_t n_rows_plus_one, uint32_t stride, float* d_norms,
                     cudaStream_t stream);

// Survivors of a complete scan are exact; each raises the best-so-far.
int launch_finalize_batch(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel,
                          uint32_t capacity, bool pruning, cudaStream_t stream);

// A valid best-so-far before the first scan: the greatest lower bound of a nearest-neighbour
// distance among the first seed_rows entries of the rarity order, from the segment-mean
// boxes (needs s.lb_means / s.lb_boxes).  d_seed_lb: seed_rows words of scratch.
int launch_seed_lower_bound(SearchState s, const uint32_t* d_order, uint32_t seed_rows, uint32_t* d_seed_lb,
                            cudaStream_t stream);
// best = max over exact, allowed rows (start of a top-k pass).
int launch_seed_best(SearchState s, cudaStream_t stream);
int launch_exclude_zone(SearchState s, uint32_t row, cudaStream_t stream);

// Finalists of a pass: exact, allowed rows whose float32 nn is within the safety band of
// the best-so-far.  d_list[0 .. min(count, cap)) = rows; d_count[0] = how many qualify.
int launch_collect_finalists(SearchState s, uint32_t* d_list, uint32_t cap, uint32_t* d_count,
                             cudaStream_t stream);

// d_keys[i] = nn key of row d_list[i].
int launch_gather_keys(SearchState s, const uint32_t* d_list, uint32_t count, uint64_t* d_keys, cudaStream_t stream);

// Exact float64 nearest-neighbour distance (squared) of one row over ALL non-self rows,
// straight from the series: d_out_bits[0] = bits of the minimum (must be preset to the
// bits of an upper bound, e.g. +inf), with early abandoning against it.
int launch_exact_nn(const double* d_series, const double* d_mean, const double* d_inv_sigma,
                    uint32_t n_rows, uint32_t n, uint32_t row, double* d_zrow, const float* d_lb_means, float lb_scale,
                    float lb_q, unsigned long long* d_out_bits, cudaStream_t stream);
// ... for up to 4 finalists in one launch (d_zrow: count x n doubles; d_out_bits: count start bounds in, results out)
int launch_exact_nn_group(const double* d_series, const double* d_mean, const double* d_inv_sigma, uint32_t n_rows,
                          uint32_t n, const uint32_t* rows, uint32_t count, double* d_zrow, const float* d_lb_means,
                          float lb_scale, float lb_q, unsigned long long* d_out_bits, cudaStream_t stream);

// ------------------------------------------------------------------ probes
int launch_fp32_probe(int which, float* d_sink, int blocks, int iters, cudaStream_t stream);
double fp32_probe_ops(int which, int blocks, int iters);

}  // namespace tsdd_b200
