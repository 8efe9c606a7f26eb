/* tsdd_cuda.h — C ABI of the B200 discord-search engine (libtsdd_cuda.so).
 *
 * This is the drop-in boundary for the ONE hot path of the reference
 * (/root/reference/proj): preparation + PhiDD/HOTSAX search, entered in the
 * reference through
 *     tsdd::run_discovery   include/tsdd/pipeline.hpp:37   (src/pipeline.cpp:53-93)
 *     tsdd::phidd_discord   include/tsdd/discovery.hpp:86  (src/discovery.cpp:360-373)
 * The reference has no FFI of its own; the C++ shim in include/tsdd/ (same
 * type and function names as the reference headers) binds these entry points
 * and re-throws the reference's exception types from the return codes.
 *
 * Plain pointers and sizes only; no exceptions cross this boundary; every
 * function returns one of the TSDD_* codes below and leaves a message for
 * tsdd_cuda_last_error().  All compute runs in hand-written sm_100a kernels;
 * there is no CPU fallback: without a CUDA device tsdd_cuda_create fails with
 * TSDD_ERR_RUNTIME.
 *
 * Threading: one call at a time per context; distinct contexts
 * may be used concurrently.  Positions are 1-based (discovery.hpp:21).
 */
#ifndef TSDD_CUDA_H
#define TSDD_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  2/3 are the reference CLI's exit codes (tools/tsdd.cpp:212-223). */
#define TSDD_OK 0
#define TSDD_ERR_PARAMETER 2  /* -> tsdd::ParameterError        (errors.hpp:10-13) */
#define TSDD_ERR_VALIDATION 3 /* -> tsdd::ValidationError       (errors.hpp:16-19) */
#define TSDD_ERR_INFEASIBLE 4 /* -> tsdd::InfeasibleInputError  (errors.hpp:22-25) */
#define TSDD_ERR_RUNTIME 5    /* CUDA / NCCL failure -> std::runtime_error */

typedef struct tsdd_cuda_ctx tsdd_cuda_ctx;

/* Counters and timings of the last prepare + search on a context.
 * calls / abandoned keep the reference's meaning (series.hpp:68-74):
 * distance evaluations started / cut short.  terms = (x-y)^2 terms actually
 * accumulated by the scan kernels (the FP32 roofline numerator).            */
typedef struct tsdd_cuda_stats {
  uint64_t rows;           /* N = m - n + 1 */
  uint64_t calls;          /* pair distances started (tile pairs with |i-j| >= n) */
  uint64_t abandoned;      /* of which stopped before the last column */
  uint64_t terms;          /* accumulated (x-y)^2 terms, all scan kernels */
  uint64_t buckets;        /* distinct SAX words present */
  uint64_t min_freq_candidates; /* size of the reference's candidate set (index.cpp:66-79) */
  uint64_t batches;        /* outer-loop batches run */
  uint64_t scanned_candidates; /* candidates that entered a full scan */
  uint64_t kernel_launches;    /* kernels launched by prepare + search */
  double prep_ms;          /* device time of the preparation stage (CUDA events) */
  double search_ms;        /* device time of the search stage (CUDA events) */
  double scan_kernel_ms;   /* device time inside the tiled distance kernel only */
  double h2d_ms;           /* series upload, when prepare was given a host pointer */
  uint64_t scan_kernel_launches;
  uint64_t scan_kernel_terms; /* terms accumulated by the tiled distance kernel only */
  double encode_ms;        /* preparation: window statistics + PAA/SAX/hash kernel */
  double build_rows_ms;    /* preparation: float32 matrix build (HBM write-bound) */
  double index_ms;         /* preparation: lower-bound summaries, radix sorts, run-length histogram, rarity order */
  uint64_t tiles;          /* candidate-tile x neighbour-tile pairs the tile kernel started */
  uint64_t tile_live_candidates; /* live candidates summed over them (128 per tile = dense tiles) */
  uint64_t lb_skipped;     /* (candidate, neighbour tile) pairs ruled out by the lower-bound filter */
  uint64_t scan_kernel_ws_launches; /* of scan_kernel_launches, those of the warp-specialised kernel */
  uint64_t scan_kernel_dot_launches; /* of those, launches of its dot-product form (one FFMA per term) */
  uint64_t scan_kernel_dot_terms;   /* of scan_kernel_terms, those computed as one FFMA */
  uint64_t finalists;      /* rows settled in float64 at the end of the passes (near-ties of the float32 search) */
  uint64_t exact_reruns;   /* of those, measured again from +inf because the float32 start bound was too low */
  uint64_t useful_terms;   /* of scan_kernel_terms: terms of pairs that were live, non-self and not padding */
  uint64_t propagated;     /* pair distances measured by the time-topology step (option "propagate") */
  uint64_t scan_kernel_tc_launches; /* of scan_kernel_dot_launches, those of the tensor-core tile kernel (dot_form 3 .. 6) */
  uint64_t scan_kernel_tc_terms;    /* of scan_kernel_dot_terms, those computed there (three MMA multiply-adds per term) */
  double scan_kernel_tc_ms;         /* of scan_kernel_ms, the device time inside the tensor-core tile kernel */
  uint64_t tail_restarts;           /* searches started over because the first batch's tensor-core tails were not warranted */
} tsdd_cuda_stats;

/* ---- lifetime ------------------------------------------------------------ */

/* Binds a context to one CUDA device (one context per GPU / per rank). */
int tsdd_cuda_create(tsdd_cuda_ctx** out, int device);
void tsdd_cuda_destroy(tsdd_cuda_ctx* ctx);

/* Message of the last failure on this context (ctx == NULL: last failure of
 * tsdd_cuda_create on this thread).  Never NULL.                            */
const char* tsdd_cuda_last_error(const tsdd_cuda_ctx* ctx);

/* Runs all further work of the context on the caller's CUDA stream (a
 * cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream) so that the
 * caller's events bracket it; NULL restores the context's own stream.      */
int tsdd_cuda_set_stream(tsdd_cuda_ctx* ctx, void* cuda_stream);

/* Tunables, by name: "batch" (candidates per outer-loop batch), "first_batch"
 * / "batch_growth" (size of the first batch of the first pass and the factor by
 * which batches grow up to "batch"), "first_range" / "growth"
 * / "rounds" (neighbour rows are visited in ranges: first_range rows, then each
 * range growth times larger, at most rounds of them; dead candidates are
 * dropped between ranges), "window_rounds" / "window_first" / "window_growth"
 * (before that covering scan, each candidate tile visits its own SAX word's
 * neighbourhood in the hash-sorted order: window_first slots, growing), "bucket_mates" (same-word
 * neighbours tried per row before the scans), "propagate" (time topology: at the start of a batch
 * and after its window rounds every live candidate c measures up to this many pairs (c, j - delta)
 * suggested by rows c + delta, |delta| <= 16, that already know a neighbour j; 0 = off), "rescore" (0/1: decide each pass
 * among the near-tied finalists by their exact float64 nn distance),
 * "margin_delta" (relative safety band of the float32 discard test; negative = from n),
 * "margin_q" (its part proportional to sqrt(best-so-far), for the float32 quantisation of the
 * rows; negative = from n), "finalist_cap" (room of the first collection of near-tied
 * finalists; a pass with more collects again and still settles all of them), "symmetric" (0/1: completed tiles
 * also lower the neighbours' bounds), "packed" (0/1: f32x2 arithmetic),
 * "wide_tile" (0/1: 128 x 128 tiles, one CTA per SM, instead of 128 x 64, two),
 * "kernel" (0: per launch; 1: the cp.async tile kernel everywhere; 2: the
 * warp-specialised cp.async.bulk + mbarrier kernel everywhere), "rotate" (0/1), "share_bounds" (0/1), "lower_bound" (0/1: in the covering scan a
 * candidate skips a neighbour tile whose segment-mean boxes are provably
 * further away than its threshold), "dot_form" (the warp-specialised kernel
 * computes d^2 as |a|^2 + |b|^2 - 2 a.b, one FFMA per term, with the discard band widened by
 * its absolute error bound: 0 never; 1 once a search has found that tiles are not abandoned
 * early anyway and the best-so-far dwarfs the bound; 2 from the first launch; 3 / 4 and 5 / 6: as 1 / 2,
 * with the dot-form tiles of batches that fill 128 candidates on the TENSOR CORES — tcgen05.mma on
 * rows split into two tf32 parts (3 / 4, kind::tf32) or two fp16 parts (5 / 6, kind::f16), three MMAs
 * per k-step, accumulators in tensor memory; 5 is the default),
 * "tc_tail" (0/1, or the greatest number of candidates: the later ranges of a covering scan of a search that
 * is NOT in the dot form move to the tensor cores — with the lower-bound filter — once the measured
 * CUDA-core time per tile says that is cheaper; default 1, at most 1,024 candidates),
 * "tc_growth" / "tc_window_rounds" / "tc_window_growth" (the ranges and window rounds of a dot-form batch on the
 * tensor cores: 2.0 / 5 / 2.5 — fewer, wider launches than on the CUDA cores),
 * "mates_form" (-1: the same-word step picks its kernel by the input; 0 float64, 1 float32, 2 along runs of consecutive rows),
 * "tc_convert" (0/1: such a tail reads the float32 matrix and makes the neighbours' fp16 parts inside the kernel,
 * instead of building split copies of the matrix first; default 1),
 * "tc_tail_first" (0/1: the first batch of a search may do so on trust, before there is a best-so-far to size the
 * band against; should its result not dwarf the band, the search starts over without the tails),
 * "encode_tol_scale" (x the window encoder's distance-to-breakpoint tolerance; 0: its exact path only),
 * "tensor_map" (0/1: the warp-specialised kernel loads the tiles of covering scans — and, in
 * the dot-product form, of window rounds, from a copy of the matrix kept in the hash-sorted
 * order — as cp.async.bulk.tensor boxes instead of one bulk copy per row),
 * "dot_window_rounds" (window rounds of a dot-form batch whose window tiles load that way),
 * "dot_window_growth" (growth of those rounds, at most "window_growth"),
 * "dot_growth" (range growth of a dot-form batch, at most "growth": without abandoning inside
 * tiles a dead candidate costs full price until the next compaction),
 * "dot_tile16" (0/1: the dot-product form runs on 256-candidate tiles with 16 x 8 pairs per
 * thread — candidate rows stored pairwise interleaved, one FFMA2 per two candidates — while a
 * batch still fills such tiles; default 1),
 * "filter_in_ws" (0/1: covering scans with the lower-bound filter run on the warp-specialised
 * kernel, the filter on the four warps of its producer warpgroup, instead of on the cp.async
 * tile kernel; measured slower on the BASELINE workloads, off by default),
 * "seed_rows" (before the first scan, the best-so-far is seeded with the greatest LOWER bound of
 * a nearest-neighbour distance among this many first entries of the rarity order, from the
 * segment-mean boxes; 0 = start from zero as the reference does),
 * "shard_prep" (0/1, default 1: ranks joined by an NCCL communicator or an in-process group
 * each compute the window statistics and hashes of ONE slice of the rows and all-gather them),
 * "time_kernels" (0/1: CUDA events around every tile-kernel launch).
 * Unknown name -> TSDD_ERR_PARAMETER.  None of them changes the result.     */
int tsdd_cuda_set_option(tsdd_cuda_ctx* ctx, const char* name, double value);

/* ---- preparation stage (replaces pipeline.cpp:60-69) --------------------- */

/* check_config alone (pipeline.cpp:21-49): the validation that prepare runs
 * first, usable without a device.  Writes the message the matching reference
 * exception would carry into `message` (may be NULL).                       */
int tsdd_cuda_check_config_f32(const float* series, size_t m, size_t n, size_t word_len,
                               size_t alphabet, char* message, size_t message_bytes);
int tsdd_cuda_check_config_f64(const double* series, size_t m, size_t n, size_t word_len,
                               size_t alphabet, char* message, size_t message_bytes);

/* Validates exactly as check_config does (pipeline.cpp:21-49: finite values,
 * 1 <= n <= m, 1 <= word_len <= n, alphabet in 2..10, N >= n+1), except that
 * the dictionary guard is 2^32 words instead of 2^24 (sax.hpp:80): the device
 * index is sort-based and never allocates |A|^w entries.  Then, on the device:
 * per-window mean / sigma in float64, the z-normalised subsequence matrix in
 * float32 (series.cpp:46-74), PAA -> SAX -> word hash (sax.cpp:63-132), and
 * the bucket / frequency / rarity index (index.cpp:12-109) by radix sort and
 * run-length histogram.  `series` is a HOST pointer.                        */
int tsdd_cuda_prepare_f32(tsdd_cuda_ctx* ctx, const float* series, size_t m, size_t n,
                          size_t word_len, size_t alphabet);
int tsdd_cuda_prepare_f64(tsdd_cuda_ctx* ctx, const double* series, size_t m, size_t n,
                          size_t word_len, size_t alphabet);
/* Same, with the float32 series already resident in device memory on the
 * context's device (no host<->device copy inside).                          */
int tsdd_cuda_prepare_device_f32(tsdd_cuda_ctx* ctx, const float* d_series, size_t m, size_t n,
                                 size_t word_len, size_t alphabet);

/* Rebuilds only what depends on the SAX shape — window encoding (sax.cpp:82-132) and
 * DiscordIndexes::build (index.cpp:101-109) — on a prepared context, keeping the resident
 * series and subsequence matrix.  This is what lets the C++ mirrors in
 * include/tsdd/cuda_engine.hpp follow the reference's two-step preparation
 * (SubsequenceMatrix::build, then DiscordIndexes::build).                    */
int tsdd_cuda_reindex(tsdd_cuda_ctx* ctx, size_t word_len, size_t alphabet);

/* ---- search stage (replaces phidd_discord, discovery.cpp:360-373) -------- */

#define TSDD_SEARCH_DISABLE_PRUNING 1u /* DiscoveryOptions::disable_pruning (discovery.hpp:31) */

/* Top-k discords of the prepared series.  k = 1 is the reference's search.
 * For k > 1, discord r is the arg-max of the nearest-neighbour distance over
 * positions at least n away from every earlier discord.
 * positions[k] are 1-based; distances[k] are Euclidean (sqrt taken once,
 * discovery.cpp:88-98).  Ties on the distance go to the smaller position
 * (discovery.cpp:158-165).  Nothing beat 0 -> position 1, distance 0.
 * With several ranks (tsdd_cuda_comm_init / tsdd_cuda_set_exchange) every
 * rank must call this with the same arguments; all ranks return the same
 * answer.                                                                   */
int tsdd_cuda_search(tsdd_cuda_ctx* ctx, int k, unsigned flags, uint64_t* positions,
                     double* distances);

int tsdd_cuda_get_stats(const tsdd_cuda_ctx* ctx, tsdd_cuda_stats* out);

/* ---- parity access to the prepared arrays (tests only) ------------------- */

#define TSDD_FETCH_ROWS 1       /* float  [N * stride]  z-normalised matrix (series.hpp:53)   */
#define TSDD_FETCH_MEAN 2       /* double [N]           window means                          */
#define TSDD_FETCH_INV_SIGMA 3  /* double [N]           1/sigma, 0 for flat windows           */
#define TSDD_FETCH_PAA 4        /* double [N * w]       segment means (sax.hpp:37)            */
#define TSDD_FETCH_SAX 5        /* uint32 [N * w]       symbols 1..|A| (sax.hpp:47)           */
#define TSDD_FETCH_HASH 6       /* uint64 [N]           1-based word hash (index.hpp:61)      */
#define TSDD_FETCH_FREQ 7       /* uint32 [N]           bucket size of each row (index.hpp:15) */
#define TSDD_FETCH_BUCKETS 8    /* uint64 [N]           1-based positions, bucket after bucket in
                                                         ascending hash order (index.hpp:29)   */
#define TSDD_FETCH_ORDER 9      /* uint64 [N]           1-based positions in rarity order      */
#define TSDD_FETCH_CANDIDATES 10 /* uint64 [min_freq_candidates] (index.hpp:20-22)            */
#define TSDD_FETCH_NN_SQ 11     /* float  [N]           current nn upper bounds (squared)      */
#define TSDD_FETCH_NN_EXACT 12  /* uint8  [N]           1 where NN_SQ is the exact nn          */

/* Row stride of TSDD_FETCH_ROWS in floats (n rounded up to a multiple of 64; padding is 0). */
size_t tsdd_cuda_row_stride(const tsdd_cuda_ctx* ctx);

/* Copies one prepared array to host memory.  bytes must be the exact size. */
int tsdd_cuda_fetch(tsdd_cuda_ctx* ctx, int what, void* dst, size_t bytes);

/* Rows [first_row, first_row + n_rows) of the matrix (0-based, n_rows * stride floats):
 * SubsequenceMatrix::row (series.hpp:53) without moving the whole matrix.   */
int tsdd_cuda_fetch_rows(tsdd_cuda_ctx* ctx, size_t first_row, size_t n_rows, float* dst);

/* ---- several GPUs: candidates sharded, best-so-far max-reduced ----------- */

/* Entry e of the rarity order belongs to rank (e mod world).  After every
 * batch the packed best-so-far (float bits of d^2 << 32 | ~position) is
 * max-reduced over all ranks, and (option "share_bounds", default on) the N
 * nn bounds are min-reduced, so that what one rank's scans learn about a row
 * prunes it on every rank.                                                  */

/* NCCL path: one 16-byte ncclAllReduce(ncclMax, ncclUint64) and one N-element
 * ncclAllReduce(ncclMin, ncclUint64) per batch on the search stream.  libnccl.so.2 is loaded at run time.  Rank 0 creates the id
 * and hands the 128 bytes to the other ranks (any transport).               */
int tsdd_cuda_comm_unique_id(char id[128]);
int tsdd_cuda_comm_init(tsdd_cuda_ctx* ctx, const char id[128], int world, int rank);
/* Ranks of the context's exchange: what ncclCommCount reports for its NCCL communicator, else
 * the world size it was given (1 for a single context).                     */
int tsdd_cuda_comm_size(const tsdd_cuda_ctx* ctx, int* nranks);

/* In-process path: `world` contexts of ONE process (one per device; the same device may carry
 * several) become ranks 0 .. world-1 of a group, each driven by its own host thread.  The
 * ranks meet in a host barrier and exchange on the devices: the per-batch keys through the
 * barrier, the N nn bounds by a kernel that min-reduces the peers' arrays read straight from
 * their memory (cudaDeviceEnablePeerAccess: NVLink / NVSwitch; staged through cudaMemcpyPeer
 * where two devices cannot map one another).  Call once, from one thread, before the rank
 * threads start; every rank must then make the same prepare / search calls.  A failure on one
 * rank releases the others with TSDD_ERR_RUNTIME.                            */
int tsdd_cuda_group_create(tsdd_cuda_ctx** ctxs, int world);

/* Host-hook path (tests, or a caller that already owns a communicator): the
 * engine hands `count` packed keys on the host; the hook must return, in
 * place, the element-wise maximum over all ranks.  Non-zero = failure.      */
typedef int (*tsdd_exchange_fn)(void* user, uint64_t* keys, size_t count);
int tsdd_cuda_set_exchange(tsdd_cuda_ctx* ctx, tsdd_exchange_fn fn, void* user, int world,
                           int rank);

/* ---- measurement helpers -------------------------------------------------- */

/* FP32 issue-rate probes on the context's device (roofline denominators the
 * driver's MEASURED_PEAKS.json does not have).  which: 0 = dependent-free
 * FFMA stream, 1 = FSUB+FFMA pairs (the distance kernel's mix), 2 = packed
 * fma.rn.f32x2, 3 = packed sub+fma f32x2; +4 = the same at 8 warps per SM, +8 = at
 * 16 warps per SM (the tile kernels' occupancies).  Returns lane-operations per second
 * in *ops_per_s (one FFMA = one op; an f32x2 instruction = two).            */
int tsdd_cuda_fp32_probe(tsdd_cuda_ctx* ctx, int which, double* ops_per_s, double* ms);

/* Exhaustive nn profile with the same tiled kernel and no pruning (the
 * Engine::brute analogue, discovery.cpp:123-173): nn_sq[N], +inf where a row
 * has no non-self match.  Needs a prepared context.                         */
int tsdd_cuda_nn_profile(tsdd_cuda_ctx* ctx, float* nn_sq_host);

#ifdef __cplusplus
}
#endif
#endif /* TSDD_CUDA_H */
