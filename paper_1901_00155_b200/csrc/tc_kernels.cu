// The dot-product form of the tile kernel on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// The default for the dot form (option dot_form = 5; 1 / 2 keep it on the CUDA-core kernels of
// search_kernels.cu, which stay the FP32 roofline evidence) and for the tails of covering scans (tc_tail).
// The dot form of the distance, d^2 = |a|^2 + |b|^2 - 2 a.b, is a dense contraction: a tile of 128
// candidates x 256 neighbours is the matrix product A (128 x n) . B^T (n x 256).  Float32 inputs do
// not fit a 16-bit or TF32 mantissa, so every row is split once into
//     x = hi + lo,   hi = fp16(x), lo = fp16(x - hi)   (22 bits between them; or two tf32 parts, dot_form 3 / 4),
// and a tile is THREE MMAs per k-step,
//     A_hi.B_hi + A_hi.B_lo + A_lo.B_hi        (the missing lo.lo term is below 2^-20 |a||b|),
// accumulated in float32 in tensor memory.  The split and the accumulation leave an absolute
// error of the same kind as the CUDA-core dot form's, within three times its bound; the engine
// widens the discard band accordingly (SearchState::margin_abs) and the float64 decision at the
// end of a pass is unchanged — positions stay those of the reference.
//
// Kernel anatomy (PERSISTENT: one CTA per SM takes work items — a candidate tile x up to 16 neighbour tiles —
// off a global counter; 256 threads, 352 when converting; no CTA-wide barrier after the set-up):
//   warp 3      the head: work items, and per tile — everything requested in one batch, the next tile's rows a
//               tile ahead — the candidates' rows / norms / thresholds, the neighbours' rows / norms / kill limits,
//               the lower-bound filter of a tail, the position bins of a window tile; four metadata slots;
//   warp 0      producer: per 64-byte row piece four TMA boxes (A_hi, A_lo: 128 rows; B_hi, B_lo: 256 rows;
//               64-byte swizzle; 48 KB) onto a "full" mbarrier, four stages deep — or, converting (format 3),
//               the float32 neighbour rows themselves as one 256 x 128-byte box where B_hi | B_lo go;
//   warp 1      MMA issuer: one elected lane issues 6 tcgen05.mma per stage (M 128, N 256, K 16 fp16 / 8 tf32;
//               operands straight from the swizzled shared-memory tiles through matrix descriptors) and
//               tcgen05.commit's the stage back to the producer; the accumulators of tile t+1 go to the other
//               half of tensor memory (2 x 256 columns);
//   warp 2      allocates / frees the 512 TMEM columns; converting: one of the four converter warps (with warps
//               8 .. 10) that split the float32 rows into the fp16 operand tiles in place;
//   warps 4..7  epilogue: thread m of the warpgroup owns candidate m (TMEM lane m); it reads its 256 accumulators
//               with tcgen05.ld (32 columns at a time, the next chunk in flight), keeps two running minima per
//               chunk and looks at a chunk pair by pair only when one of them trips; one atomicMin per
//               candidate per tile, plus the symmetric updates that kill a neighbour.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "kernels.hpp"

namespace tsdd_b200 {

namespace {

constexpr int kM = 128;                    // candidates per tile = TMEM lanes
constexpr int kN = 256;                    // neighbours per tile = accumulator columns
// A stage is one 64-byte piece of every row (64-byte swizzle): 16 tf32 columns or 32 fp16 columns,
// i.e. two MMA k-steps of 32 bytes either way; the byte geometry does not depend on the format.
constexpr int kRowPiece = 64;
constexpr int kTcStages = 4;
constexpr int kMetaSlots = 4;              // tiles whose metadata may be prepared ahead of the streams
constexpr int kABytes = kM * kRowPiece;        //  8 KB
constexpr int kBBytes = kN * kRowPiece;        // 16 KB
constexpr int kTcStageBytes = 2 * kABytes + 2 * kBBytes;  // A_hi | A_lo | B_hi | B_lo = 48 KB
constexpr int kTcThreads = 256;
constexpr uint32_t kTmemCols = 512;        // two accumulator sets of 256 columns
constexpr int kBinWords = 256;             // 8,192 position bins per tile (a bit each)

constexpr float kNoColumn = 1e30f;         // "norm" of a column that holds no row / takes no symmetric update: never the smallest

struct alignas(16) TcMeta {
  float thr[kM];               // the candidates' thresholds (their bounds; -1: dead or no candidate)
  uint32_t cand[kM];           // ... their rows
  float cnorm[kM];             // ... and squared norms
  uint32_t jrow[kN];           // the neighbours' rows (0xFFFFFFFF: none)
  float nnorm[kN];             // ... squared norms (kNoColumn: none)
  float lim[kN];               // ... the distance below which a symmetric update kills the neighbour (-1: takes none)
  float w[kN];                 // nnorm - lim (kNoColumn: takes none): the epilogue's one test per chunk
  uint32_t bins[kBinWords];    // window tiles: which position bins (row >> bin_shift, folded) hold a neighbour of the tile
  uint32_t valid;   // neighbour slots of the tile that hold a row
  uint32_t stop;    // no tile follows
  uint32_t slot0;   // first neighbour slot of the tile
  uint32_t cand0;   // first candidate slot of the tile (of the work item it belongs to)
};

struct SharedTc {
  alignas(1024) unsigned char stages[kTcStages][kTcStageBytes];
  TcMeta meta[kMetaSlots];
  unsigned long long full[kTcStages], empty[kTcStages], ready[kTcStages], tmem_full[2], tmem_empty[2], meta_full[kMetaSlots], meta_empty[kMetaSlots];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t gap(uint32_t a, uint32_t b) { return a > b ? a - b : b - a; }
__device__ __forceinline__ uint64_t ld_key(const uint64_t* p) {
  return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}

__device__ __forceinline__ void bar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(unsigned long long* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Bounded wait: a pipeline that never completes traps (after kWaitLimitNs of wall time) instead
// of hanging the GPU; `tag` says which wait it was.
constexpr unsigned long long kWaitLimitNs = 2000000000ull;
__device__ __noinline__ void bar_wait_slow(unsigned long long* bar, uint32_t parity, int tag) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t done = 0;
    for (int spin = 0; spin < 1024 && !done; ++spin) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(smem_u32(bar)), "r"(parity)
          : "memory");
    }
    if (done) return;
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > kWaitLimitNs) {
      printf("k_scan_tiles_tc: wait %d timed out (parity %u, block %u,%u thread %u)\n", tag, parity, blockIdx.x, blockIdx.y,
             threadIdx.x);
      __trap();
    }
  }
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, uint32_t parity, int tag) {
  uint32_t done = 0;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  if (!done) bar_wait_slow(bar, parity, tag);
}
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* map, uint32_t col, uint32_t row, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(col), "r"(row), "r"(smem_u32(bar))
      : "memory");
}

// Shared-memory matrix descriptor of a K-major tile whose rows are 64 bytes with the 64-byte
// swizzle (what the TMA boxes write): start address >> 4 | leading offset (unused for swizzled
// K-major) | stride between 8-row groups = 512 bytes | descriptor version 1 | SWIZZLE_64B (4).
__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr) {
  return static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4) | (1ull << 16) | (static_cast<uint64_t>((8 * kRowPiece) >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}
// Instruction descriptor: D float32; A / B tf32 (format 2) or fp16 (format 0), both K-major; N = 256, M = 128.
template <bool kHalf>
struct InstrDesc {
  static constexpr uint32_t value = (1u << 4) | ((kHalf ? 0u : 2u) << 7) | ((kHalf ? 0u : 2u) << 10) |
                                    (static_cast<uint32_t>(kN >> 3) << 17) | (static_cast<uint32_t>(kM >> 4) << 24);
};
template <bool kHalf>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t accumulate) {
  if constexpr (kHalf)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "n"(InstrDesc<true>::value), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "n"(InstrDesc<false>::value), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, "
      "%18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]),
        "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// The registers of an earlier tmem_ld32 may be read after this (they are operands, so that no use moves above the wait).
__device__ __forceinline__ void tmem_wait(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]), "+r"(v[8]),
                 "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]),
                 "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]),
                 "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

// x = hi + lo with both parts fp16 (round to nearest): 22 bits between them
__device__ __forceinline__ void split_half(const float4& x, uint2& h, uint2& l) {
  const __half2 h0 = __floats2half2_rn(x.x, x.y), h1 = __floats2half2_rn(x.z, x.w);
  const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
  const __half2 l0 = __floats2half2_rn(x.x - f0.x, x.y - f0.y), l1 = __floats2half2_rn(x.z - f1.x, x.w - f1.y);
  h = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
  l = make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
}
// -DTSDD_TC_PROFILE: cycles every role spends in each of its waits, printed by a few CTAs (development aid)
#ifdef TSDD_TC_PROFILE
#define TC_T0() const long long t0_ = clock64()
#define TC_ACC(x) (x) += clock64() - t0_
#else
#define TC_T0()
#define TC_ACC(x)
#endif

// -DTSDD_TC_EXP=bits: timing experiments (results are WRONG under them): 1 the epilogue only drains tensor
// memory, 2 the producer leaves the neighbour boxes out, 4 one MMA per k-step instead of three, 8 no A boxes
#ifndef TSDD_TC_EXP
#define TSDD_TC_EXP 0
#endif

struct TcArgs {
  const uint32_t* batch_rows;
  const uint32_t* batch_slots;
  const uint32_t* sel;
  const uint32_t* nbr_index;  // hash-sorted row list (window mode) or nullptr
  uint32_t u_begin, u_end;    // 256-row neighbour tiles of this launch
  uint32_t tiles_per_item;    // neighbour tiles of one work item
  int pruning;
  uint32_t* work;             // the launch's work-item counter (zero at launch)
  float lim_factor;
  int tail;                   // a covering scan of a search that is not in the dot form (counters: tail_calls, no tile_live)
};

// kFormat: 0 rows split into two tf32 parts, 1 into two fp16 parts (both read from split copies of the matrix), 3 fp16
// parts of the NEIGHBOUR rows made inside the kernel: the producer streams the float32 matrix itself (128-byte pieces,
// 128-byte swizzle) into a raw buffer beside each stage, and the otherwise idle warp 2 splits it into the stage's
// B_hi / B_lo tiles in the layout a 64-byte-swizzled TMA box would have written (chunk c of row r at c ^ ((r >> 1) & 3)),
// then fences the async proxy and signals the MMA warp.  No split copy of the matrix at all (16 GB and 4.8 ms at
// workload 4): the tails of covering scans, which stream every neighbour row once per candidate tile anyway.
constexpr int kConvertWarps = 4;   // warp 2 and three more (warps 8 .. 10)
constexpr int kTcThreadsConvert = kTcThreads + 32 * (kConvertWarps - 1);
template <bool kSymmetric, int kFormat>
__global__ void __launch_bounds__(kFormat == 3 ? kTcThreadsConvert : kTcThreads, 1)
k_scan_tiles_tc(SearchState s, TcArgs a, const __grid_constant__ CUtensorMap map_a_hi,
                const __grid_constant__ CUtensorMap map_a_lo, const __grid_constant__ CUtensorMap map_b_hi,
                const __grid_constant__ CUtensorMap map_b_lo) {
  extern __shared__ unsigned char smem_raw[];
  // (swizzled tiles want 1024-byte alignment: align by hand, the launch adds the slack)
  SharedTc& sh = *reinterpret_cast<SharedTc*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));

  const uint32_t count = a.sel[0];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float inf = __uint_as_float(kInfBits);

  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) bar_init(&sh.full[i], 1), bar_init(&sh.empty[i], 1), bar_init(&sh.ready[i], kConvertWarps);
    for (int i = 0; i < 2; ++i) {
      bar_init(&sh.tmem_full[i], 1);
      bar_init(&sh.tmem_empty[i], 4);   // the four epilogue warps
    }
    for (int i = 0; i < kMetaSlots; ++i) {
      bar_init(&sh.meta_full[i], 1);
      bar_init(&sh.meta_empty[i], kFormat == 3 ? 6 + kConvertWarps : 6);   // the four epilogue warps, the MMA warp, the producer (and the converter)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {  // tensor memory: all 512 columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)), "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = sh.tmem_base;

  const bool window = a.nbr_index != nullptr;
  const uint32_t bin_shift = 31 - __clz(s.n);  // position bins of 2^bin_shift <= n rows (TcMeta::bins)
  const uint32_t units = (s.n_rows + kN - 1) / kN;  // 256-row units of the (hash-sorted or positional) row order
  constexpr bool kHalf = kFormat != 0, kConvert = kFormat == 3;
  constexpr uint32_t kStageCols = kHalf ? 32 : 16;  // columns of one 64-byte row piece
  // (converting: the raw float32 neighbour rows land where B_hi | B_lo go — 256 rows x 128 bytes = 2 x 256 rows x 64 bytes —
  // and are converted in place: the stage geometry is the same)
  constexpr uint32_t kStages = kTcStages, kStageBytes = kTcStageBytes;
  unsigned char* const stage_base = &sh.stages[0][0];
  const uint32_t chunks = s.stride / kStageCols;

  if (warp == 3) {
    // ================================================================ the head of the pipeline: work items and tile metadata
    // The CTAs of a launch (one per SM) take work items — one candidate tile x `tiles_per_item`
    // neighbour tiles, candidate tiles the fast index so that the CTAs running side by side walk
    // the same neighbour tiles (those then come from L2) — off a global counter until none is
    // left: no wave quantisation, and tensor memory, barriers and pipeline are set up once per SM
    // and launch.  Everything the other roles need to know about a tile travels in its metadata
    // slot, the candidate tile included, so an item boundary is no event for them.
    const uint64_t best = a.pruning ? *s.best : 0ull;
    // the greatest distance that still kills a row (common.cuh: dead_bound); 0 while there is no best-so-far
    const float best_d = __uint_as_float(key_bits(best));
    const float kill = a.pruning ? fmaxf((best_d - fmaf(s.margin_q, sqrtf(best_d), s.margin_abs)) / s.margin, 0.f) : 0.f;
    const uint32_t cand_tiles = (count + kM - 1) / kM;
    const uint32_t span = a.u_end - a.u_begin;
    const uint32_t items_per_cand = (span + a.tiles_per_item - 1) / a.tiles_per_item;
    const uint32_t total_items = cand_tiles * items_per_cand;
    unsigned long long calls_total = 0, tiles_total = 0, live_total = 0, skipped_total = 0;
    [[maybe_unused]] long long w_a = 0;
    [[maybe_unused]] const long long t_start = clock64();
    auto slot0_of = [&](uint32_t u, uint32_t centre) -> uint32_t {
      // window mode: units around the candidate tile's own, alternating outwards; covering mode: unit u itself
      if (!window) return u * kN;
      const uint32_t step = (u + 1) >> 1;
      const uint32_t unit = (u & 1) ? (centre + step) % units : (centre + units - step % units) % units;
      return unit * kN;
    };
    // Everything a tile needs from global memory is requested in ONE batch before anything is used
    // (with its loads one behind the other this warp, not the tensor cores, set the pace: 22,000
    // cycles a tile), and the neighbour rows of the NEXT tile, on which that tile's other loads
    // depend, are requested a tile ahead.
    auto rows_of = [&](uint32_t slot0, uint32_t (&j)[kN / 32]) {
#pragma unroll
      for (int q = 0; q < kN / 32; ++q) {
        const uint32_t slot = slot0 + lane + 32 * q;
        j[q] = slot < s.n_rows ? (window ? __ldg(a.nbr_index + slot) : slot) : 0xFFFFFFFFu;
      }
    };
    uint32_t ti = 0;          // tiles published so far
    bool slot_held = false;   // the next slot has been waited for already (a tile that was not published after all)
    for (;;) {
      uint32_t item = 0;
      if (lane == 0) item = atomicAdd(a.work, 1u);
      item = __shfl_sync(0xFFFFFFFFu, item, 0);
      if (item >= total_items) break;
      const uint32_t cand0 = (item % cand_tiles) * kM;
      const uint32_t u0 = a.u_begin + (item / cand_tiles) * a.tiles_per_item;
      const uint32_t n_tiles = min(static_cast<uint32_t>(a.tiles_per_item), a.u_end - u0);
      uint32_t crow[kM / 32];
      float cnorm[kM / 32];
#pragma unroll
      for (int q = 0; q < kM / 32; ++q) {
        const uint32_t r = cand0 + lane + 32 * q;
        crow[q] = r < count ? __ldg(a.batch_rows + r) : 0xFFFFFFFFu;
      }
      const uint32_t centre = window ? __ldg(a.batch_slots + min(cand0 + kM / 2, count - 1)) / kN : 0u;
#pragma unroll
      for (int q = 0; q < kM / 32; ++q) {
        if (crow[q] != 0xFFFFFFFFu) TSDD_BOUND(crow[q], s.n_rows);
        cnorm[q] = crow[q] != 0xFFFFFFFFu ? __ldg(s.row_norms + crow[q]) : 0.f;
      }
      // the lower-bound filter of the covering scans (search_kernels.cu: k_scan_tiles<.., kLb>) for a tail: the
      // candidates' 16 segment means, kept for the whole item
      const bool filter = a.tail && a.pruning && !window && s.lb_means != nullptr;
      float means[kM / 32][kLbSegments];
      if (filter) {
#pragma unroll
        for (int q = 0; q < kM / 32; ++q) {
          const float4* pm = reinterpret_cast<const float4*>(s.lb_means + static_cast<size_t>(crow[q] != 0xFFFFFFFFu ? crow[q] : 0u) * kLbSegments);
#pragma unroll
          for (int v = 0; v < kLbSegments / 4; ++v) {
            const float4 m4 = __ldg(pm + v);
            means[q][4 * v] = m4.x, means[q][4 * v + 1] = m4.y, means[q][4 * v + 2] = m4.z, means[q][4 * v + 3] = m4.w;
          }
        }
      }
      uint32_t j_next[kN / 32];
      rows_of(slot0_of(u0, centre), j_next);
      for (uint32_t t = 0; t < n_tiles; ++t) {
        const uint32_t m = ti % kMetaSlots, use = ti / kMetaSlots;
        TcMeta& meta = sh.meta[m];
        const uint32_t slot0 = slot0_of(u0 + t, centre);
        const uint32_t valid = slot0 < s.n_rows ? min(static_cast<uint32_t>(kN), s.n_rows - slot0) : 0u;
        uint32_t j[kN / 32];
        uint64_t key_n[kN / 32], key_c[kM / 32];
        float norm_n[kN / 32];
#pragma unroll
        for (int q = 0; q < kN / 32; ++q) {
          j[q] = j_next[q];
          if (j[q] != 0xFFFFFFFFu) TSDD_BOUND(j[q], s.n_rows);
          key_n[q] = (j[q] != 0xFFFFFFFFu && kSymmetric && a.pruning) ? ld_key(s.nn + j[q]) : 0ull;
          norm_n[q] = j[q] != 0xFFFFFFFFu ? __ldg(s.row_norms + j[q]) : kNoColumn;
        }
#pragma unroll
        for (int q = 0; q < kM / 32; ++q) key_c[q] = (crow[q] != 0xFFFFFFFFu && a.pruning) ? ld_key(s.nn + crow[q]) : 0ull;
        if (t + 1 < n_tiles) rows_of(slot0_of(u0 + t + 1, centre), j_next);
        if (use >= 1 && !slot_held) { TC_T0(); bar_wait(&sh.meta_empty[m], (use - 1) & 1, 1); TC_ACC(w_a); }
        slot_held = true;
        bool any_live = false, any_needed = false;
        unsigned long long calls = 0;
        uint32_t live = 0, skipped = 0;
        float4 tile_lo[kLbSegments / 4], tile_hi[kLbSegments / 4];
        if (filter && valid > 0) {  // the box of the tile's boxes: lane l reduces component l (16 minima, 16 maxima)
          const uint32_t first_unit = slot0 / kLbBoxRows, last_unit = (slot0 + valid - 1) / kLbBoxRows;
          float comp = lane < kLbSegments ? 3.0e38f : -3.0e38f;
          for (uint32_t unit = first_unit; unit <= last_unit; ++unit) {
            const float v = __ldg(s.lb_boxes + static_cast<size_t>(unit) * 2 * kLbSegments + lane);
            comp = lane < kLbSegments ? fminf(comp, v) : fmaxf(comp, v);
          }
          float box[2 * kLbSegments];
#pragma unroll
          for (int c = 0; c < 2 * kLbSegments; ++c) box[c] = __shfl_sync(0xFFFFFFFFu, comp, c);
#pragma unroll
          for (int v = 0; v < kLbSegments / 4; ++v) {
            tile_lo[v] = make_float4(box[4 * v], box[4 * v + 1], box[4 * v + 2], box[4 * v + 3]);
            tile_hi[v] = make_float4(box[kLbSegments + 4 * v], box[kLbSegments + 4 * v + 1], box[kLbSegments + 4 * v + 2],
                                     box[kLbSegments + 4 * v + 3]);
          }
        }
#pragma unroll
        for (int q = 0; q < kM / 32; ++q) {
          const uint32_t r = lane + 32 * q, row = crow[q];
          float thr = -1.f;
          if (row != 0xFFFFFFFFu) {
            if (!a.pruning) {
              thr = inf;
            } else {
              const float bound = __uint_as_float(key_bits(key_c[q]));
              if (!dead_bound(bound, best, s.margin, s.margin_abs, s.margin_q)) thr = bound;
            }
          }
          if (thr >= 0.f) any_live = true;
          if (filter && thr >= 0.f && valid > 0) {
            // a candidate whose segment means lie further from every 16-row box of the tile than its threshold
            // cannot find a neighbour below it here: it sits the tile out.  First against the box of the whole
            // tile (a weaker bound, one test instead of sixteen), which settles most of them.
            float lb_tile = 0.f;
#pragma unroll
            for (int v = 0; v < kLbSegments / 4; ++v) {
              const float4 lo = tile_lo[v], hi = tile_hi[v];
              float g;
              g = fmaxf(fmaxf(lo.x - means[q][4 * v], means[q][4 * v] - hi.x), 0.f), lb_tile = fmaf(g, g, lb_tile);
              g = fmaxf(fmaxf(lo.y - means[q][4 * v + 1], means[q][4 * v + 1] - hi.y), 0.f), lb_tile = fmaf(g, g, lb_tile);
              g = fmaxf(fmaxf(lo.z - means[q][4 * v + 2], means[q][4 * v + 2] - hi.z), 0.f), lb_tile = fmaf(g, g, lb_tile);
              g = fmaxf(fmaxf(lo.w - means[q][4 * v + 3], means[q][4 * v + 3] - hi.w), 0.f), lb_tile = fmaf(g, g, lb_tile);
            }
            bool needed = false;
            const bool settled = lb_rules_out(lb_tile * s.lb_scale, thr, s.lb_q);
            const uint32_t first_unit = slot0 / kLbBoxRows, last_unit = (slot0 + valid - 1) / kLbBoxRows;
            for (uint32_t unit = first_unit; unit <= last_unit && !needed && !settled; ++unit) {
              const float4* pb = reinterpret_cast<const float4*>(s.lb_boxes + static_cast<size_t>(unit) * 2 * kLbSegments);
              float lb = 0.f;
#pragma unroll
              for (int v = 0; v < kLbSegments / 4; ++v) {
                const float4 lo = __ldg(pb + v), hi = __ldg(pb + kLbSegments / 4 + v);
                float g;
                g = fmaxf(fmaxf(lo.x - means[q][4 * v], means[q][4 * v] - hi.x), 0.f), lb = fmaf(g, g, lb);
                g = fmaxf(fmaxf(lo.y - means[q][4 * v + 1], means[q][4 * v + 1] - hi.y), 0.f), lb = fmaf(g, g, lb);
                g = fmaxf(fmaxf(lo.z - means[q][4 * v + 2], means[q][4 * v + 2] - hi.z), 0.f), lb = fmaf(g, g, lb);
                g = fmaxf(fmaxf(lo.w - means[q][4 * v + 3], means[q][4 * v + 3] - hi.w), 0.f), lb = fmaf(g, g, lb);
              }
              needed = !lb_rules_out(lb * s.lb_scale, thr, s.lb_q);
            }
            if (!needed) {
              thr = -1.f;
              skipped += 1;
            }
          }
          meta.thr[r] = thr;
          meta.cand[r] = row;
          meta.cnorm[r] = cnorm[q];
          if (thr >= 0.f) {
            any_needed = true;
            live += 1;
            uint32_t overlap = 0;
            if (!window) {  // (window tiles: the epilogue counts the self-match pairs)
              const uint32_t z0 = row >= s.n - 1 ? row - (s.n - 1) : 0, z1 = row + s.n;
              const uint32_t o0 = max(slot0, z0), o1 = min(slot0 + valid, z1);
              overlap = o1 > o0 ? o1 - o0 : 0;
            }
            calls += valid - overlap;
          }
        }
        any_live = __any_sync(0xFFFFFFFFu, any_live);
        if (!any_live) break;  // every candidate of the tile is dead: the rest of the item is not needed (the slot stays held)
        skipped_total += skipped;
        if (!__any_sync(0xFFFFFFFFu, any_needed)) continue;  // the filter: nobody needs this tile (the slot stays held)
        if (window) {
#pragma unroll
          for (int q = 0; q < kBinWords / 32; ++q) meta.bins[lane + 32 * q] = 0u;
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < kN / 32; ++q) {
          const uint32_t e = lane + 32 * q;
          meta.jrow[e] = j[q];
          meta.nnorm[e] = norm_n[q];  // (kNoColumn where the slot holds no row: such a column never comes out smallest)
          // Symmetric updates, d(i,j) = d(j,i), are only worth their price where they KILL the neighbour
          // (in the dot form nothing else is gained from a lower bound: no tile is abandoned early): a
          // neighbour that is dead already, or no best-so-far yet, and the column takes none.
          float lim = -1.f;
          if (kSymmetric && a.pruning && j[q] != 0xFFFFFFFFu && kill > 0.f &&
              !dead_bound(__uint_as_float(key_bits(key_n[q])), best, s.margin, s.margin_abs, s.margin_q))
            lim = fminf(__uint_as_float(key_bits(key_n[q])), kill * a.lim_factor);
          meta.lim[e] = lim;
          meta.w[e] = lim > 0.f ? norm_n[q] - lim : kNoColumn;  // |b|^2 - 2 a.b - lim < -|a|^2  <=>  d < lim
          if (window && j[q] != 0xFFFFFFFFu) {
            const uint32_t bin = (j[q] >> bin_shift) & (kBinWords * 32 - 1);
            atomicOr(&meta.bins[bin >> 5], 1u << (bin & 31));
          }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) calls += __shfl_xor_sync(0xFFFFFFFFu, calls, d);
        live_total += live;
        if (lane == 0) {
          meta.valid = valid;
          meta.slot0 = slot0;
          meta.cand0 = cand0;
          meta.stop = 0u;
        }
        __syncwarp();
        if (lane == 0) bar_arrive(&sh.meta_full[m]);
        slot_held = false;
        ++ti;
        calls_total += calls;
        tiles_total += 1;
      }
    }
    {  // the slot after the last tile: stop
      const uint32_t m = ti % kMetaSlots, use = ti / kMetaSlots;
      if (use >= 1 && !slot_held) bar_wait(&sh.meta_empty[m], (use - 1) & 1, 1);
      if (lane == 0) sh.meta[m].stop = 1u;
      __syncwarp();
      if (lane == 0) bar_arrive(&sh.meta_full[m]);
    }
#ifdef TSDD_TC_PROFILE
    if (lane == 0 && blockIdx.x % 37 == 0)
      printf("tc meta cta %u: total %lld wait meta_empty %lld tiles %llu\n", blockIdx.x, clock64() - t_start, w_a, tiles_total);
#endif
    if (lane == 0) {
      if (calls_total) atomicAdd(&s.counters->calls, calls_total);
      if (calls_total && a.tail) atomicAdd(&s.counters->tail_calls, calls_total);
      if (tiles_total) atomicAdd(&s.counters->tiles, tiles_total);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) live_total += __shfl_xor_sync(0xFFFFFFFFu, live_total, d);
    if (lane == 0 && live_total && !a.tail) atomicAdd(&s.counters->tile_live, live_total);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) skipped_total += __shfl_xor_sync(0xFFFFFFFFu, skipped_total, d);
    if (lane == 0 && skipped_total) atomicAdd(&s.counters->lb_skipped, skipped_total);
  } else if (warp == 0) {
    // ================================================================ producer: the TMA streams
    uint32_t seq = 0;
    [[maybe_unused]] long long w_meta = 0, w_a = 0;
    [[maybe_unused]] const long long t_start = clock64();
    for (uint32_t ti = 0;; ++ti) {
      const uint32_t m = ti % kMetaSlots;
      { TC_T0(); bar_wait(&sh.meta_full[m], (ti / kMetaSlots) & 1, 2); TC_ACC(w_meta); }
      const bool stop = *reinterpret_cast<volatile uint32_t*>(&sh.meta[m].stop) != 0;
      const uint32_t slot0 = *reinterpret_cast<volatile uint32_t*>(&sh.meta[m].slot0);
      const uint32_t cand0 = *reinterpret_cast<volatile uint32_t*>(&sh.meta[m].cand0);
      __syncwarp();
      if (lane == 0) bar_arrive(&sh.meta_empty[m]);
      if (stop) break;
      for (uint32_t c = 0; c < chunks; ++c) {
        const uint32_t st = seq % kStages, round = seq / kStages;
        if (round >= 1) { TC_T0(); bar_wait(&sh.empty[st], (round - 1) & 1, 3); TC_ACC(w_a); }
        if (lane == 0) {
          bar_expect_tx(&sh.full[st], ((TSDD_TC_EXP & 8) ? 0 : 2 * kABytes) + ((TSDD_TC_EXP & 2) ? 0 : 2 * kBBytes));
          unsigned char* dst = stage_base + st * kStageBytes;
          const uint32_t col = c * kStageCols;
          if (!(TSDD_TC_EXP & 8)) {
            tma_box(dst, &map_a_hi, col, cand0, &sh.full[st]);
            tma_box(dst + kABytes, &map_a_lo, col, cand0, &sh.full[st]);
          }
          if (kConvert) {  // the float32 rows themselves: 256 rows x 128 bytes, where B_hi | B_lo will be
            tma_box(dst + 2 * kABytes, &map_b_hi, col, slot0, &sh.full[st]);
          } else if (!(TSDD_TC_EXP & 2)) {
            tma_box(dst + 2 * kABytes, &map_b_hi, col, slot0, &sh.full[st]);
            tma_box(dst + 2 * kABytes + kBBytes, &map_b_lo, col, slot0, &sh.full[st]);
          }
        }
        ++seq;
      }
    }
#ifdef TSDD_TC_PROFILE
    if (lane == 0 && blockIdx.x % 37 == 0)
      printf("tc producer cta %u: total %lld wait meta %lld wait empty %lld stages %u\n", blockIdx.x, clock64() - t_start, w_meta, w_a, seq);
#endif
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    uint32_t seq = 0;
    [[maybe_unused]] long long w_meta = 0, w_a = 0, w_b = 0;
    [[maybe_unused]] const long long t_start = clock64();
    for (uint32_t ti = 0;; ++ti) {
      const uint32_t m = ti % kMetaSlots, buf = ti & 1;
      { TC_T0(); bar_wait(&sh.meta_full[m], (ti / kMetaSlots) & 1, 4); TC_ACC(w_meta); }
      const bool stop = *reinterpret_cast<volatile uint32_t*>(&sh.meta[m].stop) != 0;
      __syncwarp();
      if (lane == 0) bar_arrive(&sh.meta_empty[m]);
      if (stop) break;
      if (ti >= 2) { TC_T0(); bar_wait(&sh.tmem_empty[buf], ((ti >> 1) - 1) & 1, 5); TC_ACC(w_a); }  // the epilogue has drained this accumulator set
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tmem_d = tmem_base + buf * kN;
      for (uint32_t c = 0; c < chunks; ++c) {
        const uint32_t st = seq % kStages, round = seq / kStages;
        { TC_T0(); bar_wait(kConvert ? &sh.ready[st] : &sh.full[st], round & 1, 6); TC_ACC(w_b); }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t base = smem_u32(stage_base + st * kStageBytes);
          const uint64_t a_hi = umma_desc(base), a_lo = umma_desc(base + kABytes);
          const uint64_t b_hi = umma_desc(base + 2 * kABytes), b_lo = umma_desc(base + 2 * kABytes + kBBytes);
#pragma unroll
          for (uint32_t k = 0; k < 2; ++k) {  // two k-steps of 32 bytes (8 tf32 / 16 fp16 columns) per stage
            const uint64_t step = static_cast<uint64_t>((k * 32) >> 4);
            umma<kHalf>(tmem_d, a_hi + step, b_hi + step, (c | k) != 0 ? 1u : 0u);
            if (!(TSDD_TC_EXP & 4)) {
              umma<kHalf>(tmem_d, a_hi + step, b_lo + step, 1u);
              umma<kHalf>(tmem_d, a_lo + step, b_hi + step, 1u);
            }
          }
          umma_commit(&sh.empty[st]);                          // the stage is free once these MMAs have read it
          if (c + 1 == chunks) umma_commit(&sh.tmem_full[buf]);  // ... and the tile's accumulators are complete
        }
        __syncwarp();
        ++seq;
      }
    }
#ifdef TSDD_TC_PROFILE
    if (lane == 0 && blockIdx.x % 37 == 0)
      printf("tc mma cta %u: total %lld wait meta %lld wait tmem_empty %lld wait full %lld stages %u\n", blockIdx.x, clock64() - t_start, w_meta, w_a, w_b, seq);
#endif
  } else if (kConvert && (warp == 2 || warp >= 8)) {
    // ================================================================ converters: float32 neighbour rows -> fp16 hi / lo tiles
    const uint32_t part = warp == 2 ? 0u : warp - 7u;  // this warp's quarter of the tile's rows
    uint32_t seq = 0;
    for (uint32_t ti = 0;; ++ti) {
      const uint32_t m = ti % kMetaSlots;
      bar_wait(&sh.meta_full[m], (ti / kMetaSlots) & 1, 9);
      const bool stop = *reinterpret_cast<volatile uint32_t*>(&sh.meta[m].stop) != 0;
      __syncwarp();
      if (lane == 0) bar_arrive(&sh.meta_empty[m]);
      if (stop) break;
      for (uint32_t c = 0; c < chunks; ++c) {
        const uint32_t st = seq % kStages, round = seq / kStages;
        bar_wait(&sh.full[st], round & 1, 10);
        unsigned char* base = stage_base + st * kStageBytes;
        const float4* raw = reinterpret_cast<const float4*>(base + 2 * kABytes);
        constexpr uint32_t kRowsPerLane = kN / 32 / kConvertWarps;
        uint32_t hi[kRowsPerLane][16], lo[kRowsPerLane][16];  // 32 halves a row each: the row's two 64-byte pieces
#pragma unroll
        for (uint32_t rr = 0; rr < kRowsPerLane; ++rr) {
          const uint32_t r = part * (kN / kConvertWarps) + lane + 32 * rr;
#pragma unroll
          for (uint32_t q = 0; q < 8; ++q) {
            const float4 x = raw[r * 8 + (q ^ (r & 7u))];  // (128-byte swizzle of the raw box)
            uint2 h, l;
            split_half(x, h, l);
            hi[rr][2 * q] = h.x, hi[rr][2 * q + 1] = h.y;
            lo[rr][2 * q] = l.x, lo[rr][2 * q + 1] = l.y;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kConvertWarps) : "memory");  // every converter has read its rows: now in place
#pragma unroll
        for (uint32_t rr = 0; rr < kRowsPerLane; ++rr) {
          const uint32_t r = part * (kN / kConvertWarps) + lane + 32 * rr;
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q) {
            const uint32_t at = r * kRowPiece + ((q ^ ((r >> 1) & 3u)) << 4);  // (64-byte swizzle of the operand tile)
            *reinterpret_cast<uint4*>(base + 2 * kABytes + at) =
                make_uint4(hi[rr][4 * q], hi[rr][4 * q + 1], hi[rr][4 * q + 2], hi[rr][4 * q + 3]);
            *reinterpret_cast<uint4*>(base + 2 * kABytes + kBBytes + at) =
                make_uint4(lo[rr][4 * q], lo[rr][4 * q + 1], lo[rr][4 * q + 2], lo[rr][4 * q + 3]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> the tensor cores' reads
        __syncwarp();
        if (lane == 0) bar_arrive(&sh.ready[st]);
        ++seq;
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ================================================================ epilogue: thread = candidate = TMEM lane
    const uint32_t mrow = tid - 128;                 // candidate (TMEM lane) of this thread
    const uint32_t lane_base = (warp & 3u) * 32u;    // the TMEM lanes this warp may read
    const float d_floor = 0.5f * s.margin_abs;
    unsigned long long tiles_done = 0, useful = 0;
    uint32_t overlap_total = 0;
    [[maybe_unused]] long long w_meta = 0, w_a = 0;
    [[maybe_unused]] const long long t_start = clock64();
#ifdef TSDD_TC_PROFILE
    uint32_t n_slow = 0, n_slow_thr = 0, n_near = 0, n_part = 0;
#endif
    for (uint32_t ti = 0;; ++ti) {
      const uint32_t m = ti % kMetaSlots, buf = ti & 1;
      { TC_T0(); bar_wait(&sh.meta_full[m], (ti / kMetaSlots) & 1, 7); TC_ACC(w_meta); }
      TcMeta& meta = sh.meta[m];
      if (*reinterpret_cast<volatile uint32_t*>(&meta.stop) != 0) {
        __syncwarp();
        if (lane == 0) bar_arrive(&sh.meta_empty[m]);
        break;
      }
      const float thr = meta.thr[mrow];
      const uint32_t row = meta.cand[mrow];
      const float cn = meta.cnorm[mrow];
      const bool taking_part = thr >= 0.f && row != 0xFFFFFFFFu;
#ifdef TSDD_TC_PROFILE
      n_part += taking_part ? 1 : 0;
#endif
      // Can the tile hold a self match (|row - j| < n) of this candidate?  Covering tiles are consecutive
      // rows; of a window tile the metadata warp has marked the position bins that hold a neighbour.
      bool near = false;
      if (taking_part) {
        const uint32_t z0 = row >= s.n - 1 ? row - (s.n - 1) : 0u, z1 = row + s.n - 1;
        if (!window) {
          near = z0 < meta.slot0 + meta.valid && z1 >= meta.slot0;
        } else {
          for (uint32_t b = z0 >> bin_shift; b <= (z1 >> bin_shift); ++b) {
            const uint32_t bin = b & (kBinWords * 32 - 1);
            near |= (meta.bins[bin >> 5] >> (bin & 31)) & 1u;
          }
        }
      }
      { TC_T0(); bar_wait(&sh.tmem_full[buf], (ti >> 1) & 1, 8); TC_ACC(w_a); }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      unsigned long long key_min = ~0ull;  // (distance bits << 32) | neighbour: the 64-bit minimum settles ties by the smaller row
      // Per 32-column chunk two running minima, no branch: of |b|^2 - 2 a.b (against the candidate's own
      // threshold) and of |b|^2 - 2 a.b - lim (against -|a|^2: a distance that kills its neighbour).
      // Only a chunk in which one of them trips is looked at pair by pair — and a tile that may hold a
      // self match of the candidate, whose pairs have to be told apart.  The accumulators of chunk
      // c + 1 are on their way from tensor memory while chunk c is measured.
      const uint32_t taddr = tmem_base + (lane_base << 16) + buf * kN;
      const float thr_own = taking_part ? thr : -inf;
      auto measure = [&](const uint32_t (&v)[32], uint32_t cc) {
        const float4* pn = reinterpret_cast<const float4*>(meta.nnorm + cc * 32);
        const float4* pw = reinterpret_cast<const float4*>(meta.w + cc * 32);
        // (four independent minima each: one warp per scheduler has nobody to hide a 32-deep dependent chain behind)
        float l0 = inf, l1 = inf, l2 = inf, l3 = inf, w0 = inf, w1 = inf, w2 = inf, w3 = inf;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 nn4 = pn[q];
          l0 = fminf(l0, fmaf(-2.f, __uint_as_float(v[4 * q]), nn4.x));
          l1 = fminf(l1, fmaf(-2.f, __uint_as_float(v[4 * q + 1]), nn4.y));
          l2 = fminf(l2, fmaf(-2.f, __uint_as_float(v[4 * q + 2]), nn4.z));
          l3 = fminf(l3, fmaf(-2.f, __uint_as_float(v[4 * q + 3]), nn4.w));
          if (kSymmetric) {
            const float4 w4 = pw[q];
            w0 = fminf(w0, fmaf(-2.f, __uint_as_float(v[4 * q]), w4.x));
            w1 = fminf(w1, fmaf(-2.f, __uint_as_float(v[4 * q + 1]), w4.y));
            w2 = fminf(w2, fmaf(-2.f, __uint_as_float(v[4 * q + 2]), w4.z));
            w3 = fminf(w3, fmaf(-2.f, __uint_as_float(v[4 * q + 3]), w4.w));
          }
        }
        const float low = fminf(fminf(l0, l1), fminf(l2, l3)), low_w = fminf(fminf(w0, w1), fminf(w2, w3));
        if ((TSDD_TC_EXP & 1) && low != 12345.678f) return;
        const bool own = fmaxf(low + cn, d_floor) <= thr_own;
        const bool kills = kSymmetric && taking_part && low_w < -cn;
        if (own || kills) {
#ifdef TSDD_TC_PROFILE
          n_slow += 1; n_slow_thr += own ? 1 : 0;
#endif
#pragma unroll
          for (int i = 0; i < 32; ++i) {  // (fully unrolled: the accumulators stay in registers)
            const uint32_t n = cc * 32 + i;
            const float t = fmaf(-2.f, __uint_as_float(v[i]), meta.nnorm[n]);
            const float d = fmaxf(t + cn, d_floor);
            const float lim = kSymmetric ? meta.lim[n] : -1.f;
            if (d <= thr_own || d < lim) {
              const uint32_t j = meta.jrow[n];
              if (j != 0xFFFFFFFFu && (!near || gap(row, j) >= s.n)) {
                const uint32_t bits = __float_as_uint(d);
                if (d <= thr_own) {
                  const unsigned long long key = nn_key(bits, j);
                  key_min = key < key_min ? key : key_min;
                }
                if (d < lim) {
                  TSDD_BOUND(j, s.n_rows);
                  atomicMin(as_ull(s.nn + j), static_cast<unsigned long long>(nn_key(bits, row)));
                }
              }
            }
          }
        }
      };
      {
        uint32_t v0[32], v1[32];
        tmem_ld32(taddr, v0);
#pragma unroll 1
        for (uint32_t cc = 0; cc < kN / 32; cc += 2) {
          tmem_wait(v0);
          tmem_ld32(taddr + (cc + 1) * 32, v1);
          measure(v0, cc);
          __syncwarp();  // (the pair-by-pair path diverges; tcgen05.ld / wait are warp-wide)
          tmem_wait(v1);
          if (cc + 2 < kN / 32) tmem_ld32(taddr + (cc + 2) * 32, v0);
          measure(v1, cc + 1);
          __syncwarp();
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&sh.tmem_empty[buf]);
      if (window) {
        // Self-match pairs of a window tile (the metadata warp counted live x valid): the warp counts them
        // together, candidate by candidate, each lane looking at eight of the tile's neighbours.
        uint32_t todo = __ballot_sync(0xFFFFFFFFu, near);
        while (todo) {
          const int src = __ffs(todo) - 1;
          todo &= todo - 1;
          const uint32_t r = __shfl_sync(0xFFFFFFFFu, row, src);
#ifdef TSDD_TC_PROFILE
          n_near += lane == 0 ? 1 : 0;
#endif
#pragma unroll
          for (int q = 0; q < kN / 32; ++q) overlap_total += gap(r, meta.jrow[lane + 32 * q]) < s.n ? 1u : 0u;
        }
      }
      if (key_min != ~0ull) {
        TSDD_BOUND(row, s.n_rows);
        atomicMin(as_ull(s.nn + row), key_min);
      }
      useful += taking_part ? static_cast<unsigned long long>(meta.valid) * s.n : 0ull;
      tiles_done += 1;
      __syncwarp();
      if (lane == 0) bar_arrive(&sh.meta_empty[m]);
    }
#ifdef TSDD_TC_PROFILE
    if (blockIdx.x % 37 == 0) {
      const uint32_t any_slow = __reduce_add_sync(0xFFFFFFFFu, n_slow), any_thr = __reduce_add_sync(0xFFFFFFFFu, n_slow_thr),
                     any_near = __reduce_add_sync(0xFFFFFFFFu, n_near), any_part = __reduce_add_sync(0xFFFFFFFFu, n_part);
      if (lane == 0)
        printf("tc epilogue cta %u: total %lld wait meta %lld wait tmem_full %lld tiles %llu slow %u slowthr %u near %u part %u\n", blockIdx.x,
               clock64() - t_start, w_meta, w_a, tiles_done, any_slow, any_thr, any_near, any_part);
    }
#endif
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      useful += __shfl_xor_sync(0xFFFFFFFFu, useful, d);
      overlap_total += __shfl_xor_sync(0xFFFFFFFFu, overlap_total, d);
    }
    if (lane == 0) {
      if (warp == 4 && tiles_done) {
        const unsigned long long terms = tiles_done * kM * kN * static_cast<unsigned long long>(s.stride);
        atomicAdd(&s.counters->terms, terms);
        atomicAdd(&s.counters->tile_terms, terms);
        atomicAdd(&s.counters->dot_terms, terms);
        atomicAdd(&s.counters->tc_terms, terms);
      }
      if (useful) atomicAdd(&s.counters->useful_terms, useful);
      if (overlap_total) atomicAdd(&s.counters->calls, ~static_cast<unsigned long long>(overlap_total) + 1ull);
    }
  }

  // ---- teardown: every role is done with tensor memory before it is freed
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}


// x = hi + lo with both parts exactly representable in tf32 (low 13 mantissa bits clear)
__global__ void __launch_bounds__(256)
k_split_tf32(const float4* __restrict__ in, size_t quads, float4* __restrict__ hi, float4* __restrict__ lo) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= quads) return;
  const float4 x = in[i];
  auto top = [](float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); };
  const float4 h = make_float4(top(x.x), top(x.y), top(x.z), top(x.w));
  hi[i] = h;
  lo[i] = make_float4(top(x.x - h.x), top(x.y - h.y), top(x.z - h.z), top(x.w - h.w));
}

__global__ void __launch_bounds__(256)
k_split_f16(const float4* __restrict__ in, size_t quads, uint2* __restrict__ hi, uint2* __restrict__ lo) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= quads) return;
  uint2 h, l;
  split_half(in[i], h, l);
  hi[i] = h;
  lo[i] = l;
}

// The same split, one warp per row, with the row's squared norm as a by-product (the same sum k_row_norms
// forms): a search that moves its covering scans to the tensor cores mid-way reads the matrix once, not twice.
template <bool kHalf>
__global__ void __launch_bounds__(256)
k_split_rows_norms(const float* __restrict__ in, uint32_t n_rows, uint32_t stride, float* __restrict__ hi, float* __restrict__ lo,
                   float* __restrict__ norms, uint32_t n_norms) {
  const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const float4* p = reinterpret_cast<const float4*>(in + static_cast<size_t>(row) * stride);
  auto top = [](float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); };
  float acc = 0.f;
  for (uint32_t c = lane; c < stride / 4; c += 32) {
    const float4 x = p[c];
    acc += (x.x * x.x + x.y * x.y) + (x.z * x.z + x.w * x.w);
    if constexpr (kHalf) {
      uint2 h, l;
      split_half(x, h, l);
      reinterpret_cast<uint2*>(hi)[static_cast<size_t>(row) * (stride / 4) + c] = h;
      reinterpret_cast<uint2*>(lo)[static_cast<size_t>(row) * (stride / 4) + c] = l;
    } else {
      const float4 h = make_float4(top(x.x), top(x.y), top(x.z), top(x.w));
      reinterpret_cast<float4*>(hi)[static_cast<size_t>(row) * (stride / 4) + c] = h;
      reinterpret_cast<float4*>(lo)[static_cast<size_t>(row) * (stride / 4) + c] =
          make_float4(top(x.x - h.x), top(x.y - h.y), top(x.z - h.z), top(x.w - h.w));
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
  if (lane == 0 && row < n_norms) norms[row] = acc;
}

// The batch's rows, split the same way, dense in batch order; rows past the batch size are zero.
template <bool kHalf>
__global__ void __launch_bounds__(256)
k_gather_rows_split(SearchState s, const uint32_t* __restrict__ batch_rows, const uint32_t* __restrict__ sel,
                    uint32_t capacity_padded, float* __restrict__ hi, float* __restrict__ lo) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= capacity_padded) return;
  const uint32_t count = sel[0];
  if (r >= (count + kM - 1) / kM * kM) return;  // only the tiles the scan will touch
  if constexpr (kHalf) {
    uint2* dh = reinterpret_cast<uint2*>(hi) + static_cast<size_t>(r) * (s.stride / 4);
    uint2* dl = reinterpret_cast<uint2*>(lo) + static_cast<size_t>(r) * (s.stride / 4);
    if (r < count) {
      TSDD_BOUND(batch_rows[r], s.n_rows);
      const float4* src = reinterpret_cast<const float4*>(s.rows + static_cast<size_t>(batch_rows[r]) * s.stride);
      for (uint32_t c = lane; c < s.stride / 4; c += 32) split_half(__ldg(src + c), dh[c], dl[c]);
    } else {
      for (uint32_t c = lane; c < s.stride / 4; c += 32) dh[c] = dl[c] = make_uint2(0u, 0u);
    }
    return;
  }
  float4* dh = reinterpret_cast<float4*>(hi + static_cast<size_t>(r) * s.stride);
  float4* dl = reinterpret_cast<float4*>(lo + static_cast<size_t>(r) * s.stride);
  auto top = [](float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); };
  if (r < count) {
    TSDD_BOUND(batch_rows[r], s.n_rows);
    const float4* src = reinterpret_cast<const float4*>(s.rows + static_cast<size_t>(batch_rows[r]) * s.stride);
    for (uint32_t c = lane; c < s.stride / 4; c += 32) {
      const float4 x = __ldg(src + c);
      const float4 h = make_float4(top(x.x), top(x.y), top(x.z), top(x.w));
      dh[c] = h;
      dl[c] = make_float4(top(x.x - h.x), top(x.y - h.y), top(x.z - h.z), top(x.w - h.w));
    }
  } else {
    for (uint32_t c = lane; c < s.stride / 4; c += 32) dh[c] = dl[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

inline unsigned blocks_of(size_t items, unsigned per_block) { return static_cast<unsigned>((items + per_block - 1) / per_block); }

}  // namespace

int launch_split_rows(const float* d_in, size_t floats, bool half, float* d_hi, float* d_lo, cudaStream_t stream) {
  const size_t quads = floats / 4;
  if (half)
    k_split_f16<<<blocks_of(quads, 256), 256, 0, stream>>>(reinterpret_cast<const float4*>(d_in), quads,
                                                          reinterpret_cast<uint2*>(d_hi), reinterpret_cast<uint2*>(d_lo));
  else
    k_split_tf32<<<blocks_of(quads, 256), 256, 0, stream>>>(reinterpret_cast<const float4*>(d_in), quads,
                                                           reinterpret_cast<float4*>(d_hi), reinterpret_cast<float4*>(d_lo));
  return 1;
}

int launch_split_rows_norms(const float* d_in, uint32_t n_rows, uint32_t stride, bool half, float* d_hi, float* d_lo,
                            float* d_norms, uint32_t n_norms, cudaStream_t stream) {
  const unsigned blocks = blocks_of(static_cast<size_t>(n_rows) * 32, 256);
  if (half) k_split_rows_norms<true><<<blocks, 256, 0, stream>>>(d_in, n_rows, stride, d_hi, d_lo, d_norms, n_norms);
  else k_split_rows_norms<false><<<blocks, 256, 0, stream>>>(d_in, n_rows, stride, d_hi, d_lo, d_norms, n_norms);
  return 1;
}

int launch_gather_rows_split(SearchState s, const uint32_t* d_batch_rows, const uint32_t* d_sel, uint32_t capacity_padded,
                             bool half, float* d_hi, float* d_lo, cudaStream_t stream) {
  const unsigned blocks = blocks_of(static_cast<size_t>(capacity_padded) * 32, 256);
  if (half) k_gather_rows_split<true><<<blocks, 256, 0, stream>>>(s, d_batch_rows, d_sel, capacity_padded, d_hi, d_lo);
  else k_gather_rows_split<false><<<blocks, 256, 0, stream>>>(s, d_batch_rows, d_sel, capacity_padded, d_hi, d_lo);
  return 1;
}

int launch_scan_tiles_tc(SearchState s, const TcOperands& op, const uint32_t* d_batch_rows, const uint32_t* d_batch_slots,
                         const uint32_t* d_sel, uint32_t live_upper_bound, const uint32_t* d_nbr_index, uint32_t k_begin,
                         uint32_t k_end, bool pruning, bool symmetric, cudaStream_t stream, const char** error) {
  if (error) *error = nullptr;
  if (k_end <= k_begin || live_upper_bound == 0) return 0;
  // 128-row units of the plan -> 256-row tiles (a half tile of overlap with the neighbouring segment is harmless)
  const uint32_t u_begin = k_begin / 2, u_end = (k_end + 1) / 2;
  const uint32_t cand_tiles = (live_upper_bound + kM - 1) / kM;
  const uint64_t tiles = u_end - u_begin;
  // Work items for the persistent CTAs (one per SM): about `per_sm` items per SM, so that the last ones to finish
  // are short, of at most 16 tiles (an item whose candidates are all dead is dropped at its first tile)
  constexpr int per_sm = 6;  // (3 and 12 measure the same)
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  // a symmetric update is taken where it kills its neighbour (x 1.1 of that distance: 20 % slower, the slow path trips)
  constexpr float lim_factor = 1.f;
  const uint64_t want = tiles * cand_tiles / (static_cast<uint64_t>(sms) * per_sm);
  const uint32_t tiles_per_item = static_cast<uint32_t>(want < 1 ? 1 : want > 16 ? 16 : want);
  const uint64_t items = static_cast<uint64_t>(cand_tiles) * ((tiles + tiles_per_item - 1) / tiles_per_item);
  const bool window = d_nbr_index != nullptr;
  CUtensorMap map_a_hi{}, map_a_lo{}, map_b_hi{}, map_b_lo{};
  const float* b_hi = window ? op.sorted_hi : op.rows_hi;
  const float* b_lo = window ? op.sorted_lo : op.rows_lo;
  const uint64_t b_rows = op.rows_padded;  // (a box that reaches past the last row is zero-filled by the TMA unit)
  const uint32_t cols = op.half ? 32 : 16, elem = op.half ? 2 : 4;
  if (op.convert && (window || !op.half)) {
    if (error) *error = "the converting tensor-core kernel takes fp16 parts and covering scans only";
    return 0;
  }
  if (!make_row_map_boxed(&map_a_hi, op.batch_hi, static_cast<uint64_t>(cand_tiles) * kM, s.stride, cols, kM, elem) ||
      !make_row_map_boxed(&map_a_lo, op.batch_lo, static_cast<uint64_t>(cand_tiles) * kM, s.stride, cols, kM, elem) ||
      // (converting: the float32 matrix itself, 32 columns = 128 bytes a piece, 128-byte swizzle; b_lo unused)
      !(op.convert ? make_row_map_boxed(&map_b_hi, s.rows, b_rows, s.stride, 32, kN, 4)
                   : make_row_map_boxed(&map_b_hi, b_hi, b_rows, s.stride, cols, kN, elem)) ||
      !(op.convert ? make_row_map_boxed(&map_b_lo, s.rows, b_rows, s.stride, 32, kN, 4)
                   : make_row_map_boxed(&map_b_lo, b_lo, b_rows, s.stride, cols, kN, elem))) {
    if (error) *error = "cuTensorMapEncodeTiled failed (tensor-core tile kernel)";
    return 0;
  }
  cudaMemsetAsync(op.work, 0, sizeof(uint32_t), stream);
  TcArgs a{d_batch_rows, d_batch_slots, d_sel, d_nbr_index, u_begin, u_end, tiles_per_item, pruning ? 1 : 0, op.work,
           op.tail ? 1e30f : lim_factor,  // (a tail's neighbours take every symmetric update: the rows it meets are still to be scanned)
           op.tail ? 1 : 0};
  dim3 grid(static_cast<unsigned>(items < static_cast<uint64_t>(sms) ? items : sms));
  const int smem = static_cast<int>(sizeof(SharedTc)) + 1024;
  auto launch = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kernel<<<grid, op.convert ? kTcThreadsConvert : kTcThreads, smem, stream>>>(s, a, map_a_hi, map_a_lo, map_b_hi, map_b_lo);
  };
  if (symmetric) {
    if (op.convert) launch(k_scan_tiles_tc<true, 3>);
    else if (op.half) launch(k_scan_tiles_tc<true, 1>);
    else launch(k_scan_tiles_tc<true, 0>);
  } else {
    if (op.convert) launch(k_scan_tiles_tc<false, 3>);
    else if (op.half) launch(k_scan_tiles_tc<false, 1>);
    else launch(k_scan_tiles_tc<false, 0>);
  }
  return 1;
}

}  // namespace tsdd_b200
