// FP32 issue-rate probes: the roofline denominator of the distance kernel.
//
// MEASURED_PEAKS.json has HBM and bf16 tensor figures only.  The distance
// kernel runs on the FP32 CUDA-core pipe, so its ceiling is measured here, on
// the same device and at the same clocks, with register-resident streams of
// independent operations in the kernel's own instruction mixes:
//   0  FFMA only                      (the nominal "FP32 FMA peak")
//   1  FSUB + FFMA per term           (scalar (x-y)^2 accumulation)
//   2  packed fma.rn.f32x2 only       (sm_100 two-lane FP32 instruction)
//   3  packed add + fma f32x2 per two terms (the shipped kernel's mix)
// One "op" is one scalar-lane instruction result: an FFMA counts 1, an f32x2
// instruction counts 2.

#include "kernels.hpp"

namespace tsdd_b200 {

namespace {

constexpr int kProbeThreads = 256;
constexpr int kProbeChains = 16;  // independent accumulators per thread
constexpr int kProbeUnroll = 8;   // body repetitions per loop trip

template <int kWhich>
__global__ void __launch_bounds__(kProbeThreads)
k_fp32_probe(float* sink, int iters) {
  const float seed = static_cast<float>(threadIdx.x) * 1e-3f;
  if constexpr (kWhich == 0 || kWhich == 1) {
    float acc[kProbeChains], a[kProbeChains];
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) {
      acc[c] = seed + c;
      a[c] = seed * 0.5f + c * 0.25f;
    }
    float b = seed + 0.125f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < kProbeUnroll; ++r) {
#pragma unroll
        for (int c = 0; c < kProbeChains; ++c) {
          if constexpr (kWhich == 0) {
            acc[c] = fmaf(a[c], b, acc[c]);
          } else {
            const float d = a[c] - b;
            acc[c] = fmaf(d, d, acc[c]);
          }
        }
        // one operand moves (a loop-invariant a - b would be hoisted out of the sub+fma mix, and the
        // FFMA-only stream measured SLOWER with a constant multiplier: 55 instead of 70 TFLOP/s);
        // this one FADD per kProbeChains steps runs on the same pipe and is COUNTED (fp32_probe_ops)
        b += 1e-7f;
      }
    }
    float total = 0.f;
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) total += acc[c];
    if (total == 12345.678f) sink[blockIdx.x * blockDim.x + threadIdx.x] = total;
  } else {
    float2 acc[kProbeChains], a[kProbeChains];
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) {
      acc[c] = make_float2(seed + c, seed - c);
      a[c] = make_float2(seed * 0.5f + c * 0.25f, seed * 0.25f - c);
    }
    float2 b = make_float2(seed + 0.125f, seed - 0.125f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < kProbeUnroll; ++r) {
#pragma unroll
        for (int c = 0; c < kProbeChains; ++c) {
          if constexpr (kWhich == 2) {
            acc[c] = __ffma2_rn(a[c], b, acc[c]);
          } else {
            const float2 d = __fadd2_rn(a[c], b);
            acc[c] = __ffma2_rn(d, d, acc[c]);
          }
        }
        b.x += 1e-7f;  // (counted, see above)
      }
    }
    float total = 0.f;
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) total += acc[c].x + acc[c].y;
    if (total == 12345.678f) sink[blockIdx.x * blockDim.x + threadIdx.x] = total;
  }
}

// Packed and scalar arithmetic interleaved: kPackedChains chains of f32x2
// sub+fma and kScalarChains chains of scalar sub+fma per step.  If the packed
// instructions occupy only one of the two FP32 sub-pipes, the scalar ones can
// run beside them.
template <int kPackedChains, int kScalarChains>
__global__ void __launch_bounds__(kProbeThreads)
k_fp32_probe_dual(float* sink, int iters) {
  const float seed = static_cast<float>(threadIdx.x) * 1e-3f;
  float2 acc2[kPackedChains], a2[kPackedChains];
  float acc1[kScalarChains], a1[kScalarChains];
#pragma unroll
  for (int c = 0; c < kPackedChains; ++c) {
    acc2[c] = make_float2(seed + c, seed - c);
    a2[c] = make_float2(seed * 0.5f + c * 0.25f, seed * 0.25f - c);
  }
#pragma unroll
  for (int c = 0; c < kScalarChains; ++c) {
    acc1[c] = seed + 3 * c;
    a1[c] = seed * 0.75f + c * 0.125f;
  }
  float2 b = make_float2(seed + 0.125f, seed - 0.125f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < kProbeUnroll; ++r) {
#pragma unroll
      for (int c = 0; c < (kPackedChains > kScalarChains ? kPackedChains : kScalarChains); ++c) {
        if (c < kPackedChains) {
          const float2 d = __fadd2_rn(a2[c], b);
          acc2[c] = __ffma2_rn(d, d, acc2[c]);
        }
        if (c < kScalarChains) {
          const float d = a1[c] + b.x;
          acc1[c] = fmaf(d, d, acc1[c]);
        }
      }
      b.x += 1e-7f;
    }
  }
  float total = 0.f;
#pragma unroll
  for (int c = 0; c < kPackedChains; ++c) total += acc2[c].x + acc2[c].y;
#pragma unroll
  for (int c = 0; c < kScalarChains; ++c) total += acc1[c];
  if (total == 12345.678f) sink[blockIdx.x * blockDim.x + threadIdx.x] = total;
}

}  // namespace

int launch_fp32_probe(int which, float* d_sink, int blocks, int iters, cudaStream_t stream) {
  switch (which) {
    case 16: k_fp32_probe_dual<8, 8><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); return 1;
    case 17: k_fp32_probe_dual<12, 6><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); return 1;
    case 18: k_fp32_probe_dual<12, 4><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); return 1;
    case 19: k_fp32_probe_dual<14, 2><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); return 1;
    case 0: k_fp32_probe<0><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); break;
    case 1: k_fp32_probe<1><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); break;
    case 2: k_fp32_probe<2><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); break;
    default: k_fp32_probe<3><<<blocks, kProbeThreads, 0, stream>>>(d_sink, iters); break;
  }
  return 1;
}

double fp32_probe_ops(int which, int blocks, int iters) {
  const double lanes = static_cast<double>(blocks) * kProbeThreads;
  if (which >= 16) {
    const int packed = which == 16 ? 8 : which == 17 ? 12 : which == 18 ? 12 : 14;
    const int scalar = which == 16 ? 8 : which == 17 ? 6 : which == 18 ? 4 : 2;
    return lanes * static_cast<double>(iters) * kProbeUnroll * (packed * 4.0 + scalar * 2.0 + 1.0);  // + the moving operand's FADD
  }
  const double per_lane = static_cast<double>(iters) * kProbeUnroll * kProbeChains;
  const double instr = (which == 0 || which == 2) ? 1.0 : 2.0;  // instructions per chain step
  const double width = (which >= 2) ? 2.0 : 1.0;                 // lanes per instruction
  // every variant moves one operand with ONE scalar FADD per unroll step; it runs on the same pipe and is counted
  const double moving = static_cast<double>(iters) * kProbeUnroll;
  return lanes * (per_lane * instr * width + moving);
}

}  // namespace tsdd_b200
