// gemm.cu -- the quantized GEMMs.
//
// 1. lpq_quant_gemm: the per-op-rounded GEMM of the north star.  The
//    reference has no such kernel (its only GEMM is quantized_matmul, a
//    double-accumulated matmul quantized once, proj/src/quant_ops.cpp:191);
//    its semantics are restated from the reference's primitives in
//    oracle/lpq_oracle.h (lpqo_quant_gemm):
//        acc = +0;  for k in 0..K-1:  acc = Qa(fl32(acc + Qm(fl32(a_ik b_kj))))
//    Per-op rounding makes this a chain of 2K dependent rounded operations per
//    output, not a dense contraction, so it runs on the CUDA cores, never the
//    tensor cores, and never splits K.
//
//    Two kernels, selected ON THE DEVICE from a pre-scan of A and B (so the
//    call stays asynchronous):
//    * k_qgemm_bf16: when Qm = Qa = float(8,7), rounding is nearest-even,
//      A and B are bf16-exact and the pre-scan proves that no intermediate
//      can leave the normal bf16 range, then fl32(a*b) is exact, Q(v) equals
//      IEEE RNE to bf16 of the exact value, and double rounding through fp32
//      is innocuous (24 >= 2*8+2), so each Q(fl32(.)) is ONE hardware
//      bf16x2 op: HMUL2.BF16 for the product, HADD2.BF16 for the sum.  Two
//      outputs per instruction, one instruction per multiply-add.
//    * k_qgemm_general: any float formats and rounding modes (stochastic
//      included, with the reference RNG): fp32 __fmul_rn/__fadd_rn and the
//      exact element quantizer of quant_math.cuh after every op.
//
// 2. lpq_matmul_q: the reference's quantized_matmul with the quantizer fused
//    into the GEMM epilogue: FP64 DFMA accumulation in ascending k, which is
//    bit-identical to `acc += double(a) * double(b)` (tensor.cpp:355-376)
//    because the product of two fp32 values is exact in double.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/lpq.h"
#include "kernels.cuh"
#include "runtime.h"

namespace lpq {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// Pre-scan: finiteness, bf16-exactness and exponent ranges of A and B.
// GemmScan fields are accumulated with atomicMax; min fields are stored as
// 255 - field so a zeroed struct is the identity.
__global__ void __launch_bounds__(256)
    k_gemm_scan(const float* __restrict__ A, int64_t na,
                const float* __restrict__ B, int64_t nb,
                GemmScan* __restrict__ scan) {
  uint32_t a_min = 0, a_max = 0, b_min = 0, b_max = 0, a_low = 0, b_low = 0,
           nf = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb;
       i += stride) {
    const uint32_t u = i < na ? f2u(A[i]) : f2u(B[i - na]);
    const uint32_t f = (u >> 23) & 0xFFu;
    const uint32_t ab = u & 0x7FFFFFFFu;
    nf |= f == 0xFFu ? 1u : 0u;
    const uint32_t inv = ab ? 255u - f : 0u;
    if (i < na) {
      a_min = max(a_min, inv);
      a_max = max(a_max, f);
      a_low |= u & 0xFFFFu;
    } else {
      b_min = max(b_min, inv);
      b_max = max(b_max, f);
      b_low |= u & 0xFFFFu;
    }
  }
  a_min = __reduce_max_sync(kFull, a_min);
  a_max = __reduce_max_sync(kFull, a_max);
  b_min = __reduce_max_sync(kFull, b_min);
  b_max = __reduce_max_sync(kFull, b_max);
  a_low = __reduce_or_sync(kFull, a_low);
  b_low = __reduce_or_sync(kFull, b_low);
  nf = __reduce_or_sync(kFull, nf);
  if ((threadIdx.x & 31) == 0) {
    if (a_min) atomicMax(&scan->a_min_nz_exp_field, a_min);
    if (a_max) atomicMax(&scan->a_max_exp_field, a_max);
    if (b_min) atomicMax(&scan->b_min_nz_exp_field, b_min);
    if (b_max) atomicMax(&scan->b_max_exp_field, b_max);
    if (a_low) atomicOr(&scan->a_low_bits, a_low);
    if (b_low) atomicOr(&scan->b_low_bits, b_low);
    if (nf) atomicOr(&scan->nonfinite, nf);
  }
}

// True when the hardware bf16 path reproduces Q(fl32(.)) exactly for every
// op of this GEMM (see file comment and DESIGN.md §4).
__device__ __forceinline__ bool bf16_path_ok(const GemmScan& s, int64_t K) {
  if (s.nonfinite || s.a_low_bits || s.b_low_bits) return false;
  if (s.a_min_nz_exp_field == 0 || s.b_min_nz_exp_field == 0)
    return true;  // A or B is all zeros: every product and sum is +-0
  const int ea_min = (255 - (int)s.a_min_nz_exp_field) - 127;
  const int eb_min = (255 - (int)s.b_min_nz_exp_field) - 127;
  const int ea_max = (int)s.a_max_exp_field - 127;
  const int eb_max = (int)s.b_max_exp_field - 127;
  // every value is a multiple of 2^g, so nonzero magnitudes stay >= 2^-126
  if ((ea_min - 7) + (eb_min - 7) < -126) return false;
  // |acc| <= K * |a|max |b|max (1 + 2^-8)^(K+1) must stay below 2^127
  const double lg = log2((double)K) + (ea_max + 1) + (eb_max + 1) +
                    (double)(K + 1) * 0.00563 + 1.0;
  return lg < 126.0;
}

// Raw (not bf16-exact) fp32 operands under Qm = Qa = float(8,7) nearest:
// fl32(a*b) is the reference's product, and Qm of it is cvt.rn.bf16 when it
// is normal; the sums are of bf16 values, so HADD2.BF16 (one rounding of the
// exact sum) equals Qa(fl32(sum)) as in the exact path.  Every nonzero
// operand normal and every value a multiple of G = 2^(ea_min + eb_min - 7)
// >= 2^-126 keeps every nonzero product and sum normal; the overflow bound
// is the exact path's.
__device__ __forceinline__ bool bf16raw_path_ok(const GemmScan& s, int64_t K) {
  if (s.nonfinite) return false;
  if (s.a_min_nz_exp_field == 0 || s.b_min_nz_exp_field == 0)
    return true;  // A or B is all zeros: every product and sum is +-0
  const int fa = 255 - (int)s.a_min_nz_exp_field, fb = 255 - (int)s.b_min_nz_exp_field;
  if (fa == 0 || fb == 0) return false;  // a subnormal operand
  const int ea_min = fa - 127, eb_min = fb - 127;
  const int ea_max = (int)s.a_max_exp_field - 127;
  const int eb_max = (int)s.b_max_exp_field - 127;
  if (ea_min + eb_min - 7 < -126) return false;
  const double lg = log2((double)K) + (ea_max + 1) + (eb_max + 1) +
                    (double)(K + 1) * 0.00563 + 1.0;
  return lg < 126.0;
}

// ---------------------------------------------------------------------------
// k_qgemm_bits: any float formats whose mantissa fits the bit-domain form
// (man <= 22), NearestEven or Stochastic, when the pre-scan proves every
// product and partial sum is zero or inside both formats' normal ranges
// (bits_path_ok).  Then each Q is quant_float_bits -- an integer add of the
// rounding increment (RNE: half a step; stochastic: the reference variate's
// top bits, complemented for x >= 0) and a mask of the dropped bits -- with no
// clamp, no underflow grid and no branches; the variates of a thread's 4
// consecutive outputs share hash work (variate24_x4_top).  Same 64x64 tile
// and k order as k_qgemm_general.
//   Proof: nonzero operands normal; every product Qm(fl32(a b)) is a multiple
//   of G = 2^(ea_min + eb_min - man_m), and sums of multiples of G stay
//   multiples of G under fp32 adds and either rounding, so every nonzero
//   value is >= G >= 2^max(min_exp_m, min_exp_a); and |value| stays below
//   K |a|max |b|max (1 + 2^-man)^(K+1) < 2^min(max_exp_m, max_exp_a).
__device__ __forceinline__ bool bits_path_ok(const GemmScan& s, int64_t K,
                                             const FloatParams& qm, const FloatParams& qa) {
  if (s.nonfinite || !qm.bits_ok || !qa.bits_ok) return false;
  if (s.a_min_nz_exp_field == 0 || s.b_min_nz_exp_field == 0)
    return true;  // A or B is all zeros: every product and sum is +-0
  const int fa = 255 - (int)s.a_min_nz_exp_field, fb = 255 - (int)s.b_min_nz_exp_field;
  if (fa == 0 || fb == 0) return false;  // a subnormal operand
  const int ea_min = fa - 127, eb_min = fb - 127;
  const int ea_max = (int)s.a_max_exp_field - 127;
  const int eb_max = (int)s.b_max_exp_field - 127;
  if (ea_min + eb_min - qm.man < max(qm.min_exp, qa.min_exp)) return false;
  const int man = min(qm.man, qa.man);
  const double lg = log2((double)K) + (ea_max + 1) + (eb_max + 1) +
                    (double)(K + 1) * log2(1.0 + ldexp(1.0, -man)) + 1.0;
  return lg < (double)min(qm.max_exp, qa.max_exp);
}

// which kernel of a quant_gemm launch computes the product (each kernel
// evaluates this on the device from the pre-scan and exits unless it is the
// one): flags bit 0: float(8,7) RNE (the bf16 kernels may run), bit 1: the
// bits kernel may run.  0: exact bf16, 1: raw bf16, 2: bits, 3: general.
__device__ __forceinline__ int gemm_kernel_choice(const GemmScan& s, int64_t K, int flags,
                                                  const FloatParams& qm, const FloatParams& qa) {
  if ((flags & 1) && bf16_path_ok(s, K)) return 0;
  if ((flags & 1) && bf16raw_path_ok(s, K)) return 1;
  if ((flags & 2) && bits_path_ok(s, K, qm, qa)) return 2;
  return 3;
}

// ---------------------------------------------------------------------------
// k_qgemm_bf16: 128x128 CTA tile, 128 threads, 8x16 outputs per thread held
// as 64 bf16x2 accumulators; K staged 16 at a time into double-buffered
// shared memory as bf16 (A transposed so a thread's 8 rows are one 16-byte
// load), global tiles prefetched into registers one step ahead.  A thread's
// 16 columns are two groups of 8, 64 apart (tx*8, tx*8 + 64), so the B
// fragment loads of a quarter-warp are contiguous.
constexpr int kBM = 128, kBN = 128, kBK = 16, kQT = 128;

__device__ __forceinline__ uint32_t bmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t badd2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

template <bool VEC>
__device__ __forceinline__ float4 ld_tile4(const float* __restrict__ p,
                                           int64_t row, int64_t col,
                                           int64_t rows, int64_t cols,
                                           int64_t ld) {
  if (VEC) {
    if (row < rows && col < cols)
      return __ldg(reinterpret_cast<const float4*>(p + row * ld + col));
    return make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (row < rows) {
    const float* r = p + row * ld;
    if (col < cols) v.x = __ldg(r + col);
    if (col + 1 < cols) v.y = __ldg(r + col + 1);
    if (col + 2 < cols) v.z = __ldg(r + col + 2);
    if (col + 3 < cols) v.w = __ldg(r + col + 3);
  }
  return v;
}

__device__ __forceinline__ uint64_t pack_f32x2(float lo, float hi) {
  return ((uint64_t)f2u(hi) << 32) | f2u(lo);
}
// (lo0*lo1, hi0*hi1), each rounded to nearest like __fmul_rn
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// (lo0+lo1, hi0+hi1), each rounded to nearest like __fadd_rn
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ uint32_t cvt_bf16x2(float hi, float lo) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// RAW: operands that are not bf16-exact (bf16raw_path_ok): fp32 tiles in
// shared memory, two products per packed FMUL2 rounded by one F2FP (ALU
// pipe) into a bf16x2 word, then HADD2 -- no more FMA-pipe cycles per MAC than
// the HMUL2 form (measured: an HMUL2/HADD2 occupies both FMA half-pipes), so
// raw operands run near the exact path's rate.
template <bool VEC, bool RAW>
__global__ void __launch_bounds__(kQT)
    k_qgemm_bf16(const float* __restrict__ A, const float* __restrict__ B,
                 float* __restrict__ C, int64_t M, int64_t N, int64_t K,
                 const GemmScan* __restrict__ scan) {
  if (RAW ? (bf16_path_ok(*scan, K) || !bf16raw_path_ok(*scan, K))
          : !bf16_path_ok(*scan, K))
    return;  // another kernel of the launch runs instead
  using Elem = typename std::conditional<RAW, float, uint16_t>::type;
  __shared__ __align__(16) Elem As[2][kBK][kBM];
  __shared__ __align__(16) Elem Bs[2][kBK][kBN];
  const int t = threadIdx.x;
  const int tx = t & 7, ty = t >> 3;  // 8 column groups x 16 row groups
  const int64_t m0 = (int64_t)blockIdx.y * kBM, n0 = (int64_t)blockIdx.x * kBN;

  uint32_t acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0u;

  float4 ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int f = t + kQT * i;  // A: 128 rows x 4 float4 along k
      ra[i] = ld_tile4<VEC>(A, m0 + (f >> 2), k0 + (f & 3) * 4, M, K, K);
      const int g = t + kQT * i;  // B: 16 k-rows x 32 float4 along n
      rb[i] = ld_tile4<VEC>(B, k0 + (g >> 5), n0 + (g & 31) * 4, K, N, N);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int f = t + kQT * i;
      const int row = f >> 2, kq = (f & 3) * 4;
      const int g = t + kQT * i;
      const int kr = g >> 5, col = (g & 31) * 4;
      if constexpr (RAW) {
        As[buf][kq + 0][row] = ra[i].x;
        As[buf][kq + 1][row] = ra[i].y;
        As[buf][kq + 2][row] = ra[i].z;
        As[buf][kq + 3][row] = ra[i].w;
        *reinterpret_cast<float4*>(&Bs[buf][kr][col]) = rb[i];
      } else {
        As[buf][kq + 0][row] = (uint16_t)(f2u(ra[i].x) >> 16);
        As[buf][kq + 1][row] = (uint16_t)(f2u(ra[i].y) >> 16);
        As[buf][kq + 2][row] = (uint16_t)(f2u(ra[i].z) >> 16);
        As[buf][kq + 3][row] = (uint16_t)(f2u(ra[i].w) >> 16);
        uint2 w;
        w.x = (f2u(rb[i].x) >> 16) | (f2u(rb[i].y) & 0xFFFF0000u);
        w.y = (f2u(rb[i].z) >> 16) | (f2u(rb[i].w) & 0xFFFF0000u);
        *reinterpret_cast<uint2*>(&Bs[buf][kr][col]) = w;
      }
    }
  };

  const int64_t nk = (K + kBK - 1) / kBK;
  load(0);
  stash(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) load((kt + 1) * kBK);
    const int kk_end = (int)min((int64_t)kBK, K - kt * kBK);
    auto step = [&](int kk) {
      if constexpr (RAW) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8 + 4]);
        // columns tx*4 + 32q .. +3: a quarter-warp's float4 loads are 128
        // contiguous bytes (conflict-free; tx*16 + 4q was 4-way conflicted)
        float bf[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4 + 32 * q]);
          bf[4 * q] = b4.x;
          bf[4 * q + 1] = b4.y;
          bf[4 * q + 2] = b4.z;
          bf[4 * q + 3] = b4.w;
        }
        const float af[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        // two products per packed mul.rn.f32x2 (FMUL2): one issue slot per
        // pair (26.8 -> 28.5 TFLOP/s at 4096^3 over scalar FMUL pairs)
        uint64_t bp[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) bp[j] = pack_f32x2(bf[2 * j], bf[2 * j + 1]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t ap = pack_f32x2(af[i], af[i]);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint64_t p = fmul2(ap, bp[j]);
            acc[i][j] = badd2(acc[i][j], cvt_bf16x2(u2f((uint32_t)(p >> 32)), u2f((uint32_t)p)));
          }
        }
        return;
      }
      const uint4 av = *reinterpret_cast<const uint4*>(&As[buf][kk][ty * 8]);
      // columns tx*8 + 64q .. +7: a quarter-warp's 16-byte loads are 128
      // contiguous bytes (conflict-free; tx*16 was 2-way conflicted)
      const uint4 b0 = *reinterpret_cast<const uint4*>(&Bs[buf][kk][tx * 8]);
      const uint4 b1 = *reinterpret_cast<const uint4*>(&Bs[buf][kk][tx * 8 + 64]);
      const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
      const uint32_t bw[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t a2 = __byte_perm(aw[i >> 1], 0, (i & 1) ? 0x3232 : 0x1010);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = badd2(acc[i][j], bmul2(a2, bw[j]));
      }
    };
    if (kk_end == kBK && !RAW) {
      // full tile: unrolled so the shared-memory loads of k+1 overlap the
      // math of k (the k order of every accumulator is unchanged)
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) step(kk);
    } else if (kk_end == kBK) {
      // RAW: 256 instructions per k; a full unroll overflowed the
      // instruction cache (ncu: "no instruction" 2.9 stalls per issue)
#pragma unroll 2
      for (int kk = 0; kk < kBK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kk_end; ++kk) step(kk);
    }
    if (kt + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }

  // epilogue: bf16 -> fp32 is exact (the low half goes to the high bits)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + ty * 8 + i;
    if (row >= M) continue;
    float* crow = C + row * N;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // word j holds columns col, col + 1 (RAW: tx*4 + 32*(j/2) + 2*(j%2);
      // bf16: tx*8 + 64*(j/4) + 2*(j%4))
      const int64_t col = RAW ? n0 + tx * 4 + 32 * (j >> 1) + 2 * (j & 1)
                              : n0 + tx * 8 + 64 * (j >> 2) + 2 * (j & 3);
      const float lo = u2f(acc[i][j] << 16), hi = u2f(acc[i][j] & 0xFFFF0000u);
      if (VEC && col + 1 < N) {
        *reinterpret_cast<float2*>(crow + col) = make_float2(lo, hi);
      } else {
        if (col < N) crow[col] = lo;
        if (col + 1 < N) crow[col + 1] = hi;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_qgemm_general: 64x64 CTA tile, 256 threads, 4x4 outputs per thread, fp32
// shared tiles; any float formats and rounding modes.
constexpr int kGM = 64, kGN = 64, kGK = 16, kGT = 256;

// The streaming element forms (identical results to quant_float<M>), picked
// by the (uniform) format parameters.
template <int M>
__device__ __forceinline__ float qf(float x, const FloatParams& p, uint32_t v) {
  constexpr bool kFast = M == kNearestEven || M == kStochastic;
  constexpr int MF = kFast ? M : kNearestEven;
  if (kFast && p.scaled_ok) return quant_float_scaled<MF>(x, p, v);
  // the exp_bits == 8 streaming form: faster for stochastic rounding here
  // (0.40 -> 0.46 TFLOP/s), slower for nearest (1.02 -> 0.94)
  if (M == kStochastic && !p.tiny) return quant_float_fast<kStochastic>(x, p, v);
  return quant_float<M>(x, p, v);
}

template <int M_>
__global__ void __launch_bounds__(kGT)
    k_qgemm_general(const float* __restrict__ A, const float* __restrict__ B,
                    float* __restrict__ C, int64_t M, int64_t N, int64_t K,
                    int64_t row_base, FloatParams qm, FloatParams qa,
                    uint64_t seed, uint64_t call,
                    const GemmScan* __restrict__ scan, int flags,
                    uint32_t* __restrict__ status) {
  if (scan->nonfinite) {  // non-finite operands are rejected like quantize
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
      atomicOr(status, kStatusNonFinite);
    return;
  }
  if (gemm_kernel_choice(*scan, K, flags, qm, qa) != 3)
    return;  // another kernel of the launch did it
  __shared__ float As[kGK][kGM];
  __shared__ float Bs[kGK][kGN];
  __shared__ uint64_t keys[kGK][2];
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * kGM, n0 = (int64_t)blockIdx.x * kGN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  uint64_t idx[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      idx[i][j] = (uint64_t)(row_base + m0 + ty * 4 + i) * (uint64_t)N +
                  (uint64_t)(n0 + tx * 4 + j);

  for (int64_t k0 = 0; k0 < K; k0 += kGK) {
    for (int e = t; e < kGM * kGK; e += kGT) {
      const int r = e / kGK, c = e % kGK;  // A tile, coalesced along k
      const int64_t gr = m0 + r, gc = k0 + c;
      As[c][r] = (gr < M && gc < K) ? A[gr * K + gc] : 0.0f;
      const int kr = e / kGN, nc = e % kGN;  // B tile, coalesced along n
      const int64_t gk = k0 + kr, gn = n0 + nc;
      Bs[kr][nc] = (gk < K && gn < N) ? B[gk * N + gn] : 0.0f;
    }
    if (M_ == kStochastic && t < 2 * kGK) {
      const int kk = t >> 1, op = t & 1;
      keys[kk][op] = stream_key(seed, call + 2 * (uint64_t)(k0 + kk) + op);
    }
    __syncthreads();
    const int kk_end = (int)min((int64_t)kGK, K - k0);
    for (int kk = 0; kk < kk_end; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
      uint64_t km = 0, ka = 0;
      if (M_ == kStochastic) { km = keys[kk][0]; ka = keys[kk][1]; }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // a thread's 4 columns are consecutive flat indices: when the first
        // is a multiple of 4 their variates share work (variate24_x4)
        uint32_t vm[4] = {0u, 0u, 0u, 0u}, va[4] = {0u, 0u, 0u, 0u};
        if (M_ == kStochastic) {
          if ((idx[i][0] & 3u) == 0) {
            variate24_x4(km, idx[i][0], 32u, vm);
            variate24_x4(ka, idx[i][0], 32u, va);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              vm[j] = variate24(km, idx[i][j]);
              va[j] = variate24(ka, idx[i][j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float p = qf<M_>(fmul(a[i], b[j]), qm, vm[j]);
          acc[i][j] = qf<M_>(fadd(acc[i][j], p), qa, va[j]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + ty * 4 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + tx * 4 + j;
      if (col < N) C[row * N + col] = acc[i][j];
    }
  }
}

template <int M_, bool X4>
__global__ void __launch_bounds__(kGT)
    k_qgemm_bits(const float* __restrict__ A, const float* __restrict__ B,
                 float* __restrict__ C, int64_t M, int64_t N, int64_t K,
                 int64_t row_base, FloatParams qm, FloatParams qa,
                 uint64_t seed, uint64_t call, const GemmScan* __restrict__ scan,
                 int flags, RngMul rm) {
  if (gemm_kernel_choice(*scan, K, flags, qm, qa) != 2) return;
  __shared__ __align__(16) float As[kGK][kGM];
  __shared__ __align__(16) float Bs[kGK][kGN];
  __shared__ uint64_t keys[kGK][2];
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * kGM, n0 = (int64_t)blockIdx.x * kGN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  uint64_t idx[4];  // flat output index of column tx*4 of row i (the variates')
#pragma unroll
  for (int i = 0; i < 4; ++i)
    idx[i] = (uint64_t)(row_base + m0 + ty * 4 + i) * (uint64_t)N + (uint64_t)(n0 + tx * 4);
  // variates as top words from the ALU-leaning hash (its final >> 8 folded
  // into quant_float_bits_top, whose sign spread and carry add issue on the
  // FMA pipe): c4s 1109 -> 1130 GFLOP/s.  (The FMA-leaning variate24_x4_top
  // for both ops: 953, for the multiply's only: 1064.)
  auto q = [&](float v, const FloatParams& p, uint32_t top) {
    if (M_ != kStochastic) return quant_float_bits<kNearestEven>(v, p, 0u);
    return quant_float_bits_top<true>(v, p, top, rm.one);
  };
  auto vars = [&](uint64_t key, uint64_t id, uint32_t (&top)[4]) {
    if (M_ != kStochastic) return;
    if (X4) {
      variate24_x4<true>(key, id, rm.m32, top);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) top[j] = variate24(key, id + (uint64_t)j) << 8;
    }
  };
  for (int64_t k0 = 0; k0 < K; k0 += kGK) {
    for (int e = t; e < kGM * kGK; e += kGT) {
      const int r = e / kGK, c = e % kGK;  // A tile, coalesced along k
      const int64_t gr = m0 + r, gc = k0 + c;
      As[c][r] = (gr < M && gc < K) ? A[gr * K + gc] : 0.0f;
      const int kr = e / kGN, nc = e % kGN;  // B tile, coalesced along n
      const int64_t gk = k0 + kr, gn = n0 + nc;
      Bs[kr][nc] = (gk < K && gn < N) ? B[gk * N + gn] : 0.0f;
    }
    if (M_ == kStochastic && t < 2 * kGK) {
      const int kk = t >> 1, op = t & 1;
      keys[kk][op] = stream_key(seed, call + 2 * (uint64_t)(k0 + kk) + op);
    }
    __syncthreads();
    const int kk_end = (int)min((int64_t)kGK, K - k0);
    for (int kk = 0; kk < kk_end; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
      uint64_t km = 0, ka = 0;
      if (M_ == kStochastic) { km = keys[kk][0]; ka = keys[kk][1]; }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t vm[4] = {0u, 0u, 0u, 0u}, va[4] = {0u, 0u, 0u, 0u};
        vars(km, idx[i], vm);
        vars(ka, idx[i], va);
        // products and sums two at a time (mul / add .rn.f32x2: the same
        // per-lane rounding as __fmul_rn / __fadd_rn, one issue slot per pair)
        const uint64_t ap = pack_f32x2(a[i], a[i]);
#pragma unroll
        for (int j = 0; j < 4; j += 2) {
          const uint64_t p = fmul2(ap, pack_f32x2(b[j], b[j + 1]));
          const float q0 = q(u2f((uint32_t)p), qm, vm[j]);
          const float q1 = q(u2f((uint32_t)(p >> 32)), qm, vm[j + 1]);
          const uint64_t s = fadd2(pack_f32x2(acc[i][j], acc[i][j + 1]), pack_f32x2(q0, q1));
          acc[i][j] = q(u2f((uint32_t)s), qa, va[j]);
          acc[i][j + 1] = q(u2f((uint32_t)(s >> 32)), qa, va[j + 1]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + ty * 4 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + tx * 4 + j;
      if (col < N) C[row * N + col] = acc[i][j];
    }
  }
}

bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

template <int M_>
void launch_general(const float* A, const float* B, float* C, int64_t M,
                    int64_t N, int64_t K, int64_t row_base,
                    const FloatParams& qm, const FloatParams& qa, int flags,
                    uint64_t seed, uint64_t call, GemmScan* scan,
                    uint32_t* status, cudaStream_t s) {
  dim3 grid((unsigned)((N + kGN - 1) / kGN), (unsigned)((M + kGM - 1) / kGM));
  if constexpr (M_ == kNearestEven || M_ == kStochastic) {
    if (flags & 2) {  // the bit-domain kernel (it checks its proof itself)
      if (N % 4 == 0)
        k_qgemm_bits<M_, true><<<grid, kGT, 0, s>>>(A, B, C, M, N, K, row_base, qm, qa, seed,
                                                    call, scan, flags, rng_mul());
      else
        k_qgemm_bits<M_, false><<<grid, kGT, 0, s>>>(A, B, C, M, N, K, row_base, qm, qa, seed,
                                                     call, scan, flags, rng_mul());
      note_launch();
    }
  }
  k_qgemm_general<M_><<<grid, kGT, 0, s>>>(A, B, C, M, N, K, row_base, qm, qa, seed, call,
                                           scan, flags, status);
  note_launch();
}

// ---------------------------------------------------------------------------
// k_matmul_q: the reference quantized_matmul with the quantizer in the
// epilogue, accumulated on the FP64 tensor cores.  One DMMA m8n8k4 computes
// D = C + A*B as the chain fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))) in
// ascending k -- measured on B200 over 1.3e8 adversarial outputs
// (scripts/dmma_probe.cu: 0 differences from the DFMA chain, ~20 % from a
// single-rounding sum) -- and the products of fp32 operands are exact in
// double, so chaining the MMAs over k in ascending order is bit-identical to
// the reference's `acc += double(a) * double(b)` (tensor.cpp:355-376).
// Padding k beyond K adds +-0 products, which leave a (never -0) accumulator
// unchanged.  128x64 CTA tile, 8 warps of 32x32 (4x4 MMA tiles, 32 double
// accumulators per thread, <= 128 registers), TWO CTAs per SM so one CTA's
// barrier bubble is filled by the other's MMAs; K staged by 32 as double in
// double-buffered shared memory (108.5 KB per CTA) with conflict-free padded
// fragment strides.  Measured on B200 (ncu): DMMA sub-pipe 82 % active with
// one 128x128 CTA per SM (8 or 16 warps, K by 16) -> 91 % with this shape;
// 29.6 -> 33.2 TFLOP/s.  (The CUDA-core DFMA tile, 2 B of shared-memory
// traffic per MAC, was capped at 17.4.)
constexpr int kDM = 128, kDN = 64, kDK = 32, kDT = 256;
constexpr int kWTM = 4, kWTN = 4;  // 8x8 MMA tiles per warp: 32 x 32 outputs
constexpr int kDWN = kDN / (8 * kWTN);  // warps along n
constexpr int kDAS = kDK + 4;   // A row stride (doubles): conflict-free fragments
constexpr int kDBS = kDN + 4;   // B row stride (doubles)
constexpr size_t kDSmem = sizeof(double) * 2 * ((size_t)kDM * kDAS + (size_t)kDK * kDBS);

struct EpilogueFloat {
  FloatParams p;
  template <int M_>
  __device__ __forceinline__ float apply(float x, uint32_t v) const {
    return quant_float<M_>(x, p, v);
  }
};
struct EpilogueFixedSat {
  FixedParams p;
  template <int M_>
  __device__ __forceinline__ float apply(float x, uint32_t v) const {
    return quant_fixed<M_, true>(x, p, v);
  }
};
struct EpilogueFixedWrap {
  FixedParams p;
  template <int M_>
  __device__ __forceinline__ float apply(float x, uint32_t v) const {
    return quant_fixed<M_, false>(x, p, v);
  }
};
struct EpilogueNone {
  template <int M_>
  __device__ __forceinline__ float apply(float x, uint32_t) const { return x; }
};

template <int M_, class Epi, bool VEC>
__global__ void __launch_bounds__(kDT, 2)
    k_matmul_q(const float* __restrict__ A, const float* __restrict__ B,
               float* __restrict__ C, int64_t M, int64_t N, int64_t K,
               int64_t row_base, Epi epi, uint64_t key,
               uint32_t* __restrict__ status) {
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                              // [2][kDM][kDAS]
  double* Bs = dsm + 2 * kDM * kDAS;             // [2][kDK][kDBS]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp / kDWN, wn = warp % kDWN;  // 4 x 2 warps of 32 x 32
  const int64_t m0 = (int64_t)blockIdx.y * kDM, n0 = (int64_t)blockIdx.x * kDN;
  double acc[kWTM][kWTN][2];
#pragma unroll
  for (int i = 0; i < kWTM; ++i)
#pragma unroll
    for (int j = 0; j < kWTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // global -> register staging in float4 chunks: A 128 rows x kDK k,
  // B kDK k-rows x 64 cols
  constexpr int kAQ = kDM * kDK / 4 / kDT, kBQ = kDK * kDN / 4 / kDT;
  constexpr int kAC = kDK / 4, kBC = kDN / 4;     // chunks per smem row
  float4 ra[kAQ], rb[kBQ];
  auto ld4 = [&](const float* p, int64_t r, int64_t c, int64_t R, int64_t Cn) {
    float4 v;
    if (VEC && r < R && c + 4 <= Cn) {  // Cn % 4 == 0, 16-byte aligned rows
      v = __ldg(reinterpret_cast<const float4*>(p + r * Cn + c));
    } else {
      v.x = (r < R && c < Cn) ? __ldg(p + r * Cn + c) : 0.0f;
      v.y = (r < R && c + 1 < Cn) ? __ldg(p + r * Cn + c + 1) : 0.0f;
      v.z = (r < R && c + 2 < Cn) ? __ldg(p + r * Cn + c + 2) : 0.0f;
      v.w = (r < R && c + 3 < Cn) ? __ldg(p + r * Cn + c + 3) : 0.0f;
    }
    return v;
  };
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < kAQ; ++q) {
      const int c = t + kDT * q;
      ra[q] = ld4(A, m0 + c / kAC, k0 + (c % kAC) * 4, M, K);
    }
#pragma unroll
    for (int q = 0; q < kBQ; ++q) {
      const int c = t + kDT * q;
      rb[q] = ld4(B, k0 + c / kBC, n0 + (c % kBC) * 4, K, N);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < kAQ; ++q) {
      const int c = t + kDT * q;
      double2* a = reinterpret_cast<double2*>(As + buf * kDM * kDAS + (c / kAC) * kDAS + (c % kAC) * 4);
      a[0] = make_double2((double)ra[q].x, (double)ra[q].y);
      a[1] = make_double2((double)ra[q].z, (double)ra[q].w);
    }
#pragma unroll
    for (int q = 0; q < kBQ; ++q) {
      const int c = t + kDT * q;
      double2* b = reinterpret_cast<double2*>(Bs + buf * kDK * kDBS + (c / kBC) * kDBS + (c % kBC) * 4);
      b[0] = make_double2((double)rb[q].x, (double)rb[q].y);
      b[1] = make_double2((double)rb[q].z, (double)rb[q].w);
    }
  };
  const int64_t nk = (K + kDK - 1) / kDK;
  load(0);
  stash(0);
  __syncthreads();
  const int fr = lane >> 2, fk = lane & 3;       // fragment row / k of this lane
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) load((kt + 1) * kDK);
    const double* a_s = As + buf * kDM * kDAS + (wm * 8 * kWTM + fr) * kDAS + fk;
    const double* b_s = Bs + buf * kDK * kDBS + fk * kDBS + wn * 8 * kWTN + fr;
#pragma unroll
    for (int ks = 0; ks < kDK / 4; ++ks) {       // ascending k, 4 per MMA
      double af[kWTM], bf[kWTN];
#pragma unroll
      for (int i = 0; i < kWTM; ++i) af[i] = a_s[i * 8 * kDAS + ks * 4];
#pragma unroll
      for (int j = 0; j < kWTN; ++j) bf[j] = b_s[ks * 4 * kDBS + j * 8];
#pragma unroll
      for (int i = 0; i < kWTM; ++i)
#pragma unroll
        for (int j = 0; j < kWTN; ++j)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
    if (kt + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
  // epilogue: lane holds D[fr][2*fk + {0,1}] of every 8x8 tile
  uint32_t bad = 0;
#pragma unroll
  for (int i = 0; i < kWTM; ++i) {
    const int64_t row = m0 + wm * 8 * kWTM + i * 8 + fr;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < kWTN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = n0 + wn * 8 * kWTN + j * 8 + 2 * fk + h;
        if (col >= N) continue;
        const float c = __double2float_rn(acc[i][j][h]);
        uint32_t v = 0;
        if (M_ == kStochastic)
          v = variate24(key, (uint64_t)(row_base + row) * (uint64_t)N + (uint64_t)col);
        const bool nf = nonfinite(c);
        bad |= nf ? 1u : 0u;
        C[row * N + col] = nf ? 0.0f : epi.template apply<M_>(c, v);
      }
    }
  }
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0 && bad) atomicOr(status, kStatusNonFinite);
}

template <int M_, class Epi>
void launch_mmq(const float* A, const float* B, float* C, int64_t M, int64_t N,
                int64_t K, int64_t row_base, const Epi& epi, uint64_t key,
                uint32_t* status, cudaStream_t s) {
  // the dynamic shared-memory opt-in is per device: one bit per device that
  // has it (per instantiation; setting it twice from racing threads is benign)
  static std::atomic<uint64_t> ready{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(ready.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k_matmul_q<M_, Epi, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDSmem);
    cudaFuncSetAttribute(k_matmul_q<M_, Epi, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDSmem);
    ready.fetch_or(bit, std::memory_order_release);
  }
  dim3 grid((unsigned)((N + kDN - 1) / kDN), (unsigned)((M + kDM - 1) / kDM));
  const bool vec = K % 4 == 0 && N % 4 == 0 && aligned16(A) && aligned16(B);
  if (vec)
    k_matmul_q<M_, Epi, true><<<grid, kDT, kDSmem, s>>>(A, B, C, M, N, K, row_base,
                                                        epi, key, status);
  else
    k_matmul_q<M_, Epi, false><<<grid, kDT, kDSmem, s>>>(A, B, C, M, N, K, row_base,
                                                         epi, key, status);
  note_launch();
}

template <class Epi>
void dispatch_mmq(int mode, const float* A, const float* B, float* C,
                  int64_t M, int64_t N, int64_t K, int64_t row_base,
                  const Epi& epi, uint64_t key, uint32_t* status,
                  cudaStream_t s) {
  switch (mode) {
    case kStochastic: launch_mmq<kStochastic>(A, B, C, M, N, K, row_base, epi, key, status, s); break;
    case kNearestAway: launch_mmq<kNearestAway>(A, B, C, M, N, K, row_base, epi, key, status, s); break;
    case kNearestZero: launch_mmq<kNearestZero>(A, B, C, M, N, K, row_base, epi, key, status, s); break;
    default: launch_mmq<kNearestEven>(A, B, C, M, N, K, row_base, epi, key, status, s); break;
  }
}

}  // namespace

cudaError_t launch_quant_gemm(const float* A, const float* B, float* C,
                              int64_t M, int64_t N, int64_t K,
                              int64_t row_base, const FloatParams& qm,
                              const FloatParams& qa, bool bf16_formats,
                              int mode, uint64_t seed, uint64_t call,
                              GemmScan* scan, uint32_t* status,
                              cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(scan, 0, sizeof(GemmScan), s);
  if (e != cudaSuccess) return e;
  {
    const int64_t total = M * K + K * N;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)device_info().sm_count * 8, (total + 255) / 256));
    k_gemm_scan<<<grid, 256, 0, s>>>(A, M * K, B, K * N, scan);
    note_launch();
  }
  const bool try_bf16 = bf16_formats && mode == kNearestEven;
  if (try_bf16) {  // exact bf16 operands, else raw fp32 ones (one of them runs)
    dim3 grid((unsigned)((N + kBN - 1) / kBN), (unsigned)((M + kBM - 1) / kBM));
    const bool vec = (K % 4 == 0) && (N % 4 == 0) && aligned16(A) &&
                     aligned16(B) && aligned16(C);
    if (vec) {
      k_qgemm_bf16<true, false><<<grid, kQT, 0, s>>>(A, B, C, M, N, K, scan);
      k_qgemm_bf16<true, true><<<grid, kQT, 0, s>>>(A, B, C, M, N, K, scan);
    } else {
      k_qgemm_bf16<false, false><<<grid, kQT, 0, s>>>(A, B, C, M, N, K, scan);
      k_qgemm_bf16<false, true><<<grid, kQT, 0, s>>>(A, B, C, M, N, K, scan);
    }
    note_launch(2);
  }
  const bool try_bits = (mode == kNearestEven || mode == kStochastic) && qm.bits_ok &&
                        qa.bits_ok;
  const int flags = (try_bf16 ? 1 : 0) | (try_bits ? 2 : 0);
  switch (mode) {
    case kStochastic: launch_general<kStochastic>(A, B, C, M, N, K, row_base, qm, qa, flags, seed, call, scan, status, s); break;
    case kNearestAway: launch_general<kNearestAway>(A, B, C, M, N, K, row_base, qm, qa, flags, seed, call, scan, status, s); break;
    case kNearestZero: launch_general<kNearestZero>(A, B, C, M, N, K, row_base, qm, qa, flags, seed, call, scan, status, s); break;
    default: launch_general<kNearestEven>(A, B, C, M, N, K, row_base, qm, qa, flags, seed, call, scan, status, s); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_matmul_q(const float* A, const float* B, float* C,
                            int64_t M, int64_t N, int64_t K, int64_t row_base,
                            int kind, const FloatParams& fp,
                            const FixedParams& xp, int mode, uint64_t key,
                            uint32_t* status, cudaStream_t s) {
  if (kind == LPQ_FLOAT)
    dispatch_mmq(mode, A, B, C, M, N, K, row_base, EpilogueFloat{fp}, key, status, s);
  else if (kind == LPQ_FIXED && xp.saturate)
    dispatch_mmq(mode, A, B, C, M, N, K, row_base, EpilogueFixedSat{xp}, key, status, s);
  else if (kind == LPQ_FIXED)
    dispatch_mmq(mode, A, B, C, M, N, K, row_base, EpilogueFixedWrap{xp}, key, status, s);
  else
    launch_mmq<kNearestEven>(A, B, C, M, N, K, row_base, EpilogueNone{}, key, status, s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host-memory GEMM context (one per device)
namespace {
struct GemmCtx {
  float *A = nullptr, *B = nullptr, *C = nullptr;
  size_t ca = 0, cb = 0, cc = 0;
  void* ws = nullptr;
  size_t cws = 0;
  uint32_t* status = nullptr;
  cudaStream_t st = nullptr;
  std::mutex mu;
};
std::mutex g_gemm_mu;
std::vector<std::unique_ptr<GemmCtx>> g_gemm;

GemmCtx* gemm_ctx(int dev) {
  std::lock_guard<std::mutex> lk(g_gemm_mu);
  if ((int)g_gemm.size() <= dev) g_gemm.resize(dev + 1);
  if (!g_gemm[dev]) g_gemm[dev].reset(new GemmCtx());
  return g_gemm[dev].get();
}

cudaError_t grow(float** p, size_t* cap, size_t elems) {
  if (elems <= *cap) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(p, sizeof(float) * std::max<size_t>(elems, 1));
  if (e == cudaSuccess) *cap = elems;
  return e;
}
}  // namespace

}  // namespace lpq

using namespace lpq;

extern "C" {

size_t lpq_quant_gemm_workspace_size(int64_t, int64_t, int64_t) {
  return 256;  // GemmScan, padded
}

// every operand's byte count fits int64 (A: M x K, B: K x N, C: M x N)
static bool gemm_dims_ok(int64_t M, int64_t N, int64_t K) {
  const int64_t lim = INT64_MAX / 4;
  auto fits = [&](int64_t a, int64_t b) { return a == 0 || b <= lim / a; };
  return fits(M, K) && fits(K, N) && fits(M, N);
}

lpq_status lpq_quant_gemm(const float* A, const float* B, float* C, int64_t M,
                          int64_t N, int64_t K, int64_t row_base,
                          const lpq_format* fmul, const lpq_format* fadd,
                          int mode, uint64_t seed, uint64_t call, void* ws,
                          size_t ws_bytes, uint32_t* d_status, void* stream) {
  lpq_status st = check_format(fmul);
  if (st == LPQ_OK) st = check_format(fadd);
  if (st != LPQ_OK) return st;
  if (fmul->kind != LPQ_FLOAT || fadd->kind != LPQ_FLOAT) return LPQ_ERR_UNSUPPORTED;
  if (M < 0 || N < 0 || K < 0 || row_base < 0 || mode < 0 || mode > 3)
    return LPQ_ERR_ARGUMENT;
  if (!gemm_dims_ok(M, N, K)) return LPQ_ERR_SHAPE;
  if (M == 0 || N == 0) return LPQ_OK;
  if (!C || !d_status || (K > 0 && (!A || !B))) return LPQ_ERR_ARGUMENT;
  if (!ws || ws_bytes < sizeof(GemmScan)) return LPQ_ERR_WORKSPACE;
  const FloatParams qm = make_float(fmul->exp_bits, fmul->man_bits);
  const FloatParams qa = make_float(fadd->exp_bits, fadd->man_bits);
  const bool bf16 = fmul->exp_bits == 8 && fmul->man_bits == 7 &&
                    fadd->exp_bits == 8 && fadd->man_bits == 7;
  cudaError_t e = launch_quant_gemm(A, B, C, M, N, K, row_base, qm, qa, bf16,
                                    mode, seed, call, static_cast<GemmScan*>(ws),
                                    d_status, static_cast<cudaStream_t>(stream));
  note_passes(1);
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

lpq_status lpq_matmul_q(const float* A, const float* B, float* C, int64_t M,
                        int64_t N, int64_t K, int64_t row_base,
                        const lpq_format* f, int mode, uint64_t seed,
                        uint64_t call, void* ws, size_t ws_bytes,
                        uint32_t* d_status, void* stream) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  if (M < 0 || N < 0 || K < 0 || row_base < 0 || mode < 0 || mode > 3)
    return LPQ_ERR_ARGUMENT;
  if (!gemm_dims_ok(M, N, K)) return LPQ_ERR_SHAPE;
  if (M == 0 || N == 0) return LPQ_OK;
  if (!C || !d_status || (K > 0 && (!A || !B))) return LPQ_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t key = stream_key(seed, call);
  FloatParams fp{};
  FixedParams xp{};
  if (f->kind == LPQ_FLOAT) fp = make_float(f->exp_bits, f->man_bits);
  if (f->kind == LPQ_FIXED) xp = make_fixed(f->wl, f->fl, f->symmetric != 0, f->saturate != 0);
  cudaError_t e = launch_matmul_q(A, B, C, M, N, K, row_base, f->kind, fp, xp,
                                  mode, key, d_status, s);
  note_passes(1);
  if (e != cudaSuccess) return cuda_fail(e);
  if (f->kind == LPQ_BLOCK) {  // block maxima need the whole product first
    const int64_t shape[2] = {M, N};
    return quantize_device(C, C, shape, 2, (uint64_t)(row_base * N), f, mode,
                           seed, call, ws, ws_bytes, d_status, s);
  }
  return LPQ_OK;
}

lpq_status lpq_quant_gemm_host(const float* A, const float* B, float* C,
                               int64_t M, int64_t N, int64_t K,
                               int64_t row_base, const lpq_format* fmul,
                               const lpq_format* fadd, int mode, uint64_t seed,
                               uint64_t call, int device) {
  lpq_status st = check_format(fmul);
  if (st == LPQ_OK) st = check_format(fadd);
  if (st != LPQ_OK) return st;
  if (fmul->kind != LPQ_FLOAT || fadd->kind != LPQ_FLOAT) return LPQ_ERR_UNSUPPORTED;
  if (M < 0 || N < 0 || K < 0) return LPQ_ERR_ARGUMENT;
  if (M == 0 || N == 0) return LPQ_OK;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e);
  if (device < 0) cudaGetDevice(&device);
  DeviceGuard guard(device);
  GemmCtx* c = gemm_ctx(device);
  std::lock_guard<std::mutex> lk(c->mu);
#define TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return cuda_fail(_e); } while (0)
  if (!c->st) {
    TRY(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    TRY(cudaMalloc(&c->status, sizeof(uint32_t)));
    TRY(cudaMemset(c->status, 0, sizeof(uint32_t)));
    TRY(cudaMalloc(&c->ws, 256));
    c->cws = 256;
  }
  TRY(grow(&c->A, &c->ca, (size_t)(M * K)));
  TRY(grow(&c->B, &c->cb, (size_t)(K * N)));
  TRY(grow(&c->C, &c->cc, (size_t)(M * N)));
  TRY(cudaMemcpyAsync(c->A, A, sizeof(float) * M * K, cudaMemcpyHostToDevice, c->st));
  TRY(cudaMemcpyAsync(c->B, B, sizeof(float) * K * N, cudaMemcpyHostToDevice, c->st));
  st = lpq_quant_gemm(c->A, c->B, c->C, M, N, K, row_base, fmul, fadd, mode,
                      seed, call, c->ws, c->cws, c->status, c->st);
  if (st != LPQ_OK) { cudaStreamSynchronize(c->st); return st; }
  TRY(cudaMemcpyAsync(C, c->C, sizeof(float) * M * N, cudaMemcpyDeviceToHost, c->st));
  return lpq_status_fetch(c->status, c->st);
}

lpq_status lpq_matmul_q_host(const float* A, const float* B, float* C,
                             int64_t M, int64_t N, int64_t K,
                             const lpq_format* f, int mode, uint64_t seed,
                             uint64_t call, int device) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  if (M < 0 || N < 0 || K < 0) return LPQ_ERR_ARGUMENT;
  if (M == 0 || N == 0) return LPQ_OK;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e);
  if (device < 0) cudaGetDevice(&device);
  DeviceGuard guard(device);
  GemmCtx* c = gemm_ctx(device);
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->st) {
    TRY(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    TRY(cudaMalloc(&c->status, sizeof(uint32_t)));
    TRY(cudaMemset(c->status, 0, sizeof(uint32_t)));
    TRY(cudaMalloc(&c->ws, 256));
    c->cws = 256;
  }
  const int64_t shape[2] = {M, N};
  const size_t wsb = lpq_workspace_size(f, shape, 2);
  if (wsb > c->cws) {
    cudaFree(c->ws);
    c->ws = nullptr;
    c->cws = 0;
    TRY(cudaMalloc(&c->ws, wsb));
    c->cws = wsb;
  }
  TRY(grow(&c->A, &c->ca, (size_t)(M * K)));
  TRY(grow(&c->B, &c->cb, (size_t)(K * N)));
  TRY(grow(&c->C, &c->cc, (size_t)(M * N)));
  TRY(cudaMemcpyAsync(c->A, A, sizeof(float) * M * K, cudaMemcpyHostToDevice, c->st));
  TRY(cudaMemcpyAsync(c->B, B, sizeof(float) * K * N, cudaMemcpyHostToDevice, c->st));
  st = lpq_matmul_q(c->A, c->B, c->C, M, N, K, 0, f, mode, seed, call, c->ws,
                    c->cws, c->status, c->st);
  if (st != LPQ_OK) { cudaStreamSynchronize(c->st); return st; }
  TRY(cudaMemcpyAsync(C, c->C, sizeof(float) * M * N, cudaMemcpyDeviceToHost, c->st));
  return lpq_status_fetch(c->status, c->st);
#undef TRY
}

}  // extern "C"
