// Host build of the kernels' element math (paper_1910_04540_b200/csrc/
// quant_math.cuh) for CPU verification against the reference.
// TEST INFRASTRUCTURE ONLY: not part of the product library; exists so the
// exact source the sm_100a kernels inline can be swept over millions of
// inputs on a machine without a GPU.
#include <cstring>
#include <math.h>
#include <stdint.h>

#include "../../paper_1910_04540_b200/csrc/quant_math.cuh"

namespace {
struct Fmt { int32_t kind, exp_bits, man_bits, wl, fl, symmetric, saturate, block_dim; };

template <int M>
void run(const float* x, const uint32_t* v, float* y, int64_t n, const Fmt* f) {
  if (f->kind == 0) {
    // the kernels' dispatch: the streaming form for even/stochastic unless
    // |x| * 2^-min_exp can flush to zero
    const lpq::FloatParams p = lpq::make_float(f->exp_bits, f->man_bits);
    // the bit-domain form wherever the kernels may take it (zero or the
    // normal range of the format, after the clamp), the streaming forms
    // elsewhere
    if ((M == 0 || M == 1) && (p.scaled_ok || !p.tiny) && p.bits_ok) {
      for (int64_t i = 0; i < n; ++i) {
        const float xc = fminf(fmaxf(x[i], -p.max_value), p.max_value);
        const uint32_t vi = v ? v[i] : 0u;
        if (!(fabsf(xc) < p.min_normal && xc != 0.0f))
          y[i] = lpq::quant_float_bits<(M == 0 ? 0 : 1)>(xc, p, vi);
        else if (p.scaled_ok)
          y[i] = lpq::quant_float_scaled<(M == 0 ? 0 : 1)>(x[i], p, vi);
        else
          y[i] = lpq::quant_float_fast<(M == 0 ? 0 : 1)>(x[i], p, vi);
      }
    } else if ((M == 0 || M == 1) && p.scaled_ok)
      for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_float_scaled<(M == 0 ? 0 : 1)>(x[i], p, v ? v[i] : 0u);
    else if ((M == 0 || M == 1) && !p.tiny)
      for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_float_fast<(M == 0 ? 0 : 1)>(x[i], p, v ? v[i] : 0u);
    else
      for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_float<M>(x[i], p, v ? v[i] : 0u);
  } else if (f->saturate) {
    const lpq::FixedParams p = lpq::make_fixed(f->wl, f->fl, f->symmetric, true);
    // the kernels' dispatch: the underflow guard only when fl <= -1
    if (p.tiny)
      for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_fixed<M, true, true>(x[i], p, v ? v[i] : 0u);
    else
      for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_fixed_sat_fast<M>(x[i], p, v ? v[i] : 0u);
  } else {
    const lpq::FixedParams p = lpq::make_fixed(f->wl, f->fl, f->symmetric, false);
    for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_fixed<M, false>(x[i], p, v ? v[i] : 0u);
  }
}

template <int M>
void run_block(const float* x, const uint32_t* v, float* y, int64_t n, int wl,
               uint32_t max_bits, int* bad) {
  const lpq::BlockScale s = lpq::make_block_scale(max_bits, wl);
  *bad = s.bad;
  const float kmin = -(float)(1 << (wl - 1)), kmax = (float)((1 << (wl - 1)) - 1);
  const bool two = s.s2 != 1.0f || s.o2 != 1.0f;
  // the kernels' dispatch (block.cu)
  if ((M == 0 || M == 1) && two)
    for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_block_fast<(M == 0 ? 0 : 1), true>(x[i], s, kmin, kmax, v ? v[i] : 0u);
  else if (M == 0 || M == 1)
    for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_block_fast<(M == 0 ? 0 : 1), false>(x[i], s, kmin, kmax, v ? v[i] : 0u);
  else
    for (int64_t i = 0; i < n; ++i) y[i] = lpq::quant_block<M>(x[i], s, kmin, kmax, v ? v[i] : 0u);
}
}  // namespace

extern "C" {
// elementwise float/fixed with explicit 24-bit variates v (u = v * 2^-24)
void hm_quant(const float* x, const uint32_t* v, float* y, int64_t n, const Fmt* f, int mode) {
  switch (mode) {
    case 0: run<0>(x, v, y, n, f); break;
    case 1: run<1>(x, v, y, n, f); break;
    case 2: run<2>(x, v, y, n, f); break;
    default: run<3>(x, v, y, n, f); break;
  }
}
// one block with its maximum given as |x| bits
int hm_quant_block(const float* x, const uint32_t* v, float* y, int64_t n, int wl,
                   uint32_t max_bits, int mode) {
  int bad = 0;
  switch (mode) {
    case 0: run_block<0>(x, v, y, n, wl, max_bits, &bad); break;
    case 1: run_block<1>(x, v, y, n, wl, max_bits, &bad); break;
    case 2: run_block<2>(x, v, y, n, wl, max_bits, &bad); break;
    default: run_block<3>(x, v, y, n, wl, max_bits, &bad); break;
  }
  return bad;
}
uint32_t hm_variate24(uint64_t key, uint64_t index) { return lpq::variate24(key, index); }
void hm_variates24(uint64_t key, uint64_t base, int64_t n, uint32_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = lpq::variate24(key, base + (uint64_t)i);
}
// the kernels' pipe-balanced forms (must equal variate24)
void hm_variates24_balanced(uint64_t key, uint64_t base, int64_t n, uint32_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = lpq::variate24_zb(key ^ (base + (uint64_t)i), 32u);
}
void hm_variates24_fma(uint64_t key, uint64_t base, int64_t n, uint32_t* out) {
  const lpq::RngMul m = lpq::rng_mul();
  for (int64_t i = 0; i < n; ++i) out[i] = lpq::variate24_zf(key ^ (base + (uint64_t)i), m);
}
// the float4 form (idx % 4 == 0), n a multiple of 4
void hm_variates24_x4(uint64_t key, uint64_t base, int64_t n, uint32_t* out) {
  for (int64_t i = 0; i < n; i += 4) lpq::variate24_x4(key, base + (uint64_t)i, 32u, out + i);
}
// the ALU-leaning float4 form returning top words (variate = top >> 8)
void hm_variates24_x4_topw(uint64_t key, uint64_t base, int64_t n, uint32_t* out) {
  for (int64_t i = 0; i < n; i += 4) {
    lpq::variate24_x4<true>(key, base + (uint64_t)i, 32u, out + i);
    for (int q = 0; q < 4; ++q) out[i + q] >>= 8;
  }
}
// the top-word float4 form (variate = top >> 8)
void hm_variates24_x4_top(uint64_t key, uint64_t base, int64_t n, uint32_t* out) {
  const lpq::RngMul m = lpq::rng_mul();
  for (int64_t i = 0; i < n; i += 4) {
    lpq::variate24_x4_top(key, base + (uint64_t)i, m, out + i);
    for (int q = 0; q < 4; ++q) out[i + q] >>= 8;
  }
}
// stochastic bit-domain float quantizer from top words (v << 8 | junk):
// clamped inputs in the bit-domain range only (the caller filters)
void hm_quant_float_bits_top(const float* x, const uint32_t* top, float* y, int64_t n,
                             int exp_bits, int man_bits) {
  const lpq::FloatParams p = lpq::make_float(exp_bits, man_bits);
  for (int64_t i = 0; i < n; ++i) {
    const float xc = fminf(fmaxf(x[i], -p.max_value), p.max_value);
    y[i] = lpq::quant_float_bits_top<false>(xc, p, top[i], 1u);
    // the FMA-pipe form (the GEMM's) must agree bit for bit
    const float yf = lpq::quant_float_bits_top<true>(xc, p, top[i], 1u);
    if (memcmp(&yf, &y[i], 4) != 0) y[i] = __builtin_nanf("0x7ABCD");
  }
}
void hm_quant_float_bits(const float* x, const uint32_t* v, float* y, int64_t n,
                         int exp_bits, int man_bits) {
  const lpq::FloatParams p = lpq::make_float(exp_bits, man_bits);
  for (int64_t i = 0; i < n; ++i) {
    const float xc = fminf(fmaxf(x[i], -p.max_value), p.max_value);
    y[i] = lpq::quant_float_bits<0>(xc, p, v[i]);
  }
}
uint64_t hm_stream_key(uint64_t seed, uint64_t call) { return lpq::stream_key(seed, call); }
}
