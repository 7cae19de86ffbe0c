/*
 * lpq_oracle.c -- CPU restatement of the reference quantizer hot path.
 * TEST INFRASTRUCTURE ONLY (see lpq_oracle.h).  Compiled with
 * -ffp-contract=off and without fast-math so every double operation is a
 * single IEEE-754 round-to-nearest step, as in the reference.
 */
#include "lpq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng: proj/include/lpsim/rng.hpp:17-36 ---------------------------- */

uint64_t lpqo_mix64(uint64_t z) {
  /* splitmix64 finalizer (rng.hpp:17-22) */
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t lpqo_stream_key(uint64_t seed, uint64_t call) {
  return lpqo_mix64(lpqo_mix64(seed) ^ call); /* rng.hpp:25-27 */
}

float lpqo_variate_from_key(uint64_t key, uint64_t index) {
  /* top 24 bits scaled by 2^-24 (rng.hpp:34-36) */
  return (float)(lpqo_mix64(key ^ index) >> 40) * 0x1.0p-24f;
}

float lpqo_uniform_variate(uint64_t seed, uint64_t call, uint64_t index) {
  return lpqo_variate_from_key(lpqo_stream_key(seed, call), index);
}

/* ---- exact double rounding: proj/include/lpsim/rounding.hpp:16-85 ------ */

static double o_floor(double r) {
  /* rounding.hpp:16-20: integers beyond 2^52 pass through; below, the
     int64 truncation is exact */
  if (!(r < 0x1p52 && r > -0x1p52)) return r;
  double t = (double)(int64_t)r;
  return t > r ? t - 1.0 : t;
}

static double o_half_even(double r) {
  /* rounding.hpp:27-37 */
  if (r < 0x1p51 && r > -0x1p51) {
    volatile double s = r + 0x1.8p52; /* volatile: keep the two roundings */
    return s - 0x1.8p52;
  }
  if (!(r < 0x1p52 && r > -0x1p52)) return r;
  double f = o_floor(r);
  if (r == f) return r;
  return (((int64_t)f) & 1) == 0 ? f : f + 1.0;
}

static double o_half_away(double r) {
  /* rounding.hpp:41-46 */
  double a = r < 0.0 ? -r : r;
  if (a >= 0x1p52) return r;
  double k = o_floor(a + 0.5);
  return r < 0.0 ? -k : k;
}

static double o_half_zero(double r) {
  /* rounding.hpp:49-54 */
  double a = r < 0.0 ? -r : r;
  if (a >= 0x1p52) return r;
  double k = -o_floor(0.5 - a);
  return r < 0.0 ? -k : k;
}

static double o_stochastic(double r, double u) {
  double f = o_floor(r); /* rounding.hpp:56-59 */
  return f + (u < r - f ? 1.0 : 0.0);
}

double lpqo_round_integer(double r, int mode, double u) {
  switch (mode) {
  case LPQO_STOCHASTIC: return o_stochastic(r, u);
  case LPQO_NEAREST_AWAY: return o_half_away(r);
  case LPQO_NEAREST_ZERO: return o_half_zero(r);
  default: return o_half_even(r);
  }
}

/* ---- formats: proj/include/lpsim/formats.hpp:36-112 -------------------- */

static int f_bias(const lpqo_format* f) { return (1 << (f->exp_bits - 1)) - 1; }
static int f_min_exp(const lpqo_format* f) { return 1 - f_bias(f); }
static int f_max_exp(const lpqo_format* f) {
  int e = (1 << f->exp_bits) - 1 - f_bias(f);
  return e < 127 ? e : 127;
}

int lpqo_validate(const lpqo_format* f) {
  switch (f->kind) {
  case LPQO_FLOAT:
    if (f->exp_bits < 1 || f->exp_bits > 8) return LPQO_FORMAT_ERROR;
    if (f->man_bits < 0 || f->man_bits > 23) return LPQO_FORMAT_ERROR;
    return LPQO_OK;
  case LPQO_FIXED:
    if (f->wl < 2 || f->wl > 24) return LPQO_FORMAT_ERROR;
    if (f->fl < f->wl - 128 || f->fl > 126) return LPQO_FORMAT_ERROR;
    return LPQO_OK;
  case LPQO_BLOCK:
    if (f->wl < 2 || f->wl > 24) return LPQO_FORMAT_ERROR;
    /* block_dim: -1 encodes "whole tensor"; other negatives are rejected
       like formats.hpp:105-107 */
    if (f->block_dim < -1) return LPQO_FORMAT_ERROR;
    return LPQO_OK;
  default:
    return LPQO_FORMAT_ERROR;
  }
}

/* ---- scalar primitives: proj/include/lpsim/scalar_quant.hpp ------------ */

static double p2(int e) { return ldexp(1.0, e); } /* exact, pow2i :19-21 */

static int o_float_exponent(float x) {
  /* scalar_quant.hpp:26-33: exponent field, or leading-bit position for
     denormals */
  uint32_t bits;
  memcpy(&bits, &x, 4);
  bits &= 0x7FFFFFFFu;
  int field = (int)(bits >> 23);
  if (field != 0) return field - 127;
  return -118 - __builtin_clz(bits);
}

static double o_fixed_fold(double k, const lpqo_format* f) {
  /* FixedFolder::fold, scalar_quant.hpp:50-62 */
  double kmax = (double)((1ll << (f->wl - 1)) - 1);
  double kmin = f->symmetric ? -kmax : -(double)(1ll << (f->wl - 1));
  if (f->saturate) {
    if (k > kmax) return kmax;
    if (k < kmin) return kmin;
    return k;
  }
  double span = p2(f->wl), half = p2(f->wl - 1);
  double m = fmod(k, span);
  if (m < 0.0) m += span;
  if (m >= half) m -= span;
  if (m < kmin) m = kmin;
  return m;
}

float lpqo_quant_fixed(float x, const lpqo_format* f, int mode, float u) {
  /* quantize_scalar_fixed, scalar_quant.hpp:145-153, and the fused lambda
     quant_ops.cpp:41-48 (identical arithmetic) */
  double r = (double)x * p2(f->fl);
  double k = o_fixed_fold(lpqo_round_integer(r, mode, (double)u), f);
  return (float)(k * p2(-f->fl));
}

static float o_float_apply(float x, const lpqo_format* f, int mode, double u) {
  /* FloatQuantizer::apply_m, scalar_quant.hpp:117-134 (x nonzero) */
  int man = f->man_bits, emin = f_min_exp(f), emax = f_max_exp(f);
  double maxv = ldexp(2.0 - ldexp(1.0, -man), emax);
  int e = o_float_exponent(x);
  if (e < emin) {
    double k = lpqo_round_integer((double)x * p2(-emin), mode, u);
    return (float)(k * p2(emin));
  }
  int E = e > emax ? emax : e;
  double k = lpqo_round_integer((double)x * p2(man - E), mode, u);
  double q = k * p2(E - man);
  if (q > maxv) return (float)maxv;
  if (q < -maxv) return (float)(-maxv);
  return (float)q;
}

float lpqo_quant_float(float x, const lpqo_format* f, int mode, float u) {
  if (x == 0.0f) return x; /* scalar_quant.hpp:163, quant_ops.cpp:59 */
  return o_float_apply(x, f, mode, (double)u);
}

/* ---- tensor level: proj/src/quant_ops.cpp + tensor.cpp ----------------- */

static int64_t o_numel(const int64_t* shape, int rank) {
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) n *= shape[d];
  return n;
}

int lpqo_reduce_max_abs(const float* x, const int64_t* shape, int rank,
                        int block_dim, float* out) {
  /* tensor.cpp:320-353: `a > m` skips NaN */
  int64_t n = o_numel(shape, rank);
  if (block_dim < 0) {
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
      float a = fabsf(x[i]);
      if (a > m) m = a;
    }
    out[0] = m;
    return LPQO_OK;
  }
  if (block_dim >= rank) return LPQO_SHAPE_ERROR;
  int64_t extent = shape[block_dim], inner = 1;
  for (int d = block_dim + 1; d < rank; ++d) inner *= shape[d];
  for (int64_t c = 0; c < extent; ++c) out[c] = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = (i / inner) % extent;
    float a = fabsf(x[i]);
    if (a > out[c]) out[c] = a;
  }
  return LPQO_OK;
}

int lpqo_quantize_block_given_max(const float* x, float* y, const int64_t* shape,
                                  int rank, uint64_t index_base,
                                  const lpqo_format* f, int mode, uint64_t seed,
                                  uint64_t call, const float* mx) {
  /* fused_block pass 2 (quant_ops.cpp:73-115) with the block maxima given */
  int st = lpqo_validate(f);
  if (st) return st;
  if (f->kind != LPQO_BLOCK) return LPQO_UNSUPPORTED;
  if (f->block_dim >= 0 && f->block_dim >= rank) return LPQO_SHAPE_ERROR;
  int64_t n = o_numel(shape, rank);
  uint64_t key = lpqo_stream_key(seed, call);
  int bad = 0;
  int64_t blocks = f->block_dim < 0 ? 1 : shape[f->block_dim];
  double* delta = (double*)malloc(sizeof(double) * (size_t)(blocks ? blocks : 1));
  double* inv = (double*)malloc(sizeof(double) * (size_t)(blocks ? blocks : 1));
  for (int64_t b = 0; b < blocks; ++b) {
    if (mx[b] == 0.0f) { delta[b] = 0.0; inv[b] = 0.0; continue; }
    int E = o_float_exponent(mx[b]);
    if (E > 126) { /* check_block_range, scalar_quant.hpp:72-77 */
      free(delta); free(inv);
      return LPQO_INVALID_INPUT;
    }
    int shift = E - (f->wl - 2);
    delta[b] = p2(shift);
    inv[b] = p2(-shift);
  }
  int64_t stride = 1, extent = 1;
  if (f->block_dim >= 0) {
    extent = shape[f->block_dim];
    for (int d = f->block_dim + 1; d < rank; ++d) stride *= shape[d];
  }
  double kmax = (double)((1ll << (f->wl - 1)) - 1);
  double kmin = -p2(f->wl - 1);
  for (int64_t i = 0; i < n; ++i) {
    float v = x[i];
    if (!isfinite(v)) { bad = 1; y[i] = 0.0f; continue; }
    int64_t b = f->block_dim < 0 ? 0 : (i / stride) % extent;
    if (delta[b] == 0.0) { y[i] = 0.0f; continue; }
    double u = mode == LPQO_STOCHASTIC
                   ? (double)lpqo_variate_from_key(key, index_base + (uint64_t)i)
                   : 0.0;
    /* block_quant_one_m, scalar_quant.hpp:80-87 */
    double k = lpqo_round_integer((double)v * inv[b], mode, u);
    if (k > kmax) k = kmax;
    if (k < kmin) k = kmin;
    y[i] = (float)(k * delta[b]);
  }
  free(delta); free(inv);
  return bad ? LPQO_INVALID_INPUT : LPQO_OK;
}

int lpqo_quantize(const float* x, float* y, const int64_t* shape, int rank,
                  uint64_t index_base, const lpqo_format* f, int mode,
                  uint64_t seed, uint64_t call) {
  int st = lpqo_validate(f); /* quant_ops.cpp:156 */
  if (st) return st;
  int64_t n = o_numel(shape, rank);
  uint64_t key = lpqo_stream_key(seed, call);
  int bad = 0;
  if (f->kind == LPQO_BLOCK) {
    /* fused_block, quant_ops.cpp:68-115: pass 1 (the maxima), pass 2 */
    if (f->block_dim >= 0 && f->block_dim >= rank) return LPQO_SHAPE_ERROR;
    int64_t blocks = f->block_dim < 0 ? 1 : shape[f->block_dim];
    float* mx = (float*)malloc(sizeof(float) * (size_t)(blocks ? blocks : 1));
    lpqo_reduce_max_abs(x, shape, rank, f->block_dim, mx);
    st = lpqo_quantize_block_given_max(x, y, shape, rank, index_base, f, mode, seed,
                                       call, mx);
    free(mx);
    return st;
  }
  for (int64_t i = 0; i < n; ++i) {
    float v = x[i];
    if (!isfinite(v)) { bad = 1; y[i] = 0.0f; continue; } /* quant_ops.cpp:21-25 */
    float u = mode == LPQO_STOCHASTIC
                  ? lpqo_variate_from_key(key, index_base + (uint64_t)i)
                  : 0.0f;
    y[i] = f->kind == LPQO_FIXED ? lpqo_quant_fixed(v, f, mode, u)
                                 : lpqo_quant_float(v, f, mode, u);
  }
  return bad ? LPQO_INVALID_INPUT : LPQO_OK;
}

void lpqo_random_uniform(float* y, int64_t n, uint64_t index_base,
                         uint64_t seed, uint64_t call, float lo, float hi) {
  /* tensor.cpp:430-440 */
  double l = lo, h = hi;
  uint64_t key = lpqo_stream_key(seed, call);
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)lpqo_variate_from_key(key, index_base + (uint64_t)i);
    y[i] = (float)(l + (h - l) * u);
  }
}

void lpqo_matmul(const float* a, const float* b, float* c, int64_t m,
                 int64_t k, int64_t n) {
  /* tensor.cpp:355-376: double accumulator, ascending k */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t kk = 0; kk < k; ++kk)
        acc += (double)a[i * k + kk] * (double)b[kk * n + j];
      c[i * n + j] = (float)acc;
    }
}

static float o_q_op(float v, const lpqo_format* f, int mode, float u) {
  /* Q of the per-op GEMM: apply_m with the zero passthrough; non-finite
     intermediates saturate through apply_m's own arithmetic (E clamps to
     max_exp, q compares beyond max_value); NaN passes through. */
  if (v == 0.0f) return v;
  if (isnan(v)) return v;
  return o_float_apply(v, f, mode, (double)u);
}

int lpqo_quant_gemm(const float* a, const float* b, float* c, int64_t M,
                    int64_t N, int64_t K, int64_t row_base, int64_t r0,
                    int64_t r1, const lpqo_format* fmul,
                    const lpqo_format* fadd, int mode, uint64_t seed,
                    uint64_t call) {
  int st = lpqo_validate(fmul);
  if (st) return st;
  st = lpqo_validate(fadd);
  if (st) return st;
  if (fmul->kind != LPQO_FLOAT || fadd->kind != LPQO_FLOAT)
    return LPQO_UNSUPPORTED;
  (void)M;
  uint64_t* keys = NULL;
  if (mode == LPQO_STOCHASTIC) {
    keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(2 * K + 1));
    for (int64_t k = 0; k < 2 * K; ++k)
      keys[k] = lpqo_stream_key(seed, call + (uint64_t)k);
  }
  for (int64_t i = r0; i < r1; ++i)
    for (int64_t j = 0; j < N; ++j) {
      uint64_t idx = (uint64_t)(row_base + i) * (uint64_t)N + (uint64_t)j;
      float acc = 0.0f;
      for (int64_t k = 0; k < K; ++k) {
        float um = 0.0f, ua = 0.0f;
        if (keys) {
          um = lpqo_variate_from_key(keys[2 * k], idx);
          ua = lpqo_variate_from_key(keys[2 * k + 1], idx);
        }
        float p = (float)((double)a[i * K + k] * (double)b[k * N + j]);
        p = o_q_op(p, fmul, mode, um);
        float s = (float)((double)acc + (double)p);
        acc = o_q_op(s, fadd, mode, ua);
      }
      c[i * N + j] = acc;
    }
  free(keys);
  return LPQO_OK;
}
