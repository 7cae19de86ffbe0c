/*
 * lpq_oracle.h -- CPU restatement of the reference quantizer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (liblpq.so, the lpsim
 * drop-in shim, the Python mirror) may include, link or call this code.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs use it, and only as the checker.
 *
 * Parity pinning: this restatement is checked against
 *   (1) the golden vectors of the reference's own unit tests
 *       (proj/tests/test_rng_rounding.cpp, test_scalar_quant.cpp,
 *       test_quant_ops.cpp; transcribed in tests/test_oracle_golden.py), and
 *   (2) the reference library itself, compiled from /root/reference sources
 *       into oracle/_ref/liblpsim_ref.so (oracle/Makefile), through fixtures
 *       committed under tests/golden/ (tests/golden/make_golden.py).
 * The per-op-rounded GEMM (lpqo_quant_gemm) has no reference implementation;
 * it is a restatement built from the reference's scalar primitives and is
 * "parity unpinned" for its rounding order.
 *
 * The oracle is deliberately written in plain C with double arithmetic, the
 * way the reference computes (proj/include/lpsim/rounding.hpp), and not with
 * the integer/fp32 tricks the CUDA kernels use, so that the two are
 * independent implementations of the same semantics.
 */
#ifndef LPQ_ORACLE_H
#define LPQ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* RoundingMode order of proj/include/lpsim/formats.hpp:14-19 */
enum { LPQO_STOCHASTIC = 0, LPQO_NEAREST_EVEN = 1, LPQO_NEAREST_AWAY = 2,
       LPQO_NEAREST_ZERO = 3 };
enum { LPQO_FLOAT = 0, LPQO_FIXED = 1, LPQO_BLOCK = 2 };
/* status codes (mirror the reference exception taxonomy,
   proj/include/lpsim/errors.hpp:9-55) */
enum { LPQO_OK = 0, LPQO_FORMAT_ERROR = 1, LPQO_SHAPE_ERROR = 2,
       LPQO_INVALID_INPUT = 3, LPQO_UNSUPPORTED = 4 };

typedef struct {
  int32_t kind;       /* LPQO_FLOAT / LPQO_FIXED / LPQO_BLOCK */
  int32_t exp_bits;   /* float */
  int32_t man_bits;   /* float */
  int32_t wl;         /* fixed, block */
  int32_t fl;         /* fixed */
  int32_t symmetric;  /* fixed */
  int32_t saturate;   /* fixed */
  int32_t block_dim;  /* block: -1 = whole tensor */
} lpqo_format;

/* rng.hpp:17-36 */
uint64_t lpqo_mix64(uint64_t z);
uint64_t lpqo_stream_key(uint64_t seed, uint64_t call);
float lpqo_variate_from_key(uint64_t key, uint64_t index);
float lpqo_uniform_variate(uint64_t seed, uint64_t call, uint64_t index);

/* rounding.hpp:16-85 (round_integer_m); u used only for stochastic */
double lpqo_round_integer(double r, int mode, double u);

/* formats.hpp:82-112 */
int lpqo_validate(const lpqo_format* f);

/* scalar quantizers, scalar_quant.hpp:145-196 (x finite) */
float lpqo_quant_fixed(float x, const lpqo_format* f, int mode, float u);
float lpqo_quant_float(float x, const lpqo_format* f, int mode, float u);

/* Tensor-level fused quantization, quant_ops.cpp:13-164: output[i] for the
   flat index i uses the variate of (seed, call, index_base + i).  Returns a
   status code; on error the output content is unspecified (the reference
   discards it). */
int lpqo_quantize(const float* x, float* y, const int64_t* shape, int rank,
                  uint64_t index_base, const lpqo_format* f, int mode,
                  uint64_t seed, uint64_t call);

/* fused_block's quantization pass (quant_ops.cpp:73-115) with the block
   maxima mx[extent] given (e.g. combined across shards). */
int lpqo_quantize_block_given_max(const float* x, float* y, const int64_t* shape,
                                  int rank, uint64_t index_base,
                                  const lpqo_format* f, int mode, uint64_t seed,
                                  uint64_t call, const float* mx);

/* Per-block maxima as reduce_max_abs (tensor.cpp:320-353): whole tensor
   (block_dim < 0) gives one value. */
int lpqo_reduce_max_abs(const float* x, const int64_t* shape, int rank,
                        int block_dim, float* out);

/* random_uniform (tensor.cpp:430-440) over flat indices
   [index_base, index_base + n). */
void lpqo_random_uniform(float* y, int64_t n, uint64_t index_base,
                         uint64_t seed, uint64_t call, float lo, float hi);

/* matmul with a double accumulator, ascending k (tensor.cpp:355-376). */
void lpqo_matmul(const float* a, const float* b, float* c, int64_t m,
                 int64_t k, int64_t n);

/* Per-op-rounded GEMM restated from the reference primitives (SURVEY §8(a)
   A8, §8(c)):
     acc = +0f
     for k in 0..K-1:
       p   = Q_mul(fl32(a_ik * b_kj))      variate (seed, call + 2k,   idx)
       acc = Q_add(fl32(acc + p))          variate (seed, call + 2k+1, idx)
   idx = (row_base + i) * N + j; fl32(x op y) = float(double(x) op double(y))
   (tensor.cpp:140-156); Q = FloatQuantizer::apply_m with the x == 0
   passthrough of quantize_scalar_float (scalar_quant.hpp:117-165), applied
   also to non-finite intermediates (saturating), see DESIGN.md.
   Only rows [r0, r1) of C are computed (to bound test time). */
int lpqo_quant_gemm(const float* a, const float* b, float* c, int64_t M,
                    int64_t N, int64_t K, int64_t row_base, int64_t r0,
                    int64_t r1, const lpqo_format* fmul,
                    const lpqo_format* fadd, int mode, uint64_t seed,
                    uint64_t call);

#ifdef __cplusplus
}
#endif

#endif
