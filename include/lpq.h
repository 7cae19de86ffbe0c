/*
 * lpq.h -- C ABI of the B200-native fused quantization library (liblpq.so).
 *
 * This is the drop-in boundary for the reference's quantizer hot path
 * (lpsim, proj/include/lpsim/quant_ops.hpp:23-46).  Every entry point is
 * extern "C" with plain pointers and sizes; no exception crosses it.  The C++
 * shim that restores the reference's exact C++ API over these calls is
 * paper_1910_04540_b200/csrc/dropin/quant_ops_b200.cpp.
 *
 * Two families:
 *   * device entry points (lpq_quantize, lpq_quant_gemm, lpq_matmul_q, ...):
 *     device pointers, asynchronous on the caller's CUDA stream, no
 *     allocation, no synchronisation.  Data-dependent errors (non-finite
 *     input, block maximum out of range) are OR-ed into a caller-owned device
 *     status word; lpq_status_fetch() turns it into an lpq_status.
 *   * host entry points (lpq_quantize_host, lpq_quant_gemm_host, ...): host
 *     pointers (pinned or pageable), synchronous, returning the final status.
 *     They stage through a per-device context (streams, device buffers,
 *     pinned bounce buffers) and overlap host<->device copies with the
 *     kernels chunk by chunk.
 *
 * Semantics are bit-exact with the reference for every format and rounding
 * mode, including stochastic rounding: the variate of flat element i is the
 * reference's uniform_variate(seed, call, index_base + i)
 * (proj/include/lpsim/rng.hpp:43-46).
 */
#ifndef LPQ_H
#define LPQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPQ_ABI_VERSION 1

/* Status codes.  Each maps to one exception type of the reference
 * (proj/include/lpsim/errors.hpp:9-55). */
typedef enum {
  LPQ_OK = 0,
  LPQ_ERR_FORMAT = 1,        /* format_error           (formats.hpp:82-108)   */
  LPQ_ERR_SHAPE = 2,         /* shape_error            (quant_ops.cpp:70-71)  */
  LPQ_ERR_INVALID_INPUT = 3, /* invalid_input_error: non-finite input
                                (quant_ops.cpp:28-29)                        */
  LPQ_ERR_UNSUPPORTED = 4,   /* unsupported_format_error (quant_ops.cpp:169) */
  LPQ_ERR_BLOCK_RANGE = 5,   /* invalid_input_error: block maximum >= 2^127
                                (scalar_quant.hpp:72-77)                      */
  LPQ_ERR_ARGUMENT = 6,      /* null pointer, negative extent, bad mode     */
  LPQ_ERR_WORKSPACE = 7,     /* workspace too small                          */
  LPQ_ERR_CUDA = 8,          /* CUDA runtime error (lpq_last_cuda_error)     */
  LPQ_ERR_NO_DEVICE = 9,     /* no CUDA device / driver                      */
  LPQ_ERR_INVALID_VALUE = 10 /* invalid_value_error: non-finite result of a
                                composed-chain op (tensor.cpp:58-78)         */
} lpq_status;

/* Rounding modes, in the order of proj/include/lpsim/formats.hpp:14-19. */
typedef enum {
  LPQ_STOCHASTIC = 0,
  LPQ_NEAREST_EVEN = 1,
  LPQ_NEAREST_AWAY = 2,
  LPQ_NEAREST_ZERO = 3
} lpq_rounding;

typedef enum { LPQ_FLOAT = 0, LPQ_FIXED = 1, LPQ_BLOCK = 2 } lpq_kind;

/* One NumberFormat (proj/include/lpsim/formats.hpp:36-80) as a flat struct:
 *   LPQ_FLOAT : exp_bits in [1,8], man_bits in [0,23]        (FloatFormat)
 *   LPQ_FIXED : wl in [2,24], fl in [wl-128,126], symmetric, saturate
 *                                                            (FixedFormat)
 *   LPQ_BLOCK : wl in [2,24], block_dim = -1 (whole tensor) or d >= 0
 *                                                       (BlockFloatFormat) */
typedef struct {
  int32_t kind;
  int32_t exp_bits;
  int32_t man_bits;
  int32_t wl;
  int32_t fl;
  int32_t symmetric;
  int32_t saturate;
  int32_t block_dim;
} lpq_format;

/* ---- host-only helpers (no GPU needed) ---------------------------------- */

int lpq_abi_version(void);
const char* lpq_status_string(lpq_status s);
/* validate(fmt): proj/include/lpsim/formats.hpp:82-112 */
lpq_status lpq_validate_format(const lpq_format* f);
/* Device workspace the device entry points need for this (format, shape):
 * block formats -- the per-block maxima of the two-pass plans, or the row
 * maxima and arrival counters of the single-pass chunk plan for rows of
 * 32K+ floats (whichever is larger; the device call zeroes what it uses).
 * 0 for float/fixed.  A block call given no workspace takes a
 * workspace-free plan where one exists (rows of 32K..1M floats: thread-block
 * clusters) and returns LPQ_ERR_WORKSPACE otherwise. */
size_t lpq_workspace_size(const lpq_format* f, const int64_t* shape, int rank);
/* Number of kernel launches issued by this library so far (for benches). */
uint64_t lpq_launch_count(void);
/* Data-pass counter, the analogue of lpsim::pass_count / bump_pass
 * (proj/include/lpsim/tensor.hpp:52-66, tensor.cpp:302-311): one per HBM
 * pass a quantize call makes (1 for float/fixed and single-pass block,
 * 2 for two-pass block). */
uint64_t lpq_pass_count(void);
void lpq_reset_pass_count(void);
/* The last CUDA error string seen by the library (thread-local). */
const char* lpq_last_cuda_error(void);

/* ---- device entry points (stream-ordered, no allocation) ---------------- */

/* quantize_fused_at (proj/src/quant_ops.cpp:154-164) on device memory.
 *   x, y        : device fp32, row-major, numel = prod(shape); y may equal x
 *   index_base  : flat index of x[0] in the full tensor (RNG counter offset
 *                 for shards; 0 for a whole tensor)
 *   mode        : lpq_rounding; seed/call: RngStream seed and call id
 *   ws          : device workspace of >= lpq_workspace_size() bytes; calls
 *                 that may run concurrently (different streams) need their
 *                 own workspaces
 *   d_status    : device uint32 the kernels OR error bits into (the caller
 *                 zeroes it; read it with lpq_status_fetch)
 *   stream      : cudaStream_t (NULL = legacy default stream) */
lpq_status lpq_quantize(const float* x, float* y, const int64_t* shape,
                        int rank, uint64_t index_base, const lpq_format* f,
                        int mode, uint64_t seed, uint64_t call, void* ws,
                        size_t ws_bytes, uint32_t* d_status, void* stream);

/* Block formats split across shards (a whole-tensor block, or
 * blocks along dim d >= 1 of a tensor sharded along dim 0) need ONE exchange
 * step: every shard reduces its part of each block's maximum, the maxima are
 * combined with an elementwise max across shards (ncclAllReduce(MAX) on
 * `extent` uint32s: non-negative float bits order like the floats), then
 * every shard quantizes with the global maxima.  Both halves of fused_block
 * (proj/src/quant_ops.cpp:68-115; reduce_max_abs, tensor.cpp:320-353).
 *   lpq_block_absmax: maxima[extent] := max|x| bits over this tensor's part
 *     of each block (NaN ignored; extent = shape[block_dim], 1 for the whole
 *     tensor).  Device uint32 array, overwritten.
 *   lpq_quantize_block_apply: the quantization pass with the given maxima;
 *     index_base as in lpq_quantize (the shard's first global flat index).
 *     Flags non-finite inputs and out-of-range maxima in *d_status. */
lpq_status lpq_block_absmax(const float* x, const int64_t* shape, int rank,
                            const lpq_format* f, uint32_t* maxima, void* stream);
lpq_status lpq_quantize_block_apply(const float* x, float* y, const int64_t* shape,
                                    int rank, uint64_t index_base,
                                    const lpq_format* f, int mode, uint64_t seed,
                                    uint64_t call, const uint32_t* maxima,
                                    uint32_t* d_status, void* stream);

/* Synchronise `stream`, read and clear *d_status, map the bits to a status
 * (LPQ_ERR_BLOCK_RANGE takes precedence over LPQ_ERR_INVALID_INPUT, as the
 * reference's reduction pass throws before its quantization pass). */
lpq_status lpq_status_fetch(uint32_t* d_status, void* stream);

/* Per-op-rounded GEMM (no reference implementation; restated in
 * oracle/lpq_oracle.h from quant_ops.cpp + scalar_quant.hpp primitives):
 *   C[i][j]: acc = +0; for k = 0..K-1 (sequential):
 *              acc = Q_add(fl32(acc + Q_mul(fl32(A[i][k] * B[k][j]))))
 * A is MxK, B is KxN, C is MxN, row-major device fp32.  fmul/fadd must be
 * float formats.  Stochastic variates: (seed, call + 2k) for Q_mul and
 * (seed, call + 2k + 1) for Q_add, index (row_base + i) * N + j.
 * ws: lpq_quant_gemm_workspace_size() bytes (pre-scan results). */
size_t lpq_quant_gemm_workspace_size(int64_t M, int64_t N, int64_t K);
lpq_status lpq_quant_gemm(const float* A, const float* B, float* C, int64_t M,
                          int64_t N, int64_t K, int64_t row_base,
                          const lpq_format* fmul, const lpq_format* fadd,
                          int mode, uint64_t seed, uint64_t call, void* ws,
                          size_t ws_bytes, uint32_t* d_status, void* stream);

/* quantized_matmul (proj/src/quant_ops.cpp:191-193 over tensor.cpp:355-376):
 * C = Q(float(sum_k double(A[i][k]) * double(B[k][j]))), double accumulator,
 * ascending k, quantization fused into the epilogue.  Q's variate index is
 * (row_base + i) * N + j with (seed, call).  Block formats quantize the
 * finished product with lpq_quantize (ws: lpq_workspace_size({M, N})). */
lpq_status lpq_matmul_q(const float* A, const float* B, float* C, int64_t M,
                        int64_t N, int64_t K, int64_t row_base,
                        const lpq_format* f, int mode, uint64_t seed,
                        uint64_t call, void* ws, size_t ws_bytes,
                        uint32_t* d_status, void* stream);

/* random_uniform (proj/src/tensor.cpp:430-440) over flat indices
 * [index_base, index_base + n): y[i] = float(lo + (hi - lo) * u). */
lpq_status lpq_uniform(float* y, int64_t n, uint64_t index_base, uint64_t seed,
                       uint64_t call, float lo, float hi, void* stream);

/* variate_tensor (proj/src/tensor.cpp:281-290): y[i] = uniform_variate(seed,
 * call, index_base + i). */
lpq_status lpq_variates(float* y, int64_t n, uint64_t index_base,
                        uint64_t seed, uint64_t call, void* stream);

/* quantize_composed_at (proj/src/quant_ops.cpp:117-150, 166-177): the
 * many-kernel baseline -- the same quantization as a chain of generic tensor
 * kernels, one HBM pass and one temporary each (the paper's "many-kernel
 * approach").  Float formats -> LPQ_ERR_UNSUPPORTED.
 * ws: lpq_composed_workspace_size() bytes (three full-size temporaries). */
size_t lpq_composed_workspace_size(const lpq_format* f, const int64_t* shape,
                                   int rank);
lpq_status lpq_quantize_composed(const float* x, float* y, const int64_t* shape,
                                 int rank, uint64_t index_base,
                                 const lpq_format* f, int mode, uint64_t seed,
                                 uint64_t call, void* ws, size_t ws_bytes,
                                 uint32_t* d_status, void* stream);

/* One tensor of a grouped quantization. */
typedef struct {
  const float* x;        /* device input  */
  float* y;              /* device output (may equal x) */
  const int64_t* shape;  /* host array of rank extents */
  int32_t rank;
  int32_t reserved;
  uint64_t index_base;   /* flat index of x[0] (RNG counter offset) */
  uint64_t call;         /* this tensor's call id */
} lpq_tensor_desc;

/* quantize_fused_at over many tensors with one format/mode/seed and a call
 * id per tensor (the reference's sequence of quantize_fused calls, each
 * advancing the counter): up to 64 tensors per kernel launch for float and
 * fixed formats and for block formats along dim 0 with rows <= 8192 floats;
 * other block layouts run per tensor (ws: the largest lpq_workspace_size). */
lpq_status lpq_quantize_grouped(const lpq_tensor_desc* tensors, int count,
                                const lpq_format* f, int mode, uint64_t seed,
                                void* ws, size_t ws_bytes, uint32_t* d_status,
                                void* stream);

/* One quantizer of a fused multi-quantizer kernel: a (non-block) format, a
 * rounding mode and the RngStream (seed, call) its variates come from. */
typedef struct {
  lpq_format format;
  int32_t mode;
  int32_t enabled;  /* 0: keep full precision (an absent QuantConfig slot) */
  uint64_t seed;
  uint64_t call;
} lpq_quant_slot;

/* LowPrecisionOptimizer::step for ONE parameter tensor (proj/src/train.cpp:
 * 148-178) fused into one pass over n elements (device pointers):
 *   g = Qg(grad);  vel = Qv(fl32(fl32(momentum*vel) + g));
 *   acc = Qa(fl32(acc - fl32(lr*vel)));  weight = Qw(acc)
 * Qv and Qa are the reference's two accumulator quantizations (the same
 * spec used twice: call ids c and c+1 when stochastic).  Variates use flat
 * index index_base + i.  Block formats -> LPQ_ERR_UNSUPPORTED. */
lpq_status lpq_sgd_step(const float* grad, float* vel, float* acc,
                        float* weight, int64_t n, float momentum, float lr,
                        const lpq_quant_slot* grad_q,
                        const lpq_quant_slot* acc_q_vel,
                        const lpq_quant_slot* acc_q_acc,
                        const lpq_quant_slot* weight_q, uint64_t index_base,
                        uint32_t* d_status, void* stream);

/* One parameter tensor of a grouped optimizer step: device pointers, its
 * element count and flat-index base, and the call id of each of its four
 * quantizations (gradient, accumulator on the velocity, accumulator on the
 * accumulator, weight) -- the values the reference's per-parameter loop
 * would use (train.cpp:148-178 advances each stochastic spec per tensor). */
typedef struct {
  const float* grad;
  float* vel;
  float* acc;
  float* weight;
  int64_t n;
  uint64_t index_base;
  uint64_t call_grad, call_vel, call_acc, call_weight;
} lpq_sgd_tensor;

/* LowPrecisionOptimizer::step over `count` parameter tensors in as few
 * launches as possible (up to 64 tensors per launch; the tensor table
 * travels in the kernel parameters, so the call is graph-capturable).  Same
 * per-element semantics as lpq_sgd_step; the slots' `call` fields are
 * ignored in favour of each tensor's call ids. */
lpq_status lpq_sgd_step_grouped(const lpq_sgd_tensor* tensors, int count,
                                float momentum, float lr,
                                const lpq_quant_slot* grad_q,
                                const lpq_quant_slot* acc_q_vel,
                                const lpq_quant_slot* acc_q_acc,
                                const lpq_quant_slot* weight_q,
                                uint32_t* d_status, void* stream);

/* ---- host entry points (synchronous; host buffers) ---------------------- */

/* quantize_fused_at over host memory on CUDA device `device` (-1 = current):
 * H2D, kernels and D2H are pipelined in chunks.  For saturating fixed point
 * with wl <= 8 and float formats with 1 + exp + man <= 8 (NearestEven /
 * Stochastic) the device->host copy carries one-byte codes of the quantized
 * values, decoded on the host through a 256-entry table (bit-identical). */
lpq_status lpq_quantize_host(const float* x, float* y, const int64_t* shape,
                             int rank, uint64_t index_base,
                             const lpq_format* f, int mode, uint64_t seed,
                             uint64_t call, int device);

/* Bytes per element lpq_quantize_host moves host->device and device->host
 * for this format and mode (4 and 4, or 4 and 1 with byte codes). */
void lpq_host_bytes_per_element(const lpq_format* f, int mode, int* h2d, int* d2h);

lpq_status lpq_quantize_composed_host(const float* x, float* y,
                                      const int64_t* shape, int rank,
                                      uint64_t index_base, const lpq_format* f,
                                      int mode, uint64_t seed, uint64_t call,
                                      int device);

lpq_status lpq_quant_gemm_host(const float* A, const float* B, float* C,
                               int64_t M, int64_t N, int64_t K,
                               int64_t row_base, const lpq_format* fmul,
                               const lpq_format* fadd, int mode, uint64_t seed,
                               uint64_t call, int device);

lpq_status lpq_matmul_q_host(const float* A, const float* B, float* C,
                             int64_t M, int64_t N, int64_t K,
                             const lpq_format* f, int mode, uint64_t seed,
                             uint64_t call, int device);

/* ---- data formats on either side of the path (proj/src/io.cpp) --------- */

/* parse_format (io.cpp:132-181): "float[:E:M]", "fixed[:WL:FL[:symmetric]
 * [:wrap]]", "block[:WL[:tensor|:dimD]]" (defaults float:5:2, fixed:8:4,
 * block:8:tensor), validated; LPQ_ERR_FORMAT on any grammar/range error. */
lpq_status lpq_parse_format(const char* text, lpq_format* out);
/* parse_rounding (io.cpp:200-206): stochastic | nearest_even | nearest_away |
 * nearest_zero. */
lpq_status lpq_parse_rounding(const char* text, int* mode);
/* format_to_string (io.cpp:183-198); returns the string length. */
int lpq_format_to_string(const lpq_format* f, char* buf, size_t len);
/* LPT1 tensor files (io.cpp:54-99): header query, payload load, save. */
lpq_status lpq_tensor_file_info(const char* path, int64_t* shape /*[8]*/,
                                int* rank);
lpq_status lpq_load_tensor_file(const char* path, float* dst, int64_t n);
lpq_status lpq_save_tensor_file(const char* path, const float* data,
                                const int64_t* shape, int rank);
/* `lpsim quantize IN OUT` (proj/tools/lpsim_main.cpp:23-34) on the GPU: LPT1
 * in -> page-locked memory -> pipelined quantize -> LPT1 out. */
lpq_status lpq_quantize_file(const char* in_path, const char* out_path,
                             const lpq_format* f, int mode, uint64_t seed,
                             uint64_t call, int device);

/* Release the per-device contexts the host entry points created. */
void lpq_shutdown(void);

#ifdef __cplusplus
}
#endif

#endif /* LPQ_H */
