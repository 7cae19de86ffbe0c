// quant_ops_b200.cpp -- drop-in replacement for the reference's
// proj/src/quant_ops.cpp: the same C++ API (proj/include/lpsim/
// quant_ops.hpp:23-46, compiled against the reference's own headers), with
// every quantization running on the B200 through liblpq.so's C ABI
// (include/lpq.h).  A maintainer swaps this file for quant_ops.cpp in
// lpsim_core and links liblpq.so; nothing else changes.
//
//   quantize_fused_at     -> lpq_quantize_host          (quant_ops.cpp:154-164)
//   quantize_fused        -> + call_counter rule        (quant_ops.cpp:179-183)
//   quantize_composed_at  -> lpq_quantize_composed_host (quant_ops.cpp:166-177)
//   quantize_composed     -> + call_counter rule        (quant_ops.cpp:185-189)
//   quantized_matmul      -> lpq_matmul_q_host          (quant_ops.cpp:191-193)
//
// Status codes map back to the reference's exception types
// (proj/include/lpsim/errors.hpp), and the data-pass counter
// (detail::bump_pass) is advanced by the number of device passes each call
// made, so the pass-count contract (fused <= 2, composed >= 4 / >= 6) holds.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <variant>

#include "lpq.h"
#include "lpsim/errors.hpp"
#include "lpsim/formats.hpp"
#include "lpsim/quant_ops.hpp"
#include "lpsim/tensor.hpp"

namespace lpsim {

namespace {

lpq_format to_lpq(const NumberFormat& fmt) {
  lpq_format f{};
  f.block_dim = -1;
  if (const auto* x = std::get_if<FloatFormat>(&fmt)) {
    f.kind = LPQ_FLOAT;
    f.exp_bits = x->exp_bits;
    f.man_bits = x->man_bits;
  } else if (const auto* x = std::get_if<FixedFormat>(&fmt)) {
    f.kind = LPQ_FIXED;
    f.wl = x->wl;
    f.fl = x->fl;
    f.symmetric = x->symmetric ? 1 : 0;
    f.saturate = x->saturate ? 1 : 0;
  } else {
    const auto& b = std::get<BlockFloatFormat>(fmt);
    f.kind = LPQ_BLOCK;
    f.wl = b.wl;
    f.block_dim = b.block_dim ? *b.block_dim : -1;
  }
  return f;
}

[[noreturn]] void raise(lpq_status st, const char* what) {
  const std::string msg = std::string(what) + ": " + lpq_status_string(st);
  switch (st) {
    case LPQ_ERR_FORMAT: throw format_error(msg);
    case LPQ_ERR_SHAPE: throw shape_error(msg);
    case LPQ_ERR_INVALID_INPUT:
    case LPQ_ERR_BLOCK_RANGE: throw invalid_input_error(msg);
    case LPQ_ERR_UNSUPPORTED: throw unsupported_format_error(msg);
    case LPQ_ERR_INVALID_VALUE: throw invalid_value_error(msg);
    default:
      throw std::runtime_error(msg + " (" + lpq_last_cuda_error() + ")");
  }
}

void bump_passes(uint64_t before) {
  for (uint64_t p = before; p < lpq_pass_count(); ++p) detail::bump_pass();
}

template <typename Call>
Tensor run_quantize(const Tensor& t, const QuantSpec& spec, Call&& call,
                    const char* what) {
  validate(spec.format);  // formats.hpp:82-112 throws format_error itself
  const lpq_format f = to_lpq(spec.format);
  Tensor out(t.shape());
  const uint64_t before = lpq_pass_count();
  const lpq_status st = call(t.data(), out.data(), t.shape().data(), t.rank(), &f);
  bump_passes(before);
  if (st != LPQ_OK) raise(st, what);
  return out;
}

}  // namespace

Tensor quantize_fused_at(const Tensor& t, const QuantSpec& spec,
                         std::uint64_t call) {
  return run_quantize(
      t, spec,
      [&](const float* x, float* y, const int64_t* shape, int rank,
          const lpq_format* f) {
        return lpq_quantize_host(x, y, shape, rank, 0, f,
                                 static_cast<int>(spec.mode), spec.seed, call,
                                 -1);
      },
      "quantize_fused");
}

Tensor quantize_composed_at(const Tensor& t, const QuantSpec& spec,
                            std::uint64_t call) {
  return run_quantize(
      t, spec,
      [&](const float* x, float* y, const int64_t* shape, int rank,
          const lpq_format* f) {
        return lpq_quantize_composed_host(x, y, shape, rank, 0, f,
                                          static_cast<int>(spec.mode),
                                          spec.seed, call, -1);
      },
      "quantize_composed");
}

Tensor quantize_fused(const Tensor& t, QuantSpec& spec) {
  Tensor out = quantize_fused_at(t, spec, spec.call_counter);
  if (spec.mode == RoundingMode::Stochastic) ++spec.call_counter;
  return out;
}

Tensor quantize_composed(const Tensor& t, QuantSpec& spec) {
  Tensor out = quantize_composed_at(t, spec, spec.call_counter);
  if (spec.mode == RoundingMode::Stochastic) ++spec.call_counter;
  return out;
}

// matmul (tensor.cpp:355-376) + quantize_fused in ONE device call: DFMA
// accumulation in ascending k, the quantizer in the GEMM epilogue.
Tensor quantized_matmul(const Tensor& a, const Tensor& b, QuantSpec& spec) {
  if (a.rank() != 2 || b.rank() != 2)
    throw shape_error("matmul: operands must be rank-2");
  if (a.extent(1) != b.extent(0))
    throw shape_error("matmul: inner dimensions disagree");
  validate(spec.format);
  const int64_t m = a.extent(0), k = a.extent(1), n = b.extent(1);
  const lpq_format f = to_lpq(spec.format);
  Tensor out(Shape{m, n});
  const uint64_t before = lpq_pass_count();
  const lpq_status st = lpq_matmul_q_host(
      a.data(), b.data(), out.data(), m, n, k, &f, static_cast<int>(spec.mode),
      spec.seed, spec.call_counter, -1);
  bump_passes(before);
  if (st != LPQ_OK) raise(st, "quantized_matmul");
  if (spec.mode == RoundingMode::Stochastic) ++spec.call_counter;
  return out;
}

}  // namespace lpsim
