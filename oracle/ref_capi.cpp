// ref_capi.cpp -- extern "C" wrapper over the UNMODIFIED reference library
// (lpsim, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/liblpsim_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (fixture generation, oracle
// cross-checks) and by bench.py's cpu_baseline / --impl reference legs, which
// time the reference's own quantize_fused_at on the host cores.  It is never
// linked into the product.
//
// The signatures take plain pointers so ctypes can drive them; every call
// builds the reference's own Tensor and QuantSpec types and calls the
// reference API (proj/include/lpsim/quant_ops.hpp:23-46) unchanged.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "lpsim/errors.hpp"
#include "lpsim/formats.hpp"
#include "lpsim/io.hpp"
#include "lpsim/quant_ops.hpp"
#include "lpsim/rng.hpp"
#include "lpsim/scalar_quant.hpp"
#include "lpsim/tensor.hpp"

namespace {

struct RefFormat {  // same layout as lpqo_format / lpq_format
  int32_t kind, exp_bits, man_bits, wl, fl, symmetric, saturate, block_dim;
};

lpsim::NumberFormat to_format(const RefFormat* f) {
  if (f->kind == 0) return lpsim::FloatFormat{f->exp_bits, f->man_bits};
  if (f->kind == 1)
    return lpsim::FixedFormat{f->wl, f->fl, f->symmetric != 0, f->saturate != 0};
  lpsim::BlockFloatFormat b{f->wl, {}};
  if (f->block_dim >= 0) b.block_dim = f->block_dim;
  else if (f->block_dim < -1) b.block_dim = f->block_dim;  // let validate reject
  return b;
}

lpsim::Shape to_shape(const int64_t* shape, int rank) {
  return lpsim::Shape(shape, shape + rank);
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const lpsim::format_error&) {
    return 1;
  } catch (const lpsim::shape_error&) {
    return 2;
  } catch (const lpsim::invalid_input_error&) {
    return 3;
  } catch (const lpsim::unsupported_format_error&) {
    return 4;
  } catch (...) {
    return 9;
  }
}

}  // namespace

extern "C" {

void lpsr_set_num_threads(int n) { lpsim::set_num_threads(n); }
uint64_t lpsr_pass_count() { return lpsim::pass_count(); }
void lpsr_reset_pass_count() { lpsim::reset_pass_count(); }

float lpsr_uniform_variate(uint64_t seed, uint64_t call, uint64_t index) {
  return lpsim::uniform_variate(lpsim::RngStream{seed}, call, index);
}
uint64_t lpsr_stream_key(uint64_t seed, uint64_t call) {
  return lpsim::detail::stream_key(seed, call);
}

// round_integer (rounding.hpp:210-224); returns status, value in *out
int lpsr_round_integer(double r, int mode, double u, double* out) {
  return guarded([&] {
    *out = lpsim::round_integer(r, static_cast<lpsim::RoundingMode>(mode), u);
  });
}

int lpsr_quant_scalar(float x, const RefFormat* f, int mode, float u,
                      float* out) {
  return guarded([&] {
    const auto fmt = to_format(f);
    lpsim::validate(fmt);
    const auto m = static_cast<lpsim::RoundingMode>(mode);
    if (const auto* ff = std::get_if<lpsim::FixedFormat>(&fmt))
      *out = lpsim::quantize_scalar_fixed(x, *ff, m, u);
    else
      *out = lpsim::quantize_scalar_float(x, std::get<lpsim::FloatFormat>(fmt),
                                          m, u);
  });
}

// Vectorised scalar quantization with explicit variates (test oracle sweep).
int lpsr_quant_scalar_many(const float* x, const float* u, float* y, int64_t n,
                           const RefFormat* f, int mode) {
  return guarded([&] {
    const auto fmt = to_format(f);
    lpsim::validate(fmt);
    const auto m = static_cast<lpsim::RoundingMode>(mode);
    if (const auto* ff = std::get_if<lpsim::FixedFormat>(&fmt)) {
      for (int64_t i = 0; i < n; ++i)
        y[i] = lpsim::quantize_scalar_fixed(x[i], *ff, m, u ? u[i] : 0.0f);
    } else {
      const auto& fl = std::get<lpsim::FloatFormat>(fmt);
      for (int64_t i = 0; i < n; ++i)
        y[i] = lpsim::quantize_scalar_float(x[i], fl, m, u ? u[i] : 0.0f);
    }
  });
}

// quantize_fused_at (quant_ops.cpp:154-164) on a copy of x.  *seconds gets
// the wall time of the quantize_fused_at call alone (tensor construction and
// the copy-out are outside it).
int lpsr_quantize_fused_at(const float* x, float* y, const int64_t* shape,
                           int rank, const RefFormat* f, int mode,
                           uint64_t seed, uint64_t call, double* seconds) {
  return guarded([&] {
    const bool saved = lpsim::validation_enabled();
    lpsim::set_validation(false);  // allow non-finite inputs to reach the op
    lpsim::Tensor t(to_shape(shape, rank),
                    std::vector<float>(x, x + [&] {
                      int64_t n = 1;
                      for (int d = 0; d < rank; ++d) n *= shape[d];
                      return n;
                    }()));
    lpsim::set_validation(saved);
    lpsim::QuantSpec spec{to_format(f), static_cast<lpsim::RoundingMode>(mode),
                          seed, 0};
    const auto t0 = std::chrono::steady_clock::now();
    lpsim::Tensor q = lpsim::quantize_fused_at(t, spec, call);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(y, q.data(), sizeof(float) * static_cast<size_t>(q.numel()));
  });
}

int lpsr_quantize_composed_at(const float* x, float* y, const int64_t* shape,
                              int rank, const RefFormat* f, int mode,
                              uint64_t seed, uint64_t call) {
  return guarded([&] {
    int64_t n = 1;
    for (int d = 0; d < rank; ++d) n *= shape[d];
    lpsim::Tensor t(to_shape(shape, rank), std::vector<float>(x, x + n));
    lpsim::QuantSpec spec{to_format(f), static_cast<lpsim::RoundingMode>(mode),
                          seed, 0};
    lpsim::Tensor q = lpsim::quantize_composed_at(t, spec, call);
    std::memcpy(y, q.data(), sizeof(float) * static_cast<size_t>(n));
  });
}

int lpsr_reduce_max_abs(const float* x, const int64_t* shape, int rank,
                        int block_dim, float* out) {
  return guarded([&] {
    int64_t n = 1;
    for (int d = 0; d < rank; ++d) n *= shape[d];
    lpsim::set_validation(false);
    lpsim::Tensor t(to_shape(shape, rank), std::vector<float>(x, x + n));
    lpsim::set_validation(true);
    std::optional<int> dim;
    if (block_dim >= 0) dim = block_dim;
    lpsim::Tensor m = lpsim::reduce_max_abs(t, dim);
    std::memcpy(out, m.data(), sizeof(float) * static_cast<size_t>(m.numel()));
  });
}

int lpsr_random_uniform(float* y, const int64_t* shape, int rank,
                        uint64_t seed, uint64_t call, float lo, float hi) {
  return guarded([&] {
    lpsim::Tensor t = lpsim::random_uniform(to_shape(shape, rank),
                                            lpsim::RngStream{seed}, call, lo, hi);
    std::memcpy(y, t.data(), sizeof(float) * static_cast<size_t>(t.numel()));
  });
}

int lpsr_matmul(const float* a, const float* b, float* c, int64_t m, int64_t k,
                int64_t n) {
  return guarded([&] {
    lpsim::Tensor ta({m, k}, std::vector<float>(a, a + m * k));
    lpsim::Tensor tb({k, n}, std::vector<float>(b, b + k * n));
    lpsim::Tensor tc = lpsim::matmul(ta, tb);
    std::memcpy(c, tc.data(), sizeof(float) * static_cast<size_t>(m * n));
  });
}

// quantized_matmul (quant_ops.cpp:191-193): returns the advanced counter.
int lpsr_quantized_matmul(const float* a, const float* b, float* c, int64_t m,
                          int64_t k, int64_t n, const RefFormat* f, int mode,
                          uint64_t seed, uint64_t* call_counter) {
  return guarded([&] {
    lpsim::Tensor ta({m, k}, std::vector<float>(a, a + m * k));
    lpsim::Tensor tb({k, n}, std::vector<float>(b, b + k * n));
    lpsim::QuantSpec spec{to_format(f), static_cast<lpsim::RoundingMode>(mode),
                          seed, *call_counter};
    lpsim::Tensor tc = lpsim::quantized_matmul(ta, tb, spec);
    *call_counter = spec.call_counter;
    std::memcpy(c, tc.data(), sizeof(float) * static_cast<size_t>(m * n));
  });
}

// The per-op-rounded GEMM as the reference's OWN tensor-op composition
// (SURVEY.md §8(c) "Per-op GEMM oracle"): for k = 0..K-1, over M x N tensors,
//   P   = mul(a[:, k] (x) 1, 1 (x) b[k, :])          tensor.cpp:152-156
//   P   = quantize_fused_at(P, {fmt_mul}, call + 2k)  quant_ops.cpp:154-164
//   acc = add(acc, P)                                  tensor.cpp:140-144
//   acc = quantize_fused_at(acc, {fmt_add}, call + 2k + 1)
// with acc starting as the zero-filled Tensor({M, N}) (+0).  Variate index
// of output (i, j) = its flat index i*N + j (quant_pass, quant_ops.cpp:13-31).
// Every step is a reference API call; nothing here does arithmetic.
int lpsr_quant_gemm_composed(const float* a, const float* b, float* c, int64_t m,
                             int64_t n, int64_t k, const RefFormat* fmul,
                             const RefFormat* fadd, int mode, uint64_t seed,
                             uint64_t call) {
  return guarded([&] {
    const lpsim::QuantSpec smul{to_format(fmul), static_cast<lpsim::RoundingMode>(mode),
                                seed, 0};
    const lpsim::QuantSpec sadd{to_format(fadd), static_cast<lpsim::RoundingMode>(mode),
                                seed, 0};
    lpsim::Tensor acc({m, n});
    std::vector<float> pa(static_cast<size_t>(m * n)), pb(static_cast<size_t>(m * n));
    for (int64_t kk = 0; kk < k; ++kk) {
      for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
          pa[static_cast<size_t>(i * n + j)] = a[i * k + kk];
          pb[static_cast<size_t>(i * n + j)] = b[kk * n + j];
        }
      lpsim::Tensor p = lpsim::mul(lpsim::Tensor({m, n}, pa), lpsim::Tensor({m, n}, pb));
      p = lpsim::quantize_fused_at(p, smul, call + 2 * static_cast<uint64_t>(kk));
      acc = lpsim::add(acc, p);
      acc = lpsim::quantize_fused_at(acc, sadd, call + 2 * static_cast<uint64_t>(kk) + 1);
    }
    std::memcpy(c, acc.data(), sizeof(float) * static_cast<size_t>(m * n));
  });
}

// parse_format (io.cpp:132-181) -> flat format struct
int lpsr_parse_format(const char* text, RefFormat* out) {
  return guarded([&] {
    const auto fmt = lpsim::parse_format(text);
    RefFormat r{};
    r.block_dim = -1;
    if (const auto* f = std::get_if<lpsim::FloatFormat>(&fmt)) {
      r.kind = 0; r.exp_bits = f->exp_bits; r.man_bits = f->man_bits;
    } else if (const auto* f = std::get_if<lpsim::FixedFormat>(&fmt)) {
      r.kind = 1; r.wl = f->wl; r.fl = f->fl; r.symmetric = f->symmetric; r.saturate = f->saturate;
    } else {
      const auto& b = std::get<lpsim::BlockFloatFormat>(fmt);
      r.kind = 2; r.wl = b.wl; r.block_dim = b.block_dim ? *b.block_dim : -1;
    }
    *out = r;
  });
}

// parse_quant_config (io.cpp:294-321) -> five (present, format, mode, seed)
// slots in the category order weight, accumulator, gradient, activation,
// error.  nlohmann type errors (json::exception other than the parse error the
// reference converts) return 7.
int lpsr_parse_quant_config(const char* text, uint64_t default_seed,
                            int32_t* present, RefFormat* fmts, int32_t* modes,
                            uint64_t* seeds) {
  try {
    const lpsim::QuantConfig cfg = lpsim::parse_quant_config(text, default_seed);
    const std::optional<lpsim::QuantSpec>* slots[5] = {
        &cfg.weight, &cfg.accumulator, &cfg.gradient, &cfg.activation, &cfg.error};
    for (int i = 0; i < 5; ++i) {
      present[i] = slots[i]->has_value();
      if (!present[i]) continue;
      const auto& sp = **slots[i];
      RefFormat r{};
      r.block_dim = -1;
      if (const auto* f = std::get_if<lpsim::FloatFormat>(&sp.format)) {
        r.kind = 0; r.exp_bits = f->exp_bits; r.man_bits = f->man_bits;
      } else if (const auto* f = std::get_if<lpsim::FixedFormat>(&sp.format)) {
        r.kind = 1; r.wl = f->wl; r.fl = f->fl; r.symmetric = f->symmetric; r.saturate = f->saturate;
      } else {
        const auto& b = std::get<lpsim::BlockFloatFormat>(sp.format);
        r.kind = 2; r.wl = b.wl; r.block_dim = b.block_dim ? *b.block_dim : -1;
      }
      fmts[i] = r;
      modes[i] = static_cast<int32_t>(sp.mode);
      seeds[i] = sp.seed;
    }
    return 0;
  } catch (const lpsim::format_error&) {
    return 1;
  } catch (const std::exception&) {
    return 7;
  }
}

int lpsr_write_tensor_file(const char* path, const float* x, const int64_t* shape, int rank) {
  return guarded([&] {
    int64_t n = 1;
    for (int d = 0; d < rank; ++d) n *= shape[d];
    lpsim::set_validation(false);
    lpsim::Tensor t(to_shape(shape, rank), std::vector<float>(x, x + n));
    lpsim::set_validation(true);
    lpsim::write_tensor_file(path, t);
  });
}

int lpsr_read_tensor_file(const char* path, float* y, int64_t n, int64_t* shape, int* rank) {
  return guarded([&] {
    lpsim::Tensor t = lpsim::read_tensor_file(path);
    *rank = t.rank();
    for (int d = 0; d < t.rank(); ++d) shape[d] = t.extent(d);
    if (t.numel() <= n) std::memcpy(y, t.data(), sizeof(float) * static_cast<size_t>(t.numel()));
  });
}

}  // extern "C"
