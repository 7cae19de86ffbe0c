"""ctypes handles on the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -- oracle/liblpq_oracle.so, the C restatement (oracle/lpq_oracle.c)
* ``RefLib``  -- oracle/_ref/liblpsim_ref.so, the unmodified reference library
  (compiled from /root/reference sources by oracle/Makefile) behind
  oracle/ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liblpq_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "liblpsim_ref.so")

STOCHASTIC, NEAREST_EVEN, NEAREST_AWAY, NEAREST_ZERO = 0, 1, 2, 3
ALL_MODES = (NEAREST_EVEN, NEAREST_AWAY, NEAREST_ZERO, STOCHASTIC)
FLOAT, FIXED, BLOCK = 0, 1, 2
OK, FORMAT_ERROR, SHAPE_ERROR, INVALID_INPUT, UNSUPPORTED = 0, 1, 2, 3, 4


class Fmt(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "exp_bits", "man_bits", "wl", "fl", "symmetric", "saturate",
        "block_dim")]

    def __repr__(self):
        if self.kind == FLOAT:
            return f"float:{self.exp_bits}:{self.man_bits}"
        if self.kind == FIXED:
            return (f"fixed:{self.wl}:{self.fl}"
                    + (":symmetric" if self.symmetric else "")
                    + ("" if self.saturate else ":wrap"))
        return f"block:{self.wl}:" + ("tensor" if self.block_dim < 0
                                      else f"dim{self.block_dim}")


def float_fmt(e, m):
    return Fmt(FLOAT, e, m, 0, 0, 0, 0, -1)


def fixed_fmt(wl, fl, symmetric=False, saturate=True):
    return Fmt(FIXED, 0, 0, wl, fl, int(symmetric), int(saturate), -1)


def block_fmt(wl, dim=None):
    return Fmt(BLOCK, 0, 0, wl, 0, 0, 0, -1 if dim is None else dim)


_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_FP = C.POINTER(C.c_float)


def _ensure_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")],
                       check=True)


class Oracle:
    """The C restatement."""

    def __init__(self):
        _ensure_built()
        L = C.CDLL(ORACLE_SO)
        L.lpqo_mix64.restype = C.c_uint64
        L.lpqo_mix64.argtypes = [C.c_uint64]
        L.lpqo_stream_key.restype = C.c_uint64
        L.lpqo_stream_key.argtypes = [C.c_uint64, C.c_uint64]
        L.lpqo_uniform_variate.restype = C.c_float
        L.lpqo_uniform_variate.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.lpqo_round_integer.restype = C.c_double
        L.lpqo_round_integer.argtypes = [C.c_double, C.c_int, C.c_double]
        L.lpqo_validate.argtypes = [C.POINTER(Fmt)]
        for fn in (L.lpqo_quant_fixed, L.lpqo_quant_float):
            fn.restype = C.c_float
            fn.argtypes = [C.c_float, C.POINTER(Fmt), C.c_int, C.c_float]
        L.lpqo_quantize.argtypes = [_fp, _fp, _i64p, C.c_int, C.c_uint64,
                                    C.POINTER(Fmt), C.c_int, C.c_uint64,
                                    C.c_uint64]
        L.lpqo_reduce_max_abs.argtypes = [_fp, _i64p, C.c_int, C.c_int, _fp]
        L.lpqo_quantize_block_given_max.argtypes = [_fp, _fp, _i64p, C.c_int, C.c_uint64,
                                                    C.POINTER(Fmt), C.c_int, C.c_uint64,
                                                    C.c_uint64, _fp]
        L.lpqo_random_uniform.argtypes = [_fp, C.c_int64, C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_float,
                                          C.c_float]
        L.lpqo_matmul.argtypes = [_fp, _fp, _fp, C.c_int64, C.c_int64,
                                  C.c_int64]
        L.lpqo_quant_gemm.argtypes = [_fp, _fp, _fp, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_int64,
                                      C.c_int64, C.POINTER(Fmt),
                                      C.POINTER(Fmt), C.c_int, C.c_uint64,
                                      C.c_uint64]
        self.L = L

    def variate(self, seed, call, index):
        return self.L.lpqo_uniform_variate(seed, call, index)

    def round_integer(self, r, mode, u=0.0):
        return self.L.lpqo_round_integer(r, mode, u)

    def quant_scalar(self, x, fmt, mode, u=0.0):
        fn = self.L.lpqo_quant_fixed if fmt.kind == FIXED else self.L.lpqo_quant_float
        return fn(x, C.byref(fmt), mode, u)

    def quantize(self, x, fmt, mode, seed=0, call=0, index_base=0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        shape = np.array(x.shape, dtype=np.int64)
        st = self.L.lpqo_quantize(x.reshape(-1) if x.ndim == 0 else x, y,
                                  shape, x.ndim, index_base, C.byref(fmt),
                                  mode, seed, call)
        return st, y

    def quantize_block_given_max(self, x, fmt, mode, mx, seed=0, call=0, index_base=0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        mx = np.ascontiguousarray(mx, dtype=np.float32)
        st = self.L.lpqo_quantize_block_given_max(
            x, y, np.array(x.shape, dtype=np.int64), x.ndim, index_base, C.byref(fmt),
            mode, seed, call, mx)
        return st, y

    def reduce_max_abs(self, x, dim):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.zeros(1 if dim is None else x.shape[dim], dtype=np.float32)
        st = self.L.lpqo_reduce_max_abs(x, np.array(x.shape, dtype=np.int64),
                                        x.ndim, -1 if dim is None else dim, out)
        return st, out

    def random_uniform(self, n, seed, call, lo, hi, index_base=0):
        y = np.empty(n, dtype=np.float32)
        self.L.lpqo_random_uniform(y, n, index_base, seed, call, lo, hi)
        return y

    def matmul(self, a, b):
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.float32)
        self.L.lpqo_matmul(np.ascontiguousarray(a), np.ascontiguousarray(b),
                           c, m, k, n)
        return c

    def quant_gemm(self, a, b, fmul, fadd, mode=NEAREST_EVEN, seed=0, call=0,
                   rows=None, row_base=0):
        M, K = a.shape
        N = b.shape[1]
        r0, r1 = (0, M) if rows is None else rows
        c = np.zeros((M, N), dtype=np.float32)
        st = self.L.lpqo_quant_gemm(np.ascontiguousarray(a),
                                    np.ascontiguousarray(b), c, M, N, K,
                                    row_base, r0, r1, C.byref(fmul),
                                    C.byref(fadd), mode, seed, call)
        return st, c


class RefLib:
    """The reference library itself (oracle/_ref/liblpsim_ref.so)."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        L = C.CDLL(REF_SO)
        L.lpsr_uniform_variate.restype = C.c_float
        L.lpsr_uniform_variate.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.lpsr_stream_key.restype = C.c_uint64
        L.lpsr_stream_key.argtypes = [C.c_uint64, C.c_uint64]
        L.lpsr_round_integer.argtypes = [C.c_double, C.c_int, C.c_double,
                                         C.POINTER(C.c_double)]
        L.lpsr_quant_scalar.argtypes = [C.c_float, C.POINTER(Fmt), C.c_int,
                                        C.c_float, C.POINTER(C.c_float)]
        L.lpsr_quant_scalar_many.argtypes = [_fp, C.c_void_p, _fp, C.c_int64,
                                             C.POINTER(Fmt), C.c_int]
        L.lpsr_quantize_fused_at.argtypes = [_fp, _fp, _i64p, C.c_int,
                                             C.POINTER(Fmt), C.c_int,
                                             C.c_uint64, C.c_uint64,
                                             C.POINTER(C.c_double)]
        L.lpsr_quantize_composed_at.argtypes = [_fp, _fp, _i64p, C.c_int,
                                                C.POINTER(Fmt), C.c_int,
                                                C.c_uint64, C.c_uint64]
        L.lpsr_reduce_max_abs.argtypes = [_fp, _i64p, C.c_int, C.c_int, _fp]
        L.lpsr_random_uniform.argtypes = [_fp, _i64p, C.c_int, C.c_uint64,
                                          C.c_uint64, C.c_float, C.c_float]
        L.lpsr_matmul.argtypes = [_fp, _fp, _fp, C.c_int64, C.c_int64,
                                  C.c_int64]
        L.lpsr_quantized_matmul.argtypes = [_fp, _fp, _fp, C.c_int64,
                                            C.c_int64, C.c_int64,
                                            C.POINTER(Fmt), C.c_int,
                                            C.c_uint64,
                                            C.POINTER(C.c_uint64)]
        L.lpsr_set_num_threads.argtypes = [C.c_int]
        L.lpsr_quant_gemm_composed.argtypes = [_fp, _fp, _fp, C.c_int64, C.c_int64,
                                               C.c_int64, C.POINTER(Fmt), C.POINTER(Fmt),
                                               C.c_int, C.c_uint64, C.c_uint64]
        L.lpsr_parse_format.argtypes = [C.c_char_p, C.POINTER(Fmt)]
        L.lpsr_write_tensor_file.argtypes = [C.c_char_p, _fp, _i64p, C.c_int]
        L.lpsr_read_tensor_file.argtypes = [C.c_char_p, _fp, C.c_int64, _i64p,
                                            C.POINTER(C.c_int)]
        L.lpsr_parse_quant_config.argtypes = [
            C.c_char_p, C.c_uint64, np.ctypeslib.ndpointer(np.int32, flags="C"),
            C.POINTER(Fmt), np.ctypeslib.ndpointer(np.int32, flags="C"),
            np.ctypeslib.ndpointer(np.uint64, flags="C")]
        L.lpsr_pass_count.restype = C.c_uint64
        self.L = L

    def set_num_threads(self, n):
        self.L.lpsr_set_num_threads(n)

    def parse_format(self, text):
        f = Fmt()
        st = self.L.lpsr_parse_format(text.encode(), C.byref(f))
        return st, f

    def parse_quant_config(self, text, default_seed):
        """-> (status, [None | (Fmt, mode, seed)] x 5)"""
        present = np.zeros(5, np.int32)
        fmts = (Fmt * 5)()
        modes = np.zeros(5, np.int32)
        seeds = np.zeros(5, np.uint64)
        st = self.L.lpsr_parse_quant_config(text.encode(), C.c_uint64(default_seed),
                                            present, fmts, modes, seeds)
        out = [(fmts[i], int(modes[i]), int(seeds[i])) if present[i] else None
               for i in range(5)]
        return st, out

    def write_tensor_file(self, path, x):
        x = np.asarray(x, dtype=np.float32, order="C")  # keeps rank 0
        return self.L.lpsr_write_tensor_file(path.encode(), x.reshape(-1),
                                             np.array(x.shape, np.int64), x.ndim)

    def read_tensor_file(self, path, n):
        y = np.empty(max(n, 1), np.float32)
        shape = np.zeros(8, np.int64)
        rank = C.c_int()
        st = self.L.lpsr_read_tensor_file(path.encode(), y, n, shape, C.byref(rank))
        return st, y[:n], tuple(int(v) for v in shape[:rank.value])

    def variate(self, seed, call, index):
        return self.L.lpsr_uniform_variate(seed, call, index)

    def round_integer(self, r, mode, u=0.0):
        out = C.c_double()
        st = self.L.lpsr_round_integer(r, mode, u, C.byref(out))
        return st, out.value

    def quant_scalar_many(self, x, fmt, mode, u=None):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        up = None
        if u is not None:
            u = np.ascontiguousarray(u, dtype=np.float32)
            up = u.ctypes.data
        st = self.L.lpsr_quant_scalar_many(x, up, y, x.size, C.byref(fmt),
                                           mode)
        return st, y

    def quantize(self, x, fmt, mode, seed=0, call=0, timed=False):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        secs = C.c_double()
        st = self.L.lpsr_quantize_fused_at(x.reshape(-1) if x.ndim == 0 else x,
                                           y, np.array(x.shape, np.int64),
                                           x.ndim, C.byref(fmt), mode, seed,
                                           call, C.byref(secs))
        return (st, y, secs.value) if timed else (st, y)

    def quantize_composed(self, x, fmt, mode, seed=0, call=0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        st = self.L.lpsr_quantize_composed_at(x, y, np.array(x.shape, np.int64),
                                              x.ndim, C.byref(fmt), mode, seed,
                                              call)
        return st, y

    def reduce_max_abs(self, x, dim):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.zeros(1 if dim is None else x.shape[dim], dtype=np.float32)
        st = self.L.lpsr_reduce_max_abs(x, np.array(x.shape, np.int64), x.ndim,
                                        -1 if dim is None else dim, out)
        return st, out

    def random_uniform(self, shape, seed, call, lo, hi):
        y = np.empty(shape, dtype=np.float32)
        self.L.lpsr_random_uniform(y.reshape(-1), np.array(shape, np.int64),
                                   len(shape), seed, call, lo, hi)
        return y

    def matmul(self, a, b):
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.float32)
        st = self.L.lpsr_matmul(np.ascontiguousarray(a), np.ascontiguousarray(b),
                                c, m, k, n)
        assert st == 0
        return c

    def quant_gemm_composed(self, a, b, fmul, fadd, mode, seed=0, call=0):
        """The per-op GEMM as the reference's own mul -> quantize_fused_at ->
        add -> quantize_fused_at composition per k (ref_capi.cpp)."""
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.float32)
        st = self.L.lpsr_quant_gemm_composed(np.ascontiguousarray(a, np.float32),
                                             np.ascontiguousarray(b, np.float32), c,
                                             m, n, k, C.byref(fmul), C.byref(fadd),
                                             mode, seed, call)
        return st, c

    def quantized_matmul(self, a, b, fmt, mode, seed=0, call=0):
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.float32)
        cc = C.c_uint64(call)
        st = self.L.lpsr_quantized_matmul(np.ascontiguousarray(a),
                                          np.ascontiguousarray(b), c, m, k, n,
                                          C.byref(fmt), mode, seed,
                                          C.byref(cc))
        return st, c, cc.value


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def f32_from_bits(u):
    return np.asarray(u, dtype=np.uint32).view(np.float32)
