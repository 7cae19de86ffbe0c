// io.cu -- the data formats on either side of the hot path (SURVEY.md §8(f)
// row 3): LPT1 tensor files and the format / rounding spec strings of the
// reference (proj/src/io.cpp:54-206), plus lpq_quantize_file, the GPU
// counterpart of `lpsim quantize` (proj/tools/lpsim_main.cpp:23-34):
// read an LPT1 file straight into page-locked memory, quantize it through
// the pipelined host path, write the result.
//
// LPT1 layout (io.cpp:54-99): "LPT1", u32 rank (<= 8), rank x u64 extents
// (each <= 2^40), then numel x u32 IEEE-754 float bits, all little-endian.
// Host-only code (no device work except inside lpq_quantize_file).
#include <cuda_runtime.h>

#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lpq.h"
#include "runtime.h"

namespace lpq {

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  out.push_back(cur);
  return out;
}

bool to_int(const std::string& s, int* v) {
  if (s.empty()) return false;
  char* end = nullptr;
  errno = 0;
  const long x = std::strtol(s.c_str(), &end, 10);
  if (errno || *end != '\0' || x < -2147483647L || x > 2147483647L) return false;
  *v = (int)x;
  return true;
}

struct Header {
  int rank = 0;
  int64_t shape[8] = {};
  int64_t numel = 1;
  long payload = 0;  // byte offset of the data
};

bool get_le(FILE* f, void* dst, int bytes) {
  unsigned char b[8];
  if (fread(b, 1, (size_t)bytes, f) != (size_t)bytes) return false;
  uint64_t v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[i];
  if (bytes == 4) *static_cast<uint32_t*>(dst) = (uint32_t)v;
  else *static_cast<uint64_t*>(dst) = v;
  return true;
}

lpq_status read_header(FILE* f, Header* h) {
  char magic[4];
  if (fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "LPT1", 4) != 0)
    return LPQ_ERR_FORMAT;  // "tensor file: bad magic"
  uint32_t rank = 0;
  if (!get_le(f, &rank, 4)) return LPQ_ERR_FORMAT;  // truncated
  if (rank > 8) return LPQ_ERR_FORMAT;              // rank exceeds 8
  h->rank = (int)rank;
  h->numel = 1;
  for (uint32_t d = 0; d < rank; ++d) {
    uint64_t e = 0;
    if (!get_le(f, &e, 8)) return LPQ_ERR_FORMAT;
    if (e > (uint64_t(1) << 40)) return LPQ_ERR_FORMAT;  // extent too large
    h->shape[d] = (int64_t)e;
    h->numel *= (int64_t)e;
  }
  h->payload = ftell(f);
  return LPQ_OK;
}

// little-endian host: the payload is the float array itself
bool read_payload(FILE* f, float* dst, int64_t n) {
  const size_t kStep = size_t(64) << 20;
  char* p = reinterpret_cast<char*>(dst);
  size_t left = sizeof(float) * (size_t)n;
  while (left) {
    const size_t k = left < kStep ? left : kStep;
    if (fread(p, 1, k, f) != k) return false;
    p += k;
    left -= k;
  }
  return true;
}

lpq_status write_file(const char* path, const int64_t* shape, int rank,
                      const float* data, int64_t n) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return LPQ_ERR_FORMAT;  // "cannot open ... for writing"
  unsigned char hdr[4 + 4 + 8 * 8];
  std::memcpy(hdr, "LPT1", 4);
  for (int i = 0; i < 4; ++i) hdr[4 + i] = (unsigned char)(((uint32_t)rank >> (8 * i)) & 0xFF);
  for (int d = 0; d < rank; ++d)
    for (int i = 0; i < 8; ++i)
      hdr[8 + 8 * d + i] = (unsigned char)(((uint64_t)shape[d] >> (8 * i)) & 0xFF);
  bool ok = fwrite(hdr, 1, (size_t)(8 + 8 * rank), f) == (size_t)(8 + 8 * rank);
  const size_t bytes = sizeof(float) * (size_t)n;
  ok = ok && fwrite(data, 1, bytes, f) == bytes;
  ok = (std::fclose(f) == 0) && ok;
  return ok ? LPQ_OK : LPQ_ERR_FORMAT;  // "failed writing ..."
}

}  // namespace

}  // namespace lpq

using namespace lpq;

extern "C" {

// parse_format (io.cpp:132-181): float[:E:M] | fixed[:WL:FL[:symmetric][:wrap]]
// | block[:WL[:tensor|:dimD]], defaults float:5:2, fixed:8:4, block:8:tensor
lpq_status lpq_parse_format(const char* text, lpq_format* out) {
  if (!text || !out) return LPQ_ERR_ARGUMENT;
  const auto parts = split(text, ':');
  lpq_format f{};
  f.block_dim = -1;
  const std::string& kind = parts[0];
  if (kind == "float") {
    f.kind = LPQ_FLOAT;
    f.exp_bits = 5;
    f.man_bits = 2;
    if (parts.size() == 3) {
      if (!to_int(parts[1], &f.exp_bits) || !to_int(parts[2], &f.man_bits)) return LPQ_ERR_FORMAT;
    } else if (parts.size() != 1) {
      return LPQ_ERR_FORMAT;
    }
  } else if (kind == "fixed") {
    f.kind = LPQ_FIXED;
    f.wl = 8;
    f.fl = 4;
    f.saturate = 1;
    if (parts.size() >= 3) {
      if (!to_int(parts[1], &f.wl) || !to_int(parts[2], &f.fl)) return LPQ_ERR_FORMAT;
      for (size_t i = 3; i < parts.size(); ++i) {
        if (parts[i] == "symmetric") f.symmetric = 1;
        else if (parts[i] == "wrap") f.saturate = 0;
        else return LPQ_ERR_FORMAT;
      }
    } else if (parts.size() != 1) {
      return LPQ_ERR_FORMAT;
    }
  } else if (kind == "block") {
    f.kind = LPQ_BLOCK;
    f.wl = 8;
    if (parts.size() >= 2 && !to_int(parts[1], &f.wl)) return LPQ_ERR_FORMAT;
    if (parts.size() == 3) {
      const std::string& a = parts[2];
      if (a == "tensor") f.block_dim = -1;
      else if (a.rfind("dim", 0) == 0) {
        if (!to_int(a.substr(3), &f.block_dim)) return LPQ_ERR_FORMAT;
        if (f.block_dim < 0) f.block_dim = -2;  // validate rejects it
      } else {
        return LPQ_ERR_FORMAT;
      }
    } else if (parts.size() > 3) {
      return LPQ_ERR_FORMAT;
    }
  } else {
    return LPQ_ERR_FORMAT;
  }
  const lpq_status st = check_format(&f);  // validate (formats.hpp:82-112)
  if (st != LPQ_OK) return st;
  *out = f;
  return LPQ_OK;
}

// parse_rounding (io.cpp:200-206)
lpq_status lpq_parse_rounding(const char* text, int* mode) {
  if (!text || !mode) return LPQ_ERR_ARGUMENT;
  const std::string t(text);
  if (t == "stochastic") *mode = LPQ_STOCHASTIC;
  else if (t == "nearest_even") *mode = LPQ_NEAREST_EVEN;
  else if (t == "nearest_away") *mode = LPQ_NEAREST_AWAY;
  else if (t == "nearest_zero") *mode = LPQ_NEAREST_ZERO;
  else return LPQ_ERR_FORMAT;
  return LPQ_OK;
}

// format_to_string (io.cpp:183-198); returns the length written (excl. NUL)
int lpq_format_to_string(const lpq_format* f, char* buf, size_t len) {
  if (!f || !buf || len == 0) return -1;
  int n;
  if (f->kind == LPQ_FLOAT) {
    n = std::snprintf(buf, len, "float:%d:%d", f->exp_bits, f->man_bits);
  } else if (f->kind == LPQ_FIXED) {
    n = std::snprintf(buf, len, "fixed:%d:%d%s%s", f->wl, f->fl,
                      f->symmetric ? ":symmetric" : "", f->saturate ? "" : ":wrap");
  } else if (f->block_dim >= 0) {
    n = std::snprintf(buf, len, "block:%d:dim%d", f->wl, f->block_dim);
  } else {
    n = std::snprintf(buf, len, "block:%d:tensor", f->wl);
  }
  return n;
}

// read_tensor_file header (io.cpp:69-88): rank, shape[8]
lpq_status lpq_tensor_file_info(const char* path, int64_t* shape, int* rank) {
  if (!path || !shape || !rank) return LPQ_ERR_ARGUMENT;
  FILE* f = std::fopen(path, "rb");
  if (!f) return LPQ_ERR_FORMAT;
  Header h;
  const lpq_status st = read_header(f, &h);
  std::fclose(f);
  if (st != LPQ_OK) return st;
  *rank = h.rank;
  for (int d = 0; d < h.rank; ++d) shape[d] = h.shape[d];
  return LPQ_OK;
}

// read_tensor_file payload into caller memory of n floats
lpq_status lpq_load_tensor_file(const char* path, float* dst, int64_t n) {
  if (!path || (n > 0 && !dst)) return LPQ_ERR_ARGUMENT;
  FILE* f = std::fopen(path, "rb");
  if (!f) return LPQ_ERR_FORMAT;
  Header h;
  lpq_status st = read_header(f, &h);
  if (st == LPQ_OK && h.numel != n) st = LPQ_ERR_SHAPE;
  if (st == LPQ_OK && !read_payload(f, dst, n)) st = LPQ_ERR_FORMAT;  // truncated
  std::fclose(f);
  return st;
}

// write_tensor_file (io.cpp:89-94)
lpq_status lpq_save_tensor_file(const char* path, const float* data,
                                const int64_t* shape, int rank) {
  if (!path || rank < 0 || rank > 8 || (rank > 0 && !shape)) return LPQ_ERR_ARGUMENT;
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) n *= shape[d];
  if (n > 0 && !data) return LPQ_ERR_ARGUMENT;
  return write_file(path, shape, rank, data, n);
}

// `lpsim quantize IN OUT --format F --rounding R --seed S` on the GPU
// (lpsim_main.cpp:23-34): LPT1 in -> page-locked buffer -> pipelined
// quantize -> LPT1 out.
lpq_status lpq_quantize_file(const char* in_path, const char* out_path,
                             const lpq_format* fmt, int mode, uint64_t seed,
                             uint64_t call, int device) {
  if (!in_path || !out_path) return LPQ_ERR_ARGUMENT;
  lpq_status st = check_format(fmt);
  if (st != LPQ_OK) return st;
  FILE* f = std::fopen(in_path, "rb");
  if (!f) return LPQ_ERR_FORMAT;
  Header h;
  st = read_header(f, &h);
  if (st != LPQ_OK) {
    std::fclose(f);
    return st;
  }
  float* buf = nullptr;
  const size_t bytes = sizeof(float) * (size_t)(h.numel > 0 ? h.numel : 1);
  cudaError_t e = cudaMallocHost(&buf, bytes);
  if (e != cudaSuccess) {
    std::fclose(f);
    return cuda_fail(e);
  }
  const bool ok = read_payload(f, buf, h.numel);
  std::fclose(f);
  if (!ok) {
    cudaFreeHost(buf);
    return LPQ_ERR_FORMAT;
  }
  // in place: the host path streams chunks H2D -> kernel -> D2H
  st = lpq_quantize_host(buf, buf, h.shape, h.rank, 0, fmt, mode, seed, call, device);
  if (st == LPQ_OK) st = write_file(out_path, h.shape, h.rank, buf, h.numel);
  cudaFreeHost(buf);
  return st;
}

}  // extern "C"
