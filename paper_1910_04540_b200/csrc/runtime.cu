// runtime.cu -- host-memory entry points of liblpq.so.
//
// The reference API takes and returns host tensors (lpsim::Tensor, a
// std::vector<float>; proj/include/lpsim/tensor.hpp:19-46).  These entry
// points give that API a B200 path: a per-device context owns three CUDA
// streams, device chunk buffers and pinned bounce buffers; a call streams the
// tensor through them so that chunk c's host->device copy, chunk c-1's kernel
// and chunk c-2's device->host copy run concurrently (two copy engines + the
// SMs).  Pinned caller memory is copied directly; pageable memory (a plain
// std::vector, as the drop-in shim passes) is bounced through the pinned
// buffers with a multi-threaded memcpy.  Block formats whose blocks are not
// contiguous rows need the whole tensor resident for the reduction pass and
// take the resident path (copy in, two device passes, copy out).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include "../../include/lpq.h"
#include "kernels.cuh"
#include "runtime.h"

namespace lpq {

namespace {

constexpr int kStreams = 3;
constexpr int64_t kChunkElems = int64_t(1) << 24;  // 64 MiB of fp32

struct HostCtx {
  int dev = 0;
  cudaStream_t st[kStreams] = {};
  cudaEvent_t done[kStreams] = {};
  float* dbuf[kStreams] = {};
  float* pin_in[kStreams] = {};
  float* pin_out[kStreams] = {};
  uint8_t* dcode[kStreams] = {};   // device byte codes of a chunk
  uint8_t* pcode[kStreams] = {};   // page-locked byte codes of a chunk
  void* sws[kStreams] = {};        // device workspace of a chunk's call
  size_t sws_bytes = 0;
  int64_t chunk_cap = 0;  // elements per chunk buffer
  uint32_t* d_status = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  float* dfull = nullptr;
  int64_t dfull_cap = 0;
  // direct path (tensors <= 16 MB): page-locked staging of pageable
  // inputs / outputs, byte codes of the whole tensor, block maxima + flag
  float* pstage = nullptr;
  int64_t pstage_cap = 0;
  uint8_t* dcodef = nullptr;
  uint8_t* pcodef = nullptr;
  int64_t codef_cap = 0;
  uint32_t* daux = nullptr;  // device: encode flag
  uint32_t* paux = nullptr;  // page-locked: block maxima [extent] + flag
  int64_t paux_cap = 0;
  uint32_t* pstatus = nullptr;  // page-locked status word (status fetch)
  std::mutex mu;

  ~HostCtx() { release(); }

  void release() {
    DeviceGuard g(dev);
    for (int k = 0; k < kStreams; ++k) {
      if (dbuf[k]) cudaFree(dbuf[k]);
      if (pin_in[k]) cudaFreeHost(pin_in[k]);
      if (pin_out[k]) cudaFreeHost(pin_out[k]);
      if (dcode[k]) cudaFree(dcode[k]);
      if (pcode[k]) cudaFreeHost(pcode[k]);
      if (sws[k]) cudaFree(sws[k]);
      dcode[k] = nullptr;
      pcode[k] = nullptr;
      sws[k] = nullptr;
      if (done[k]) cudaEventDestroy(done[k]);
      if (st[k]) cudaStreamDestroy(st[k]);
      dbuf[k] = pin_in[k] = pin_out[k] = nullptr;
      done[k] = nullptr;
      st[k] = nullptr;
    }
    if (d_status) cudaFree(d_status);
    if (ws) cudaFree(ws);
    if (dfull) cudaFree(dfull);
    if (pstage) cudaFreeHost(pstage);
    if (dcodef) cudaFree(dcodef);
    if (pcodef) cudaFreeHost(pcodef);
    if (daux) cudaFree(daux);
    if (paux) cudaFreeHost(paux);
    if (pstatus) cudaFreeHost(pstatus);
    pstatus = nullptr;
    pstage = nullptr;
    dcodef = nullptr;
    pcodef = nullptr;
    daux = paux = nullptr;
    pstage_cap = codef_cap = paux_cap = 0;
    d_status = nullptr;
    ws = nullptr;
    dfull = nullptr;
    chunk_cap = dfull_cap = 0;
    ws_bytes = sws_bytes = 0;
  }

  cudaError_t init() {
    if (st[0]) return cudaSuccess;
    for (int k = 0; k < kStreams; ++k) {
      cudaError_t e = cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaMallocHost(&pstatus, sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&d_status, sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    return cudaMemset(d_status, 0, sizeof(uint32_t));
  }

  // lpq_status_fetch through the page-locked status word (a pageable
  // 4-byte copy costs tens of microseconds)
  lpq_status fetch_status(cudaStream_t s) {
    cudaError_t e = cudaMemcpyAsync(pstatus, d_status, sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    const uint32_t bits = *pstatus;
    if (e == cudaSuccess && bits) e = cudaMemsetAsync(d_status, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return cuda_fail(e);
    return map_status_bits(bits);
  }

  cudaError_t ensure_chunks(int64_t elems) {
    if (elems <= chunk_cap) return cudaSuccess;
    for (int k = 0; k < kStreams; ++k) {
      if (dbuf[k]) cudaFree(dbuf[k]);
      if (pin_in[k]) cudaFreeHost(pin_in[k]);
      if (pin_out[k]) cudaFreeHost(pin_out[k]);
      if (dcode[k]) cudaFree(dcode[k]);
      if (pcode[k]) cudaFreeHost(pcode[k]);
      if (sws[k]) cudaFree(sws[k]);
      dbuf[k] = pin_in[k] = pin_out[k] = nullptr;
      dcode[k] = pcode[k] = nullptr;
      sws[k] = nullptr;
    }
    chunk_cap = 0;
    sws_bytes = 0;
    const size_t bytes = sizeof(float) * (size_t)elems;
    // a chunk's block call: the row plans' state for rows > 32768 floats
    const size_t wsb = block_chunks_workspace(elems / 32768 + 1);
    for (int k = 0; k < kStreams; ++k) {
      cudaError_t e = cudaMalloc(&dbuf[k], bytes);
      if (e == cudaSuccess) e = cudaMallocHost(&pin_in[k], bytes);
      if (e == cudaSuccess) e = cudaMallocHost(&pin_out[k], bytes);
      if (e == cudaSuccess) e = cudaMalloc(&dcode[k], (size_t)elems);
      if (e == cudaSuccess) e = cudaMallocHost(&pcode[k], (size_t)elems);
      if (e == cudaSuccess) e = cudaMalloc(&sws[k], wsb);
      if (e != cudaSuccess) return e;
    }
    chunk_cap = elems;
    sws_bytes = wsb;
    return cudaSuccess;
  }

  cudaError_t ensure_full(int64_t elems) {
    if (elems <= dfull_cap) return cudaSuccess;
    if (dfull) cudaFree(dfull);
    dfull = nullptr;
    dfull_cap = 0;
    cudaError_t e = cudaMalloc(&dfull, sizeof(float) * (size_t)elems);
    if (e == cudaSuccess) dfull_cap = elems;
    return e;
  }

  cudaError_t ensure_stage(int64_t elems) {
    if (elems <= pstage_cap) return cudaSuccess;
    if (pstage) cudaFreeHost(pstage);
    pstage = nullptr;
    pstage_cap = 0;
    cudaError_t e = cudaMallocHost(&pstage, sizeof(float) * (size_t)elems);
    if (e == cudaSuccess) pstage_cap = elems;
    return e;
  }

  cudaError_t ensure_codes(int64_t elems, int64_t extent) {
    cudaError_t e = cudaSuccess;
    if (elems > codef_cap) {
      if (dcodef) cudaFree(dcodef);
      if (pcodef) cudaFreeHost(pcodef);
      dcodef = nullptr;
      pcodef = nullptr;
      codef_cap = 0;
      e = cudaMalloc(&dcodef, (size_t)elems);
      if (e == cudaSuccess) e = cudaMallocHost(&pcodef, (size_t)elems);
      if (e != cudaSuccess) return e;
      codef_cap = elems;
    }
    if (!daux) {
      e = cudaMalloc(&daux, sizeof(uint32_t));
      if (e != cudaSuccess) return e;
    }
    if (extent + 1 > paux_cap) {
      if (paux) cudaFreeHost(paux);
      paux = nullptr;
      paux_cap = 0;
      e = cudaMallocHost(&paux, sizeof(uint32_t) * (size_t)(extent + 1));
      if (e != cudaSuccess) return e;
      paux_cap = extent + 1;
    }
    return cudaSuccess;
  }

  cudaError_t ensure_ws(size_t bytes) {
    if (bytes <= ws_bytes) return cudaSuccess;
    if (ws) cudaFree(ws);
    ws = nullptr;
    ws_bytes = 0;
    cudaError_t e = cudaMalloc(&ws, bytes);
    if (e == cudaSuccess) ws_bytes = bytes;
    return e;
  }
};

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<HostCtx>> g_ctx;

HostCtx* context_for(int dev) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1);
  if (!g_ctx[dev]) {
    g_ctx[dev].reset(new HostCtx());
    g_ctx[dev]->dev = dev;
  }
  return g_ctx[dev].get();
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// How the host turns one-byte codes back into fp32 (bit-identical to the
// device's quantized values).
struct Decode {
  enum Kind { kLut = 1, kFixed = 2, kBlock = 3 };
  int kind = 0;
  const float* lut = nullptr;    // kLut: 256 entries
  float scale = 0.0f;            // kFixed: 2^-fl
  const double* delta = nullptr; // kBlock: delta per block
  int64_t extent = 1, stride = 1;
};

// Copy into page-locked staging memory with non-temporal (streaming) stores:
// the lines go to DRAM instead of staying dirty in the CPU caches, so the
// DMA that reads them next does not have to snoop them out of the caches
// (criterion 7's 2^20-float host call: fused 460 -> 400 us, composed 525 ->
// 495 us on the B200 host, scripts/gpu_stage_nt.sh).
static void memcpy_stage(void* dst_, const void* src_, size_t len) {
#if defined(__x86_64__)
  char* dst = static_cast<char*>(dst_);
  const char* src = static_cast<const char*>(src_);
  size_t head = (16u - ((uintptr_t)dst & 15u)) & 15u;
  if (head > len) head = len;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  len -= head;
  const size_t n64 = len / 64;
  for (size_t i = 0; i < n64; ++i) {
    const __m128i* s4 = reinterpret_cast<const __m128i*>(src + 64 * i);
    __m128i* d4 = reinterpret_cast<__m128i*>(dst + 64 * i);
    const __m128i a = _mm_loadu_si128(s4), b = _mm_loadu_si128(s4 + 1);
    const __m128i c = _mm_loadu_si128(s4 + 2), d = _mm_loadu_si128(s4 + 3);
    _mm_stream_si128(d4, a);
    _mm_stream_si128(d4 + 1, b);
    _mm_stream_si128(d4 + 2, c);
    _mm_stream_si128(d4 + 3, d);
  }
  std::memcpy(dst + 64 * n64, src + 64 * n64, len - 64 * n64);
  _mm_sfence();
#else
  std::memcpy(dst_, src_, len);
#endif
}

// Persistent copy workers for parallel_memcpy (spawning threads per call
// cost more than a 4 MB copy).  Parts of >= 512 KB, at most 16 threads
// including the caller.
class CopyPool {
  struct Job;

 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  int width() const { return (int)workers_.size() + 1; }

  // count units (bytes, or codes when dec) split over `parts` threads; a
  // unit of the destination is dst_unit bytes; first: element index of
  // src[0] within the tensor (block decode)
  void run(char* dst, const char* src, size_t count, int parts,
           const Decode* dec = nullptr, size_t first = 0, bool stage = false) {
    const size_t dst_unit = dec ? sizeof(float) : 1;
    // ceil(count / parts) rounded up to 64 units, so the parts cover count
    // (rounding count / parts down lost the remainder when the quotient was
    // already a multiple of 64: e.g. 1048577 codes over 16 parts)
    const size_t part = ((count + parts - 1) / parts + 63) & ~size_t(63);
    std::vector<Job> jobs;
    for (int t = 0; t < parts; ++t) {
      const size_t b = part * t;
      if (b >= count) break;
      jobs.push_back(Job{dst + b * dst_unit, src + b, std::min(part, count - b), dec,
                         first + b, stage});
    }
    run_list(std::move(jobs));
  }

 private:
  // jobs[0] runs on the caller, the rest on whichever thread takes them
  void run_list(std::vector<Job>&& all) {
    if (all.empty()) return;
    const Job first_job = all[0];
    std::unique_lock<std::mutex> lk(mu_);
    jobs_.assign(all.begin() + 1, all.end());
    next_ = 0;
    pending_ = jobs_.size();
    apending_.store(pending_, std::memory_order_release);
    ++gen_;
    agen_.store(gen_, std::memory_order_release);
    lk.unlock();
    cv_.notify_all();
    exec(first_job);
    lk.lock();
    // help with whatever the workers have not picked up, then wait
    while (next_ < jobs_.size()) {
      const Job j = jobs_[next_++];
      lk.unlock();
      exec(j);
      lk.lock();
      --pending_;
      apending_.fetch_sub(1, std::memory_order_acq_rel);
    }
    if (pending_ != 0) {  // spin briefly (the parts finish within microseconds)
      lk.unlock();
      spin_until([&] { return apending_.load(std::memory_order_acquire) == 0; });
      lk.lock();
    }
    done_.wait(lk, [&] { return pending_ == 0; });
  }

  struct Job {
    char* dst;
    const char* src;
    size_t len;          // bytes (copy) or codes (decode)
    const Decode* dec;   // null: memcpy
    size_t first;        // element index of src[0] (block decode)
    bool stage;          // memcpy into staging memory (memcpy_stage)
  };
  static void exec(const Job& j) {
    if (!j.dec) {
      if (j.stage) memcpy_stage(j.dst, j.src, j.len);
      else std::memcpy(j.dst, j.src, j.len);
      return;
    }
    float* d = reinterpret_cast<float*>(j.dst);
    const uint8_t* c = reinterpret_cast<const uint8_t*>(j.src);
    const Decode& dc = *j.dec;
    if (dc.kind == Decode::kLut) {
      for (size_t i = 0; i < j.len; ++i) d[i] = dc.lut[c[i]];
    } else if (dc.kind == Decode::kFixed) {  // k * 2^-fl: exact, +0 for k = 0
      const float sc = dc.scale;
      for (size_t i = 0; i < j.len; ++i) d[i] = (float)(int8_t)c[i] * sc;
    } else {  // block: float(double(k) * delta_b), b = (idx / stride) % extent
      size_t i = 0;
      while (i < j.len) {
        const uint64_t idx = j.first + i;
        const uint64_t blk = idx / (uint64_t)dc.stride;
        const double dl = dc.delta[blk % (uint64_t)dc.extent];
        const size_t end = std::min<size_t>(j.len, (size_t)((blk + 1) * dc.stride - j.first));
        for (; i < end; ++i) d[i] = (float)((double)(int8_t)c[i] * dl);
      }
    }
  }
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int n = (int)std::max(1u, std::min(hw, 16u)) - 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // poll pred for up to ~200 us before the caller falls back to blocking:
  // a host call issues its pool jobs back to back, and a condition-variable
  // wake-up costs tens of microseconds on this host
  template <class P>
  static bool spin_until(P pred) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0;; ++i) {
      if (pred()) return true;
#if defined(__x86_64__)
      __builtin_ia32_pause();  // leave the core's issue slots to its sibling
#endif
      if ((i & 63) == 63 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200))
        return false;
    }
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      if (!stop_ && !(gen_ != seen && next_ < jobs_.size())) {
        lk.unlock();
        spin_until([&] { return agen_.load(std::memory_order_acquire) != seen; });
        lk.lock();
      }
      cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < jobs_.size()); });
      if (stop_) return;
      while (next_ < jobs_.size()) {
        const Job j = jobs_[next_++];
        lk.unlock();
        exec(j);
        lk.lock();
        apending_.fetch_sub(1, std::memory_order_acq_rel);
        if (--pending_ == 0) done_.notify_all();
      }
      seen = gen_;
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::vector<Job> jobs_;
  size_t next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  std::atomic<uint64_t> agen_{0};      // gen_, for the spinning workers
  std::atomic<size_t> apending_{0};    // pending_, for the spinning caller
  bool stop_ = false;
};

std::mutex g_copy_mu;  // one parallel copy at a time (the pool is shared)

void parallel_memcpy(void* dst, const void* src, size_t bytes,
                     size_t serial_below = size_t(8) << 20, bool stage = false) {
  // below serial_below the workers' wake-up costs more than the copy; parts
  // of >= 256 KB (4 MB: 16 threads 11 us, 4 threads 28 us, 1 thread 228 us,
  // scripts/host_copy_probe.cpp)
  const size_t kMinPart = size_t(256) << 10;
  const size_t want = bytes < serial_below ? 1 : bytes / kMinPart;
  if (want <= 1) {
    if (stage) memcpy_stage(dst, src, bytes);
    else std::memcpy(dst, src, bytes);
    return;
  }
  std::lock_guard<std::mutex> lk(g_copy_mu);
  CopyPool& pool = CopyPool::get();
  const int parts = (int)std::min<size_t>(want, (size_t)pool.width());
  if (parts <= 1) {
    if (stage) memcpy_stage(dst, src, bytes);
    else std::memcpy(dst, src, bytes);
    return;
  }
  pool.run(static_cast<char*>(dst), static_cast<const char*>(src), bytes, parts, nullptr, 0,
           stage);
}

// dst[i] = decode(codes[i]) over the copy pool (256K codes = 1 MB of output
// per part, like the copies); first: tensor index of codes[0]
void parallel_decode(float* dst, const uint8_t* codes, size_t n, const Decode& dec,
                     size_t first = 0) {
  const size_t kMinPart = size_t(1) << 15;  // 32K codes (1M: 8 threads 14 us)
  const size_t want = std::max<size_t>(1, n / kMinPart);
  std::lock_guard<std::mutex> lk(g_copy_mu);
  CopyPool& pool = CopyPool::get();
  const int parts = (int)std::min<size_t>(want, (size_t)pool.width());
  pool.run(reinterpret_cast<char*>(dst), reinterpret_cast<const char*>(codes), n, parts,
           &dec, first);
}

// One-byte codes for the device->host copy of quantized results: saturating
// fixed point with wl <= 8 and float formats with 1 + exp + man <= 8, under
// NearestEven / Stochastic (whose zero results are +0 for fixed point; the
// float code keeps the sign, so a passed-through -0 survives).  Every
// quantized value of those formats is one of <= 256 bit patterns; the code
// is a bijection on them and the host decodes with a 256-entry table, so the
// output is bit-identical to copying the fp32 values -- at a quarter of the
// PCIe bytes.
bool byte_code_for(const lpq_format* f, int mode, ByteCode* bc, float* lut) {
  if (mode != kNearestEven && mode != kStochastic) return false;
  if (f->kind == LPQ_FIXED && f->saturate && f->wl <= 8) {
    bc->kind = 1;
    bc->scale = std::ldexp(1.0f, f->fl);
    const float down = std::ldexp(1.0f, -f->fl);
    for (int c = 0; c < 256; ++c) lut[c] = (float)(int8_t)(uint8_t)c * down + 0.0f;
    return true;
  }
  if (f->kind == LPQ_FLOAT && 1 + f->exp_bits + f->man_bits <= 8 && f->exp_bits >= 2) {
    const int bias = (1 << (f->exp_bits - 1)) - 1;
    bc->kind = 2;
    bc->man = f->man_bits;
    bc->min_exp = 1 - bias;
    const int nexp = 1 << f->exp_bits;  // E code 0 = zero, 1.. = min_exp..
    for (int c = 0; c < 256; ++c) {
      const int sign = (c >> 7) & 1;
      const int ei = (c >> f->man_bits) & (nexp - 1);
      const int mt = c & ((1 << f->man_bits) - 1);
      float v = 0.0f;
      if (ei != 0) {
        const int e = bc->min_exp + ei - 1;
        v = std::ldexp(1.0f + (float)mt / (float)(1 << f->man_bits), e);
      }
      lut[c] = sign ? -v : v;
    }
    return true;
  }
  return false;
}

// The host decoder of a ByteCode (fixed: arithmetic, float: the table).
Decode decoder_for(const lpq_format* f, const ByteCode& bc, const float* lut) {
  Decode d;
  if (bc.kind == 1) {
    d.kind = Decode::kFixed;
    d.scale = std::ldexp(1.0f, -f->fl);
  } else {
    d.kind = Decode::kLut;
    d.lut = lut;
  }
  return d;
}

int resolve_device(int device, lpq_status* st) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    *st = cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e);
    return -1;
  }
  if (device < 0) cudaGetDevice(&device);
  if (device >= count) {
    *st = LPQ_ERR_ARGUMENT;
    return -1;
  }
  *st = LPQ_OK;
  return device;
}

#define LPQ_TRY(expr)                          \
  do {                                         \
    cudaError_t _e = (expr);                   \
    if (_e != cudaSuccess) return cuda_fail(_e); \
  } while (0)

// Streaming path: chunks of `unit`-aligned elements, each quantized as an
// independent piece with its own flat index base (elementwise formats, or
// block formats whose blocks are whole contiguous rows of length `unit`).
lpq_status stream_quantize(HostCtx* c, const float* x, float* y, int64_t n,
                           int64_t unit, bool rows, uint64_t index_base,
                           const lpq_format* f, int mode, uint64_t seed,
                           uint64_t call) {
  // Chunks of 1 MB .. 64 MB.  Into page-locked output memory (the decode
  // runs at memory speed) at least ~16 chunks, so mid-size tensors overlap
  // copy-in, kernel, copy-out and decode: the 64 MB C1 tensor's e2e 64 ->
  // 84-88 GB/s with 16 chunks of 4 MB instead of 4 of 16 MB (8: 75-76, 32:
  // 72-73).  Into pageable memory not yet touched, the decode also takes the
  // page faults and smaller chunks stall the three-deep pipeline behind it
  // (32 MB: 2.47 / 2.66 / 4.28 ms with 4 / 8 / 16 chunks), so ~4 there.  1 GB
  // tensors keep 64 MB chunks either way.
  const bool pin_x = is_pinned(x), pin_y = is_pinned(y);
  const int64_t min_chunks = pin_y ? 16 : 4;
  const int64_t target = std::min<int64_t>(
      kChunkElems, std::max<int64_t>(int64_t(1) << 18, (n + min_chunks - 1) / min_chunks));
  const int64_t chunk = std::max<int64_t>(1, target / unit) * unit;
  LPQ_TRY(c->ensure_chunks(std::max<int64_t>(chunk, c->chunk_cap)));
  const int64_t nchunks = (n + chunk - 1) / chunk;
  lpq_format fr = *f;
  if (rows) fr.block_dim = 0;
  lpq_status qst = LPQ_OK;
  ByteCode bc{};
  float lut[256];
  const bool coded = !rows && byte_code_for(f, mode, &bc, lut);
  note_passes(1);   // one data pass for the whole call:
  PassScope scope;  // the chunks' device calls do not count again
  const Decode dec = coded ? decoder_for(f, bc, lut) : Decode{};
  auto finish = [&](int64_t ci) {
    const int k = (int)(ci % kStreams);
    cudaEventSynchronize(c->done[k]);
    const int64_t off = ci * chunk, len = std::min(chunk, n - off);
    if (coded) parallel_decode(y + off, c->pcode[k], (size_t)len, dec);
    else if (!pin_y) parallel_memcpy(y + off, c->pin_out[k], sizeof(float) * (size_t)len);
  };
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int k = (int)(ci % kStreams);
    if (ci >= kStreams) finish(ci - kStreams);
    const int64_t off = ci * chunk, len = std::min(chunk, n - off);
    const size_t bytes = sizeof(float) * (size_t)len;
    const float* src = x + off;
    if (!pin_x) {
      parallel_memcpy(c->pin_in[k], x + off, bytes, size_t(8) << 20, true);
      src = c->pin_in[k];
    }
    float* dst = pin_y ? y + off : c->pin_out[k];
    LPQ_TRY(cudaMemcpyAsync(c->dbuf[k], src, bytes, cudaMemcpyHostToDevice, c->st[k]));
    int64_t shp[2];
    int rank;
    if (rows) { shp[0] = len / unit; shp[1] = unit; rank = 2; }
    else { shp[0] = len; rank = 1; }
    qst = quantize_device(c->dbuf[k], c->dbuf[k], shp, rank,
                          index_base + (uint64_t)off, &fr, mode, seed, call,
                          c->sws[k], c->sws_bytes, c->d_status, c->st[k]);
    if (qst != LPQ_OK) break;
    if (coded) {  // a quarter of the bytes across PCIe; decoded in finish()
      LPQ_TRY(launch_encode8(c->dbuf[k], c->dcode[k], len, bc, c->st[k]));
      LPQ_TRY(cudaMemcpyAsync(c->pcode[k], c->dcode[k], (size_t)len,
                              cudaMemcpyDeviceToHost, c->st[k]));
    } else {
      LPQ_TRY(cudaMemcpyAsync(dst, c->dbuf[k], bytes, cudaMemcpyDeviceToHost, c->st[k]));
    }
    LPQ_TRY(cudaEventRecord(c->done[k], c->st[k]));
  }
  for (int64_t ci = std::max<int64_t>(0, nchunks - kStreams); ci < nchunks; ++ci)
    finish(ci);
  if (qst != LPQ_OK) {
    for (int k = 0; k < kStreams; ++k) cudaStreamSynchronize(c->st[k]);
    return qst;
  }
  return lpq_status_fetch(c->d_status, c->st[0]);
}

// Resident path: the whole tensor on the device (two-pass block formats).
lpq_status resident_quantize(HostCtx* c, const float* x, float* y,
                             const int64_t* shape, int rank, int64_t n,
                             uint64_t index_base, const lpq_format* f,
                             int mode, uint64_t seed, uint64_t call) {
  LPQ_TRY(c->ensure_full(n));
  const size_t wsb = lpq_workspace_size(f, shape, rank);
  if (wsb) LPQ_TRY(c->ensure_ws(wsb));
  cudaStream_t s = c->st[0];
  const size_t bytes = sizeof(float) * (size_t)n;
  if (is_pinned(x)) {
    LPQ_TRY(cudaMemcpyAsync(c->dfull, x, bytes, cudaMemcpyHostToDevice, s));
  } else {
    LPQ_TRY(c->ensure_chunks(std::min<int64_t>(n, kChunkElems)));
    for (int64_t off = 0; off < n; off += c->chunk_cap) {
      const int64_t len = std::min(c->chunk_cap, n - off);
      const int k = (int)((off / c->chunk_cap) % 2);
      LPQ_TRY(cudaEventSynchronize(c->done[k]));
      parallel_memcpy(c->pin_in[k], x + off, sizeof(float) * (size_t)len, size_t(8) << 20,
                      true);
      LPQ_TRY(cudaMemcpyAsync(c->dfull + off, c->pin_in[k],
                              sizeof(float) * (size_t)len,
                              cudaMemcpyHostToDevice, s));
      LPQ_TRY(cudaEventRecord(c->done[k], s));
    }
  }
  lpq_status qst = quantize_device(c->dfull, c->dfull, shape, rank, index_base,
                                   f, mode, seed, call, c->ws, c->ws_bytes,
                                   c->d_status, s);
  if (qst != LPQ_OK) {
    cudaStreamSynchronize(s);
    return qst;
  }
  if (is_pinned(y)) {
    LPQ_TRY(cudaMemcpyAsync(y, c->dfull, bytes, cudaMemcpyDeviceToHost, s));
  } else {
    LPQ_TRY(c->ensure_chunks(std::min<int64_t>(n, kChunkElems)));
    for (int64_t off = 0; off < n; off += c->chunk_cap) {
      const int64_t len = std::min(c->chunk_cap, n - off);
      LPQ_TRY(cudaMemcpyAsync(c->pin_out[0], c->dfull + off,
                              sizeof(float) * (size_t)len,
                              cudaMemcpyDeviceToHost, s));
      LPQ_TRY(cudaStreamSynchronize(s));
      parallel_memcpy(y + off, c->pin_out[0], sizeof(float) * (size_t)len);
    }
  }
  return lpq_status_fetch(c->d_status, s);
}

// Host -> device copy of a whole (small) tensor: pinned memory directly;
// pageable memory through the context's page-locked staging buffer, filled
// by the copy pool (the driver's own staging of pageable copies runs at
// ~18 GB/s on the B200 host, scripts/host_copy_probe.cpp: 232 us for 4 MB
// against ~11 us of pool memcpy + 86 us of DMA).
cudaError_t h2d_small(HostCtx* c, float* d, const float* x, int64_t n, cudaStream_t s) {
  const size_t bytes = sizeof(float) * (size_t)n;
  if (is_pinned(x) || bytes < (size_t(256) << 10))
    return cudaMemcpyAsync(d, x, bytes, cudaMemcpyHostToDevice, s);
  cudaError_t e = c->ensure_stage(n);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(s);  // the staging buffer may still feed a copy
  if (e != cudaSuccess) return e;
  parallel_memcpy(c->pstage, x, bytes, size_t(256) << 10, true);
  return cudaMemcpyAsync(d, c->pstage, bytes, cudaMemcpyHostToDevice, s);
}

// Device -> host copy of a whole (small) tensor, then the status fetch
// (which synchronises the stream); pageable destinations through the
// staging buffer (DMA, then the copy pool).
lpq_status d2h_small_and_fetch(HostCtx* c, float* y, const float* d, int64_t n,
                               cudaStream_t s) {
  const size_t bytes = sizeof(float) * (size_t)n;
  if (is_pinned(y) || bytes < (size_t(256) << 10)) {
    LPQ_TRY(cudaMemcpyAsync(y, d, bytes, cudaMemcpyDeviceToHost, s));
    return c->fetch_status(s);
  }
  LPQ_TRY(c->ensure_stage(n));
  LPQ_TRY(cudaMemcpyAsync(c->pstage, d, bytes, cudaMemcpyDeviceToHost, s));
  const lpq_status st = c->fetch_status(s);
  if (st != LPQ_OK) return st;
  parallel_memcpy(y, c->pstage, bytes, size_t(256) << 10);
  return LPQ_OK;
}

// Small tensors (<= 16 MB): one staged copy in, the device call, one copy
// out on one stream.  Formats whose every quantized value has a one-byte code
// (ByteCode: fixed wl <= 8 saturating, float 1 + exp + man <= 8; block wl <=
// 8 on the plans that leave the block maxima in the workspace) copy the codes
// back instead of fp32 -- a quarter of the device->host bytes, decoded
// bit-exactly on the host by the copy pool.  (Pipelining the call in parts
// over two streams was measured on the B200 host, scripts/host_crit7.cpp:
// the part's H2D and the previous part's D2H complete together -- the copies
// do not overlap here -- so 2..8 parts only added ~15 us of API calls each.)
lpq_status direct_quantize(HostCtx* c, const float* x, float* y,
                           const int64_t* shape, int rank, int64_t n,
                           uint64_t index_base, const lpq_format* f, int mode,
                           uint64_t seed, uint64_t call) {
  LPQ_TRY(c->ensure_full(n));
  const size_t wsb = lpq_workspace_size(f, shape, rank);
  if (wsb) LPQ_TRY(c->ensure_ws(wsb));
  cudaStream_t s = c->st[0];
  ByteCode bc{};
  float lut[256];
  const bool coded = byte_code_for(f, mode, &bc, lut);
  LPQ_TRY(h2d_small(c, c->dfull, x, n, s));
  const lpq_status qst = quantize_device(c->dfull, c->dfull, shape, rank, index_base,
                                         f, mode, seed, call, c->ws, c->ws_bytes,
                                         c->d_status, s);
  if (qst != LPQ_OK) {
    cudaStreamSynchronize(s);
    return qst;
  }
  if (coded) {
    LPQ_TRY(c->ensure_codes(n, 1));
    LPQ_TRY(launch_encode8(c->dfull, c->dcodef, n, bc, s));
    LPQ_TRY(cudaMemcpyAsync(c->pcodef, c->dcodef, (size_t)n, cudaMemcpyDeviceToHost, s));
    const lpq_status st = c->fetch_status(s);
    if (st != LPQ_OK) return st;
    parallel_decode(y, c->pcodef, (size_t)n, decoder_for(f, bc, lut));
    return LPQ_OK;
  }
  BlockGeom g{1, 1, n};
  bool bcoded = false;
  if (!coded && f->kind == LPQ_BLOCK && f->wl <= 8 &&
      (mode == kNearestEven || mode == kStochastic) &&
      block_geometry(f, shape, rank, &g) == LPQ_OK)
    bcoded = block_plan_maxima_in_ws(block_plan(g, c->dfull, c->dfull));
  if (!bcoded) return d2h_small_and_fetch(c, y, c->dfull, n, s);
  LPQ_TRY(c->ensure_codes(n, g.extent));
  LPQ_TRY(cudaMemsetAsync(c->daux, 0, sizeof(uint32_t), s));
  LPQ_TRY(launch_encode_block8(c->dfull, c->dcodef, g, static_cast<const uint32_t*>(c->ws),
                               f->wl, c->daux, s));
  LPQ_TRY(cudaMemcpyAsync(c->paux, c->ws, sizeof(uint32_t) * (size_t)g.extent,
                          cudaMemcpyDeviceToHost, s));
  LPQ_TRY(cudaMemcpyAsync(c->paux + g.extent, c->daux, sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, s));
  LPQ_TRY(cudaMemcpyAsync(c->pcodef, c->dcodef, (size_t)n, cudaMemcpyDeviceToHost, s));
  const lpq_status st = c->fetch_status(s);
  if (st != LPQ_OK) return st;
  if (c->paux[g.extent] != 0u)  // a result in the subnormal range: fp32 copy
    return d2h_small_and_fetch(c, y, c->dfull, n, s);
  std::vector<double> delta((size_t)g.extent);
  for (int64_t b = 0; b < g.extent; ++b) {
    const uint32_t m = c->paux[b];
    delta[(size_t)b] = m ? std::ldexp(1.0, float_exponent_bits(m) - (f->wl - 2)) : 0.0;
  }
  Decode dec;
  dec.kind = Decode::kBlock;
  dec.delta = delta.data();
  dec.extent = g.extent;
  dec.stride = g.stride;
  parallel_decode(y, c->pcodef, (size_t)n, dec);
  return LPQ_OK;
}

}  // namespace

lpq_status host_context_quantize(const float* x, float* y,
                                 const int64_t* shape, int rank,
                                 uint64_t index_base, const lpq_format* f,
                                 int mode, uint64_t seed, uint64_t call,
                                 int device) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  int64_t n = 0;
  st = check_shape(shape, rank, &n);
  if (st != LPQ_OK) return st;
  if (mode < 0 || mode > 3) return LPQ_ERR_ARGUMENT;
  BlockGeom g{1, 1, n};
  if (f->kind == LPQ_BLOCK) {
    st = block_geometry(f, shape, rank, &g);
    if (st != LPQ_OK) return st;
  }
  if (n == 0) return LPQ_OK;
  if (!x || !y) return LPQ_ERR_ARGUMENT;
  const int dev = resolve_device(device, &st);
  if (dev < 0) return st;
  DeviceGuard guard(dev);
  HostCtx* c = context_for(dev);
  std::lock_guard<std::mutex> lk(c->mu);
  cudaError_t e = c->init();
  if (e != cudaSuccess) return cuda_fail(e);
  // one staged call up to 16 MB of pageable input; page-locked inputs need no
  // staging copy and gain from the chunked overlap sooner (8 / 12 / 16 MB:
  // 580 / 941 / 1266 us direct vs 347 / 478 / 637 us streamed; pageable ones
  // the other way round, 607 / 995 / 1092 vs 691 / 1057 / 1327 us)
  const int64_t direct_max = is_pinned(x) ? (int64_t(4) << 20) : (int64_t(16) << 20);
  if ((int64_t)sizeof(float) * n <= direct_max)
    return direct_quantize(c, x, y, shape, rank, n, index_base, f, mode, seed, call);
  if (f->kind != LPQ_BLOCK)
    return stream_quantize(c, x, y, n, 1, false, index_base, f, mode, seed, call);
  // an aligned device buffer decides the plan exactly as the device call will
  static const float* kAligned = reinterpret_cast<const float*>(uintptr_t(256));
  if (block_plan_single_pass(block_plan(g, kAligned, kAligned)))
    return stream_quantize(c, x, y, n, g.stride, true, index_base, f, mode,
                           seed, call);
  return resident_quantize(c, x, y, shape, rank, n, index_base, f, mode, seed,
                           call);
}

lpq_status host_context_composed(const float* x, float* y,
                                 const int64_t* shape, int rank,
                                 uint64_t index_base, const lpq_format* f,
                                 int mode, uint64_t seed, uint64_t call,
                                 int device) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  if (f->kind == LPQ_FLOAT) return LPQ_ERR_UNSUPPORTED;
  int64_t n = 0;
  st = check_shape(shape, rank, &n);
  if (st != LPQ_OK) return st;
  if (f->kind == LPQ_BLOCK) {
    BlockGeom g;
    st = block_geometry(f, shape, rank, &g);
    if (st != LPQ_OK) return st;
  }
  if (n == 0) return LPQ_OK;
  if (!x || !y) return LPQ_ERR_ARGUMENT;
  const int dev = resolve_device(device, &st);
  if (dev < 0) return st;
  DeviceGuard guard(dev);
  HostCtx* c = context_for(dev);
  std::lock_guard<std::mutex> lk(c->mu);
  LPQ_TRY(c->init());
  LPQ_TRY(c->ensure_full(n));
  const size_t wsb = lpq_composed_workspace_size(f, shape, rank);
  LPQ_TRY(c->ensure_ws(wsb));
  cudaStream_t s = c->st[0];
  // the same host staging as the fused direct path (fp32 both ways: the
  // many-kernel chain's last op writes fp32)
  LPQ_TRY(h2d_small(c, c->dfull, x, n, s));
  st = quantize_composed_device(c->dfull, c->dfull, shape, rank, index_base, f,
                                mode, seed, call, c->ws, c->ws_bytes,
                                c->d_status, s);
  if (st != LPQ_OK) {
    cudaStreamSynchronize(s);
    return st;
  }
  return d2h_small_and_fetch(c, y, c->dfull, n, s);
}

void shutdown_contexts() {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  g_ctx.clear();
}

}  // namespace lpq

extern "C" {

lpq_status lpq_quantize_host(const float* x, float* y, const int64_t* shape,
                             int rank, uint64_t index_base,
                             const lpq_format* f, int mode, uint64_t seed,
                             uint64_t call, int device) {
  return lpq::host_context_quantize(x, y, shape, rank, index_base, f, mode,
                                    seed, call, device);
}

lpq_status lpq_quantize_composed_host(const float* x, float* y,
                                      const int64_t* shape, int rank,
                                      uint64_t index_base, const lpq_format* f,
                                      int mode, uint64_t seed, uint64_t call,
                                      int device) {
  return lpq::host_context_composed(x, y, shape, rank, index_base, f, mode,
                                    seed, call, device);
}

void lpq_shutdown(void) { lpq::shutdown_contexts(); }

void lpq_host_bytes_per_element(const lpq_format* f, int mode, int* h2d, int* d2h) {
  lpq::ByteCode bc{};
  float lut[256];
  const bool coded = f && lpq::check_format(f) == LPQ_OK && f->kind != LPQ_BLOCK &&
                     lpq::byte_code_for(f, mode, &bc, lut);
  if (h2d) *h2d = 4;
  if (d2h) *d2h = coded ? 1 : 4;
}

}  // extern "C"
