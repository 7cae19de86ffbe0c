// host_copy_probe.cpp -- diagnostic for the small-tensor host path
// (criterion 7 of the reference's acceptance suite: 2^20 floats through the
// host API).  Medians of 41 runs of each phase on pageable buffers shaped
// like the drop-in's std::vector<float> (freshly value-initialised output):
//   driver pageable H2D / D2H, pinned H2D / D2H, our own staging (T threads
//   memcpy into pinned + DMA, chunked), T-thread int8 -> fp32 decode.
// Build: nvcc -O3 -std=c++17 scripts/host_copy_probe.cpp -o build/host_copy_probe -lpthread
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

using Clock = std::chrono::steady_clock;

static double med(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

template <class F>
static double time_us(F f, int reps = 41) {
  for (int i = 0; i < 3; ++i) f();
  std::vector<double> ts;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = Clock::now();
    f();
    ts.push_back(std::chrono::duration<double, std::micro>(Clock::now() - t0).count());
  }
  return med(ts);
}

// run fn(part) for part in [0, parts) on `parts` threads (spawned per call:
// an upper bound on a pool's wake-up cost)
struct Pool {
  std::vector<std::thread> th;
  std::atomic<int> gen{0}, done{0};
  std::function<void(int)> job;
  int n;
  std::atomic<bool> stop{false};
  explicit Pool(int n_) : n(n_) {
    for (int i = 1; i < n; ++i)
      th.emplace_back([this, i] {
        int seen = 0;
        while (!stop.load()) {
          const int g = gen.load(std::memory_order_acquire);
          if (g == seen) { std::this_thread::yield(); continue; }
          seen = g;
          job(i);
          done.fetch_add(1, std::memory_order_acq_rel);
        }
      });
  }
  ~Pool() {
    stop = true;
    for (auto& t : th) t.join();
  }
  void run(std::function<void(int)> f) {
    job = f;
    done.store(0);
    gen.fetch_add(1, std::memory_order_acq_rel);
    f(0);
    while (done.load(std::memory_order_acquire) < n - 1) {}
  }
};

int main() {
  const size_t n = size_t(1) << 20, bytes = 4 * n;
  std::vector<float> x(n);
  for (size_t i = 0; i < n; ++i) x[i] = (float)(i % 1000) * 0.01f - 5.0f;
  float *d = nullptr, *pin = nullptr;
  uint8_t *dc = nullptr, *pc = nullptr;
  cudaMalloc(&d, bytes);
  cudaMalloc(&dc, n);
  cudaMallocHost(&pin, bytes);
  cudaMallocHost(&pc, n);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  printf("driver pageable H2D 4MB: %.1f us\n", time_us([&] {
           cudaMemcpyAsync(d, x.data(), bytes, cudaMemcpyHostToDevice, s);
           cudaStreamSynchronize(s);
         }));
  printf("pinned H2D 4MB: %.1f us\n", time_us([&] {
           cudaMemcpyAsync(d, pin, bytes, cudaMemcpyHostToDevice, s);
           cudaStreamSynchronize(s);
         }));
  printf("pinned D2H 4MB: %.1f us\n", time_us([&] {
           cudaMemcpyAsync(pin, d, bytes, cudaMemcpyDeviceToHost, s);
           cudaStreamSynchronize(s);
         }));
  printf("pinned D2H 1MB codes: %.1f us\n", time_us([&] {
           cudaMemcpyAsync(pc, dc, n, cudaMemcpyDeviceToHost, s);
           cudaStreamSynchronize(s);
         }));
  printf("driver pageable D2H 4MB into fresh vector: %.1f us\n", time_us([&] {
           std::vector<float> y(n);
           cudaMemcpyAsync(y.data(), d, bytes, cudaMemcpyDeviceToHost, s);
           cudaStreamSynchronize(s);
         }));
  printf("fresh vector<float>(2^20) alone: %.1f us\n", time_us([&] {
           std::vector<float> y(n);
           asm volatile("" ::"r"(y.data()) : "memory");
         }));
  for (int T : {1, 2, 4, 8, 16}) {
    Pool pool(T);
    printf("T=%2d memcpy 4MB pageable->pinned: %.1f us\n", T, time_us([&] {
             pool.run([&](int p) {
               const size_t part = bytes / T;
               std::memcpy((char*)pin + p * part, (const char*)x.data() + p * part, part);
             });
           }));
    for (int chunks : {1, 2, 4, 8}) {
      printf("T=%2d staged H2D 4MB in %d chunks: %.1f us\n", T, chunks, time_us([&] {
               const size_t cb = bytes / chunks;
               for (int c = 0; c < chunks; ++c) {
                 pool.run([&](int p) {
                   const size_t part = cb / T;
                   std::memcpy((char*)pin + c * cb + p * part,
                               (const char*)x.data() + c * cb + p * part, part);
                 });
                 cudaMemcpyAsync((char*)d + c * cb, (char*)pin + c * cb, cb,
                                 cudaMemcpyHostToDevice, s);
               }
               cudaStreamSynchronize(s);
             }));
    }
    std::vector<float> y(n);
    printf("T=%2d decode 1M int8->fp32 (existing output): %.1f us\n", T, time_us([&] {
             pool.run([&](int p) {
               const size_t part = n / T;
               float* o = y.data() + p * part;
               const int8_t* c = (const int8_t*)pc + p * part;
               for (size_t i = 0; i < part; ++i) o[i] = (float)c[i] * 0.0625f;
             });
           }));
    printf("T=%2d memcpy 4MB pinned->pageable: %.1f us\n", T, time_us([&] {
             pool.run([&](int p) {
               const size_t part = bytes / T;
               std::memcpy((char*)y.data() + p * part, (const char*)pin + p * part, part);
             });
           }));
  }
  printf("cpus %u\n", std::thread::hardware_concurrency());
  return 0;
}
