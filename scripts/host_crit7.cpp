// host_crit7.cpp -- the reference acceptance suite's criterion 7 timing
// (proj/tests/acceptance.cpp:340-377 via bench.cpp:43-95) restated against
// liblpq.so's host API, with per-phase detail: 2^20 floats shaped {16384, 64},
// NearestEven, fixed(8,4) and block(8, whole tensor); each call allocates and
// value-initialises its output like the drop-in's Tensor; median of 7 after 2
// warm-ups, fused then composed, several rounds.
// Build: g++ -O2 -std=c++17 scripts/host_crit7.cpp -Iinclude \
//          -Lpaper_1910_04540_b200/lib -llpq -Wl,-rpath,$PWD/paper_1910_04540_b200/lib
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "lpq.h"

using Clock = std::chrono::steady_clock;

static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  const int64_t n = 1 << 20;
  const int64_t shape[2] = {16384, 64};
  std::vector<float> x(n);
  for (int64_t i = 0; i < n; ++i) x[i] = -4.0f + 8.0f * (float)((i * 2654435761u) % 1000003) / 1000003.0f;
  lpq_format fx{};
  fx.kind = LPQ_FIXED;
  fx.wl = 8;
  fx.fl = 4;
  fx.saturate = 1;
  fx.block_dim = -1;
  lpq_format fb{};
  fb.kind = LPQ_BLOCK;
  fb.wl = 8;
  fb.block_dim = -1;
  for (int round = 0; round < 3; ++round) {
    for (const lpq_format* f : {&fx, &fb}) {
      double med[2];
      for (int impl = 0; impl < 2; ++impl) {
        auto call = [&]() {
          std::vector<float> y(n);
          const lpq_status st =
              impl == 0 ? lpq_quantize_host(x.data(), y.data(), shape, 2, 0, f, 0, 0x15EED, 0, -1)
                        : lpq_quantize_composed_host(x.data(), y.data(), shape, 2, 0, f, 0,
                                                     0x15EED, 0, -1);
          if (st != LPQ_OK) std::printf("status %d\n", (int)st);
        };
        for (int w = 0; w < 2; ++w) call();
        std::vector<double> ts;
        for (int r = 0; r < 7; ++r) {
          const auto t0 = Clock::now();
          call();
          ts.push_back(std::chrono::duration<double, std::micro>(Clock::now() - t0).count());
        }
        med[impl] = median(ts);
      }
      std::printf("round %d %s: fused %.1f us composed %.1f us ratio %.3f\n", round,
                  f == &fx ? "fixed(8,4)" : "block(8)", med[0], med[1], med[0] / med[1]);
    }
  }
  // the value-initialised output alone
  std::vector<double> ts;
  for (int r = 0; r < 9; ++r) {
    const auto t0 = Clock::now();
    std::vector<float> y(n);
    asm volatile("" ::"r"(y.data()) : "memory");
    ts.push_back(std::chrono::duration<double, std::micro>(Clock::now() - t0).count());
  }
  std::printf("vector<float>(2^20) alone: %.1f us\n", median(ts));
  return 0;
}
