// Breakdown of the C++ API call monoalign::align at the acceptance suite's
// scaling-law sizes (B8, S = 4T): output allocation alone, the C-ABI host
// entry into a pre-faulted pageable buffer, and the whole call.
// build: g++ -O2 -std=c++20 -Iinclude tools/host_path_timing.cpp \
//          -Lpaper_2409_07704_b200/_lib -lmonoalign_b200 -Wl,-rpath,$PWD/paper_2409_07704_b200/_lib
#include <chrono>
#include <cstdio>
#include <vector>

#include "monoalign/align.hpp"
#include "monoalign/bench.hpp"
#include "monoalign_b200.h"

int main() {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  for (int t : {512, 640, 768, 896, 1024}) {
    const int s = 4 * t, B = 8;
    const auto batch = monoalign::bench::generate_random_batch(B, t, s, 5005);
    monoalign::MasConfig cfg;
    cfg.engine = monoalign::EngineKind::Reference;
    for (int w = 0; w < 2; ++w) (void)monoalign::align(batch, cfg);
    double a_alloc = 1e9, a_host = 1e9, a_full = 1e9;
    std::vector<uint8_t> pre(static_cast<size_t>(B) * t * s, 0);
    mas_config_t c;
    mas_config_default(&c);
    c.engine = MAS_ENGINE_REFERENCE;
    mas_error_t err;
    for (int r = 0; r < 7; ++r) {
      auto t0 = clk::now();
      { std::vector<uint8_t> v(static_cast<size_t>(B) * t * s); }
      auto t1 = clk::now();
      mas_align_host(batch.values.data(), B, t, s, nullptr, &c, pre.data(), nullptr, &err);
      auto t2 = clk::now();
      (void)monoalign::align(batch, cfg);
      auto t3 = clk::now();
      a_alloc = std::min(a_alloc, ms(t0, t1));
      a_host = std::min(a_host, ms(t1, t2));
      a_full = std::min(a_full, ms(t2, t3));
    }
    std::printf("T=%d S=%d: out alloc %.2f ms, mas_align_host(prefaulted out) %.2f ms, align %.2f ms\n",
                t, s, a_alloc, a_host, a_full);
  }
  return 0;
}
