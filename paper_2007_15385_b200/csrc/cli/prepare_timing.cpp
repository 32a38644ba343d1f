// prepare_timing -- host-visible cost of the C-ABI preparation, measured by a
// C++ caller (bench.py's `convert` block runs it; Python's own call overhead
// would otherwise dominate a ~10 us figure).
//
//   prepare_timing N [N ...]   -> one JSON line per N: medians over 200 warm
//   calls of vpipg_prepare (returns after host validation + enqueue) and of
//   vpipg_prepare + vpipg_poly_status (until the handle is usable), in us.
// The polygon is the regular N-gon of radius 1 (vpip::regular_polygon's
// vertices), prepared with all three kinds on device 0.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vpipg.h"

int main(int argc, char** argv) {
  using clk = std::chrono::steady_clock;
  auto us = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count();
  };
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  for (int i = 1; i < argc; ++i) {
    const int n = std::atoi(argv[i]);
    std::vector<double> vx(n), vy(n);
    if (vpipg_regular_polygon(n, 1.0, 0.0, 0.0, vx.data(), vy.data()) != 0) return 2;
    std::vector<double> enq, rdy;
    for (int it = 0; it < 250; ++it) {
      vpipg_poly* p = nullptr;
      const auto t0 = clk::now();
      const int rc = vpipg_prepare(vx.data(), vy.data(), n, VPIPG_KIND_ALL, 0, nullptr, &p);
      const auto t1 = clk::now();
      const int st = rc ? rc : vpipg_poly_status(p);
      const auto t2 = clk::now();
      vpipg_destroy(p);
      if (st) {
        std::fprintf(stderr, "prepare n=%d: %s\n", n, vpipg_strerror(st));
        return 1;
      }
      if (it >= 50) {
        enq.push_back(us(t0, t1));
        rdy.push_back(us(t0, t2));
      }
    }
    std::printf("{\"n\": %d, \"prepare_enqueue_us\": %.2f, \"prepare_ready_us\": %.2f}\n", n,
                med(enq), med(rdy));
  }
  return 0;
}
