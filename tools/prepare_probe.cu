// Host-visible cost of vpipg_prepare and of the CUDA calls it is made of
// (B200, warm): medians of 200 calls, microseconds.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "vpipg.h"

using clk = std::chrono::steady_clock;
static double us(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::micro>(b - a).count();
}
static double med(std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; }
struct Big { double v[512]; };
__global__ void empty_k(int) {}
__global__ void big_k(const __grid_constant__ Big b) { if (b.v[0] == 123.0) printf("x"); }

int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  for (int n : {8, 32, 1024}) {
    std::vector<double> vx(n), vy(n);
    for (int i = 0; i < n; ++i) { vx[i] = cos(2 * M_PI * i / n); vy[i] = sin(2 * M_PI * i / n); }
    std::vector<double> e, r;
    for (int it = 0; it < 250; ++it) {
      vpipg_poly* p = nullptr;
      auto t0 = clk::now();
      vpipg_prepare(vx.data(), vy.data(), n, VPIPG_KIND_ALL, 0, s, &p);
      auto t1 = clk::now();
      vpipg_poly_status(p);
      auto t2 = clk::now();
      vpipg_destroy(p);
      if (it >= 50) { e.push_back(us(t0, t1)); r.push_back(us(t0, t2)); }
    }
    printf("{\"n\": %d, \"prepare_us\": %.2f, \"ready_us\": %.2f}\n", n, med(e), med(r));
  }
  cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0);
  void* hp; cudaHostAlloc(&hp, 1 << 20, 0);
  void* d; cudaMalloc(&d, 1 << 20);
  cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  Big big{};
  std::vector<double> ta, tl, tb, tm, te, tf, ts;
  for (int it = 0; it < 250; ++it) {
    void* p;
    auto t0 = clk::now(); cudaMallocFromPoolAsync(&p, 65536, pool, s);
    auto t1 = clk::now(); empty_k<<<1, 256, 0, s>>>(0);
    auto t2 = clk::now(); big_k<<<1, 256, 0, s>>>(big);
    auto t3 = clk::now(); cudaMemcpyAsync(hp, d, 4096, cudaMemcpyDeviceToHost, s);
    auto t4 = clk::now(); cudaEventRecord(ev, s);
    auto t5 = clk::now(); cudaFreeAsync(p, s);
    auto t6 = clk::now(); cudaStreamSynchronize(s);
    auto t7 = clk::now();
    if (it >= 50) { ta.push_back(us(t0, t1)); tl.push_back(us(t1, t2)); tb.push_back(us(t2, t3));
                    tm.push_back(us(t3, t4)); te.push_back(us(t4, t5)); tf.push_back(us(t5, t6));
                    ts.push_back(us(t6, t7)); }
  }
  printf("{\"mallocFromPoolAsync\": %.2f, \"launch\": %.2f, \"launch_4KB_params\": %.2f, "
         "\"memcpyAsync_D2H_pinned\": %.2f, \"eventRecord\": %.2f, \"freeAsync\": %.2f, \"sync\": %.2f}\n",
         med(ta), med(tl), med(tb), med(tm), med(te), med(tf), med(ts));
  return 0;
}
