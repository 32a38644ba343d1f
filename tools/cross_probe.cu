// Crossing-engine formulation probe (sm_100a). Each thread holds P points in
// registers and runs the ray-crossing parity over an n-edge table held in the
// kernel parameter bank (uniform registers), R times; the variants must give
// identical parity words (checked) and are timed per point-edge.
//  V0: (H_k ^ H_{k-1}) & ~D, XOR-reduced (2 FADD + FFMA + 1.5 LOP3)
//  V1: sign(h_k * h_{k-1}) & ~D, par ^= P & ~D (2 FADD + FFMA + FMUL + LOP3)
//  V2: predicates: FSETP A_k, FSETP.XOR in_k, FFMA x-intercept, FSETP.AND, PLOP3
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

constexpr int kMax = 64;
struct Tab { float4 v[kMax]; float4 w[kMax]; int n; };  // v: (u.x, u.y, z, w.x); w: (e, u.y, 0, 0)
constexpr int P = 12;

template <int V>
__global__ void __launch_bounds__(256, 2) probe(const __grid_constant__ Tab t, int reps, uint32_t* out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  float x[P], y[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    uint32_t s = (tid * P + p) * 2654435761u;
    s ^= s >> 13; s *= 0x5bd1e995u; s ^= s >> 15;
    x[p] = ((s & 0xffff) / 65536.f) * 3.f - 1.5f;
    y[p] = ((s >> 16) / 65536.f) * 3.f - 1.5f;
  }
  uint32_t res = 0;
  const int n = t.n;
  for (int r = 0; r < reps; ++r) {
    uint32_t par[P];
#pragma unroll
    for (int p = 0; p < P; ++p) par[p] = 0;
    if constexpr (V == 3) {
      float hp[P];
      const float4 last = t.v[n - 1];
#pragma unroll
      for (int p = 0; p < P; ++p) hp[p] = y[p] - last.y;
#pragma unroll 1
      for (int k = 0; k < n; k += 4) {  // n % 4 == 0 here
        const float4 v0 = t.v[k], v1 = t.v[k + 1], v2 = t.v[k + 2], v3 = t.v[k + 3];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float h0 = y[p] - v0.y, g0 = v0.x - x[p], h1 = y[p] - v1.y;
          const float h2 = y[p] - v2.y, g2 = v2.x - x[p], h3 = y[p] - v3.y;
          const uint32_t t0 = (__float_as_uint(h0) ^ __float_as_uint(hp[p])) & ~__float_as_uint(fmaf(h0, v0.z, g0));
          const uint32_t t1 = (__float_as_uint(h1) ^ __float_as_uint(h0)) & ~__float_as_uint(fmaf(h0, v1.z, g0));
          const uint32_t t2 = (__float_as_uint(h2) ^ __float_as_uint(h1)) & ~__float_as_uint(fmaf(h2, v2.z, g2));
          const uint32_t t3 = (__float_as_uint(h3) ^ __float_as_uint(h2)) & ~__float_as_uint(fmaf(h2, v3.z, g2));
          par[p] ^= t0 ^ t1 ^ t2 ^ t3;
          hp[p] = h3;
        }
      }
    } else if constexpr (V == 0 || V == 1) {
      float hp[P], gp[P];
      const float4 last = t.v[n - 1];
#pragma unroll
      for (int p = 0; p < P; ++p) { hp[p] = y[p] - last.y; gp[p] = last.x - x[p]; }
#pragma unroll 2
      for (int k = 0; k < n; ++k) {
        const float4 v = t.v[k];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float h = y[p] - v.y;
          const float d = fmaf(hp[p], v.z, gp[p]);
          if (V == 0) par[p] ^= (__float_as_uint(h) ^ __float_as_uint(hp[p])) & ~__float_as_uint(d);
          else par[p] ^= __float_as_uint(h * hp[p]) & ~__float_as_uint(d);
          hp[p] = h;
          gp[p] = v.x - x[p];
        }
      }
    } else {
      // predicates; A = (u.y > qy), crossing iff in range and qx < x-intercept
      const float4 last = t.v[n - 1];
      uint32_t ap[P];
#pragma unroll
      for (int p = 0; p < P; ++p) ap[p] = last.y > y[p];
#pragma unroll 2
      for (int k = 0; k < n; ++k) {
        const float4 v = t.v[k];
        const float e = t.w[k].x;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          uint32_t a, c;
          asm("{\n\t.reg .pred pa, pprev, pin, pc, ppar;\n\t"
              "setp.ne.u32 pprev, %2, 0;\n\t"
              "setp.ne.u32 ppar, %3, 0;\n\t"
              "setp.gt.f32 pa, %4, %5;\n\t"
              "setp.gt.xor.f32 pin, %4, %5, pprev;\n\t"
              "setp.lt.and.f32 pc, %6, %7, pin;\n\t"
              "xor.pred ppar, ppar, pc;\n\t"
              "selp.u32 %0, 1, 0, pa;\n\t"
              "selp.u32 %1, 0x80000000, 0, ppar;\n\t}"
              : "=r"(a), "=r"(c)
              : "r"(ap[p]), "r"(par[p]), "f"(v.y), "f"(y[p]), "f"(x[p]), "f"(fmaf(y[p], v.z, e)));
          ap[p] = a;
          par[p] = c;
        }
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) res += (par[p] >> 31) << p;
  }
  out[tid] = res;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32;
  Tab t{};
  t.n = n;
  std::vector<double> vx(n), vy(n);
  for (int i = 0; i < n; ++i) {
    const double a = 2 * M_PI * (i + 0.3 * (i % 3) / 3.0) / n;
    vx[i] = cos(a) * (1 + 0.05 * ((i * 7) % 5 - 2) / 2.0);
    vy[i] = sin(a) * (1 + 0.05 * ((i * 3) % 5 - 2) / 2.0);
  }
  for (int k = 0; k < n; ++k) {
    const int j = (k + n - 1) % n;
    const float ux = (float)vx[k], uy = (float)vy[k], wx = (float)vx[j], wy = (float)vy[j];
    const double dvy = (double)uy - wy, dvx = (double)ux - wx;
    const float z = dvy != 0 ? (float)(dvx / dvy) : 0.f;
    t.v[k] = make_float4(ux, uy, z, wx);
    t.w[k] = make_float4((float)((double)wx - (double)wy * z), uy, 0, 0);
  }
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = prop.multiProcessorCount * 2, threads = 256, reps = 400;
  const size_t nt = (size_t)blocks * threads;
  uint32_t* out; CK(cudaMalloc(&out, nt * 4 * 4));
  std::vector<uint32_t> h[4];
  auto run = [&](auto kern, int vi, const char* name) {
    for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(t, reps, out + vi * nt);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(t, reps, out + vi * nt);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double wpe = (double)nt / 32 * P * n * reps * 5;  // warp point-edges
    const double cyc = ms * 1e-3 * clk * 1e3 * prop.multiProcessorCount * 4;
    h[vi].resize(nt);
    CK(cudaMemcpy(h[vi].data(), out + vi * nt, nt * 4, cudaMemcpyDeviceToHost));
    printf("{\"variant\": \"%s\", \"n\": %d, \"ms\": %.3f, \"cycles_per_warp_point_edge\": %.3f}\n", name, n, ms, cyc / wpe);
  };
  run(probe<0>, 0, "V0 lop3");
  run(probe<1>, 1, "V1 fmul+lop3");
  run(probe<2>, 2, "V2 predicates");
  run(probe<3>, 3, "V3 paired anchoring");
  size_t bad1 = 0, bad2 = 0, bad3 = 0, ins = 0;
  for (size_t i = 0; i < nt; ++i) { bad1 += h[0][i] != h[1][i]; bad2 += h[0][i] != h[2][i]; bad3 += h[0][i] != h[3][i]; ins += __builtin_popcount(h[0][i]); }
  printf("{\"mismatch_v1\": %zu, \"mismatch_v2\": %zu, \"mismatch_v3\": %zu, \"inside_bits\": %zu}\n", bad1, bad2, bad3, ins);
  return 0;
}
