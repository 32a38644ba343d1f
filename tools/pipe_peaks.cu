// Pipe-throughput microbenchmark for the roofline denominators of the point
// tests (FFMA / FFMA2 / DFMA / LOP3 / FMNMX3 issue rates on sm_100a).
// Each thread runs kChains independent dependency chains so the pipes, not
// latency, bound the loop. Reports warp-instructions and lane-ops per second
// and the SM clock seen by the kernel (clock64 delta / globaltimer delta).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int kChains = 8;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

template <int kOp>
__global__ void __launch_bounds__(256) pipe_kernel(float* out, int iters, float a, float b,
                                                    unsigned long long* clk) {
  uint64_t c0 = clock64();
  uint64_t t0 = gtimer();
  float v[kChains];
  uint64_t p[kChains];
  double d[kChains];
  unsigned u[kChains];
  float w[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    v[i] = out[threadIdx.x] + i;
    p[i] = (uint64_t)__float_as_uint(v[i]) | ((uint64_t)__float_as_uint(v[i] + 1.f) << 32);
    d[i] = v[i];
    u[i] = __float_as_uint(v[i]);
    w[i] = v[i] * 0.5f;
  }
  uint64_t ab = (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(a) << 32);
  uint64_t bb = (uint64_t)__float_as_uint(b) | ((uint64_t)__float_as_uint(b) << 32);
  double da = a, db = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      if constexpr (kOp == 0) {  // FFMA, register operands
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 1) % kChains]), "f"(b));
      } else if constexpr (kOp == 1) {  // FFMA, uniform operands
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
      } else if constexpr (kOp == 2) {  // FFMA2 packed pair
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(ab), "l"(bb));
      } else if constexpr (kOp == 3) {  // DFMA
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(da), "d"(db));
      } else if constexpr (kOp == 4) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(u[(i + 1) % kChains]), "r"(u[(i + 3) % kChains]));
      } else if constexpr (kOp == 5) {  // FMNMX3
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 1) % kChains]), "f"(v[(i + 2) % kChains]));
      } else if constexpr (kOp == 6) {  // 2x FFMA2 + 1 LOP3 (the affine half-plane inner loop)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(ab), "l"(bb));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[(i + 4) % kChains]) : "l"(ab), "l"(bb));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xfe;" : "+r"(u[i]) : "r"((unsigned)p[i]), "r"((unsigned)(p[i] >> 32)));

      } else if constexpr (kOp == 7) {  // 4 FFMA + 1 LOP3 (two edges, scalar FFMA)
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 1) % kChains]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 2) % kChains]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 3) % kChains]) : "f"(a), "f"(b));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xfe;" : "+r"(u[i]) : "r"(__float_as_uint(v[i])), "r"(__float_as_uint(v[(i + 1) % kChains])));
      } else if constexpr (kOp == 8) {  // 4 FFMA + 1 FMNMX3
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 1) % kChains]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 2) % kChains]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 3) % kChains]) : "f"(a), "f"(b));
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(w[i]) : "f"(v[i]), "f"(v[(i + 1) % kChains]));
      } else if constexpr (kOp == 9) {  // FADD
        asm volatile("add.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(v[(i + 1) % kChains]));
      } else if constexpr (kOp == 10) {  // IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[i]) : "r"(u[(i + 1) % kChains]), "r"(u[(i + 2) % kChains]));
      } else if constexpr (kOp == 11) {  // IADD3
        asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) % kChains]));
      } else if constexpr (kOp == 12) {  // 2 FFMA + 1 LOP3
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 1) % kChains]) : "f"(a), "f"(b));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xfe;" : "+r"(u[i]) : "r"(__float_as_uint(v[i])), "r"(__float_as_uint(v[(i + 1) % kChains])));
      } else if constexpr (kOp == 13) {  // FFMA.SAT
        asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
      } else if constexpr (kOp == 14) {  // 4 FFMA + 2 FADD + 3 LOP3 (crossing, two edges)
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 1) % kChains]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 2) % kChains]) : "f"(a), "f"(b));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[(i + 3) % kChains]) : "f"(a), "f"(b));
        asm volatile("add.f32 %0, %0, %1;" : "+f"(w[i]) : "f"(a));
        asm volatile("add.f32 %0, %0, %1;" : "+f"(w[(i + 1) % kChains]) : "f"(a));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(__float_as_uint(v[i])), "r"(__float_as_uint(w[i])));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[(i + 1) % kChains]) : "r"(__float_as_uint(v[(i + 1) % kChains])), "r"(__float_as_uint(w[(i + 1) % kChains])));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(u[(i + 1) % kChains]), "r"(__float_as_uint(v[(i + 2) % kChains])));
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i)
    acc += v[i] + __uint_as_float((unsigned)p[i]) + (float)d[i] + __uint_as_float(u[i]) + w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    clk[0] = clock64() - c0;
    clk[1] = gtimer() - t0;
  }
}

template <int kOp>
int run(const char* name, int inst_per_iter_chain, int lanes_per_inst, int sms) {
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float* out; unsigned long long* clk;
  CK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  CK(cudaMemset(out, 0, sizeof(float) * blocks * threads));
  CK(cudaMalloc(&clk, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) pipe_kernel<kOp><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f, clk);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) pipe_kernel<kOp><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f, clk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2]; CK(cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost));
  double warp_inst = (double)blocks * (threads / 32) * iters * kChains * inst_per_iter_chain * reps;
  double s = ms * 1e-3;
  double mhz = (double)h[0] / (double)h[1] * 1e3;
  printf("{\"op\": \"%s\", \"warp_inst_per_s\": %.4e, \"lane_ops_per_s\": %.4e, "
         "\"warp_inst_per_clk_per_sm\": %.3f, \"sm_mhz_seen\": %.0f}\n",
         name, warp_inst / s, warp_inst * 32 * lanes_per_inst / s,
         warp_inst / s / (mhz * 1e6) / sms, mhz);
  cudaFree(out); cudaFree(clk);
  return 0;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", prop.name, prop.multiProcessorCount,
         prop.major, prop.minor);
  const int sms = prop.multiProcessorCount;
  run<0>("ffma_reg", 1, 1, sms);
  run<1>("ffma_uniform", 1, 1, sms);
  run<2>("ffma2", 1, 2, sms);
  run<3>("dfma", 1, 1, sms);
  run<4>("lop3", 1, 1, sms);
  run<5>("fmnmx3", 1, 1, sms);
  run<6>("2xffma2+lop3", 3, 1, sms);
  run<7>("4xffma+lop3", 5, 1, sms);
  run<8>("4xffma+fmnmx3", 5, 1, sms);
  run<9>("fadd", 1, 1, sms);
  run<10>("imad", 1, 1, sms);
  run<11>("iadd", 1, 1, sms);
  run<12>("2xffma+lop3", 3, 1, sms);
  run<13>("ffma_sat", 1, 1, sms);
  run<14>("4xffma+2xfadd+3xlop3", 9, 1, sms);
  return 0;
}
