// Issue-rate microbenchmark, part 2 (sm_100a): which instructions issue at
// full rate (1 warp-instruction / clk / SMSP) and which block dispatch for two
// cycles, for the crossing engine's formulation search.
// Each thread runs kChains independent chains; the kernel-argument operands
// are uniform registers unless the op says "3v" (three vector registers).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int kChains = 8;

template <int kOp>
__global__ void __launch_bounds__(256) pipe_kernel(float* out, int iters, float a, float b) {
  float v[kChains], w[kChains];
  unsigned u[kChains];
  double dv[kChains], dw[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    v[i] = out[threadIdx.x] + i;
    w[i] = v[i] * 0.5f + 1.f;
    u[i] = __float_as_uint(v[i]);
    dv[i] = v[i];
    dw[i] = w[i];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      const int j = (i + 1) % kChains, k = (i + 3) % kChains;
      if constexpr (kOp == 0) {  // FFMA, 3 vector registers
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(w[j]), "f"(w[k]));
      } else if constexpr (kOp == 1) {  // FFMA, 2 vector + uniform
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(w[j]), "f"(a));
      } else if constexpr (kOp == 2) {  // FMUL 2 vector
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(w[j]));
      } else if constexpr (kOp == 3) {  // FSETP + accumulate predicate (setp.and)
        asm volatile("{.reg .pred p; setp.lt.f32 p, %1, %2; @p add.f32 %0, %0, 0f3f800000;}" : "+f"(v[i]) : "f"(w[j]), "f"(w[k]));
      } else if constexpr (kOp == 4) {  // FMNMX 2-input
        asm volatile("max.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(w[j]));
      } else if constexpr (kOp == 5) {  // FSEL (selp.f32 on a predicate)
        asm volatile("{.reg .pred p; setp.lt.f32 p, %1, %2; selp.f32 %0, %1, %0, p;}" : "+f"(v[i]) : "f"(w[j]), "f"(w[k]));
      } else if constexpr (kOp == 6) {  // LOP3 3 vector
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(u[j]), "r"(u[k]));
      } else if constexpr (kOp == 7) {  // SHF (funnel shift)
        asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(u[i]) : "r"(u[j]));
      } else if constexpr (kOp == 8) {  // FADD.SAT 2 vector
        asm volatile("add.sat.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(w[j]));
      } else if constexpr (kOp == 9) {  // IMNMX
        asm volatile("max.s32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[j]));
      } else if constexpr (kOp == 10) {  // PRMT
        asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(u[i]) : "r"(u[j]));
      } else if constexpr (kOp == 12) {  // DADD
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(dv[i]) : "d"(dw[j]));
      } else if constexpr (kOp == 13) {  // DMUL
        asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(dv[i]) : "d"(dw[j]));
      } else if constexpr (kOp == 14) {  // DSETP + predicated integer add (the flag count)
        asm volatile("{.reg .pred p; setp.lt.f64 p, %1, %2; @p add.u32 %0, %0, 1;}" : "+r"(u[i]) : "d"(dv[j]), "d"(dw[k]));
      } else if constexpr (kOp == 15) {  // DSETP into a bool AND (the Voronoi accumulation)
        asm volatile("{.reg .pred p, q; setp.ne.u32 q, %0, 0; setp.le.and.f64 p, %1, %2, q; selp.u32 %0, 1, 0, p;}" : "+r"(u[i]) : "d"(dv[j]), "d"(dw[k]));
      } else if constexpr (kOp == 11) {  // FFMA 3v + FADD 2v, 1:1
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(w[j]), "f"(w[k]));
        asm volatile("add.f32 %0, %0, %1;" : "+f"(w[i]) : "f"(v[k]));
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc += v[i] + w[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int kOp>
int run(const char* name, int inst_per_iter_chain, int sms, int clk_mhz) {
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float* out;
  CK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  CK(cudaMemset(out, 0, sizeof(float) * blocks * threads));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) pipe_kernel<kOp><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) pipe_kernel<kOp><<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_inst = (double)blocks * (threads / 32) * iters * kChains * inst_per_iter_chain * reps;
  printf("{\"op\": \"%s\", \"warp_inst_per_s\": %.4e, \"warp_inst_per_clk_per_smsp\": %.3f}\n",
         name, warp_inst / (ms * 1e-3), warp_inst / (ms * 1e-3) / (clk_mhz * 1e6) / sms / 4);
  cudaFree(out);
  return 0;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount, mhz = clk / 1000;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"max_mhz\": %d}\n", prop.name, sms, mhz);
  run<0>("ffma_3v", 1, sms, mhz);
  run<1>("ffma_2v_ur", 1, sms, mhz);
  run<2>("fmul_2v", 1, sms, mhz);
  run<3>("fsetp+pred_fadd", 2, sms, mhz);
  run<4>("fmnmx2", 1, sms, mhz);
  run<5>("fsetp+fsel", 2, sms, mhz);
  run<6>("lop3_3v", 1, sms, mhz);
  run<7>("shf", 1, sms, mhz);
  run<8>("fadd_sat", 1, sms, mhz);
  run<9>("imnmx", 1, sms, mhz);
  run<10>("prmt", 1, sms, mhz);
  run<11>("ffma3v+fadd", 2, sms, mhz);
  run<12>("dadd", 1, sms, mhz);
  run<13>("dmul", 1, sms, mhz);
  run<14>("dsetp+pred_iadd", 2, sms, mhz);
  run<15>("dsetp.and+sel", 3, sms, mhz);
  return 0;
}
