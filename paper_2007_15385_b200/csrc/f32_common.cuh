// f32_common.cuh -- device helpers shared by the fp32 streaming kernels
// (test_f32.cu: per-engine and fused kernels; tri_small.cu: the small-polygon
// fused kernel): the CTA shape, the NaN-propagating three-input max / min,
// the crossing bit, the ballot vote with its predicated count, the count
// flush, the persistent slice schedule and the L2 prefetch.
#pragma once

#include <cstdint>
#include <type_traits>

#include "vpipg_internal.h"

#define VPIPG_PRAGMA(x) _Pragma(#x)
#define VPIPG_UNROLL(n) VPIPG_PRAGMA(unroll n)

#ifndef VPIPG_INLINE
#define VPIPG_INLINE 1
#endif

namespace vpipg {

namespace {

constexpr int kWarps = 8;             // warps per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kGroupXlo = 0, kGroupYlo = 2;  // slab group order (vpipg_device.cuh)

// NaN-propagating three-input max / min (FMNMX3 .NAN, same issue cost): a
// point with a NaN coordinate turns every bound of its sections into NaN, so
// the final compare sees NaN and the engine's NaN rule decides (SlabEngine)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// ---------------------------------------------------------------------------
// Crossing engine (engines.cpp:165-204). For edge w = v[k-1] -> u = v[k]:
//   in_range <=> (u.y > qy) != (w.y > qy) <=> sign(h_k) ^ sign(h_{k-1}),
//                h = qy - v.y (a -0.0 from qy = -0.0 merely moves vertex k to
//                "above" for both of its edges at once, which keeps the parity)
//   on_left  <=> qx < x-of-edge-at-qy <=> d = (a.x - qx) + (qy - a.y) * dvx/dvy > 0
//                for either endpoint a of the edge
// crossing bit = (H_k ^ H_{k-1}) & ~D (one LOP3), XOR-reduced into the parity
// word's bit 31 two bits per LOP3.
//
// Paired anchoring: edges k (v[k-1] -> v[k]) and k+1 (v[k] -> v[k+1]) both
// take their x-intercept from their shared vertex v[k], so g = v[k].x - qx is
// formed for every other vertex only and h_k serves both d's: per edge
// 1 FADD (h) + 1/2 FADD (g) + 1 FFMA (d) + 3/2 LOP3, 5.5 dispatch cycles
// against 6 for one g per vertex (B200, profiles/crossing_forms_r02.json:
// C5 crossing 12.18 -> 11.20 ms at P = 12). The per-edge constants come from
// the parameter bank as uniform registers (VPIPG_INLINE), so the FFMA has two
// vector sources: with three (table in shared memory) it issues at 0.61 per
// cycle instead of 0.96 (tools/pipe_peaks2.cu).
// Points exactly on an edge line lie inside the 1e-5 parity band, so the
// reference's closed-boundary latch (engines.cpp:194-196) is repeated only by
// the exact f64 kernel.
__device__ __forceinline__ uint32_t cross_bit(float h, float hprev, float d) {
  return (__float_as_uint(h) ^ __float_as_uint(hprev)) & ~__float_as_uint(d);
}
// ---------------------------------------------------------------------------
// Output: ballot words (PIPM order), optional byte mask, per-lane inside count.
// The P words of a slice are warp-uniform; lane 0 writes them with 16-byte
// streaming stores (a slice's words are 64 contiguous, 64-byte aligned bytes).
// kVote 0: inside = (a >= b); 1: (a >= b or unordered), the NaN-inside rule;
// 2: a's bit pattern is negative as an int (the crossing parity word, no
// float conversion). One compare feeds both the ballot and a predicated count.
// Per-lane inside counts: integer-valued floats (VPIPG_FCOUNT, the predicated
// FADD issues at full rate on the FMA pipe) or u32; exact either way below
// 2^24 points per lane (2^24 x 75,776 resident lanes per launch).
#ifndef VPIPG_FCOUNT
#define VPIPG_FCOUNT 1
#endif
using cnt_t = std::conditional_t<VPIPG_FCOUNT != 0, float, uint32_t>;
#if VPIPG_FCOUNT
#define VPIPG_CNT_ADD "@q add.f32 %1, %1, 0f3F800000;\n\t}"
#define VPIPG_CNT_C "+f"
#else
#define VPIPG_CNT_ADD "@q add.u32 %1, %1, 1;\n\t}"
#define VPIPG_CNT_C "+r"
#endif
template <int kVote>
__device__ __forceinline__ uint32_t vote_in(float a, float b, cnt_t& cnt) {
  uint32_t w;
  if (kVote == 2)
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.lt.s32 q, %2, 0;\n\t"
        "vote.sync.ballot.b32 %0, q, 0xffffffff;\n\t"
        VPIPG_CNT_ADD
        : "=r"(w), VPIPG_CNT_C(cnt)
        : "r"(__float_as_uint(a)));
  else if (kVote == 1)
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.geu.f32 q, %2, %3;\n\t"
        "vote.sync.ballot.b32 %0, q, 0xffffffff;\n\t"
        VPIPG_CNT_ADD
        : "=r"(w), VPIPG_CNT_C(cnt)
        : "f"(a), "f"(b));
  else
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ge.f32 q, %2, %3;\n\t"
        "vote.sync.ballot.b32 %0, q, 0xffffffff;\n\t"
        VPIPG_CNT_ADD
        : "=r"(w), VPIPG_CNT_C(cnt)
        : "f"(a), "f"(b));
  return w;
}

__device__ __forceinline__ void flush_count(cnt_t fcnt, const TestArgs& a) {
  uint32_t cnt = static_cast<uint32_t>(fcnt);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
  if ((threadIdx.x & 31) == 0 && a.inside && cnt) atomicAdd(a.inside, (unsigned long long)cnt);
}

// Persistent slice schedule: warp w of CTA b takes slices (b + r * grid) *
// kWarps + w for rounds r = 0 .. rounds - 1. `rounds` depends on the CTA
// only, so every loop over it is uniform control flow for the compiler (the
// per-edge table reads can then use the uniform datapath); a warp whose slot
// in the last round lies past the end re-reads the last full slice and stores
// nothing (emit's `live`).
struct SliceRounds {
  uint64_t W, b0, g0, rounds, last;
  __device__ SliceRounds(uint64_t full_slices, int warp) {
    W = (uint64_t)gridDim.x * kWarps;
    b0 = (uint64_t)blockIdx.x * kWarps;
    g0 = b0 + warp;
    rounds = full_slices > b0 ? (full_slices - b0 + W - 1) / W : 0;
    last = full_slices ? full_slices - 1 : 0;
  }
  __device__ uint64_t slice(uint64_t r) const {
    const uint64_t g = g0 + r * W;
    return g < last ? g : last;
  }
  __device__ bool live(uint64_t r) const { return g0 + r * W <= last; }
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}


}  // namespace

// a crossing record (u.x, u.y, dvx/dvy, w.x) from the local frame of the
// device tables to the absolute frame of the parameter-bank launches (test_f32.cu)
float4 cross_record_abs(const float4& r, float ox, float oy);

}  // namespace vpipg
