// tri_small.cu -- the small-polygon fused kernel's route: its plan, its entry
// points and the instantiations for 3..8 vertices (tri_small.cuh; 9..12 in
// tri_small_hi.cu).
#include "tri_small.cuh"

namespace vpipg {

namespace {

template <int MODE, int NC = 3>
SmallLaunch small_for(int nc, int k) {
  if constexpr (NC > 8) return nullptr;
  else return nc == NC ? small_for_k<NC, MODE>(k) : small_for<MODE, NC + 1>(nc, k);
}

// the small kernel's launcher for these tables and this batch, or null
SmallLaunch small_plan(const DevTables& t, const TestArgs* a) {
  const uint64_t kWarpPts = 32u * small_p((int)t.cross.n);
  if (!VPIPG_TRI_SMALL || !VPIPG_INLINE || !t.h_cross || !t.h_slab[0] || !t.h_slab[1] ||
      t.cross.n < 3 || t.cross.n > (uint32_t)kSmallMaxN)
    return nullptr;
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(a[0].xs) | reinterpret_cast<uintptr_t>(a[0].ys)) & 15) == 0;
  if (!aligned || a[0].m / kWarpPts < (uint64_t)kWarps) return nullptr;
  for (int e = 0; e < 3; ++e)
    if (a[e].bytes || (reinterpret_cast<uintptr_t>(a[e].words) & 15)) return nullptr;
  auto form = [](const SlabTable& s) { return s.cnt[kGroupXlo] == 0 ? 1 : s.cnt[kGroupYlo] == 0 ? 2 : 0; };
  const int mode = form(t.slab[0]);
  if (mode == 0 || form(t.slab[1]) != mode) return nullptr;
  const int glo = mode == 1 ? kGroupYlo : kGroupXlo;
  uint32_t k = small_kmin((int)t.cross.n);  // smaller groups are padded
  for (int e = 0; e < 2; ++e)
    for (int s = 0; s < 2; ++s) {
      const uint32_t c = t.slab[e].cnt[glo + s] / 2;
      if (c == 0) return nullptr;
      k = c > k ? c : k;
    }
  return t.cross.n <= 8 ? small_launcher_lo((int)t.cross.n, (int)k, mode)
                        : small_launcher_hi((int)t.cross.n, (int)k, mode);
}

}  // namespace

SmallLaunch small_launcher_lo(int nc, int k, int mode) {
  return mode == 1 ? small_for<1>(nc, k) : small_for<2>(nc, k);
}

bool test_f32_small_plan(const DevTables& t, const TestArgs* a) { return small_plan(t, a) != nullptr; }

cudaError_t launch_test_f32_small(const DevTables& t, const TestArgs* a, cudaStream_t stream) {
  const SmallLaunch launch = small_plan(t, a);
  return launch ? launch(t, a, stream) : cudaErrorNotSupported;
}

}  // namespace vpipg
