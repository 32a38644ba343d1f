// tri_small_hi.cu -- the small-polygon fused kernel's instantiations for
// 9..12 vertices (tri_small.cuh), compiled beside tri_small.cu.
#include "tri_small.cuh"

namespace vpipg {

namespace {

template <int MODE, int NC = 9>
SmallLaunch small_for(int nc, int k) {
  if constexpr (NC > kSmallMaxN) return nullptr;
  else return nc == NC ? small_for_k<NC, MODE>(k) : small_for<MODE, NC + 1>(nc, k);
}

}  // namespace

SmallLaunch small_launcher_hi(int nc, int k, int mode) {
  return mode == 1 ? small_for<1>(nc, k) : small_for<2>(nc, k);
}

}  // namespace vpipg
