// K1 instantiations with the Gauss / 3M complex product (see
// cheb_step_kernel.cuh): three real DMMA.8x8x4 per complex 8x8x4 block
// instead of four. The first entry of a (bm, bn, groups) key is its default;
// `warps` selects the others (tuning).
#include "cheb_step_kernel.cuh"

namespace chfsi {
namespace k1 {

const Variant* variant_3m(int bm, int bn, int groups, int warps, bool conj) {
#define CHFSI_V(BM_, BN_, WM_, WN_, ST_, MB_, GR_)                                            \
  if (bm == BM_ && bn == BN_ && groups == GR_ && (warps == 0 || warps == WM_ * WN_)) {        \
    static const Variant a = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, false, GR_, true>();  \
    static const Variant b = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, true, GR_, true>();   \
    return conj ? &b : &a;                                                                    \
  }
  CHFSI_V(64, 16, 8, 1, 4, 2, 1)
  CHFSI_V(64, 16, 4, 1, 4, 2, 1)   // 4 warps of 16x16: more registers per warp
  CHFSI_V(64, 32, 4, 2, 4, 2, 1)
  CHFSI_V(64, 32, 2, 2, 4, 2, 1)   // 4 warps of 32x16
  CHFSI_V(128, 16, 8, 1, 6, 1, 1)
  CHFSI_V(128, 32, 4, 2, 5, 1, 1)  // 8 warps of 32x16, one CTA per SM
  CHFSI_V(128, 32, 8, 2, 5, 1, 1)
  CHFSI_V(64, 16, 8, 1, 10, 1, 2)
  CHFSI_V(64, 32, 4, 2, 8, 1, 2)
#undef CHFSI_V
  return nullptr;
}

// 32-complex-deep k-slabs (NH = 4): same shared memory as twice the stages
// of the 16-deep ones, half the slab boundaries (CHFSI_K1_NH=4 / chfsi_set_k1_slab)
const Variant* variant_3m_deep(int bm, int bn, int groups, int warps, bool conj) {
#define CHFSI_V(BM_, BN_, WM_, WN_, ST_, MB_, GR_)                                                \
  if (bm == BM_ && bn == BN_ && groups == GR_ && (warps == 0 || warps == WM_ * WN_)) {            \
    static const Variant a = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, false, GR_, true, 4>();   \
    static const Variant b = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, true, GR_, true, 4>();    \
    return conj ? &b : &a;                                                                        \
  }
  CHFSI_V(64, 16, 4, 1, 2, 2, 1)
  CHFSI_V(64, 32, 2, 2, 2, 2, 1)
  CHFSI_V(128, 32, 4, 2, 2, 1, 1)
#undef CHFSI_V
  return nullptr;
}

}  // namespace k1
}  // namespace chfsi
