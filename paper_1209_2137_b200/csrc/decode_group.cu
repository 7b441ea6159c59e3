// decode_group.cu — instantiations of the SIMD-BP128 group kernels of
// group.cuh (KW warps per chunk, iterations round robin, mailbox carry).
#include "group.cuh"

namespace izg {

using GroupFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                         uint32_t*, uint32_t*, const CUtensorMap, int);

template <int KW>
GroupFn pick_group_kw(int delta) {
  switch (delta) {
    case IZG_DELTA_NONE: return group_kernel<IZG_DELTA_NONE, KW>;
    case IZG_DELTA_D1: return group_kernel<IZG_DELTA_D1, KW>;
    case IZG_DELTA_D4: return group_kernel<IZG_DELTA_D4, KW>;
    case IZG_DELTA_D2: return group_kernel<IZG_DELTA_D2, KW>;
    case IZG_DELTA_DM: return group_kernel<IZG_DELTA_DM, KW>;
  }
  return nullptr;
}

GroupFn pick_group(int kw, int delta) {
  switch (kw) {
    case 2: return pick_group_kw<2>(delta);
    case 4: return pick_group_kw<4>(delta);
    case 8: return pick_group_kw<8>(delta);
  }
  return nullptr;
}

}  // namespace izg
