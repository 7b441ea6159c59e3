// decode_split.cu — instantiations of the split (several warps per chunk,
// decoupled look-back) decode kernels of split.cuh.
#include "split.cuh"

namespace izg {

using SplitFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                         uint32_t*, SplitArgs, IdxView);

template <int CODEC>
SplitFn pick_split_codec(int delta) {
  switch (delta) {
    case IZG_DELTA_NONE: return split_kernel<CODEC, IZG_DELTA_NONE>;
    case IZG_DELTA_D1: return split_kernel<CODEC, IZG_DELTA_D1>;
    case IZG_DELTA_D4: return split_kernel<CODEC, IZG_DELTA_D4>;
    case IZG_DELTA_D2: return split_kernel<CODEC, IZG_DELTA_D2>;
    case IZG_DELTA_DM: return split_kernel<CODEC, IZG_DELTA_DM>;
  }
  return nullptr;
}

SplitFn pick_split(int codec, int delta) {
  if (codec == IZG_SIMDBP128) return pick_split_codec<IZG_SIMDBP128>(delta);
  if (codec == IZG_SIMDFASTPFOR) return pick_split_codec<IZG_SIMDFASTPFOR>(delta);
  return nullptr;
}

}  // namespace izg
