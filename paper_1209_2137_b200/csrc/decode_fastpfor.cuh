#pragma once
#include "izg_common.cuh"

namespace izg {

template <int DELTA>
__device__ int32_t fastpfor_core(WarpRing& r, OutStage& os, const uint32_t* page, uint32_t nw,
                                 uint32_t nblocks, uint32_t* out, bool out_aligned, int64_t orow,
                                 uint4& carry, uint32_t* pos_out) {
  return IZG_E_FP_TRUNC_PAGE;
}

}  // namespace izg
