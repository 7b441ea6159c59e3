#pragma once
#include "izg_common.cuh"

namespace izg {

template <int DELTA>
__device__ int32_t fastpfor_core(RingView& rv, uint64_t* full, uint64_t* empty, uint4 (*tot)[kCW],
                                 uint32_t& tbuf, uint32_t nw, uint32_t nblocks, uint32_t* out,
                                 bool out_aligned, uint4& carry, uint32_t* pos_out) {
  return IZG_E_FP_TRUNC_PAGE;
}

}  // namespace izg
