// decode_relay.cu — instantiations of the SIMD-BP128 relay kernel of
// relay.cuh (segments of a chunk claimed level by level, state handed on in
// order; batches of a few waves of warp slots).
#include "relay.cuh"

namespace izg {

RelayFn pick_relay(int delta) {
  switch (delta) {
    case IZG_DELTA_NONE: return relay_kernel<IZG_DELTA_NONE>;
    case IZG_DELTA_D1: return relay_kernel<IZG_DELTA_D1>;
    case IZG_DELTA_D4: return relay_kernel<IZG_DELTA_D4>;
    case IZG_DELTA_D2: return relay_kernel<IZG_DELTA_D2>;
    case IZG_DELTA_DM: return relay_kernel<IZG_DELTA_DM>;
  }
  return nullptr;
}

}  // namespace izg
