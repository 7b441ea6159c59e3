// decode_cta.cu — instantiations of the CTA-cooperative SIMD-BP128 kernel
// of cta.cuh (one CTA per SM, shared staging ring, units of 1,024 integers
// round robin over 16 consumer warps, mailbox carry), array modes only.
#include "cta.cuh"

namespace izg {

using GroupFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                         uint32_t*, uint32_t*, const CUtensorMap, int);

GroupFn pick_cta(int delta) {
  switch (delta) {
    case IZG_DELTA_D1: return cta_kernel<IZG_DELTA_D1>;
    case IZG_DELTA_D4: return cta_kernel<IZG_DELTA_D4>;
    case IZG_DELTA_D2: return cta_kernel<IZG_DELTA_D2>;
    case IZG_DELTA_DM: return cta_kernel<IZG_DELTA_DM>;
  }
  return nullptr;
}

size_t cta_smem_bytes() { return CtaLayout::kSmem; }
int cta_threads() { return kCtaWarps * 32; }

}  // namespace izg
