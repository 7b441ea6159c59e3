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

}  // namespace izg

#ifdef IZG_CTA_PROF
extern "C" int izg_debug_cta_trace(void* host) {
  return cudaMemcpyFromSymbol(host, izg::g_cta_trace, sizeof(izg::g_cta_trace)) == cudaSuccess ? 0 : -1;
}
extern "C" int izg_debug_cta_prof(void* host, size_t bytes, int reset) {
  if (bytes > sizeof(izg::g_cta_prof)) bytes = sizeof(izg::g_cta_prof);
  if (cudaMemcpyFromSymbol(host, izg::g_cta_prof, bytes) != cudaSuccess) return -1;
  if (reset) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, izg::g_cta_prof) != cudaSuccess) return -1;
    cudaMemset(p, 0, sizeof(izg::g_cta_prof));
  }
  return 0;
}
#endif

namespace izg {
int cta_threads() { return kCtaWarps * 32; }

}  // namespace izg
