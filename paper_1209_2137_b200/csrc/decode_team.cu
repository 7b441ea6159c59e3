// decode_team.cu — instantiations of the team SIMD-FastPFOR decode of
// team.cuh (one CTA of 8 warps per page, shared TMA staging, windowed bulk
// unpack of the exception arrays, two-level prefix sum).
#include "team.cuh"

namespace izg {

using TeamFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                        uint32_t*, uint32_t*, const CUtensorMap, int, IdxView);

TeamFn pick_team(int delta) {
  switch (delta) {
    case IZG_DELTA_NONE: return fp_team_kernel<IZG_DELTA_NONE>;
    case IZG_DELTA_D1: return fp_team_kernel<IZG_DELTA_D1>;
    case IZG_DELTA_D4: return fp_team_kernel<IZG_DELTA_D4>;
    case IZG_DELTA_D2: return fp_team_kernel<IZG_DELTA_D2>;
    case IZG_DELTA_DM: return fp_team_kernel<IZG_DELTA_DM>;
  }
  return nullptr;
}

size_t team_smem_bytes() { return TeamLayout::kSmem; }
int team_threads() { return kTeamThreads; }

}  // namespace izg

#ifdef IZG_TEAM_PROF
extern "C" int izg_debug_team_prof(void* host, int reset) {
  if (cudaMemcpyFromSymbol(host, izg::g_team_prof, sizeof(izg::g_team_prof)) != cudaSuccess) return -1;
  if (reset) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, izg::g_team_prof) != cudaSuccess) return -1;
    cudaMemset(p, 0, sizeof(izg::g_team_prof));
  }
  return 0;
}
#endif

#ifdef IZG_BOUNDS
// {violations, kind of the first, its chunk, its offset}; reset != 0 clears the counters.
extern "C" int izg_debug_bounds(void* host, int reset) {
  if (cudaMemcpyFromSymbol(host, izg::g_izg_oob, sizeof(izg::g_izg_oob)) != cudaSuccess) return -1;
  if (reset) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, izg::g_izg_oob) != cudaSuccess) return -1;
    cudaMemset(p, 0, sizeof(izg::g_izg_oob));
  }
  return 0;
}
#endif
