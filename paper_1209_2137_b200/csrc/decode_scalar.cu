// decode_scalar.cu — the scalar-array FastPFOR decode kernels
// (codec_patched.cpp:292-417, PatchStorage::scalar_arrays), in their own
// translation unit.
//
// History: in round 1 these kernels, built at ptxas -O2/-O3,
// faulted ("misaligned address" / "illegal memory access") on pages with
// exceptions — deterministically, e.g. any single 128-integer page with one
// exception at b = 3 (tools/repro_scalar_fault.py) — while -O0/-O1 or any
// change to the exception loop decoded exactly; this file was built at
// -Xptxas -O1.  Round 2 replaced the patch loop by the lean one
// (decode_fastpfor.cuh: fp_patch_lean — every address from a valid base,
// no address selects), and at -O3 the repro, tests/test_collisions.py and
// tests/test_gpu_f3.py pass; the special build flag is gone.  The fault's
// root cause was never pinned down (the pool refuses compute-sanitizer and
// GPU core dumps).
#include "decode_kernel.cuh"

namespace izg {

KernelFn pick_fastpfor_scalar(int delta) { return pick<IZG_FASTPFOR, false>(delta); }
KernelFn pick_probe_fastpfor_scalar(int delta) { return pick_probe<IZG_FASTPFOR>(delta); }

}  // namespace izg
