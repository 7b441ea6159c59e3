// decode_scalar.cu — the scalar-array FastPFOR decode kernels
// (codec_patched.cpp:292-417, PatchStorage::scalar_arrays), in their own
// translation unit so build.py can compile them with ptxas -O1.
//
// Why: built at ptxas -O2/-O3 (this library's default), these kernels faulted
// with "misaligned address" / "illegal memory access" on pages with
// exceptions — deterministically, e.g. any single 128-integer page with one
// exception at b = 3 (tests/test_collisions.py reproduces it) — while the same
// source at -O0/-O1, or with any change to the exception loop (a printf, no
// inlining, dropping either its loads or its shared-memory ORs), decoded
// exactly.  Every address the loop forms was checked in range and aligned in
// an instrumented build, and the vertical-array instantiation of the same
// code (SIMD-FastPFOR) is unaffected.  Without a faulting PC in this sandbox
// (no compute-sanitizer, no core dumps) the cause is not pinned down;
// DESIGN.md §9 records it.
#include "decode_kernel.cuh"

namespace izg {

KernelFn pick_fastpfor_scalar(int delta) { return pick<IZG_FASTPFOR, false>(delta); }
KernelFn pick_probe_fastpfor_scalar(int delta) { return pick_probe<IZG_FASTPFOR>(delta); }

}  // namespace izg
