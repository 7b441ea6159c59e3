// decode_probe.cu — instantiations of the probe-sink decode kernels
// (decode -> intersect, probe.cuh), kept out of decode.cu so the two
// translation units compile in parallel.  Scalar-array FastPFOR lives in
// decode_scalar.cu with the rest of that codec's kernels.
#include "decode_kernel.cuh"

namespace izg {

KernelFn pick_probe_fastpfor_scalar(int delta);

KernelFn pick_probe_kernel(int codec, int delta) {
  switch (codec) {
    case IZG_SIMDBP128: return pick_probe<IZG_SIMDBP128>(delta);
    case IZG_SIMDFASTPFOR: return pick_probe<IZG_SIMDFASTPFOR>(delta);
    case IZG_BP32: return pick_probe<IZG_BP32>(delta);
    case IZG_FASTPFOR: return pick_probe_fastpfor_scalar(delta);
    case IZG_SIMPLEPFOR: return pick_probe<IZG_SIMPLEPFOR>(delta);
  }
  return nullptr;
}

}  // namespace izg
