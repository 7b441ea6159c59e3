// decode_kernel.cuh — the persistent decode kernel template, shared by the
// translation units that instantiate it (decode.cu, decode_scalar.cu).
//
// Kernel shape: persistent CTAs of kWarps independent warps.
// Each warp claims whole chunks, streams the chunk's compressed payload into
// its private shared-memory ring with TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx), decodes straight out of the ring with the prefix sum
// fused, and writes every decoded integer to HBM exactly once.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/intzip_b200.h"
#include "decode_bp128.cuh"
#include "decode_fastpfor.cuh"
#include "index_fastpfor.cuh"
#include "izg_common.cuh"
#include "probe.cuh"

namespace izg {

// Per-chunk argument checks applied before touching the payload:
// decode_array's length check (codec.cpp:43-44) or decode_deltas' count
// checks (codec_binpack.cpp:12-15, codec_patched.cpp:52-57).
__device__ __forceinline__ int32_t precheck(int codec, bool array_mode, uint32_t n) {
  if (array_mode) {
    if (n == 0 || n > IZG_CHUNK_SIZE) return IZG_E_CHUNK_LENGTH;
  } else {
    if (n % 128) return IZG_E_COUNT_MULTIPLE;
    if (codec != IZG_SIMDBP128 && codec != IZG_BP32 && n > IZG_CHUNK_SIZE)
      return IZG_E_PAGE_TOO_LARGE;
  }
  return IZG_OK;
}

// Persistent kernel: every warp repeatedly claims the next chunk (one atomic
// per chunk) and decodes it end to end: stream, unpack, patch, prefix sum,
// VByte remainder, consumption check, status.  IDX (SIMD-FastPFOR only):
// pages were indexed by fp_index_kernel into `ix`.  OS is the output sink:
// OutStage writes the decoded integers to `out`; ProbeStage (probe.cuh)
// intersects them with `pa.s` instead and `out` is unused.
template <int CODEC, int DELTA, bool IDX, typename OS = OutStage, int SHAPE = 0>
__global__ void __launch_bounds__((Layout<CODEC, IDX, SHAPE>::kWarps * 32))
    __maxnreg__((Layout<CODEC, IDX, SHAPE>::kMaxRegs))
    decode_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                  uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                  uint32_t* __restrict__ consumed, uint32_t* __restrict__ next_chunk,
                  const __grid_constant__ CUtensorMap omap, int tma_out, IdxView ix,
                  ProbeArgs pa) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using LY = Layout<CODEC, IDX, SHAPE>;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpRing r;
  r.base = smem_u32(smem + warp * kRingBytes);
  r.bar = smem_u32(smem + LY::kBarOff) + warp * kNS * 8u;
  FpScratch* fsc = reinterpret_cast<FpScratch*>(smem + LY::kTabOff + warp * LY::kTabBytes);
  OS os;
  os.base = smem_u32(smem + LY::kOutOff + warp * LY::kTiles * kStageOut);
  os.leader = lane == 0;
  if constexpr (OS::kProbe) {
    os.pa = pa;
  } else {
    os.buf = 0;
    os.tmap = &omap;
  }
  r.g = 0;
  r.leader = lane == 0;
  r.policy = policy_evict_first();
  if (lane == 0) {
    for (uint32_t i = 0; i < kNS; ++i) mbar_init_s(r.bar + 8u * i, 1);
    fence_barrier_init();
  }
  __syncwarp();

  for (;;) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 1u);
    c = __shfl_sync(0xFFFFFFFFu, c, 0);
    if (c >= n_chunks) break;
    const izg_chunk ch = chunks[c];
    int32_t st = precheck(CODEC, kArray, ch.n);
    uint32_t pos = 0;
    os.begin_chunk();
    if (st == IZG_OK) {
      const uint32_t* p = words + ch.word_off;
      // probe sink: no output; every full iteration takes the put/commit path
      uint32_t* o = OS::kProbe ? nullptr : out + ch.out_off;
      const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
      const int64_t orow = OS::kProbe                                ? 0
                           : tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5)
                                                                   : -1;
      const uint32_t core = kArray ? ch.n / 128 * 128 : ch.n;
      uint4 carry = make_uint4(0, 0, 0, 0);
      constexpr int ST = CODEC == IZG_SIMDFASTPFOR ? kVertical
                         : CODEC == IZG_FASTPFOR ? kScalar
                                                 : kSimple8b;
      if (CODEC == IZG_SIMDBP128) {
        r.begin(p, ch.n_words);
        if (r.phase == 0)
          st = bp128_core<DELTA, true>(r, os, ch.n_words, core / 128, o, oal, orow, carry, &pos);
        else
          st = bp128_core<DELTA, false>(r, os, ch.n_words, core / 128, o, oal, orow, carry,
                                        &pos);
        r.end();
      } else if (CODEC == IZG_BP32) {
        r.begin(p, ch.n_words);
        st = bp32_core<DELTA>(r, os, ch.n_words, core / 128, o, oal, orow, carry, &pos);
        r.end();
      } else if (IDX) {
        st = fastpfor_core_idx<DELTA, ST>(r, os, reinterpret_cast<uint32_t*>(fsc), p, c,
                                          core / 128, ix, o, oal, orow, carry, &pos);
      } else {
        st = fastpfor_core<DELTA, ST>(r, os, *fsc, p, ch.n_words, core / 128, o, oal, orow,
                                      carry, &pos);
      }
      if (kArray && st == IZG_OK) {
        if (core < ch.n) {
          // Variable Byte remainder (codec.cpp:56-62).
          uint32_t rb = 0;
          const uint32_t cnt = ch.n - core;
          // probe sink: the tail goes to the warp's (now idle) tile,
          // linear, then through the probe like any short iteration
          // (vbyte_tail writes out[core + i], hence the offset base)
          uint32_t* tail = nullptr;
          if constexpr (OS::kProbe)
            tail = reinterpret_cast<uint32_t*>(smem + LY::kOutOff +
                                               warp * LY::kTiles * kStageOut);
          if (lane == 0)
            st = vbyte_tail<DELTA>(reinterpret_cast<const uint8_t*>(p + pos),
                                   4u * (ch.n_words - pos), core, cnt, carry,
                                   OS::kProbe ? tail - core : o, &rb);
          st = __shfl_sync(0xFFFFFFFFu, st, 0);
          rb = __shfl_sync(0xFFFFFFFFu, rb, 0);
          if (st == IZG_OK) pos += (rb + 3) / 4;
          if constexpr (OS::kProbe) {
            if (st == IZG_OK) {
              __syncwarp();
              uint32_t v[4][4];
#pragma unroll
              for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint32_t i = 16u * lane + 4u * k + j;
                  v[k][j] = i < cnt ? tail[i] : 0u;
                }
              os.direct(v, nullptr, false, true, cnt, lane);
            }
          }
        }
        if (st == IZG_OK && pos != ch.n_words) st = IZG_E_PAYLOAD_SIZE;  // codec.cpp:63-64
      }
    }
    if (lane == 0) {
      status[c] = st;
      if (consumed) consumed[c] = st == IZG_OK ? pos : 0;
    }
  }
  os.drain();
}

using KernelFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                          uint32_t*, uint32_t*, const CUtensorMap, int, IdxView, ProbeArgs);

template <int CODEC, bool IDX, int SHAPE = 0>
KernelFn pick(int delta) {
  using OS = OutStageT<Layout<CODEC, IDX, SHAPE>::kTiles>;
  switch (delta) {
    case IZG_DELTA_NONE: return decode_kernel<CODEC, IZG_DELTA_NONE, IDX, OS, SHAPE>;
    case IZG_DELTA_D1: return decode_kernel<CODEC, IZG_DELTA_D1, IDX, OS, SHAPE>;
    case IZG_DELTA_D4: return decode_kernel<CODEC, IZG_DELTA_D4, IDX, OS, SHAPE>;
    case IZG_DELTA_D2: return decode_kernel<CODEC, IZG_DELTA_D2, IDX, OS, SHAPE>;
    case IZG_DELTA_DM: return decode_kernel<CODEC, IZG_DELTA_DM, IDX, OS, SHAPE>;
  }
  return nullptr;
}

}  // namespace izg

namespace izg {

// Probe-sink kernels (decode -> intersect), array modes D1 / D4 only.
template <int CODEC>
KernelFn pick_probe(int delta) {
  switch (delta) {
    case IZG_DELTA_D1: return decode_kernel<CODEC, IZG_DELTA_D1, false, ProbeStage>;
    case IZG_DELTA_D4: return decode_kernel<CODEC, IZG_DELTA_D4, false, ProbeStage>;
  }
  return nullptr;
}

}  // namespace izg
