// encode.cuh — GPU encoder (secondary path).
//
// Restates, fused per chunk:
//   encode_array's chunk body       codec.cpp:21-35 (delta, core, VByte tail)
//   delta_encode_scalar / _stride4  delta.cpp:18-23, 53-58 (+ D2/DM extensions)
//   SimdBp128Codec::encode_deltas   codec_binpack.cpp:70-92
//   max_bitwidth / pack_vertical128 bitpack.cpp:287-291, 87-120
//   vbyte_encode                    codec_basic.cpp:16-25
// Output words are bit-identical to the reference encoder's
// (tests/test_gpu_encode.py compares them word for word).
//
// One warp encodes one chunk, four blocks per iteration in the same register
// layout as the decoder (lane 8q+s8 holds 16 consecutive integers of block
// q).  A block's width is an 8-lane OR reduction; its packed rows are built
// with shared-memory OR reductions in a per-warp tile and copied out
// coalesced.  A meta-block's 16-byte descriptor precedes its payloads but
// only earlier widths determine a block's offset, so the descriptor is
// written after the meta-block's last block.
#pragma once
#include <cstdint>

#include "../../include/intzip_b200.h"
#include "izg_ptx.cuh"

namespace izg {

constexpr int kEncWarps = 8;

__device__ __forceinline__ uint32_t bitw(uint32_t v) { return 32u - __clz(v); }

template <int DELTA, bool WRAP>
__global__ void __launch_bounds__(kEncWarps * 32)
    bp128_encode_kernel(const uint32_t* __restrict__ values, izg_chunk* __restrict__ chunks,
                        uint32_t n_chunks, uint32_t* __restrict__ words,
                        int32_t* __restrict__ status, uint32_t* __restrict__ next_chunk) {
  __shared__ uint32_t tiles[kEncWarps][512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  uint32_t* tile = tiles[warp];
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  for (;;) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 1u);
    c = __shfl_sync(0xFFFFFFFFu, c, 0);
    if (c >= n_chunks) break;
    const izg_chunk ch = chunks[c];
    const uint32_t n = ch.n;
    int32_t st = IZG_OK;
    if (kArray && (n == 0 || n > IZG_CHUNK_SIZE)) st = IZG_E_CHUNK_LENGTH;
    if (!kArray && n % 128 != 0) st = IZG_E_COUNT_MULTIPLE;
    uint32_t pos = 0;
    if (st == IZG_OK) {
      const uint32_t* x = values + ch.out_off;
      uint32_t* o = words + ch.word_off;
      const bool xal = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
      const uint32_t core = kArray ? n / 128 * 128 : n;
      const uint32_t nb = core / 128;
      bool bad = false;
      uint4 carry = make_uint4(0, 0, 0, 0);  // last slot of the previous iteration
      for (uint32_t mb0 = 0; mb0 < nb; mb0 += 16) {
        const uint32_t G = min(16u, nb - mb0);
        const uint32_t desc = pos;
        pos += 4;
        uint32_t wdesc = 0;  // lane g < 16: width of group g
        for (uint32_t g0 = 0; g0 < G; g0 += 4) {
          const bool live = g0 + q < G;
          const uint32_t* xb = x + (size_t)(mb0 + g0 + q) * 128 + 16 * s8;
          uint32_t v[4][4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (live) {
              if (xal) {
                const uint4 t = __ldg(reinterpret_cast<const uint4*>(xb) + k);
                v[k][0] = t.x; v[k][1] = t.y; v[k][2] = t.z; v[k][3] = t.w;
              } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) v[k][j] = __ldg(xb + 4 * k + j);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) v[k][j] = 0;
            }
          }
          // previous slot (4 values) of each thread's first slot
          uint4 prev;
          prev.x = __shfl_up_sync(0xFFFFFFFFu, v[3][0], 1);
          prev.y = __shfl_up_sync(0xFFFFFFFFu, v[3][1], 1);
          prev.z = __shfl_up_sync(0xFFFFFFFFu, v[3][2], 1);
          prev.w = __shfl_up_sync(0xFFFFFFFFu, v[3][3], 1);
          if (lane == 0) prev = carry;
          carry.x = __shfl_sync(0xFFFFFFFFu, v[3][0], 31);
          carry.y = __shfl_sync(0xFFFFFFFFu, v[3][1], 31);
          carry.z = __shfl_sync(0xFFFFFFFFu, v[3][2], 31);
          carry.w = __shfl_sync(0xFFFFFFFFu, v[3][3], 31);
          // differences (delta.cpp:18-23, 53-58), computed from the top slot down
          uint32_t d[4][4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t p0 = k ? v[k - 1][0] : prev.x, p1 = k ? v[k - 1][1] : prev.y;
            const uint32_t p2 = k ? v[k - 1][2] : prev.z, p3 = k ? v[k - 1][3] : prev.w;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t pr = 0;
              if (DELTA == IZG_DELTA_D4) pr = j == 0 ? p0 : j == 1 ? p1 : j == 2 ? p2 : p3;
              if (DELTA == IZG_DELTA_D1) pr = j ? v[k][j - 1] : p3;
              if (DELTA == IZG_DELTA_D2) pr = j >= 2 ? v[k][j - 2] : (j == 0 ? p2 : p3);
              if (DELTA == IZG_DELTA_DM) pr = p3;
              if (DELTA == IZG_DELTA_NONE) pr = 0;
              if (!WRAP && kArray && live && v[k][j] < pr) bad = true;
              d[k][j] = v[k][j] - pr;
            }
          }
          // block width: OR over the block's 8 lanes (bitpack.cpp:287-291)
          uint32_t acc = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) acc |= d[k][0] | d[k][1] | d[k][2] | d[k][3];
          acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
          acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 2);
          acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 4);
          const uint32_t b = live ? bitw(acc) : 0u;
          // payload offsets of the four blocks (words), from the block widths
          const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, b, 0), b1 = __shfl_sync(0xFFFFFFFFu, b, 8);
          const uint32_t b2 = __shfl_sync(0xFFFFFFFFu, b, 16), b3 = __shfl_sync(0xFFFFFFFFu, b, 24);
          const uint32_t off = 4u * (q == 0 ? 0 : q == 1 ? b0 : q == 2 ? b0 + b1 : b0 + b1 + b2);
          const uint32_t total = 4u * (b0 + b1 + b2 + b3);
          if (lane >= (int)g0 && lane < (int)g0 + 4) {
            const uint32_t k = lane - g0;
            wdesc = k == 0 ? b0 : k == 1 ? b1 : k == 2 ? b2 : b3;
          }
          // vertical pack into the tile (bitpack.h:18-23): value of slot s,
          // lane j -> bits [s*b, s*b+b) of lane j's stream
          for (uint32_t i = lane; i < total; i += 32) tile[i] = 0;
          __syncwarp();
          if (b) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t bit = (4u * s8 + k) * b;
              const uint32_t w0 = off + 4u * (bit >> 5), sh = bit & 31u;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                atomicOr(&tile[w0 + j], d[k][j] << sh);
                if (sh + b > 32) atomicOr(&tile[w0 + 4 + j], d[k][j] >> (32 - sh));
              }
            }
          }
          __syncwarp();
          for (uint32_t i = lane; i < total; i += 32) o[pos + i] = tile[i];
          pos += total;
          __syncwarp();
        }
        // descriptor: byte g = width of group g, absent groups 0 (codec_binpack.cpp:86-89)
        const uint32_t wv = lane < 16 ? wdesc : 0u;
        const uint32_t g4 = (lane & 3) * 4;
        const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, wv, g4), w1 = __shfl_sync(0xFFFFFFFFu, wv, g4 + 1);
        const uint32_t w2 = __shfl_sync(0xFFFFFFFFu, wv, g4 + 2), w3 = __shfl_sync(0xFFFFFFFFu, wv, g4 + 3);
        if (lane < 4) o[desc + lane] = w0 | w1 << 8 | w2 << 16 | w3 << 24;
      }
      if (__any_sync(0xFFFFFFFFu, bad)) st = IZG_E_DECREASING;
      if (st == IZG_OK && kArray && core < n && lane == 0) {
        // Variable Byte remainder (codec.cpp:29-33; codec_basic.cpp:16-25)
        uint32_t acc = 0, nbytes = 0;
        for (uint32_t i = core; i < n; ++i) {
          const uint32_t xi = x[i];
          uint32_t pr = 0;
          if (DELTA == IZG_DELTA_D4) pr = i >= 4 ? x[i - 4] : 0u;
          if (DELTA == IZG_DELTA_D1) pr = i >= 1 ? x[i - 1] : 0u;
          if (DELTA == IZG_DELTA_D2) pr = i >= 2 ? x[i - 2] : 0u;
          if (DELTA == IZG_DELTA_DM) pr = i >= 4 ? x[(i & ~3u) - 1] : 0u;
          if (!WRAP && xi < pr) {
            st = IZG_E_DECREASING;
            break;
          }
          uint32_t dv = xi - pr;
          for (;;) {
            const uint32_t byte = dv >= 128 ? (dv & 0x7Fu) : (dv | 0x80u);
            acc |= byte << (8 * (nbytes & 3));
            if ((++nbytes & 3) == 0) {
              o[pos++] = acc;
              acc = 0;
            }
            if (dv < 128) break;
            dv >>= 7;
          }
        }
        if (nbytes & 3) o[pos++] = acc;
      }
      st = __shfl_sync(0xFFFFFFFFu, st, 0);
      pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
    }
    if (lane == 0) {
      status[c] = st;
      chunks[c].n_words = st == IZG_OK ? pos : 0;
    }
  }
}

inline uint64_t izg_encode_bound_impl(int codec, uint32_t n) {
  const uint64_t nb = n / 128;
  const uint64_t rem = 159;  // 127 VByte values of at most 5 bytes
  if (codec == IZG_SIMDBP128) return 4 * ((nb + 15) / 16) + 128 * nb + rem + 4;
  return 2 + 128 * nb + 1 + (131 * nb + 3) / 4 + 1 + 32 * 4 + 128 * nb + 32 * 128 + rem + 4;
}

}  // namespace izg
