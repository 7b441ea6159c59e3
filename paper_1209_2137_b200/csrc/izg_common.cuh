// izg_common.cuh — pieces shared by the fused decode kernels:
//   * the TMA ring that streams each chunk's compressed payload into shared
//     memory (producer side and the consumer-side view),
//   * the fused inverse differential coding + output stage for a warp that
//     holds four 128-integer blocks in "slot-major" registers.
//
// Register layout of a warp's four blocks ("mapping C"): lane
// l = 8q + s8 owns block q (0..3) of the warp and, in that block, vertical
// slots 4*s8 .. 4*s8+3 of all four lanes.  Slot s of lane j is integer 4s+j
// of the block (bitpack.h:18-23), so each lane holds 16 CONSECUTIVE integers
// v[c][j] = block[16*s8 + 4c + j] and the warp holds 512 consecutive
// integers.  D4's four residue classes are the four vertical lanes
// (delta.h:13-15), so every prefix sum is a short in-thread scan plus one
// warp scan of per-lane totals.
#pragma once
#include <cstdint>

#include "../../include/intzip_b200.h"
#include "izg_ptx.cuh"

namespace izg {

constexpr uint32_t kStage = 4096;                // bytes per ring stage
constexpr uint32_t kNStage = 16;                 // stages per ring
constexpr uint32_t kRing = kStage * kNStage;     // 64 KiB
constexpr uint32_t kRingMask = kRing - 1;
constexpr int kCW = 8;                           // consumer warps per CTA
constexpr int kConsumers = kCW * 32;
constexpr int kThreads = kConsumers + 32;        // + one producer warp
constexpr int kBlocksPerIter = kCW * 4;          // 32 blocks = 2 meta-blocks

// Geometry of a chunk's payload as streamed through the ring: the 16-byte
// aligned span [a16, a16 + total) covering the payload, `phase` = byte offset
// of payload word 0 inside that span.  Every chunk starts on a fresh stage.
struct StreamGeom {
  const uint8_t* a16;
  uint32_t total;
  uint32_t phase;
  uint32_t nst;
};

__device__ __forceinline__ StreamGeom stream_geom(const uint32_t* words, uint64_t word_off,
                                                  uint32_t n_words) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(words + word_off);
  const uintptr_t a16 = a0 & ~uintptr_t(15);
  const uintptr_t e16 = (a0 + 4ull * n_words + 15) & ~uintptr_t(15);
  StreamGeom g;
  g.a16 = reinterpret_cast<const uint8_t*>(a16);
  g.total = static_cast<uint32_t>(e16 - a16);
  g.phase = static_cast<uint32_t>(a0 - a16);
  g.nst = n_words ? (g.total + kStage - 1) / kStage : 0;
  return g;
}

// Producer: stream one chunk's span into consecutive ring stages.
__device__ __forceinline__ void produce_chunk(uint8_t* ring, uint64_t* full, uint64_t* empty,
                                              const StreamGeom& sg, uint32_t& g,
                                              uint64_t policy) {
  for (uint32_t k = 0; k < sg.nst; ++k, ++g) {
    const uint32_t slot = g % kNStage;
    mbar_wait(&empty[slot], ((g / kNStage) & 1u) ^ 1u);
    const uint32_t off = k * kStage;
    const uint32_t bytes = min(kStage, sg.total - off);
    mbar_arrive_expect_tx(&full[slot], bytes);
    bulk_g2s(ring + slot * kStage, sg.a16 + off, bytes, &full[slot], policy);
  }
}

// Consumer-side view of one chunk in the ring.  Every consumer thread keeps
// an identical copy; only consumer thread 0 arrives on `empty`.
struct RingView {
  uint32_t ring;      // shared-memory address of the ring
  uint32_t g0;        // global stage index of the chunk's first stage
  uint32_t phase;     // byte offset of payload word 0 in the first stage
  uint32_t nst;       // stages of the chunk
  uint32_t waited;    // stages known complete
  uint32_t released;  // stages handed back to the producer

  // Shared-memory address of payload byte `o`.
  __device__ __forceinline__ uint32_t addr(uint32_t o) const {
    return ring + (((g0 % kNStage) * kStage + phase + o) & kRingMask);
  }
  __device__ __forceinline__ uint32_t word_addr(uint32_t w) const { return addr(4u * w); }

  // Block until payload bytes [0, end) have landed.
  __device__ __forceinline__ void ensure(uint64_t* full, uint32_t end) {
    const uint32_t need = phase + end;
    while (waited * kStage < need && waited < nst) {
      const uint32_t gg = g0 + waited;
      mbar_wait(&full[gg % kNStage], (gg / kNStage) & 1u);
      ++waited;
    }
  }

  // Hand back every stage that lies entirely below payload byte `o`.
  __device__ __forceinline__ void release_below(uint64_t* empty, uint32_t o, bool leader) {
    uint32_t upto = (phase + o) / kStage;
    if (upto > waited) upto = waited;
    while (released < upto) {
      if (leader) mbar_arrive(&empty[(g0 + released) % kNStage]);
      ++released;
    }
  }

  // End of chunk (call after a consumer barrier): wait for and hand back
  // every remaining stage so the producer's phases stay in step.
  __device__ __forceinline__ void finish(uint64_t* full, uint64_t* empty, bool leader) {
    if (leader) {
      for (uint32_t k = released; k < nst; ++k) {
        const uint32_t gg = g0 + k;
        if (k >= waited) mbar_wait(&full[gg % kNStage], (gg / kNStage) & 1u);
        mbar_arrive(&empty[gg % kNStage]);
      }
    }
    waited = released = nst;
  }
};

__device__ __forceinline__ uint4 u4add(uint4 a, uint4 b) {
  return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ uint4 u4sub(uint4 a, uint4 b) {
  return make_uint4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}

template <int NC>
__device__ __forceinline__ uint4 warp_incl_scan(uint4 t, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, t.x, d);
    uint32_t y1 = NC > 1 ? __shfl_up_sync(0xFFFFFFFFu, t.y, d) : 0u;
    uint32_t y2 = NC > 2 ? __shfl_up_sync(0xFFFFFFFFu, t.z, d) : 0u;
    uint32_t y3 = NC > 3 ? __shfl_up_sync(0xFFFFFFFFu, t.w, d) : 0u;
    if (lane >= d) {
      t.x += y0;
      if (NC > 1) t.y += y1;
      if (NC > 2) t.z += y2;
      if (NC > 3) t.w += y3;
    }
  }
  return t;
}

// Fused inverse differential coding + store for one warp iteration.
//   v        : the thread's 16 deltas, v[c][j] = block[16*s8 + 4c + j]
//   carry    : running state entering the iteration (identical in all
//              consumer threads); updated to the state after the iteration
//   tot      : shared scratch [kCW] for warp totals (double-buffered by caller)
//   out      : &output[16*s8] of the thread's block, or nullptr if inactive
// Contains the per-iteration consumer barrier.
//   D4 (delta.cpp:60-75): carry.{x,y,z,w} = last value of vertical lane j.
//   D1 (delta.cpp:25-51): carry.x = last value.
//   D2 (ext):             carry.x / .y = last even / odd value.
//   DM (ext):             carry.x = last value of the last 4-vector.
template <int DELTA>
__device__ __forceinline__ void scan_store(uint32_t (&v)[4][4], uint4& carry, uint4* tot,
                                           int warp, int lane, uint32_t* out,
                                           bool out_aligned) {
  uint4 T = make_uint4(0, 0, 0, 0);
  uint32_t q3[4] = {0, 0, 0, 0};  // DM: inclusive prefix of lane-3 deltas
  if (DELTA == IZG_DELTA_D4) {
#pragma unroll
    for (int c = 1; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) v[c][j] += v[c - 1][j];
    T = make_uint4(v[3][0], v[3][1], v[3][2], v[3][3]);
  } else if (DELTA == IZG_DELTA_D1) {
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s += v[c][j];
        v[c][j] = s;
      }
    T.x = s;
  } else if (DELTA == IZG_DELTA_D2) {
    uint32_t se = 0, so = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      se += v[c][0]; v[c][0] = se;
      so += v[c][1]; v[c][1] = so;
      se += v[c][2]; v[c][2] = se;
      so += v[c][3]; v[c][3] = so;
    }
    T.x = se;
    T.y = so;
  } else if (DELTA == IZG_DELTA_DM) {
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s += v[c][3];
      q3[c] = s;
    }
    T.x = s;
  }

  if (DELTA != IZG_DELTA_NONE) {
    constexpr int NC = DELTA == IZG_DELTA_D4 ? 4 : DELTA == IZG_DELTA_D2 ? 2 : 1;
    const uint4 I = warp_incl_scan<NC>(T, lane);
    if (lane == 31) tot[warp] = I;
    named_bar_sync(1, kConsumers);
    uint4 P = carry, S = carry;
#pragma unroll
    for (int w = 0; w < kCW; ++w) {
      const uint4 t = tot[w];
      if (w < warp) P = u4add(P, t);
      S = u4add(S, t);
    }
    carry = S;
    const uint4 base = u4add(P, u4sub(I, T));
    if (DELTA == IZG_DELTA_D4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[c][0] += base.x; v[c][1] += base.y; v[c][2] += base.z; v[c][3] += base.w;
      }
    } else if (DELTA == IZG_DELTA_D1) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[c][j] += base.x;
    } else if (DELTA == IZG_DELTA_D2) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[c][0] += base.x; v[c][1] += base.y; v[c][2] += base.x; v[c][3] += base.y;
      }
    } else {  // DM: x[c][j] = L_{c-1} + d[c][j]
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t L = base.x + (c ? q3[c - 1] : 0u);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[c][j] += L;
      }
    }
  } else {
    named_bar_sync(1, kConsumers);
  }

  if (out) {
    if (out_aligned) {
#pragma unroll
      for (int c = 0; c < 4; ++c) stg128_cs(out + 4 * c, v[c][0], v[c][1], v[c][2], v[c][3]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) out[4 * c + j] = v[c][j];
    }
  }
}

// Variable Byte remainder (codec_basic.cpp:27-51) of a chunk, decoded by one
// thread from the ring, continued through the prefix sum with `carry`
// (codec.cpp:56-66).  Returns an izg_status; *rem_bytes = bytes consumed.
template <int DELTA>
__device__ int32_t vbyte_tail(const RingView& rv, uint32_t byte_pos, uint32_t nbytes,
                              uint32_t core, uint32_t count, uint4 carry, uint32_t* out,
                              uint32_t* rem_bytes) {
  uint32_t pos = 0;
  uint32_t c4[4] = {carry.x, carry.y, carry.z, carry.w};
  for (uint32_t i = 0; i < count; ++i) {
    uint32_t v = 0, shift = 0;
    for (;;) {
      if (pos >= nbytes) return IZG_E_VBYTE_TRUNCATED;
      const uint32_t b = lds8(rv.addr(byte_pos + pos));
      ++pos;
      if (b & 0x80u) {
        if (shift == 28 && (b & 0x70u)) return IZG_E_VBYTE_OVERFLOW;
        v |= (b & 0x7Fu) << shift;
        break;
      }
      if (shift == 28) return IZG_E_VBYTE_TOO_LONG;
      v |= b << shift;
      shift += 7;
    }
    const uint32_t idx = core + i;
    uint32_t x = v;
    if (DELTA == IZG_DELTA_D4) {
      x += c4[idx & 3];
      c4[idx & 3] = x;
    } else if (DELTA == IZG_DELTA_D1) {
      x += c4[0];
      c4[0] = x;
    } else if (DELTA == IZG_DELTA_D2) {
      x += c4[idx & 1];
      c4[idx & 1] = x;
    } else if (DELTA == IZG_DELTA_DM) {
      x += c4[0];  // c4[0] = x_{4k-1}
      if ((idx & 3) == 3) c4[0] = x;
    }
    out[idx] = x;
  }
  *rem_bytes = pos;
  return IZG_OK;
}

}  // namespace izg
