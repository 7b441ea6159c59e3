// izg_common.cuh — pieces shared by the fused decode kernels.
//
// Execution model: one WARP decodes one chunk at a time and
// owns a private shared-memory ring that its lane 0 fills with TMA bulk
// copies (cp.async.bulk global->shared, completion on an mbarrier).  No
// inter-warp synchronisation exists on the hot path: the prefix-sum carry
// lives in the warp's registers, so tens of independent chunks are in
// flight per SM and the per-chunk dependency chains overlap.
//
// Register layout of one warp iteration ("mapping C"): lane
// l = 8q + s8 owns block q (0..3) of the iteration and, in that block,
// vertical slots 4*s8 .. 4*s8+3 of all four lanes.  Slot s of lane j is
// integer 4s+j of the block (bitpack.h:18-23), so every lane holds 16
// CONSECUTIVE integers v[c][j] = block[16*s8 + 4c + j] and the warp holds 512
// consecutive integers.  D4's four residue classes are the four vertical
// lanes (delta.h:13-15): each prefix sum is a 3-add in-thread scan plus one
// warp scan of per-lane totals.
#pragma once
#include <cstdint>

#include "../../include/intzip_b200.h"
#include "izg_ptx.cuh"

namespace izg {

// IZG_BOUNDS (developer build; the pool refuses compute-sanitizer): every
// global access range the team decode and the lane index pass form is checked against the
// chunk's own span — reads inside the 16-byte-aligned cover of [page, page + n_words),
// writes inside [out + out_off, + n) — and violations are counted (izg_debug_bounds).
#ifdef IZG_BOUNDS
__device__ unsigned int g_izg_oob[4];  // count, kind of the first, its chunk, its offset
__device__ __forceinline__ void izg_check(bool ok, uint32_t kind, uint32_t chunk, uint32_t off) {
  if (!ok && atomicAdd(&g_izg_oob[0], 1u) == 0) {
    g_izg_oob[1] = kind;
    g_izg_oob[2] = chunk;
    g_izg_oob[3] = off;
  }
}
// [a, a + len) inside the 16-byte-aligned cover of [page, page + 4 nw)
__device__ __forceinline__ bool izg_in_span(uintptr_t a, uint64_t len, const void* page, uint32_t nw) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(page) & ~uintptr_t(15);
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(page) + 4ull * nw + 15) & ~uintptr_t(15);
  return a >= lo && a + len <= hi;
}
#define IZG_CHECK(ok, kind, chunk, off) izg_check((ok), (kind), (chunk), (off))
#else
#define IZG_CHECK(ok, kind, chunk, off)
#endif

constexpr uint32_t kSB = 1024;                // bytes per ring stage
constexpr uint32_t kNS = 4;                   // stages per warp ring
constexpr uint32_t kRingBytes = kSB * kNS;    // 4 KiB per warp
constexpr uint32_t kRingMask = kRingBytes - 1;
constexpr uint32_t kStageOut = 2048;          // one warp iteration of output (512 ints)

// Shared memory per CTA: the warps' rings, then 2 output staging tiles per
// warp (1024-byte aligned for the 128-byte TMA swizzle), then per-warp
// SIMD-FastPFOR block tables, then the ring barriers.
// SHAPE (indexed SIMD-FastPFOR only): 0 = 4 warps per CTA at 96 registers
// (20 warps per SM), 1 = 6 warps at 80 registers (24 per SM) for very large
// batches, whose page records come from HBM rather than L2.
template <int CODEC, bool IDX = false, int SHAPE = 0>
struct Layout {
  // page codecs (byte array + exceptions) vs binary packing
  static constexpr bool kPaged = CODEC == IZG_SIMDFASTPFOR || CODEC == IZG_FASTPFOR ||
                                 CODEC == IZG_SIMPLEPFOR;
#ifndef IZG_IDX_WARPS
#define IZG_IDX_WARPS 4  // with 96 registers: 5 CTAs, 20 warps per SM
#endif
#ifndef IZG_PAGED_WARPS
#define IZG_PAGED_WARPS 4  // fused page kernels: 5 CTAs of 4 warps at 96 registers
#endif
#ifndef IZG_BIG_TILES
#define IZG_BIG_TILES 1
#endif
#ifndef IZG_IDX_TILES
#define IZG_IDX_TILES 1
#endif
#ifndef IZG_PAGED_TILES
#define IZG_PAGED_TILES 1
#endif
#ifndef IZG_BIG_WARPS
#define IZG_BIG_WARPS 6  // indexed SIMD-FastPFOR, SHAPE 1 (80 registers)
#endif
#ifndef IZG_BP_WARPS
#define IZG_BP_WARPS 8
#endif
#ifndef IZG_BP_MAXREGS
#define IZG_BP_MAXREGS 80
#endif
  static constexpr int kWarps =
      kPaged ? (IDX ? (SHAPE ? IZG_BIG_WARPS : IZG_IDX_WARPS) : IZG_PAGED_WARPS) : IZG_BP_WARPS;
  // registers per thread: 3 CTAs per SM for the fused kernels; the indexed
  // page decode runs 5 CTAs of 4 warps at 96 registers (no spills; measured
  // better than 24 warps at 80 registers)
#ifndef IZG_PAGED_MAXREGS
#define IZG_PAGED_MAXREGS 96
#endif
#ifndef IZG_IDX_MAXREGS
#define IZG_IDX_MAXREGS 96
#endif
  static constexpr int kMaxRegs = !kPaged ? IZG_BP_MAXREGS
                                 : IDX    ? (SHAPE ? 80 : IZG_IDX_MAXREGS)
                                          : IZG_PAGED_MAXREGS;
  // per-warp scratch, 16-byte multiple: the fused page kernels' FpScratch
  // (decode_fastpfor.cuh), the indexed one's exception directory only
  static constexpr uint32_t kTabBytes = !kPaged ? 0 : IDX ? 144 : 2048 + 512 + 2 * 33 * 4 + 8;
  // output tiles per warp: 2, or 1 for the large-batch indexed shape
  // (IZG_BIG_TILES) — less shared memory, more L1 for the exception loads
  static constexpr int kTiles = !kPaged ? 2
                                : IDX   ? (SHAPE ? IZG_BIG_TILES : IZG_IDX_TILES)
                                        : IZG_PAGED_TILES;
  static constexpr uint32_t kOutOff = kWarps * kRingBytes;
  static constexpr uint32_t kTabOff = kOutOff + kWarps * kTiles * kStageOut;
  static constexpr uint32_t kBarOff = kTabOff + kWarps * kTabBytes;
  static constexpr size_t kSmem = kBarOff + kWarps * kNS * 8;
};

// A warp's private TMA ring.  All lanes keep identical counters; lane 0
// issues the copies.  Chunk payloads stream as the 16-byte-aligned span
// covering them; `phase` is payload word 0's byte offset in that span.
struct WarpRing {
  static constexpr uint32_t kMask = kRingMask;
  uint32_t base;        // shared address of the ring
  uint32_t bar;         // shared address of its kNS mbarriers (8 bytes each)
  uint32_t g;           // stages consumed before the current chunk
  const uint8_t* a16;   // current chunk span
  uint32_t total, phase, nst;
  uint32_t issued, waited, released;
  uint64_t policy;
  bool leader;

  __device__ __forceinline__ uint32_t addr(uint32_t o) const {
    return base + (((g % kNS) * kSB + phase + o) & kRingMask);
  }
  __device__ __forceinline__ uint32_t word_addr(uint32_t w) const { return addr(4u * w); }
  // Unmasked ring offset of payload byte 0 (add a byte offset, mask, add base).
  __device__ __forceinline__ uint32_t ring_off() const { return (g % kNS) * kSB + phase; }

  __device__ __forceinline__ void refill() {
    while (issued < nst && issued < released + kNS) {
      if (leader) {
        const uint32_t slot = (g + issued) % kNS;
        const uint32_t off = issued * kSB;
        const uint32_t bytes = min(kSB, total - off);
        mbar_arrive_expect_tx_s(bar + 8u * slot, bytes);
        bulk_g2s_s(base + slot * kSB, a16 + off, bytes, bar + 8u * slot, policy);
      }
      ++issued;
    }
  }

  __device__ __forceinline__ void begin(const uint32_t* p, uint32_t n_words) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p);
    const uintptr_t s = a0 & ~uintptr_t(15);
    const uintptr_t e = (a0 + 4ull * n_words + 15) & ~uintptr_t(15);
    a16 = reinterpret_cast<const uint8_t*>(s);
    total = static_cast<uint32_t>(e - s);
    phase = static_cast<uint32_t>(a0 - s);
    nst = n_words ? (total + kSB - 1) / kSB : 0;
    issued = waited = released = 0;
    refill();
  }

  // Block until payload bytes [0, end) have landed.
  __device__ __forceinline__ void ensure(uint32_t end) {
    const uint32_t need = phase + end;
    while (waited * kSB < need && waited < issued) {
      const uint32_t gg = g + waited;
      mbar_wait_s(bar + 8u * (gg % kNS), (gg / kNS) & 1u);
      ++waited;
    }
  }

  // Recycle every stage lying entirely below payload byte `o`.
  __device__ __forceinline__ void release_below(uint32_t o) {
    uint32_t upto = (phase + o) / kSB;
    if (upto > waited) upto = waited;
    if (upto > released) {
      __syncwarp();
      fence_proxy_async_smem();  // generic reads before the async-proxy refill
      released = upto;
      refill();
    }
  }

  // End of chunk: drain copies still in flight so slots and phases stay
  // consistent for the next chunk.
  __device__ __forceinline__ void end() {
    ensure(0xFFFFFFF0u - phase);
    __syncwarp();
    fence_proxy_async_smem();
    g += issued;
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
    const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, t.x, d);
    const uint32_t y1 = NC > 1 ? __shfl_up_sync(0xFFFFFFFFu, t.y, d) : 0u;
    const uint32_t y2 = NC > 2 ? __shfl_up_sync(0xFFFFFFFFu, t.z, d) : 0u;
    const uint32_t y3 = NC > 3 ? __shfl_up_sync(0xFFFFFFFFu, t.w, d) : 0u;
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
//   v     : the thread's 16 deltas, v[c][j] = block[16*s8 + 4c + j]
//   carry : running state entering the iteration (identical in all lanes),
//           updated to the state after the iteration:
//     D4 (delta.cpp:60-75): carry.{x,y,z,w} = last value of vertical lane j
//     D1 (delta.cpp:25-51): carry.x = last value
//     D2 (ext):             carry.x / .y = last even / odd value
//     DM (ext):             carry.x = last value of the last 4-vector
//   out   : &output[16*s8] of the thread's block, or nullptr if inactive
template <int DELTA>
__device__ __forceinline__ void scan(uint32_t (&v)[4][4], uint4& carry, int lane) {
  if (DELTA != IZG_DELTA_NONE) {
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
    } else {  // DM
      uint32_t s = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        s += v[c][3];
        q3[c] = s;
      }
      T.x = s;
    }
    constexpr int NC = DELTA == IZG_DELTA_D4 ? 4 : DELTA == IZG_DELTA_D2 ? 2 : 1;
    const uint4 I = warp_incl_scan<NC>(T, lane);
    const uint4 base = u4add(carry, u4sub(I, T));
    uint4 tot;
    tot.x = __shfl_sync(0xFFFFFFFFu, I.x, 31);
    tot.y = NC > 1 ? __shfl_sync(0xFFFFFFFFu, I.y, 31) : 0u;
    tot.z = NC > 2 ? __shfl_sync(0xFFFFFFFFu, I.z, 31) : 0u;
    tot.w = NC > 3 ? __shfl_sync(0xFFFFFFFFu, I.w, 31) : 0u;
    carry = u4add(carry, tot);
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
  }
}

// Direct global store of the thread's 16 consecutive integers.
__device__ __forceinline__ void store_direct(const uint32_t (&v)[4][4], uint32_t* out,
                                             bool out_aligned) {
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

// Output path for full warp iterations: the warp's 512 consecutive integers
// go to a 2 KiB shared tile in the 128-byte-swizzled layout (conflict-free
// for mapping C: the 8 lanes of a quarter-warp land in 8 distinct 16-byte
// bank groups), then one TMA tensor store writes 16 full 128-byte rows.
// NT = 2: two tiles per warp alternate (SIMD-BP128, whose short iterations
// need the overlap); NT = 1: the page decoders, whose long iterations hide
// the wait and whose exception loads want the shared memory back as L1.
// A tile is reused once its store has read it.
template <int NT = 2>
struct OutStageT {
  static constexpr bool kProbe = false;  // see ProbeStage (probe.cuh)
  static constexpr bool kAgg = false;    // see AggStage (split.cuh)
  uint32_t base;     // shared address of the warp's two tiles (1024-aligned)
  uint32_t buf;
  const void* tmap;  // 2-D map of the output: rows of 32 integers, box 16 rows
  bool leader;

  __device__ __forceinline__ void begin_chunk() {}
  // Iterations that do not take the TMA path (short tails, unaligned output).
  __device__ __forceinline__ void direct(const uint32_t (&v)[4][4], uint32_t* o, bool oal,
                                         bool live, uint32_t /*nvalid*/, int /*lane*/) {
    if (live) store_direct(v, o, oal);
  }

  __device__ __forceinline__ void put(const uint32_t (&v)[4][4], int lane, uint32_t row) {
    if (leader) bulk_wait_read<NT - 1>();
    __syncwarp();
    const uint32_t t = base + buf * kStageOut;
    const uint32_t q = lane >> 3, s8 = lane & 7;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t L = 512u * q + 64u * s8 + 16u * k;
      const uint32_t r = L >> 7, c = (L >> 4) & 7u;
      sts128(t + (r << 7) + ((c ^ (r & 7u)) << 4), v[k][0], v[k][1], v[k][2], v[k][3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (leader) {
      tma_store_2d(tmap, t, 0, (int)row);
      bulk_commit();
    }
    buf = NT == 2 ? buf ^ 1u : 0u;
  }
  // Split form for SIMD-FastPFOR, which patches the tile in place:
  // acquire() -> write/patch/read the tile -> commit() or abandon().
  __device__ __forceinline__ uint32_t acquire() {
    if (leader) bulk_wait_read<NT - 1>();
    __syncwarp();
    return base + buf * kStageOut;
  }
  __device__ __forceinline__ void commit(const uint32_t (&v)[4][4], int lane, uint32_t row) {
    const uint32_t t = base + buf * kStageOut;
    write(t, v, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (leader) {
      tma_store_2d(tmap, t, 0, (int)row);
      bulk_commit();
    }
    buf = NT == 2 ? buf ^ 1u : 0u;
  }
  __device__ __forceinline__ void abandon() { __syncwarp(); }

  // Swizzled byte address of integer p (0..511) of a warp tile.
  __device__ __forceinline__ static uint32_t swz(uint32_t t, uint32_t p) {
    const uint32_t L = 4u * p, r = L >> 7, c = (L >> 4) & 7u;
    return t + (r << 7) + ((c ^ (r & 7u)) << 4) + (L & 15u);
  }
  __device__ __forceinline__ static void write(uint32_t t, const uint32_t (&v)[4][4], int lane) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      sts128(swz(t, 16u * lane + 4u * k), v[k][0], v[k][1], v[k][2], v[k][3]);
  }
  __device__ __forceinline__ static void read(uint32_t t, uint32_t (&v)[4][4], int lane) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 x = lds128(swz(t, 16u * lane + 4u * k));
      v[k][0] = x.x; v[k][1] = x.y; v[k][2] = x.z; v[k][3] = x.w;
    }
  }
  __device__ __forceinline__ void drain() {
    if (leader) bulk_wait<0>();
    __syncwarp();
  }
};
using OutStage = OutStageT<2>;

// Variable Byte remainder (codec_basic.cpp:27-51) of a chunk (at most 127
// integers), decoded by one lane straight from global memory and continued
// through the prefix sum from `carry` (codec.cpp:56-66).  Returns an
// izg_status; *rem_bytes = bytes consumed.
// `out` is the chunk's output (integer `core + i` goes to out[core + i]).
template <int DELTA>
__device__ int32_t vbyte_tail(const uint8_t* bytes, uint32_t nbytes, uint32_t core,
                              uint32_t count, uint4 carry, uint32_t* out, uint32_t* rem_bytes) {
  uint32_t pos = 0;
  uint32_t c0 = carry.x, c1 = carry.y, c2 = carry.z, c3 = carry.w;
  for (uint32_t i = 0; i < count; ++i) {
    uint32_t v = 0, shift = 0;
    for (;;) {
      if (pos >= nbytes) return IZG_E_VBYTE_TRUNCATED;
      const uint32_t b = __ldg(bytes + pos);
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
      const uint32_t k = idx & 3;
      x += k == 0 ? c0 : k == 1 ? c1 : k == 2 ? c2 : c3;
      if (k == 0) c0 = x; else if (k == 1) c1 = x; else if (k == 2) c2 = x; else c3 = x;
    } else if (DELTA == IZG_DELTA_D1) {
      x += c0;
      c0 = x;
    } else if (DELTA == IZG_DELTA_D2) {
      if (idx & 1) { x += c1; c1 = x; } else { x += c0; c0 = x; }
    } else if (DELTA == IZG_DELTA_DM) {
      x += c0;  // c0 = x_{4k-1}
      if ((idx & 3) == 3) c0 = x;
    }
    out[idx] = x;
  }
  *rem_bytes = pos;
  return IZG_OK;
}

}  // namespace izg
