// decode_bp128.cuh — one warp decodes one SIMD-BP128 chunk.
//
// Restates, fused into a single pass out of the warp's shared-memory ring:
//   SimdBp128Codec::decode_deltas   codec_binpack.cpp:94-119 (meta-block walk,
//                                   width/truncation checks, words consumed)
//   unpack_vertical128              bitpack.cpp:122-161, 324-328
//   delta_decode (D1/D4)            delta.cpp:25-89 (+ D2/DM extensions)
// The 16-byte meta-block descriptor is read once per meta-block by all
// lanes; lanes 0..15 each own one group width and a 16-lane scan yields the
// block offsets, so the descriptor chain costs one shared-memory round trip
// per 2048 integers and never a dependent global load.
#pragma once
#include "izg_common.cuh"

namespace izg {

struct MetaWalk {
  uint32_t width;  // lane g's group width (lanes 0..15; lanes 16..31 mirror)
  uint32_t excl;   // payload words from the end of the descriptor to block g
  uint32_t size;   // payload words of all present blocks (uniform)
  int32_t err;     // first error in the reference's check order (uniform)
};

// One meta-block descriptor at payload word `pos` with `groups` present
// groups (codec_binpack.cpp:104-117): for each present group in order, a
// width byte > 32 is an error, then a payload running past `nw` words.
template <bool ALIGNED, typename R>
__device__ __forceinline__ MetaWalk walk_meta(const R& r, uint32_t pos, uint32_t groups,
                                              uint32_t nw, int lane) {
  uint32_t d0, d1, d2, d3;
  if (ALIGNED) {
    const uint4 d = lds128(r.word_addr(pos));
    d0 = d.x; d1 = d.y; d2 = d.z; d3 = d.w;
  } else {
    d0 = lds32(r.word_addr(pos));
    d1 = lds32(r.word_addr(pos + 1));
    d2 = lds32(r.word_addr(pos + 2));
    d3 = lds32(r.word_addr(pos + 3));
  }
  const uint32_t g = lane & 15;
  const uint32_t word = g < 4 ? d0 : g < 8 ? d1 : g < 12 ? d2 : d3;
  const uint32_t w = (word >> (8 * (g & 3))) & 0xFFu;
  const bool valid = g < groups;
  const uint32_t sz = valid ? 4u * min(w, 33u) : 0u;
  uint32_t incl = sz;
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d, 16);
    if (g >= (uint32_t)d) incl += y;
  }
  const bool bad_w = valid && w > 32;
  const bool bad_t = valid && (pos + 4 + incl > nw);
  const uint32_t mw = __ballot_sync(0xFFFFFFFFu, bad_w) & 0xFFFFu;
  const uint32_t mt = __ballot_sync(0xFFFFFFFFu, bad_t) & 0xFFFFu;
  MetaWalk m;
  m.err = IZG_OK;
  if (mw | mt) {
    const int first = __ffs(mw | mt) - 1;
    m.err = ((mw >> first) & 1u) ? IZG_E_BP_WIDTH : IZG_E_BP_TRUNC_PAYLOAD;
  }
  m.width = w;
  m.excl = incl - sz;
  m.size = __shfl_sync(0xFFFFFFFFu, incl, groups - 1);
  return m;
}

// Unpack one thread's 4 slots x 4 lanes of a block whose payload starts at
// unmasked ring byte `bb`, sliding a two-row window (lo, hi) down the block:
// a 16-byte row is fetched only when the bit cursor enters it, so each lane
// reads each row it needs once (bitpack.cpp:122-143 restated per lane).
template <typename R>
__device__ __forceinline__ void unpack_slots_aligned(const R& r, uint32_t bb, uint32_t width,
                                                     uint32_t s8, uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
  uint32_t bit = 4u * s8 * width;
  uint32_t row = bit >> 5;
  uint32_t ra = bb + 16u * row;
  uint4 lo = lds128(r.base + (ra & R::kMask));
  uint4 hi = lds128(r.base + ((ra + 16u) & R::kMask));
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c) {
      bit += width;
      if ((bit >> 5) != row) {
        ++row;
        ra += 16u;
        lo = hi;
        hi = lds128(r.base + ((ra + 16u) & R::kMask));
      }
    }
    const uint32_t sh = bit & 31u;
    v[c][0] = funnel_r(lo.x, hi.x, sh) & mask;
    v[c][1] = funnel_r(lo.y, hi.y, sh) & mask;
    v[c][2] = funnel_r(lo.z, hi.z, sh) & mask;
    v[c][3] = funnel_r(lo.w, hi.w, sh) & mask;
  }
}

// Same, two row loads per slot and no window: fewer instructions, more
// shared-memory wavefronts.
__device__ __forceinline__ void unpack_slots_rows(const WarpRing& r, uint32_t bb, uint32_t width,
                                                  uint32_t s8, uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
  uint32_t bit = 4u * s8 * width;
#pragma unroll
  for (int c = 0; c < 4; ++c, bit += width) {
    const uint32_t ra = bb + 16u * (bit >> 5), sh = bit & 31u;
    const uint4 lo = lds128(r.base + (ra & kRingMask));
    const uint4 hi = lds128(r.base + ((ra + 16u) & kRingMask));
    v[c][0] = funnel_r(lo.x, hi.x, sh) & mask;
    v[c][1] = funnel_r(lo.y, hi.y, sh) & mask;
    v[c][2] = funnel_r(lo.z, hi.z, sh) & mask;
    v[c][3] = funnel_r(lo.w, hi.w, sh) & mask;
  }
}

// Same for a payload that is not 16-byte aligned in the ring: word loads.
template <typename R>
__device__ __forceinline__ void unpack_slots_unaligned(const R& r, uint32_t bword,
                                                       uint32_t width, uint32_t s8,
                                                       uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t bit = (4u * s8 + c) * width;
    const uint32_t w0 = bword + 4 * (bit >> 5), sh = bit & 31u;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      v[c][j] = funnel_r(lds32(r.word_addr(w0 + j)), lds32(r.word_addr(w0 + 4 + j)), sh) & mask;
  }
}

// Scalar 32-integer groups (bitpack.h:12-16: value i of a group at bits
// [i*b, i*b+b) of its b-word stream), as used by BP32 and the scalar
// FastPFOR family: a 128-integer block is 4 groups of `width` words from
// stream word `bword`.  Mapping C gives lane 8q+s8 block values
// 16*s8 .. 16*s8+15, i.e. half (s8 & 1) of group s8/2; the lane slides a
// two-word window along its 16*width bits (one shared load per word).
__device__ __forceinline__ void unpack_scalar_slots(const WarpRing& r, uint32_t bword,
                                                    uint32_t width, uint32_t s8,
                                                    uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
  const uint32_t gbase = bword + (s8 >> 1) * width;
  uint32_t bit = 16u * (s8 & 1u) * width;
  uint32_t wi = bit >> 5;
  uint32_t lo = lds32(r.word_addr(gbase + wi));
  uint32_t hi = lds32(r.word_addr(gbase + wi + 1));
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (k) {
      bit += width;
      if ((bit >> 5) != wi) {
        ++wi;
        lo = hi;
        hi = lds32(r.word_addr(gbase + wi + 1));
      }
    }
    v[k >> 2][k & 3] = funnel_r(lo, hi, bit & 31u) & mask;
  }
}

// One 32-integer scalar group "by value": lane l extracts value l (bits
// [l*w, l*w+w) of the w-word stream at payload word `off`) and stores it at
// integer 32*row + l of the warp's output tile `t`.  The tile row is uniform,
// so the 128-byte swizzle (OutStage::swz) reduces to an XOR of the lane's
// 16-byte chunk with row & 7; 32 consecutive integers of one row are
// conflict-free.  `roff` = r.ring_off().
__device__ __forceinline__ void scalar_group_to_tile(const WarpRing& r, uint32_t roff,
                                                     uint32_t off, uint32_t w, uint32_t t,
                                                     uint32_t row, int lane) {
  const uint32_t bit = (uint32_t)lane * w;
  const uint32_t a = roff + 4u * off + ((bit >> 5) << 2);  // unmasked ring byte of word 0
  const uint32_t lo = lds32(r.base + (a & kRingMask));
  const uint32_t hi = lds32(r.base + ((a + 4u) & kRingMask));
  const uint32_t dst = t + (row << 7) + ((((uint32_t)lane >> 2) ^ (row & 7u)) << 4) +
                       (((uint32_t)lane & 3u) << 2);
  sts32(dst, funnel_r(lo, hi, bit & 31u) & low_mask(w));
}

// Bp32Codec::decode_deltas (codec_binpack.cpp:43-60) fused like bp128_core:
// per 128 integers one descriptor word (byte g = width of scalar group g)
// and the four groups.  Per warp iteration the four descriptors are read as
// a short dependent chain with a one-instruction width check (__vcmpgtu4)
// and a byte-sum bound check; only a failing descriptor re-runs the
// reference's per-group checks in order.  The 16 groups are unpacked by
// value into the output tile and read back in mapping C for the scan.
template <int DELTA, typename OS>
__device__ int32_t bp32_core(WarpRing& r, OS& os, uint32_t nw, uint32_t nblocks,
                             uint32_t* out, bool out_aligned, int64_t orow, uint4& carry,
                             uint32_t* pos_out) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  uint32_t pos = 0;
#pragma unroll 1
  for (uint32_t g0 = 0; g0 < nblocks; g0 += 4) {
    const uint32_t ng = min(4u, nblocks - g0);
    // everything before this iteration is consumed: free it first, so the
    // ring can take the whole iteration (<= 4 x 129 words) before ensure()
    r.release_below(4u * pos);
    uint32_t desc[4], dpos[4];
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      desc[k] = 0;
      dpos[k] = pos;
      if (k < ng) {
        if (pos >= nw) return IZG_E_BP32_TRUNC_DESC;
        r.ensure(4u * (pos + 1));
        const uint32_t d = lds32(r.word_addr(pos));
        const uint32_t sum = __dp4a(d, 0x01010101u, 0u);  // the four widths
        if (__vcmpgtu4(d, 0x20202020u) || pos + 1 + sum > nw) {
          uint32_t at = pos + 1;  // codec_binpack.cpp:49-53, group by group
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t w = (d >> (8 * g)) & 0xFFu;
            if (w > 32) return IZG_E_BP32_WIDTH;
            if (at + w > nw) return IZG_E_BP32_TRUNC_PAYLOAD;
            at += w;
          }
        }
        desc[k] = d;
        dpos[k] = pos + 1;
        pos += 1 + sum;
      }
    }
    r.ensure(4u * pos);
    const uint32_t t = os.acquire();
    const uint32_t roff = r.ring_off();
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      if (k < ng) {
        uint32_t off = dpos[k];
#pragma unroll
        for (uint32_t g = 0; g < 4; ++g) {
          const uint32_t w = (desc[k] >> (8 * g)) & 0xFFu;
          scalar_group_to_tile(r, roff, off, w, t, 4u * k + g, lane);
          off += w;
        }
      }
    }
    __syncwarp();
    uint32_t v[4][4];
    OutStage::read(t, v, lane);
    const bool active = q < ng;
    if (!active) {  // blocks past the end: zero deltas keep the carry exact
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[c][j] = 0;
    }
    scan<DELTA>(v, carry, lane);
    if (orow >= 0 && ng == 4) {
      os.commit(v, lane, (uint32_t)(orow + 4 * g0));
    } else {
      os.abandon();
      os.direct(v, out + (size_t)(g0 + q) * 128 + 16 * s8, out_aligned, active, 128u * ng, lane);
    }
  }
  *pos_out = pos;
  return IZG_OK;
}

// Decode `nblocks` core blocks of the chunk streaming through `r`.
// Returns an izg_status; on success *pos_out = payload words consumed.
// `orow` is the chunk's first output row (32 integers) for the TMA path, or
// -1 when the output is not 128-byte aligned (direct stores then).
// Split decode (split.cuh): blocks [blk_begin, nblocks) only, blk_begin a
// multiple of 16 with the ring and `nw` starting at its meta-block; output
// indices stay chunk-relative.
// OS::kAgg (AggStage, split.cuh): nothing is written; the deltas are only
// summed per carry component, and `carry` is advanced by the segment's
// aggregate (what the scan would have carried out of it).
template <int DELTA>
__device__ __forceinline__ void accumulate(const uint32_t (&v)[4][4], uint4& a) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (DELTA == IZG_DELTA_D4) {
      a.x += v[c][0]; a.y += v[c][1]; a.z += v[c][2]; a.w += v[c][3];
    } else if (DELTA == IZG_DELTA_D1) {
      a.x += v[c][0] + v[c][1] + v[c][2] + v[c][3];
    } else if (DELTA == IZG_DELTA_D2) {
      a.x += v[c][0] + v[c][2];
      a.y += v[c][1] + v[c][3];
    } else if (DELTA == IZG_DELTA_DM) {
      a.x += v[c][3];  // DM carries the last value of each 4-vector
    }
  }
}

template <int DELTA, bool ALIGNED, typename OS>
__device__ int32_t bp128_core(WarpRing& r, OS& os, uint32_t nw, uint32_t nblocks,
                              uint32_t* out, bool out_aligned, int64_t orow, uint4& carry,
                              uint32_t* pos_out, uint32_t blk_begin = 0) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  uint32_t pos = 0;
  uint4 acc = make_uint4(0, 0, 0, 0);  // OS::kAgg: this lane's sums
  for (uint32_t mb0 = blk_begin; mb0 < nblocks; mb0 += 16) {
    const uint32_t groups = min(16u, nblocks - mb0);
    if (pos + 4 > nw) return IZG_E_BP_TRUNC_DESC;
    r.release_below(4u * pos);
    r.ensure(4u * (pos + 4));
    const MetaWalk m = walk_meta<ALIGNED>(r, pos, groups, nw, lane);
    if (m.err) return m.err;
    const uint32_t pay = pos + 4;  // first block's payload word
#pragma unroll 1
    for (uint32_t g0 = 0; g0 < groups; g0 += 4) {
      const uint32_t gi = g0 + q;
      const bool active = gi < groups;
      uint32_t width = __shfl_sync(0xFFFFFFFFu, m.width, gi & 15);
      const uint32_t excl = __shfl_sync(0xFFFFFFFFu, m.excl, gi & 15);
      // Stream window of this iteration: its first block to its last.
      const uint32_t first = __shfl_sync(0xFFFFFFFFu, m.excl, g0);
      const uint32_t lastg = min(g0 + 3, groups - 1);
      const uint32_t endw = __shfl_sync(0xFFFFFFFFu, m.excl + 4 * m.width, lastg);
      r.release_below(4u * (pay + first));
      r.ensure(4u * (pay + endw));
      if (!active) width = 0;  // reads stay in the ring; values are zero
      uint32_t v[4][4];
      if (ALIGNED)
        unpack_slots_aligned(r, r.ring_off() + 4u * (pay + excl), width, s8, v);
      else
        unpack_slots_unaligned(r, pay + excl, width, s8, v);
      if constexpr (OS::kAgg) {
        accumulate<DELTA>(v, acc);
        continue;
      }
#ifndef IZG_ABL_BP_NOSCAN  // developer ablation (wrong output): no prefix sum
      scan<DELTA>(v, carry, lane);
#endif
#ifdef IZG_ABL_BP_NOSTORE  // developer ablation (no output): nothing stored
      if (v[0][0] == 0xFFFFFFFFu && v[3][3] == 0x12345678u) carry.x += 1;
      continue;
#endif
      if (orow >= 0 && g0 + 4 <= groups) {
        os.put(v, lane, (uint32_t)(orow + 4 * (mb0 + g0)));
      } else {
        os.direct(v, out + (size_t)(mb0 + gi) * 128 + 16 * s8, out_aligned, active,
                  128u * min(4u, groups - g0), lane);
      }
    }
    pos = pay + m.size;
  }
  if constexpr (OS::kAgg) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      acc.x += __shfl_xor_sync(0xFFFFFFFFu, acc.x, d);
      if (DELTA == IZG_DELTA_D4 || DELTA == IZG_DELTA_D2)
        acc.y += __shfl_xor_sync(0xFFFFFFFFu, acc.y, d);
      if (DELTA == IZG_DELTA_D4) {
        acc.z += __shfl_xor_sync(0xFFFFFFFFu, acc.z, d);
        acc.w += __shfl_xor_sync(0xFFFFFFFFu, acc.w, d);
      }
    }
    carry = u4add(carry, acc);
  }
  *pos_out = pos;
  return IZG_OK;
}

}  // namespace izg
