// decode_bp128.cuh — consumer side of the fused SIMD-BP128 decoder.
//
// Restates, fused into one pass over shared memory:
//   SimdBp128Codec::decode_deltas   codec_binpack.cpp:94-119 (meta-block walk,
//                                   width/truncation checks)
//   unpack_vertical128              bitpack.cpp:122-161, 324-328
//   delta_decode (D1/D4)            delta.cpp:25-89
//   decode_array's chunk body       codec.cpp:50-68 (remainder, consumption)
//
// One CTA iteration = 2 meta-blocks = 32 blocks of 128 integers; consumer
// warp w takes blocks 4w..4w+3.  Every consumer thread walks the two 16-byte
// descriptors itself (lanes 0..15 hold one group each; a 16-lane scan gives
// the block offsets), so the 32-hop descriptor chain costs one shared-memory
// round trip per meta-block and never touches global memory.
#pragma once
#include "izg_common.cuh"

namespace izg {

struct MetaWalk {
  uint32_t width;  // this lane's group width (lanes 0..15)
  uint32_t excl;   // words from payload start of the meta-block to its block
  uint32_t size;   // payload words of the whole meta-block (uniform)
  int32_t err;     // first error (uniform)
};

// Walk one meta-block descriptor at payload word `pos` with `groups` present
// groups (codec_binpack.cpp:98-117); checks in the reference's order.
template <bool ALIGNED>
__device__ __forceinline__ MetaWalk walk_meta(const RingView& rv, uint32_t pos, uint32_t groups,
                                              uint32_t nw, int lane) {
  MetaWalk m;
  uint32_t d0, d1, d2, d3;
  if (ALIGNED) {
    const uint4 d = lds128(rv.word_addr(pos));
    d0 = d.x; d1 = d.y; d2 = d.z; d3 = d.w;
  } else {
    d0 = lds32(rv.word_addr(pos));
    d1 = lds32(rv.word_addr(pos + 1));
    d2 = lds32(rv.word_addr(pos + 2));
    d3 = lds32(rv.word_addr(pos + 3));
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
  m.err = IZG_OK;
  if (mw | mt) {
    const int first = __ffs(mw | mt) - 1;
    m.err = ((mw >> first) & 1u) ? IZG_E_BP_WIDTH : IZG_E_BP_TRUNC_PAYLOAD;
  }
  m.width = w;
  m.excl = incl - sz;
  m.size = __shfl_sync(0xFFFFFFFFu, incl, groups ? groups - 1 : 0);
  if (!groups) m.size = 0;
  return m;
}

// Decode the core blocks of one chunk.  Returns an izg_status; on success
// *pos_out = payload words consumed by the core (decode_deltas' return).
template <int DELTA, bool ALIGNED>
__device__ int32_t bp128_core(RingView& rv, uint64_t* full, uint64_t* empty, uint4 (*tot)[kCW],
                              uint32_t& tbuf, uint32_t nw, uint32_t nblocks, uint32_t* out,
                              bool out_aligned, uint4& carry, uint32_t* pos_out) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int q = lane >> 3, s8 = lane & 7;
  const int bi = 4 * warp + q;       // block within the iteration
  const int mbl = bi >> 4;           // meta-block within the iteration
  const uint32_t gi = bi & 15;       // group within the meta-block
  uint32_t pos = 0;
  for (uint32_t blk0 = 0; blk0 < nblocks; blk0 += kBlocksPerIter) {
    // --- descriptor walk: meta-blocks A and B of this iteration ---------
    const uint32_t gA = min(16u, nblocks - blk0);
    if (pos + 4 > nw) return IZG_E_BP_TRUNC_DESC;
    rv.ensure(full, 4u * (pos + 4));
    const MetaWalk A = walk_meta<ALIGNED>(rv, pos, gA, nw, lane);
    if (A.err) return A.err;
    const uint32_t posA = pos;
    pos += 4 + A.size;
    uint32_t gB = 0, posB = pos;
    MetaWalk B;
    B.width = 0; B.excl = 0; B.size = 0; B.err = 0;
    if (nblocks - blk0 > 16) {
      gB = min(16u, nblocks - blk0 - 16);
      if (pos + 4 > nw) return IZG_E_BP_TRUNC_DESC;
      rv.ensure(full, 4u * (pos + 4));
      B = walk_meta<ALIGNED>(rv, pos, gB, nw, lane);
      if (B.err) return B.err;
      pos += 4 + B.size;
    }
    rv.ensure(full, 4u * pos);

    // --- unpack this thread's 4 slots x 4 lanes -------------------------
    const uint32_t width = __shfl_sync(0xFFFFFFFFu, mbl ? B.width : A.width, gi);
    const uint32_t excl = __shfl_sync(0xFFFFFFFFu, mbl ? B.excl : A.excl, gi);
    const bool active = mbl ? gi < gB : gi < gA;
    uint32_t v[4][4];
    if (active) {
      const uint32_t bstart = (mbl ? posB : posA) + 4 + excl;  // block payload word
      const uint32_t mask = low_mask(width);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t bit = (4u * s8 + c) * width;
        const uint32_t r = bit >> 5, sh = bit & 31u;
        const uint32_t w0 = bstart + 4 * r;
        if (ALIGNED) {
          const uint4 lo = lds128(rv.word_addr(w0));
          const uint4 hi = lds128(rv.word_addr(w0 + 4));
          v[c][0] = funnel_r(lo.x, hi.x, sh) & mask;
          v[c][1] = funnel_r(lo.y, hi.y, sh) & mask;
          v[c][2] = funnel_r(lo.z, hi.z, sh) & mask;
          v[c][3] = funnel_r(lo.w, hi.w, sh) & mask;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[c][j] = funnel_r(lds32(rv.word_addr(w0 + j)), lds32(rv.word_addr(w0 + 4 + j)), sh) &
                      mask;
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[c][j] = 0;
    }

    // --- fused prefix sum + store (contains the iteration barrier) -----
    uint32_t* o = active ? out + (size_t)(blk0 + bi) * 128 + 16 * s8 : nullptr;
    scan_store<DELTA>(v, carry, tot[tbuf], warp, lane, o, out_aligned);
    tbuf ^= 1;
    rv.release_below(empty, 4u * pos, tid == 0);
  }
  *pos_out = pos;
  return IZG_OK;
}

}  // namespace izg
