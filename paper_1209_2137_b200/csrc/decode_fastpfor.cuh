// decode_fastpfor.cuh — one warp decodes one SIMD-FastPFOR page.
//
// Restates FastPforCodec::decode_deltas for PatchStorage::vertical_arrays
// (codec_patched.cpp:292-417) fused with the prefix sum, in three phases:
//
//   1. byte array (codec_patched.cpp:309-336): streamed through the warp's
//      TMA ring and walked serially by every lane in lockstep (broadcast
//      shared loads), checking each entry in the reference's order.  Each
//      block's entry is packed into a 32-bit shared table word
//      {byte offset of its positions : 17, c : 8, w = maxbits - b : 6} plus a
//      width byte.  The position-range check runs lane-parallel beside the
//      serial walk and is resolved at the end (a bad position can only
//      precede, never follow, a structural error found later in the walk).
//   2. exception directory (codec_patched.cpp:346-379): at most 32 dependent
//      loads from L2 (the page tail was bulk-prefetched into L2 up front);
//      lane w-1 keeps array w's base word and count.  Arrays are NOT
//      bulk-unpacked: each high is extracted on demand (vertical layout:
//      value r lies in group r/128, lane r%4, slot (r%128)/4).
//   3. blocks (codec_patched.cpp:381-415): the packed area streams through
//      the ring; four blocks per warp iteration are unpacked (mapping C),
//      written to the warp's swizzled output tile, patched there with
//      shared-memory atomic OR (o[pos] |= high << b; duplicate positions OR
//      like the reference), read back, prefix-summed and TMA-stored.
// Per-width cursors live in lane w-1 and advance in block order, which
// yields the reference's "exception array exhausted" check exactly.
#pragma once
#include "decode_bp128.cuh"
#include "izg_common.cuh"

namespace izg {

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ldg_u8(const uint8_t* p) { return __ldg(p); }

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
                 : "memory");
}

// Phase 1.  Walks the byte array serially (every lane in lockstep, shared
// loads broadcast) with the reference's structural checks, filling tab/tab_b.
// Position bytes are NOT range-checked here: they are read anyway when the
// exceptions are patched, and fp_positions_bad() settles the precedence of
// a bad position on every error path.  *parsed = blocks whose entry passed.
__device__ int32_t fp_parse(WarpRing& r, uint32_t* tab, uint8_t* tab_b, uint64_t L,
                            uint32_t nblocks, int lane, uint32_t* parsed) {
  uint32_t bpos = 0;
  uint32_t k = 0;
  int32_t st = IZG_OK;
  uint32_t limit = 0;  // bytes [0, limit) of the stream are resident
  for (; k < nblocks; ++k) {
    if (bpos + 258u > limit) {  // an entry spans at most 3 + 255 bytes
      r.release_below(bpos);
      r.ensure(bpos + 512u);
      limit = r.waited * kSB - r.phase;
    }
    const uint32_t a = r.ring_off() + bpos;
    const uint32_t b = lds8(r.base + (a & kRingMask));
    const uint32_t mb = lds8(r.base + ((a + 1) & kRingMask));
    const uint32_t c = lds8(r.base + ((a + 2) & kRingMask));
    const bool exc = mb > b;
    // codec_patched.cpp:313-330, in order
    if (bpos + 2ull > L) { st = IZG_E_FP_TRUNC_META; break; }
    if (b > 32 || mb > 32 || b > mb) { st = IZG_E_FP_WIDTHS; break; }
    if (exc) {
      if (bpos + 2ull >= L) { st = IZG_E_FP_TRUNC_META; break; }
      if (c == 0) { st = IZG_E_FP_EMPTY_EXC; break; }
      if (bpos + 3ull + c > L) { st = IZG_E_FP_TRUNC_POS; break; }
    }
    if (lane == 0) {
      tab[k] = exc ? (bpos + 3) | (c << 17) | ((mb - b) << 25) : 0u;
      tab_b[k] = (uint8_t)b;
    }
    bpos += exc ? 3 + c : 2;
  }
  *parsed = k;
  if (st) return st;
  if (bpos != L) return IZG_E_FP_BA_LEN;
  return IZG_OK;
}

// Slow path for error statuses: does any exception position of blocks
// [0, nb) reach 128 (codec_patched.cpp:328-330)?  The reference validates
// every position during its byte-array walk, before any later check.
__device__ bool fp_positions_bad(const uint32_t* tab, const uint8_t* ba, uint32_t nb, int lane) {
  bool bad = false;
  for (uint32_t k = 0; k < nb; ++k) {
    const uint32_t e = tab[k];
    const uint32_t c = (e >> 17) & 0xFFu, bp = e & 0x1FFFFu;
    for (uint32_t i = lane; i < c; i += 32) bad |= ldg_u8(ba + bp + i) >= 128u;
  }
  return __any_sync(0xFFFFFFFFu, bad);
}

// Phase 2.  `pos` = page word after the byte array.  On success lane w-1
// holds array w's base word and count; *end = words consumed by the page.
__device__ int32_t fp_directory(const uint32_t* page, uint32_t nw, uint64_t pos, int lane,
                                uint32_t* base, uint32_t* count, uint32_t* end) {
  *base = 0;
  *count = 0;
  if (pos >= nw) return IZG_E_FP_NO_BITSET;
  uint32_t bits = ldg_u32(page + pos);
  ++pos;
  while (bits) {
    const uint32_t w = __ffs(bits);  // width w <-> bit w-1
    bits &= bits - 1;
    if (pos >= nw) return IZG_E_FP_TRUNC_EXC;
    const uint32_t n = ldg_u32(page + pos);
    pos = (pos + 1 + 3) & ~uint64_t{3};  // 16-byte alignment in the page
    const uint64_t nwords = ((uint64_t)n + 127) / 128 * 4 * w;
    if (pos + nwords > nw) return IZG_E_FP_TRUNC_EXC;
    if (lane == (int)w - 1) {
      *base = (uint32_t)pos;
      *count = n;
    }
    pos += nwords;
  }
  *end = (uint32_t)pos;
  return IZG_OK;
}

// High bits of exception r of the width-w vertical array at page word `base`.
__device__ __forceinline__ uint32_t fp_high(const uint32_t* page, uint32_t base, uint32_t w,
                                            uint32_t r) {
  const uint32_t t = r & 127u;
  const uint32_t bit = (t >> 2) * w;
  const uint32_t word = base + (r >> 7) * 4u * w + 4u * (bit >> 5) + (t & 3u);
  const uint32_t sh = bit & 31u;
  const uint32_t lo = ldg_u32(page + word);
  const uint32_t hi = ldg_u32(page + word + (sh + w > 32 ? 4u : 0u));
  return funnel_r(lo, hi, sh) & low_mask(w);
}

template <class T>
__device__ __forceinline__ T pick4(uint32_t k, T a, T b, T c, T d) {
  return k == 0 ? a : k == 1 ? b : k == 2 ? c : d;
}

// Per-block exception parameters of one warp iteration, in shared memory so
// a lane finds its exception's block with one broadcast load.
struct ExcParam {
  int32_t pbase;  // byte-array offset of exception e is pbase + e
  int32_t rbase;  // index in its width array is rbase + e
  uint32_t base;  // page word of that array
  uint32_t wb;    // w | b << 8
};

// Phase 3.  Returns an izg_status; *bad_pos is set when a position >= 128
// was met (the caller resolves precedence).
template <int DELTA>
__device__ int32_t fp_blocks(WarpRing& r, OutStage& os, const uint32_t* tab, const uint8_t* tab_b,
                             ExcParam* prm, const uint32_t* page, uint32_t A, uint32_t nblocks,
                             uint32_t dir_base, uint32_t dir_n, uint32_t* out, bool oal,
                             int64_t orow, uint4& carry, bool* bad_pos) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);
  uint32_t packed = 1;   // page word of the next block's payload
  uint32_t used = 0;     // lane w-1: exceptions consumed from array w
  bool bad = false;
#pragma unroll 1
  for (uint32_t g0 = 0; g0 < nblocks; g0 += 4) {
    const uint32_t ng = min(4u, nblocks - g0);
    uint32_t bq[4], offq[4], cx[4];
    int32_t err = IZG_OK;
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool live = (uint32_t)k < ng;
      const uint32_t e = live ? tab[g0 + k] : 0u;
      const uint32_t b = live ? tab_b[g0 + k] : 0u;
      const uint32_t c = (e >> 17) & 0xFFu, w = e >> 25;
      bq[k] = b;
      offq[k] = packed;
      cx[k] = tot;
      // codec_patched.cpp:387-388 then 406-407, block by block
      if (live && err == IZG_OK && packed + 4ull * b > A) err = IZG_E_FP_OVERRUN;
      packed += 4u * b;
      uint32_t cur = 0, base = 0;
      if (c) {
        const int src = (int)w - 1;
        cur = __shfl_sync(0xFFFFFFFFu, used, src);
        base = __shfl_sync(0xFFFFFFFFu, dir_base, src);
        const uint32_t n = __shfl_sync(0xFFFFFFFFu, dir_n, src);
        if (lane == src) used += c;
        if (err == IZG_OK && (uint64_t)cur + c > n) err = IZG_E_FP_EXHAUSTED;
      }
      if (lane == k) {
        ExcParam x;
        x.pbase = (int32_t)(e & 0x1FFFFu) - (int32_t)tot;
        x.rbase = (int32_t)cur - (int32_t)tot;
        x.base = base;
        x.wb = w | b << 8;
        prm[k] = x;
      }
      tot += c;
    }
    if (err) return err;

    // Stream window: packed words [offq[0], packed) (the stream starts at word 1).
    r.release_below(4u * (offq[0] - 1));
    r.ensure(4u * (packed - 1));
    const bool live = q < ng;
    const uint32_t myb = live ? pick4(q, bq[0], bq[1], bq[2], bq[3]) : 0u;
    const uint32_t myoff = pick4(q, offq[0], offq[1], offq[2], offq[3]);
    uint32_t v[4][4];
    if (r.phase == 0)
      unpack_slots_aligned(r, r.ring_off() + 4u * (myoff - 1), myb, s8, v);
    else
      unpack_slots_unaligned(r, myoff - 1, myb, s8, v);

    const uint32_t t = os.acquire();
    OutStage::write(t, v, lane);
    __syncwarp();
    // Exceptions, 8 rounds of 32 per batch: every load of a batch is issued
    // before the first shared-memory OR (lanes past the end re-read the last
    // exception and skip the OR), so a batch costs one L2 round trip.
    for (uint32_t e0 = 0; e0 < tot; e0 += 256) {
      uint32_t where[8], what[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t e = min(e0 + 32u * j + lane, tot - 1);
        const uint32_t k = (e >= cx[1]) + (e >= cx[2]) + (e >= cx[3]);
        const ExcParam x = prm[k];
        const uint32_t w = x.wb & 0xFFu, b = x.wb >> 8;
        const uint32_t p = ldg_u8(ba + (x.pbase + (int32_t)e));
        what[j] = fp_high(page, x.base, w, (uint32_t)(x.rbase + (int32_t)e)) << b;
        where[j] = p < 128u ? OutStage::swz(t, 128u * k + p) : 0xFFFFFFFFu;
        bad |= p >= 128u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (e0 + 32u * j + lane < tot && where[j] != 0xFFFFFFFFu)
          asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(where[j]), "r"(what[j]));
    }
    __syncwarp();
    OutStage::read(t, v, lane);
    scan<DELTA>(v, carry, lane);
    if (orow >= 0 && ng == 4) {
      os.commit(v, lane, (uint32_t)(orow + 4 * g0));
    } else {
      os.abandon();
      if (live) store_direct(v, out + (size_t)(g0 + q) * 128 + 16 * s8, oal);
    }
  }
  *bad_pos = __any_sync(0xFFFFFFFFu, bad);
  if (packed != A) return IZG_E_FP_PACKED_SIZE;
  return IZG_OK;
}

// Whole page.  `nblocks` = count / 128; *pos_out = words consumed.
template <int DELTA>
__device__ int32_t fastpfor_core(WarpRing& r, OutStage& os, uint32_t* tab, uint8_t* tab_b,
                                 ExcParam* prm, const uint32_t* page, uint32_t nw,
                                 uint32_t nblocks, uint32_t* out, bool oal, int64_t orow,
                                 uint4& carry, uint32_t* pos_out) {
  const int lane = threadIdx.x & 31;
  if (nblocks == 0) {  // decode_deltas(count == 0) reads nothing (codec_patched.cpp:295)
    *pos_out = 0;
    return IZG_OK;
  }
  if (nw == 0) return IZG_E_FP_TRUNC_PAGE;
  const uint32_t A = ldg_u32(page);
  if (A < 1 || A >= nw) return IZG_E_FP_BA_OFFSET;
  if (lane == 0) prefetch_l2(page + A, 4u * (nw - A));
  const uint32_t L = ldg_u32(page + A);
  const uint64_t ba_words = ((uint64_t)L + 3) / 4;
  if (A + 1 + ba_words > nw) return IZG_E_FP_TRUNC_BA;
  const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);

  r.begin(page + A + 1, (uint32_t)ba_words);
  uint32_t parsed = 0;
  int32_t st = fp_parse(r, tab, tab_b, L, nblocks, lane, &parsed);
  r.end();
  __syncwarp();  // table written by lane 0 -> visible to all lanes
  if (st) return fp_positions_bad(tab, ba, parsed, lane) ? IZG_E_FP_POS_RANGE : st;

  uint32_t dir_base, dir_n, end = 0;
  st = fp_directory(page, nw, A + 1 + ba_words, lane, &dir_base, &dir_n, &end);
  if (st) return fp_positions_bad(tab, ba, nblocks, lane) ? IZG_E_FP_POS_RANGE : st;

  r.begin(page + 1, A - 1);
  bool bad_pos = false;
  st = fp_blocks<DELTA>(r, os, tab, tab_b, prm, page, A, nblocks, dir_base, dir_n, out, oal,
                        orow, carry, &bad_pos);
  r.end();
  if (st) return fp_positions_bad(tab, ba, nblocks, lane) ? IZG_E_FP_POS_RANGE : st;
  if (bad_pos) return IZG_E_FP_POS_RANGE;
  *pos_out = end;
  return IZG_OK;
}

}  // namespace izg
