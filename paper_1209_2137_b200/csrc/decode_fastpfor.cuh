// decode_fastpfor.cuh — one warp decodes one SIMD-FastPFOR page.
//
// Restates FastPforCodec::decode_deltas for PatchStorage::vertical_arrays
// (codec_patched.cpp:292-417) fused with the prefix sum, in three phases:
//
//   1. byte array (codec_patched.cpp:309-336): streamed through the warp's
//      TMA ring and walked in 128-byte windows (one shuffle per entry on the
//      serial chain; checks lane-parallel, in the reference's order).  Each
//      block's entry goes to a 32-bit shared table word {b : 6, w : 6, c : 8}
//      (w = maxbits - b); byte-array offsets, packed offsets and per-width
//      cursors are running sums rebuilt four blocks at a time in phase 3
//      (lane w-1 keeps width w's count).  Positions are checked when the
//      patch reads them; fp_positions_bad() settles precedence on error paths.
//   2. exception directory (codec_patched.cpp:346-379): at most 32 dependent
//      loads from L2 (the page tail was bulk-prefetched into L2 up front);
//      array w's base word and count go to the warp's shared scratch.  Arrays are NOT
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
// Coherent (non-.nc) loads for the patch loop: with ld.global.nc there, the
// indexed scalar-array FastPFOR kernel faulted ("misaligned address") on
// every page with exceptions although every address is 4-byte aligned, and
// the fault vanished with any change to the loop (printf, no inlining, no
// shared-memory ORs); plain ld.global is immune and costs nothing here.
__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p) {
#ifdef IZG_PATCH_LDG  // sanitizer repro builds only
  return __ldg(p);
#endif
  uint32_t v;
  asm("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_u8(const uint8_t* p) {
#ifdef IZG_PATCH_LDG
  return __ldg(p);
#endif
  uint32_t v;
  asm("ld.global.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_u8(const uint8_t* p) { return __ldg(p); }

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
                 : "memory");
}

// Per-warp scratch of the SIMD-FastPFOR decoder (shared memory).
struct __align__(16) FpScratch {
  uint32_t tab[512];       // per block: b | w << 6 | c << 12 (w = maxbits - b)
  uint32_t win[128];       // fp_parse: per window byte, len | len2 << 16
  uint32_t dir_base[33];   // by width w = 1..32
  uint32_t dir_n[33];
};

// Phase 1.  Walk of the byte array (codec_patched.cpp:309-336) in 128-byte
// windows.  Lane l decodes window bytes 4l..4l+3 as speculative entry starts:
// len (2, or 3 + c when maxbits > b) and len2 = len + the len of the entry
// that would follow (0 when that entry's header is not inside the window).
// The serial chain of entry starts then reads one broadcast word from the
// warp's window table per TWO entries; up to 32 entries of a window are
// validated and tabulated lane-parallel, and the first failing entry (in
// order) ends the walk with the reference's status.  *parsed = entries that
// passed.
static __device__ int32_t fp_parse(WarpRing& r, FpScratch& sc, uint64_t L, uint32_t nblocks, int lane,
                            uint32_t* parsed) {
  const uint32_t Lc = L > 0x7FFFFFF0ull ? 0x7FFFFFF0u : (uint32_t)L;
  uint32_t s = 0;   // next entry start (byte offset in the byte array)
  uint32_t k0 = 0;  // entries tabulated so far
  while (k0 < nblocks) {
    const uint32_t W = s & ~3u;
    r.release_below(W);
    r.ensure(W + 128);
    const uint32_t word = lds32(r.base + ((r.ring_off() + W + 4u * lane) & kRingMask));
    const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, word, 1);
    uint32_t len[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t x = funnel_r(word, nxt, 8 * k);
      const uint32_t b = x & 0xFFu, mb = (x >> 8) & 0xFFu, c = (x >> 16) & 0xFFu;
      len[k] = mb > b ? 3 + c : 2;
    }
    __syncwarp();  // previous window's chain is done with sc.win
    reinterpret_cast<uint4*>(sc.win)[lane] = make_uint4(len[0], len[1], len[2], len[3]);
    __syncwarp();
    uint32_t pair[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t d2 = 4u * lane + k + len[k];  // the following entry's start
      const uint32_t l2 = d2 <= 125 ? sc.win[d2] : 0u;
      pair[k] = len[k] | (l2 ? len[k] + l2 : 0u) << 16;
    }
    __syncwarp();
    reinterpret_cast<uint4*>(sc.win)[lane] = make_uint4(pair[0], pair[1], pair[2], pair[3]);
    __syncwarp();
    // serial chain of starts inside the window (uniform), two entries a step
    uint32_t m = 0, mystart = 0;
    const uint32_t cap = min(32u, nblocks - k0);
    while (m < cap && s <= W + 125) {
      const uint32_t v = sc.win[s - W];
      const uint32_t l1 = v & 0xFFFFu, l2 = v >> 16;
      if ((uint32_t)lane == m) mystart = s;
      const bool two = l2 != 0 && m + 1 < cap;
      if (two && (uint32_t)lane == m + 1) mystart = s + l1;
      s += two ? l2 : l1;
      m += two ? 2u : 1u;
    }
    // lane-parallel checks of entries k0 .. k0+m-1, in the reference's order
    int32_t code = IZG_OK;
    uint32_t b = 0, mb = 0, c = 0;
    if ((uint32_t)lane < m) {
      const uint32_t a = r.ring_off() + mystart;
      b = lds8(r.base + (a & kRingMask));
      mb = lds8(r.base + ((a + 1) & kRingMask));
      c = lds8(r.base + ((a + 2) & kRingMask));
      const bool exc = mb > b;
      if (mystart + 2 > Lc) code = IZG_E_FP_TRUNC_META;
      else if (b > 32 || mb > 32 || b > mb) code = IZG_E_FP_WIDTHS;
      else if (exc && mystart + 2 >= Lc) code = IZG_E_FP_TRUNC_META;
      else if (exc && c == 0) code = IZG_E_FP_EMPTY_EXC;
      else if (exc && mystart + 3 + c > Lc) code = IZG_E_FP_TRUNC_POS;
      else
        sc.tab[k0 + lane] = exc ? b | ((mb - b) << 6) | (c << 12) : b;
    }
    const uint32_t badm = __ballot_sync(0xFFFFFFFFu, code != IZG_OK);
    if (badm) {
      const int f = __ffs(badm) - 1;
      *parsed = k0 + f;
      return __shfl_sync(0xFFFFFFFFu, code, f);
    }
    k0 += m;
  }
  *parsed = k0;
  if (s != L) return IZG_E_FP_BA_LEN;
  return IZG_OK;
}

// Slow path for error statuses: does any exception position of blocks
// [0, nb) reach 128 (codec_patched.cpp:328-330)?  The reference validates
// every position during its byte-array walk, before any later check.
static __device__ bool fp_positions_bad(const FpScratch& sc, const uint8_t* ba, uint32_t nb, int lane) {
  bool bad = false;
  uint32_t bp = 0;  // entry start in the byte array
  for (uint32_t k = 0; k < nb; ++k) {
    const uint32_t e = sc.tab[k], c = e >> 12;
    if (c)
      for (uint32_t i = lane; i < c; i += 32) bad |= ldg_u8(ba + bp + 3 + i) >= 128u;
    bp += c ? 3 + c : 2;
  }
  return __any_sync(0xFFFFFFFFu, bad);
}

// Patch storage of the exception highs (codec_patched.cpp:195-199).
enum { kVertical = 0, kScalar = 1, kSimple8b = 2 };

// ---- Simple-8b exception highs (SimplePFOR) ------------------------------
// One stream of 64-bit words (low half first) after the byte array
// (codec_patched.cpp:284-287, 342-345); selector = low 4 bits, then
// cap(sel) values of bits(sel) bits each (codec_basic.h:45-60); zero-run
// selectors 0/1 code 240/120 zeros; values truncate to 32 bits
// (simple8b_decode's 32-bit overload, codec_basic.cpp:227-300).
__device__ __forceinline__ uint32_t s8_cap(uint32_t sel) {
  const uint64_t lo = 0x0A0C0F141E3C78F0ull;  // sel 0..7: 240,120,60,30,20,15,12,10
  const uint64_t hi = 0x0102030405060708ull;  // sel 8..15: 8,7,6,5,4,3,2,1
  return (uint32_t)((sel < 8 ? lo : hi) >> (8 * (sel & 7))) & 0xFFu;
}
__device__ __forceinline__ uint32_t s8_bits(uint32_t sel) {
  const uint64_t lo = 0x0605040302010000ull;  // sel 0..7: 0,0,1,2,3,4,5,6
  const uint64_t hi = 0x3C1E140F0C0A0807ull;  // sel 8..15: 7,8,10,12,15,20,30,60
  return (uint32_t)((sel < 8 ? lo : hi) >> (8 * (sel & 7))) & 0xFFu;
}

// simple8b_decode's bounds walk (codec_basic.cpp:296-305) over `T` values
// from page word `pos`, 32 words per step: *end = first word after the last
// word needed, or IZG_E_S8_EXHAUSTED when the page ends first.
static __device__ int32_t s8_scan(const uint32_t* page, uint32_t nw, uint32_t pos, uint32_t T, int lane,
                           uint32_t* end) {
  if (T == 0) {
    *end = pos;
    return IZG_OK;
  }
  uint32_t done = 0;
  for (uint64_t k = 0;; k += 32) {
    const uint64_t at = pos + 2 * (k + lane);
    const bool valid = at + 2 <= nw;
    const uint32_t cnt = valid ? s8_cap(ldg_u32(page + at) & 15u) : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    const uint32_t hit = __ballot_sync(0xFFFFFFFFu, valid && done + incl >= T);
    const uint32_t inv = __ballot_sync(0xFFFFFFFFu, !valid);
    if (hit && (!inv || __ffs(hit) < __ffs(inv))) {
      *end = (uint32_t)(pos + 2 * (k + __ffs(hit)));
      return IZG_OK;
    }
    if (inv) return IZG_E_S8_EXHAUSTED;
    done += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
}

// Window of 32 Simple-8b words (lane l holds word wk+l: halves and the value
// index of its first value) over the stream at page word `pos`.
struct S8Window {
  uint32_t pos, nw;
  uint32_t wk;     // stream word index of lane 0's word
  uint32_t lo, hi, start, cnt, total;
  __device__ __forceinline__ void load(const uint32_t* page, uint32_t k, uint32_t v0, int lane) {
    wk = k;
    const uint64_t at = pos + 2 * ((uint64_t)k + lane);
    const bool valid = at + 2 <= nw;
    lo = valid ? ldg_u32(page + at) : 0u;
    hi = valid ? ldg_u32(page + at + 1) : 0u;
    cnt = valid ? s8_cap(lo & 15u) : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += y;
    }
    start = v0 + incl - cnt;
    total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  // Re-centre so that lane 0's word holds value e (e >= start of lane 0).
  __device__ __forceinline__ void seek(const uint32_t* page, uint32_t e, int lane) {
    uint32_t v0 = __shfl_sync(0xFFFFFFFFu, start, 0);
    while (e >= v0 + total) {
      load(page, wk + 32, v0 + total, lane);
      v0 = __shfl_sync(0xFFFFFFFFu, start, 0);
    }
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, start <= e && cnt);
    const uint32_t l0 = m ? 31 - __clz(m) : 0u;
    if (l0) load(page, wk + l0, __shfl_sync(0xFFFFFFFFu, start, l0), lane);
  }
};

// Patch one warp iteration of a SimplePFOR page: its `tot` exceptions are
// values E0 .. E0+tot-1 of the stream, dealt one per lane per round in block
// order (blocks' exception prefixes p1 < p2 < p3 within the iteration).
static __device__ bool fp_patch_s8(uint32_t t, const uint32_t* page, const uint8_t* ba, S8Window& win,
                            uint32_t E0, uint32_t tot, uint32_t myb, uint32_t myc, uint32_t mybp,
                            int lane) {
  const uint32_t p1 = __shfl_sync(0xFFFFFFFFu, myc, 0);
  const uint32_t p2 = p1 + __shfl_sync(0xFFFFFFFFu, myc, 8);
  const uint32_t p3 = p2 + __shfl_sync(0xFFFFFFFFu, myc, 16);
  bool bad = false;
#pragma unroll 1
  for (uint32_t base = 0; base < tot; base += 32) {
    win.seek(page, E0 + base, lane);
    const uint32_t x = base + lane;  // exception index within the iteration
    const bool ok = x < tot;
    const uint32_t e = E0 + x;
    uint32_t l = 0;  // last window word whose first value is <= e
#pragma unroll
    for (uint32_t st = 16; st; st >>= 1) {
      const uint32_t v = __shfl_sync(0xFFFFFFFFu, win.start, (l + st) & 31);
      if (l + st < 32 && v <= e) l += st;
    }
    const uint32_t wlo = __shfl_sync(0xFFFFFFFFu, win.lo, l);
    const uint32_t whi = __shfl_sync(0xFFFFFFFFu, win.hi, l);
    const uint32_t j = e - __shfl_sync(0xFFFFFFFFu, win.start, l);
    const uint32_t q = (x >= p1) + (x >= p2) + (x >= p3);
    const uint32_t b = __shfl_sync(0xFFFFFFFFu, myb, 8 * q);
    const uint32_t bp = __shfl_sync(0xFFFFFFFFu, mybp, 8 * q);
    if (ok) {
      const uint32_t i = x - (q == 0 ? 0u : q == 1 ? p1 : q == 2 ? p2 : p3);
      const uint32_t bits = s8_bits(wlo & 15u);
      const uint64_t word = (uint64_t)whi << 32 | wlo;
      const uint32_t high =
          bits ? (uint32_t)((word >> (4 + j * bits)) & ((1ull << bits) - 1)) : 0u;
      const uint32_t pp = ld_u8(ba + bp + i);
      if (pp >= 128u)
        bad = true;
      else if (high)
        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(OutStage::swz(t, 128u * q + pp)),
                     "r"(high << b));
    }
  }
  return bad;
}

// Phase 2.  `pos` = page word after the byte array; *end = words consumed.
// ST = kVertical: 16-byte-aligned vertical groups of 128 (simdfastpfor);
// kScalar: scalar groups of 32, no alignment (fastpfor).
template <int ST>
static __device__ int32_t fp_directory(FpScratch& sc, const uint32_t* page, uint32_t nw, uint64_t pos,
                                int lane, uint32_t* end) {
  sc.dir_n[lane + 1] = 0;
  sc.dir_base[lane + 1] = 0;
  if (lane == 0) sc.dir_base[0] = 0;  // width 0 (no exceptions): the page start
  __syncwarp();
  if (pos >= nw) return IZG_E_FP_NO_BITSET;
  uint32_t bits = ldg_u32(page + pos);
  ++pos;
  while (bits) {
    const uint32_t w = __ffs(bits);  // width w <-> bit w-1
    bits &= bits - 1;
    if (pos >= nw) return IZG_E_FP_TRUNC_EXC;
    const uint32_t n = ldg_u32(page + pos);
    uint64_t nwords;
    if (ST == kVertical) {
      pos = (pos + 1 + 3) & ~uint64_t{3};  // 16-byte alignment in the page
      nwords = ((uint64_t)n + 127) / 128 * 4 * w;
    } else {
      pos = pos + 1;
      nwords = ((uint64_t)n + 31) / 32 * w;
    }
    if (pos + nwords > nw) return IZG_E_FP_TRUNC_EXC;
    if (lane == 0) {
      sc.dir_base[w] = (uint32_t)pos;
      sc.dir_n[w] = n;
    }
    pos += nwords;
  }
  __syncwarp();
  *end = (uint32_t)pos;
  return IZG_OK;
}

// Patch one warp iteration's exceptions into its output tile `t`
// (codec_patched.cpp:390-404: o[pos] |= high << b).  Lanes 8q..8q+7 carry
// block q's parameters (b, exception width w, count c, first position byte
// bp in the byte array, cursor cur in array w, array base word) and patch
// block q, sixteen exceptions per round with every load issued before the
// first OR; the round count is set by the longest of the four lists.
// Duplicate positions OR together like the reference.  Returns true when a
// position >= 128 was met (the caller resolves precedence).
#ifndef IZG_PATCH_SLOTS
#define IZG_PATCH_SLOTS 2  // exceptions per lane per round (8 lanes per block)
#endif
// Lean patch (vertical arrays of SIMD-FastPFOR, scalar arrays of FastPFOR):
// every address is formed from a valid base, so no slot needs a select on
// its addresses — an idle slot (e >= c)
// re-reads the block's exception 0, and a block without exceptions reads
// width 0's base, which callers set to 0 (dir_base[0] = 0) — and the tile
// address of position p in block q is built from per-lane constants (the
// 128-byte swizzle's row parity depends only on q and p >> 5).
#ifndef IZG_PATCH_LEAN
#define IZG_PATCH_LEAN 1
#endif
template <int ST>
__device__ __forceinline__ bool fp_patch_lean(uint32_t t, const uint32_t* page,
                                              const uint8_t* ba, uint32_t myb, uint32_t myw,
                                              uint32_t myc, uint32_t mybp, uint32_t mycur,
                                              uint32_t mybase, int lane, uint32_t nw = 0,
                                              uint32_t chunk = 0) {
  (void)nw;
  (void)chunk;
  const uint32_t q = (lane >> 3) & 3u, s8 = lane & 7;
  uint32_t mxc = max(myc, __shfl_xor_sync(0xFFFFFFFFu, myc, 8));
  mxc = max(mxc, __shfl_xor_sync(0xFFFFFFFFu, mxc, 16));
  const uint32_t wmask = low_mask(myw), w4 = 4u * myw;
  const uint32_t* arr = page + mybase;
  const uint8_t* pb = ba + mybp;
  const uint32_t tq = t + (q << 9), rq = (q & 1u) << 2;
  bool bad = false;
  for (uint32_t e0 = s8; e0 < mxc; e0 += 8 * IZG_PATCH_SLOTS) {
    uint32_t pp[IZG_PATCH_SLOTS], lo[IZG_PATCH_SLOTS], hi[IZG_PATCH_SLOTS], sh[IZG_PATCH_SLOTS];
    bool ok[IZG_PATCH_SLOTS];
#pragma unroll
    for (int j = 0; j < IZG_PATCH_SLOTS; ++j) {
      const uint32_t e = e0 + 8u * j;
      ok[j] = e < myc;
      const uint32_t rr = mycur + (ok[j] ? e : 0u);
      uint32_t word, step;
      if (ST == kVertical) {  // group r/128, lane r%4, slot (r%128)/4
        const uint32_t tt = rr & 127u, bit = (tt >> 2) * myw;
        word = (rr >> 7) * w4 + 4u * (bit >> 5) + (tt & 3u);
        sh[j] = bit & 31u;
        step = 4u;
      } else {  // group r/32, bits [(r%32)*w, +w) of its w-word stream
        const uint32_t bit = (rr & 31u) * myw;
        word = (rr >> 5) * myw + (bit >> 5);
        sh[j] = bit & 31u;
        step = 1u;
      }
      IZG_CHECK(!nw || !ok[j] || izg_in_span(reinterpret_cast<uintptr_t>(pb + e), 1, page, nw), 6,
                chunk, e);
      IZG_CHECK(!nw || (izg_in_span(reinterpret_cast<uintptr_t>(arr + word), 4, page, nw) &&
                        izg_in_span(reinterpret_cast<uintptr_t>(
                                        arr + word + (sh[j] + myw > 32 ? step : 0u)), 4, page, nw)),
                7, chunk, word);
      pp[j] = ok[j] ? ld_u8(pb + e) : 0u;
      lo[j] = ld_u32(arr + word);
      hi[j] = ld_u32(arr + word + (sh[j] + myw > 32 ? step : 0u));
    }
#pragma unroll
    for (int j = 0; j < IZG_PATCH_SLOTS; ++j) {
      if (ok[j]) {
        const uint32_t p = pp[j];
        if (p < 128u) {
          const uint32_t hv = (funnel_r(lo[j], hi[j], sh[j]) & wmask) << myb;
          const uint32_t r = p >> 5;
          const uint32_t a = tq + (r << 7) + (((((p >> 2) & 7u) ^ (rq + r))) << 4) + ((p & 3u) << 2);
          asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(hv));
        } else {
          bad = true;
        }
      }
    }
  }
  return bad;
}

template <int ST>
__device__ __forceinline__ bool fp_patch(uint32_t t, const uint32_t* page, const uint8_t* ba,
                                         uint32_t myb, uint32_t myw, uint32_t myc, uint32_t mybp,
                                         uint32_t mycur, uint32_t mybase, int lane, uint32_t nw = 0,
                                         uint32_t chunk = 0) {
#if IZG_PATCH_LEAN
  return fp_patch_lean<ST>(t, page, ba, myb, myw, myc, mybp, mycur, mybase, lane, nw, chunk);
#endif
  const uint32_t q = (lane >> 3) & 3u, s8 = lane & 7;
  uint32_t mxc = max(myc, __shfl_xor_sync(0xFFFFFFFFu, myc, 8));
  mxc = max(mxc, __shfl_xor_sync(0xFFFFFFFFu, mxc, 16));
  const uint32_t wmask = low_mask(myw), w4 = 4u * myw;
  bool bad = false;
  for (uint32_t e0 = s8; e0 < mxc; e0 += 8 * IZG_PATCH_SLOTS) {
    uint32_t pp[IZG_PATCH_SLOTS], lo[IZG_PATCH_SLOTS], hi[IZG_PATCH_SLOTS], sh[IZG_PATCH_SLOTS];
    bool ok[IZG_PATCH_SLOTS];
#pragma unroll
    for (int j = 0; j < IZG_PATCH_SLOTS; ++j) {
      const uint32_t e = e0 + 8u * j;
      ok[j] = e < myc;
      const uint32_t ee = ok[j] ? e : 0u;
      const uint32_t rr = mycur + ee;
      uint32_t word, step;
      if (ST == kVertical) {  // group r/128, lane r%4, slot (r%128)/4
        const uint32_t tt = rr & 127u, bit = (tt >> 2) * myw;
        word = mybase + (rr >> 7) * w4 + 4u * (bit >> 5) + (tt & 3u);
        sh[j] = bit & 31u;
        step = 4u;
      } else {  // group r/32, bits [(r%32)*w, +w) of its w-word stream
        const uint32_t bit = (rr & 31u) * myw;
        word = mybase + (rr >> 5) * myw + (bit >> 5);
        sh[j] = bit & 31u;
        step = 1u;
      }
      // an idle slot reads the page's first words (always in bounds)
      pp[j] = ok[j] ? ld_u8(ba + mybp + ee) : 0u;
      lo[j] = ld_u32(page + (ok[j] ? word : 0u));
      hi[j] = ld_u32(page + (ok[j] ? word + (sh[j] + myw > 32 ? step : 0u) : 0u));
    }
#pragma unroll
    for (int j = 0; j < IZG_PATCH_SLOTS; ++j) {
      if (ok[j]) {
        const uint32_t high = funnel_r(lo[j], hi[j], sh[j]) & wmask;
        if (pp[j] < 128u)
          asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(OutStage::swz(t, 128u * q + pp[j])),
                       "r"(high << myb));
        else
          bad = true;
      }
    }
  }
  return bad;
}

// Phase 3.  Returns an izg_status; *bad_pos is set when a position >= 128
// was met (the caller resolves precedence).
// SimplePFOR (ST == kSimple8b): exceptions are consumed in block order from
// one stream starting at page word `s8pos` (nw = page words), so a block's
// cursor is the running exception count and there is no exhaustion check.
template <int DELTA, int ST, typename OS>
__device__ int32_t fp_blocks(WarpRing& r, OS& os, FpScratch& sc, const uint32_t* page,
                             uint32_t A, uint32_t nblocks, uint32_t* out, bool oal, int64_t orow,
                             uint4& carry, bool* bad_pos, uint32_t s8pos = 0, uint32_t nw = 0) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);
  uint32_t packed = 1;  // page word of the next block's payload
  uint32_t bpos = 0;    // byte-array offset of the next block's entry
  uint32_t used = 0;    // lane w-1: exceptions consumed from array w
  uint32_t E = 0;       // SimplePFOR: exceptions consumed so far
  S8Window win;
  if (ST == kSimple8b) {
    win.pos = s8pos;
    win.nw = nw;
    win.load(page, 0, 0, lane);
  }
  bool bad = false;
#pragma unroll 1
  for (uint32_t g0 = 0; g0 < nblocks; g0 += 4) {
    const uint32_t ng = min(4u, nblocks - g0);
    // Lanes 0..3 own blocks g0..g0+3: fields, running sums over the four
    // blocks (packed words, exceptions), checks, exception parameters.
    uint32_t b = 0, c = 0, w = 0;
    if ((uint32_t)lane < ng) {
      const uint32_t e = sc.tab[g0 + lane];
      b = e & 63u;
      w = (e >> 6) & 63u;
      c = e >> 12;
    }
    // cursor of each block in its width array: the lane-distributed running
    // count (lane w-1) plus earlier same-width blocks of this iteration
    uint32_t acc = 0, add = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t wc = __shfl_sync(0xFFFFFFFFu, w | c << 8, j);
      const uint32_t wj = wc & 0xFFu, cj = wc >> 8;
      if (j < lane && wj == w) acc += cj;
      if (cj && wj == (uint32_t)lane + 1) add += cj;
    }
    const uint32_t cur = __shfl_sync(0xFFFFFFFFu, used, (w - 1) & 31) + acc;
    used += add;
    // inclusive scans over lanes 0..3: packed words, exceptions, entry bytes
    uint32_t pk = 4u * b, ce = c, bl = (uint32_t)lane < ng ? (c ? 3 + c : 2) : 0u;
#pragma unroll
    for (int d = 1; d < 4; d <<= 1) {
      const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, pk, d, 4);
      const uint32_t y1 = __shfl_up_sync(0xFFFFFFFFu, ce, d, 4);
      const uint32_t y2 = __shfl_up_sync(0xFFFFFFFFu, bl, d, 4);
      if ((lane & 3) >= d) {
        pk += y0;
        ce += y1;
        bl += y2;
      }
    }
    const uint32_t bp = bpos + bl - (c ? c : 0u);  // this block's first position byte
    const uint32_t pk_ex = pk - 4u * b;
    // codec_patched.cpp:387-388 then 406-407, block by block
    const bool ov = (uint32_t)lane < ng && packed + pk > A;
    const bool ex = ST != kSimple8b && c && cur + c > sc.dir_n[w];
    const uint32_t em = __ballot_sync(0xFFFFFFFFu, ov || ex) & 0xFu;
    if (em) {
      const int k = __ffs(em) - 1;
      return (__ballot_sync(0xFFFFFFFFu, ov) >> k) & 1u ? IZG_E_FP_OVERRUN : IZG_E_FP_EXHAUSTED;
    }
    // per-lane view of its own block q (lanes 8q..8q+7 patch block q)
    const uint32_t myb = __shfl_sync(0xFFFFFFFFu, b, q);
    const uint32_t myoff = packed + __shfl_sync(0xFFFFFFFFu, pk_ex, q);
    const uint32_t myc = __shfl_sync(0xFFFFFFFFu, c, q);
    const uint32_t myw = __shfl_sync(0xFFFFFFFFu, w, q);
    const uint32_t mybp = __shfl_sync(0xFFFFFFFFu, bp, q);
    const uint32_t mycur = __shfl_sync(0xFFFFFFFFu, cur, q);
    const uint32_t mybase = ST == kSimple8b ? 0u : sc.dir_base[myw];
    const uint32_t first = packed;
    packed += __shfl_sync(0xFFFFFFFFu, pk, 3);
    bpos += __shfl_sync(0xFFFFFFFFu, bl, 3);
    const uint32_t tot = __shfl_sync(0xFFFFFFFFu, ce, 3);
    const uint32_t E0 = E;  // SimplePFOR: first stream value of this iteration
    E += tot;

    // Stream window: packed words [first, packed) (the stream starts at word 1).
    r.release_below(4u * (first - 1));
    r.ensure(4u * (packed - 1));
    const bool live = q < ng;
    uint32_t v[4][4];
    if (ST != kVertical)
      unpack_scalar_slots(r, myoff - 1, myb, s8, v);
    else if (r.phase == 0)
      unpack_slots_aligned(r, r.ring_off() + 4u * (myoff - 1), myb, s8, v);
    else
      unpack_slots_unaligned(r, myoff - 1, myb, s8, v);
    if (tot) {
      // Patch through the warp's output tile (swizzled; see OutStage).
      const uint32_t t = os.acquire();
      OutStage::write(t, v, lane);
      __syncwarp();

      if (ST == kSimple8b)
        bad |= fp_patch_s8(t, page, ba, win, E0, tot, myb, myc, mybp, lane);
      else
        bad |= fp_patch<ST>(t, page, ba, myb, myw, myc, mybp, mycur, mybase, lane);
      __syncwarp();
      OutStage::read(t, v, lane);
      scan<DELTA>(v, carry, lane);
      if (orow >= 0 && ng == 4) {
        os.commit(v, lane, (uint32_t)(orow + 4 * g0));
      } else {
        os.abandon();
        os.direct(v, out + (size_t)(g0 + q) * 128 + 16 * s8, oal, live, 128u * ng, lane);
      }
    } else {
      scan<DELTA>(v, carry, lane);
      if (orow >= 0 && ng == 4)
        os.put(v, lane, (uint32_t)(orow + 4 * g0));
      else
        os.direct(v, out + (size_t)(g0 + q) * 128 + 16 * s8, oal, live, 128u * ng, lane);
    }
  }
  *bad_pos = __any_sync(0xFFFFFFFFu, bad);
  if (packed != A) return IZG_E_FP_PACKED_SIZE;
  return IZG_OK;
}

// Whole page.  `nblocks` = count / 128; *pos_out = words consumed.
template <int DELTA, int ST, typename OS>
__device__ int32_t fastpfor_core(WarpRing& r, OS& os, FpScratch& sc, const uint32_t* page,
                                 uint32_t nw, uint32_t nblocks, uint32_t* out, bool oal,
                                 int64_t orow, uint4& carry, uint32_t* pos_out) {
  const int lane = threadIdx.x & 31;
  if (nblocks == 0) {  // decode_deltas(count == 0) reads nothing (codec_patched.cpp:295)
    *pos_out = 0;
    return IZG_OK;
  }
  if (nw == 0) return IZG_E_FP_TRUNC_PAGE;
  const uint32_t A = ldg_u32(page);
  if (A < 1 || A >= nw) return IZG_E_FP_BA_OFFSET;
  const uint32_t L = ldg_u32(page + A);
  const uint64_t ba_words = ((uint64_t)L + 3) / 4;
  if (A + 1 + ba_words > nw) return IZG_E_FP_TRUNC_BA;
  const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);

  const uint64_t keep = r.policy;
  r.policy = policy_evict_last();  // the patch re-reads the position bytes
  r.begin(page + A + 1, (uint32_t)ba_words);
  uint32_t parsed = 0;
  int32_t st = fp_parse(r, sc, L, nblocks, lane, &parsed);
  r.end();
  r.policy = keep;
  __syncwarp();  // table written by lane 0 -> visible to all lanes
  if (st) return fp_positions_bad(sc, ba, parsed, lane) ? IZG_E_FP_POS_RANGE : st;

  uint32_t end = 0;
  if (ST == kSimple8b) {
    // simple8b_decode of all the page's highs up front (codec_patched.cpp:342-345)
    uint32_t T = 0;
    for (uint32_t k = lane; k < nblocks; k += 32) T += sc.tab[k] >> 12;
#pragma unroll
    for (int d = 16; d; d >>= 1) T += __shfl_xor_sync(0xFFFFFFFFu, T, d);
    st = s8_scan(page, nw, A + 1 + (uint32_t)ba_words, T, lane, &end);
  } else {
    st = fp_directory<ST>(sc, page, nw, A + 1 + ba_words, lane, &end);
  }
  if (st) return fp_positions_bad(sc, ba, nblocks, lane) ? IZG_E_FP_POS_RANGE : st;

  // exception arrays: warm L2 while the packed area streams
  if (lane == 0) {
    const uint32_t x0 = A + 1 + (uint32_t)ba_words;
    prefetch_l2(page + x0, 4u * (end - x0));
  }
  r.begin(page + 1, A - 1);
  bool bad_pos = false;
  st = fp_blocks<DELTA, ST>(r, os, sc, page, A, nblocks, out, oal, orow, carry, &bad_pos,
                            A + 1 + (uint32_t)ba_words, nw);
  r.end();
  if (st) return fp_positions_bad(sc, ba, nblocks, lane) ? IZG_E_FP_POS_RANGE : st;
  if (bad_pos) return IZG_E_FP_POS_RANGE;
  *pos_out = end;
  return IZG_OK;
}

}  // namespace izg
