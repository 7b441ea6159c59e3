// team.cuh — SIMD-FastPFOR decode with one CTA (a "team": 8 decoding warps
// and a staging warp) per page, from the records of the page index pass
// (index_fastpfor.cuh).  DESIGN.md 3 has the measurements and the history.
//
// The warp-per-page decode (decode_fastpfor.cuh / index_fastpfor.cuh) runs a
// staging ring per warp and fetches every exception with two scattered global
// loads plus the address arithmetic of the vertical layout, and a batch of a
// few thousand pages leaves most of its warp slots empty.  Here a page is
// decoded in super-iterations of 32 blocks (4,096 integers), one warp
// iteration of 4 blocks per decoding warp:
//
//   * the staging warp is the front end, ahead of the decoders.  It claims
//     pages, settles the ones that need no decode, publishes a descriptor
//     per page, and feeds two in-order streams of TMA bulk copies: (a) per
//     super-iteration the packed words, the 32 block records and the
//     position bytes, into linear staging buffers (one mbarrier per slot,
//     four slots); (b) per exception WINDOW the packed exception arrays
//     (codec_patched.cpp:346-379), one copy per width: the page index pass
//     records every width's cursor at each 32-block boundary
//     (IdxView::snap), and a window is the longest run of super-iterations
//     whose groups fit half of the buffer;
//   * a decoding warp waits for its slot, unpacks its four blocks from the
//     staging buffer, and patches in its output tile with the position byte
//     and the exception high both read from shared memory
//     (codec_patched.cpp:390-404: o[pos] |= high << b);
//   * the prefix sum is a carry chain: each warp scans its 512 integers from
//     a zero carry, takes the running prefix from its mailbox, posts prefix +
//     own total to the next warp's, adds the prefix and stores the tile with
//     TMA (delta.cpp:60-75 for D4; the same split for D1 / D2 / DM).
//
// No CTA barrier after initialisation: pages, windows, slots and mailboxes
// are all handed over through mbarriers.  Everything the index pass checked
// stays checked there; exception positions >= 128 are detected while
// patching (codec_patched.cpp:328-330), as in the warp-per-page kernels.
// What does not fit the staged paths (a super-iteration with over 5 KiB of
// position bytes, a window that does not fit even for one super-iteration,
// cursors past 65,535, packed rows that are not 16-byte aligned) is patched
// from global memory with fp_patch / unpacked with word loads inside the
// same kernel: same results (tests/test_gpu_team.py).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "decode_kernel.cuh"

namespace izg {

constexpr int kTeamWarps = 8;
constexpr uint32_t kTeamSI = 4 * kTeamWarps;  // blocks per super-iteration
#ifndef IZG_TEAM_SLOTS
#define IZG_TEAM_SLOTS 4
#endif
constexpr uint32_t kTeamSlots = IZG_TEAM_SLOTS;  // super-iterations staged ahead
#ifndef IZG_TEAM_PK
#define IZG_TEAM_PK 16896
#endif
#ifndef IZG_TEAM_XB
#define IZG_TEAM_XB 14336  // per window; two windows (8 KiB: C4 10 % 0.372 ms, 1 % 0.235; 14 KiB: 0.360, 0.222; C5 equal)
#endif
constexpr uint32_t kTeamPk = IZG_TEAM_PK;     // packed words staging (>= 16 KiB + 16)
constexpr uint32_t kTeamPs = 5 * 1024;        // position bytes staging
constexpr uint32_t kTeamXb = IZG_TEAM_XB;     // packed exception arrays of a window
#ifndef IZG_TEAM_UNPACK
#define IZG_TEAM_UNPACK team_unpack_window  // or team_unpack_rows (more row loads, fewer moves)
#endif
#ifndef IZG_TEAM_NARROW
#define IZG_TEAM_NARROW 1  // separate unpack for iterations whose four widths are all <= 8
#endif
#ifndef IZG_TEAM_IDLE_NS
#define IZG_TEAM_IDLE_NS 64  // staging warp: sleep after a pass without progress
#endif
#ifndef IZG_TEAM_MINCTAS
#define IZG_TEAM_MINCTAS 3  // CTAs per SM the register allocation allows for
#endif
constexpr int kTeamThreads = (kTeamWarps + 1) * 32;  // 8 decoding warps + the staging warp
#define IZG_TEAM_LB_THREADS ((kTeamWarps + 1) * 32)

#ifdef IZG_TEAM_PROF  // developer build: where a page's time goes (cycles, summed over pages)
// decoding warp 0, cycles: [0] pages, [1] waits for a page descriptor, [2] for an exception
// window, [3] for staged data, [4] for the carry mailbox, [5] whole pages; staging warp:
// [6] passes without progress
__device__ unsigned long long g_team_prof[8];
#define TEAM_PROF_T(x) const long long x = clock64()
#define TEAM_PROF_ADD(i, v) atomicAdd(&g_team_prof[i], (unsigned long long)(v))
#else
#define TEAM_PROF_T(x)
#define TEAM_PROF_ADD(i, v)
#endif

struct TeamLayout {
  static constexpr uint32_t kTiles = 0;  // one 2 KiB output tile per decoding warp (1024-aligned)
  static constexpr uint32_t kPk = kTiles + kTeamWarps * kStageOut;  // packed words staging
  static constexpr uint32_t kPs = kPk + kTeamPk;                    // position bytes staging
  static constexpr uint32_t kRec = kPs + kTeamPs;                   // block records [slots][32]
  static constexpr uint32_t kXb = kRec + kTeamSlots * kTeamSI * 16; // exception highs, two windows
  // staging warp's page contexts [2]: bounds P[20], S[20], array bases [32], scalars [24],
  // cursor snapshots u16 [16][32]
  static constexpr uint32_t kCtxBytes = (20 + 20 + 32 + 24) * 4 + 1024;
  static constexpr uint32_t kCtx = kXb + 2 * kTeamXb;
  // per window, per width: {shared address of the first staged group, its first value's index}
  static constexpr uint32_t kXrel = kCtx + 2 * kCtxBytes;  // uint2 [2][36]
  static constexpr uint32_t kDirb = kXrel + 2 * 36 * 8;   // u32 [2][36]: per page, array base word
  static constexpr uint32_t kTot = kDirb + 2 * 36 * 4;    // uint4 [warps]: carry mailboxes
  static constexpr uint32_t kDesc = kTot + kTeamWarps * 16;        // u32 [2][16]: page descriptors
  static constexpr uint32_t kXinfo = kDesc + 2 * 64;               // uint2 [2] {window end, fast}
  static constexpr uint32_t kInfo = kXinfo + 2 * 8;                // uint2 [slots] {pkrel, psrel}
  static constexpr uint32_t kAlloc = kInfo + kTeamSlots * 8;       // uint2 [slots] {pk off, ps off}
  static constexpr uint32_t kBar = kAlloc + kTeamSlots * 8;        // u64 [slots]: staging landed
  static constexpr uint32_t kEmpty = kBar + kTeamSlots * 8;        // u64 [slots]: staging read by all warps
  static constexpr uint32_t kMbx = kEmpty + kTeamSlots * 8;        // u64 [warps]: mailbox posted
  static constexpr uint32_t kXfull = kMbx + kTeamWarps * 8;        // u64 [2]: window prepared
  static constexpr uint32_t kXempty = kXfull + 16;                 // u64 [2]: window consumed
  static constexpr uint32_t kPfull = kXempty + 16;                 // u64 [2]: descriptor written
  static constexpr uint32_t kPdone = kPfull + 16;                  // u64 [2]: warps 0..6 left the page
  static constexpr uint32_t kPfree = kPdone + 16;                  // u64 [2]: page finished
  static constexpr uint32_t kBad = kPfree + 16;                    // u32 [2]: a position >= 128 was met
  static constexpr size_t kSmem = kBad + 16;
};
static_assert(TeamLayout::kXrel % 16 == 0 && TeamLayout::kTot % 16 == 0 &&
                  TeamLayout::kDesc % 16 == 0 && TeamLayout::kBar % 8 == 0,
              "team layout");
static_assert(IZG_TEAM_MINCTAS * (TeamLayout::kSmem + 1024) <= 228 * 1024, "team shared memory");
static_assert(kTeamPk >= 16384 + 16 && kTeamPk % 16 == 0 && kTeamPs % 16 == 0, "team staging");

// Linear staging: unpack_slots_aligned's "ring" without a wrap.
struct LinBuf {
  static constexpr uint32_t kMask = 0xFFFFFFFFu;
  uint32_t base;
};

__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}

// One warp's 2 KiB output tile in the 128-byte-swizzled layout of OutStageT
// (izg_common.cuh), with the lane's four 16-byte chunk addresses held as two
// registers: integers 16 lane + 4 k .. + 3 (mapping C) live at byte
// ta0 | (16 k ^ tm3) — row lane / 2, chunk (4 (lane & 1) + k) ^ (row & 7).
struct TeamTile {
  uint32_t t;      // shared address of the tile (1024-aligned)
  uint32_t ta0, tm3;
  const void* tmap;
  bool leader;
  __device__ __forceinline__ void init(uint32_t tile, int lane, const void* map) {
    t = tile;
    tmap = map;
    leader = lane == 0;
    const uint32_t m = ((uint32_t)lane >> 1) & 7u;
    ta0 = tile + (((uint32_t)lane >> 1) << 7) + (((4u * ((uint32_t)lane & 1u)) ^ (m & 4u)) << 4);
    tm3 = (m & 3u) << 4;
  }
  __device__ __forceinline__ uint32_t addr(int k) const { return ta0 | ((16u * k) ^ tm3); }
  // the tile's previous TMA store has read it
  __device__ __forceinline__ void wait_free() const {
    if (leader) bulk_wait_read<0>();
    __syncwarp();
  }
  __device__ __forceinline__ void write(const uint32_t (&v)[4][4]) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) sts128(addr(k), v[k][0], v[k][1], v[k][2], v[k][3]);
  }
  __device__ __forceinline__ void read(uint32_t (&v)[4][4]) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 x = lds128(addr(k));
      v[k][0] = x.x; v[k][1] = x.y; v[k][2] = x.z; v[k][3] = x.w;
    }
  }
  // after write(): 16 rows of 32 integers to output row `row`
  __device__ __forceinline__ void store(uint32_t row) const {
    fence_proxy_async_smem();
    __syncwarp();
    if (leader) {
      tma_store_2d(tmap, t, 0, (int)row);
      bulk_commit();
    }
  }
  __device__ __forceinline__ void drain() const {
    if (leader) bulk_wait<0>();
    __syncwarp();
  }
};

// t += (value of lane - d) for lanes >= d: the shuffle's own in-range
// predicate guards the add (no compare, no select).
__device__ __forceinline__ void shfl_up_add(uint32_t& t, uint32_t d) {
  asm volatile(
      "{\n\t.reg .u32 y;\n\t.reg .pred p;\n\t"
      "shfl.sync.up.b32 y|p, %0, %1, 0, 0xffffffff;\n\t"
      "@p add.u32 %0, %0, y;\n\t}"
      : "+r"(t)
      : "r"(d));
}
template <int NC>
__device__ __forceinline__ uint4 team_incl_scan(uint4 t) {
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    shfl_up_add(t.x, d);
    if (NC > 1) shfl_up_add(t.y, d);
    if (NC > 2) shfl_up_add(t.z, d);
    if (NC > 3) shfl_up_add(t.w, d);
  }
  return t;
}

// Unpack the thread's 4 slots x 4 lanes of a block at shared byte address
// `bb` (16-byte aligned rows, linear buffer): two row loads per slot, no
// window to slide (bitpack.cpp:122-143 restated per lane).
__device__ __forceinline__ void team_unpack_rows(uint32_t bb, uint32_t width, uint32_t s8,
                                                 uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
  uint32_t bit = 4u * s8 * width;
#pragma unroll
  for (int c = 0; c < 4; ++c, bit += width) {
    const uint32_t ra = bb + 16u * (bit >> 5), sh = bit & 31u;
    const uint4 lo = lds128(ra);
    const uint4 hi = lds128(ra + 16u);
    v[c][0] = funnel_r(lo.x, hi.x, sh) & mask;
    v[c][1] = funnel_r(lo.y, hi.y, sh) & mask;
    v[c][2] = funnel_r(lo.z, hi.z, sh) & mask;
    v[c][3] = funnel_r(lo.w, hi.w, sh) & mask;
  }
}

// Widths up to 8: the lane's four slots are 4 b <= 32 consecutive bits of each
// vertical lane's stream, inside two rows: one funnel shift per lane brings
// them into a word, then a shift and a mask per value.
__device__ __forceinline__ void team_unpack_narrow(uint32_t bb, uint32_t width, uint32_t s8,
                                                   uint32_t (&v)[4][4]) {
  const uint32_t mask = (1u << width) - 1u;
  const uint32_t bit = 4u * s8 * width;
  const uint32_t ra = bb + 16u * (bit >> 5), sh = bit & 31u;
  const uint4 lo = lds128(ra);
  const uint4 hi = lds128(ra + 16u);
  const uint32_t w0 = funnel_r(lo.x, hi.x, sh), w1 = funnel_r(lo.y, hi.y, sh);
  const uint32_t w2 = funnel_r(lo.z, hi.z, sh), w3 = funnel_r(lo.w, hi.w, sh);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t s = c * width;
    v[c][0] = (w0 >> s) & mask;
    v[c][1] = (w1 >> s) & mask;
    v[c][2] = (w2 >> s) & mask;
    v[c][3] = (w3 >> s) & mask;
  }
}

__device__ __forceinline__ void team_unpack_window(uint32_t bb, uint32_t width, uint32_t s8,
                                                   uint32_t (&v)[4][4]) {
  unpack_slots_aligned(LinBuf{0u}, bb, width, s8, v);
}

// Word-load unpack for pages whose packed rows are not 16-byte aligned
// (unpack_slots_unaligned over a linear buffer): `bw` = shared byte address
// of the block's first word.
__device__ __forceinline__ void team_unpack_words(uint32_t bw, uint32_t width, uint32_t s8,
                                                  uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t bit = (4u * s8 + c) * width;
    const uint32_t a = bw + 16u * (bit >> 5), sh = bit & 31u;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      v[c][j] = funnel_r(lds32(a + 4u * j), lds32(a + 16u + 4u * j), sh) & mask;
  }
}

// Patch one warp iteration from shared memory: lanes 8q..8q+7 patch block q,
// sixteen exceptions per round.  `ps` = shared address of the block's first
// position byte; the block's width-w array is staged packed (vertical
// groups of 128, codec_patched.cpp:346-379) from shared address `xa`, and
// its exceptions are values rc, rc + 1, ... counted from the first staged
// group: value r lies in group r / 128, lane r % 4, slot (r % 128) / 4.
__device__ __forceinline__ bool team_patch(uint32_t t, uint32_t ps, uint32_t xa, uint32_t rc,
                                           uint32_t myw, uint32_t myb, uint32_t myc, int lane) {
  const uint32_t q = (lane >> 3) & 3u, s8 = lane & 7;
  uint32_t mxc = max(myc, __shfl_xor_sync(0xFFFFFFFFu, myc, 8));
  mxc = max(mxc, __shfl_xor_sync(0xFFFFFFFFu, mxc, 16));
  // integer p of block q: tile byte 512 q + (4 p ^ 16 ((row & 7))), row = 4 q + p / 32,
  // i.e. (t + 512 q) ^ 64 (q & 1) ^ (4 p) ^ 16 (p / 32)
  const uint32_t tqr = (t + (q << 9)) ^ ((q & 1u) << 6);
  const uint32_t wmask = low_mask(myw), w16 = 16u * myw;
  uint32_t badp = 0;
  for (uint32_t e0 = s8; e0 < mxc; e0 += 16) {
    uint32_t pp[2], lo[2], hi[2], sh[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t e = e0 + 8u * j;
      pp[j] = 0x100u;  // idle slot: no patch, not a position error
      lo[j] = hi[j] = sh[j] = 0;
      if (e < myc) {
        const uint32_t r = rc + e, tt = r & 127u, bit = (tt >> 2) * myw;
        const uint32_t a = xa + (r >> 7) * w16 + ((bit >> 5) << 4) + ((tt & 3u) << 2);
        sh[j] = bit & 31u;
        pp[j] = lds8(ps + e);
        lo[j] = lds32(a);
        hi[j] = lds32(a + 16u);
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t p = pp[j];
      const uint32_t a = tqr ^ (((p >> 1) & 0x30u) ^ (p << 2));
      const uint32_t hv = (funnel_r(lo[j], hi[j], sh[j]) & wmask) << myb;
      if (p < 128u) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(hv) : "memory");
      badp |= p;  // bit 7: a position in 128..255 (codec_patched.cpp:328-330)
    }
  }
  return (badp & 0x80u) != 0;
}

// First half of the two-level prefix sum: in-thread scan and warp scan of the
// lane totals from a zero carry.  ex = exclusive prefix of the lane totals,
// incl = inclusive (lane 31: the warp total), q3 = DM's lane-3 prefixes.
template <int DELTA>
__device__ __forceinline__ void team_scan_local(uint32_t (&v)[4][4], uint4& ex, uint4& incl,
                                                uint32_t (&q3)[4], int lane) {
  uint4 T = make_uint4(0, 0, 0, 0);
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
  incl = team_incl_scan<NC>(T);
  ex = u4sub(incl, T);
}

// Second half: `base` = page carry + totals of the warps before this one +
// the lane's exclusive prefix.
template <int DELTA>
__device__ __forceinline__ void team_scan_apply(uint32_t (&v)[4][4], const uint4 base,
                                                const uint32_t (&q3)[4]) {
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

// Staging state (the staging warp; lane 0 allocates and issues the copies).
struct TeamProducer {
  uint32_t gi, gd;            // super-iterations staged / read by every warp (all pages)
  uint32_t pk_head, ps_head;  // allocation heads of the two staging buffers
  uint64_t policy;
};

// Wait with a suspend-time hint: the waiting warp sleeps in hardware until
// the phase completes (or the hint expires) instead of re-issuing try_wait.
#ifndef IZG_TEAM_WAIT_NS
#define IZG_TEAM_WAIT_NS 4000
#endif
#ifndef IZG_TEAM_WAIT_SLEEP
#define IZG_TEAM_WAIT_SLEEP 0  // ns slept between polls (0: re-issue try_wait at once)
#endif
__device__ __forceinline__ void team_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
#if IZG_TEAM_WAIT_SLEEP
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@p bra TD_%=;\n\t"
      "TW_%=:\n\t"
      "nanosleep.u32 %3;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TW_%=;\n\t"
      "TD_%=:\n\t}"
      :
      : "r"(bar), "r"(parity), "r"((uint32_t)IZG_TEAM_WAIT_NS), "r"((uint32_t)IZG_TEAM_WAIT_SLEEP)
      : "memory");
#else
      "{\n\t.reg .pred p;\n\t"
      "TW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TW_%=;\n\t}"
      :
      : "r"(bar), "r"(parity), "r"((uint32_t)IZG_TEAM_WAIT_NS)
      : "memory");
#endif
}

__device__ __forceinline__ bool mbar_test_s(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Place `len` bytes in a staging buffer of `size` whose unconsumed data
// spans [tail, head) in allocation order (tail == 0xFFFFFFFF: nothing in
// flight).  A placement never wraps.  Returns the offset or 0xFFFFFFFF.
__device__ __forceinline__ uint32_t team_place(uint32_t head, uint32_t tail, uint32_t len,
                                               uint32_t size) {
  if (tail == 0xFFFFFFFFu) return len <= size ? 0u : 0xFFFFFFFFu;
  if (head > tail) {
    if (head + len <= size) return head;
    return len <= tail ? 0u : 0xFFFFFFFFu;
  }
  return head + len <= tail ? head : 0xFFFFFFFFu;
}

// Stage super-iteration j of a page (global number pr.gi) if its data fit
// the staging buffers next to what is still unread: the packed words
// [P_j, P_j+1), its block records, and the byte-array bytes [S_j, S_j+1)
// (skipped when they exceed the buffer: that super-iteration patches from
// global memory), each as the 16-byte-aligned span covering it, all
// completing on the slot's `full` barrier.  info[slot] = {shared address of
// page word 0, shared address of byte-array byte 0 (0: not staged)}.
// `ctx` = the page's context (bounds P at +0, S at +80).  Lane 0 only.
__device__ __forceinline__ bool team_issue(TeamProducer& pr, uint32_t sb, uint32_t ctx, uint32_t j,
                                           uint32_t nb, const uint32_t* page, const uint8_t* ba,
                                           const uint4* rec, uint32_t nw, uint32_t c) {
  using LY = TeamLayout;
  const uint32_t P0 = lds32(ctx + 4u * j), P1 = lds32(ctx + 4u * j + 4u);
  const uint32_t S0 = lds32(ctx + 80u + 4u * j), S1 = lds32(ctx + 84u + 4u * j);
  const uintptr_t gp0 = reinterpret_cast<uintptr_t>(page + P0) & ~uintptr_t(15);
  const uintptr_t gp1 = (reinterpret_cast<uintptr_t>(page + P1) + 15) & ~uintptr_t(15);
  const uintptr_t gs0 = reinterpret_cast<uintptr_t>(ba + S0) & ~uintptr_t(15);
  const uintptr_t gs1 = (reinterpret_cast<uintptr_t>(ba + S1) + 15) & ~uintptr_t(15);
  const uint32_t lenp = P1 > P0 ? (uint32_t)(gp1 - gp0) : 0u;
  uint32_t lens = S1 > S0 ? (uint32_t)(gs1 - gs0) : 0u;
  const bool pskip = lens > kTeamPs;
  if (pskip) lens = 0;
#ifdef IZG_BOUNDS_SELFTEST  // the checker must fire: pretend the chunk is half as long
  IZG_CHECK(izg_in_span(gp0, lenp, page, nw / 2), 1, c, P0);
#else
  IZG_CHECK(izg_in_span(gp0, lenp, page, nw), 1, c, P0);
#endif
  IZG_CHECK(pskip || izg_in_span(gs0, lens, page, nw), 2, c, S0);
  (void)nw;
  (void)c;
  uint32_t tp = 0xFFFFFFFFu, ts = 0xFFFFFFFFu;
  if (pr.gi != pr.gd) {  // oldest unread super-iteration: gd
    const uint2 al = lds64(sb + LY::kAlloc + 8u * (pr.gd % kTeamSlots));
    tp = al.x;
    ts = al.y;
  } else {
    pr.pk_head = pr.ps_head = 0;
  }
  const uint32_t op = team_place(pr.pk_head, tp, lenp, kTeamPk);
  const uint32_t ops = team_place(pr.ps_head, ts, lens, kTeamPs);
  if (op == 0xFFFFFFFFu || ops == 0xFFFFFFFFu) return false;
  const uint32_t slot = pr.gi % kTeamSlots;
  const uint32_t bar = sb + LY::kBar + 8u * slot;
  const uint32_t nrec = min(kTeamSI, nb - j * kTeamSI);
  const uint32_t pkrel = sb + LY::kPk + op - (uint32_t)(gp0 - reinterpret_cast<uintptr_t>(page));
  const uint32_t psrel =
      pskip ? 0u : sb + LY::kPs + ops - (uint32_t)(gs0 - reinterpret_cast<uintptr_t>(ba));
  sts64(sb + LY::kInfo + 8u * slot, pkrel, psrel);
  sts64(sb + LY::kAlloc + 8u * slot, op, ops);
  fence_proxy_async_smem();  // earlier generic reads of the buffers, then async writes
  mbar_arrive_expect_tx_s(bar, lenp + lens + 16u * nrec);
  if (lenp) bulk_g2s_s(sb + LY::kPk + op, reinterpret_cast<const void*>(gp0), lenp, bar, pr.policy);
  bulk_g2s_s(sb + LY::kRec + slot * (kTeamSI * 16u), rec + j * kTeamSI, 16u * nrec, bar, pr.policy);
  if (lens) bulk_g2s_s(sb + LY::kPs + ops, reinterpret_cast<const void*>(gs0), lens, bar, pr.policy);
  pr.pk_head = op + lenp;
  pr.ps_head = ops + lens;
  return true;
}

// End of a chunk (one warp): VByte remainder (codec.cpp:56-62), exact
// consumption (codec.cpp:63-64), status and words consumed.
template <int DELTA>
__device__ __forceinline__ void team_finish(int32_t st, uint32_t pos, uint4 carry,
                                            const izg_chunk& ch, const uint32_t* page, uint32_t* o,
                                            uint32_t c, int32_t* status, uint32_t* consumed,
                                            int lane) {
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  if (kArray && st == IZG_OK) {
    const uint32_t core = ch.n / 128 * 128;
    if (core < ch.n) {
      uint32_t rb = 0;
      if (lane == 0)
        st = vbyte_tail<DELTA>(reinterpret_cast<const uint8_t*>(page + pos), 4u * (ch.n_words - pos),
                               core, ch.n - core, carry, o, &rb);
      st = __shfl_sync(0xFFFFFFFFu, st, 0);
      rb = __shfl_sync(0xFFFFFFFFu, rb, 0);
      if (st == IZG_OK) pos += (rb + 3) / 4;
    }
    if (st == IZG_OK && pos != ch.n_words) st = IZG_E_PAYLOAD_SIZE;
  }
  if (lane == 0) {
    status[c] = st;
    if (consumed) consumed[c] = st == IZG_OK ? pos : 0;
  }
}

template <int DELTA>
__global__ void __launch_bounds__(IZG_TEAM_LB_THREADS, IZG_TEAM_MINCTAS)
    fp_team_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                   uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                   uint32_t* __restrict__ consumed, uint32_t* __restrict__ next_chunk,
                   const __grid_constant__ CUtensorMap omap, int tma_out, IdxView ix) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using LY = TeamLayout;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t sb = smem_u32(smem);
  asm volatile("mov.u32 %0, %0;" : "+r"(sb));  // one register, never rematerialised
  if (tid == 0) {
    for (uint32_t i = 0; i < kTeamSlots; ++i) {
      mbar_init_s(sb + LY::kBar + 8u * i, 1);
      mbar_init_s(sb + LY::kEmpty + 8u * i, kTeamWarps);
    }
    for (uint32_t i = 0; i < kTeamWarps; ++i) mbar_init_s(sb + LY::kMbx + 8u * i, 1);
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init_s(sb + LY::kXfull + 8u * i, 1);
      mbar_init_s(sb + LY::kXempty + 8u * i, kTeamWarps);
      mbar_init_s(sb + LY::kPfull + 8u * i, 1);
      mbar_init_s(sb + LY::kPdone + 8u * i, kTeamWarps - 1);
      mbar_init_s(sb + LY::kPfree + 8u * i, 1);
    }
    fence_barrier_init();
    if (kArray) {  // the first page's initial carry, posted to warp 0's mailbox
      sts128(sb + LY::kTot, 0, 0, 0, 0);
      mbar_arrive_s(sb + LY::kMbx);
    }
  }
  __syncthreads();

  if (warp == kTeamWarps) {
    // ======================= staging warp ====================================
    // Runs ahead of the decoding warps as two in-order streams over the
    // pages it claims: (a) staging of super-iterations (TMA), (b) exception
    // windows (bulk unpack into the free half of xbuf, one batch of groups
    // per pass), stream (b) up to a page ahead of (a).  Pages that need no
    // decode (argument errors, index-pass errors, arrays shorter than a
    // block) are settled here.  Each decodable page gets a context (bounds,
    // array bases, snapshots; two contexts, by page parity) and a published
    // descriptor for the decoding warps.
    TeamProducer pr;
    pr.policy = policy_evict_first();
    pr.gi = pr.gd = pr.pk_head = pr.ps_head = 0;
    auto claim = [&]() -> uint32_t {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(next_chunk, 1u);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      if (c < n_chunks) {  // its index records towards L2: read one page later
        const uint8_t* p = nullptr;
        if (lane == 0) p = reinterpret_cast<const uint8_t*>(chunks + c);
        else if (lane == 1) p = reinterpret_cast<const uint8_t*>(ix.hdr + c);
        else if (lane == 2) p = reinterpret_cast<const uint8_t*>(ix.dir + (size_t)c * 32);
        else if (lane < 11) p = reinterpret_cast<const uint8_t*>(ix.snap + (size_t)c * 512) + 128 * (lane - 3);
        else if (lane < 28) p = reinterpret_cast<const uint8_t*>(ix.page_rec(c) + min(32u * (lane - 11), kMaxBlocks - 1));
        if (p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
      }
      return c;
    };
    // context scalars (u32 index from +288): 0 c, 1 nb, 2 K, 3 A, 4 flags (1 ovf, 2 exception rows
    // aligned), 5..6 word_off, 7 n_words
    constexpr uint32_t kScal = 288, kSnapOff = (20 + 20 + 32 + 24) * 4;
    uint32_t c_next = claim();
    uint32_t pprep = 0;   // decodable pages prepared so far (contexts / descriptors written)
    bool ended = false;   // the END descriptor is out
    uint32_t pa = 0, ka = 0;    // stream (a): page, next super-iteration to stage
    uint32_t pb = 0, wkb = 0;   // stream (b): page, first super-iteration without a window
    uint32_t wprep = 0;         // windows prepared so far
    for (;;) {
      bool progress = false;
      // ---- a new page, when a stream needs one and a context is free ----------
      if (!ended && (pa == pprep || pb == pprep) && min(pa, pb) + 2 > pprep) {
        const uint32_t c = c_next;
        const uint32_t pp = pprep & 1u;
        if (c >= n_chunks) {  // no more pages: tell the decoding warps
          if (pprep >= 2) mbar_wait_s(sb + LY::kPfree + 8u * pp, ((pprep >> 1) - 1u) & 1u);
          if (lane == 0) {
            sts128(sb + LY::kDesc + 64u * pp, 0, 1u, 0, 0);
            mbar_arrive_s(sb + LY::kPfull + 8u * pp);
          }
          ended = true;
        } else {
          c_next = claim();
          const izg_chunk ch = chunks[c];
          int32_t st = precheck(IZG_SIMDFASTPFOR, kArray, ch.n);
          const uint32_t* page = words + ch.word_off;
          const uint32_t nb = (kArray ? ch.n / 128 * 128 : ch.n) / 128;
          uint4 h = make_uint4(0, 0, 0, 0);
          const uint4* rec = ix.page_rec(c);
          bool decode = false;
          if (st == IZG_OK && nb) {
            h = ix.hdr[c];
            st = (int32_t)(h.x & 0xFFu);
            if (st == IZG_OK)
              decode = true;
            else if (!(st == IZG_E_FP_TRUNC_PAGE || st == IZG_E_FP_BA_OFFSET ||
                       st == IZG_E_FP_TRUNC_BA) &&
                     fp_positions_bad_idx(rec, reinterpret_cast<const uint8_t*>(page + h.w + 1),
                                          (h.x >> 8) & 0xFFFFu, lane))
              st = IZG_E_FP_POS_RANGE;
          }
          if (!decode) {
            team_finish<DELTA>(st, 0, make_uint4(0, 0, 0, 0), ch, page, out + ch.out_off, c, status,
                               consumed, lane);
          } else {
            const uint32_t A = h.w;
            const bool ovf = (h.x >> 31) != 0;  // a cursor passed 65,535: no snapshots
            const bool xal = (reinterpret_cast<uintptr_t>(page) & 15) == 0;
            const uint32_t K = (nb + kTeamSI - 1) / kTeamSI;
            const uint32_t ctx = sb + LY::kCtx + pp * LY::kCtxBytes;
            // Super-iteration bounds, lane l <-> boundary l (0..16): packed
            // word and byte-array offset of block 32 l, or the ends.
            uint32_t bP = A, bS = 4u * (h.y - A - 1);
            if ((uint32_t)lane * kTeamSI < nb) {
              const uint4 e = rec[(uint32_t)lane * kTeamSI];
              bP = e.y;
              bS = e.z - 3u;
            }
            const uint32_t dirv = ix.dir[(size_t)c * 32 + lane];  // lane <-> width lane + 1
            if (lane < 20) {
              sts32(ctx + 4u * lane, bP);
              sts32(ctx + 80u + 4u * lane, bS);
            }
            sts32(ctx + 160u + 4u * lane, dirv);
            if (!ovf) {
              const uint32_t* sp = reinterpret_cast<const uint32_t*>(ix.snap + (size_t)c * 512);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                sts32(ctx + kSnapOff + 4u * (lane + 32 * i), __ldg(sp + lane + 32 * i));
            }
            if (lane == 0) {
              prefetch_l2(page + h.y, 4u * (h.z - h.y));  // exception arrays
              sts128(ctx + kScal, c, nb, K, A);
              sts128(ctx + kScal + 16, (ovf ? 1u : 0u) | (xal ? 2u : 0u), (uint32_t)ch.word_off,
                     (uint32_t)(ch.word_off >> 32), ch.n_words);
            }
            if (pprep >= 2) mbar_wait_s(sb + LY::kPfree + 8u * pp, ((pprep >> 1) - 1u) & 1u);
            sts32(sb + LY::kDirb + 4u * (36u * pp + lane + 1), dirv);
            if (lane == 0) {
              const uint32_t d = sb + LY::kDesc + 64u * pp;
              sts128(d, c, ovf ? 2u : 0u, nb, K);
              sts128(d + 16, A, h.z, ch.n, ch.n_words);
              sts128(d + 32, (uint32_t)ch.word_off, (uint32_t)(ch.word_off >> 32),
                     (uint32_t)ch.out_off, (uint32_t)(ch.out_off >> 32));
              sts32(sb + LY::kDirb + 4u * 36u * pp, 0);
              sts32(sb + LY::kBad + 4u * pp, 0);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_s(sb + LY::kPfull + 8u * pp);
            ++pprep;
          }
        }
        progress = true;
      }
      // ---- stream (a): staging --------------------------------------------------
      if (pa < pprep) {
        const uint32_t ctx = sb + LY::kCtx + (pa & 1u) * LY::kCtxBytes;
        uint32_t r = 0;  // bit 0: staged something, bit 1: page complete
        if (lane == 0) {
          const uint4 sc = lds128(ctx + kScal);        // c, nb, K, A
          const uint4 sc2 = lds128(ctx + kScal + 16);  // flags, word_off
          while (pr.gd < pr.gi &&
                 mbar_test_s(sb + LY::kEmpty + 8u * (pr.gd % kTeamSlots), (pr.gd / kTeamSlots) & 1u))
            ++pr.gd;
          const uint32_t* page = words + ((uint64_t)sc2.z << 32 | sc2.y);
          const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + sc.w + 1);
          while (ka < sc.z && pr.gi < pr.gd + kTeamSlots) {
            if (!team_issue(pr, sb, ctx, ka, sc.y, page, ba, ix.page_rec(sc.x), sc2.w, sc.x)) break;
            ++pr.gi;
            ++ka;
            r |= 1u;
          }
          if (ka == sc.z) r |= 2u;
        }
        r = __shfl_sync(0xFFFFFFFFu, r, 0);
        ka = __shfl_sync(0xFFFFFFFFu, ka, 0);
        if (r & 1u) progress = true;
        if (r & 2u) {
          ++pa;
          ka = 0;
          progress = true;
        }
      }
      // ---- stream (b): exception windows ---------------------------------------
      if (pb < pprep) {
        const uint32_t ctx = sb + LY::kCtx + (pb & 1u) * LY::kCtxBytes;
        const uint32_t xb = wprep & 1u;
        const uint4 sc = lds128(ctx + kScal);        // c, nb, K, A
        const uint4 sc2 = lds128(ctx + kScal + 16);  // flags, word_off
        const uint32_t K = sc.z;
        const bool ovf = (sc2.x & 1u) != 0;
        uint32_t fr = 1;
        if (wprep >= 2 && lane == 0)
          fr = mbar_test_s(sb + LY::kXempty + 8u * xb, ((wprep >> 1) - 1u) & 1u);
        if (__shfl_sync(0xFFFFFFFFu, fr, 0)) {
          // lane <-> width w = lane + 1; lo / hi = its cursor at the window's
          // ends; the longest window whose packed groups (16 w bytes each,
          // plus the 16-byte alignment of each array's span) fit this half
          const uint32_t w = (uint32_t)lane + 1u;
          const uint32_t lo = (wkb && !ovf) ? lds16(ctx + kSnapOff + 2u * ((wkb - 1) * 32 + lane)) : 0u;
          uint32_t m = K - wkb, g = 0, bytes = 0, tot = 0;
          bool fast = false;
          if (!ovf) {
            for (;; --m) {
              const uint32_t hi = lds16(ctx + kSnapOff + 2u * ((wkb + m - 1) * 32 + lane));
              g = hi > lo ? ((hi + 127u) >> 7) - (lo >> 7) : 0u;
              bytes = g ? g * 16u * w + 32u : 0u;
              tot = bytes;
#pragma unroll
              for (int d = 16; d; d >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, d);
              if (tot <= kTeamXb) {
                fast = true;
                break;
              }
              if (m == 1) break;
            }
          }
          const uint32_t bar = sb + LY::kXfull + 8u * xb;
          if (fast && tot) {
            uint32_t off = bytes;  // exclusive prefix of the spans over the widths
#pragma unroll
            for (uint32_t d = 1; d < 32; d <<= 1) shfl_up_add(off, d);
            off -= bytes;
            const uint32_t* page = words + ((uint64_t)sc2.z << 32 | sc2.y);
            const uint32_t* src = page + lds32(ctx + 160u + 4u * lane) + (size_t)(lo >> 7) * 4u * w;
            const uintptr_t s0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
            const uintptr_t s1 = (reinterpret_cast<uintptr_t>(src) + g * 16u * w + 15) & ~uintptr_t(15);
            const uint32_t len = g ? (uint32_t)(s1 - s0) : 0u;  // <= bytes - 16
            const uint32_t dst = sb + LY::kXb + xb * kTeamXb + off;
            uint32_t sum = len;
#pragma unroll
            for (int d = 16; d; d >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, d);
            // value r of width w: packed group r / 128 - lo / 128 from this address on
            if (g)
              sts64(sb + LY::kXrel + 8u * (36u * xb + w),
                    dst + (uint32_t)(reinterpret_cast<uintptr_t>(src) - s0), lo & ~127u);
            if (lane == 0) {
              sts64(sb + LY::kXinfo + 8u * xb, wkb + m, 1u);
              fence_proxy_async_smem();
              mbar_arrive_expect_tx_s(bar, sum);
            }
            __syncwarp();
            IZG_CHECK(!g || izg_in_span(s0, len, page, sc2.w), 3, sc.x, lane);
            if (g) bulk_g2s_s(dst, reinterpret_cast<const void*>(s0), len, bar, pr.policy);
          } else {
            if (lane == 0) {
              sts64(sb + LY::kXinfo + 8u * xb, wkb + m, fast ? 1u : 0u);
              mbar_arrive_s(bar);
            }
          }
          __syncwarp();
          ++wprep;
          wkb += m;
          if (wkb >= K) {
            ++pb;
            wkb = 0;
          }
          progress = true;
        }
      }
      if (ended && pa == pprep && pb == pprep) break;
#ifdef IZG_TEAM_PROF
      if (!progress && lane == 0) TEAM_PROF_ADD(6, 1);
#endif
      if (!progress) __nanosleep(IZG_TEAM_IDLE_NS);
    }
    return;
  }

  // ========================= decoding warps ==================================
  constexpr int NC = DELTA == IZG_DELTA_D4 ? 4 : DELTA == IZG_DELTA_D2 ? 2 : 1;
  (void)NC;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  TeamTile tile;
  tile.init(sb + LY::kTiles + warp * kStageOut, lane, &omap);
  uint32_t git = 0;     // super-iterations consumed so far, all pages (slot and parity)
  uint32_t wcount = 0;  // exception windows entered so far
  for (uint32_t pcount = 0;; ++pcount) {
    const uint32_t pp = pcount & 1u;
    TEAM_PROF_T(pq0);
    team_wait(sb + LY::kPfull + 8u * pp, (pcount >> 1) & 1u);
    TEAM_PROF_T(pq1);
#ifdef IZG_TEAM_PROF
    long long pxw = 0, pfw = 0, pmw = 0;
#endif
    const uint4 d0 = lds128(sb + LY::kDesc + 64u * pp);
    if (d0.y & 1u) break;
    const uint4 d1 = lds128(sb + LY::kDesc + 64u * pp + 16);
    const uint4 d2 = lds128(sb + LY::kDesc + 64u * pp + 32);
    const uint32_t c = d0.x, nb = d0.z, K = d0.w, A = d1.x;
    izg_chunk ch;
    ch.word_off = (uint64_t)d2.y << 32 | d2.x;
    ch.out_off = (uint64_t)d2.w << 32 | d2.z;
    ch.n = d1.z;
    ch.n_words = d1.w;
    const uint32_t* page = words + ch.word_off;
    uint32_t* o = out + ch.out_off;
    const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    const int64_t orow = tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5) : -1;
    const bool pal = (reinterpret_cast<uintptr_t>(page + 1) & 15) == 0;  // packed rows aligned
    uint32_t win_end = 0, xb = 0;
    bool xfast = false, bad = false;
    uint4 fin = make_uint4(0, 0, 0, 0);  // warp 7, lane 31: the page's final carry
#pragma unroll 1
    for (uint32_t k = 0; k < K; ++k, ++git) {
      if (k == win_end) {  // next exception window
        if (k) {
          __syncwarp();
          if (lane == 0) mbar_arrive_s(sb + LY::kXempty + 8u * xb);
        }
        xb = wcount & 1u;
        TEAM_PROF_T(px0);
        team_wait(sb + LY::kXfull + 8u * xb, (wcount >> 1) & 1u);
#ifdef IZG_TEAM_PROF
        pxw += clock64() - px0;
#endif
        const uint2 xi = lds64(sb + LY::kXinfo + 8u * xb);
        win_end = xi.x;
        xfast = xi.y != 0;
        ++wcount;
      }
      const uint32_t slot = git % kTeamSlots;
      TEAM_PROF_T(pf0);
      team_wait(sb + LY::kBar + 8u * slot, (git / kTeamSlots) & 1u);
#ifdef IZG_TEAM_PROF
      pfw += clock64() - pf0;
#endif
      const uint2 info = lds64(sb + LY::kInfo + 8u * slot);
      const uint32_t blk0 = k * kTeamSI + 4u * warp;
      const bool live = blk0 + q < nb;
      // a block past the page's last decodes width 0 at the first block's rows
      uint4 e = lds128(sb + LY::kRec + slot * (kTeamSI * 16u) + (live ? 16u * (4u * warp + q) : 0u));
      if (!live) e.x = 0;
      const uint32_t myb = e.x & 63u, myw = (e.x >> 6) & 63u, myc = e.x >> 12;
      const uint32_t myoff = e.y, mybp = e.z, mycur = e.w;
#ifdef IZG_ABL_TEAM_NOPATCH  // developer ablation (wrong output): no exception path
      const bool tot = false;
#else
      const bool tot = __any_sync(0xFFFFFFFFu, myc != 0);
#endif
      uint32_t v[4][4];
      if (pal) {
#if IZG_TEAM_NARROW
        if (__all_sync(0xFFFFFFFFu, myb <= 8u))
          team_unpack_narrow(info.x + 4u * myoff, myb, s8, v);
        else
#endif
          IZG_TEAM_UNPACK(info.x + 4u * myoff, myb, s8, v);
      } else {
        team_unpack_words(info.x + 4u * myoff, myb, s8, v);
      }
      if (tot) {
        tile.wait_free();
        tile.write(v);
        __syncwarp();
        if (xfast && info.y) {
          const uint2 xr = lds64(sb + LY::kXrel + 8u * (36u * xb + myw));
          bad |= team_patch(tile.t, info.y + mybp, xr.x, mycur - xr.y, myw, myb, myc, lane);
        } else {
          bad |= fp_patch<kVertical>(tile.t, page, ba, myb, myw, myc, mybp, mycur,
                                     lds32(sb + LY::kDirb + 4u * (36u * pp + myw)), lane, ch.n_words, c);
        }
        __syncwarp();
        tile.read(v);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_s(sb + LY::kEmpty + 8u * slot);  // done with the staging
#ifdef IZG_ABL_TEAM_NOSCAN  // developer ablation (wrong output): no prefix sum, no carry chain
      if (false) {
#else
      if (kArray) {
#endif
        uint4 ex, incl;
        uint32_t q3[4] = {0, 0, 0, 0};
        team_scan_local<DELTA>(v, ex, incl, q3, lane);
        // carry chain: the prefix up to the previous warp iteration arrives
        // in this warp's mailbox; ours goes to the next warp's (the page's
        // last one posts the next page's zero carry instead)
#ifndef IZG_ABL_TEAM_NOCHAIN  // developer ablation (wrong output): no wait on the carry chain
        TEAM_PROF_T(pm0);
        team_wait(sb + LY::kMbx + 8u * warp, git & 1u);
#ifdef IZG_TEAM_PROF
        pmw += clock64() - pm0;
#endif
#endif
        const uint4 pv = lds128(sb + LY::kTot + 16u * warp);
        __syncwarp();  // everyone has read the mailbox before the chain can refill it
        if (lane == 31) {
          fin = u4add(pv, incl);
          const bool wrap = warp == kTeamWarps - 1;
          const uint32_t dst = wrap ? 0u : (uint32_t)warp + 1u;
          if (wrap && k + 1 == K)
            sts128(sb + LY::kTot, 0, 0, 0, 0);
          else
            sts128(sb + LY::kTot + 16u * dst, fin.x, fin.y, fin.z, fin.w);
          mbar_arrive_s(sb + LY::kMbx + 8u * dst);
        }
        team_scan_apply<DELTA>(v, u4add(pv, ex), q3);
      }
#ifdef IZG_ABL_TEAM_NOSTORE  // developer ablation (no output): nothing stored
      if (v[0][0] == 0xFFFFFFFFu && v[3][3] == 0x12345678u && v[1][2] == 77u) bad = true;
      if (true) {
      } else
#endif
      if (orow >= 0 && blk0 + 4 <= nb) {
        IZG_CHECK(128u * (blk0 + 4) <= ch.n, 4, c, blk0);
        if (!tot) tile.wait_free();
        tile.write(v);
        tile.store((uint32_t)(orow + 4 * (int64_t)blk0));
      } else {
        __syncwarp();
        IZG_CHECK(!live || 128u * (blk0 + q) + 16u * s8 + 16u <= ch.n, 5, c, blk0);
        if (live) store_direct(v, o + (size_t)(blk0 + q) * 128 + 16 * s8, oal);
      }
    }
    // ---- end of the page ------------------------------------------------------
#ifdef IZG_TEAM_PROF
    if (tid == 0) {
      TEAM_PROF_ADD(0, 1); TEAM_PROF_ADD(1, pq1 - pq0); TEAM_PROF_ADD(2, pxw); TEAM_PROF_ADD(3, pfw);
      TEAM_PROF_ADD(4, pmw); TEAM_PROF_ADD(5, clock64() - pq0);
    }
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive_s(sb + LY::kXempty + 8u * xb);  // done with its last window
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) sts32(sb + LY::kBad + 4u * pp, 1);
    if (warp != kTeamWarps - 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive_s(sb + LY::kPdone + 8u * pp);
    } else {  // the last warp of the chain holds the final carry: it ends the chunk
      team_wait(sb + LY::kPdone + 8u * pp, (pcount >> 1) & 1u);
      uint4 carry;
      carry.x = __shfl_sync(0xFFFFFFFFu, fin.x, 31);
      carry.y = __shfl_sync(0xFFFFFFFFu, fin.y, 31);
      carry.z = __shfl_sync(0xFFFFFFFFu, fin.z, 31);
      carry.w = __shfl_sync(0xFFFFFFFFu, fin.w, 31);
      const int32_t st = lds32(sb + LY::kBad + 4u * pp) ? IZG_E_FP_POS_RANGE : IZG_OK;
      team_finish<DELTA>(st, d1.y, carry, ch, page, o, c, status, consumed, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(sb + LY::kPfree + 8u * pp);
    }
  }
  tile.drain();
}

}  // namespace izg
