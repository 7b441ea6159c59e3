// team.cuh — SIMD-FastPFOR decode with one CTA (a "team" of 8 warps) per page.
//
// The warp-per-page decode (decode_fastpfor.cuh / index_fastpfor.cuh) is
// issue-bound: every warp runs its own staging ring, and every exception
// costs two scattered global loads plus the address arithmetic of the
// vertical layout (codec_patched.cpp:338-379 bulk-unpacks the exception
// arrays instead).  Here a CTA decodes one page in lockstep super-iterations
// of 32 blocks (4,096 integers), one warp iteration of 4 blocks per warp:
//
//   * staging is shared: per super-iteration one thread issues TMA bulk
//     copies of the packed words, the 32 block records of the page index
//     pass and the position bytes into linear shared-memory buffers (one
//     mbarrier per slot, four slots in flight), so no warp manages a ring;
//   * exception highs are bulk-unpacked the way the reference does
//     (codec_patched.cpp:346-379), but only for a WINDOW of super-iterations
//     at a time: the page index pass records every width's cursor at each
//     32-block boundary (IdxView::snap), the team takes the longest window
//     whose vertical groups fit its 16 KiB buffer, and its warps unpack
//     those groups (one warp per group of 128, lane = slot, straight from
//     global memory).  A patch then costs one position byte and one value
//     from shared memory (codec_patched.cpp:390-404: o[pos] |= high << b);
//   * the prefix sum is two-level: each warp scans its 512 integers from a
//     zero carry, lane 31 publishes the warp total, one CTA barrier, and
//     every warp adds the page carry plus the totals of the warps before it
//     (delta.cpp:60-75 for D4; the same split for D1 / D2 / DM).
//
// Everything the index pass checked stays checked there; exception
// positions >= 128 are detected while patching (codec_patched.cpp:328-330),
// as in the warp-per-page kernels.  Pages whose exception windows or
// position bytes do not fit (a single super-iteration over 32 groups or
// 5 KiB of positions, cursors past 65,535) patch from global memory with
// fp_patch for the super-iterations concerned: same results.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "decode_kernel.cuh"

namespace izg {

constexpr int kTeamWarps = 8;
constexpr uint32_t kTeamSI = 4 * kTeamWarps;  // blocks per super-iteration
constexpr uint32_t kTeamSlots = 4;            // super-iterations staged ahead
#ifndef IZG_TEAM_PK
#define IZG_TEAM_PK (20 * 1024)
#endif
#ifndef IZG_TEAM_XB
#define IZG_TEAM_XB (16 * 1024)
#endif
constexpr uint32_t kTeamPk = IZG_TEAM_PK;     // packed words staging (>= 16 KiB + 16)
constexpr uint32_t kTeamPs = 5 * 1024;        // position bytes staging
constexpr uint32_t kTeamXb = IZG_TEAM_XB;     // unpacked exception highs of a window
constexpr uint32_t kTeamXGroups = kTeamXb / 512;
#ifndef IZG_TEAM_UNPACK
#define IZG_TEAM_UNPACK team_unpack_window  // or team_unpack_rows (more row loads, fewer moves)
#endif
#ifndef IZG_TEAM_AHEAD
#define IZG_TEAM_AHEAD 2  // warp 0 stages more once fewer than this many lie ahead
#endif
#ifndef IZG_TEAM_MINCTAS
#define IZG_TEAM_MINCTAS 3  // CTAs per SM the register allocation allows for
#endif
constexpr int kTeamThreads = (kTeamWarps + 1) * 32;  // 8 decoding warps + the staging warp
#define IZG_TEAM_LB_THREADS ((kTeamWarps + 1) * 32)

#ifdef IZG_TEAM_PROF  // developer build: where a page's time goes (cycles, summed over pages)
// [0] pages, [1] claim -> setup barrier, [2] setup barrier -> first staging landed (warp 0),
// [3] window set-ups (warp 0, incl. barriers), [4] iterations (warp 0), [5] loop end -> page end
// [6] warp 0: waits on `full`, [7] warp 0: waits on the carry mailbox
__device__ unsigned long long g_team_prof[8];
#define TEAM_PROF_T(x) const long long x = clock64()
#define TEAM_PROF_ADD(i, v) atomicAdd(&g_team_prof[i], (unsigned long long)(v))
#else
#define TEAM_PROF_T(x)
#define TEAM_PROF_ADD(i, v)
#endif

struct TeamLayout {
  static constexpr uint32_t kTiles = 0;  // one 2 KiB output tile per warp (1024-aligned)
  static constexpr uint32_t kPk = kTiles + kTeamWarps * kStageOut;
  static constexpr uint32_t kPs = kPk + kTeamPk;
  static constexpr uint32_t kRec = kPs + kTeamPs;
  static constexpr uint32_t kXb = kRec + kTeamSlots * kTeamSI * 16;
  static constexpr uint32_t kSnap = kXb + kTeamXb;       // u16 [16][32]
  static constexpr uint32_t kXrel = kSnap + 1024;        // i32 [36]
  static constexpr uint32_t kDirb = kXrel + 36 * 4;      // u32 [36]
  static constexpr uint32_t kTot = kDirb + 36 * 4;       // uint4 [warps + 1]: carry mailboxes, final carry
  static constexpr uint32_t kInfo = kTot + (kTeamWarps + 1) * 16;  // uint2 [slots] {pkrel, psrel}
  static constexpr uint32_t kAlloc = kInfo + kTeamSlots * 8;     // uint2 [slots] {pk off, ps off}
  static constexpr uint32_t kBar = kAlloc + kTeamSlots * 8;      // u64 [slots]: staging landed
  static constexpr uint32_t kEmpty = kBar + kTeamSlots * 8;      // u64 [slots]: staging read by all warps
  static constexpr uint32_t kMbx = kEmpty + kTeamSlots * 8;      // u64 [warps]: mailbox posted
  static constexpr uint32_t kPage = kMbx + kTeamWarps * 8;       // u32 page, u32 bad flag
  static constexpr size_t kSmem = kPage + 16;
};
static_assert(TeamLayout::kXrel % 16 == 0 && TeamLayout::kTot % 16 == 0, "team layout");
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
// position byte, `xa` = shared address of its first exception high.
__device__ __forceinline__ bool team_patch(uint32_t t, uint32_t ps, uint32_t xa, uint32_t myb,
                                           uint32_t myc, int lane) {
  const uint32_t q = (lane >> 3) & 3u, s8 = lane & 7;
  uint32_t mxc = max(myc, __shfl_xor_sync(0xFFFFFFFFu, myc, 8));
  mxc = max(mxc, __shfl_xor_sync(0xFFFFFFFFu, mxc, 16));
  // integer p of block q: tile byte 512 q + (4 p ^ 16 ((row & 7))), row = 4 q + p / 32,
  // i.e. (t + 512 q) ^ 64 (q & 1) ^ (4 p) ^ 16 (p / 32)
  const uint32_t tqr = (t + (q << 9)) ^ ((q & 1u) << 6);
  uint32_t badp = 0;
  for (uint32_t e0 = s8; e0 < mxc; e0 += 16) {
    uint32_t pp[2], xv[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t e = e0 + 8u * j;
      pp[j] = 0x100u;  // idle slot: no patch, not a position error
      xv[j] = 0;
      if (e < myc) {
        pp[j] = lds8(ps + e);
        xv[j] = lds32(xa + 4u * e);
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t p = pp[j];
      const uint32_t a = tqr ^ (((p >> 1) & 0x30u) ^ (p << 2));
      if (p < 128u) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(xv[j] << myb) : "memory");
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

// Producer state of a page (warp 0; lane 0 issues the copies).
struct TeamProducer {
  uint32_t issued;            // super-iterations of this page staged so far
  uint32_t done;              // super-iterations every warp has finished reading
  uint32_t pk_head, ps_head;  // allocation heads of the two staging buffers
  uint64_t policy;
};

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

// Stage super-iterations until number `need` is staged, and beyond it while
// they fit, up to kTeamSlots past the `done` consumed ones.  All lanes of
// warp 0 call (the bounds live in lanes 0..16); lane 0 allocates and issues.
// A super-iteration counts as consumed once every warp has arrived on its
// slot's `empty` barrier.  Per super-iteration j: the packed words
// [P_j, P_j+1), its block records, and the byte-array bytes [S_j, S_j+1)
// (skipped when they exceed the buffer: that super-iteration patches from
// global memory), each as the 16-byte-aligned span covering it, all
// completing on the slot's `full` barrier.  info[slot] = {shared address of
// page word 0, shared address of byte-array byte 0 (0: not staged)}.
__device__ __forceinline__ void team_produce(TeamProducer& pr, uint32_t sb, uint32_t git0,
                                             uint32_t need, uint32_t K, uint32_t nb, uint32_t bP,
                                             uint32_t bS, const uint32_t* page, const uint8_t* ba,
                                             const uint4* rec, int lane) {
  using LY = TeamLayout;
  for (;;) {
    // consumed super-iterations: `empty` phases already complete
    uint32_t adv = 0;
    if (lane == 0) {
      while (pr.done + adv < pr.issued) {
        const uint32_t g = git0 + pr.done + adv;
        if (!mbar_test_s(sb + LY::kEmpty + 8u * (g % kTeamSlots), (g / kTeamSlots) & 1u)) break;
        ++adv;
      }
    }
    pr.done += __shfl_sync(0xFFFFFFFFu, adv, 0);
    while (pr.issued < K && pr.issued < pr.done + kTeamSlots) {
      const uint32_t j = pr.issued;
      const uint32_t P0 = __shfl_sync(0xFFFFFFFFu, bP, j), P1 = __shfl_sync(0xFFFFFFFFu, bP, j + 1);
      const uint32_t S0 = __shfl_sync(0xFFFFFFFFu, bS, j), S1 = __shfl_sync(0xFFFFFFFFu, bS, j + 1);
      uint32_t fit = 1;
      if (lane == 0) {
        const uintptr_t gp0 = reinterpret_cast<uintptr_t>(page + P0) & ~uintptr_t(15);
        const uintptr_t gp1 = (reinterpret_cast<uintptr_t>(page + P1) + 15) & ~uintptr_t(15);
        const uintptr_t gs0 = reinterpret_cast<uintptr_t>(ba + S0) & ~uintptr_t(15);
        const uintptr_t gs1 = (reinterpret_cast<uintptr_t>(ba + S1) + 15) & ~uintptr_t(15);
        const uint32_t lenp = P1 > P0 ? (uint32_t)(gp1 - gp0) : 0u;
        uint32_t lens = S1 > S0 ? (uint32_t)(gs1 - gs0) : 0u;
        const bool pskip = lens > kTeamPs;
        if (pskip) lens = 0;
        uint32_t tp = 0xFFFFFFFFu, ts = 0xFFFFFFFFu;
        if (j != pr.done) {  // oldest unconsumed super-iteration: `done`
          const uint2 al = lds64(sb + LY::kAlloc + 8u * ((git0 + pr.done) % kTeamSlots));
          tp = al.x;
          ts = al.y;
        } else {
          pr.pk_head = pr.ps_head = 0;
        }
        const uint32_t op = team_place(pr.pk_head, tp, lenp, kTeamPk);
        const uint32_t ops = team_place(pr.ps_head, ts, lens, kTeamPs);
        if (op == 0xFFFFFFFFu || ops == 0xFFFFFFFFu) {
          fit = 0;
        } else {
          const uint32_t slot = (git0 + j) % kTeamSlots;
          const uint32_t bar = sb + LY::kBar + 8u * slot;
          const uint32_t nrec = min(kTeamSI, nb - j * kTeamSI);
          const uint32_t pkrel =
              sb + LY::kPk + op - (uint32_t)(gp0 - reinterpret_cast<uintptr_t>(page));
          const uint32_t psrel =
              pskip ? 0u : sb + LY::kPs + ops - (uint32_t)(gs0 - reinterpret_cast<uintptr_t>(ba));
          sts64(sb + LY::kInfo + 8u * slot, pkrel, psrel);
          sts64(sb + LY::kAlloc + 8u * slot, op, ops);
          fence_proxy_async_smem();  // earlier generic reads of the buffers, then async writes
          mbar_arrive_expect_tx_s(bar, lenp + lens + 16u * nrec);
          if (lenp)
            bulk_g2s_s(sb + LY::kPk + op, reinterpret_cast<const void*>(gp0), lenp, bar, pr.policy);
          bulk_g2s_s(sb + LY::kRec + slot * (kTeamSI * 16u), rec + j * kTeamSI, 16u * nrec, bar,
                     pr.policy);
          if (lens)
            bulk_g2s_s(sb + LY::kPs + ops, reinterpret_cast<const void*>(gs0), lens, bar, pr.policy);
          pr.pk_head = op + lenp;
          pr.ps_head = ops + lens;
        }
      }
      fit = __shfl_sync(0xFFFFFFFFu, fit, 0);
      if (!fit) break;
      ++pr.issued;
    }
    if (pr.issued > need || pr.issued >= K) return;
    // `need` does not fit yet: wait until the oldest staged one is consumed
    const uint32_t g = git0 + pr.done;
    mbar_wait_s(sb + LY::kEmpty + 8u * (g % kTeamSlots), (g / kTeamSlots) & 1u);
    ++pr.done;
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
  constexpr int NC = DELTA == IZG_DELTA_D4 ? 4 : DELTA == IZG_DELTA_D2 ? 2 : 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  uint32_t sb = smem_u32(smem);
  asm volatile("mov.u32 %0, %0;" : "+r"(sb));  // one register, never rematerialised
  TeamTile tile;  // decoding warps only
  tile.init(sb + LY::kTiles + (warp & (kTeamWarps - 1)) * kStageOut, lane, &omap);
  if (tid == 0) {
    for (uint32_t i = 0; i < kTeamSlots; ++i) {
      mbar_init_s(sb + LY::kBar + 8u * i, 1);
      mbar_init_s(sb + LY::kEmpty + 8u * i, kTeamWarps);
    }
    for (uint32_t i = 0; i < kTeamWarps; ++i) mbar_init_s(sb + LY::kMbx + 8u * i, 1);
    fence_barrier_init();
  }
  TeamProducer pr;
  pr.policy = policy_evict_first();
  pr.issued = pr.done = pr.pk_head = pr.ps_head = 0;
  uint32_t git = 0;  // super-iterations consumed so far, all pages (slot and parity)
  volatile uint32_t* s_page = reinterpret_cast<volatile uint32_t*>(smem + LY::kPage);

  for (;;) {
    TEAM_PROF_T(pt0);
    if (tid == 0) {
      s_page[0] = atomicAdd(next_chunk, 1u);
      s_page[1] = 0;  // a position >= 128 was met
    }
    __syncthreads();
    const uint32_t c = s_page[0];
    if (c >= n_chunks) break;
    const izg_chunk ch = chunks[c];
    int32_t st = precheck(IZG_SIMDFASTPFOR, kArray, ch.n);
    uint32_t pos = 0;
    uint4 carry = make_uint4(0, 0, 0, 0);
    const uint32_t* page = words + ch.word_off;
    uint32_t* o = out + ch.out_off;
    const uint32_t core = kArray ? ch.n / 128 * 128 : ch.n;
    const uint32_t nb = core / 128;
    bool decoded = false;
    if (st == IZG_OK && nb) {
      const uint4 h = ix.hdr[c];
      st = (int32_t)(h.x & 0xFFu);
      const uint4* rec = ix.page_rec(c);
      if (st) {
        if (!(st == IZG_E_FP_TRUNC_PAGE || st == IZG_E_FP_BA_OFFSET || st == IZG_E_FP_TRUNC_BA) &&
            fp_positions_bad_idx(rec, reinterpret_cast<const uint8_t*>(page + h.w + 1),
                                 (h.x >> 8) & 0xFFFFu, lane))
          st = IZG_E_FP_POS_RANGE;
      } else {
        decoded = true;
        const uint32_t A = h.w;
        const bool ovf = (h.x >> 31) != 0;  // a cursor passed 65,535: no snapshots
        const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);
        const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
        const int64_t orow = tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5) : -1;
        const bool pal = (reinterpret_cast<uintptr_t>(page + 1) & 15) == 0;  // packed rows aligned
        const bool xal = (reinterpret_cast<uintptr_t>(page) & 15) == 0;      // exception rows aligned
        const uint32_t K = (nb + kTeamSI - 1) / kTeamSI;
        // Super-iteration bounds, lane l <-> boundary l (0..16): packed word
        // and byte-array offset of block 32 l, or the ends.
        uint32_t bP = A, bS = 4u * (h.y - A - 1);
        if ((uint32_t)lane * kTeamSI < nb) {
          const uint4 e = rec[(uint32_t)lane * kTeamSI];
          bP = e.y;
          bS = e.z - 3u;
        }
        const uint32_t dirv = ix.dir[(size_t)c * 32 + lane];  // lane <-> width lane + 1
        if (warp == 0) {
          sts32(sb + LY::kDirb + 4u * (lane + 1), dirv);
          sts32(sb + LY::kXrel + 4u * (lane + 1), 0);
          if (lane == 0) {
            sts32(sb + LY::kDirb, 0);
            sts32(sb + LY::kXrel, 0);
          }
        }
        if (!ovf && tid < 256)
          sts32(sb + LY::kSnap + 4u * tid,
                reinterpret_cast<const uint32_t*>(ix.snap + (size_t)c * 512)[tid]);
        const uint32_t git0 = git;
        if (kArray && tid == 0) {  // the page's initial carry, posted to warp 0's mailbox
          sts128(sb + LY::kTot, 0, 0, 0, 0);
          mbar_arrive_s(sb + LY::kMbx);
        }
        __syncthreads();
        TEAM_PROF_T(pt1);
#ifdef IZG_TEAM_PROF
        long long pwin = 0, pfull = 0, pmbx = 0, pt2 = 0;
#endif
        if (warp == kTeamWarps) {
          // ---- staging warp: every super-iteration of the page, as space frees up
          pr.issued = pr.done = 0;
          while (pr.issued < K)
            team_produce(pr, sb, git0, pr.issued, K, nb, bP, bS, page, ba, rec, lane);
          while (pr.done < K) {  // observe every `empty` phase (keeps the parities in step)
            const uint32_t g = git0 + pr.done;
            mbar_wait_s(sb + LY::kEmpty + 8u * (g % kTeamSlots), (g / kTeamSlots) & 1u);
            ++pr.done;
          }
          git += K;
        } else {

        uint32_t win_end = 0;  // super-iteration at which the next exception window starts
        bool xfast = false;    // this window's highs are unpacked in shared memory
        bool bad = false;
#pragma unroll 1
        for (uint32_t k = 0; k < K; ++k, ++git) {
          // ---- exception window --------------------------------------------
          TEAM_PROF_T(pw0);
          if (k == win_end) {
            if (k) named_bar_sync(1, kTeamWarps * 32);  // every warp is done with the previous window's highs
            // lane <-> width lane + 1; lo / hi = its cursor at the window's ends
            const uint32_t lo = (k && !ovf) ? lds16(sb + LY::kSnap + 2u * ((k - 1) * 32 + lane)) : 0u;
            uint32_t m = K - k, g = 0, G = 0;
            xfast = false;
            if (!ovf) {
              for (;;) {
                const uint32_t hi = lds16(sb + LY::kSnap + 2u * ((k + m - 1) * 32 + lane));
                g = hi > lo ? ((hi + 127u) >> 7) - (lo >> 7) : 0u;
                G = g;
#pragma unroll
                for (int d = 16; d; d >>= 1) G += __shfl_xor_sync(0xFFFFFFFFu, G, d);
                if (G <= kTeamXGroups) {
                  xfast = true;
                  break;
                }
                if (m == 1) break;
                m = (m + 1) / 2;
              }
            } else {
              m = K - k;
            }
            win_end = k + m;
            if (xfast && G) {
              uint32_t goff = g;  // exclusive prefix of the groups over the widths
#pragma unroll
              for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, goff, d);
                if (lane >= d) goff += y;
              }
              goff -= g;
              // value r of width w sits at xbuf[xrel[w] + r]
              if (warp == 0) sts32(sb + LY::kXrel + 4u * (lane + 1), 128u * goff - (lo & ~127u));
              for (uint32_t i = warp; i < G; i += kTeamWarps) {
                const uint32_t own = __ballot_sync(0xFFFFFFFFu, g != 0 && goff <= i);
                const int ow = 31 - __clz(own);
                const uint32_t w = (uint32_t)ow + 1u;
                const uint32_t gi = (__shfl_sync(0xFFFFFFFFu, lo, ow) >> 7) +
                                    (i - __shfl_sync(0xFFFFFFFFu, goff, ow));
                const uint32_t* src = page + __shfl_sync(0xFFFFFFFFu, dirv, ow) + (size_t)gi * 4u * w;
                // lane = vertical slot: its four lanes' values are integers
                // 4 lane .. 4 lane + 3 of the group
                const uint32_t bit = (uint32_t)lane * w, sh = bit & 31u;
                const uint32_t* rp = src + 4u * (bit >> 5);
                uint4 a, b = make_uint4(0, 0, 0, 0);
                const bool two = sh + w > 32u;
                if (xal) {
                  a = __ldg(reinterpret_cast<const uint4*>(rp));
                  if (two) b = __ldg(reinterpret_cast<const uint4*>(rp + 4));
                } else {
                  a = make_uint4(__ldg(rp), __ldg(rp + 1), __ldg(rp + 2), __ldg(rp + 3));
                  if (two) b = make_uint4(__ldg(rp + 4), __ldg(rp + 5), __ldg(rp + 6), __ldg(rp + 7));
                }
                const uint32_t mask = low_mask(w);
                sts128(sb + LY::kXb + 512u * i + 16u * lane, funnel_r(a.x, b.x, sh) & mask,
                       funnel_r(a.y, b.y, sh) & mask, funnel_r(a.z, b.z, sh) & mask,
                       funnel_r(a.w, b.w, sh) & mask);
              }
            }
            named_bar_sync(1, kTeamWarps * 32);  // the window's highs and xrel are in place
          }

          // ---- this warp's four blocks ---------------------------------------
          const uint32_t slot = git % kTeamSlots;
          TEAM_PROF_T(pw1);
          mbar_wait_s(sb + LY::kBar + 8u * slot, (git / kTeamSlots) & 1u);
#ifdef IZG_TEAM_PROF
          { const long long now = clock64(); pwin += pw1 - pw0; pfull += now - pw1; if (k == 0) pt2 = now; }
#endif
          const uint2 info = lds64(sb + LY::kInfo + 8u * slot);
          const uint32_t blk0 = k * kTeamSI + 4u * warp;
          const bool live = blk0 + q < nb;
          // a block past the page's last decodes width 0 at the first block's rows
          uint4 e = lds128(sb + LY::kRec + slot * (kTeamSI * 16u) + (live ? 16u * (4u * warp + q) : 0u));
          if (!live) e.x = 0;
          const uint32_t myb = e.x & 63u, myw = (e.x >> 6) & 63u, myc = e.x >> 12;
          const uint32_t myoff = e.y, mybp = e.z, mycur = e.w;
          const bool tot = __any_sync(0xFFFFFFFFu, myc != 0);
          uint32_t v[4][4];
          if (pal)
            IZG_TEAM_UNPACK(info.x + 4u * myoff, myb, s8, v);
          else
            team_unpack_words(info.x + 4u * myoff, myb, s8, v);
          if (tot) {
            tile.wait_free();
            tile.write(v);
            __syncwarp();
            if (xfast && info.y) {
              const uint32_t xa = sb + LY::kXb + 4u * (lds32(sb + LY::kXrel + 4u * myw) + mycur);
              bad |= team_patch(tile.t, info.y + mybp, xa, myb, myc, lane);
            } else {
              bad |= fp_patch<kVertical>(tile.t, page, ba, myb, myw, myc, mybp, mycur,
                                         lds32(sb + LY::kDirb + 4u * myw), lane);
            }
            __syncwarp();
            tile.read(v);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_s(sb + LY::kEmpty + 8u * slot);  // done with the staging
          if (kArray) {
            uint4 ex, incl;
            uint32_t q3[4] = {0, 0, 0, 0};
            team_scan_local<DELTA>(v, ex, incl, q3, lane);
            // carry chain: the prefix up to the previous warp iteration arrives
            // in this warp's mailbox; post ours to the next warp's
#ifndef IZG_ABL_TEAM_NOCHAIN  // developer ablation (wrong output): no wait on the carry chain
            TEAM_PROF_T(pm0);
            mbar_wait_s(sb + LY::kMbx + 8u * warp, git & 1u);
#ifdef IZG_TEAM_PROF
            pmbx += clock64() - pm0;
#endif
#endif
            const uint4 pv = lds128(sb + LY::kTot + 16u * warp);
            __syncwarp();  // everyone has read the mailbox before the chain can refill it
            if (lane == 31) {
              const bool last = warp == kTeamWarps - 1;
              const uint32_t dst = last ? (k + 1 == K ? kTeamWarps : 0) : warp + 1;
              sts128(sb + LY::kTot + 16u * dst, pv.x + incl.x, pv.y + incl.y, pv.z + incl.z,
                     pv.w + incl.w);
              if (dst != kTeamWarps) mbar_arrive_s(sb + LY::kMbx + 8u * dst);
            }
            team_scan_apply<DELTA>(v, u4add(pv, ex), q3);
          }
          if (orow >= 0 && blk0 + 4 <= nb) {
            if (!tot) tile.wait_free();
            tile.write(v);
            tile.store((uint32_t)(orow + 4 * (int64_t)blk0));
          } else {
            __syncwarp();
            if (live) store_direct(v, o + (size_t)(blk0 + q) * 128 + 16 * s8, oal);
          }
        }
        if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) s_page[1] = 1;
#ifdef IZG_TEAM_PROF
        if (tid == 0) {
          const long long pt3 = clock64();
          TEAM_PROF_ADD(0, 1); TEAM_PROF_ADD(1, pt1 - pt0); TEAM_PROF_ADD(2, pt2 - pt1);
          TEAM_PROF_ADD(3, pwin); TEAM_PROF_ADD(4, pt3 - pt2); TEAM_PROF_ADD(6, pfull);
          TEAM_PROF_ADD(7, pmbx);
          s_page[2] = (uint32_t)pt3;
        }
#endif
        }  // decoding warps
        pos = h.z;
      }
    }
    __syncthreads();  // bad flag, final carry; s_page[0] read by everyone before the next claim
#ifdef IZG_TEAM_PROF
    if (tid == 0 && decoded) TEAM_PROF_ADD(5, (uint32_t)((uint32_t)clock64() - s_page[2]));
#endif
    if (warp == 0) {
      if (decoded && s_page[1]) st = IZG_E_FP_POS_RANGE;
      if (decoded && kArray) carry = lds128(sb + LY::kTot + 16u * kTeamWarps);
      __syncwarp();
      if (kArray && st == IZG_OK) {
        if (core < ch.n) {  // Variable Byte remainder (codec.cpp:56-62)
          uint32_t rb = 0;
          if (lane == 0)
            st = vbyte_tail<DELTA>(reinterpret_cast<const uint8_t*>(page + pos),
                                   4u * (ch.n_words - pos), core, ch.n - core, carry, o, &rb);
          st = __shfl_sync(0xFFFFFFFFu, st, 0);
          rb = __shfl_sync(0xFFFFFFFFu, rb, 0);
          if (st == IZG_OK) pos += (rb + 3) / 4;
        }
        if (st == IZG_OK && pos != ch.n_words) st = IZG_E_PAYLOAD_SIZE;  // codec.cpp:63-64
      }
      if (lane == 0) {
        status[c] = st;
        if (consumed) consumed[c] = st == IZG_OK ? pos : 0;
      }
    }
  }
  if (warp < kTeamWarps) tile.drain();
}

}  // namespace izg
