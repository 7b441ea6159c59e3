// team_bp.cuh — SIMD-BP128 decode with one CTA (8 decoding warps and a
// staging warp) per chunk: team.cuh's structure for the codec without
// exceptions.  One warp per chunk (decode_bp128.cuh) leaves most warp slots
// empty on batches of a few thousand chunks (C1: 1,024; C3: 4,096), and every
// warp streams its own ring.  Here:
//
//   * the staging warp copies the chunk, which is one contiguous span, into a
//     32 KiB shared ring as 4 KiB pieces (TMA bulk copies, an mbarrier per
//     piece), as far ahead as the ring allows; it walks the 16-byte
//     meta-block descriptors in the ring (SimdBp128Codec::decode_deltas,
//     codec_binpack.cpp:94-119: walk_meta, every check in the reference's
//     order) and publishes, per super-iteration of 32 blocks, each block's
//     width and ring position; it claims chunks one ahead and settles the
//     ones that need no decode;
//   * the 8 decoding warps take 4 blocks of each super-iteration, unpack them
//     from the ring (unpack_vertical128, bitpack.cpp:122-161), run the prefix
//     sum as a carry chain through per-warp mailboxes (delta.cpp:25-89) and
//     store their tile with TMA — exactly team.cuh's decoders without the
//     patch.
//
// After a descriptor error the remaining blocks of the chunk decode width 0
// (the chunk's status is the error; its output is unspecified, as in the
// other kernels); nothing reads outside the ring.
#pragma once
#include "team.cuh"

namespace izg {

#ifndef IZG_BP_PIECE
#define IZG_BP_PIECE 4096
#endif
#ifndef IZG_BP_PIECES
#define IZG_BP_PIECES 8
#endif
#ifndef IZG_BP_SLOTS
#define IZG_BP_SLOTS 4
#endif
constexpr uint32_t kBpPiece = IZG_BP_PIECE;          // bytes per ring piece
constexpr uint32_t kBpPieces = IZG_BP_PIECES;        // pieces in the ring
constexpr uint32_t kBpRing = kBpPiece * kBpPieces;   // 32 KiB >= a super-iteration + 2 pieces
constexpr uint32_t kBpSlots = IZG_BP_SLOTS;          // super-iterations published ahead
#ifndef IZG_BPTEAM_MINCTAS
#define IZG_BPTEAM_MINCTAS 3
#endif

struct BpTeamLayout {
  static constexpr uint32_t kTiles = 0;  // 2 KiB output tiles, two per decoding warp (1024-aligned)
  static constexpr uint32_t kRing = kTiles + 2 * kTeamWarps * kStageOut;
  static constexpr uint32_t kTab = kRing + kBpRing;               // uint2 [slots][32] {width, ring byte}
  static constexpr uint32_t kTot = kTab + kBpSlots * kTeamSI * 8; // uint4 [warps]: carry mailboxes
  static constexpr uint32_t kDesc = kTot + kTeamWarps * 16;       // u32 [2][16]: chunk descriptors
  static constexpr uint32_t kEnd = kDesc + 2 * 64;                // uint2 [2] {words consumed, status}
  static constexpr uint32_t kStart = kEnd + 16;                   // u32 [slots]: first ring byte
  static constexpr uint32_t kPieceBar = kStart + kBpSlots * 4;    // u64 [pieces]: piece landed
  static constexpr uint32_t kFull = kPieceBar + kBpPieces * 8;    // u64 [slots]: table published
  static constexpr uint32_t kEmpty = kFull + kBpSlots * 8;        // u64 [slots]: read by all warps
  static constexpr uint32_t kMbx = kEmpty + kBpSlots * 8;         // u64 [warps]: mailbox posted
  static constexpr uint32_t kPfull = kMbx + kTeamWarps * 8;       // u64 [2]: descriptor written
  static constexpr uint32_t kPdone = kPfull + 16;                 // u64 [2]: warps 0..6 left the chunk
  static constexpr uint32_t kPfree = kPdone + 16;                 // u64 [2]: chunk finished
  static constexpr size_t kSmem = kPfree + 16;
};
static_assert(BpTeamLayout::kTot % 16 == 0 && BpTeamLayout::kPieceBar % 8 == 0, "bp team layout");

// The ring seen from unmasked ring bytes (walk_meta's and unpack_slots_aligned's view).
struct BpRingView {
  static constexpr uint32_t kMask = kBpRing - 1;
  uint32_t base;  // shared address of the ring
  uint32_t off;   // unmasked ring byte of the chunk's payload byte 0
  __device__ __forceinline__ uint32_t addr(uint32_t o) const { return base + ((off + o) & kMask); }
  __device__ __forceinline__ uint32_t word_addr(uint32_t w) const { return addr(4u * w); }
};

// Word-load unpack from the ring for chunks whose rows are not 16-byte aligned.
__device__ __forceinline__ void bp_unpack_words(uint32_t base, uint32_t rb, uint32_t width,
                                                uint32_t s8, uint32_t (&v)[4][4]) {
  const uint32_t mask = low_mask(width);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t bit = (4u * s8 + c) * width;
    const uint32_t a = rb + 16u * (bit >> 5), sh = bit & 31u;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      v[c][j] = funnel_r(lds32(base + ((a + 4u * j) & (kBpRing - 1))),
                         lds32(base + ((a + 16u + 4u * j) & (kBpRing - 1))), sh) & mask;
  }
}

template <int DELTA>
__global__ void __launch_bounds__(IZG_TEAM_LB_THREADS, IZG_BPTEAM_MINCTAS)
    bp_team_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                   uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                   uint32_t* __restrict__ consumed, uint32_t* __restrict__ next_chunk,
                   const __grid_constant__ CUtensorMap omap, int tma_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using LY = BpTeamLayout;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t sb = smem_u32(smem);
  asm volatile("mov.u32 %0, %0;" : "+r"(sb));  // one register, never rematerialised
  if (tid == 0) {
    for (uint32_t i = 0; i < kBpPieces; ++i) mbar_init_s(sb + LY::kPieceBar + 8u * i, 1);
    for (uint32_t i = 0; i < kBpSlots; ++i) {
      mbar_init_s(sb + LY::kFull + 8u * i, 1);
      mbar_init_s(sb + LY::kEmpty + 8u * i, kTeamWarps);
    }
    for (uint32_t i = 0; i < kTeamWarps; ++i) mbar_init_s(sb + LY::kMbx + 8u * i, 1);
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init_s(sb + LY::kPfull + 8u * i, 1);
      mbar_init_s(sb + LY::kPdone + 8u * i, kTeamWarps - 1);
      mbar_init_s(sb + LY::kPfree + 8u * i, 1);
    }
    fence_barrier_init();
    if (kArray) {  // the first chunk's initial carry, posted to warp 0's mailbox
      sts128(sb + LY::kTot, 0, 0, 0, 0);
      mbar_arrive_s(sb + LY::kMbx);
    }
  }
  __syncthreads();

  if (warp == kTeamWarps) {
    // ======================= staging warp ====================================
    const uint64_t policy = policy_evict_first();
    uint32_t gp = 0;        // pieces issued so far (all chunks)
    uint32_t gw = 0;        // pieces known landed (waited)
    uint32_t gi = 0, gd = 0;  // super-iterations published / read by every warp (all chunks)
    uint32_t cons = 0;      // unmasked ring byte below which everything has been read
    uint32_t cur_start = 0; // first ring byte of the super-iteration being prepared
    uint32_t pcount = 0;    // chunks handed to the decoding warps
    auto claim = [&]() -> uint32_t {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(next_chunk, 1u);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      if (c < n_chunks && lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(chunks + c));
      return c;
    };
    // one `empty` phase: the oldest published super-iteration has been read by every warp
    auto retire = [&](bool block) -> bool {
      if (gd == gi) return false;
      const uint32_t bar = sb + LY::kEmpty + 8u * (gd % kBpSlots), par = (gd / kBpSlots) & 1u;
      uint32_t ok = 1;
      if (block)
        mbar_wait_s(bar, par);
      else {
        if (lane == 0) ok = mbar_test_s(bar, par);
        ok = __shfl_sync(0xFFFFFFFFu, ok, 0);
      }
      if (!ok) return false;
      ++gd;
      // everything below the next unread super-iteration's first byte is free
      cons = gd == gi ? cur_start : lds32(sb + LY::kStart + 4u * (gd % kBpSlots));
      return true;
    };
    uint32_t c_next = claim();
    for (;;) {
      const uint32_t c = c_next;
      const uint32_t pp = pcount & 1u;
      if (c >= n_chunks) {  // no more chunks: tell the decoding warps
        if (pcount >= 2) mbar_wait_s(sb + LY::kPfree + 8u * pp, ((pcount >> 1) - 1u) & 1u);
        if (lane == 0) {
          sts128(sb + LY::kDesc + 64u * pp, 0, 1u, 0, 0);
          mbar_arrive_s(sb + LY::kPfull + 8u * pp);
        }
        break;
      }
      c_next = claim();
      const izg_chunk ch = chunks[c];
      int32_t st = precheck(IZG_SIMDBP128, kArray, ch.n);
      const uint32_t* p = words + ch.word_off;
      const uint32_t nb = (kArray ? ch.n / 128 * 128 : ch.n) / 128;
      if (st != IZG_OK || nb == 0) {
        team_finish<DELTA>(st, 0, make_uint4(0, 0, 0, 0), ch, p, out + ch.out_off, c, status,
                           consumed, lane);
        continue;
      }
      const uint32_t nw = ch.n_words;
      const uint32_t K = (nb + kTeamSI - 1) / kTeamSI;
      if (pcount >= 2) mbar_wait_s(sb + LY::kPfree + 8u * pp, ((pcount >> 1) - 1u) & 1u);
      if (lane == 0) {
        const uint32_t d = sb + LY::kDesc + 64u * pp;
        sts128(d, c, 0, nb, K);
        sts128(d + 16, 0, 0, ch.n, ch.n_words);
        sts128(d + 32, (uint32_t)ch.word_off, (uint32_t)(ch.word_off >> 32), (uint32_t)ch.out_off,
               (uint32_t)(ch.out_off >> 32));
        mbar_arrive_s(sb + LY::kPfull + 8u * pp);
      }
      ++pcount;

      // the chunk's 16-byte-aligned span, as pieces gp0 .. gp0 + npieces - 1
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(p);
      const uintptr_t s16 = a0 & ~uintptr_t(15);
      const uint32_t total = (uint32_t)(((a0 + 4ull * nw + 15) & ~uintptr_t(15)) - s16);
      const uint32_t npieces = (total + kBpPiece - 1) / kBpPiece;
      const uint32_t gp0 = gp;
      const uint32_t off0 = gp0 * kBpPiece + (uint32_t)(a0 - s16);  // unmasked ring byte of payload byte 0
      const BpRingView rv{sb + LY::kRing, off0};
      for (; gw < gp; ++gw)  // copies of the chunk before that nothing waited for
        mbar_wait_s(sb + LY::kPieceBar + 8u * (gw % kBpPieces), (gw / kBpPieces) & 1u);
      cur_start = off0;
      if (gd == gi) cons = cur_start;
      // issue pieces while the ring has room: the pieces from `cons` on must stay
      auto issue = [&]() {
        while (gp < gp0 + npieces && gp < cons / kBpPiece + kBpPieces) {
          if (lane == 0) {
            const uint32_t i = gp - gp0, sl = gp % kBpPieces;
            const uint32_t bytes = min(kBpPiece, total - i * kBpPiece);
            const uint32_t bar = sb + LY::kPieceBar + 8u * sl;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx_s(bar, bytes);
            bulk_g2s_s(sb + LY::kRing + sl * kBpPiece,
                       reinterpret_cast<const uint8_t*>(s16) + (size_t)i * kBpPiece, bytes, bar, policy);
          }
          ++gp;
        }
      };
      // chunk bytes [0, end) (payload-relative) have landed
      auto need = [&](uint32_t end) {
        const uint32_t last = gp0 + min(npieces, ((uint32_t)(a0 - s16) + end + kBpPiece - 1) / kBpPiece);
        for (;;) {
          issue();
          if (gp >= last) break;
          retire(true);  // the ring is full of unread data: wait for the decoders
        }
        for (; gw < last; ++gw)
          mbar_wait_s(sb + LY::kPieceBar + 8u * (gw % kBpPieces), (gw / kBpPieces) & 1u);
      };
      uint32_t pos = 0;  // payload word of the next descriptor
      for (uint32_t j = 0; j < K; ++j, ++gi) {
        while (gi >= gd + kBpSlots) retire(true);
        while (retire(false)) {
        }
        const uint32_t tab = sb + LY::kTab + (gi % kBpSlots) * (kTeamSI * 8u);
        cur_start = off0 + 4u * pos;  // first byte of this super-iteration
        if (gd == gi) cons = cur_start;
        if (lane == 0) sts32(sb + LY::kStart + 4u * (gi % kBpSlots), cur_start);
#pragma unroll 1
        for (uint32_t h = 0; h < 2; ++h) {
          const uint32_t mb0 = j * kTeamSI + 16u * h;
          uint32_t wv = 0, ra = off0;  // a dead block: width 0 at a valid place
          if (mb0 < nb && st == IZG_OK) {
            const uint32_t groups = min(16u, nb - mb0);
            if (pos + 4 > nw) {
              st = IZG_E_BP_TRUNC_DESC;
            } else {
              need(4u * (pos + 4));
              MetaWalk m;
              if ((off0 & 15u) == 0)
                m = walk_meta<true>(rv, pos, groups, nw, lane);
              else
                m = walk_meta<false>(rv, pos, groups, nw, lane);
              if (m.err) {
                st = m.err;
              } else {
                need(4u * (pos + 4 + m.size));
                if ((uint32_t)(lane & 15) < groups) {
                  wv = m.width;
                  ra = off0 + 4u * (pos + 4 + m.excl);
                }
                pos += 4 + m.size;
              }
            }
          }
          if (lane < 16) sts64(tab + 8u * (16u * h + lane), wv, ra);
        }
        if (j + 1 == K && lane == 0) sts64(sb + LY::kEnd + 8u * pp, pos, (uint32_t)st);
        __syncwarp();
        if (lane == 0) mbar_arrive_s(sb + LY::kFull + 8u * (gi % kBpSlots));
      }
    }
    return;
  }

  // ========================= decoding warps ==================================
  const uint32_t q = lane >> 3, s8 = lane & 7;
  TeamTile tile;
  tile.init(sb + LY::kTiles + 2 * warp * kStageOut, lane, &omap);  // two tiles, alternating
  uint32_t git = 0;  // super-iterations consumed so far, all chunks (slot and parity)
  for (uint32_t pcount = 0;; ++pcount) {
    const uint32_t pp = pcount & 1u;
    team_wait(sb + LY::kPfull + 8u * pp, (pcount >> 1) & 1u);
    const uint4 d0 = lds128(sb + LY::kDesc + 64u * pp);
    if (d0.y & 1u) break;
    const uint4 d1 = lds128(sb + LY::kDesc + 64u * pp + 16);
    const uint4 d2 = lds128(sb + LY::kDesc + 64u * pp + 32);
    const uint32_t c = d0.x, nb = d0.z, K = d0.w;
    izg_chunk ch;
    ch.word_off = (uint64_t)d2.y << 32 | d2.x;
    ch.out_off = (uint64_t)d2.w << 32 | d2.z;
    ch.n = d1.z;
    ch.n_words = d1.w;
    const uint32_t* p = words + ch.word_off;
    uint32_t* o = out + ch.out_off;
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    const int64_t orow = tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5) : -1;
    const bool pal = (reinterpret_cast<uintptr_t>(p) & 15) == 0;  // rows 16-byte aligned
    uint4 fin = make_uint4(0, 0, 0, 0);  // warp 7, lane 31: the chunk's final carry
#pragma unroll 1
    for (uint32_t k = 0; k < K; ++k, ++git) {
      const uint32_t slot = git % kBpSlots;
      team_wait(sb + LY::kFull + 8u * slot, (git / kBpSlots) & 1u);
      const uint32_t blk0 = k * kTeamSI + 4u * warp;
      const bool live = blk0 + q < nb;
      const uint2 e = lds64(sb + LY::kTab + slot * (kTeamSI * 8u) + 8u * (4u * warp + q));
      uint32_t v[4][4];
      if (pal)
        unpack_slots_aligned(BpRingView{sb + LY::kRing, 0u}, e.y, e.x, s8, v);
      else
        bp_unpack_words(sb + LY::kRing, e.y, e.x, s8, v);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(sb + LY::kEmpty + 8u * slot);  // done with the ring and the table
      if (kArray) {
        uint4 ex, incl;
        uint32_t q3[4] = {0, 0, 0, 0};
        team_scan_local<DELTA>(v, ex, incl, q3, lane);
        team_wait(sb + LY::kMbx + 8u * warp, git & 1u);
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
      if (orow >= 0 && blk0 + 4 <= nb) {
        const uint32_t tb = (git & 1u) * kStageOut;  // the other tile's store may still be reading
        if (tile.leader) bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sts128(tile.addr(kk) + tb, v[kk][0], v[kk][1], v[kk][2], v[kk][3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (tile.leader) {
          tma_store_2d(tile.tmap, tile.t + tb, 0, (int)(uint32_t)(orow + 4 * (int64_t)blk0));
          bulk_commit();
        }
      } else {
        __syncwarp();
        if (live) store_direct(v, o + (size_t)(blk0 + q) * 128 + 16 * s8, oal);
      }
    }
    // ---- end of the chunk -------------------------------------------------------
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
      const uint2 en = lds64(sb + LY::kEnd + 8u * pp);
      team_finish<DELTA>((int32_t)en.y, en.x, carry, ch, p, o, c, status, consumed, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(sb + LY::kPfree + 8u * pp);
    }
  }
  tile.drain();
}

}  // namespace izg
