// cta.cuh — SIMD-BP128 decode with a whole CTA per SM cooperating on each
// chunk (small and mid-size batches: C1's 1,024 chunks, C3's 4,096).
//
// Why: one warp per chunk is a dependent chain of 128 warp iterations
// (~1,750 cycles each), so a batch with fewer chunks than the
// ~3,500 resident warp slots is latency-bound (C1: 7 warps per SM, 12%
// occupancy).  The group kernel (group.cuh) lets a few warps share a chunk,
// but every one of them streams the whole chunk through its own ring.
//
// Here one persistent CTA per SM runs a warp-specialised pipeline over a
// SINGLE shared staging ring (kCtaRing bytes of 4 KiB pieces, TMA bulk
// copies, one mbarrier per piece):
//   * producer warp (the last one): claims chunks (one atomic each),
//     publishes each chunk's record in a slot, copies the chunk's compressed
//     span into the ring piece by piece as consumers free space, and walks
//     the meta-block descriptor chain in shared memory (codec_binpack.cpp:
//     94-119, walk_meta: every width / truncation check in the reference's
//     order), publishing each meta-block's payload position in the slot's
//     table;
//   * kCtaConsumers consumer warps: the chunk stream is cut into UNITS of
//     eight blocks (half a meta-block, 1,024 integers, two warp iterations);
//     unit U belongs to warp U % kCtaConsumers, so the warps work on
//     consecutive units of the same chunk at once.  A unit is unpacked and
//     prefix-summed from a zero carry in registers, then waits for the carry
//     out of unit U-1 in a shared-memory mailbox (group.cuh's mbx_wait /
//     mbx_post), adds it, posts its own, frees the ring up to its end, and
//     stores both iterations with TMA tensor stores.  The chain between
//     warps is one mailbox hop per 1,024 integers; every compressed byte is
//     read from HBM once and every integer written once.
//   The last unit of a chunk decodes the VByte remainder from the final
//   carry (codec.cpp:56-62), checks exact consumption (codec.cpp:63-64) and
//   writes the chunk's status and words consumed.
// Statuses equal the one-warp kernel's: the producer's walk finds the first
// failing meta-block; units from that meta-block on are not decoded.
#pragma once
#include "group.cuh"

namespace izg {

constexpr int kCtaConsumers = 16;
constexpr int kCtaWarps = kCtaConsumers + 1;
constexpr uint32_t kCtaPiece = 4096;                      // bytes per ring piece
constexpr uint32_t kCtaPieces = 32;                        // pieces in the ring
constexpr uint32_t kCtaRing = kCtaPiece * kCtaPieces;      // 128 KiB
constexpr uint32_t kCtaSlots = 8;                          // chunk records in flight
constexpr uint32_t kCtaUnitBlocks = 8;                     // blocks per unit
constexpr uint32_t kCtaSpin = 1u << 26;                    // stuck chain: report, do not hang

// Per-chunk record published by the producer (shared memory, volatile use).
struct CtaSlot {
  uint32_t seq;        // chunk sequence number (the slot's validity tag)
  uint32_t chunk;      // index in the chunk table
  uint32_t piece0;     // global index of the chunk's first ring piece
  uint32_t phase;      // payload word 0's byte offset in its 16-byte span
  uint32_t nw, n, nblocks;
  uint32_t u0, nunits; // the chunk's units: [u0, u0 + nunits) of the stream
  uint32_t npieces;
  uint32_t walked;     // meta-blocks whose table entry is valid
  uint32_t walk_done;  // 1 once the walk ended (walk_err / end_pos final)
  int32_t walk_err;    // first error of the walk (or of the length check)
  uint32_t end_pos;    // payload word after the last meta-block
  uint32_t pad[2];
  uint32_t table[32];  // payload word of each meta-block's descriptor
};

struct CtaLayout {
  static constexpr uint32_t kRingOff = 0;
  static constexpr uint32_t kTileOff = kCtaRing;                              // 2 tiles / consumer
  static constexpr uint32_t kSlotOff = kTileOff + kCtaConsumers * 2 * kStageOut;
  static constexpr uint32_t kMbxOff = kSlotOff + kCtaSlots * sizeof(CtaSlot);  // 32 B / consumer
  static constexpr uint32_t kCtlOff = kMbxOff + kCtaConsumers * 32;            // control words
  static constexpr uint32_t kBarOff = (kCtlOff + 64 + 7) & ~7u;                // piece mbarriers
  static constexpr size_t kSmem = kBarOff + kCtaPieces * 8;
};
// control words (u32 at kCtlOff + 4 * k)
//   published: chunk records published (slots 0 .. published-1 valid unless recycled)
//   total:     chunk records the producer will ever publish (~0 until known)
//   release:   ring pieces below this global index are free (consumers, in chain order)
//   done:      chunks completed, in order (the last unit of chunk k sets it to k + 1)
//   issued:    ring pieces issued so far (a piece's mbarrier phase is only waited on
//              once it is issued, so parity waits never see a stale phase)
enum { kCtlPublished = 0, kCtlTotal = 1, kCtlRelease = 2, kCtlDone = 3, kCtlIssued = 4 };

// Read-only view of the ring for the walk / unpack helpers (decode_bp128.cuh).
struct CtaView {
  static constexpr uint32_t kMask = kCtaRing - 1;
  uint32_t base;  // ring
  uint32_t off;   // unmasked ring byte of payload byte 0
  __device__ __forceinline__ uint32_t addr(uint32_t o) const { return base + ((off + o) & kMask); }
  __device__ __forceinline__ uint32_t word_addr(uint32_t w) const { return addr(4u * w); }
  __device__ __forceinline__ uint32_t ring_off() const { return off; }
};

__device__ __forceinline__ uint32_t ldv(uint32_t a) { return lds32_volatile(a); }
__device__ __forceinline__ void stv(uint32_t a, uint32_t v) { sts32_volatile(a, v); }

// Wait (all lanes) for ring pieces [waited, to) (global indices) to land.
// `waited` must not lie below a piece that may have been recycled.
__device__ __forceinline__ void cta_wait_pieces(uint32_t bars, uint32_t& waited, uint32_t to) {
  for (; waited < to; ++waited)
    mbar_wait_s(bars + 8u * (waited % kCtaPieces), (waited / kCtaPieces) & 1u);
}
// Consumer side: the pieces must also have been issued (otherwise their
// barrier still shows the previous lap's phase).
__device__ __forceinline__ void cta_wait_issued(uint32_t ctl, uint32_t bars, uint32_t& waited,
                                                uint32_t from, uint32_t to, bool* stalled) {
  if (waited < from) waited = from;
  if (waited >= to) return;
  for (uint32_t spin = 0; lds32_volatile(ctl + 4 * kCtlIssued) < to;) {
    if (++spin > kCtaSpin) {
      *stalled = true;
      return;
    }
  }
  cta_wait_pieces(bars, waited, to);
}

template <int DELTA>
__global__ void __launch_bounds__(kCtaWarps * 32, 1)
    cta_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
               uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
               uint32_t* __restrict__ consumed, uint32_t* __restrict__ next_chunk,
               const __grid_constant__ CUtensorMap omap, int tma_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring = smem_u32(smem + CtaLayout::kRingOff);
  const uint32_t bars = smem_u32(smem + CtaLayout::kBarOff);
  const uint32_t ctl = smem_u32(smem + CtaLayout::kCtlOff);
  const uint32_t slots = smem_u32(smem + CtaLayout::kSlotOff);
  CtaSlot* slotp = reinterpret_cast<CtaSlot*>(smem + CtaLayout::kSlotOff);
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < kCtaPieces; ++i) mbar_init_s(bars + 8u * i, 1);
    for (uint32_t i = 0; i < 16; ++i) stv(ctl + 4 * i, 0);
    stv(ctl + 4 * kCtlTotal, 0xFFFFFFFFu);
    for (uint32_t i = 0; i < kCtaSlots; ++i) stv(slots + i * sizeof(CtaSlot), 0xFFFFFFFFu);
    for (uint32_t i = 0; i < kCtaConsumers; ++i)
      stv(smem_u32(smem + CtaLayout::kMbxOff + 32 * i) + 16, 0xFFFFFFFFu);
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCtaConsumers) {
    // ---------------------------------------------------------------- producer
    const uint64_t policy = policy_evict_first();
    uint32_t seq = 0, piece_next = 0, u_next = 0, waited = 0;
    for (;; ++seq) {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(next_chunk, 1u);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      if (c >= n_chunks) break;
      // the slot is free once the chunk that last used it is done
      if (seq >= kCtaSlots) {
        uint32_t n = 0;
        while (ldv(ctl + 4 * kCtlDone) + kCtaSlots <= seq && ++n < kCtaSpin) {
        }
      }
      const izg_chunk ch = chunks[c];
      const int32_t pre = precheck(IZG_SIMDBP128, kArray, ch.n);
      const uint32_t core = pre ? 0u : (kArray ? ch.n / 128 * 128 : ch.n);
      const uint32_t nblocks = core / 128;
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(words + ch.word_off);
      const uintptr_t s16 = a0 & ~uintptr_t(15);
      const uint32_t nw = pre ? 0u : ch.n_words;
      const uint32_t total = nw ? (uint32_t)(((a0 + 4ull * nw + 15) & ~uintptr_t(15)) - s16) : 0u;
      const uint32_t npieces = (total + kCtaPiece - 1) / kCtaPiece;
      const uint32_t nunits = max(1u, (nblocks + kCtaUnitBlocks - 1) / kCtaUnitBlocks);
      const uint32_t sa = slots + (seq % kCtaSlots) * sizeof(CtaSlot);
      if (lane == 0) {
        CtaSlot* S = slotp + seq % kCtaSlots;
        S->chunk = c;
        S->piece0 = piece_next;
        S->phase = (uint32_t)(a0 - s16);
        S->nw = nw;
        S->n = ch.n;
        S->nblocks = nblocks;
        S->u0 = u_next;
        S->nunits = nunits;
        S->npieces = npieces;
        S->walked = 0;
        S->walk_done = pre ? 1u : 0u;
        S->walk_err = pre;
        S->end_pos = 0;
        __threadfence_block();
        stv(sa, seq);  // the tag last: the record is valid
        __threadfence_block();
        stv(ctl + 4 * kCtlPublished, seq + 1);
      }
      __syncwarp();
      const CtaView vw{ring, (piece_next % kCtaPieces) * kCtaPiece + (uint32_t)(a0 - s16)};
      uint32_t issued = 0, pos = 0, mb = 0;
      bool walking = !pre && nblocks > 0;
      int32_t err = IZG_OK;
      uint32_t spin = 0;
      while (issued < npieces || walking) {
        // 1. copies, as far as the consumers have freed the ring
        if (issued < npieces) {
          const uint32_t rel = ldv(ctl + 4 * kCtlRelease);
          const uint32_t i0 = issued;
          while (issued < npieces && piece_next + issued < rel + kCtaPieces) {
            if (lane == 0) {
              const uint32_t k = piece_next + issued, sl = k % kCtaPieces;
              const uint32_t bytes = min(kCtaPiece, total - issued * kCtaPiece);
              fence_proxy_async_smem();
              mbar_arrive_expect_tx_s(bars + 8u * sl, bytes);
              bulk_g2s_s(ring + sl * kCtaPiece,
                         reinterpret_cast<const uint8_t*>(s16) + (size_t)issued * kCtaPiece, bytes,
                         bars + 8u * sl, policy);
            }
            ++issued;
          }
          if (issued != i0) {
            spin = 0;
            if (lane == 0) stv(ctl + 4 * kCtlIssued, piece_next + issued);
          }
        }
        // 2. the walk, as far as the landed data goes
        bool progressed = false;
        while (walking) {
          const uint32_t groups = min(16u, nblocks - 16 * mb);
          if (pos + 4 > nw) {
            err = IZG_E_BP_TRUNC_DESC;
            walking = false;
            break;
          }
          const uint32_t need = (vw.off % kCtaPiece + 4u * (pos + 4) + kCtaPiece - 1) / kCtaPiece;
          if (need > issued) break;  // descriptor not copied yet
          cta_wait_pieces(bars, waited, piece_next + need);
          const MetaWalk m = walk_meta<false>(vw, pos, groups, nw, lane);
          if (m.err) {
            err = m.err;
            walking = false;
            break;
          }
          if (lane == 0) {
            CtaSlot* S = slotp + seq % kCtaSlots;
            S->table[mb] = pos;
            __threadfence_block();
            stv(sa + offsetof(CtaSlot, walked), mb + 1);
          }
          pos += 4 + m.size;
          ++mb;
          progressed = true;
          if (16 * mb >= nblocks) walking = false;
        }
        if (!walking && !(issued < npieces)) break;
        if (progressed) spin = 0;
        else if (++spin > kCtaSpin) {  // a broken pipeline: report, do not hang
          err = IZG_E_SPLIT_STALL;
          walking = false;
        }
        __syncwarp();
      }
      if (lane == 0) {
        CtaSlot* S = slotp + seq % kCtaSlots;
        if (!pre) {
          S->walk_err = err;
          S->end_pos = pos;
        }
        __threadfence_block();
        stv(sa + offsetof(CtaSlot, walk_done), 1u);
      }
      // copies still outstanding (a walk error stopped early): issue them so
      // the piece sequence stays consistent for the consumers' waits
      while (issued < npieces) {
        const uint32_t rel = ldv(ctl + 4 * kCtlRelease);
        while (issued < npieces && piece_next + issued < rel + kCtaPieces) {
          if (lane == 0) {
            const uint32_t k = piece_next + issued, sl = k % kCtaPieces;
            const uint32_t bytes = min(kCtaPiece, total - issued * kCtaPiece);
            fence_proxy_async_smem();
            mbar_arrive_expect_tx_s(bars + 8u * sl, bytes);
            bulk_g2s_s(ring + sl * kCtaPiece,
                       reinterpret_cast<const uint8_t*>(s16) + (size_t)issued * kCtaPiece, bytes,
                       bars + 8u * sl, policy);
            stv(ctl + 4 * kCtlIssued, k + 1);
          }
          ++issued;
        }
        __syncwarp();
      }
      // the producer's own waits must not fall behind the pieces it skips
      waited = max(waited, piece_next + npieces);
      piece_next += npieces;
      u_next += nunits;
    }
    if (lane == 0) stv(ctl + 4 * kCtlTotal, seq);
    // drain: the pieces issued last must land before the CTA may exit
    for (uint32_t k = piece_next >= kCtaPieces ? piece_next - kCtaPieces : 0; k < piece_next; ++k)
      mbar_wait_s(bars + 8u * (k % kCtaPieces), (k / kCtaPieces) & 1u);
    return;
  }

  // ---------------------------------------------------------------- consumers
  const uint32_t q = lane >> 3, s8 = lane & 7;
  OutStage os;
  os.base = smem_u32(smem + CtaLayout::kTileOff + warp * 2 * kStageOut);
  os.leader = lane == 0;
  os.buf = 0;
  os.tmap = &omap;
  const uint32_t mbx_base = smem_u32(smem + CtaLayout::kMbxOff);
  uint32_t waited = 0;  // ring pieces this warp has waited for (global index)
  uint32_t si = 0;      // slot sequence number of the current chunk
  bool stalled = false;
  for (uint32_t U = (uint32_t)warp;; U += kCtaConsumers) {
    // ---- the chunk that holds unit U
    uint32_t sa = 0;
    bool found = false, ended = false;
    for (uint32_t spin = 0; !found && !ended;) {
      const uint32_t pub = ldv(ctl + 4 * kCtlPublished);
      if (si >= pub) {
        if (ldv(ctl + 4 * kCtlTotal) <= si) ended = true;
        else if (++spin > kCtaSpin) ended = stalled = true;
        continue;
      }
      sa = slots + (si % kCtaSlots) * sizeof(CtaSlot);
      const uint32_t t1 = ldv(sa);
      const uint32_t u0 = ldv(sa + offsetof(CtaSlot, u0));
      const uint32_t nu = ldv(sa + offsetof(CtaSlot, nunits));
      __threadfence_block();
      const uint32_t t2 = ldv(sa);
      if (t1 != si || t2 != si) {  // recycled: that chunk is done, U lies further on
        ++si;
        continue;
      }
      if (U < u0 + nu) found = true;
      else ++si;
    }
    if (ended) break;
    const CtaSlot* S = slotp + si % kCtaSlots;
    const uint32_t c = ldv(sa + offsetof(CtaSlot, chunk));
    const uint32_t u = U - ldv(sa + offsetof(CtaSlot, u0));
    const uint32_t nunits = ldv(sa + offsetof(CtaSlot, nunits));
    const uint32_t piece0 = ldv(sa + offsetof(CtaSlot, piece0));
    const uint32_t phase = ldv(sa + offsetof(CtaSlot, phase));
    const uint32_t nw = ldv(sa + offsetof(CtaSlot, nw));
    const uint32_t nblocks = ldv(sa + offsetof(CtaSlot, nblocks));
    const uint32_t npieces = ldv(sa + offsetof(CtaSlot, npieces));
    const izg_chunk ch = chunks[c];
    const CtaView vw{ring, (piece0 % kCtaPieces) * kCtaPiece + phase};
    uint32_t* o = out + ch.out_off;
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    const int64_t orow = tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5) : -1;
    // ---- the unit's meta-block: wait for its table entry (or the walk's end)
    const uint32_t mb = u / 2, half = u & 1;
    bool live = nblocks > 0;
    uint32_t pos = 0;
    if (live) {
      for (uint32_t spin = 0;;) {
        if (ldv(sa + offsetof(CtaSlot, walked)) > mb) break;
        if (ldv(sa + offsetof(CtaSlot, walk_done))) {
          if (ldv(sa + offsetof(CtaSlot, walked)) <= mb) live = false;
          break;
        }
        if (++spin > kCtaSpin) {
          stalled = true;
          live = false;
          break;
        }
      }
      __threadfence_block();
      if (live) pos = S->table[mb];
    }
    // ---- unpack + local scan of the unit's (up to) two iterations
    uint4 local = make_uint4(0, 0, 0, 0);
    uint32_t v[2][4][4];
    uint32_t g_lo = 0, groups = 0;
    uint32_t endw = 0;  // payload word after the unit's last block
    if (live) {
      groups = min(16u, nblocks - 16 * mb);
      g_lo = 8 * half;
      // descriptor + the unit's blocks: landed?  (phase < 16: byte b of the
      // chunk span is byte phase + b of its first piece)
      const uint32_t first_piece = piece0 + (phase + 4u * pos) / kCtaPiece;
      cta_wait_issued(ctl, bars, waited, first_piece,
                      piece0 + (phase + 4u * (pos + 4) + kCtaPiece - 1) / kCtaPiece, &stalled);
      const MetaWalk m = walk_meta<false>(vw, pos, groups, nw, lane);  // checked by the producer
      const uint32_t pay = pos + 4;
      const uint32_t lastg = min(g_lo + 7, groups - 1);
      endw = pay + __shfl_sync(0xFFFFFFFFu, m.excl + 4 * m.width, lastg);
      cta_wait_issued(ctl, bars, waited, first_piece,
                      piece0 + (phase + 4u * endw + kCtaPiece - 1) / kCtaPiece, &stalled);
#pragma unroll
      for (uint32_t it = 0; it < 2; ++it) {
        const uint32_t g0 = g_lo + 4 * it;
        const uint32_t gi = g0 + q;
        const bool active = gi < groups && g0 < groups;
        uint32_t width = __shfl_sync(0xFFFFFFFFu, m.width, gi & 15);
        const uint32_t excl = __shfl_sync(0xFFFFFFFFu, m.excl, gi & 15);
        if (!active) width = 0;
        if (phase == 0)
          unpack_slots_aligned(vw, vw.ring_off() + 4u * (pay + excl), width, s8, v[it]);
        else
          unpack_slots_unaligned(vw, pay + excl, width, s8, v[it]);
        if (kArray) scan<DELTA>(v[it], local, lane);
      }
    }
    // ---- the carry chain (one hop per unit, across chunks too, so the
    // ring's release point only ever moves forward)
    const uint32_t my_mbx = mbx_base + 32 * (U % kCtaConsumers);
    uint4 cin = make_uint4(0, 0, 0, 0);
    if (U > 0) {
      const uint4 prev =
          mbx_wait(mbx_base + 32 * ((U - 1) % kCtaConsumers), U - 1, lane, &stalled);
      if (u > 0) cin = prev;  // a chunk's first unit starts from zero
    }
    if (kArray && live) {
      add_carry<DELTA>(v[0], cin);
      add_carry<DELTA>(v[1], cin);
    }
    const uint4 cout = u4add(cin, local);
    // every read of this unit's ring bytes is done: free up to its end
    __syncwarp();
    fence_proxy_async_smem();
    if (lane == 0) {
      // a meta-block's first half keeps its descriptor (the second half
      // re-reads it); its second half, or the chunk's last unit, frees all
      const uint32_t rel = u + 1 == nunits ? piece0 + npieces
                           : !live         ? 0u
                           : half == 0     ? piece0 + (phase + 4u * pos) / kCtaPiece
                                           : piece0 + (phase + 4u * endw) / kCtaPiece;
      if (rel > ldv(ctl + 4 * kCtlRelease)) stv(ctl + 4 * kCtlRelease, rel);
    }
    mbx_post(my_mbx, cout, U, lane);
    // ---- stores
    if (live) {
#pragma unroll
      for (uint32_t it = 0; it < 2; ++it) {
        const uint32_t g0 = g_lo + 4 * it;
        if (g0 >= groups) break;
        const uint32_t gi = g0 + q;
        const uint32_t blk0 = 16 * mb + g0;
        if (orow >= 0 && g0 + 4 <= groups) {
          os.put(v[it], lane, (uint32_t)(orow + 4 * blk0));
        } else {
          os.direct(v[it], o + (size_t)(16 * mb + gi) * 128 + 16 * s8, oal, gi < groups,
                    128u * min(4u, groups - g0), lane);
        }
      }
    }
    // ---- the chunk's last unit: remainder, consumption, status
    if (u + 1 == nunits) {
      // the walk is final once it published its end (all units are past it)
      for (uint32_t spin = 0; !ldv(sa + offsetof(CtaSlot, walk_done)) && ++spin < kCtaSpin;) {
      }
      __threadfence_block();
      int32_t st = (int32_t)ldv(sa + offsetof(CtaSlot, walk_err));
      uint32_t end = ldv(sa + offsetof(CtaSlot, end_pos));
      const uint32_t n = ch.n;
      if (stalled) st = IZG_E_SPLIT_STALL;
      const uint32_t core = kArray ? n / 128 * 128 : n;
      if (kArray && st == IZG_OK) {
        if (core < n) {  // Variable Byte remainder (codec.cpp:56-62)
          uint32_t rb = 0;
          const uint32_t* p = words + ch.word_off;
          if (lane == 0)
            st = vbyte_tail<DELTA>(reinterpret_cast<const uint8_t*>(p + end),
                                   4u * (nw - end), core, n - core, cout, o, &rb);
          st = __shfl_sync(0xFFFFFFFFu, st, 0);
          rb = __shfl_sync(0xFFFFFFFFu, rb, 0);
          if (st == IZG_OK) end += (rb + 3) / 4;
        }
        if (st == IZG_OK && end != nw) st = IZG_E_PAYLOAD_SIZE;  // codec.cpp:63-64
      }
      if (lane == 0) {
        status[c] = st;
        if (consumed) consumed[c] = st == IZG_OK ? end : 0;
        // chunks complete in order: the producer recycles a slot only once
        // every earlier chunk is done too
        for (uint32_t spin = 0; ldv(ctl + 4 * kCtlDone) != si && ++spin < kCtaSpin;) {
        }
        __threadfence_block();
        stv(ctl + 4 * kCtlDone, si + 1);
      }
    }
  }
  os.drain();
}

}  // namespace izg
