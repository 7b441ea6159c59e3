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
//     out of unit U-1 in a shared-memory mailbox (value + an mbarrier that
//     completes one phase per post: the waiting warp sleeps in
//     mbarrier.try_wait instead of spinning on a flag and stealing issue
//     slots), adds it, posts its own, frees the ring up to its end, and
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

#ifndef IZG_CTA_SLEEP
#define IZG_CTA_SLEEP 256  // ns between polls of the walk's progress
#endif
// Warp w runs on SM sub-partition w % 4.  The producer (warp 0) gets
// sub-partition 0 to itself — warps 4, 8, ... exit at once — so its serial
// descriptor walk never waits for issue slots behind consumers; the
// consumers are the other warps (consumer k = warp 4 (k / 3) + 1 + k % 3).
#ifndef IZG_CTA_GROUPS
#define IZG_CTA_GROUPS 5  // sub-partition rounds: 3 consumers each
#endif
constexpr int kCtaConsumers = 3 * IZG_CTA_GROUPS;
constexpr int kCtaWarps = 4 * IZG_CTA_GROUPS;
constexpr uint32_t kCtaPiece = 4096;                      // bytes per ring piece
#ifndef IZG_CTA_PIECES
#define IZG_CTA_PIECES 32
#endif
constexpr uint32_t kCtaPieces = IZG_CTA_PIECES;            // pieces in the ring (power of 2)
constexpr uint32_t kCtaRing = kCtaPiece * kCtaPieces;      // 128 KiB
constexpr uint32_t kCtaSlots = 8;                          // chunk records in flight
constexpr uint32_t kCtaUnitBlocks = 8;                     // blocks per unit
constexpr uint32_t kCtaSpin = 1u << 26;                    // stuck chain: report, do not hang

// Per-chunk record published by the producer (shared memory, volatile use).
// The fields consumers read per chunk sit in the first three 16-byte words
// (three vector loads).
struct __align__(16) CtaSlot {
  uint32_t seq;        // chunk sequence number (the slot's validity tag)
  uint32_t chunk;      // index in the chunk table
  uint32_t piece0;     // global index of the chunk's first ring piece
  uint32_t phase;      // payload word 0's byte offset in its 16-byte span
  uint32_t nw, n, nblocks;
  uint32_t u0;         // the chunk's units: [u0, u0 + nunits) of the stream
  uint32_t nunits;
  uint32_t npieces;
  uint32_t out_lo, out_hi;    // izg_chunk::out_off
  uint32_t word_lo, word_hi;  // izg_chunk::word_off
  uint32_t walk_done;  // 1 once the walk ended (walk_err / end_pos final)
  int32_t walk_err;    // first error of the walk (or of the length check)
  uint32_t end_pos;    // payload word after the last meta-block
  uint32_t pad[3];
  uint32_t table[32];  // payload word of each meta-block's descriptor | 1 << 31 once walked
};

__device__ __forceinline__ uint4 ldv4(uint32_t a) { return lds128_volatile(a); }

struct CtaLayout {
  static constexpr uint32_t kRingOff = 0;
  static constexpr uint32_t kTileOff = kCtaRing;                              // 2 tiles / consumer
  static constexpr uint32_t kSlotOff = kTileOff + kCtaConsumers * 2 * kStageOut;  // 16-aligned
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

// Mailbox of consumer warp k: the carry out of its latest unit (uint4 at +0)
// and an mbarrier (+16) whose phase p completes when unit 16p + k posts.
// The chain orders every post after the previous reader of the mailbox
// (unit U + 16 posts only after unit U + 1 has read unit U's carry), so a
// waiter never sees a phase two laps ahead or behind.
__device__ __forceinline__ void cta_mbx_post(uint32_t mbx, uint4 c, int lane) {
  if (lane == 0) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(mbx), "r"(c.x), "r"(c.y),
                 "r"(c.z), "r"(c.w)
                 : "memory");
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(mbx + 16)
                 : "memory");
  }
}
__device__ __forceinline__ uint4 cta_mbx_wait(uint32_t mbx, uint32_t unit, bool* stalled) {
  for (uint32_t n = 0; !mbar_try_wait_s(mbx + 16, (unit / kCtaConsumers) & 1u);)
    if (++n > kCtaSpin) {  // a broken chain is a bug: report it, never hang the GPU
      *stalled = true;
      break;
    }
  return lds128(mbx);
}

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
    __nanosleep(64);
    if (++spin > kCtaSpin) {
      *stalled = true;
      return;
    }
  }
  cta_wait_pieces(bars, waited, to);
}

#ifdef IZG_CTA_PROF  // developer build: per-warp time split of the consumers' units
__device__ unsigned long long g_cta_prof[160][kCtaWarps][8];
__device__ long long g_cta_trace[64][6];  // CTA 0: per chunk seq: claim, published, walk done, first unit, last unit done
#define CTA_T(k)                                                              \
  do {                                                                        \
    const long long _t = clock64();                                           \
    if (lane == 0) g_cta_prof[blockIdx.x][warp][k] += (unsigned long long)(_t - t_last); \
    t_last = _t;                                                              \
  } while (0)
#else
#define CTA_T(k) \
  do {           \
  } while (0)
#endif

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
      mbar_init_s(smem_u32(smem + CtaLayout::kMbxOff + 32 * i) + 16, 1);
    fence_barrier_init();
  }
  __syncthreads();

  if (warp % 4 == 0 && warp > 0) return;  // sub-partition 0 belongs to the producer
  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    const uint64_t policy = policy_evict_first();
    uint32_t seq = 0, piece_next = 0, u_next = 0, waited = 0;
    for (;; ++seq) {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(next_chunk, 1u);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      if (c >= n_chunks) break;
#ifdef IZG_CTA_PROF
      if (blockIdx.x == 0 && lane == 0 && seq < 64) g_cta_trace[seq][0] = clock64();
#endif
      // the slot is free once the chunk that last used it is done
      if (seq >= kCtaSlots) {
        uint32_t n = 0;
        while (ldv(ctl + 4 * kCtlDone) + kCtaSlots <= seq && ++n < kCtaSpin) __nanosleep(64);
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
        S->out_lo = (uint32_t)ch.out_off;
        S->out_hi = (uint32_t)(ch.out_off >> 32);
        S->word_lo = (uint32_t)ch.word_off;
        S->word_hi = (uint32_t)(ch.word_off >> 32);
        for (int k = 0; k < 32; ++k) S->table[k] = 0;  // no valid bit: not walked yet
        S->walk_done = pre ? 1u : 0u;
        S->walk_err = pre;
        S->end_pos = 0;
        __threadfence_block();
        stv(sa, seq);  // the tag last: the record is valid
        __threadfence_block();
        stv(ctl + 4 * kCtlPublished, seq + 1);
#ifdef IZG_CTA_PROF
        if (blockIdx.x == 0 && seq < 64) g_cta_trace[seq][1] = clock64();
#endif
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
        // 2. the walk, as far as the landed data goes: lane 0 hops alone (a
        // tight loop: four shared loads, dp4a, vcmpgtu4 per meta-block) and
        // publishes each meta-block's position with its valid bit in one
        // store, so consumers need no fence to read it
        bool progressed = false;
        if (walking) {
          uint32_t bad = 0;  // 1: truncated descriptor; 2: run walk_meta for the error
          if (lane == 0) {
            while (16 * mb < nblocks) {
              const uint32_t groups = min(16u, nblocks - 16 * mb);
              if (pos + 4 > nw) {
                bad = 1;
                break;
              }
              const uint32_t need = (vw.off % kCtaPiece + 4u * (pos + 4) + kCtaPiece - 1) / kCtaPiece;
              if (need > issued) break;  // descriptor not copied yet
#ifdef IZG_CTA_PROF
              const long long tw0 = clock64();
#endif
              cta_wait_pieces(bars, waited, piece_next + need);
#ifdef IZG_CTA_PROF
              g_cta_prof[blockIdx.x][warp][6] += (unsigned long long)(clock64() - tw0);
#endif
              uint32_t d[4];
              if (((vw.off + 4u * pos) & 15u) == 0) {
                const uint4 dv = lds128(vw.word_addr(pos));
                d[0] = dv.x; d[1] = dv.y; d[2] = dv.z; d[3] = dv.w;
              } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) d[k] = lds32(vw.word_addr(pos + k));
              }
              if (groups < 16) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  d[k] &= groups >= 4u * k + 4 ? 0xFFFFFFFFu
                          : groups <= 4u * k   ? 0u
                                               : (1u << (8 * (groups - 4 * k))) - 1u;
              }
              const uint32_t sum = __dp4a(d[0], 0x01010101u, __dp4a(d[1], 0x01010101u,
                                   __dp4a(d[2], 0x01010101u, __dp4a(d[3], 0x01010101u, 0u))));
              const uint32_t wide = __vcmpgtu4(d[0], 0x20202020u) | __vcmpgtu4(d[1], 0x20202020u) |
                                    __vcmpgtu4(d[2], 0x20202020u) | __vcmpgtu4(d[3], 0x20202020u);
              if (wide || (uint64_t)pos + 4 + 4ull * sum > nw) {
                bad = 2;
                break;
              }
              stv(sa + offsetof(CtaSlot, table) + 4 * mb, pos | 0x80000000u);
              pos += 4 + 4 * sum;
              ++mb;
              progressed = true;
            }
          }
          bad = __shfl_sync(0xFFFFFFFFu, bad, 0);
          pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
          mb = __shfl_sync(0xFFFFFFFFu, mb, 0);
          progressed = __shfl_sync(0xFFFFFFFFu, (uint32_t)progressed, 0) != 0;
          waited = __shfl_sync(0xFFFFFFFFu, waited, 0);
          if (bad == 1) {
            err = IZG_E_BP_TRUNC_DESC;
            walking = false;
          } else if (bad == 2) {  // the reference's first error inside this meta-block
            const MetaWalk m = walk_meta<false>(vw, pos, min(16u, nblocks - 16 * mb), nw, lane);
            err = m.err ? m.err : IZG_E_BP_TRUNC_PAYLOAD;
            walking = false;
          } else if (16 * mb >= nblocks) {
            walking = false;
          }
        }
        if (!walking && !(issued < npieces)) break;
        if (progressed) {
          spin = 0;
        } else {
          if (++spin > kCtaSpin) {  // a broken pipeline: report, do not hang
            err = IZG_E_SPLIT_STALL;
            walking = false;
          }
#ifdef IZG_CTA_PROF
          const long long ts0 = clock64();
#endif
          __nanosleep(32);
#ifdef IZG_CTA_PROF
          if (lane == 0) g_cta_prof[blockIdx.x][warp][7] += (unsigned long long)(clock64() - ts0);
#endif
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
#ifdef IZG_CTA_PROF
        if (blockIdx.x == 0 && seq < 64) g_cta_trace[seq][2] = clock64();
#endif
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
  const uint32_t ci = (uint32_t)(warp / 4) * 3 + (uint32_t)(warp % 4) - 1;  // consumer index
  os.base = smem_u32(smem + CtaLayout::kTileOff + ci * 2 * kStageOut);
  os.leader = lane == 0;
  os.buf = 0;
  os.tmap = &omap;
  const uint32_t mbx_base = smem_u32(smem + CtaLayout::kMbxOff);
  uint32_t waited = 0;  // ring pieces this warp has waited for (global index)
  uint32_t si = 0;      // slot sequence number of the current chunk
  bool stalled = false;
#ifdef IZG_CTA_PROF
  long long t_last = clock64();
#endif
  // the current chunk's record, cached across this warp's units of it
  uint32_t sa = 0, c = 0, u0 = 0, nunits = 0, piece0 = 0, phase = 0, nw = 0, n = 0;
  uint32_t nblocks = 0, npieces = 0;
  uint64_t out_off = 0, word_off = 0;
  bool have = false;
  for (uint32_t U = ci;; U += kCtaConsumers) {
    // ---- the chunk that holds unit U
    bool ended = false;
    if (!have || U >= u0 + nunits) {
      have = false;
      for (uint32_t spin = 0; !have && !ended;) {
        const uint32_t pub = ldv(ctl + 4 * kCtlPublished);
        if (si >= pub) {
          if (ldv(ctl + 4 * kCtlTotal) <= si) ended = true;
          else if (++spin > kCtaSpin) ended = stalled = true;
          else __nanosleep(64);
          continue;
        }
        sa = slots + (si % kCtaSlots) * sizeof(CtaSlot);
        const uint4 w0 = ldv4(sa), w1 = ldv4(sa + 16), w2 = ldv4(sa + 32), w3 = ldv4(sa + 48);
        __threadfence_block();
        const uint32_t t2 = ldv(sa);
        if (w0.x != si || t2 != si) {  // recycled: that chunk is done, U lies further on
          ++si;
          continue;
        }
        c = w0.y;
        piece0 = w0.z;
        phase = w0.w;
        nw = w1.x;
        n = w1.y;
        nblocks = w1.z;
        u0 = w1.w;
        nunits = w2.x;
        npieces = w2.y;
        out_off = (uint64_t)w2.w << 32 | w2.z;
        word_off = (uint64_t)w3.y << 32 | w3.x;
        if (U < u0 + nunits) have = true;
        else ++si;
      }
    }
    if (ended) break;
    CTA_T(0);  // finding the unit's chunk
    const uint32_t u = U - u0;
#ifdef IZG_CTA_PROF
    if (blockIdx.x == 0 && lane == 0 && u == 0 && si < 64) g_cta_trace[si][3] = clock64();
#endif
    const CtaView vw{ring, (piece0 % kCtaPieces) * kCtaPiece + phase};
    uint32_t* o = out + out_off;
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    const int64_t orow = tma_out && (out_off & 31) == 0 ? (int64_t)(out_off >> 5) : -1;
    // ---- the unit's meta-block: wait for its table entry (or the walk's end)
    const uint32_t mb = u / 2, half = u & 1;
    bool live = nblocks > 0;
    uint32_t pos = 0;
    if (live) {
      for (uint32_t spin = 0;;) {
        const uint32_t t = ldv(sa + offsetof(CtaSlot, table) + 4 * mb);
        if (t >> 31) {
          pos = t & 0x7FFFFFFFu;
          break;
        }
        if (ldv(sa + offsetof(CtaSlot, walk_done))) {  // ended before this meta-block
          live = (ldv(sa + offsetof(CtaSlot, table) + 4 * mb) >> 31) != 0;
          if (live) pos = ldv(sa + offsetof(CtaSlot, table) + 4 * mb) & 0x7FFFFFFFu;
          break;
        }
        if (++spin > kCtaSpin) {
          stalled = true;
          live = false;
          break;
        }
        __nanosleep(IZG_CTA_SLEEP);  // leave the issue slots to the producer's walk
      }
    }
    CTA_T(1);  // waiting for the walk to reach the unit's meta-block
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
      const MetaWalk m = phase == 0 ? walk_meta<true>(vw, pos, groups, nw, lane)
                                    : walk_meta<false>(vw, pos, groups, nw, lane);
      const uint32_t pay = pos + 4;
      const uint32_t lastg = min(g_lo + 7, groups - 1);
      endw = pay + __shfl_sync(0xFFFFFFFFu, m.excl + 4 * m.width, lastg);
      cta_wait_issued(ctl, bars, waited, first_piece,
                      piece0 + (phase + 4u * endw + kCtaPiece - 1) / kCtaPiece, &stalled);
      CTA_T(2);  // waiting for the unit's ring pieces
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
    CTA_T(3);  // unpack + local scan
    // ---- the carry chain (one hop per unit, across chunks too, so the
    // ring's release point only ever moves forward)
    const uint32_t my_mbx = mbx_base + 32 * (U % kCtaConsumers);
    uint4 cin = make_uint4(0, 0, 0, 0);
#ifdef IZG_ABL_CTA_NOCHAIN  // developer ablation (wrong output): no carry wait
    if (false) {
#else
    if (U > 0) {
#endif
      const uint4 prev = cta_mbx_wait(mbx_base + 32 * ((U - 1) % kCtaConsumers), U - 1, &stalled);
      if (u > 0) cin = prev;  // a chunk's first unit starts from zero
    }
    CTA_T(4);  // carry wait
    // post first: the hop to the next unit's warp is the chain's critical path
    const uint4 cout = u4add(cin, local);
    cta_mbx_post(my_mbx, cout, lane);
    if (kArray && live) {
      add_carry<DELTA>(v[0], cin);
      add_carry<DELTA>(v[1], cin);
    }
    // every read of this unit's ring bytes has returned (its values are in
    // registers): free them (a release may land after a later unit's; the
    // producer only reads a lower bound and fences before refilling)
    if (lane == 0) {
      // a meta-block's first half keeps its descriptor (the second half
      // re-reads it); its second half, or the chunk's last unit, frees all
      const uint32_t rel = u + 1 == nunits ? piece0 + npieces
                           : !live         ? 0u
                           : half == 0     ? piece0 + (phase + 4u * pos) / kCtaPiece
                                           : piece0 + (phase + 4u * endw) / kCtaPiece;
      if (rel > ldv(ctl + 4 * kCtlRelease)) stv(ctl + 4 * kCtlRelease, rel);
    }
    // ---- stores
    if (live) {
      if (orow >= 0 && g_lo + 8 <= groups) {
        // both iterations through the warp's two tiles: one wait for their
        // previous stores, one proxy fence, two TMA tensor stores
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        OutStage::write(os.base, v[0], lane);
        OutStage::write(os.base + kStageOut, v[1], lane);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const uint32_t row = (uint32_t)(orow + 4 * (16 * mb + g_lo));
          tma_store_2d(&omap, os.base, 0, (int)row);
          tma_store_2d(&omap, os.base + kStageOut, 0, (int)(row + 16));
          bulk_commit();
        }
      } else {
#pragma unroll
        for (uint32_t it = 0; it < 2; ++it) {
          const uint32_t g0 = g_lo + 4 * it;
          if (g0 >= groups) break;
          const uint32_t gi = g0 + q;
          if (orow >= 0 && g0 + 4 <= groups) {
            os.put(v[it], lane, (uint32_t)(orow + 4 * (16 * mb + g0)));
          } else {
            os.direct(v[it], o + (size_t)(16 * mb + gi) * 128 + 16 * s8, oal, gi < groups,
                      128u * min(4u, groups - g0), lane);
          }
        }
      }
    }
    CTA_T(5);  // post, release, stores
    // ---- the chunk's last unit: remainder, consumption, status
    if (u + 1 == nunits) {
      // the walk is final once it published its end (all units are past it)
      for (uint32_t spin = 0; !ldv(sa + offsetof(CtaSlot, walk_done)) && ++spin < kCtaSpin;) {
      }
      __threadfence_block();
      int32_t st = (int32_t)ldv(sa + offsetof(CtaSlot, walk_err));
      uint32_t end = ldv(sa + offsetof(CtaSlot, end_pos));
      if (stalled) st = IZG_E_SPLIT_STALL;
      const uint32_t core = kArray ? n / 128 * 128 : n;
      if (kArray && st == IZG_OK) {
        if (core < n) {  // Variable Byte remainder (codec.cpp:56-62)
          uint32_t rb = 0;
          const uint32_t* p = words + word_off;
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
#ifdef IZG_CTA_PROF
        if (blockIdx.x == 0 && si < 64) g_cta_trace[si][4] = clock64();
#endif
      }
    }
  }
  os.drain();
}

}  // namespace izg
