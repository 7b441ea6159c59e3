// group.cuh — SIMD-BP128 decode with KW warps per chunk (mid-size batches).
//
// One warp per chunk runs a chunk in ~0.114 ms whatever the batch: its 128
// iterations form one dependent chain (~1,750 cycles each), so
// a batch with fewer chunks than resident warps (C1: 1,024 chunks against
// 3,552 warp slots) leaves the GPU latency-bound.  Here KW warps of one CTA
// share a chunk and take its warp iterations (512 integers) round robin:
// iteration i belongs to warp i % KW.  Every warp streams the chunk through
// its own TMA ring and walks every meta-block descriptor (so every warp
// makes the reference's checks in the same order and stops at the same
// error), but unpacks, scans and stores only its own iterations.  The
// prefix-sum carry is the only thing the warps exchange: each iteration is
// scanned with a zero carry, then waits for the carry out of iteration i-1
// in a shared-memory mailbox, adds it (per residue class), publishes its own
// carry out and stores.  The wait sits after the unpack and the local scan,
// so the chain between warps is one mailbox hop per iteration instead of a
// whole iteration.  No workspace, no second pass, every integer written
// once (TMA tensor stores, as the one-warp kernel).
#pragma once
#include "decode_kernel.cuh"

namespace izg {

// Per group of KW warps (64 bytes): carry (uint4) at +0, tag at +16, the
// claimed chunk at +24 / +28 (alternating rounds).
struct GroupLayout {
  static constexpr size_t kMbxOff = (Layout<IZG_SIMDBP128>::kSmem + 63) & ~size_t(63);
  static constexpr size_t kSmem = kMbxOff + 8 * 64;
};
constexpr uint32_t kGroupSpin = 1u << 26;  // a stuck mailbox is a bug: report, do not hang

__device__ __forceinline__ uint32_t lds32_volatile(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds128_volatile(uint32_t addr) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void sts32_volatile(uint32_t addr, uint32_t v) {
  asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Carry into the iteration tagged `want` (tag = round << 16 | iteration):
// lane 0 polls the mailbox; uniform result.  *stalled on a broken chain.
__device__ __forceinline__ uint4 mbx_wait(uint32_t mbx, uint32_t want, int lane, bool* stalled) {
  uint32_t ok = 1;
  if (lane == 0) {
    uint32_t n = 0;
    while (lds32_volatile(mbx + 16) != want) {
      if (++n >= kGroupSpin) {
        ok = 0;
        break;
      }
    }
  }
  ok = __shfl_sync(0xFFFFFFFFu, ok, 0);
  if (!ok) *stalled = true;
  __threadfence_block();
  return lds128_volatile(mbx);
}

// Lane 0: carry out of the iteration, then its tag.
__device__ __forceinline__ void mbx_post(uint32_t mbx, uint4 c, uint32_t tag, int lane) {
  if (lane == 0) {
    asm volatile("st.volatile.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(mbx), "r"(c.x), "r"(c.y),
                 "r"(c.z), "r"(c.w)
                 : "memory");
    __threadfence_block();
    sts32_volatile(mbx + 16, tag);
  }
}

// Add the carry entering an iteration that was scanned from zero (scan()'s
// carry layout: D4 per residue class, D2 per parity, D1/DM one value).
template <int DELTA>
__device__ __forceinline__ void add_carry(uint32_t (&v)[4][4], uint4 c) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (DELTA == IZG_DELTA_D4) {
      v[k][0] += c.x; v[k][1] += c.y; v[k][2] += c.z; v[k][3] += c.w;
    } else if (DELTA == IZG_DELTA_D2) {
      v[k][0] += c.x; v[k][1] += c.y; v[k][2] += c.x; v[k][3] += c.y;
    } else if (DELTA != IZG_DELTA_NONE) {
      v[k][0] += c.x; v[k][1] += c.x; v[k][2] += c.x; v[k][3] += c.x;
    }
  }
}

// bp128_core for warp `wi` of a group of `kw`: same walk, same checks, same
// status; only iterations i with i % kw == wi are unpacked, scanned and
// stored.  `tag0` = round << 16.  *stalled when a mailbox wait gave up.
template <int DELTA, bool ALIGNED, typename OS>
__device__ int32_t bp128_core_grp(WarpRing& r, OS& os, uint32_t nw, uint32_t nblocks,
                                  uint32_t* out, bool out_aligned, int64_t orow,
                                  uint32_t* pos_out, uint32_t wi, uint32_t kw, uint32_t mbx,
                                  uint32_t tag0, bool* stalled) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  uint32_t pos = 0, it = 0;
  for (uint32_t mb0 = 0; mb0 < nblocks; mb0 += 16) {
    const uint32_t groups = min(16u, nblocks - mb0);
    if (pos + 4 > nw) return IZG_E_BP_TRUNC_DESC;
    r.release_below(4u * pos);
    r.ensure(4u * (pos + 4));
    const MetaWalk m = walk_meta<ALIGNED>(r, pos, groups, nw, lane);
    if (m.err) return m.err;
    const uint32_t pay = pos + 4;
#pragma unroll 1
    for (uint32_t g0 = 0; g0 < groups; g0 += 4, ++it) {
      // every warp moves its ring over every iteration (stages are only
      // recycled once waited for), but only its own are decoded
      const uint32_t first = __shfl_sync(0xFFFFFFFFu, m.excl, g0);
      const uint32_t lastg = min(g0 + 3, groups - 1);
      const uint32_t endw = __shfl_sync(0xFFFFFFFFu, m.excl + 4 * m.width, lastg);
      r.release_below(4u * (pay + first));
      r.ensure(4u * (pay + endw));
      if (it % kw != wi) continue;
      const uint32_t gi = g0 + q;
      const bool active = gi < groups;
      uint32_t width = __shfl_sync(0xFFFFFFFFu, m.width, gi & 15);
      const uint32_t excl = __shfl_sync(0xFFFFFFFFu, m.excl, gi & 15);
      if (!active) width = 0;
      uint32_t v[4][4];
      if (ALIGNED)
        unpack_slots_aligned(r, r.ring_off() + 4u * (pay + excl), width, s8, v);
      else
        unpack_slots_unaligned(r, pay + excl, width, s8, v);
      if (DELTA != IZG_DELTA_NONE) {
        uint4 local = make_uint4(0, 0, 0, 0);
        scan<DELTA>(v, local, lane);
        const uint4 cin = it ? mbx_wait(mbx, tag0 | it, lane, stalled) : make_uint4(0, 0, 0, 0);
        add_carry<DELTA>(v, cin);
        mbx_post(mbx, u4add(cin, local), tag0 | (it + 1), lane);
      }
      if (orow >= 0 && g0 + 4 <= groups) {
        os.put(v, lane, (uint32_t)(orow + 4 * (mb0 + g0)));
      } else {
        os.direct(v, out + (size_t)(mb0 + gi) * 128 + 16 * s8, out_aligned, active,
                  128u * min(4u, groups - g0), lane);
      }
    }
    pos = pay + m.size;
  }
  *pos_out = pos;
  return IZG_OK;
}

// Persistent kernel: groups of KW warps claim whole chunks (the group's
// warp 0 takes the atomic, a named barrier shares it); warp 0 also decodes
// the VByte remainder from the final carry and writes status / consumed.
template <int DELTA, int KW>
__global__ void __maxnreg__((Layout<IZG_SIMDBP128>::kMaxRegs))
    group_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                 uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                 uint32_t* __restrict__ consumed, uint32_t* __restrict__ next_chunk,
                 const __grid_constant__ CUtensorMap omap, int tma_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using LY = Layout<IZG_SIMDBP128>;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t grp = (uint32_t)warp / KW, wi = (uint32_t)warp % KW;
  const uint32_t mbx = smem_u32(smem + GroupLayout::kMbxOff + 64 * grp);
  WarpRing r;
  r.base = smem_u32(smem + warp * kRingBytes);
  r.bar = smem_u32(smem + LY::kBarOff) + warp * kNS * 8u;
  OutStage os;
  os.base = smem_u32(smem + LY::kOutOff + warp * 2 * kStageOut);
  os.leader = lane == 0;
  os.buf = 0;
  os.tmap = &omap;
  r.g = 0;
  r.leader = lane == 0;
  r.policy = policy_evict_first();
  if (lane == 0) {
    for (uint32_t i = 0; i < kNS; ++i) mbar_init_s(r.bar + 8u * i, 1);
    fence_barrier_init();
    if (wi == 0) sts32_volatile(mbx + 16, 0xFFFFFFFFu);
  }
  __syncwarp();

  for (uint32_t round = 0;; ++round) {
    const uint32_t slot = mbx + 24 + 4 * (round & 1);
    if (wi == 0 && lane == 0) sts32_volatile(slot, atomicAdd(next_chunk, 1u));
    named_bar_sync(1 + grp, KW * 32);
    const uint32_t c = lds32_volatile(slot);
    if (c >= n_chunks) break;
    // every warp is past the previous chunk: clear its last tag, so no stale
    // tag can ever match this round's (the first post of the round is warp
    // 0's own, after this store)
    if (wi == 0 && lane == 0) sts32_volatile(mbx + 16, 0xFFFFFFFFu);
    const izg_chunk ch = chunks[c];
    int32_t st = precheck(IZG_SIMDBP128, kArray, ch.n);
    uint32_t pos = 0;
    bool stalled = false;
    const uint32_t tag0 = (round & 0xFFFFu) << 16;
    uint32_t n_it = 0;
    uint32_t* o = out + ch.out_off;
    const uint32_t core = kArray ? ch.n / 128 * 128 : ch.n;
    if (st == IZG_OK) {
      const uint32_t* p = words + ch.word_off;
      const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
      const int64_t orow = tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5) : -1;
      r.begin(p, ch.n_words);
      if (r.phase == 0)
        st = bp128_core_grp<DELTA, true>(r, os, ch.n_words, core / 128, o, oal, orow, &pos, wi,
                                         KW, mbx, tag0, &stalled);
      else
        st = bp128_core_grp<DELTA, false>(r, os, ch.n_words, core / 128, o, oal, orow, &pos,
                                          wi, KW, mbx, tag0, &stalled);
      r.end();
      const uint32_t nb = core / 128;
      for (uint32_t mb0 = 0; mb0 < nb; mb0 += 16) n_it += (min(16u, nb - mb0) + 3) / 4;
    }
    if (wi == 0) {
      if (kArray && st == IZG_OK) {
        const uint4 carry =
            n_it ? mbx_wait(mbx, tag0 | n_it, lane, &stalled) : make_uint4(0, 0, 0, 0);
        if (stalled) {
          st = IZG_E_SPLIT_STALL;
        } else if (core < ch.n) {  // Variable Byte remainder (codec.cpp:56-62)
          uint32_t rb = 0;
          const uint32_t* p = words + ch.word_off;
          if (lane == 0)
            st = vbyte_tail<DELTA>(reinterpret_cast<const uint8_t*>(p + pos),
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
  os.drain();
}

}  // namespace izg
