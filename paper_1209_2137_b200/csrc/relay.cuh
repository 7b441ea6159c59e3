// relay.cuh — SIMD-BP128 batches of a few waves: chunks cut into segments
// that are claimed level by level and hand their state on in order.
//
// One warp per chunk (decode_kernel.cuh) quantises a batch into waves of the
// resident warp slots (3,552 on a B200): BASELINE's C2 / C3 batches of 4,096
// chunks run one full wave and then a second one of 544 chunks on a mostly
// idle GPU, and lose 15-25 % to it.  Here every
// chunk is cut into S segments of whole meta-blocks and the warps claim
// (segment, chunk) tasks in segment-major order — segment k of every chunk
// before segment k+1 of any.  With at least as many chunks as warp slots,
// task (k, c) is claimed a whole level after (k-1, c), which has then
// finished, so the task reads its predecessor's published state — payload
// word of its first meta-block (the descriptor chain of
// codec_binpack.cpp:96-117 is serial), the prefix-sum carry (delta.cpp:25-89)
// and the chunk's first error — without waiting, decodes its blocks ONCE with
// the true carry through the one-warp kernel's own core (ring, unpack, scan,
// TMA stores) and publishes the state for (k+1, c).  No reduce pass, no
// fix-up, every integer written once; the tail of the batch is quantised in
// segments instead of chunks.  The last segment decodes the VByte remainder
// (codec.cpp:56-62), checks exact consumption (codec.cpp:63-64) and writes
// the status; a failing segment writes it and its successors pass the error
// on.  The published state is six single-copy-atomic 64-bit words (value <<
// 32 | tag, tag = level | error << 8) in a workspace zeroed before the
// launch: no fences (the state does not depend on the task's output stores).
// A task whose predecessor is still running (fewer chunks than slots, or a
// straggler) polls, bounded like the split kernel's look-back.
#pragma once
#include "split.cuh"  // relaxed 64-bit accesses, kSpinLimit; decode_kernel.cuh

namespace izg {

struct RelayState {
  unsigned long long w[8];  // 0..3 carry, 4 payload word, 5..7 unused (64-byte stride)
};

struct RelayArgs {
  RelayState* st;       // one per chunk, zeroed
  uint32_t* next_task;  // zeroed
  unsigned long long* summary;  // zeroed; see the kernel
  uint32_t seg_blocks;  // blocks per segment, a multiple of 16 (whole meta-blocks)
  uint32_t levels;      // segments of a full chunk
};

__host__ __device__ inline uint64_t relay_state_bytes(uint32_t n_chunks) {
  return (uint64_t)n_chunks * sizeof(RelayState);
}

template <int DELTA>
__global__ void __launch_bounds__((Layout<(DELTA >= 0 ? IZG_SIMDBP128 : 0)>::kWarps * 32))
    __maxnreg__((Layout<(DELTA >= 0 ? IZG_SIMDBP128 : 0)>::kMaxRegs))
    relay_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                 uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                 uint32_t* __restrict__ consumed, RelayArgs ra,
                 const __grid_constant__ CUtensorMap omap, int tma_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using LY = Layout<IZG_SIMDBP128>;
  using OS = OutStageT<LY::kTiles>;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpRing r;
  r.base = smem_u32(smem + warp * kRingBytes);
  r.bar = smem_u32(smem + LY::kBarOff) + warp * kNS * 8u;
  OS os;
  os.base = smem_u32(smem + LY::kOutOff + warp * LY::kTiles * kStageOut);
  os.leader = lane == 0;
  os.buf = 0;
  os.tmap = &omap;
  r.g = 0;
  r.leader = lane == 0;
  r.policy = policy_evict_first();
  if (lane == 0) {
    for (uint32_t i = 0; i < kNS; ++i) mbar_init_s(r.bar + 8u * i, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const uint32_t SB = ra.seg_blocks;

  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(ra.next_task, 1u);
    t = __shfl_sync(0xFFFFFFFFu, t, 0);
    const uint32_t k = t / n_chunks, c = t - k * n_chunks;
    if (k >= ra.levels) break;
    const izg_chunk ch = chunks[c];
    const uint32_t core = kArray ? ch.n / 128 * 128 : ch.n;
    const uint32_t nblocks = core / 128;
    // segments of this chunk: SB blocks each, the last one takes what is left (raw-mode
    // chunks may hold more than 65,536 integers: more blocks than levels * SB)
    const uint32_t nseg = nblocks ? min(ra.levels, (nblocks + SB - 1) / SB) : 1u;
    if (k == 0 && lane == 0) {
      // batch summary, one 64-bit word: low half = level-0 tasks seen, high half bit j =
      // some chunk has a segment j.  Both updates hit one address from one thread, so the
      // count never runs ahead of the bits it vouches for (no fence needed).
      const uint32_t sbits = (nseg >= 32 ? 0xFFFFFFFFu : (1u << nseg) - 1u) & ~1u;
      if (sbits) atomicOr(ra.summary, (unsigned long long)sbits << 32);
      atomicAdd(ra.summary, 1ull);
    }
    if (k >= nseg) {
      // every chunk's first task has been seen and none has a segment k: nor has any
      // later task (levels only grow), so this warp is done — batches of short chunks
      // do not pay for claiming and skipping the upper levels
      // (level-0 tasks post the summary first thing, so the wait below is a microsecond
      // at the start of the launch and nothing afterwards; bounded like every spin here)
      unsigned long long sm = ld_relaxed64(ra.summary);
      for (uint32_t spins = 0; (uint32_t)sm != n_chunks && spins < 4096; ++spins) {
        __nanosleep(128);
        sm = ld_relaxed64(ra.summary);
      }
      if ((uint32_t)sm == n_chunks && !((sm >> (32 + k)) & 1ull)) break;
      continue;
    }
    int32_t st = precheck(IZG_SIMDBP128, kArray, ch.n);
    if (st != IZG_OK) {  // every task of the chunk sees it; task 0 reports
      if (k == 0 && lane == 0) {
        status[c] = st;
        if (consumed) consumed[c] = 0;
      }
      continue;
    }
    const bool last = k == nseg - 1;
    const uint32_t b0 = k * SB, b1 = last ? nblocks : b0 + SB;
    unsigned long long* const sw = ra.st[c].w;
    uint4 carry = make_uint4(0, 0, 0, 0);
    uint32_t pos0 = 0;
    if (k) {
      // state out of (k-1, c): lanes 0..4 each poll one word for tag k
      unsigned long long x = 0;
      uint32_t spins = 0;
      for (;;) {
        if (lane < 5) x = ld_relaxed64(sw + lane);
        const bool ready = lane >= 5 || (uint32_t)(x & 0xFFu) == k;
        if (__all_sync(0xFFFFFFFFu, ready)) break;
        if (++spins > kSpinLimit) break;
        __nanosleep(64);
      }
      const uint32_t val = (uint32_t)(x >> 32);
      carry.x = __shfl_sync(0xFFFFFFFFu, val, 0);
      carry.y = __shfl_sync(0xFFFFFFFFu, val, 1);
      carry.z = __shfl_sync(0xFFFFFFFFu, val, 2);
      carry.w = __shfl_sync(0xFFFFFFFFu, val, 3);
      pos0 = __shfl_sync(0xFFFFFFFFu, val, 4);
      uint32_t perr = __shfl_sync(0xFFFFFFFFu, (uint32_t)(x >> 8) & 0xFFFFFFu, 4);
      if (spins > kSpinLimit) {  // a broken chain: report instead of hanging
        perr = IZG_E_SPLIT_STALL;
        if (lane == 0) {
          status[c] = (int32_t)perr;
          if (consumed) consumed[c] = 0;
        }
      }
      if (perr) {  // the failing task wrote the status; pass the error on
        if (!last && lane < 5)
          st_relaxed64(sw + lane, (unsigned long long)(k + 1) | (unsigned long long)perr << 8);
        continue;
      }
    }
    const uint32_t* p = words + ch.word_off;
    uint32_t* o = out + ch.out_off;
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    const int64_t orow = tma_out && (ch.out_off & 31) == 0 ? (int64_t)(ch.out_off >> 5) : -1;
    const uint32_t nw = ch.n_words - pos0;
    uint32_t used = 0;
    os.begin_chunk();
    r.begin(p + pos0, nw);
    if (r.phase == 0)
      st = bp128_core<DELTA, true>(r, os, nw, b1, o, oal, orow, carry, &used, b0);
    else
      st = bp128_core<DELTA, false>(r, os, nw, b1, o, oal, orow, carry, &used, b0);
    r.end();
    uint32_t pos = pos0 + used;
    if (!last) {
      if (st != IZG_OK && lane == 0) {
        status[c] = st;
        if (consumed) consumed[c] = 0;
      }
      if (lane < 5) {
        const uint32_t val = lane == 0   ? carry.x
                             : lane == 1 ? carry.y
                             : lane == 2 ? carry.z
                             : lane == 3 ? carry.w
                                         : pos;
        st_relaxed64(sw + lane, (unsigned long long)val << 32 | (unsigned long long)(k + 1) |
                                    (unsigned long long)(uint32_t)st << 8);
      }
      continue;
    }
    if (kArray && st == IZG_OK) {
      if (core < ch.n) {  // Variable Byte remainder (codec.cpp:56-62)
        uint32_t rb = 0;
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
  os.drain();
}

using RelayFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                         uint32_t*, RelayArgs, const CUtensorMap, int);

}  // namespace izg
