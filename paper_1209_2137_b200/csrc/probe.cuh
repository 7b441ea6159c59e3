// probe.cuh — decode → intersect without materialising the decoded list
// (the paper's "process the decoded posting lists" use,
// PAPER.md:1697-1719).  The reference has no such API; semantics follow
// numpy.intersect1d and are documented with izg_decode_intersect.
//
// ProbeStage replaces OutStage as the decode kernel's output sink.  Each
// decoded 512-integer iteration stays in registers (16 consecutive integers
// per lane) instead of going to HBM; the warp merges it against the sorted
// probe list S, which it walks with a per-chunk cursor: 32 elements of S per
// round (one coalesced 128-byte load, prefetched during the previous
// iteration), each lane locates its element among the lanes' segments by
// shuffle, and hits are recorded as one bit per S element (atomicOr of the
// round's ballot).  A decoded chunk is nondecreasing (the
// sorted-list use of D1/D4), so the cursor only moves forward and each tile
// costs ceil(matching S elements / 32) rounds.  Compaction of the hit bits
// into the sorted distinct intersection is in intersect.cu.
#pragma once
#include <cstdint>

#include "izg_common.cuh"

namespace izg {

struct ProbeArgs {
  const uint32_t* s;  // probe list, nondecreasing
  uint64_t ns;
  uint32_t* hits;     // ceil(ns / 32) + 1 words, zeroed by the launcher
};

// Warp-cooperative lower_bound of x in s[a, b): 32-ary search, one round
// of 32 probes per factor 32 of the range.
__device__ __forceinline__ uint64_t warp_lower_bound(const uint32_t* __restrict__ s, uint64_t a,
                                                     uint64_t b, uint32_t x, int lane) {
  while (b - a > 32) {
    const uint64_t step = (b - a + 31) / 32;
    const uint64_t i = a + (uint64_t)lane * step;
    const bool lt = i < b && __ldg(s + i) < x;
    const uint32_t k = __popc(__ballot_sync(0xFFFFFFFFu, lt));  // lanes 0..k-1
    if (k == 0) return a;
    const uint64_t a0 = a;
    a = a0 + (uint64_t)(k - 1) * step + 1;
    if (a0 + (uint64_t)k * step < b) b = a0 + (uint64_t)k * step;
  }
  const uint64_t i = a + lane;
  const bool lt = i < b && __ldg(s + i) < x;
  return a + __popc(__ballot_sync(0xFFFFFFFFu, lt));
}

// Element k (0..15) of a lane's 16 decoded integers, k dynamic (select chain).
__device__ __forceinline__ uint32_t pick16(const uint32_t (&v)[4][4], uint32_t k) {
  uint32_t r = v[0][0];
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c)
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j)
      if (4 * c + j == k) r = v[c][j];
  return r;
}

struct ProbeStage {
  static constexpr bool kProbe = true;
  static constexpr bool kAgg = false;
  uint32_t base;  // shared address of the warp's tile (FastPFOR patches there)
  bool leader;
  ProbeArgs pa;
  uint64_t cur;   // cursor into s for the current chunk; ~0 = not placed yet
  uint32_t w0, w1;  // s[cur + lane], s[cur + 32 + lane]: prefetched windows

  __device__ __forceinline__ void begin_chunk() { cur = ~0ull; }
  __device__ __forceinline__ void put(const uint32_t (&v)[4][4], int lane, uint32_t) {
    probe(v, 512u, lane);
  }
  __device__ __forceinline__ uint32_t acquire() {
    __syncwarp();
    return base;
  }
  __device__ __forceinline__ void commit(const uint32_t (&v)[4][4], int lane, uint32_t) {
    probe(v, 512u, lane);
  }
  __device__ __forceinline__ void abandon() { __syncwarp(); }
  // Warp-collective (every lane calls it): the first `nvalid` integers of
  // the iteration (lane L holds integers 16L..16L+15) are decoded values.
  __device__ __forceinline__ void direct(const uint32_t (&v)[4][4], uint32_t*, bool, bool,
                                         uint32_t nvalid, int lane) {
    probe(v, nvalid, lane);
  }
  __device__ __forceinline__ void drain() {}

  __device__ __forceinline__ uint32_t window(uint64_t at, int lane) const {
    const uint64_t i = at + lane;
    return i < pa.ns ? __ldg(pa.s + i) : 0u;
  }

  // Merge the iteration's sorted integers (registers, mapping C) against s
  // from the cursor: per round, lane j takes s[cur + j]; the lane holding
  // its segment is found by a 5-step shuffle search over the lanes' first
  // integers, and the 16 integers of that lane are compared by shuffle.
  __device__ __forceinline__ void probe(const uint32_t (&v)[4][4], uint32_t nvalid, int lane) {
    const uint32_t first = v[0][0];
    const uint32_t lo = __shfl_sync(0xFFFFFFFFu, first, 0);
    const uint32_t nl = (nvalid + 15) >> 4;  // lanes holding valid integers
    const uint32_t hi = nvalid == 512u ? __shfl_sync(0xFFFFFFFFu, v[3][3], 31)
                                       : __shfl_sync(0xFFFFFFFFu, pick16(v, (nvalid - 1) & 15u),
                                                     (int)nl - 1);
    if (cur == ~0ull) {
      cur = warp_lower_bound(pa.s, 0, pa.ns, lo, lane);
      w0 = window(cur, lane);
      w1 = window(cur + 32, lane);
    }
#pragma unroll 1
    for (int r = 0;; ++r) {
      const uint32_t x = r == 0 ? w0 : r == 1 ? w1 : window(cur, lane);
      const bool le = cur + lane < pa.ns && x <= hi;
      const bool want = le && x >= lo;
      if (__any_sync(0xFFFFFFFFu, want)) {
        uint32_t sg = 0;  // last lane whose first integer is <= x
#pragma unroll
        for (uint32_t st = 16; st; st >>= 1) {
          const uint32_t f = __shfl_sync(0xFFFFFFFFu, first, (int)(sg + st));
          if (sg + st < nl && f <= x) sg += st;
        }
        bool found = false;
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c)
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t y = __shfl_sync(0xFFFFFFFFu, v[c][j], (int)sg);
            found |= y == x && 16u * sg + 4u * c + j < nvalid;
          }
        const uint32_t fm = __ballot_sync(0xFFFFFFFFu, want && found);
        if (fm && lane == 0) {
          const uint64_t w = cur >> 5;
          const uint32_t sh = (uint32_t)cur & 31u;
          atomicOr(pa.hits + w, fm << sh);
          if (sh && (fm >> (32 - sh))) atomicOr(pa.hits + w + 1, fm >> (32 - sh));
        }
      }
      const uint32_t adv = __popc(__ballot_sync(0xFFFFFFFFu, le));
      cur += adv;
      if (adv < 32) break;
    }
    // next iteration's windows, in flight while it decodes
    w0 = window(cur, lane);
    w1 = window(cur + 32, lane);
  }
};

}  // namespace izg
