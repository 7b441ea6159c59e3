// split.cuh — small batches: several warps per chunk, with a decoupled
// look-back carry across the segments of one array (north_star item 2).
//
// One warp per chunk (decode_kernel.cuh) leaves most of the GPU idle when a
// batch has few chunks: C1's 1,024 chunks give 7 warps per SM, and a 64-chunk
// posting list less than one.  The split kernel cuts every chunk into
// segments of kSegBlocks 128-integer blocks (4,096 integers) and lets warps
// claim (segment, chunk) units level by level — segment k of every chunk
// before segment k+1 of any — so a unit's predecessor (k-1, c) is always
// already claimed by a running warp.
//
// Per unit:
//  1. Start offset.  SIMD-FastPFOR (indexed): the page records of
//     fp_index_kernel give every block's packed word, position byte and
//     exception cursors directly.  SIMD-BP128: the meta-block descriptor
//     chain (codec_binpack.cpp:96-117) is serial; every unit walks it from
//     the chunk start itself (unit 0 first pulls the chunk into L2 with one
//     bulk prefetch, so the hops are L2 hits), making every reference check
//     in order on its own two descriptors.
//  2. SIMD-BP128 array modes, reduce-then-scan: unless the predecessor's
//     inclusive prefix is already out, one unpack pass sums the segment's
//     deltas (no stores), the unit looks back (3.) and publishes its
//     inclusive prefix, then decodes once with the true carry.  Otherwise
//     (and for SIMD-FastPFOR): decode with a zero carry (the same cores as
//     the one-warp kernel), storing to HBM with plain stores so the lines
//     stay in L2.
//  3. Decoupled look-back (Merrill & Garland's single-pass scan): publish the
//     segment's aggregate (the local carry: last value per D4 lane class,
//     etc.), then walk back over predecessors, adding aggregates until one
//     publishes an inclusive prefix; publish this unit's inclusive prefix.
//     The first error of the chunk in stream order travels with the
//     prefixes.
//  4. Fix-up (decode-first units only): every lane re-reads exactly the
//     integers it stored (L2 hits) and adds the exclusive prefix per residue
//     class.  Skipped when the predecessor's inclusive prefix was already
//     published at step 2.
// The last segment decodes the VByte remainder and writes the chunk's
// status; an error on the BP128 offset chain stops the chunk's later units.
// Spins are bounded (a broken chain reports IZG_E_SPLIT_STALL instead of
// hanging the GPU).
#pragma once
#include <cstdint>

#include "decode_kernel.cuh"  // precheck, the decode cores

namespace izg {

#ifndef IZG_SPLIT_MIN_SEG
#define IZG_SPLIT_MIN_SEG 32  // blocks: 4,096 integers (16: 7% faster at 64 chunks, 15% slower at 128)
#endif
constexpr uint32_t kSegBlocks = IZG_SPLIT_MIN_SEG;  // smallest segment (BP128 meta-blocks)
constexpr uint32_t kFpSegBlocks = 32;  // SIMD-FastPFOR segments: 4,096 integers
#ifndef IZG_SPLIT_RTS
#define IZG_SPLIT_RTS 1  // SIMD-BP128: reduce-then-scan instead of decode + fix-up
#endif
constexpr uint32_t kMaxSegs = IZG_CHUNK_SIZE / 128 / kSegBlocks;

// Look-back state of one unit (80 bytes, zeroed before the launch).  Every
// published value is a 64-bit word (value << 32 | tag), tag = kind | err << 8
// (kind 1: aggregate, 2: inclusive prefix; err: first error so far), written
// and read with single-copy-atomic relaxed 64-bit accesses — no fences, so
// publishing never waits for the unit's own output stores to drain.
struct SegState {
  uint32_t pad[4];
  unsigned long long agg[4];  // per residue class (scan()'s carry layout)
  unsigned long long pre[4];
};
constexpr uint32_t kSpinLimit = 1u << 22;  // ~seconds of polling: a stall is a bug

__host__ __device__ inline uint64_t split_state_bytes(uint32_t n_chunks) {
  return (uint64_t)n_chunks * kMaxSegs * sizeof(SegState);
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Number of carry components a delta mode uses.
template <int DELTA>
__host__ __device__ constexpr int carry_words() {
  return DELTA == IZG_DELTA_D4 ? 4 : DELTA == IZG_DELTA_D2 ? 2 : 1;
}

template <int DELTA>
__device__ __forceinline__ void publish(unsigned long long* w, uint4 v, uint32_t kind,
                                        uint32_t err) {
  const uint32_t vals[4] = {v.x, v.y, v.z, v.w};
  const unsigned long long tag = kind | (unsigned long long)err << 8;
#pragma unroll
  for (int i = 0; i < carry_words<DELTA>(); ++i)
    st_relaxed64(w + i, (unsigned long long)vals[i] << 32 | tag);
}

// Read a published value: true when all its words carry `kind`.
template <int DELTA>
__device__ __forceinline__ bool try_read(const unsigned long long* w, uint32_t kind, uint4* v,
                                         uint32_t* err) {
  uint32_t vals[4] = {0, 0, 0, 0};
  bool ok = true;
#pragma unroll
  for (int i = 0; i < carry_words<DELTA>(); ++i) {
    const unsigned long long x = ld_relaxed64(w + i);
    ok &= (x & 0xFFu) == kind;
    vals[i] = (uint32_t)(x >> 32);
    if (i == 0) *err = (uint32_t)(x >> 8) & 0xFFFFFFu;
  }
  *v = make_uint4(vals[0], vals[1], vals[2], vals[3]);
  return ok;
}

// Output sink of the split kernel: like OutStage but plain 16-byte stores
// (no TMA: the fix-up re-reads each lane's own stores, which needs them in
// the generic proxy and in L2).
struct SegStage {
  static constexpr bool kProbe = false;
  static constexpr bool kAgg = false;
  uint32_t base;  // the warp's shared tile (SIMD-FastPFOR patches there)
  uint32_t* out;  // chunk output (rows are chunk-relative)
  __device__ __forceinline__ void begin_chunk() {}
  __device__ __forceinline__ void store(const uint32_t (&v)[4][4], int lane, uint32_t row) const {
    uint32_t* o = out + (size_t)row * 32 + 16 * lane;
#pragma unroll
    for (int c = 0; c < 4; ++c) stg128_cg(o + 4 * c, make_uint4(v[c][0], v[c][1], v[c][2], v[c][3]));
  }
  __device__ __forceinline__ void put(const uint32_t (&v)[4][4], int lane, uint32_t row) {
    store(v, lane, row);
  }
  __device__ __forceinline__ uint32_t acquire() {
    __syncwarp();
    return base;
  }
  __device__ __forceinline__ void commit(const uint32_t (&v)[4][4], int lane, uint32_t row) {
    __syncwarp();  // every lane's read of the patched tile is done
    store(v, lane, row);
  }
  __device__ __forceinline__ void abandon() { __syncwarp(); }
  __device__ __forceinline__ void direct(const uint32_t (&v)[4][4], uint32_t* o, bool oal,
                                         bool live, uint32_t, int) {
    if (!live) return;
    if (oal) {
#pragma unroll
      for (int c = 0; c < 4; ++c) stg128_cg(o + 4 * c, make_uint4(v[c][0], v[c][1], v[c][2], v[c][3]));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) o[4 * c + j] = v[c][j];
    }
  }
  __device__ __forceinline__ void drain() {}
};

// Sink of the aggregate pass (reduce-then-scan, SIMD-BP128): bp128_core
// only sums the deltas; nothing reaches memory.
struct AggStage {
  static constexpr bool kProbe = false;
  static constexpr bool kAgg = true;
  __device__ __forceinline__ void put(const uint32_t (&)[4][4], int, uint32_t) {}
  __device__ __forceinline__ void direct(const uint32_t (&)[4][4], uint32_t*, bool, bool,
                                         uint32_t, int) {}
};

// Add the exclusive prefix P to the integers of blocks [b0, b1) (b0 a
// multiple of 4) that this lane stored, per residue class (scan()'s carry
// layout), and to the VByte remainder [core, n) that lane 0 stored.
template <int DELTA>
__device__ __forceinline__ void seg_fixup(uint32_t* out, bool oal, uint32_t b0, uint32_t b1,
                                          uint32_t core, uint32_t n, uint4 P, int lane) {
  const uint32_t q = lane >> 3, s8 = lane & 7;
  auto add = [&](uint4 x) {
    if (DELTA == IZG_DELTA_D4) {
      x.x += P.x; x.y += P.y; x.z += P.z; x.w += P.w;
    } else if (DELTA == IZG_DELTA_D2) {
      x.x += P.x; x.y += P.y; x.z += P.x; x.w += P.y;
    } else {
      x.x += P.x; x.y += P.x; x.z += P.x; x.w += P.x;
    }
    return x;
  };
  if (oal) {  // two blocks' loads in flight before any store
    for (uint32_t g = b0 + q; g < b1; g += 8) {
      uint4* o0 = reinterpret_cast<uint4*>(out + (size_t)g * 128 + 16 * s8);
      uint4* o1 = o0 + 128;  // block g + 4
      const bool two = g + 4 < b1;
      uint4 x[4], y[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) x[c] = o0[c];
      if (two) {
#pragma unroll
        for (int c = 0; c < 4; ++c) y[c] = o1[c];
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) o0[c] = add(x[c]);
      if (two) {
#pragma unroll
        for (int c = 0; c < 4; ++c) o1[c] = add(y[c]);
      }
    }
  } else {
    for (uint32_t g = b0 + q; g < b1; g += 4) {
      uint32_t* o = out + (size_t)g * 128 + 16 * s8;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 x = add(make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]));
        o[4 * c] = x.x; o[4 * c + 1] = x.y; o[4 * c + 2] = x.z; o[4 * c + 3] = x.w;
      }
    }
  }
  if (lane == 0) {
    for (uint32_t i = core; i < n; ++i) {
      const uint32_t add = DELTA == IZG_DELTA_D4   ? ((i & 3) == 0 ? P.x : (i & 3) == 1 ? P.y
                                                      : (i & 3) == 2 ? P.z : P.w)
                           : DELTA == IZG_DELTA_D2 ? ((i & 1) ? P.y : P.x)
                                                   : P.x;
      out[i] += add;
    }
  }
}

// One SIMD-BP128 meta-block descriptor at chunk word `pos`, straight from
// global memory, warp-collective like walk_meta (lane g < 16 owns group g's
// width; a 16-lane scan gives the sizes): the reference's checks in order
// (codec_binpack.cpp:96-117).  Returns the meta-block's words including the
// descriptor, or 0 with *err (uniform).
__device__ __forceinline__ uint32_t bp_meta_words(const uint32_t* p, uint32_t pos,
                                                  uint32_t groups, uint32_t nw, int lane,
                                                  int32_t* err) {
  if (pos + 4 > nw) {
    *err = IZG_E_BP_TRUNC_DESC;
    return 0;
  }
  const uint32_t g = lane & 15;
  const uint32_t word = __ldg(p + pos + (g >> 2));  // 4-byte loads: containers
  const uint32_t w = (word >> (8 * (g & 3))) & 0xFFu;
  const bool valid = g < groups;
  const uint32_t sz = valid ? 4u * min(w, 33u) : 0u;
  uint32_t incl = sz;
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d, 16);
    if (g >= (uint32_t)d) incl += y;
  }
  const uint32_t mw = __ballot_sync(0xFFFFFFFFu, valid && w > 32) & 0xFFFFu;
  const uint32_t mt = __ballot_sync(0xFFFFFFFFu, valid && pos + 4 + incl > nw) & 0xFFFFu;
  if (mw | mt) {
    const int first = __ffs(mw | mt) - 1;
    *err = ((mw >> first) & 1u) ? IZG_E_BP_WIDTH : IZG_E_BP_TRUNC_PAYLOAD;
    return 0;
  }
  return 4u + __shfl_sync(0xFFFFFFFFu, incl, groups - 1);
}

struct SplitArgs {
  SegState* seg;       // n_chunks * kMaxSegs states, zeroed
  uint32_t* next_unit;
  uint32_t seg_blocks;  // blocks per segment: kSegBlocks << s (split_seg_blocks)
};

// Segment size for a batch: about four units per resident warp, so that
// larger batches pay for fewer descriptor walks, look-backs and unit
// start-ups (powers of two from 4,096 to 65,536 integers).
__host__ __device__ inline uint32_t split_seg_blocks(uint32_t n_chunks, uint32_t warp_slots) {
  uint32_t segs = kMaxSegs;
  while (segs > 1 && (uint64_t)n_chunks * segs > 4ull * warp_slots) segs >>= 1;
  return (IZG_CHUNK_SIZE / 128) / segs;
}

// Persistent split kernel: CODEC = IZG_SIMDBP128 or IZG_SIMDFASTPFOR
// (indexed pages; fp_index_kernel ran first).  Array modes (DELTA != NONE)
// and codec-level decode (NONE, no carry) alike.
template <int CODEC, int DELTA>
__global__ void __launch_bounds__((Layout<CODEC, CODEC == IZG_SIMDFASTPFOR>::kWarps * 32))
    __maxnreg__((Layout<CODEC, CODEC == IZG_SIMDFASTPFOR>::kMaxRegs))
    split_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                 uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                 uint32_t* __restrict__ consumed, SplitArgs sa, IdxView ix) {
  constexpr bool IDX = CODEC == IZG_SIMDFASTPFOR;
  using LY = Layout<CODEC, IDX>;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpRing r;
  r.base = smem_u32(smem + warp * kRingBytes);
  r.bar = smem_u32(smem + LY::kBarOff) + warp * kNS * 8u;
  r.g = 0;
  r.leader = lane == 0;
  r.policy = policy_evict_first();
  uint32_t* dir_base = reinterpret_cast<uint32_t*>(smem + LY::kTabOff + warp * LY::kTabBytes);
  SegStage os;
  os.base = smem_u32(smem + LY::kOutOff + warp * LY::kTiles * kStageOut);
  if (lane == 0) {
    for (uint32_t i = 0; i < kNS; ++i) mbar_init_s(r.bar + 8u * i, 1);
    fence_barrier_init();
  }
  __syncwarp();

  for (;;) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(sa.next_unit, 1u);
    u = __shfl_sync(0xFFFFFFFFu, u, 0);
    const uint32_t k = u / n_chunks, c = u - k * n_chunks;
    if (k >= (IZG_CHUNK_SIZE / 128) / sa.seg_blocks) break;
    const izg_chunk ch = chunks[c];
    const uint32_t core = kArray ? ch.n / 128 * 128 : ch.n;
    const uint32_t nblocks = core / 128;
    const uint32_t SB = sa.seg_blocks;
    const uint32_t nseg = nblocks ? (nblocks + SB - 1) / SB : 1u;
    if (k >= nseg) continue;
    const bool last = k == nseg - 1;
    const uint32_t b0 = k * SB;
    const uint32_t b1 = last ? nblocks : b0 + SB;
    SegState* const st = sa.seg + (size_t)c * kMaxSegs;
    int32_t err = precheck(CODEC, kArray, ch.n);
    if (err != IZG_OK) {  // every unit sees it; unit 0 reports
      if (k == 0 && lane == 0) {
        status[c] = err;
        if (consumed) consumed[c] = 0;
      }
      continue;
    }
    const uint32_t* p = words + ch.word_off;
    uint32_t* o = out + ch.out_off;
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    os.out = o;
    const int64_t orow = oal ? 0 : -1;  // SegStage rows are relative to o
    bool stalled = false;

    // ---- 1. start offset (BP128: the descriptor chain) -------------------
    uint32_t pos0 = 0, pos_end = 0;
    uint4 hdr = make_uint4(0, 0, 0, 0);
    if (CODEC == IZG_SIMDBP128) {
      // Every unit walks the descriptor chain from the chunk start itself
      // (no waiting on its predecessor): unit 0 pulls the chunk into L2 and
      // the other units' hops over earlier segments are L2 hits with a
      // 4-lane size check; an error there belongs to an earlier unit, which
      // reports it, so this unit just stops.
      int32_t werr = IZG_OK;
      if (k == 0 && lane == 0) prefetch_l2(p, 4u * ch.n_words);
      uint32_t pos = 0;
      for (uint32_t mb = 0; mb < b0; mb += 16) {
        const bool fits = pos + 4 <= ch.n_words;
        const uint32_t word = fits && lane < 4 ? __ldg(p + pos + lane) : 0u;
        uint32_t sz = __dp4a(word, 0x01010101u, 0u);
        sz += __shfl_xor_sync(0xFFFFFFFFu, sz, 1);
        sz += __shfl_xor_sync(0xFFFFFFFFu, sz, 2);
        sz = __shfl_sync(0xFFFFFFFFu, sz, 0);
        const bool bad = !fits || __any_sync(0xFFFFFFFFu, __vcmpgtu4(word, 0x20202020u) != 0) ||
                         pos + 4 + 4 * sz > ch.n_words;
        if (bad) {
          werr = -1;  // an earlier unit reports it
          break;
        }
        pos += 4 + 4 * sz;
      }
      pos0 = pos;
      for (uint32_t mb = b0; werr == IZG_OK && mb < b1; mb += 16)
        pos += bp_meta_words(p, pos, min(16u, nblocks - mb), ch.n_words, lane, &werr);
      pos_end = pos;
      if (lane == 0 && werr > 0) {  // first error of the chunk in stream order
        status[c] = werr;
        if (consumed) consumed[c] = 0;
      }
      if (werr != IZG_OK) continue;
    } else if (nblocks) {
      hdr = ix.hdr[c];
      const int32_t hs = (int32_t)(hdr.x & 0xFFu);
      if (hs != IZG_OK) {  // page-level error: unit 0 resolves it as the fused path does
        if (k == 0) {
          int32_t e = hs;
          if (hs != IZG_E_FP_TRUNC_PAGE && hs != IZG_E_FP_BA_OFFSET && hs != IZG_E_FP_TRUNC_BA &&
              fp_positions_bad_idx(ix.page_rec(c), reinterpret_cast<const uint8_t*>(p + hdr.w + 1),
                                   (hdr.x >> 8) & 0xFFFFu, lane))
            e = IZG_E_FP_POS_RANGE;
          if (lane == 0) {
            status[c] = e;
            if (consumed) consumed[c] = 0;
          }
        }
        continue;
      }
    }

    // ---- 2. decode with a zero carry (or the predecessor's prefix) --------
    uint4 carry = make_uint4(0, 0, 0, 0);
    bool have_prefix = k == 0;
    uint32_t pre_err = 0;
    if (k > 0) {
      uint32_t f = 0;
      if (lane == 0) {  // a partly published prefix must not leak into the carry
        uint4 v;
        uint32_t e = 0;
        if (try_read<DELTA>(st[k - 1].pre, 2u, &v, &e)) {
          f = 1u;
          carry = v;
          pre_err = e;
        }
      }
      f = __shfl_sync(0xFFFFFFFFu, f, 0);
      if (f) {
        have_prefix = true;
        carry.x = __shfl_sync(0xFFFFFFFFu, carry.x, 0);
        carry.y = __shfl_sync(0xFFFFFFFFu, carry.y, 0);
        carry.z = __shfl_sync(0xFFFFFFFFu, carry.z, 0);
        carry.w = __shfl_sync(0xFFFFFFFFu, carry.w, 0);
      }
    }
    // ---- 2'. reduce-then-scan (SIMD-BP128 array modes): when the
    // predecessor's prefix is not out yet, sum this segment's deltas (one
    // unpack pass, no stores), look back, publish the inclusive prefix
    // before decoding, and decode once with the true carry — no fix-up
    // traffic.  Step 1 already made every check this segment's payload
    // needs, so the aggregate is error-free.
    bool looked_back = false;
    uint32_t first_err = 0;
    if (CODEC == IZG_SIMDBP128 && kArray && !have_prefix && nblocks && IZG_SPLIT_RTS) {
      uint4 agg = make_uint4(0, 0, 0, 0);
      AggStage as;
      uint32_t used = 0;
      r.begin(p + pos0, ch.n_words - pos0);
      if (r.phase == 0)
        bp128_core<DELTA, true>(r, as, ch.n_words - pos0, b1, o, oal, orow, agg, &used, b0);
      else
        bp128_core<DELTA, false>(r, as, ch.n_words - pos0, b1, o, oal, orow, agg, &used, b0);
      r.end();
      uint4 excl = make_uint4(0, 0, 0, 0);
      if (lane == 0) {
        publish<DELTA>(st[k].agg, agg, 1u, 0u);
        for (int32_t j = (int32_t)k - 1; j >= 0; --j) {
          uint4 v;
          uint32_t e = 0;
          for (uint32_t it = 0;; ++it) {
            if (try_read<DELTA>(st[j].pre, 2u, &v, &e)) {
              j = -1;
              break;
            }
            if (try_read<DELTA>(st[j].agg, 1u, &v, &e)) break;
            if (it >= kSpinLimit) {
              stalled = true;
              break;
            }
            if (it > 32) __nanosleep(64);
          }
          if (stalled) break;
          excl = u4add(excl, v);
          if (e) first_err = e;
        }
        if (stalled) first_err = IZG_E_SPLIT_STALL;
        publish<DELTA>(st[k].pre, u4add(excl, agg), 2u, first_err);
      }
      carry.x = __shfl_sync(0xFFFFFFFFu, excl.x, 0);
      carry.y = __shfl_sync(0xFFFFFFFFu, excl.y, 0);
      carry.z = __shfl_sync(0xFFFFFFFFu, excl.z, 0);
      carry.w = __shfl_sync(0xFFFFFFFFu, excl.w, 0);
      first_err = __shfl_sync(0xFFFFFFFFu, first_err, 0);
      have_prefix = looked_back = true;
    }
    int32_t derr = IZG_OK;
    uint32_t pos = 0;
    if (nblocks) {
      if (CODEC == IZG_SIMDBP128) {
        r.begin(p + pos0, ch.n_words - pos0);
        uint32_t used = 0;
        if (r.phase == 0)
          derr = bp128_core<DELTA, true>(r, os, ch.n_words - pos0, b1, o, oal, orow, carry, &used,
                                         b0);
        else  // payload not 16-byte aligned (containers decoded in place)
          derr = bp128_core<DELTA, false>(r, os, ch.n_words - pos0, b1, o, oal, orow, carry,
                                          &used, b0);
        r.end();
        pos = pos0 + used;
      } else {
        const uint4* rec = ix.page_rec(c);
        dir_base[lane + 1] = ix.dir[(size_t)c * 32 + lane];
        if (lane == 0) dir_base[0] = 0;  // width 0 (no exceptions): the page start
        __syncwarp();
        const uint32_t A = hdr.w;
        const uint32_t wfirst = rec[b0].y;  // first packed word of the segment
        if (lane == 0 && k == 0) prefetch_l2(p + hdr.y, 4u * (hdr.z - hdr.y));
        r.begin(p + wfirst, A - wfirst);
        const bool bad = fp_blocks_idx<DELTA, kVertical>(r, os, dir_base, rec + b0, p, A, b1 - b0,
                                                         o + (size_t)b0 * 128, oal,
                                                         orow < 0 ? -1 : orow + 4 * b0, carry,
                                                         wfirst);
        r.end();
        if (bad) derr = IZG_E_FP_POS_RANGE;
        pos = hdr.z;
      }
    } else if (CODEC == IZG_SIMDFASTPFOR) {
      pos = 0;  // decode_deltas(count == 0) reads nothing
    }
    // VByte remainder (last unit, codec.cpp:56-62), decoded from the local carry
    int32_t terr = IZG_OK;
    if (kArray && last && core < ch.n && derr == IZG_OK) {
      uint32_t rb = 0;
      if (lane == 0)
        terr = vbyte_tail<DELTA>(reinterpret_cast<const uint8_t*>(p + pos),
                                 4u * (ch.n_words - pos), core, ch.n - core, carry, o, &rb);
      terr = __shfl_sync(0xFFFFFFFFu, terr, 0);
      rb = __shfl_sync(0xFFFFFFFFu, rb, 0);
      if (terr == IZG_OK) pos += (rb + 3) / 4;
    }
    if (kArray && last && terr == IZG_OK && derr == IZG_OK && pos != ch.n_words)
      terr = IZG_E_PAYLOAD_SIZE;  // codec.cpp:63-64
    if (!kArray && last && derr == IZG_OK && CODEC == IZG_SIMDBP128) pos = pos_end;

    // ---- 3. look-back (every mode: the chunk's first error travels with
    // the prefixes; the carry is zero without delta coding) ----------------
    uint4 excl = make_uint4(0, 0, 0, 0);
    if (looked_back) {
      if (first_err == 0 && derr != IZG_OK) first_err = (uint32_t)derr;  // (not expected)
    } else if (lane == 0) {
      if (have_prefix) {
        first_err = pre_err;  // the predecessor's prefix is inside `carry`
      } else {
        publish<DELTA>(st[k].agg, carry, 1u, (uint32_t)derr);
        for (int32_t j = (int32_t)k - 1; j >= 0; --j) {
          uint4 v;
          uint32_t e = 0;
          for (uint32_t it = 0;; ++it) {
            if (try_read<DELTA>(st[j].pre, 2u, &v, &e)) {
              j = -1;  // inclusive prefix found: last step
              break;
            }
            if (try_read<DELTA>(st[j].agg, 1u, &v, &e)) break;
            if (it >= kSpinLimit) {
              stalled = true;
              break;
            }
            if (it > 32) __nanosleep(64);
          }
          if (stalled) break;
          excl = u4add(excl, v);
          if (e) first_err = e;
        }
      }
      const uint32_t own = stalled ? (uint32_t)IZG_E_SPLIT_STALL
                                   : first_err ? first_err : (uint32_t)derr;
      publish<DELTA>(st[k].pre, u4add(excl, carry), 2u, own);
      first_err = own;
    }
    if (!looked_back) {
      excl.x = __shfl_sync(0xFFFFFFFFu, excl.x, 0);
      excl.y = __shfl_sync(0xFFFFFFFFu, excl.y, 0);
      excl.z = __shfl_sync(0xFFFFFFFFu, excl.z, 0);
      excl.w = __shfl_sync(0xFFFFFFFFu, excl.w, 0);
      first_err = __shfl_sync(0xFFFFFFFFu, first_err, 0);
    }
    // ---- 4. fix-up ---------------------------------------------------------
    if (kArray && !have_prefix && first_err == 0)
      seg_fixup<DELTA>(o, oal, b0, b1, core, last ? ch.n : core, excl, lane);
    if (lane == 0 && last) {
      int32_t s2 = (int32_t)first_err;
      if (s2 == IZG_OK) s2 = terr;
      status[c] = s2;
      if (consumed) consumed[c] = s2 == IZG_OK ? pos : 0;
    }
  }
}

}  // namespace izg
