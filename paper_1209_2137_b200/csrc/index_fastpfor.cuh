// index_fastpfor.cuh — page index pass of the two-kernel SIMD-FastPFOR path.
//
// The fused decoder (decode_fastpfor.cuh) spends about a quarter of its
// instructions on the page's metadata: walking the byte array and turning
// each block's entry into packed offsets, position offsets and per-width
// exception cursors four blocks at a time.  With a workspace, izg_decode_ws
// moves all of that into this kernel (one warp per page, 32 blocks per step,
// at high occupancy), and the decode kernel reads one 16-byte record per
// block instead.
//
// Per page one warp restates every check the reference makes before it
// touches a packed word (codec_patched.cpp:292-416), in the reference's
// order: page header (:296-305), the byte-array walk (:309-336, the fused
// decoder's windowed fp_parse), the exception directory (:339-379) and the
// block loop's overrun / exhaustion / packed-size checks (:381-415) over 32
// blocks per step.  Exception positions are
// NOT checked here — the decode kernel sees every position while patching,
// and on error paths resolves POS_RANGE precedence from the records
// (fp_positions_bad_idx), exactly as the fused path does.
//
// Workspace layout (izg_decode_workspace_size): for n chunks,
//   hdr[n]        uint4 {status | parsed entries << 8, first word after the
//                 byte array, end word (words consumed), A}
//   dir[n][32]    uint32 base word of exception array w (index w-1)
//   rec[n][512]   uint4 per block {b | w<<6 | c<<12, packed word, first
//                 position byte (byte-array offset), cursor in array w}
//   snap[n][16][32] uint16 cursor of every width (index w-1) after each 32
//                 blocks (row j: after block 32 (j + 1), or the page's last),
//                 for the team decode's exception windows (team.cuh); bit 31
//                 of hdr.x is set when a cursor passed 65,535 (rows invalid)
#pragma once
#include <cstdio>

#include "decode_fastpfor.cuh"
#include "izg_common.cuh"

namespace izg {

constexpr uint32_t kMaxBlocks = IZG_CHUNK_SIZE / 128;  // 512 records per page

struct IdxView {
  uint4* hdr;
  uint32_t* dir;
  uint4* rec;
  uint16_t* snap;
  __device__ __forceinline__ uint4* page_rec(uint32_t c) const {
    return rec + (size_t)c * kMaxBlocks;
  }
};

__host__ __device__ inline uint64_t idx_workspace_bytes(uint32_t n_chunks) {
  return (uint64_t)n_chunks * (16u + 32u * 4u + kMaxBlocks * 16u + 16u * 32u * 2u);
}

__host__ __device__ inline IdxView idx_view(void* ws, uint32_t n_chunks) {
  IdxView v;
  uint8_t* p = static_cast<uint8_t*>(ws);
  v.hdr = reinterpret_cast<uint4*>(p);
  v.dir = reinterpret_cast<uint32_t*>(p + (size_t)n_chunks * 16u);
  v.rec = reinterpret_cast<uint4*>(p + (size_t)n_chunks * (16u + 128u));
  v.snap = reinterpret_cast<uint16_t*>(p + (size_t)n_chunks * (16u + 128u + kMaxBlocks * 16u));
  return v;
}

// Metadata pass over the parsed table, 32 blocks per step (lane = block):
// packed word and first position byte (warp scans of 4b and entry lengths),
// cursor in the block's width array (earlier same-width blocks of the step
// plus the warp's running per-width count `cnt`), and — when `checks` — the
// block loop's overrun / exhaustion checks in block order
// (codec_patched.cpp:387-388, 406-407).  Records go out coalesced.
static __device__ int32_t fp_meta(const FpScratch& sc, uint32_t* cnt, uint4* rec, uint16_t* snap,
                           uint32_t nb, uint32_t A, bool checks, int lane, uint32_t* packed_end,
                           bool* cursor_ovf) {
  cnt[lane + 1] = 0;
  __syncwarp();
  uint32_t packed = 1, bpos = 0;
  int32_t err = IZG_OK;
  bool ovf = false;
#pragma unroll 1
  for (uint32_t j0 = 0; j0 < nb; j0 += 32) {
    const uint32_t k = j0 + lane;
    const bool live = k < nb;
    const uint32_t e = live ? sc.tab[k] : 0u;
    const uint32_t b = e & 63u, w = (e >> 6) & 63u, c = e >> 12;
    const uint32_t len = live ? (c ? 3 + c : 2u) : 0u;
    const uint4 inc = warp_incl_scan<2>(make_uint4(4u * b, len, 0, 0), lane);
    // exceptions of earlier same-width blocks of this step, by bit planes
    const uint32_t grp = __match_any_sync(0xFFFFFFFFu, c ? w : 64u + lane);
    const uint32_t below = grp & ((1u << lane) - 1u);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      acc += (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, (c >> j) & 1u) & below) << j;
    const uint32_t cur = c ? cnt[w] + acc : 0u;
    __syncwarp();
    if (c && lane == 31 - __clz(grp)) cnt[w] = cur + c;  // last block of its width
    __syncwarp();
    {  // every width's cursor after this step (team.cuh's exception windows)
      const uint32_t cv = cnt[lane + 1];
      ovf |= cv > 65535u;
      snap[(j0 >> 5) * 32 + lane] = (uint16_t)min(cv, 65535u);
    }
    if (checks && err == IZG_OK) {
      const bool ov = live && packed + inc.x > A;
      const bool ex = c && (uint64_t)cur + c > sc.dir_n[w];
      const uint32_t bm = __ballot_sync(0xFFFFFFFFu, ov || ex);
      if (bm) {
        const int f = __ffs(bm) - 1;
        err = (__ballot_sync(0xFFFFFFFFu, ov) >> f) & 1u ? IZG_E_FP_OVERRUN : IZG_E_FP_EXHAUSTED;
      }
    }
    if (live) stg128_cg(rec + k, make_uint4(e, packed + inc.x - 4u * b, bpos + inc.y - len + 3u, cur));
    packed += __shfl_sync(0xFFFFFFFFu, inc.x, 31);
    bpos += __shfl_sync(0xFFFFFFFFu, inc.y, 31);
  }
  *packed_end = packed;
  *cursor_ovf = __any_sync(0xFFFFFFFFu, ovf);
  return err;
}

// Shared memory of the index kernel: per warp a TMA ring, an FpScratch, the
// running per-width counts and the ring barriers.
constexpr int kIdxWarps = 8;
struct IdxLayout {
  static constexpr uint32_t kScOff = kIdxWarps * kRingBytes;
  static constexpr uint32_t kScBytes = (sizeof(FpScratch) + 15) & ~15u;
  static constexpr uint32_t kCntOff = kScOff + kIdxWarps * kScBytes;
  static constexpr uint32_t kBarOff = kCntOff + kIdxWarps * 36 * 4;
  static constexpr size_t kSmem = kBarOff + kIdxWarps * kNS * 8;
};

// One warp indexes one page: header checks (codec_patched.cpp:296-305), the
// windowed byte-array walk (fp_parse), the exception directory
// (fp_directory), then fp_meta.  Statuses follow the reference's order;
// positions are left to the decode kernel (see the file comment).
template <bool ARRAY, int ST>
__global__ void __launch_bounds__(kIdxWarps * 32)
    fp_index_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                    uint32_t n_chunks, IdxView ix) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kIdxWarps + warp;
  if (c >= n_chunks) return;  // warp-uniform
  const izg_chunk ch = chunks[c];
  // decode_array's length check or decode_deltas' count checks: the decode
  // kernel repeats them and never reads this page's record when they fail
  if (ARRAY ? (ch.n == 0 || ch.n > IZG_CHUNK_SIZE) : (ch.n % 128 || ch.n > IZG_CHUNK_SIZE)) {
    if (lane == 0) ix.hdr[c] = make_uint4(IZG_OK, 0, 0, 0);
    return;
  }
  const uint32_t nblocks = (ARRAY ? ch.n / 128 * 128 : ch.n) / 128;
  const uint32_t* page = words + ch.word_off;
  const uint32_t nw = ch.n_words;
  uint4 h = make_uint4(IZG_OK, 0, 0, 0);
  if (nblocks == 0) {  // decode_deltas(count == 0) reads nothing (codec_patched.cpp:295)
    if (lane == 0) ix.hdr[c] = h;
    return;
  }
  const uint32_t A = nw ? __ldg(page) : 0u;
  const uint32_t L = (nw && A >= 1 && A < nw) ? __ldg(page + A) : 0u;
  const uint64_t ba_words = ((uint64_t)L + 3) / 4;
  if (nw == 0) h.x = IZG_E_FP_TRUNC_PAGE;
  else if (A < 1 || A >= nw) h.x = IZG_E_FP_BA_OFFSET;
  else if (A + 1 + ba_words > nw) h.x = IZG_E_FP_TRUNC_BA;
  if (h.x) {
    if (lane == 0) ix.hdr[c] = h;
    return;
  }
  WarpRing r;
  r.base = smem_u32(smem + warp * kRingBytes);
  r.bar = smem_u32(smem + IdxLayout::kBarOff) + warp * kNS * 8u;
  r.g = 0;
  r.leader = lane == 0;
  r.policy = policy_evict_last();  // the decode kernel re-reads the position bytes
  FpScratch& sc = *reinterpret_cast<FpScratch*>(smem + IdxLayout::kScOff + warp * IdxLayout::kScBytes);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + IdxLayout::kCntOff) + warp * 36;
  if (lane == 0) {
    for (uint32_t i = 0; i < kNS; ++i) mbar_init_s(r.bar + 8u * i, 1);
    fence_barrier_init();
  }
  __syncwarp();
  r.begin(page + A + 1, (uint32_t)ba_words);
  uint32_t parsed = 0;
  int32_t st = fp_parse(r, sc, L, nblocks, lane, &parsed);
  r.end();
  __syncwarp();
  uint32_t end = 0;
  if (st == IZG_OK) {
    st = fp_directory<ST>(sc, page, nw, A + 1 + ba_words, lane, &end);
    if (st == IZG_OK) ix.dir[(size_t)c * 32 + lane] = sc.dir_base[lane + 1];
  }
  uint32_t packed = 0;
  bool ovf = false;
  const int32_t bst = fp_meta(sc, cnt, ix.page_rec(c), ix.snap + (size_t)c * 512, parsed, A,
                              st == IZG_OK, lane, &packed, &ovf);
  if (st == IZG_OK) st = bst ? bst : (packed != A ? IZG_E_FP_PACKED_SIZE : IZG_OK);
  if (lane == 0)
    ix.hdr[c] = make_uint4((uint32_t)st | parsed << 8 | (ovf ? 0x80000000u : 0u),
                           A + 1 + (uint32_t)ba_words, end, A);
}

// ---- lane-per-page index pass (round 2) -------------------------------------
//
// The warp-per-page pass above spends ~132 warp-instructions per 512
// integers, mostly on the windowed walk: per 128-byte window every lane
// decodes speculative entry lengths at four byte offsets, and the chain of
// entry starts is serial anyway.  Here each LANE indexes its own page: the
// byte-array walk is a serial loop of a handful of instructions per entry
// (codec_patched.cpp:309-336, every check in the reference's order), so a
// warp walks 32 pages at once and the pass costs a few instructions per 512
// integers; its time is the latency of the walks (every page's walk runs at
// once), which is why the byte array is read from per-lane rings in shared
// memory filled by cp.async copies ahead of the walk (below).  The exception directory (:338-379) is read
// first (its errors still rank after the walk's, as in the reference); each
// block's cursor in its width array is a running count per width, kept per
// lane in shared memory ([width][lane]: conflict-free); the block loop's
// overrun / exhaustion checks (:387-388, 406-407) and the packed-size check
// are made during the walk.  Output: the same header, directory and block
// records as fp_index_kernel, so the decode kernel is unchanged.
__device__ __forceinline__ uint32_t ld_ca_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
constexpr int kIdxLaneWarps = 4;
#ifndef IZG_IDXL_AHEAD
#define IZG_IDXL_AHEAD 256  // 65,536 C5 pages: 128 / 256 / 512 / 1024 B ahead -> 0.93 / 0.90 / 1.00 / 1.10 ms
#endif
constexpr uint32_t kIdxLaneAhead = IZG_IDXL_AHEAD;  // bytes the L1 prefetches run ahead of the walk
// The walk reads the byte array from a per-lane ring in shared memory that
// the lane fills with 16-byte cp.async copies running ahead of it, in rounds:
// wait for the copies of the round before, top the ring up, walk up to
// IZG_IDXL_ROUND entries of what has landed.  All lanes of a warp wait at the
// same instruction once per round, and every entry is read at shared-memory
// latency.  (The first version loaded each entry from global memory with L1
// prefetches ahead: 0.93 ms on 65,536 C5 pages, one exposed L2 / HBM latency
// per entry since ~450 independent streams per SM thrash L1.)
#ifndef IZG_IDXL_RING
#define IZG_IDXL_RING 8  // 16-byte chunks per lane (0: the global-load walk)
#endif
#ifndef IZG_IDXL_ROUND
#define IZG_IDXL_ROUND 2  // entries per round (65,536 C5 pages: 2 / 3 / 4 / 6 -> 0.49 / 0.54 / 0.52 / 0.60 ms)
#endif
#ifndef IZG_IDXL_DEPTH
#define IZG_IDXL_DEPTH 2  // rounds of copies in flight
#endif
#ifndef IZG_IDXL_PAIR
#define IZG_IDXL_PAIR 1  // store records in pairs (whole sectors)
#endif
constexpr uint32_t kIdxRingChunks = IZG_IDXL_RING;
struct IdxLaneLayout {
  // per warp: running counts cnt[33][32], array sizes nn[33][32] (u32), then the lanes' rings
  static constexpr uint32_t kWarpBytes = 2 * 33 * 32 * 4;
  static constexpr uint32_t kRingOff = kIdxLaneWarps * kWarpBytes;
  static constexpr size_t kSmem = kRingOff + kIdxLaneWarps * 32 * 16 * kIdxRingChunks;
};
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <bool ARRAY, int ST>
__global__ void __launch_bounds__(kIdxLaneWarps * 32)
    fp_index_lanes_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                          uint32_t n_chunks, IdxView ix) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + warp * IdxLaneLayout::kWarpBytes);
  uint32_t* nn = cnt + 33 * 32;
  const uint32_t c = (blockIdx.x * kIdxLaneWarps + warp) * 32u + lane;
  if (c >= n_chunks) return;  // the lanes work independently from here on
  const izg_chunk ch = chunks[c];
  // decode_array's length check or decode_deltas' count checks: the decode
  // kernel repeats them and never reads this page's record when they fail
  if (ARRAY ? (ch.n == 0 || ch.n > IZG_CHUNK_SIZE) : (ch.n % 128 || ch.n > IZG_CHUNK_SIZE)) {
    ix.hdr[c] = make_uint4(IZG_OK, 0, 0, 0);
    return;
  }
  const uint32_t nblocks = (ARRAY ? ch.n / 128 * 128 : ch.n) / 128;
  const uint32_t* page = words + ch.word_off;
  const uint32_t nw = ch.n_words;
  if (nblocks == 0) {  // decode_deltas(count == 0) reads nothing (codec_patched.cpp:295)
    ix.hdr[c] = make_uint4(IZG_OK, 0, 0, 0);
    return;
  }
  const uint32_t A = nw ? __ldg(page) : 0u;
  const uint32_t L = (nw && A >= 1 && A < nw) ? __ldg(page + A) : 0u;
  const uint64_t ba_words = ((uint64_t)L + 3) / 4;
  int32_t hst = IZG_OK;
  if (nw == 0) hst = IZG_E_FP_TRUNC_PAGE;
  else if (A < 1 || A >= nw) hst = IZG_E_FP_BA_OFFSET;
  else if (A + 1 + ba_words > nw) hst = IZG_E_FP_TRUNC_BA;
  if (hst) {
    ix.hdr[c] = make_uint4((uint32_t)hst, 0, 0, 0);
    return;
  }
  // the whole byte array to L2 now (one bulk prefetch per page), so the
  // serial walk below meets L2 hits, and L1 prefetches run ahead of it
#ifndef IZG_IDXL_NOL2
  prefetch_l2(page + A + 1, 4u * (uint32_t)ba_words);
#endif
  // exception directory (codec_patched.cpp:339-379); its error, if any, is
  // reported only after the byte-array walk has passed
  int32_t dst = IZG_OK;
  uint64_t pos = A + 1 + ba_words;
  uint32_t* dir = ix.dir + (size_t)c * 32;
  for (uint32_t w = 0; w <= 32; ++w) nn[w * 32 + lane] = 0;
  uint32_t bits = 0;
  if (pos >= nw) {
    dst = IZG_E_FP_NO_BITSET;
  } else {
    bits = __ldg(page + pos);
    ++pos;
  }
  for (uint32_t w = 1; w <= 32; ++w) {
    uint32_t base = 0;
    if (dst == IZG_OK && ((bits >> (w - 1)) & 1u)) {
      if (pos >= nw) {
        dst = IZG_E_FP_TRUNC_EXC;
      } else {
        const uint32_t n = __ldg(page + pos);
        uint64_t nwords;
        if (ST == kVertical) {
          pos = (pos + 1 + 3) & ~uint64_t{3};  // 16-byte alignment in the page
          nwords = ((uint64_t)n + 127) / 128 * 4 * w;
        } else {
          pos = pos + 1;
          nwords = ((uint64_t)n + 31) / 32 * w;
        }
        if (pos + nwords > nw) {
          dst = IZG_E_FP_TRUNC_EXC;
        } else {
          base = (uint32_t)pos;
          nn[w * 32 + lane] = n;
          pos += nwords;
        }
      }
    }
    dir[w - 1] = dst == IZG_OK ? base : 0u;
  }
  const uint32_t end = (uint32_t)pos;
  // the byte-array walk (codec_patched.cpp:309-336) with every block's record
  for (uint32_t w = 0; w <= 32; ++w) cnt[w * 32 + lane] = 0;
  const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);
  const uint32_t Lc = L > 0x7FFFFFF0u ? 0x7FFFFFF0u : L;
  uint4* rec = ix.page_rec(c);
  int32_t wst = IZG_OK, lst = IZG_OK;  // walk error; first block-loop error
  uint32_t s = 0, packed = 1, k = 0;
  bool ovf = false;  // a cursor passed 65,535 (snapshot rows are 16-bit)
  uint4* snap = reinterpret_cast<uint4*>(ix.snap + (size_t)c * 512);
#if IZG_IDXL_RING
  {
    constexpr uint32_t kRingBytes16 = 16u * kIdxRingChunks;
    const uint32_t ring = smem_u32(smem) + IdxLaneLayout::kRingOff +
                          (uint32_t)(warp * 32 + lane) * kRingBytes16;
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(ba) & ~uintptr_t(15);
    const uint32_t phase = (uint32_t)(reinterpret_cast<uintptr_t>(ba) - g0);
    const uint32_t nchunks = (phase + 4u * (uint32_t)ba_words + 15u) >> 4;  // covering the byte array
    uint32_t pf = 0;  // next chunk to copy; chunks below it were issued
    uint32_t pfh[IZG_IDXL_DEPTH];  // `pf` after the issue of each of the last rounds, newest first
#pragma unroll
    for (int i = 0; i < IZG_IDXL_DEPTH; ++i) pfh[i] = 0;
    bool walking = true;
    uint4 held = make_uint4(0, 0, 0, 0);  // an even block's record, stored with the next one
    while (walking && k < nblocks) {
      const uint32_t curc = (s + phase) >> 4;
      // Up to IZG_IDXL_DEPTH rounds of copies are in flight.  Chunks below pfh[DEPTH-1]
      // were issued DEPTH or more rounds ago: complete after wait_group DEPTH-1.  When the
      // walk has reached younger chunks (or a long entry skipped over them) wait for
      // everything — always BEFORE issuing new copies: a late copy must not land on a newer
      // chunk's slot, and the slots refilled below hold chunks under `curc`.
      uint32_t landed = pfh[IZG_IDXL_DEPTH - 1];
      if (curc + 1 >= landed) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        if (pf < curc) pf = curc;  // a long entry jumped past the ring
        landed = pf;
#pragma unroll
        for (int i = 0; i < IZG_IDXL_DEPTH; ++i) pfh[i] = pf;
      } else {
        asm volatile("cp.async.wait_group %0;" ::"n"(IZG_IDXL_DEPTH - 1) : "memory");
      }
      while (pf < curc + kIdxRingChunks && pf < nchunks) {
        IZG_CHECK(izg_in_span(g0 + 16u * pf, 16, page, nw), 8, c, pf);
        cp_async16(ring + 16u * (pf % kIdxRingChunks), reinterpret_cast<const void*>(g0 + 16u * pf));
        ++pf;
      }
#pragma unroll
      for (int i = IZG_IDXL_DEPTH - 1; i > 0; --i) pfh[i] = pfh[i - 1];
      pfh[0] = pf;
      asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll 1
      for (uint32_t step = 0; step < IZG_IDXL_ROUND && k < nblocks; ++step, ++k) {
        if (s + 2 > Lc) {
          wst = IZG_E_FP_TRUNC_META;
          walking = false;
          break;
        }
        const bool have3 = s + 2 < Lc;
        if (((s + (have3 ? 2u : 1u) + phase) >> 4) >= landed) break;  // next round
        const uint32_t o = s + phase;
        const uint32_t b = lds8(ring + (o % kRingBytes16));
        const uint32_t mb = lds8(ring + ((o + 1) % kRingBytes16));
        const uint32_t c3 = have3 ? lds8(ring + ((o + 2) % kRingBytes16)) : 0u;
#ifdef IZG_IDXL_DEBUG
        if (b != ba[s] || mb != ba[s + 1])
          printf("ring mismatch page %u k %u s %u o %u got %u %u want %u %u pf %u landed %u curc %u nch %u\n",
                 c, k, s, o, b, mb, (uint32_t)ba[s], (uint32_t)ba[s + 1], pf, landed, curc, nchunks);
#endif
        walking = false;  // left false by every error exit of the step
        do {
      if (b > 32 || mb > 32 || b > mb) {
        wst = IZG_E_FP_WIDTHS;
        break;
      }
      uint32_t e = b, cc = 0, cur = 0;
      if (mb > b) {
        if (s + 2 >= Lc) {
          wst = IZG_E_FP_TRUNC_META;
          break;
        }
        cc = c3;
        if (cc == 0) {
          wst = IZG_E_FP_EMPTY_EXC;
          break;
        }
        if (s + 3 + cc > Lc) {
          wst = IZG_E_FP_TRUNC_POS;
          break;
        }
        const uint32_t w = mb - b;
        cur = cnt[w * 32 + lane];
        cnt[w * 32 + lane] = cur + cc;
        ovf |= cur + cc > 65535u;
        e = b | w << 6 | cc << 12;
        if (lst == IZG_OK && (uint64_t)cur + cc > nn[w * 32 + lane] && packed + 4 * b <= A)
          lst = IZG_E_FP_EXHAUSTED;
      }
      if (lst == IZG_OK && packed + 4 * b > A) lst = IZG_E_FP_OVERRUN;
#ifndef IZG_ABL_IDX_NOREC  // developer ablation (decode broken): no record stores
#if IZG_IDXL_PAIR
      // records leave two at a time: a whole 32-byte sector per pair
      if (k & 1u) {
        stg128_cg(rec + k - 1, held);
        stg128_cg(rec + k, make_uint4(e, packed, s + 3, cur));
      } else if (k + 1 == nblocks) {
        stg128_cg(rec + k, make_uint4(e, packed, s + 3, cur));
      } else {
        held = make_uint4(e, packed, s + 3, cur);
      }
#else
      stg128_cg(rec + k, make_uint4(e, packed, s + 3, cur));
#endif
#endif
      packed += 4 * b;
      s += cc ? 3 + cc : 2;
      if ((k & 31u) == 31u || k + 1 == nblocks) {  // cursors after 32 (k / 32 + 1) blocks
#pragma unroll
        for (uint32_t w4 = 0; w4 < 4; ++w4) {
          uint32_t x[4];
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t w = 8 * w4 + 2 * j + 1;  // widths w, w + 1 -> one word
            x[j] = min(cnt[w * 32 + lane], 65535u) | min(cnt[(w + 1) * 32 + lane], 65535u) << 16;
          }
          stg128_cg(snap + (k >> 5) * 4 + w4, make_uint4(x[0], x[1], x[2], x[3]));
        }
      }
          walking = true;
        } while (false);
        if (!walking) break;
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#if IZG_IDXL_PAIR
    if (!walking && (k & 1u)) stg128_cg(rec + k - 1, held);  // the walk stopped on an odd block
#endif
  }
#else
#pragma unroll
  for (uint32_t a = 0; a < kIdxLaneAhead; a += 128)
    if (a < Lc) asm volatile("prefetch.global.L1 [%0];" ::"l"(ba + a));
  uint32_t line = 0;
  for (; k < nblocks; ++k) {
    if ((s >> 7) != line) {  // entered a new 128-byte line: fetch one further ahead
      line = s >> 7;
      const uint32_t a = 128 * line + kIdxLaneAhead;  // prefetch only inside the byte array
#ifndef IZG_IDXL_NOL1
      if (a < Lc) asm volatile("prefetch.global.L1 [%0];" ::"l"(ba + a));
#endif
    }
    if (s + 2 > Lc) {
      wst = IZG_E_FP_TRUNC_META;
      break;
    }
    // bytes s .. s+3 from the two words holding them (L1-cached loads;
    // the byte array is word-aligned and padded to a word, so both words
    // are inside the page whenever s + 2 <= L)
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(ba) + (s >> 2);
    uint32_t x = ld_ca_u32(bw);
    if (s & 3) x = funnel_r(x, (s >> 2) + 1 < (Lc + 3) / 4 ? ld_ca_u32(bw + 1) : 0u, 8 * (s & 3));
    const uint32_t b = x & 0xFFu, mb = (x >> 8) & 0xFFu, c3 = (x >> 16) & 0xFFu;
    if (b > 32 || mb > 32 || b > mb) {
      wst = IZG_E_FP_WIDTHS;
      break;
    }
    uint32_t e = b, cc = 0, cur = 0;
    if (mb > b) {
      if (s + 2 >= Lc) {
        wst = IZG_E_FP_TRUNC_META;
        break;
      }
      cc = c3;
      if (cc == 0) {
        wst = IZG_E_FP_EMPTY_EXC;
        break;
      }
      if (s + 3 + cc > Lc) {
        wst = IZG_E_FP_TRUNC_POS;
        break;
      }
      const uint32_t w = mb - b;
      cur = cnt[w * 32 + lane];
      cnt[w * 32 + lane] = cur + cc;
      ovf |= cur + cc > 65535u;
      e = b | w << 6 | cc << 12;
      if (lst == IZG_OK && (uint64_t)cur + cc > nn[w * 32 + lane] && packed + 4 * b <= A)
        lst = IZG_E_FP_EXHAUSTED;
    }
    if (lst == IZG_OK && packed + 4 * b > A) lst = IZG_E_FP_OVERRUN;
#ifndef IZG_ABL_IDX_NOREC  // developer ablation (decode broken): no record stores
    stg128_cg(rec + k, make_uint4(e, packed, s + 3, cur));
#endif
    packed += 4 * b;
    s += cc ? 3 + cc : 2;
    if ((k & 31u) == 31u || k + 1 == nblocks) {  // cursors after 32 (k / 32 + 1) blocks
#pragma unroll
      for (uint32_t w4 = 0; w4 < 4; ++w4) {
        uint32_t x[4];
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
          const uint32_t w = 8 * w4 + 2 * j + 1;  // widths w, w + 1 -> one word
          x[j] = min(cnt[w * 32 + lane], 65535u) | min(cnt[(w + 1) * 32 + lane], 65535u) << 16;
        }
        stg128_cg(snap + (k >> 5) * 4 + w4, make_uint4(x[0], x[1], x[2], x[3]));
      }
    }
  }
#endif
  int32_t st = wst;
  if (st == IZG_OK && s != L) st = IZG_E_FP_BA_LEN;
  const bool dir_ok = st == IZG_OK && dst == IZG_OK;  // fp_index_kernel reports `end` only then
  if (st == IZG_OK) st = dst;
  if (st == IZG_OK) st = lst;
  if (st == IZG_OK && packed != A) st = IZG_E_FP_PACKED_SIZE;
  ix.hdr[c] = make_uint4((uint32_t)st | k << 8 | (ovf ? 0x80000000u : 0u),
                         A + 1 + (uint32_t)ba_words, dir_ok ? end : 0u, A);
}

// ---- decode side -----------------------------------------------------------

// Error paths: does any exception position of records [0, nb) reach 128
// (codec_patched.cpp:328-330)?  Checked before every later error, as the
// reference validates positions during its byte-array walk.
static __device__ bool fp_positions_bad_idx(const uint4* rec, const uint8_t* ba, uint32_t nb, int lane) {
  bool bad = false;
  for (uint32_t k = lane; k < nb; k += 32) {
    const uint4 e = rec[k];
    const uint32_t c = e.x >> 12;
    for (uint32_t i = 0; i < c; ++i) bad |= ldg_u8(ba + e.z + i) >= 128u;
  }
  return __any_sync(0xFFFFFFFFu, bad);
}

// Blocks of an indexed page (codec_patched.cpp:381-415 minus the checks the
// index pass already made): as fp_blocks, but each lane reads its block's
// record (lanes 8q..8q+7 share block q's 16 bytes) one iteration ahead.
// Returns true when an exception position >= 128 was met.
template <int DELTA, int ST, typename OS>
__device__ bool fp_blocks_idx(WarpRing& r, OS& os, const uint32_t* dir_base, const uint4* rec,
                              const uint32_t* page, uint32_t A, uint32_t nblocks, uint32_t* out,
                              bool oal, int64_t orow, uint4& carry, uint32_t wbase = 1) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  const uint8_t* ba = reinterpret_cast<const uint8_t*>(page + A + 1);
  bool bad = false;
  uint4 nx = rec[min(q, nblocks - 1)];
#pragma unroll 1
  for (uint32_t g0 = 0; g0 < nblocks; g0 += 4) {
    const uint32_t ng = min(4u, nblocks - g0);
    const bool live = q < ng;
    const uint4 e = nx;
    if (g0 + 4 < nblocks) nx = rec[min(g0 + 4 + q, nblocks - 1)];
    const uint32_t myb = live ? e.x & 63u : 0u;
    const uint32_t myw = (e.x >> 6) & 63u;
    const uint32_t myc = live ? e.x >> 12 : 0u;
    const uint32_t myoff = e.y, mybp = e.z, mycur = e.w;
    const uint32_t first = __shfl_sync(0xFFFFFFFFu, myoff, 0);
    const uint32_t after = __shfl_sync(0xFFFFFFFFu, myoff + 4u * myb, 8 * (ng - 1));
#ifdef IZG_ABL_NOEXC  // developer ablation (wrong output): no patch path
    const bool tot = false;
#else
    const bool tot = __any_sync(0xFFFFFFFFu, myc != 0);
#endif

    // Stream window: packed words [first, after) (the stream starts at word 1).
    r.release_below(4u * (first - wbase));
    r.ensure(4u * (after - wbase));
    uint32_t v[4][4];
    if (ST != kVertical)
      unpack_scalar_slots(r, myoff - wbase, myb, s8, v);
    else if (r.phase == 0)
      unpack_slots_aligned(r, r.ring_off() + 4u * (myoff - wbase), myb, s8, v);
    else
      unpack_slots_unaligned(r, myoff - wbase, myb, s8, v);
    if (tot) {
      const uint32_t mybase = dir_base[myw];
      const uint32_t t = os.acquire();
      OutStage::write(t, v, lane);
      __syncwarp();
#ifndef IZG_ABL_NOPATCH  // developer ablation (wrong output): tile round trip only
      bad |= fp_patch<ST>(t, page, ba, myb, myw, myc, mybp, mycur, mybase, lane);
#endif
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
  return __any_sync(0xFFFFFFFFu, bad);
}

// Blocks of one page from its records `rec` (split.cuh passes a range:
// `wbase` = page word the ring starts at, 1 for a whole page).

// Whole indexed page `c` (record written by fp_index_kernel); same contract
// as fastpfor_core.
template <int DELTA, int ST, typename OS>
__device__ int32_t fastpfor_core_idx(WarpRing& r, OS& os, uint32_t* dir_base,
                                     const uint32_t* page, uint32_t c, uint32_t nblocks,
                                     const IdxView& ix, uint32_t* out, bool oal, int64_t orow,
                                     uint4& carry, uint32_t* pos_out) {
  const int lane = threadIdx.x & 31;
  if (nblocks == 0) {
    *pos_out = 0;
    return IZG_OK;
  }
  const uint4 h = ix.hdr[c];
  const int32_t st = (int32_t)(h.x & 0xFFu);
  const uint4* rec = ix.page_rec(c);
  if (st) {
    if (st == IZG_E_FP_TRUNC_PAGE || st == IZG_E_FP_BA_OFFSET || st == IZG_E_FP_TRUNC_BA)
      return st;
    return fp_positions_bad_idx(rec, reinterpret_cast<const uint8_t*>(page + h.w + 1),
                                (h.x >> 8) & 0xFFFFu, lane)
               ? IZG_E_FP_POS_RANGE
               : st;
  }
  const uint32_t A = h.w;
  dir_base[lane + 1] = ix.dir[(size_t)c * 32 + lane];
  if (lane == 0) dir_base[0] = 0;  // width 0 (no exceptions): the page start
  __syncwarp();
  if (lane == 0) prefetch_l2(page + h.y, 4u * (h.z - h.y));  // exception arrays
  r.begin(page + 1, A - 1);
  const bool bad =
      fp_blocks_idx<DELTA, ST>(r, os, dir_base, rec, page, A, nblocks, out, oal, orow, carry);
  r.end();
  if (bad) return IZG_E_FP_POS_RANGE;
  *pos_out = h.z;
  return IZG_OK;
}

}  // namespace izg
