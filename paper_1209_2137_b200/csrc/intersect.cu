// intersect.cu — consumer of the decoded arrays: sorted
// intersection of two nondecreasing uint32 arrays resident in HBM, the query
// the paper names for processing decoded posting lists.
// The reference has no intersection API; semantics follow numpy.intersect1d
// (distinct values present in both, ascending), and the tests check exactly
// that.  Decoding stays in izg_decode; only the intersection needs to leave
// the device.
//
// Algorithm: the shorter array drives.  Each thread takes kPer consecutive
// elements of it, drops repeats (a[i] == a[i-1]) and looks each one up in
// the longer array by binary search (neighbouring elements walk the same
// L2-resident path).  Two passes keep the output sorted without atomics:
// per-tile match counts, an exclusive scan of the counts, then each tile
// writes its matches at its offset in element order.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/intzip_b200.h"

namespace izg {
namespace {

constexpr int kThreads = 256, kPer = 4, kTile = kThreads * kPer;

__device__ __forceinline__ bool contains(const uint32_t* __restrict__ b, uint64_t nb, uint32_t x) {
  uint64_t lo = 0, hi = nb;  // lower_bound
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(b + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < nb && __ldg(b + lo) == x;
}

// Match mask (bit k = element base+k matches) of this thread's elements.
__device__ __forceinline__ uint32_t matches(const uint32_t* __restrict__ a, uint64_t na,
                                            const uint32_t* __restrict__ b, uint64_t nb,
                                            uint64_t base) {
  uint32_t m = 0;
  uint32_t prev = base ? __ldg(a + base - 1) : 0u;
  bool have_prev = base != 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint64_t i = base + k;
    if (i >= na) break;
    const uint32_t x = __ldg(a + i);
    if (!(have_prev && x == prev) && contains(b, nb, x)) m |= 1u << k;
    prev = x;
    have_prev = true;
  }
  return m;
}

// Exclusive block scan of per-thread counts; returns this thread's offset
// and writes the block total to *total.
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  uint32_t before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) before += warp_sums[w];
    all += warp_sums[w];
  }
  *total = all;
  return before + incl - v;
}

__global__ void __launch_bounds__(kThreads)
    isect_count(const uint32_t* __restrict__ a, uint64_t na, const uint32_t* __restrict__ b,
                uint64_t nb, uint32_t* __restrict__ tile_count) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kPer;
  const uint32_t m = matches(a, na, b, nb, base);
  uint32_t total;
  block_scan(__popc(m), &total);
  if (threadIdx.x == 0) tile_count[blockIdx.x] = total;
}

// In-place exclusive scan of the tile counts by one CTA; *count = total.
__global__ void __launch_bounds__(kThreads)
    isect_scan(uint32_t* __restrict__ tile_count, uint32_t ntiles, uint64_t* __restrict__ count) {
  uint64_t carry = 0;
  for (uint32_t t0 = 0; t0 < ntiles; t0 += kThreads) {
    const uint32_t i = t0 + threadIdx.x;
    const uint32_t v = i < ntiles ? tile_count[i] : 0u;
    uint32_t total;
    const uint32_t off = block_scan(v, &total);
    if (i < ntiles) tile_count[i] = (uint32_t)(carry + off);
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = carry;
}

__global__ void __launch_bounds__(kThreads)
    isect_write(const uint32_t* __restrict__ a, uint64_t na, const uint32_t* __restrict__ b,
                uint64_t nb, const uint32_t* __restrict__ tile_off, uint32_t* __restrict__ out) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kPer;
  const uint32_t m = matches(a, na, b, nb, base);
  uint32_t total;
  uint32_t o = tile_off[blockIdx.x] + block_scan(__popc(m), &total);
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (m >> k & 1u) out[o++] = __ldg(a + base + k);
}

// ---- compaction of the probe sink's hit bits (izg_decode_intersect) -----
// Bit i of `hits` is set when s[i] was found in a decoded tile.  Equal
// elements of s are either all found or none (a value's repeats are merged
// in the same round or the next), so repeats are dropped by keeping bit i
// only when bit i-1 is clear or s[i-1] != s[i].  One warp per group of 32
// hit words (1,024 elements of s), lane j on element j of each word; loads
// of s are coalesced and issued only for set bits.

constexpr int kGroupWords = 32;

// Calls f(keep_mask, x) for the group's words in order; x = s[32w+lane]
// when this lane's bit is set.  The loads of 8 words are issued together;
// lane 0's predecessor is lane 31 of the previous word (loaded whenever
// both bits are set, which is the only case the comparison needs it).
template <typename F>
__device__ __forceinline__ void for_group(const uint32_t* __restrict__ s,
                                          const uint32_t* __restrict__ hits, uint64_t nw,
                                          uint64_t g, F&& f) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = g * kGroupWords;
  const uint32_t mw = w0 + lane < nw ? hits[w0 + lane] : 0u;
  uint32_t prev_m = w0 ? hits[w0 - 1] : 0u;  // previous group's last word
  uint32_t prev_x = (prev_m >> 31) && lane == 31 ? __ldg(s + 32 * w0 - 1) : 0u;
#pragma unroll 1
  for (int k0 = 0; k0 < kGroupWords; k0 += 8) {
    uint32_t ms[8], xs[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      ms[t] = __shfl_sync(0xFFFFFFFFu, mw, k0 + t);
      xs[t] = (ms[t] >> lane) & 1u ? __ldg(s + 32 * (w0 + k0 + t) + lane) : 0u;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t m = ms[t], x = xs[t];
      if (m) {
        const bool bit = (m >> lane) & 1u;
        const bool pbit = lane ? (m >> (lane - 1)) & 1u : prev_m >> 31;
        uint32_t px = __shfl_up_sync(0xFFFFFFFFu, x, 1);
        const uint32_t carry = __shfl_sync(0xFFFFFFFFu, prev_x, 31);
        if (lane == 0) px = carry;
        f(__ballot_sync(0xFFFFFFFFu, bit && !(pbit && px == x)), x);
      }
      prev_m = m;
      prev_x = x;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    hits_count(const uint32_t* __restrict__ s, const uint32_t* __restrict__ hits, uint64_t nw,
               uint64_t ngroups, uint32_t* __restrict__ group_count) {
  const uint64_t g = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (g >= ngroups) return;
  uint32_t total = 0;
  for_group(s, hits, nw, g, [&](uint32_t keep, uint32_t) { total += __popc(keep); });
  if ((threadIdx.x & 31) == 0) group_count[g] = total;
}

__global__ void __launch_bounds__(kThreads)
    hits_write(const uint32_t* __restrict__ s, const uint32_t* __restrict__ hits, uint64_t nw,
               uint64_t ngroups, const uint32_t* __restrict__ group_off,
               uint32_t* __restrict__ out) {
  const uint64_t g = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (g >= ngroups) return;
  const int lane = threadIdx.x & 31;
  uint32_t o = group_off[g];
  for_group(s, hits, nw, g, [&](uint32_t keep, uint32_t x) {
    if ((keep >> lane) & 1u) out[o + __popc(keep & ((1u << lane) - 1u))] = x;
    o += __popc(keep);
  });
}

}  // namespace

// Words of hit bits for a probe list of n_s (one spare word: a round's
// ballot may straddle two words) and compaction groups.
uint64_t hit_words(uint64_t n_s) { return (n_s + 31) / 32 + 1; }
uint64_t compact_tiles(uint64_t n_s) { return ((n_s + 31) / 32 + kGroupWords - 1) / kGroupWords; }

int compact_hits(const uint32_t* d_s, uint64_t n_s, const uint32_t* hits, uint32_t* groups,
                 uint32_t* d_out, uint64_t* d_count, cudaStream_t st) {
  if (n_s == 0)
    return cudaMemsetAsync(d_count, 0, sizeof(uint64_t), st) == cudaSuccess ? IZG_SUCCESS
                                                                           : IZG_ERR_CUDA;
  const uint64_t nw = (n_s + 31) / 32, ng = compact_tiles(n_s);
  const uint64_t grid = (ng + kThreads / 32 - 1) / (kThreads / 32);
  if (ng > 0x7FFFFFFFu) return IZG_ERR_INVALID_ARGUMENT;
  hits_count<<<(unsigned)grid, kThreads, 0, st>>>(d_s, hits, nw, ng, groups);
  isect_scan<<<1, kThreads, 0, st>>>(groups, (uint32_t)ng, d_count);
  hits_write<<<(unsigned)grid, kThreads, 0, st>>>(d_s, hits, nw, ng, groups, d_out);
  return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
}

}  // namespace izg

extern "C" uint64_t izg_intersect_workspace_size(uint64_t n_a, uint64_t n_b) {
  const uint64_t n = n_a < n_b ? n_a : n_b;
  return ((n + izg::kTile - 1) / izg::kTile) * 4 + 16;
}

extern "C" int izg_intersect_sorted(const uint32_t* d_a, uint64_t n_a, const uint32_t* d_b,
                                    uint64_t n_b, uint32_t* d_out, uint64_t* d_count,
                                    void* d_ws, uint64_t ws_bytes, void* stream) {
  using namespace izg;
  if (!d_count || (n_a && !d_a) || (n_b && !d_b)) return IZG_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_a > n_b) {  // the shorter array drives
    const uint32_t* t = d_a;
    d_a = d_b;
    d_b = t;
    const uint64_t u = n_a;
    n_a = n_b;
    n_b = u;
  }
  if (n_a == 0 || n_b == 0) {
    return cudaMemsetAsync(d_count, 0, sizeof(uint64_t), s) == cudaSuccess ? IZG_SUCCESS
                                                                          : IZG_ERR_CUDA;
  }
  const uint64_t ntiles = (n_a + kTile - 1) / kTile;
  if (!d_out || !d_ws || ws_bytes < izg_intersect_workspace_size(n_a, n_b) ||
      ntiles > 0x7FFFFFFFu)
    return IZG_ERR_INVALID_ARGUMENT;
  uint32_t* tiles = static_cast<uint32_t*>(d_ws);
  isect_count<<<(unsigned)ntiles, kThreads, 0, s>>>(d_a, n_a, d_b, n_b, tiles);
  isect_scan<<<1, kThreads, 0, s>>>(tiles, (uint32_t)ntiles, d_count);
  isect_write<<<(unsigned)ntiles, kThreads, 0, s>>>(d_a, n_a, d_b, n_b, tiles, d_out);
  return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
}
