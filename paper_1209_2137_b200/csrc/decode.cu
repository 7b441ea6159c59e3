// decode.cu — fused decode kernels and the izg_decode / izg_checksum C ABI.
//
// Kernel shape: persistent CTAs of kWarps independent warps.
// Each warp claims whole chunks, streams the chunk's compressed payload into
// its private 4 KiB shared-memory ring with TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx), decodes straight out of the ring with the prefix sum
// fused, and writes every decoded integer to HBM exactly once.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/intzip_b200.h"
#include "decode_kernel.cuh"
#include "group.cuh"
#include "split.cuh"
#include "relay.cuh"
#include "encode.cuh"

namespace izg {

// ---- checksum ------------------------------------------------------------

__global__ void checksum_kernel(const uint32_t* __restrict__ d, uint64_t n,
                                unsigned long long* __restrict__ res) {
  unsigned long long s = 0, x = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w = d[i];
    s += (w + 1) * (2 * i + 1);
    x ^= w;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    x ^= __shfl_xor_sync(0xFFFFFFFFu, x, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&res[0], s);
    atomicXor(&res[1], x);
  }
}

// ---- launch plumbing -------------------------------------------------------



// 2-D view of the output for TMA stores: rows of 32 integers (128 B), box
// of 16 rows (one warp iteration), 128-byte swizzle.  The row extent is
// nominal (the kernel only stores rows of real chunks).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

#ifndef IZG_TMA_STORE
#define IZG_TMA_STORE 1  // full iterations leave through TMA tensor stores (else st.global.v4)
#endif
bool make_out_map(CUtensorMap* m, uint32_t* out) {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  if (!fn || (reinterpret_cast<uintptr_t>(out) & 127)) return false;
  const cuuint64_t dims[2] = {32, cuuint64_t{1} << 31};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, 16};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Scalar-array FastPFOR kernels live in decode_scalar.cu (ptxas -O1, see
// there); every other decode kernel is instantiated in this file.
KernelFn pick_fastpfor_scalar(int delta);
// Probe-sink (decode -> intersect) kernels: decode_probe.cu.
KernelFn pick_probe_kernel(int codec, int delta);
// Split (several warps per chunk) kernels: decode_split.cu.
using SplitFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                         uint32_t*, SplitArgs, IdxView);
SplitFn pick_split(int codec, int delta);

// SIMD-BP128 group kernels (KW warps per chunk): decode_group.cu.
using GroupFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                         uint32_t*, uint32_t*, const CUtensorMap, int);
GroupFn pick_group(int kw, int delta);
// CTA-cooperative SIMD-BP128 kernels (one CTA per SM): decode_cta.cu.
GroupFn pick_cta(int delta);
RelayFn pick_relay(int delta);
size_t cta_smem_bytes();
int cta_threads();
// Team SIMD-FastPFOR decode (one CTA per page, indexed path): decode_team.cu.
using TeamFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                        uint32_t*, uint32_t*, const CUtensorMap, int, IdxView);
TeamFn pick_team(int delta);
size_t team_smem_bytes();
int team_threads();

// Indexed SIMD-FastPFOR batches of at least IZG_TEAM_MIN pages decode with
// the team kernel (team.cuh: one CTA of 8 decoding warps + a staging warp
// per page).  Measured on B200 (tools/team_sweep.py, 65,536-integer pages,
// ms, team vs the path taken otherwise; C5 data / C4 10 % outliers): 64
// pages 0.093 vs 0.092 (split) / 0.142 vs 0.137; 256: 0.103 vs 0.129 / 0.152
// vs 0.186; 1,024: 0.192 vs 0.259 / 0.249 vs 0.357; 2,048: 0.269 vs 0.353
// (one warp per page) / 0.379 vs 0.564; 8,192: 0.867 vs 0.997 / 1.30 vs
// 1.72; 32,768: 3.08 vs 3.15 / 4.17 vs 5.08.  IZG_TEAM=0 / 1 forces it off /
// on; IZG_SPLIT=1 (the split kernel forced) also turns it off.
#ifndef IZG_TEAM_MIN
#define IZG_TEAM_MIN 128
#endif
int env_switch(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : -1;
}
bool team_wanted(uint32_t n_chunks) {
  static const int force = env_switch("IZG_TEAM");
  static const int split_force = env_switch("IZG_SPLIT");
  if (force >= 0) return force != 0;
  return split_force != 1 && n_chunks >= IZG_TEAM_MIN;
}

// SIMD-BP128 array-mode batches of up to IZG_CTA_MAX chunks take the
// CTA-cooperative kernel (cta.cuh): with fewer chunks than ~2 per resident
// warp, one warp per chunk is latency-bound.  Measured on B200
// (tools/cta_sweep.py, 65,536-integer ClusterData d=29 chunks, ms, CTA vs
// the path taken otherwise): 64: 0.025 vs 0.041 (split); 128: 0.025 vs
// 0.047; 256: 0.037 vs 0.074; 384: 0.049 vs 0.083; 512: 0.061 vs 0.090
// (group KW 4); 768: 0.086 vs 0.110; 1,024 (C1): 0.102 vs 0.115 (one warp
// per chunk); 1,536: 0.148 vs 0.151; 2,048: 0.190 vs 0.151.  IZG_CTA=0 / 1
// forces it off / on (tests, sweeps).
#ifndef IZG_CTA_MIN
#define IZG_CTA_MIN 1
#endif
#ifndef IZG_CTA_MAX
#define IZG_CTA_MAX 1600
#endif
bool cta_wanted(int codec, int delta, uint32_t n_chunks) {
  if (codec != IZG_SIMDBP128 || delta == IZG_DELTA_NONE) return false;
  static const int force = [] {
    const char* e = std::getenv("IZG_CTA");
    return e ? std::atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  return n_chunks >= IZG_CTA_MIN && n_chunks <= IZG_CTA_MAX;
}

// Warps per chunk for a SIMD-BP128 batch that does not take the split
// kernel, by batch size against the resident warp slots.  IZG_GROUP=1, 2, 4
// or 8 forces it (tuning sweeps).
uint32_t group_warps(uint32_t n_chunks, uint32_t warp_slots) {
  static const int force = [] {
    const char* e = std::getenv("IZG_GROUP");
    const int v = e ? std::atoi(e) : 0;
    return v == 1 || v == 2 || v == 4 || v == 8 ? v : 0;
  }();
  if (force) return (uint32_t)force;
  // measured (tools/group_ab.sh, 65,536-integer chunks, 3,552 slots): KW 8
  // best up to ~200 chunks, KW 4 up to ~900, one warp per chunk from 1,024
  constexpr uint32_t kMaxKw = Layout<IZG_SIMDBP128>::kWarps;  // a group lives in one CTA
  if ((uint64_t)n_chunks * 16 <= warp_slots) return kMaxKw >= 8 ? 8 : kMaxKw;
  if ((uint64_t)n_chunks * 4 <= warp_slots) return kMaxKw >= 4 ? 4 : kMaxKw;
  return 1;
}

// Small batches decode with the split kernel (split.cuh) when the caller
// gives a workspace: with few chunks one warp per chunk leaves SMs idle.
// Crossovers measured with tools/split_sweep.py on B200 (65,536-integer
// chunks): SIMD-BP128 split wins up to ~300 chunks against the group kernel
// (64: 0.035 vs 0.066 ms; 256: 0.067 vs 0.076; 512: 0.101 vs 0.089), and
// SIMD-FastPFOR up to ~1,024 pages against one warp per page (64: 0.154 vs
// 0.379 ms; 1,024: 0.398 vs 0.504 ms).  IZG_SPLIT=0 / 1 in the environment
// forces it off / on.
constexpr uint32_t kSplitMaxChunksBp = 384, kSplitMaxChunksFp = 1024;
// Indexed SIMD-FastPFOR batches from this many pages on use the 24-warp,
// 80-register decode shape (C5's 65,536 pages: 7.00 vs 7.09 ms); below it
// the 20-warp, 96-register one (8,192 C5 pages: 1.038 vs 1.053 ms; C4's
// 2,048: 0.571 vs 0.617).
#ifndef IZG_BIG_IDX_BATCH
#define IZG_BIG_IDX_BATCH 24576
#endif
constexpr uint32_t kBigIdxBatch = IZG_BIG_IDX_BATCH;
// SIMD-FastPFOR page index pass: one lane per page from IZG_INDEX_LANES_MIN
// pages on, one warp per page below (identical workspace contents).  The
// lane walk is latency-bound (~0.4 ms whatever the batch: every page's walk
// runs at once), the warp walk issue-bound: measured (tools/idx_only.py, C5
// pages, ms, lane / warp): 8,192: 0.39 / 0.19; 16,384: 0.40 / 0.34; 32,768:
// 0.46 / 0.62; 65,536: 0.49 / 1.19 (round 2's first lane walk, loading each
// entry from global memory: 0.93).  IZG_INDEX_LANES_MIN=0 / huge forces it.
#ifndef IZG_INDEX_LANES_MIN
#define IZG_INDEX_LANES_MIN 20480
#endif
bool split_wanted(int codec, uint32_t n_chunks) {
  if (codec != IZG_SIMDBP128 && codec != IZG_SIMDFASTPFOR) return false;
  static const int force = [] {
    const char* e = std::getenv("IZG_SPLIT");
    return e ? std::atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  return n_chunks <= (codec == IZG_SIMDBP128 ? kSplitMaxChunksBp : kSplitMaxChunksFp);
}
// SIMD-BP128 batches of one to a few waves of the 3,552 resident warp slots
// (BASELINE's C2 / C3: 4,096 chunks) take the relay kernel (relay.cuh) when
// the caller gives a workspace: segments of a chunk claimed level by level,
// so the batch's tail is quantised in segments instead of whole chunks.
// IZG_RELAY=0 / 1 forces it off / on; IZG_RELAY_SEGS=1..32 (a power of two) sets the levels.
#ifndef IZG_RELAY_MIN
#define IZG_RELAY_MIN 2432
#endif
#ifndef IZG_RELAY_MAX
#define IZG_RELAY_MAX 14208
#endif
// Measured (tools/relay_sweep.py, SIMD-BP128+D4, ClusterData d=29, ms, one warp per chunk
// vs relay with 2 / 4 / 8 / 16 levels): 3,552 chunks 0.250 vs 0.247 / 0.239 / 0.232 / 0.241;
// 4,096: 0.297 vs 0.269 / 0.265 / 0.261 / 0.273; 6,144: 0.397 vs 0.388 / 0.386 / 0.380 / 0.400;
// 8,192: 0.510 vs 0.511 / 0.499 / 0.503 / 0.531; 12,288: 0.768 vs 0.747 / 0.732 / 0.744 /
// 0.793; 16,384: 0.967 vs 0.970 / 0.969 / 0.985 / 1.051 — eight levels up to 7,168 chunks,
// four above, none past four waves.  Below one wave (relay 8 vs one warp per chunk): 1,700
// chunks 0.163 vs 0.150; 2,048: 0.175 vs 0.152; 2,560: 0.192 vs 0.203; 3,072: 0.206 vs 0.227;
// 3,400: 0.228 vs 0.242 — from 2,432 chunks on.
#ifndef IZG_RELAY_SPLIT8
#define IZG_RELAY_SPLIT8 7168
#endif
bool relay_wanted(int codec, uint32_t n_chunks) {
  if (codec != IZG_SIMDBP128) return false;
  static const int force = env_switch("IZG_RELAY");
  if (force >= 0) return force != 0;
  return n_chunks >= IZG_RELAY_MIN && n_chunks <= IZG_RELAY_MAX;
}
uint64_t relay_ws_bytes(uint32_t n_chunks) { return relay_state_bytes(n_chunks) + 64; }
uint64_t split_ws_offset(int codec, uint32_t n_chunks) {
  return codec == IZG_SIMDFASTPFOR ? (idx_workspace_bytes(n_chunks) + 15) / 16 * 16 : 0;
}
uint64_t workspace_bytes(int codec, uint32_t n_chunks) {
  const uint64_t base = codec == IZG_SIMDFASTPFOR ? idx_workspace_bytes(n_chunks) : 0;
  if (relay_wanted(codec, n_chunks) && !split_wanted(codec, n_chunks))
    return relay_ws_bytes(n_chunks);
  if (!split_wanted(codec, n_chunks)) return base;
  return split_ws_offset(codec, n_chunks) + split_state_bytes(n_chunks);
}


constexpr uint32_t kCounterSlots = 1024;
static_assert(sizeof(FpScratch) <= Layout<IZG_SIMDFASTPFOR>::kTabBytes, "FpScratch layout");
constexpr int kCodecs = 5;  // SIMD-BP128, SIMD-FastPFOR, BP32, FastPFOR, SimplePFOR
static_assert(Layout<IZG_SIMDFASTPFOR>::kTabBytes % 16 == 0, "FpScratch alignment");

struct DeviceInfo {
  bool init = false;
  bool ok = false;
  int sms = 0;
  // [codec (+ kCodecs: indexed page path, + 2 kCodecs: probe sink,
  //  + 3 kCodecs: split kernels, 4 kCodecs + 0..2: group kernels KW = 2, 4, 8)][delta]
  int occ[4 * kCodecs + 7][5] = {};  // + 4 kCodecs + 3: big indexed, + 4: CTA kernel, + 5: team, + 6: relay
  uint32_t* counters = nullptr;  // chunk-claim counters, one per in-flight launch
  uint32_t next_slot = 0;
};

DeviceInfo g_dev[64];
std::mutex g_dev_mu;

// Device of a pointer (the caller's buffers decide where we run).
int device_of(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return -1;
  return a.device;
}

// `variant` = codec, + kCodecs for the indexed page decode kernels, + 2 kCodecs
// for the probe-sink kernels, + 3 kCodecs for the split kernels.
int prepare(int dev, int variant, int delta, const void* fn, int threads, size_t smem,
            int* grid_per_sm, int* sms, uint32_t** counter) {
  if (dev < 0 || dev >= 64) return IZG_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& d = g_dev[dev];
  if (!d.init) {
    d.init = true;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return IZG_ERR_CUDA;
    d.ok = p.major == 10;  // sm_100 family only: no fallback path exists
    d.sms = p.multiProcessorCount;
    if (d.ok && cudaMalloc(&d.counters, kCounterSlots * sizeof(uint32_t)) != cudaSuccess) {
      d.ok = false;
      return IZG_ERR_CUDA;
    }
  }
  if (!d.ok) return IZG_ERR_NO_DEVICE;
  if (!d.occ[variant][delta]) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return IZG_ERR_CUDA;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) !=
            cudaSuccess ||
        occ < 1)
      return IZG_ERR_CUDA;
    d.occ[variant][delta] = occ;
  }
  *grid_per_sm = d.occ[variant][delta];
  *sms = d.sms;
  *counter = d.counters + (d.next_slot++ % kCounterSlots);
  return IZG_SUCCESS;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace izg

namespace izg {

// `probe` non-null: decode -> intersect (ProbeStage sink, no output; d_out
// is unused and the indexed path is not taken).
// `phase` (SIMD-FastPFOR's indexed path only): 0 = index pass + decode,
// 1 = the page index pass alone, 2 = the decode alone from a workspace that
// phase 1 filled for the same words and table (stream order).
int decode_impl(int codec, int delta, const uint32_t* d_words, const izg_chunk* d_chunks,
                uint32_t n_chunks, uint32_t* d_out, int32_t* d_status, uint32_t* d_consumed,
                void* d_ws, uint64_t ws_bytes, void* stream, const ProbeArgs* probe = nullptr,
                int phase = 0) {
  if (codec < IZG_SIMDBP128 || codec > IZG_SIMPLEPFOR) return IZG_ERR_INVALID_ARGUMENT;
  if (delta < IZG_DELTA_NONE || delta > IZG_DELTA_DM) return IZG_ERR_INVALID_ARGUMENT;
  if (probe && delta != IZG_DELTA_D1 && delta != IZG_DELTA_D4) return IZG_ERR_INVALID_ARGUMENT;
  if (n_chunks == 0) return IZG_SUCCESS;
  if (!d_words || !d_chunks || (!d_out && !probe) || !d_status) return IZG_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(d_words) & 15) return IZG_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return IZG_ERR_NO_DEVICE;
  }
  const int dev = device_of(d_status);
  if (dev < 0) return IZG_ERR_INVALID_ARGUMENT;
  const bool paged = codec == IZG_SIMDFASTPFOR || codec == IZG_FASTPFOR ||
                     codec == IZG_SIMPLEPFOR;
  // The indexed path serves SIMD-FastPFOR.  Scalar-array FastPFOR pages
  // decode with the fused kernel: its indexed variant faulted on pages with
  // exceptions in a code-layout-dependent way, so it is not
  // built until that is understood.
  const bool idx = !probe && codec == IZG_SIMDFASTPFOR && d_ws &&
                   (reinterpret_cast<uintptr_t>(d_ws) & 15) == 0 &&
                   ws_bytes >= idx_workspace_bytes(n_chunks);
  // very large indexed batches: the 24-warp shape (Layout SHAPE 1)
  static const uint32_t big_from = [] {  // IZG_BIG_IDX_BATCH=n: tests / tuning
    const char* e = std::getenv("IZG_BIG_IDX_BATCH");
    return e ? (uint32_t)std::strtoul(e, nullptr, 10) : kBigIdxBatch;
  }();
  const bool big = idx && n_chunks >= big_from;
  KernelFn fn = nullptr;
  switch (codec) {
    case IZG_SIMDBP128: fn = pick<IZG_SIMDBP128, false>(delta); break;
    case IZG_BP32: fn = pick<IZG_BP32, false>(delta); break;
    case IZG_SIMDFASTPFOR:
      fn = big ? pick<IZG_SIMDFASTPFOR, true, 1>(delta)
           : idx ? pick<IZG_SIMDFASTPFOR, true>(delta)
                 : pick<IZG_SIMDFASTPFOR, false>(delta);
      break;
    case IZG_FASTPFOR: fn = pick_fastpfor_scalar(delta); break;
    case IZG_SIMPLEPFOR: fn = pick<IZG_SIMPLEPFOR, false>(delta); break;
  }
  if (probe) fn = pick_probe_kernel(codec, delta);
  DeviceGuard guard(dev);
  int per_sm = 0, sms = 0;
  uint32_t* counter = nullptr;
  const int warps = big     ? Layout<IZG_SIMDFASTPFOR, true, 1>::kWarps
                    : idx   ? Layout<IZG_SIMDFASTPFOR, true>::kWarps
                    : paged ? Layout<IZG_SIMDFASTPFOR>::kWarps
                            : Layout<IZG_SIMDBP128>::kWarps;
  const size_t smem = big     ? Layout<IZG_SIMDFASTPFOR, true, 1>::kSmem
                      : idx   ? Layout<IZG_SIMDFASTPFOR, true>::kSmem
                      : paged ? Layout<IZG_SIMDFASTPFOR>::kSmem
                              : Layout<IZG_SIMDBP128>::kSmem;
  const bool team = idx && team_wanted(n_chunks);
  const bool split = !team && !probe && split_wanted(codec, n_chunks) && d_ws &&
                     (reinterpret_cast<uintptr_t>(d_ws) & 15) == 0 &&
                     ws_bytes >= workspace_bytes(codec, n_chunks);
  const void* kfn = split ? reinterpret_cast<const void*>(pick_split(codec, delta))
                          : reinterpret_cast<const void*>(fn);
  // phases only exist where a page index pass runs (the indexed decode and
  // SIMD-FastPFOR's split decode): elsewhere phase 1 has nothing to do and
  // phase 2 is the whole decode
  if (phase == 1 && !idx) return IZG_SUCCESS;
  int rc = prepare(dev, big ? 4 * kCodecs + 3
                           : codec + (split ? 3 * kCodecs : idx ? kCodecs : probe ? 2 * kCodecs : 0),
                   delta, kfn, warps * 32, smem, &per_sm, &sms,
                   &counter);
  if (rc != IZG_SUCCESS) return rc;
  const bool relay = !probe && !split && relay_wanted(codec, n_chunks) && d_ws &&
                     (reinterpret_cast<uintptr_t>(d_ws) & 15) == 0 &&
                     ws_bytes >= relay_ws_bytes(n_chunks);
  if (!probe && !relay && cta_wanted(codec, delta, n_chunks)) {
    GroupFn cfn = pick_cta(delta);
    int cper_sm = 0, csms = 0;
    uint32_t* ccounter = nullptr;
    rc = prepare(dev, 4 * kCodecs + 4, delta, reinterpret_cast<const void*>(cfn), cta_threads(),
                 cta_smem_bytes(), &cper_sm, &csms, &ccounter);
    if (rc != IZG_SUCCESS) return rc;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(ccounter, 0, sizeof(uint32_t), cs) != cudaSuccess) return IZG_ERR_CUDA;
    const uint32_t grid = (uint32_t)std::min<uint64_t>(n_chunks, (uint64_t)csms);
    CUtensorMap omap;
    std::memset(&omap, 0, sizeof(omap));
    const int tma_out = IZG_TMA_STORE && make_out_map(&omap, d_out) ? 1 : 0;
    cfn<<<grid, cta_threads(), cta_smem_bytes(), cs>>>(d_words, d_chunks, n_chunks, d_out,
                                                       d_status, d_consumed, ccounter, omap,
                                                       tma_out);
    return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
  }
  if (relay) {
    RelayFn rfn = pick_relay(delta);
    int rper_sm = 0, rsms = 0;
    uint32_t* rcounter = nullptr;
    rc = prepare(dev, 4 * kCodecs + 6, delta, reinterpret_cast<const void*>(rfn), warps * 32,
                 smem, &rper_sm, &rsms, &rcounter);
    if (rc != IZG_SUCCESS) return rc;
    cudaStream_t rs = static_cast<cudaStream_t>(stream);
    // per-chunk states and, behind them, the task counter: one memset
    if (cudaMemsetAsync(d_ws, 0, relay_ws_bytes(n_chunks), rs) != cudaSuccess)
      return IZG_ERR_CUDA;
    static const int force_segs = [] {
      const char* e = std::getenv("IZG_RELAY_SEGS");
      const int v = e ? std::atoi(e) : 0;
      return v >= 1 && v <= 32 && (v & (v - 1)) == 0 ? v : 0;
    }();
    RelayArgs ra;
    ra.st = static_cast<RelayState*>(d_ws);
    ra.next_task = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(d_ws) +
                                               relay_state_bytes(n_chunks));
    ra.summary = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(d_ws) +
                                                       relay_state_bytes(n_chunks) + 8);
    ra.levels = (uint32_t)(force_segs ? force_segs : n_chunks <= IZG_RELAY_SPLIT8 ? 8 : 4);
    ra.seg_blocks = (IZG_CHUNK_SIZE / 128) / ra.levels;
    const uint64_t tasks = (uint64_t)n_chunks * ra.levels;
    const uint32_t grid =
        (uint32_t)std::min<uint64_t>((tasks + warps - 1) / warps, (uint64_t)rper_sm * rsms);
    CUtensorMap omap;
    std::memset(&omap, 0, sizeof(omap));
    const int tma_out = IZG_TMA_STORE && make_out_map(&omap, d_out) ? 1 : 0;
    rfn<<<grid, warps * 32, smem, rs>>>(d_words, d_chunks, n_chunks, d_out, d_status, d_consumed,
                                        ra, omap, tma_out);
    return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
  }
  if (codec == IZG_SIMDBP128 && !probe && !split) {
    // SIMD-BP128 small batches: KW warps per chunk (group.cuh); the one-warp
    // kernel's warp slots (same registers and ring) set KW
    // (warp slots as designed: 3 CTAs of 8 warps per SM at 80 registers)
    const uint32_t kw = group_warps(n_chunks, (uint32_t)(24 * sms));
    if (kw > 1) {
      GroupFn gfn = pick_group((int)kw, delta);
      const size_t gsmem = GroupLayout::kSmem;
      const int variant = 4 * kCodecs + (kw == 2 ? 0 : kw == 4 ? 1 : 2);
      int gper_sm = 0, gsms = 0;
      uint32_t* gcounter = nullptr;
      rc = prepare(dev, variant, delta, reinterpret_cast<const void*>(gfn), warps * 32, gsmem,
                   &gper_sm, &gsms, &gcounter);
      if (rc != IZG_SUCCESS) return rc;
      cudaStream_t gs = static_cast<cudaStream_t>(stream);
      if (cudaMemsetAsync(gcounter, 0, sizeof(uint32_t), gs) != cudaSuccess) return IZG_ERR_CUDA;
      const uint64_t want = ((uint64_t)n_chunks * kw + warps - 1) / warps;
      const uint32_t grid = (uint32_t)std::min<uint64_t>(want, (uint64_t)gper_sm * gsms);
      CUtensorMap omap;
      std::memset(&omap, 0, sizeof(omap));
      const int tma_out = IZG_TMA_STORE && make_out_map(&omap, d_out) ? 1 : 0;
      gfn<<<grid, warps * 32, gsmem, gs>>>(d_words, d_chunks, n_chunks, d_out, d_status,
                                           d_consumed, gcounter, omap, tma_out);
      return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  IdxView ix{};
  if (idx && phase != 2) {
    static const bool attr = [] {
      const int b = (int)IdxLayout::kSmem;
      cudaFuncSetAttribute(fp_index_kernel<false, kVertical>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, b);
      cudaFuncSetAttribute(fp_index_kernel<true, kVertical>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, b);
      const int bl = (int)IdxLaneLayout::kSmem;
      cudaFuncSetAttribute(fp_index_lanes_kernel<false, kVertical>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, bl);
      cudaFuncSetAttribute(fp_index_lanes_kernel<true, kVertical>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, bl);
      return true;
    }();
    (void)attr;
    ix = idx_view(d_ws, n_chunks);
    static const uint32_t lanes_min = [] {  // IZG_INDEX_LANES_MIN: tests / tuning
      const char* e = std::getenv("IZG_INDEX_LANES_MIN");
      return e ? (uint32_t)std::strtoul(e, nullptr, 10) : (uint32_t)IZG_INDEX_LANES_MIN;
    }();
    if (n_chunks >= lanes_min) {  // one lane per page (index_fastpfor.cuh)
      const uint32_t g = (n_chunks + 32 * kIdxLaneWarps - 1) / (32 * kIdxLaneWarps);
      auto* lfn = delta == IZG_DELTA_NONE ? fp_index_lanes_kernel<false, kVertical>
                                          : fp_index_lanes_kernel<true, kVertical>;
      lfn<<<g, kIdxLaneWarps * 32, IdxLaneLayout::kSmem, s>>>(d_words, d_chunks, n_chunks, ix);
    } else {
      const uint32_t g = (n_chunks + kIdxWarps - 1) / kIdxWarps;
      auto* ifn = delta == IZG_DELTA_NONE ? fp_index_kernel<false, kVertical>
                                          : fp_index_kernel<true, kVertical>;
      ifn<<<g, kIdxWarps * 32, IdxLayout::kSmem, s>>>(d_words, d_chunks, n_chunks, ix);
    }
    if (phase == 1) return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
  } else if (idx) {
    ix = idx_view(d_ws, n_chunks);
  }
  if (cudaMemsetAsync(counter, 0, sizeof(uint32_t), s) != cudaSuccess) return IZG_ERR_CUDA;
  if (team) {
    TeamFn tfn = pick_team(delta);
    int tper_sm = 0, tsms = 0;
    uint32_t* tcounter = nullptr;
    rc = prepare(dev, 4 * kCodecs + 5, delta, reinterpret_cast<const void*>(tfn), team_threads(),
                 team_smem_bytes(), &tper_sm, &tsms, &tcounter);
    if (rc != IZG_SUCCESS) return rc;
    if (cudaMemsetAsync(tcounter, 0, sizeof(uint32_t), s) != cudaSuccess) return IZG_ERR_CUDA;
    const uint32_t grid = (uint32_t)std::min<uint64_t>(n_chunks, (uint64_t)tper_sm * tsms);
    CUtensorMap omap;
    std::memset(&omap, 0, sizeof(omap));
    const int tma_out = IZG_TMA_STORE && make_out_map(&omap, d_out) ? 1 : 0;
    tfn<<<grid, team_threads(), team_smem_bytes(), s>>>(d_words, d_chunks, n_chunks, d_out,
                                                        d_status, d_consumed, tcounter, omap,
                                                        tma_out, ix);
    return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
  }
  if (split) {
    SplitArgs sa;
    sa.seg = reinterpret_cast<SegState*>(static_cast<uint8_t*>(d_ws) +
                                         split_ws_offset(codec, n_chunks));
    sa.next_unit = counter;
    if (cudaMemsetAsync(sa.seg, 0, split_state_bytes(n_chunks), s) != cudaSuccess)
      return IZG_ERR_CUDA;
    // SIMD-BP128 sizes segments to the batch; SIMD-FastPFOR keeps the
    // smallest (measured best at every batch size it is selected for)
    sa.seg_blocks = codec == IZG_SIMDBP128
                        ? split_seg_blocks(n_chunks, (uint32_t)(per_sm * sms * warps))
                        : kFpSegBlocks;
    static const int force_segs = [] {  // IZG_SPLIT_SEGS=1..16: tuning sweeps
      const char* e = std::getenv("IZG_SPLIT_SEGS");
      const int v = e ? std::atoi(e) : 0;
      return v >= 1 && v <= (int)kMaxSegs && (v & (v - 1)) == 0 ? v : 0;
    }();
    if (force_segs) sa.seg_blocks = (IZG_CHUNK_SIZE / 128) / force_segs;
    const uint64_t units = (uint64_t)n_chunks * ((IZG_CHUNK_SIZE / 128) / sa.seg_blocks);
    const uint32_t grid =
        (uint32_t)std::min<uint64_t>((units + warps - 1) / warps, (uint64_t)per_sm * sms);
    pick_split(codec, delta)<<<grid, warps * 32, smem, s>>>(d_words, d_chunks, n_chunks, d_out,
                                                             d_status, d_consumed, sa, ix);
    return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
  }
  const uint64_t want = (n_chunks + warps - 1) / warps;
  static const int cap_ctas = [] {  // IZG_BP_MAX_CTAS: co-residency experiments (SIMD-BP128)
    const char* e = std::getenv("IZG_BP_MAX_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  const int eff_per_sm =
      cap_ctas > 0 && codec == IZG_SIMDBP128 ? std::min(per_sm, cap_ctas) : per_sm;
  const uint32_t grid = (uint32_t)std::min<uint64_t>(want, (uint64_t)eff_per_sm * sms);
  CUtensorMap omap;
  std::memset(&omap, 0, sizeof(omap));
  const int tma_out = !probe && IZG_TMA_STORE && make_out_map(&omap, d_out) ? 1 : 0;
  fn<<<grid, warps * 32, smem, s>>>(d_words, d_chunks, n_chunks, d_out, d_status, d_consumed,
                                    counter, omap, tma_out, ix, probe ? *probe : ProbeArgs{});
  return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
}

}  // namespace izg

extern "C" int izg_decode(int codec, int delta, const uint32_t* d_words,
                          const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
                          int32_t* d_status, uint32_t* d_consumed, void* stream) {
  return izg::decode_impl(codec, delta, d_words, d_chunks, n_chunks, d_out, d_status, d_consumed,
                          nullptr, 0, stream);
}

namespace izg {
// intersect.cu: hit bits of the probe list -> sorted distinct values
int compact_hits(const uint32_t* d_s, uint64_t n_s, const uint32_t* hits, uint32_t* tiles,
                 uint32_t* d_out, uint64_t* d_count, cudaStream_t s);
uint64_t hit_words(uint64_t n_s);
uint64_t compact_tiles(uint64_t n_s);
}  // namespace izg

extern "C" uint64_t izg_decode_intersect_workspace_size(uint64_t n_s) {
  return 4 * (izg::hit_words(n_s) + izg::compact_tiles(n_s)) + 16;
}

extern "C" int izg_decode_intersect(int codec, int delta, const uint32_t* d_words,
                                    const izg_chunk* d_chunks, uint32_t n_chunks,
                                    const uint32_t* d_s, uint64_t n_s, uint32_t* d_out,
                                    uint64_t* d_count, int32_t* d_status, void* d_ws,
                                    uint64_t ws_bytes, void* stream) {
  using namespace izg;
  if (!d_count || (n_s && (!d_s || !d_out)) || !d_ws ||
      ws_bytes < izg_decode_intersect_workspace_size(n_s) ||
      (reinterpret_cast<uintptr_t>(d_ws) & 3))
    return IZG_ERR_INVALID_ARGUMENT;
  if (delta != IZG_DELTA_D1 && delta != IZG_DELTA_D4) return IZG_ERR_INVALID_ARGUMENT;
  const int dev = device_of(d_count);
  if (dev < 0) return IZG_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* hits = static_cast<uint32_t*>(d_ws);
  uint32_t* tiles = hits + hit_words(n_s);
  if (cudaMemsetAsync(hits, 0, 4 * hit_words(n_s), s) != cudaSuccess) return IZG_ERR_CUDA;
  const ProbeArgs pa{d_s, n_s, hits};
  const int rc = decode_impl(codec, delta, d_words, d_chunks, n_chunks, nullptr, d_status,
                             nullptr, nullptr, 0, stream, &pa);
  if (rc != IZG_SUCCESS) return rc;
  return compact_hits(d_s, n_s, hits, tiles, d_out, d_count, s);
}

extern "C" uint64_t izg_decode_workspace_size(int codec, uint32_t n_chunks) {
  return izg::workspace_bytes(codec, n_chunks);
}

extern "C" uint64_t izg_decode_index_workspace_size(int codec, uint32_t n_chunks) {
  return codec == IZG_SIMDFASTPFOR ? izg::idx_workspace_bytes(n_chunks) : 0;
}

extern "C" int izg_decode_ws(int codec, int delta, const uint32_t* d_words,
                             const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
                             int32_t* d_status, uint32_t* d_consumed, void* d_workspace,
                             uint64_t workspace_bytes, void* stream) {
  return izg::decode_impl(codec, delta, d_words, d_chunks, n_chunks, d_out, d_status, d_consumed,
                          d_workspace, workspace_bytes, stream);
}

extern "C" int izg_decode_ws_phase(int codec, int delta, const uint32_t* d_words,
                                   const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
                                   int32_t* d_status, uint32_t* d_consumed, void* d_workspace,
                                   uint64_t workspace_bytes, int phase, void* stream) {
  if (phase < 0 || phase > 2) return IZG_ERR_INVALID_ARGUMENT;
  return izg::decode_impl(codec, delta, d_words, d_chunks, n_chunks, d_out, d_status, d_consumed,
                          d_workspace, workspace_bytes, stream, nullptr, phase);
}

extern "C" int izg_checksum(const uint32_t* d_data, uint64_t n, uint64_t* d_result,
                            void* stream) {
  using namespace izg;
  if (!d_result || (n && !d_data)) return IZG_ERR_INVALID_ARGUMENT;
  const int dev = device_of(d_result);
  if (dev < 0) return IZG_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(d_result, 0, 16, s) != cudaSuccess) return IZG_ERR_CUDA;
  if (n) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (n + 255) / 256;
    const unsigned grid = (unsigned)std::min<uint64_t>(want, (uint64_t)sms * 8);
    checksum_kernel<<<grid, 256, 0, s>>>(d_data, n,
                                         reinterpret_cast<unsigned long long*>(d_result));
  }
  return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
}

// ---- encoder (secondary path) ---------------------------------------------

namespace izg {

using EncodeFn = void (*)(const uint32_t*, izg_chunk*, uint32_t, uint32_t*, int32_t*, uint32_t*);

template <bool WRAP>
EncodeFn pick_enc(int codec, int delta) {
  if (codec == IZG_SIMDBP128) {
    switch (delta) {
      case IZG_DELTA_NONE: return bp128_encode_kernel<IZG_DELTA_NONE, WRAP>;
      case IZG_DELTA_D1: return bp128_encode_kernel<IZG_DELTA_D1, WRAP>;
      case IZG_DELTA_D4: return bp128_encode_kernel<IZG_DELTA_D4, WRAP>;
      case IZG_DELTA_D2: return bp128_encode_kernel<IZG_DELTA_D2, WRAP>;
      case IZG_DELTA_DM: return bp128_encode_kernel<IZG_DELTA_DM, WRAP>;
    }
  } else {
    switch (delta) {
      case IZG_DELTA_NONE: return fastpfor_encode_kernel<IZG_DELTA_NONE, WRAP>;
      case IZG_DELTA_D1: return fastpfor_encode_kernel<IZG_DELTA_D1, WRAP>;
      case IZG_DELTA_D4: return fastpfor_encode_kernel<IZG_DELTA_D4, WRAP>;
      case IZG_DELTA_D2: return fastpfor_encode_kernel<IZG_DELTA_D2, WRAP>;
      case IZG_DELTA_DM: return fastpfor_encode_kernel<IZG_DELTA_DM, WRAP>;
    }
  }
  return nullptr;
}

}  // namespace izg

extern "C" uint64_t izg_encode_bound(int codec, uint32_t n) {
  return izg::izg_encode_bound_impl(codec, n);
}

extern "C" int izg_encode(int codec, int delta, const uint32_t* d_values, izg_chunk* d_chunks,
                          uint32_t n_chunks, uint32_t* d_words, int32_t* d_status, int allow_wrap,
                          void* stream) {
  using namespace izg;
  if (codec != IZG_SIMDBP128 && codec != IZG_SIMDFASTPFOR) return IZG_ERR_INVALID_ARGUMENT;
  if (delta < IZG_DELTA_NONE || delta > IZG_DELTA_DM) return IZG_ERR_INVALID_ARGUMENT;
  if (n_chunks == 0) return IZG_SUCCESS;
  if (!d_values || !d_chunks || !d_words || !d_status) return IZG_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return IZG_ERR_NO_DEVICE;
  }
  const int dev = device_of(d_status);
  if (dev < 0) return IZG_ERR_INVALID_ARGUMENT;
  EncodeFn fn = allow_wrap ? pick_enc<true>(codec, delta) : pick_enc<false>(codec, delta);
  const size_t esmem = codec == IZG_SIMDBP128 ? 0 : kEncWarps * sizeof(FpEncScratch);
  DeviceGuard guard(dev);
  int per_sm = 0, sms = 0;
  uint32_t* counter = nullptr;
  // occupancy slot 0 of the (unused) BP128 raw-mode table is not shared with
  // decode kernels: encode uses static shared memory only
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo& d = g_dev[dev];
    if (!d.init) {
      d.init = true;
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return IZG_ERR_CUDA;
      d.ok = p.major == 10;
      d.sms = p.multiProcessorCount;
      if (d.ok && cudaMalloc(&d.counters, kCounterSlots * sizeof(uint32_t)) != cudaSuccess) {
        d.ok = false;
        return IZG_ERR_CUDA;
      }
    }
    if (!d.ok) return IZG_ERR_NO_DEVICE;
    sms = d.sms;
    counter = d.counters + (d.next_slot++ % kCounterSlots);
  }
  if (esmem && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)esmem) != cudaSuccess)
    return IZG_ERR_CUDA;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kEncWarps * 32, esmem) !=
          cudaSuccess ||
      per_sm < 1)
    return IZG_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t want = (n_chunks + kEncWarps - 1) / kEncWarps;
  const uint32_t grid = (uint32_t)std::min<uint64_t>(want, (uint64_t)per_sm * sms);
  if (cudaMemsetAsync(counter, 0, sizeof(uint32_t), s) != cudaSuccess) return IZG_ERR_CUDA;
  fn<<<grid, kEncWarps * 32, esmem, s>>>(d_values, d_chunks, n_chunks, d_words, d_status, counter);
  return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
}

#ifdef IZG_BOUNDS
// Bounds-check build: this translation unit's counters (the page index kernels).
extern "C" int izg_debug_bounds_index(void* host, int reset) {
  if (cudaMemcpyFromSymbol(host, izg::g_izg_oob, sizeof(izg::g_izg_oob)) != cudaSuccess) return -1;
  if (reset) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, izg::g_izg_oob) != cudaSuccess) return -1;
    cudaMemset(p, 0, sizeof(izg::g_izg_oob));
  }
  return 0;
}
#endif
