// decode.cu — fused decode kernels and the izg_decode / izg_checksum C ABI.
//
// Kernel shape: persistent CTAs, one producer warp whose lane 0
// streams each chunk's compressed payload into a 64 KiB shared-memory ring
// with TMA bulk copies (cp.async.bulk + mbarrier complete_tx), and eight
// consumer warps that decode straight out of the ring, fuse the prefix sum,
// and write every decoded integer to HBM exactly once.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/intzip_b200.h"
#include "decode_bp128.cuh"
#include "decode_fastpfor.cuh"
#include "izg_common.cuh"

namespace izg {

struct SmemHead {
  uint64_t full[kNStage];
  uint64_t empty[kNStage];
  uint4 tot[2][kCW];
};

// Per-chunk argument checks every role applies identically before touching
// the payload: decode_array's length check (codec.cpp:43-44) or
// decode_deltas' count checks (codec_binpack.cpp:12-15,
// codec_patched.cpp:52-57).
__device__ __forceinline__ int32_t precheck(int codec, bool array_mode, uint32_t n) {
  if (array_mode) {
    if (n == 0 || n > IZG_CHUNK_SIZE) return IZG_E_CHUNK_LENGTH;
  } else {
    if (n % 128) return IZG_E_COUNT_MULTIPLE;
    if (codec == IZG_SIMDFASTPFOR && n > IZG_CHUNK_SIZE) return IZG_E_PAGE_TOO_LARGE;
  }
  return IZG_OK;
}

template <int CODEC, int DELTA>
__global__ void __launch_bounds__(kThreads, 1)
    decode_kernel(const uint32_t* __restrict__ words, const izg_chunk* __restrict__ chunks,
                  uint32_t n_chunks, uint32_t* __restrict__ out, int32_t* __restrict__ status,
                  uint32_t* __restrict__ consumed) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  SmemHead* head = reinterpret_cast<SmemHead*>(smem + kRing);
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (uint32_t i = 0; i < kNStage; ++i) {
      mbar_init(&head->full[i], 1);
      mbar_init(&head->empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCW) {
    // ---------------- producer ----------------
    if ((tid & 31) != 0) return;
    const uint64_t pol = policy_evict_first();
    uint32_t g = 0;
    for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
      const izg_chunk ch = chunks[c];
      if (precheck(CODEC, kArray, ch.n) != IZG_OK) continue;
      const StreamGeom sg = stream_geom(words, ch.word_off, ch.n_words);
      produce_chunk(ring, head->full, head->empty, sg, g, pol);
    }
    return;
  }

  // ---------------- consumers ----------------
  uint32_t g = 0, tbuf = 0;
  for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const izg_chunk ch = chunks[c];
    int32_t st = precheck(CODEC, kArray, ch.n);
    if (st != IZG_OK) {
      if (tid == 0) {
        status[c] = st;
        if (consumed) consumed[c] = 0;
      }
      continue;
    }
    const StreamGeom sg = stream_geom(words, ch.word_off, ch.n_words);
    RingView rv{smem_u32(ring), g, sg.phase, sg.nst, 0, 0};
    g += sg.nst;
    uint32_t* o = out + ch.out_off;
    const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    const uint32_t core = kArray ? ch.n / 128 * 128 : ch.n;
    uint4 carry = make_uint4(0, 0, 0, 0);
    uint32_t pos = 0;
    if (CODEC == IZG_SIMDBP128) {
      if (sg.phase == 0)
        st = bp128_core<DELTA, true>(rv, head->full, head->empty, head->tot, tbuf, ch.n_words,
                                     core / 128, o, oal, carry, &pos);
      else
        st = bp128_core<DELTA, false>(rv, head->full, head->empty, head->tot, tbuf, ch.n_words,
                                      core / 128, o, oal, carry, &pos);
    } else {
      st = fastpfor_core<DELTA>(rv, head->full, head->empty, head->tot, tbuf, ch.n_words,
                                core / 128, o, oal, carry, &pos);
    }
    if (kArray && st == IZG_OK) {
      if (core < ch.n) {
        // Variable Byte remainder (codec.cpp:56-62), then exact consumption.
        rv.ensure(head->full, 4u * ch.n_words);
        if (tid == 0) {
          uint32_t rb = 0;
          st = vbyte_tail<DELTA>(rv, 4u * pos, 4u * (ch.n_words - pos), core, ch.n - core, carry,
                                 o, &rb);
          if (st == IZG_OK) pos += (rb + 3) / 4;
        }
      }
      if (tid == 0 && st == IZG_OK && pos != ch.n_words) st = IZG_E_PAYLOAD_SIZE;
    }
    named_bar_sync(1, kConsumers);
    rv.finish(head->full, head->empty, tid == 0);
    if (tid == 0) {
      status[c] = st;
      if (consumed) consumed[c] = st == IZG_OK ? pos : 0;
    }
  }
}

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

constexpr size_t kSmemBytes = kRing + sizeof(SmemHead);

using KernelFn = void (*)(const uint32_t*, const izg_chunk*, uint32_t, uint32_t*, int32_t*,
                          uint32_t*);

template <int CODEC>
KernelFn pick(int delta) {
  switch (delta) {
    case IZG_DELTA_NONE: return decode_kernel<CODEC, IZG_DELTA_NONE>;
    case IZG_DELTA_D1: return decode_kernel<CODEC, IZG_DELTA_D1>;
    case IZG_DELTA_D4: return decode_kernel<CODEC, IZG_DELTA_D4>;
    case IZG_DELTA_D2: return decode_kernel<CODEC, IZG_DELTA_D2>;
    case IZG_DELTA_DM: return decode_kernel<CODEC, IZG_DELTA_DM>;
  }
  return nullptr;
}

struct DeviceInfo {
  bool init = false;
  bool ok = false;
  int sms = 0;
  int occ[2][5] = {};
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

int prepare(int dev, int codec, int delta, KernelFn fn, int* grid_per_sm, int* sms) {
  if (dev < 0 || dev >= 64) return IZG_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& d = g_dev[dev];
  if (!d.init) {
    d.init = true;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return IZG_ERR_CUDA;
    d.ok = p.major == 10;  // sm_100 family only: no fallback path exists
    d.sms = p.multiProcessorCount;
  }
  if (!d.ok) return IZG_ERR_NO_DEVICE;
  if (!d.occ[codec][delta]) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSmemBytes) != cudaSuccess)
      return IZG_ERR_CUDA;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, kSmemBytes) !=
            cudaSuccess ||
        occ < 1)
      return IZG_ERR_CUDA;
    d.occ[codec][delta] = occ;
  }
  *grid_per_sm = d.occ[codec][delta];
  *sms = d.sms;
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

extern "C" int izg_decode(int codec, int delta, const uint32_t* d_words,
                          const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
                          int32_t* d_status, uint32_t* d_consumed, void* stream) {
  using namespace izg;
  if (codec != IZG_SIMDBP128 && codec != IZG_SIMDFASTPFOR) return IZG_ERR_INVALID_ARGUMENT;
  if (delta < IZG_DELTA_NONE || delta > IZG_DELTA_DM) return IZG_ERR_INVALID_ARGUMENT;
  if (n_chunks == 0) return IZG_SUCCESS;
  if (!d_words || !d_chunks || !d_out || !d_status) return IZG_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(d_words) & 15) return IZG_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return IZG_ERR_NO_DEVICE;
  }
  const int dev = device_of(d_status);
  if (dev < 0) return IZG_ERR_INVALID_ARGUMENT;
  KernelFn fn = codec == IZG_SIMDBP128 ? pick<IZG_SIMDBP128>(delta) : pick<IZG_SIMDFASTPFOR>(delta);
  DeviceGuard guard(dev);
  int per_sm = 0, sms = 0;
  int rc = prepare(dev, codec, delta, fn, &per_sm, &sms);
  if (rc != IZG_SUCCESS) return rc;
  const uint32_t grid = std::min<uint64_t>(n_chunks, (uint64_t)per_sm * sms);
  fn<<<grid, kThreads, kSmemBytes, static_cast<cudaStream_t>(stream)>>>(
      d_words, d_chunks, n_chunks, d_out, d_status, d_consumed);
  return cudaGetLastError() == cudaSuccess ? IZG_SUCCESS : IZG_ERR_CUDA;
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
