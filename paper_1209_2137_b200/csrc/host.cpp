// host.cpp — host half of the C ABI: codec registry mirror, status strings,
// buffer placement, and the synchronous host-buffer decode (the end-to-end
// entry point a user of decode_array would call).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string_view>
#include <vector>

#include "../../include/intzip_b200.h"

extern "C" const char* izg_status_string(int32_t s) {
  switch (s) {
    case IZG_OK: return "ok";
    case IZG_E_CHUNK_LENGTH: return "chunk: bad original length";
    case IZG_E_PAYLOAD_SIZE: return "chunk: payload size mismatch";
    case IZG_E_VBYTE_TRUNCATED: return "vbyte: truncated stream";
    case IZG_E_VBYTE_OVERFLOW: return "vbyte: value exceeds 32 bits";
    case IZG_E_VBYTE_TOO_LONG: return "vbyte: integer longer than 5 bytes";
    case IZG_E_BP_TRUNC_DESC: return "simdbp128: truncated descriptor";
    case IZG_E_BP_WIDTH: return "simdbp128: width byte exceeds 32";
    case IZG_E_BP_TRUNC_PAYLOAD: return "simdbp128: truncated payload";
    case IZG_E_FP_TRUNC_PAGE: return "fastpfor: truncated page";
    case IZG_E_FP_BA_OFFSET: return "fastpfor: bad byte-array offset";
    case IZG_E_FP_TRUNC_BA: return "fastpfor: truncated byte array";
    case IZG_E_FP_TRUNC_META: return "fastpfor: truncated block metadata";
    case IZG_E_FP_WIDTHS: return "fastpfor: bad block widths";
    case IZG_E_FP_EMPTY_EXC: return "fastpfor: empty exception list";
    case IZG_E_FP_TRUNC_POS: return "fastpfor: truncated exception positions";
    case IZG_E_FP_POS_RANGE: return "fastpfor: exception position out of range";
    case IZG_E_FP_BA_LEN: return "fastpfor: byte array length mismatch";
    case IZG_E_FP_NO_BITSET: return "fastpfor: missing exception bitset";
    case IZG_E_FP_TRUNC_EXC: return "fastpfor: truncated exception array";
    case IZG_E_FP_OVERRUN: return "fastpfor: packed blocks overrun byte array";
    case IZG_E_FP_EXHAUSTED: return "fastpfor: exception array exhausted";
    case IZG_E_FP_PACKED_SIZE: return "fastpfor: packed area size mismatch";
    case IZG_E_CT_TRUNCATED: return "container: truncated";
    case IZG_E_CT_MAGIC: return "container: bad magic";
    case IZG_E_CT_NAME_LENGTH: return "container: bad codec name length";
    case IZG_E_CT_FOUND_RAW: return "container: expected encoded data, found RAW";
    case IZG_E_CT_TRUNC_PAYLOAD: return "container: truncated payload";
    case IZG_E_CT_TRUNC_RECORD: return "container: truncated chunk record";
    case IZG_E_CT_CHUNK_LENGTH: return "container: bad chunk length";
    case IZG_E_CT_CHUNK_WORDS: return "container: bad chunk word count";
    case IZG_E_CT_ARRAY_LENGTH: return "container: array length mismatch";
    case IZG_E_CT_NOT_RAW: return "container: expected RAW data, found codec";
    case IZG_E_CT_RAW_COUNT: return "container: RAW word count mismatch";
    case IZG_E_BP32_TRUNC_DESC: return "bp32: truncated descriptor";
    case IZG_E_BP32_WIDTH: return "bp32: width byte exceeds 32";
    case IZG_E_BP32_TRUNC_PAYLOAD: return "bp32: truncated payload";
    case IZG_E_S8_EXHAUSTED: return "simple8b: stream exhausted before count";
    case IZG_E_SPLIT_STALL: return "internal: split decode look-back stalled";
    case IZG_E_COUNT_MULTIPLE: return "count must be a multiple of 128";
    case IZG_E_PAGE_TOO_LARGE: return "patched codec: page exceeds 65536 integers";
    case IZG_E_DECREASING: return "delta encode: input is not nondecreasing";
    default: return "unknown status";
  }
}

// make_codec (codec.cpp:99-109) for the codecs with a device decoder;
// "-d2"/"-dm" are the D2/DM extensions (not in the reference registry).
extern "C" int izg_parse_codec_name(const char* name, int* codec, int* delta) {
  if (!name || !codec || !delta) return IZG_ERR_INVALID_ARGUMENT;
  std::string_view s(name);
  int d = IZG_DELTA_D1;
  auto strip = [&](std::string_view suf, int mode) {
    if (s.size() >= suf.size() && s.substr(s.size() - suf.size()) == suf) {
      s.remove_suffix(suf.size());
      d = mode;
      return true;
    }
    return false;
  };
  strip("-s4", IZG_DELTA_D4) || strip("-d2", IZG_DELTA_D2) || strip("-dm", IZG_DELTA_DM);
  if (s == "simdbp128")
    *codec = IZG_SIMDBP128;
  else if (s == "simdfastpfor")
    *codec = IZG_SIMDFASTPFOR;
  else if (s == "bp32")
    *codec = IZG_BP32;
  else if (s == "fastpfor")
    *codec = IZG_FASTPFOR;
  else if (s == "simplepfor")
    *codec = IZG_SIMPLEPFOR;
  else
    return IZG_ERR_UNKNOWN_CODEC;
  *delta = d;
  return IZG_SUCCESS;
}

extern "C" uint64_t izg_layout_chunks(int codec, const uint32_t* n_words, uint32_t n_chunks,
                                      uint64_t* word_off_out) {
  // SIMD-BP128 payload word 0 on a 16-byte boundary (codec_binpack.h:17-23);
  // SIMD-FastPFOR page word 0 at 12 mod 16 so packed rows (word 1 + 4k,
  // codec_patched.cpp:225,250-253) are 16-byte aligned.  The scalar-group
  // codecs read words and take any placement (16-byte aligned here).
  const uint64_t phase = codec == IZG_SIMDFASTPFOR ? 3 : 0;
  uint64_t pos = 0;
  for (uint32_t i = 0; i < n_chunks; ++i) {
    pos = (pos + 3 - phase) / 4 * 4 + phase;
    if (pos < phase) pos = phase;
    word_off_out[i] = pos;
    pos += n_words[i];
  }
  return (pos + 3) / 4 * 4 + 4;  // whole 16-byte rows plus one spare row
}

// ---- synchronous host-buffer decode -----------------------------------

namespace {

constexpr int kSlots = 4;

struct Slot {
  cudaStream_t stream = nullptr;
  uint32_t* words = nullptr;
  uint64_t words_cap = 0;
  izg_chunk* table = nullptr;
  uint32_t table_cap = 0;
  uint32_t* out = nullptr;
  uint64_t out_cap = 0;
  int32_t* status = nullptr;
  uint64_t status_cap = 0;
  uint8_t* ws = nullptr;  // izg_decode_ws workspace (SIMD-FastPFOR index pass)
  uint64_t ws_cap = 0;
  cudaEvent_t decoded = nullptr;   // piece decoded: its D2H may start
  cudaEvent_t drained[6] = {};     // piece's D2H parts done: the slot may be reused
};

struct Scratch {
  int device = -1;
  Slot slot[kSlots];
  // device->host copies: each piece's output goes out as kParts concurrent
  // copies on kParts streams (several copies in flight keep D2H, the
  // pipeline's bottleneck, at ~56 GB/s instead of ~50 for one stream)
  static constexpr int kMaxParts = 6;
  int kParts = 3;  // IZG_HOST_PARTS=1..6 (tuning knob)
  cudaStream_t d2h[kMaxParts] = {};
  // pinned staging for the chunk table and the statuses, so every copy of
  // the pipeline is truly asynchronous (pageable copies block the host)
  izg_chunk* pin_table = nullptr;
  int32_t* pin_status = nullptr;
  uint64_t pin_cap = 0;
  void release() {
    if (pin_table) cudaFreeHost(pin_table);
    if (pin_status) cudaFreeHost(pin_status);
    pin_table = nullptr;
    pin_status = nullptr;
    pin_cap = 0;
    for (auto& s : slot) {
      if (s.words) cudaFree(s.words);
      if (s.table) cudaFree(s.table);
      if (s.out) cudaFree(s.out);
      if (s.status) cudaFree(s.status);
      if (s.ws) cudaFree(s.ws);
      if (s.decoded) cudaEventDestroy(s.decoded);
      for (auto& e : s.drained)
        if (e) cudaEventDestroy(e);
      if (s.stream) cudaStreamDestroy(s.stream);
      s = Slot{};
    }
    for (auto& d : d2h)
      if (d) cudaStreamDestroy(d);
    for (auto& d : d2h) d = nullptr;
    device = -1;
  }
  ~Scratch() { release(); }
};

thread_local Scratch t_scratch;

template <class T>
bool grow(T*& p, uint64_t& cap, uint64_t need) {
  if (need <= cap) return true;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  const uint64_t n = std::max<uint64_t>(need, 1024);
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return false;
  cap = n;
  return true;
}

}  // namespace

extern "C" void izg_release_host_scratch(void) { t_scratch.release(); }

// Pipelined over pieces of the chunk table: H2D and decode of each piece on
// one of four slot streams, every D2H on one stream in piece order (event
// ordered), so the host->device copy of piece k+1, the decode of piece k and
// the device->host copy of piece k-1 overlap on separate copy engines.  Chunks must be ordered
// by word_off and out_off (as encode_array / izg_layout_chunks produce);
// otherwise the whole batch is one piece.
extern "C" int izg_decode_host(int codec, int delta, const uint32_t* h_words, uint64_t n_words,
                               const izg_chunk* h_chunks, uint32_t n_chunks, uint32_t* h_out,
                               uint64_t n_out, int32_t* h_status) {
  if (n_chunks == 0) return IZG_SUCCESS;
  if (!h_words || !h_chunks || !h_out) return IZG_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return IZG_ERR_NO_DEVICE;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  Scratch& S = t_scratch;
  if (S.device != dev) {
    S.release();
    S.device = dev;
    for (auto& s : S.slot)
      if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.decoded, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.drained[0], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.drained[1], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.drained[2], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.drained[3], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.drained[4], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s.drained[5], cudaEventDisableTiming) != cudaSuccess)
        return IZG_ERR_CUDA;
    if (const char* e = std::getenv("IZG_HOST_PARTS")) {
      const int v = std::atoi(e);
      if (v >= 1 && v <= Scratch::kMaxParts) S.kParts = v;
    }
    for (auto& d : S.d2h)
      if (cudaStreamCreateWithFlags(&d, cudaStreamNonBlocking) != cudaSuccess) return IZG_ERR_CUDA;
  }
  // Validate the table against the host buffers (bounds of the copies).
  bool ordered = true;
  for (uint32_t i = 0; i < n_chunks; ++i) {
    const izg_chunk& c = h_chunks[i];
    if (c.word_off + c.n_words > n_words || c.out_off + c.n > n_out)
      return IZG_ERR_INVALID_ARGUMENT;
    if (i && (c.word_off < h_chunks[i - 1].word_off || c.out_off < h_chunks[i - 1].out_off))
      ordered = false;
  }
  // Pieces of 16..64 Mi integers of output, about an eighth of the batch
  // (enough chunks per launch to fill the GPU, enough pieces to overlap the
  // H2D, decode and D2H stages; B200 + PCIe Gen5, 2^30-integer batches:
  // 16 Mi pieces 51.0 GB/s D2H, 64 Mi 52.3, against 52.4 for one bare copy).
  std::vector<uint32_t> cuts{0};
  static const uint64_t forced_piece = [] {
    const char* e = std::getenv("IZG_HOST_PIECE_MI");  // tuning knob (integers, in Mi)
    const long v = e ? std::atol(e) : 0;
    return (uint64_t)(v > 0 ? v : 0) << 20;
  }();
  uint64_t total_ints = 0;
  for (uint32_t i = 0; i < n_chunks; ++i) total_ints += h_chunks[i].n;
  const uint64_t piece_ints =
      forced_piece ? forced_piece
                   : std::max<uint64_t>(16ull << 20, std::min<uint64_t>(64ull << 20, total_ints / 8));
  // (and at most 2^20 chunks, so batches of tiny chunks still pipeline)
  if (ordered) {
    uint64_t acc = 0;
    for (uint32_t i = 0; i < n_chunks; ++i) {
      acc += h_chunks[i].n;
      if ((acc >= piece_ints || i + 1 - cuts.back() >= (1u << 20)) && i + 1 < n_chunks) {
        cuts.push_back(i + 1);
        acc = 0;
      }
    }
  }
  cuts.push_back(n_chunks);
  if (S.pin_cap < n_chunks) {
    if (S.pin_table) cudaFreeHost(S.pin_table);
    if (S.pin_status) cudaFreeHost(S.pin_status);
    S.pin_table = nullptr;
    S.pin_status = nullptr;
    S.pin_cap = 0;
    if (cudaHostAlloc(&S.pin_table, sizeof(izg_chunk) * n_chunks, cudaHostAllocDefault) !=
            cudaSuccess ||
        cudaHostAlloc(&S.pin_status, sizeof(int32_t) * n_chunks, cudaHostAllocDefault) !=
            cudaSuccess)
      return IZG_ERR_CUDA;
    S.pin_cap = n_chunks;
  }
  std::memcpy(S.pin_table, h_chunks, sizeof(izg_chunk) * n_chunks);
  int32_t* st_host = S.pin_status;
  int rc = IZG_SUCCESS;
  std::vector<std::pair<uint64_t, uint64_t>> runs;  // output ranges to copy back
  for (size_t p = 0; p + 1 < cuts.size() && rc == IZG_SUCCESS; ++p) {
    Slot& s = S.slot[p % kSlots];
    const uint32_t c0 = cuts[p], c1 = cuts[p + 1], nc = c1 - c0;
    uint64_t wlo = UINT64_MAX, whi = 0, olo = UINT64_MAX, ohi = 0;
    for (uint32_t i = c0; i < c1; ++i) {
      wlo = std::min(wlo, h_chunks[i].word_off);
      whi = std::max(whi, h_chunks[i].word_off + h_chunks[i].n_words);
      olo = std::min(olo, h_chunks[i].out_off);
      ohi = std::max(ohi, h_chunks[i].out_off + h_chunks[i].n);
    }
    wlo &= ~uint64_t{3};                              // keep 16-byte alignment
    const uint64_t wcopy = std::min<uint64_t>(n_words, (whi + 3) & ~uint64_t{3}) - wlo;
    const uint64_t wneed = ((whi + 3) & ~uint64_t{3}) - wlo + 4;  // + the contract's pad row
    uint64_t tcap = s.table_cap;
    // SIMD-BP128 pieces never take the relay kernel here: it pays for chunks of tens of
    // thousands of integers at 2,432+ chunks per launch, and a piece (at most 64 Mi
    // integers) with that many chunks holds short ones, where it costs 5-15 %
    // (tools/relay_short.py).  Small pieces keep the split kernel's workspace.
    const uint64_t wsb =
        codec == IZG_SIMDBP128 && nc >= 2432 ? 0 : izg_decode_workspace_size(codec, nc);
    if (!grow(s.words, s.words_cap, wneed) || !grow(s.table, tcap, nc) ||
        !grow(s.out, s.out_cap, std::max<uint64_t>(ohi - olo, 1)) ||
        (wsb && !grow(s.ws, s.ws_cap, wsb))) {
      rc = IZG_ERR_CUDA;
      break;
    }
    s.table_cap = (uint32_t)tcap;
    if (!grow(s.status, s.status_cap, nc)) {
      rc = IZG_ERR_CUDA;
      break;
    }
    // The piece's table, rebased onto the slot's buffers (word wlo and
    // output olo become offset 0).
    for (uint32_t i = c0; i < c1; ++i) {
      S.pin_table[i].word_off -= wlo;
      S.pin_table[i].out_off -= olo;
    }
    for (auto& e : s.drained) cudaStreamWaitEvent(s.stream, e, 0);  // previous D2H done
    cudaMemsetAsync(s.words + wcopy, 0, (wneed - wcopy) * 4, s.stream);
    cudaMemcpyAsync(s.words, h_words + wlo, wcopy * 4, cudaMemcpyHostToDevice, s.stream);
    cudaMemcpyAsync(s.table, S.pin_table + c0, sizeof(izg_chunk) * nc, cudaMemcpyHostToDevice,
                    s.stream);
    const int r = izg_decode_ws(codec, delta, s.words, s.table, nc, s.out, s.status, nullptr,
                                s.ws, wsb, s.stream);
    if (r != IZG_SUCCESS) {
      rc = r;
      break;
    }
    cudaEventRecord(s.decoded, s.stream);
    // Copy back only what the chunks decoded: the output ranges of the
    // piece, merged where they touch.  Gaps between chunks in h_out keep the
    // caller's contents (the device buffer holds no data for them).
    runs.clear();
    for (uint32_t i = c0; i < c1; ++i)
      if (h_chunks[i].n) runs.push_back({h_chunks[i].out_off - olo, h_chunks[i].n});
    if (!ordered) std::sort(runs.begin(), runs.end());
    size_t m = 0;
    for (size_t i = 0; i < runs.size(); ++i) {
      if (m && runs[i].first <= runs[m - 1].first + runs[m - 1].second) {
        const uint64_t e = std::max(runs[m - 1].first + runs[m - 1].second,
                                    runs[i].first + runs[i].second);
        runs[m - 1].second = e - runs[m - 1].first;
      } else {
        runs[m++] = runs[i];
      }
    }
    runs.resize(m);
    if (runs.size() == 1) {  // contiguous: kParts concurrent copies keep D2H at ~56 GB/s
      const uint64_t r0 = runs[0].first, nout = runs[0].second;
      static const uint64_t sub = [] {  // IZG_HOST_SUB_MI: copies of this many Mi integers
        const char* e = std::getenv("IZG_HOST_SUB_MI");
        const long v = e ? std::atol(e) : 0;
        return (uint64_t)(v > 0 ? v : 0) << 20;
      }();
      const uint64_t part =
          sub ? sub : std::max<uint64_t>(1024, (nout / S.kParts + 1023) & ~uint64_t{1023});
      runs.clear();
      for (uint64_t a = 0; a < nout; a += part)
        runs.push_back({r0 + a, std::min<uint64_t>(part, nout - a)});
      if (!sub && runs.size() > (size_t)S.kParts) {  // rounding left a sliver: fold it in
        runs[S.kParts - 1].second += runs.back().second;
        runs.pop_back();
      }
    }
    for (int k = 0; k < S.kParts; ++k) cudaStreamWaitEvent(S.d2h[k], s.decoded, 0);
    for (size_t i = 0; i < runs.size(); ++i)
      cudaMemcpyAsync(h_out + olo + runs[i].first, s.out + runs[i].first, runs[i].second * 4,
                      cudaMemcpyDeviceToHost, S.d2h[i % S.kParts]);
    cudaMemcpyAsync(st_host + c0, s.status, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost,
                    S.d2h[0]);
    for (int k = 0; k < S.kParts; ++k) cudaEventRecord(s.drained[k], S.d2h[k]);
  }
  for (auto& s : S.slot)
    if (cudaStreamSynchronize(s.stream) != cudaSuccess) rc = IZG_ERR_CUDA;
  for (auto& d : S.d2h)
    if (cudaStreamSynchronize(d) != cudaSuccess) rc = IZG_ERR_CUDA;
  if (rc != IZG_SUCCESS) return rc;
  if (h_status) std::memcpy(h_status, st_host, sizeof(int32_t) * n_chunks);
  for (uint32_t i = 0; i < n_chunks; ++i)
    if (st_host[i] != IZG_OK) return IZG_ERR_CORRUPT;
  return IZG_SUCCESS;
}
