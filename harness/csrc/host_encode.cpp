// host_encode.cpp — host encoder for the hot-path codecs (bench/test
// HARNESS, libizh.so; not in the product library): produces device inputs
// for bench.py and the tests, word-for-word equal to the reference encoder.
//
// Restates, word-level and multithreaded over chunks:
//   encode_array                      codec.cpp:14-37
//   delta_encode_scalar / _stride4    delta.cpp:18-23, 53-58 (+ D2/DM ext)
//   SimdBp128Codec::encode_deltas     codec_binpack.cpp:70-92
//   FastPforCodec::encode_deltas      codec_patched.cpp:219-290 (vertical)
//   fastpfor_choose_width             codec_patched.cpp:15-48
//   vbyte_encode                      codec_basic.cpp:16-25
// Output words are bit-identical to the reference (tests/test_host_encode.py
// checks them against the reference compiled from source).
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "izh.h"

namespace izh {
namespace {

inline uint32_t bit_width(uint32_t v) { return v ? 32u - (uint32_t)__builtin_clz(v) : 0u; }
inline uint32_t mask_of(uint32_t b) { return b >= 32 ? 0xFFFFFFFFu : (1u << b) - 1u; }

// pack_vertical128_masked (bitpack.cpp:87-120,318-322): lane j holds values
// j, j+4, ...; lane word i is stream word 4i+j.  `out` gets 4b words.
void pack_vertical(const uint32_t* v, uint32_t b, uint32_t* out) {
  if (b == 0) return;
  std::memset(out, 0, sizeof(uint32_t) * 4 * b);
  const uint32_t m = mask_of(b);
  for (uint32_t s = 0; s < 32; ++s) {
    const uint32_t bit = s * b, w = bit >> 5, sh = bit & 31;
    for (uint32_t j = 0; j < 4; ++j) {
      const uint32_t x = v[4 * s + j] & m;
      out[4 * w + j] |= x << sh;
      if (sh + b > 32) out[4 * (w + 1) + j] |= x >> (32 - sh);
    }
  }
}

bool delta_encode(int delta, uint32_t* v, size_t n, bool wrap) {
  size_t i;
  switch (delta) {
    case IZG_DELTA_D1:
      for (i = n; i-- > 1;) {
        if (!wrap && v[i] < v[i - 1]) return false;
        v[i] -= v[i - 1];
      }
      return true;
    case IZG_DELTA_D4:
      for (i = n; i-- > 4;) {
        if (!wrap && v[i] < v[i - 4]) return false;
        v[i] -= v[i - 4];
      }
      return true;
    case IZG_DELTA_D2:
      for (i = n; i-- > 2;) {
        if (!wrap && v[i] < v[i - 2]) return false;
        v[i] -= v[i - 2];
      }
      return true;
    case IZG_DELTA_DM:
      for (size_t k = (n + 3) / 4; k-- > 1;) {
        const uint32_t base = v[4 * k - 1];
        const size_t end = std::min(n, 4 * k + 4);
        for (i = 4 * k; i < end; ++i) {
          if (!wrap && v[i] < base) return false;
          v[i] -= base;
        }
      }
      return true;
    default:
      return true;
  }
}

void bp128_encode(const uint32_t* d, size_t count, std::vector<uint32_t>& out) {
  for (size_t base = 0; base < count; base += 2048) {
    const size_t groups = std::min<size_t>(16, (count - base) / 128);
    uint8_t widths[16] = {0};
    for (size_t g = 0; g < groups; ++g) {
      uint32_t acc = 0;
      const uint32_t* blk = d + base + 128 * g;
      for (int i = 0; i < 128; ++i) acc |= blk[i];
      widths[g] = (uint8_t)bit_width(acc);
    }
    for (int w = 0; w < 4; ++w)
      out.push_back((uint32_t)widths[4 * w] | (uint32_t)widths[4 * w + 1] << 8 |
                    (uint32_t)widths[4 * w + 2] << 16 | (uint32_t)widths[4 * w + 3] << 24);
    for (size_t g = 0; g < groups; ++g) {
      const size_t old = out.size();
      out.resize(old + 4 * (size_t)widths[g]);
      pack_vertical(d + base + 128 * g, widths[g], out.data() + old);
    }
  }
}

struct WidthChoice {
  uint32_t b, maxbits;
};

// fastpfor_cost_bits / fastpfor_choose_width (codec_patched.cpp:21-48).
WidthChoice choose_width(const uint32_t* h, uint32_t block_len) {
  uint32_t maxbits = 0;
  for (uint32_t w = 0; w <= 32; ++w)
    if (h[w]) maxbits = w;
  uint32_t best_b = 0;
  uint64_t best = ~uint64_t{0};
  uint64_t above = 0;  // values wider than b, for b = maxbits downward
  // cost(b) = b*len + (8 + maxbits - b) * c(b) when c(b) > 0; evaluate every
  // b in 0..maxbits and keep the last minimum (ties toward larger b).
  std::array<uint64_t, 34> c{};
  for (int b = 32; b >= 0; --b) {
    c[b] = above;
    above += h[b];
  }
  for (uint32_t b = 0; b <= maxbits; ++b) {
    uint64_t cost = (uint64_t)b * block_len;
    if (c[b] > 0) cost += (uint64_t)(8 + maxbits - b) * c[b];
    if (cost <= best) {
      best = cost;
      best_b = b;
    }
  }
  return {best_b, maxbits};
}

void fastpfor_encode(const uint32_t* d, size_t count, std::vector<uint32_t>& out) {
  if (count == 0) return;
  const size_t page = out.size();
  out.push_back(0);
  std::vector<uint8_t> ba;
  ba.reserve(count / 128 * 8);
  std::array<std::vector<uint32_t>, 33> arrays;
  for (size_t base = 0; base < count; base += 128) {
    const uint32_t* v = d + base;
    uint32_t h[33] = {0};
    for (int i = 0; i < 128; ++i) ++h[bit_width(v[i])];
    const WidthChoice wc = choose_width(h, 128);
    ba.push_back((uint8_t)wc.b);
    ba.push_back((uint8_t)wc.maxbits);
    if (wc.maxbits > wc.b) {
      const size_t cpos = ba.size();
      ba.push_back(0);
      uint32_t c = 0;
      auto& arr = arrays[wc.maxbits - wc.b];
      for (uint32_t i = 0; i < 128; ++i)
        if (v[i] >> wc.b) {
          ba.push_back((uint8_t)i);
          arr.push_back(v[i] >> wc.b);
          ++c;
        }
      ba[cpos] = (uint8_t)c;
    }
    const size_t old = out.size();
    out.resize(old + 4 * (size_t)wc.b);
    pack_vertical(v, wc.b, out.data() + old);
  }
  out[page] = (uint32_t)(out.size() - page);
  out.push_back((uint32_t)ba.size());
  {
    const size_t nw = (ba.size() + 3) / 4, old = out.size();
    out.resize(old + nw, 0);
    std::memcpy(out.data() + old, ba.data(), ba.size());
  }
  uint32_t bitset = 0;
  for (uint32_t w = 1; w <= 32; ++w)
    if (!arrays[w].empty()) bitset |= 1u << (w - 1);
  out.push_back(bitset);
  for (uint32_t w = 1; w <= 32; ++w) {
    auto& vals = arrays[w];
    if (vals.empty()) continue;
    out.push_back((uint32_t)vals.size());
    while ((out.size() - page) % 4 != 0) out.push_back(0);
    vals.resize((vals.size() + 127) / 128 * 128, 0);
    const size_t old = out.size();
    out.resize(old + vals.size() / 128 * 4 * w);
    for (size_t g = 0; g < vals.size() / 128; ++g)
      pack_vertical(vals.data() + 128 * g, w, out.data() + old + g * 4 * w);
  }
}

void vbyte_append(const uint32_t* v, size_t n, std::vector<uint32_t>& out) {
  std::vector<uint8_t> b;
  for (size_t i = 0; i < n; ++i) {
    uint32_t x = v[i];
    while (x >= 128) {
      b.push_back((uint8_t)(x & 0x7F));
      x >>= 7;
    }
    b.push_back((uint8_t)(x | 0x80));
  }
  const size_t nw = (b.size() + 3) / 4, old = out.size();
  out.resize(old + nw, 0);
  std::memcpy(out.data() + old, b.data(), b.size());
}

}  // namespace

// Placement of izg_layout_chunks (include/intzip_b200.h): SIMD-BP128
// payloads start on a 16-byte boundary, SIMD-FastPFOR pages at 12 mod 16 so
// that their packed rows (word 1 + 4k) are 16-byte aligned; returns the
// buffer size in words (whole 16-byte rows plus one spare row).
uint64_t place(int codec, const uint32_t* n_words, uint32_t n_chunks, uint64_t* off) {
  const uint64_t phase = codec == IZG_SIMDFASTPFOR ? 3 : 0;
  uint64_t pos = phase;
  for (uint32_t i = 0; i < n_chunks; ++i) {
    pos += (phase - pos) & 3;  // next word at `phase` mod 4
    off[i] = pos;
    pos += n_words[i];
  }
  return (pos + 3) / 4 * 4 + 4;
}

// One chunk of encode_array; returns false on a decreasing input (no wrap).
bool encode_chunk(int codec, int delta, const uint32_t* values, uint32_t n, bool wrap,
                  std::vector<uint32_t>& scratch, std::vector<uint32_t>& out) {
  scratch.assign(values, values + n);
  if (delta != IZG_DELTA_NONE && !delta_encode(delta, scratch.data(), n, wrap)) return false;
  const size_t core = delta == IZG_DELTA_NONE ? n : (size_t)n / 128 * 128;
  if (codec == IZG_SIMDBP128)
    bp128_encode(scratch.data(), core, out);
  else
    fastpfor_encode(scratch.data(), core, out);
  if (core < n) vbyte_append(scratch.data() + core, n - core, out);
  return true;
}

}  // namespace izh

// ---- C ABI -----------------------------------------------------------------

struct izh_encoded {
  std::vector<std::vector<uint32_t>> payloads;
  std::vector<izg_chunk> table;
  std::vector<uint64_t> offs;
  uint64_t total_words = 0;
  int codec = 0;
};

extern "C" izh_encoded* izh_encode_batch(int codec, int delta, const uint32_t* values,
                                              const uint64_t* value_off, const uint32_t* counts,
                                              uint32_t n_chunks, int allow_wrap, int threads,
                                              int* status) {
  *status = IZG_SUCCESS;
  if ((codec != IZG_SIMDBP128 && codec != IZG_SIMDFASTPFOR) || delta < 0 || delta > 4) {
    *status = IZG_ERR_INVALID_ARGUMENT;
    return nullptr;
  }
  for (uint32_t i = 0; i < n_chunks; ++i) {
    const bool bad = delta == IZG_DELTA_NONE
                         ? (counts[i] % 128 != 0 ||
                            (codec == IZG_SIMDFASTPFOR && counts[i] > IZG_CHUNK_SIZE))
                         : (counts[i] == 0 || counts[i] > IZG_CHUNK_SIZE);
    if (bad) {
      *status = IZG_ERR_INVALID_ARGUMENT;
      return nullptr;
    }
  }
  auto* e = new izh_encoded;
  e->codec = codec;
  e->payloads.resize(n_chunks);
  std::vector<int> bad(std::max(threads, 1), 0);
  auto work = [&](int t, uint32_t lo, uint32_t hi) {
    std::vector<uint32_t> scratch;
    for (uint32_t i = lo; i < hi; ++i) {
      auto& out = e->payloads[i];
      out.reserve(counts[i] / 2 + 64);
      if (!izh::encode_chunk(codec, delta, values + value_off[i], counts[i], allow_wrap != 0,
                             scratch, out))
        bad[t] = 1;
    }
  };
  threads = std::max(1, std::min<int>(threads, (int)std::max<uint32_t>(n_chunks, 1)));
  if (threads == 1) {
    work(0, 0, n_chunks);
  } else {
    std::vector<std::thread> pool;
    const uint32_t per = (n_chunks + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const uint32_t lo = std::min<uint32_t>(n_chunks, per * t);
      const uint32_t hi = std::min<uint32_t>(n_chunks, per * (t + 1));
      pool.emplace_back(work, t, lo, hi);
    }
    for (auto& th : pool) th.join();
  }
  for (int b : bad)
    if (b) {
      delete e;
      *status = IZG_ERR_INVALID_ARGUMENT;  // decreasing input (delta.cpp:13)
      return nullptr;
    }
  std::vector<uint32_t> sizes(n_chunks);
  for (uint32_t i = 0; i < n_chunks; ++i) sizes[i] = (uint32_t)e->payloads[i].size();
  e->offs.resize(n_chunks);
  e->total_words = izh::place(codec, sizes.data(), n_chunks, e->offs.data());
  e->table.resize(n_chunks);
  for (uint32_t i = 0; i < n_chunks; ++i)
    e->table[i] = izg_chunk{e->offs[i], sizes[i], counts[i], value_off[i]};
  return e;
}

extern "C" uint64_t izh_encoded_words(const izh_encoded* e) { return e ? e->total_words : 0; }

extern "C" int izh_encoded_copy(const izh_encoded* e, uint32_t* words, izg_chunk* table,
                                int threads) {
  if (!e) return IZG_ERR_INVALID_ARGUMENT;
  const uint32_t n = (uint32_t)e->payloads.size();
  if (table) std::memcpy(table, e->table.data(), sizeof(izg_chunk) * n);
  if (words) {
    auto work = [&](uint32_t lo, uint32_t hi) {
      for (uint32_t i = lo; i < hi; ++i) {
        const uint64_t start = i ? e->offs[i - 1] + e->payloads[i - 1].size() : 0;
        std::memset(words + start, 0, (e->offs[i] - start) * 4);  // alignment pad
        std::memcpy(words + e->offs[i], e->payloads[i].data(), e->payloads[i].size() * 4);
      }
      if (hi == n && n) {
        const uint64_t end = e->offs[n - 1] + e->payloads[n - 1].size();
        std::memset(words + end, 0, (e->total_words - end) * 4);
      }
    };
    threads = std::max(1, std::min<int>(threads, (int)std::max<uint32_t>(n, 1)));
    std::vector<std::thread> pool;
    const uint32_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const uint32_t lo = std::min<uint32_t>(n, per * t), hi = std::min<uint32_t>(n, per * (t + 1));
      if (lo < hi) pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
    if (n == 0) std::memset(words, 0, e->total_words * 4);
  }
  return IZG_SUCCESS;
}

extern "C" void izh_encoded_free(izh_encoded* e) { delete e; }
