// ref_shim.cpp — C entry points over the REFERENCE library compiled from its
// own sources (/root/reference/proj/core/src, see oracle/Makefile), so tests
// and bench.py's reference arm can call it through ctypes.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Nothing in the product links this.
// All the algorithmic work happens inside the unmodified reference functions
// (intzip::encode_array, decode_array, Codec::encode_deltas/decode_deltas,
// unpack_vertical128, ...); this file only marshals buffers and catches the
// reference's exceptions into return codes:
//   0 = ok, 1 = intzip::CorruptError, 2 = std::invalid_argument, 3 = other.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "intzip/bitpack.h"
#include "intzip/codec.h"
#include "intzip/codec_basic.h"
#include "intzip/codec_patched.h"
#include "intzip/container.h"
#include "intzip/datagen.h"
#include "intzip/delta.h"
#include "intzip/errors.h"
#include "intzip/wordbytes.h"

namespace {

struct ChunkRec {  // same layout as izg_chunk (include/intzip_b200.h)
  uint64_t word_off;
  uint32_t n_words;
  uint32_t n;
  uint64_t out_off;
};

void set_err(char* err, int cap, const char* what) {
  if (err && cap > 0) {
    std::strncpy(err, what, static_cast<size_t>(cap) - 1);
    err[cap - 1] = 0;
  }
}

template <class F>
int guarded(char* err, int cap, F&& f) {
  try {
    f();
    set_err(err, cap, "");
    return 0;
  } catch (const intzip::CorruptError& e) {
    set_err(err, cap, e.what());
    return 1;
  } catch (const std::invalid_argument& e) {
    set_err(err, cap, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_err(err, cap, e.what());
    return 3;
  }
}

}  // namespace

extern "C" {

int izr_codec_names(char* out, int cap) {
  std::string all;
  for (const auto& n : intzip::codec_names()) all += n + ",";
  set_err(out, cap, all.c_str());
  return 0;
}

// encode_array over `n` values (codec.cpp:14-37).  Payloads are written
// back to back from words[0]; the chunk table receives offsets.
int izr_encode_array(const char* name, const uint32_t* values, uint64_t n,
                     uint32_t* words, uint64_t words_cap, ChunkRec* chunks,
                     uint32_t chunks_cap, uint64_t* n_words, uint32_t* n_chunks,
                     char* err, int errcap) {
  return guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    const auto cs = intzip::encode_array(*codec, {values, n});
    uint64_t pos = 0, out = 0;
    if (cs.size() > chunks_cap) throw std::runtime_error("chunk table too small");
    for (size_t i = 0; i < cs.size(); ++i) {
      if (pos + cs[i].payload.size() > words_cap)
        throw std::runtime_error("word buffer too small");
      std::memcpy(words + pos, cs[i].payload.data(), cs[i].payload.size() * 4);
      chunks[i] = {pos, static_cast<uint32_t>(cs[i].payload.size()),
                   cs[i].original_length, out};
      pos += cs[i].payload.size();
      out += cs[i].original_length;
    }
    *n_words = pos;
    *n_chunks = static_cast<uint32_t>(cs.size());
  });
}

// As encode_array for ONE chunk, but with differences taken mod 2^32 instead
// of delta_encode's monotonicity check (delta.cpp:13).  Used for the config-4
// inputs whose prefix sums wrap; decode_array accepts the
// result because its prefix sums wrap too.  The core and remainder coding are
// the reference's Codec::encode_deltas and vbyte_encode.
int izr_encode_chunk_wrapping(const char* name, const uint32_t* values,
                              uint32_t n, uint32_t* words, uint64_t words_cap,
                              uint64_t* n_words, char* err, int errcap) {
  return guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    if (n == 0 || n > intzip::kChunkSize) throw std::invalid_argument("bad n");
    std::vector<uint32_t> d(values, values + n);
    const size_t stride = codec->delta_mode() == intzip::DeltaMode::stride4 ? 4 : 1;
    for (size_t i = d.size(); i-- > stride;) d[i] -= d[i - stride];
    const size_t core = n / codec->block_multiple() * codec->block_multiple();
    std::vector<uint32_t> payload;
    codec->encode_deltas(d.data(), core, payload);
    if (core < n) {
      std::vector<uint8_t> rem;
      intzip::vbyte_encode({d.data() + core, n - core}, rem);
      intzip::append_bytes_as_words(rem, payload);
    }
    if (payload.size() > words_cap) throw std::runtime_error("word buffer too small");
    std::memcpy(words, payload.data(), payload.size() * 4);
    *n_words = payload.size();
  });
}

// decode_array (codec.cpp:39-69) over a chunk table; output placed at
// out_off of each chunk (the reference writes chunks back to back, which is
// what the table describes for a single array).
int izr_decode_array(const char* name, const uint32_t* words,
                     const ChunkRec* table, uint32_t n_chunks, uint32_t* out,
                     uint64_t out_cap, char* err, int errcap) {
  return guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    std::vector<intzip::Chunk> cs(n_chunks);
    for (uint32_t i = 0; i < n_chunks; ++i) {
      cs[i].original_length = table[i].n;
      cs[i].payload.assign(words + table[i].word_off,
                           words + table[i].word_off + table[i].n_words);
    }
    std::vector<uint32_t> res;
    intzip::decode_array(*codec, cs, res);
    if (res.size() > out_cap) throw std::runtime_error("output buffer too small");
    std::memcpy(out, res.data(), res.size() * 4);
  });
}

int izr_encode_deltas(const char* name, const uint32_t* deltas, uint64_t count,
                      uint32_t* words, uint64_t words_cap, uint64_t* n_words,
                      char* err, int errcap) {
  return guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    std::vector<uint32_t> out;
    codec->encode_deltas(deltas, count, out);
    if (out.size() > words_cap) throw std::runtime_error("word buffer too small");
    std::memcpy(words, out.data(), out.size() * 4);
    *n_words = out.size();
  });
}

int izr_decode_deltas(const char* name, const uint32_t* words, uint64_t nwords,
                      uint32_t* out, uint64_t count, uint64_t* consumed,
                      char* err, int errcap) {
  return guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    *consumed = codec->decode_deltas({words, nwords}, out, count);
  });
}

int izr_unpack_vertical128(const uint32_t* words, uint32_t b, uint32_t* out) {
  return guarded(nullptr, 0, [&] { intzip::unpack_vertical128(words, b, out); });
}

int izr_pack_vertical128(const uint32_t* values, uint32_t b, uint32_t* out,
                         int masked) {
  return guarded(nullptr, 0, [&] {
    if (masked)
      intzip::pack_vertical128_masked(values, b, out);
    else
      intzip::pack_vertical128(values, b, out);
  });
}

uint32_t izr_max_bitwidth(const uint32_t* values, uint64_t n) {
  return intzip::max_bitwidth({values, n});
}

int izr_delta(int encode, int stride4, uint32_t* values, uint64_t n) {
  return guarded(nullptr, 0, [&] {
    const auto mode = stride4 ? intzip::DeltaMode::stride4 : intzip::DeltaMode::scalar;
    if (encode)
      intzip::delta_encode(mode, {values, n});
    else
      intzip::delta_decode(mode, {values, n});
  });
}

int izr_vbyte_encode(const uint32_t* values, uint64_t n, uint8_t* out,
                     uint64_t* nbytes) {
  return guarded(nullptr, 0, [&] {
    std::vector<uint8_t> b;
    intzip::vbyte_encode({values, n}, b);
    std::memcpy(out, b.data(), b.size());
    *nbytes = b.size();
  });
}

int izr_vbyte_decode(const uint8_t* bytes, uint64_t nbytes, uint32_t* out,
                     uint64_t count, uint64_t* consumed, char* err, int errcap) {
  return guarded(err, errcap, [&] {
    *consumed = intzip::vbyte_decode({bytes, nbytes}, out, count);
  });
}

int izr_choose_width(const uint32_t* counts33, uint32_t block_len, uint32_t* b,
                     uint32_t* maxbits, uint64_t* cost) {
  intzip::Histogram33 h;
  for (int i = 0; i < 33; ++i) h.counts[i] = counts33[i];
  const auto c = intzip::fastpfor_choose_width(h, block_len);
  *b = c.b;
  *maxbits = c.maxbits;
  *cost = intzip::fastpfor_cost_bits(h, block_len, c.b);
  return 0;
}

// The reference's own generators (datagen.cpp:110-127): model 0 uniform,
// 1 cluster.  Used for cross-checks of compressed sizes only.
int izr_gen(int model, uint64_t n, uint64_t range, uint64_t seed, uint32_t* out) {
  return guarded(nullptr, 0, [&] {
    const auto v = model ? intzip::gen_clusterdata(n, range, seed)
                         : intzip::gen_uniform(n, range, seed);
    std::memcpy(out, v.data(), v.size() * 4);
  });
}

// ---- threaded batch encode with the reference encoder -------------------
//
// Entry i is one array values[value_off[i] .. + counts[i]) encoded by
// intzip::encode_array (codec.cpp:14-37), or — wrap != 0, arrays of at most
// one chunk — by the izr_encode_chunk_wrapping rule above (C4's wrapped
// inputs).  Arrays are encoded on `threads` threads; all the coding work is
// the reference's.
struct Encoded {
  std::vector<std::vector<intzip::Chunk>> arrays;
};

}  // extern "C"

namespace {

std::vector<intzip::Chunk> encode_one(const intzip::Codec& codec, const uint32_t* v, uint32_t n,
                                      bool wrap) {
  if (!wrap) return intzip::encode_array(codec, {v, n});
  if (n == 0 || n > intzip::kChunkSize) throw std::invalid_argument("wrap: bad n");
  std::vector<uint32_t> d(v, v + n);
  const size_t stride = codec.delta_mode() == intzip::DeltaMode::stride4 ? 4 : 1;
  for (size_t i = d.size(); i-- > stride;) d[i] -= d[i - stride];
  const size_t core = n / codec.block_multiple() * codec.block_multiple();
  intzip::Chunk c;
  c.original_length = n;
  codec.encode_deltas(d.data(), core, c.payload);
  if (core < n) {
    std::vector<uint8_t> rem;
    intzip::vbyte_encode({d.data() + core, n - core}, rem);
    intzip::append_bytes_as_words(rem, c.payload);
  }
  return {std::move(c)};
}

template <class F>
void ranges(uint32_t count, int threads, F&& f) {
  threads = std::max(1, std::min<int>(threads, (int)std::max<uint32_t>(count, 1)));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const uint32_t lo = (uint64_t)count * t / threads, hi = (uint64_t)count * (t + 1) / threads;
    if (lo < hi) pool.emplace_back(f, lo, hi);
  }
  for (auto& th : pool) th.join();
}

// First word of every chunk at `phase` mod 4 (phase < 0: back to back).
uint64_t place(const Encoded& e, int phase, ChunkRec* table) {
  uint64_t pos = phase < 0 ? 0 : (uint64_t)phase, out = 0;
  uint32_t k = 0;
  for (const auto& a : e.arrays)
    for (const auto& c : a) {
      if (phase >= 0) pos += ((uint64_t)phase - pos) & 3;
      if (table) table[k] = {pos, (uint32_t)c.payload.size(), c.original_length, out};
      ++k;
      pos += c.payload.size();
      out += c.original_length;
    }
  return (pos + 3) / 4 * 4 + 4;
}

}  // namespace

extern "C" {

void* izr_encode_batch(const char* name, const uint32_t* values, const uint64_t* value_off,
                       const uint32_t* counts, uint32_t n_arrays, int wrap, int threads,
                       char* err, int errcap) {
  auto* e = new Encoded;
  const int rc = guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    e->arrays.resize(n_arrays);
    std::atomic<int> failed{0};
    std::string what;
    std::mutex mu;
    ranges(n_arrays, threads, [&](uint32_t lo, uint32_t hi) {
      for (uint32_t i = lo; i < hi && !failed; ++i) {
        try {
          e->arrays[i] = encode_one(*codec, values + value_off[i], counts[i], wrap != 0);
        } catch (const std::exception& x) {
          std::lock_guard<std::mutex> g(mu);
          if (!failed.exchange(1)) what = x.what();
        }
      }
    });
    if (failed) throw std::invalid_argument(what);
  });
  if (rc) {
    delete e;
    return nullptr;
  }
  return e;
}

// Sizes of the placed words buffer and of the chunk table.
void izr_encoded_size(void* h, int phase, uint64_t* n_words, uint32_t* n_chunks) {
  const auto* e = static_cast<Encoded*>(h);
  uint32_t k = 0;
  for (const auto& a : e->arrays) k += (uint32_t)a.size();
  *n_chunks = k;
  *n_words = place(*e, phase, nullptr);
}

// Copy out the payloads (placed, gaps zero) and the chunk table.
void izr_encoded_copy(void* h, int phase, uint32_t* words, ChunkRec* table) {
  const auto* e = static_cast<Encoded*>(h);
  const uint64_t total = place(*e, phase, table);
  std::memset(words, 0, total * 4);
  uint32_t k = 0;
  for (const auto& a : e->arrays)
    for (const auto& c : a) {
      std::memcpy(words + table[k].word_off, c.payload.data(), c.payload.size() * 4);
      ++k;
    }
}

void izr_encoded_free(void* h) { delete static_cast<Encoded*>(h); }

// ---- timed batch decode: the reference arm / cpu_baseline --------------
//
// A batch holds arrays of intzip::Chunk objects and one output vector per
// array, so a timed pass is exactly `decode_array(codec, chunks_i, out_i)`
// per array (codec.cpp:39-69) into pre-faulted, reused per-array outputs,
// spread over T threads in contiguous ranges (number 1).
struct Batch {
  std::unique_ptr<intzip::Codec> codec;
  std::vector<std::vector<intzip::Chunk>> arrays;
  std::vector<std::vector<uint32_t>> outs;
};

// Each table entry is its own array of one chunk.
void* izr_batch_create(const char* name, const uint32_t* words,
                       const ChunkRec* table, uint32_t n_chunks) {
  auto* b = new Batch;
  b->codec = intzip::make_codec(name);
  b->arrays.resize(n_chunks);
  b->outs.resize(n_chunks);
  for (uint32_t i = 0; i < n_chunks; ++i) {
    b->arrays[i].resize(1);
    b->arrays[i][0].original_length = table[i].n;
    b->arrays[i][0].payload.assign(words + table[i].word_off,
                                   words + table[i].word_off + table[i].n_words);
    b->outs[i].assign(table[i].n, 0u);  // pre-fault
  }
  return b;
}

// Empty batch for `name`; arrays are appended with izr_batch_adopt.
void* izr_batch_new(const char* name) {
  auto* b = new Batch;
  b->codec = intzip::make_codec(name);
  return b;
}

// Move the arrays of an izr_encode_batch result into the batch (the handle
// is consumed) and pre-fault their outputs on `threads` threads.
void izr_batch_adopt(void* handle, void* enc, int threads) {
  auto* b = static_cast<Batch*>(handle);
  auto* e = static_cast<Encoded*>(enc);
  const size_t first = b->arrays.size();
  for (auto& a : e->arrays) b->arrays.push_back(std::move(a));
  b->outs.resize(b->arrays.size());
  delete e;
  ranges((uint32_t)(b->arrays.size() - first), threads, [&](uint32_t lo, uint32_t hi) {
    for (uint32_t i = lo; i < hi; ++i) {
      size_t n = 0;
      for (const auto& c : b->arrays[first + i]) n += c.original_length;
      b->outs[first + i].assign(n, 0u);
    }
  });
}

uint32_t izr_batch_size(void* handle) {
  return (uint32_t) static_cast<Batch*>(handle)->arrays.size();
}

// Compressed payload words of the whole batch.
uint64_t izr_batch_payload_words(void* handle) {
  uint64_t w = 0;
  for (const auto& a : static_cast<Batch*>(handle)->arrays)
    for (const auto& c : a) w += c.payload.size();
  return w;
}

// One pass over `count` arrays starting at `first` on `threads` threads;
// returns wall seconds, or a negative value if any decode threw.
double izr_batch_decode(void* handle, uint32_t first, uint32_t count,
                        int threads) {
  auto* b = static_cast<Batch*>(handle);
  if (first + count > b->arrays.size()) return -2.0;
  std::atomic<int> failed{0};
  auto work = [&](uint32_t lo, uint32_t hi) {
    for (uint32_t i = lo; i < hi; ++i) {
      try {
        intzip::decode_array(*b->codec, b->arrays[i], b->outs[i]);
      } catch (...) {
        failed = 1;
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  if (threads <= 1) {
    work(first, first + count);
  } else {
    std::vector<std::thread> pool;
    const uint32_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const uint32_t lo = first + std::min<uint32_t>(count, per * t);
      const uint32_t hi = first + std::min<uint32_t>(count, per * (t + 1));
      if (lo < hi) pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (failed) return -1.0;
  return std::chrono::duration<double>(t1 - t0).count();
}

// Copy array i's decoded output (after a pass) for verification.
int izr_batch_output(void* handle, uint32_t i, uint32_t* out) {
  auto* b = static_cast<Batch*>(handle);
  std::memcpy(out, b->outs[i].data(), b->outs[i].size() * 4);
  return 0;
}

// Checksum (izh_checksum_host's definition) of arrays [first, first+count)
// decoded back to back, the first integer having global index `base`.
void izr_batch_checksum(void* handle, uint32_t first, uint32_t count, uint64_t base,
                        uint64_t* out) {
  auto* b = static_cast<Batch*>(handle);
  uint64_t s = 0, x = 0, i = base;
  for (uint32_t a = first; a < first + count; ++a)
    for (uint32_t v : b->outs[a]) {
      s += (uint64_t(v) + 1) * (2 * i + 1);
      x ^= v;
      ++i;
    }
  out[0] = s;
  out[1] = x;
}

void izr_batch_free(void* handle) { delete static_cast<Batch*>(handle); }

// ---- container (container.cpp) -------------------------------------------

// container_write_encoded over encode_array of each array (values of array i
// at values[offs[i] .. offs[i] + lens[i])).  *len_out = bytes written (the
// buffer may be null to size it).
int izr_container_write_encoded(const char* name, const uint32_t* values,
                                const uint64_t* offs, const uint32_t* lens,
                                uint32_t n_arrays, uint8_t* buf, uint64_t cap,
                                uint64_t* len_out, char* err, int errcap) {
  return guarded(err, errcap, [&] {
    const auto codec = intzip::make_codec(name);
    std::vector<std::vector<intzip::Chunk>> arrays(n_arrays);
    for (uint32_t i = 0; i < n_arrays; ++i)
      arrays[i] = intzip::encode_array(*codec, {values + offs[i], lens[i]});
    std::ostringstream os;
    intzip::container_write_encoded(os, codec->name(), arrays);
    const std::string s = os.str();
    *len_out = s.size();
    if (buf) {
      if (s.size() > cap) throw std::runtime_error("buffer too small");
      std::memcpy(buf, s.data(), s.size());
    }
  });
}

int izr_container_write_raw(const uint32_t* values, const uint64_t* offs,
                            const uint32_t* lens, uint32_t n_arrays, uint8_t* buf,
                            uint64_t cap, uint64_t* len_out, char* err, int errcap) {
  return guarded(err, errcap, [&] {
    std::vector<std::vector<uint32_t>> arrays(n_arrays);
    for (uint32_t i = 0; i < n_arrays; ++i)
      arrays[i].assign(values + offs[i], values + offs[i] + lens[i]);
    std::ostringstream os;
    intzip::container_write_raw(os, arrays);
    const std::string s = os.str();
    *len_out = s.size();
    if (buf) {
      if (s.size() > cap) throw std::runtime_error("buffer too small");
      std::memcpy(buf, s.data(), s.size());
    }
  });
}

// container_read_encoded: codec name, then every chunk's payload packed back
// to back into `words` with its record in `chunks` (out_off consecutive over
// all arrays) and array i's first chunk at array_chunk0[i].
int izr_container_read_encoded(const uint8_t* buf, uint64_t len, char* name, int namecap,
                               uint32_t* words, uint64_t words_cap, ChunkRec* chunks,
                               uint32_t chunks_cap, uint32_t* array_chunk0,
                               uint32_t arrays_cap, uint32_t* n_arrays, uint32_t* n_chunks,
                               char* err, int errcap) {
  return guarded(err, errcap, [&] {
    std::istringstream is(std::string(reinterpret_cast<const char*>(buf), len));
    const intzip::EncodedContainer c = intzip::container_read_encoded(is);
    set_err(name, namecap, c.codec_name.c_str());
    if (c.arrays.size() + 1 > arrays_cap) throw std::runtime_error("array table too small");
    uint64_t pos = 0, out = 0;
    uint32_t k = 0;
    for (size_t a = 0; a < c.arrays.size(); ++a) {
      array_chunk0[a] = k;
      for (const intzip::Chunk& ch : c.arrays[a]) {
        if (k >= chunks_cap || pos + ch.payload.size() > words_cap)
          throw std::runtime_error("output too small");
        std::memcpy(words + pos, ch.payload.data(), ch.payload.size() * 4);
        chunks[k++] = {pos, static_cast<uint32_t>(ch.payload.size()), ch.original_length, out};
        pos += ch.payload.size();
        out += ch.original_length;
      }
    }
    array_chunk0[c.arrays.size()] = k;
    *n_arrays = static_cast<uint32_t>(c.arrays.size());
    *n_chunks = k;
  });
}

int izr_container_read_raw(const uint8_t* buf, uint64_t len, uint32_t* values, uint64_t cap,
                           uint32_t* lens, uint32_t lens_cap, uint32_t* n_arrays, char* err,
                           int errcap) {
  return guarded(err, errcap, [&] {
    std::istringstream is(std::string(reinterpret_cast<const char*>(buf), len));
    const auto arrays = intzip::container_read_raw(is);
    if (arrays.size() > lens_cap) throw std::runtime_error("array table too small");
    uint64_t pos = 0;
    for (size_t a = 0; a < arrays.size(); ++a) {
      if (pos + arrays[a].size() > cap) throw std::runtime_error("output too small");
      std::memcpy(values + pos, arrays[a].data(), arrays[a].size() * 4);
      lens[a] = static_cast<uint32_t>(arrays[a].size());
      pos += arrays[a].size();
    }
    *n_arrays = static_cast<uint32_t>(arrays.size());
  });
}

}  // extern "C"
