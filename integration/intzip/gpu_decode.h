// intzip/gpu_decode.h — the C++ binding a reference maintainer adds to the
// reference tree (proj/core/include/intzip/) to run decode_array on a B200.
//
// Drop-in for intzip::decode_array (proj/core/include/intzip/codec.h:64-71,
// proj/core/src/codec.cpp:39-76): same arguments, same output, same
// exceptions — intzip::CorruptError with the reference's what() text where
// the reference throws it, std::invalid_argument at its misuse sites.  The
// work happens in libintzip_b200.so behind the C ABI of include/intzip_b200.h
// (izg_decode_host: H2D of the placed words, the fused sm_100a decode, D2H).
// Built and run against the reference by tests/cpp/test_integration.cpp
// (oracle/Makefile), which INTEGRATION.md points at.
#pragma once
#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "intzip/codec.h"
#include "intzip/errors.h"
#include "intzip_b200.h"

namespace intzip {

inline void decode_array_b200(const Codec& codec, std::span<const Chunk> chunks,
                              std::vector<uint32_t>& out) {
  int c = 0, d = 0;
  if (izg_parse_codec_name(codec.name().c_str(), &c, &d) != IZG_SUCCESS)
    throw std::invalid_argument("b200: unsupported codec " + codec.name());
  // place payloads (16-byte aligned rows) and build the chunk table
  std::vector<uint32_t> sizes;
  sizes.reserve(chunks.size());
  for (const Chunk& ch : chunks) sizes.push_back(static_cast<uint32_t>(ch.payload.size()));
  std::vector<uint64_t> offs(chunks.size());
  const uint64_t total =
      izg_layout_chunks(c, sizes.data(), static_cast<uint32_t>(chunks.size()), offs.data());
  std::vector<uint32_t> words(total, 0);
  std::vector<izg_chunk> table(chunks.size());
  uint64_t n_out = 0;
  for (size_t i = 0; i < chunks.size(); ++i) {
    std::copy(chunks[i].payload.begin(), chunks[i].payload.end(), words.begin() + offs[i]);
    table[i] = {offs[i], sizes[i], chunks[i].original_length, n_out};
    n_out += chunks[i].original_length;
  }
  out.resize(n_out);
  if (chunks.empty()) return;
  std::vector<int32_t> status(chunks.size());
  const int rc = izg_decode_host(c, d, words.data(), total, table.data(),
                                 static_cast<uint32_t>(chunks.size()), out.data(), n_out,
                                 status.data());
  if (rc == IZG_ERR_CORRUPT) {
    for (int32_t s : status)  // the first failing chunk, as the reference's loop
      if (s) {
        if (s >= IZG_E_COUNT_MULTIPLE) throw std::invalid_argument(izg_status_string(s));
        throw CorruptError(izg_status_string(s));
      }
  }
  if (rc != IZG_SUCCESS) throw std::runtime_error("b200 decode failed: " + std::to_string(rc));
}

}  // namespace intzip
