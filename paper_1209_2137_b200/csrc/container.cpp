// container.cpp — INTZPK01 container ingest (host side of the C ABI).
//
// Restates the reference's container reader (container.cpp:62-169 of the
// reference, format container.h:14-26) over a host buffer instead of a
// std::istream.  Nothing is copied: a first pass validates the container and
// counts chunks (statuses in the reference's throw order), a second pass
// writes the chunk table with every payload indexed where it lies.  The body
// (all array records) is word-structured, so after one H2D copy of the body
// the device decodes the chunks in place; the per-record headers between
// payloads are simply never referenced.
#include <cstdint>
#include <cstring>
#include <new>
#include <string_view>

#include "../../include/intzip_b200.h"

namespace {

constexpr char kMagic[8] = {'I', 'N', 'T', 'Z', 'P', 'K', '0', '1'};
constexpr uint32_t kMaxCodecNameLength = 256;  // container.cpp:13

struct Reader {
  const uint8_t* p;
  uint64_t len, pos;
  bool u32(uint32_t* v) {  // get_u32 (container.cpp:22-30), little-endian
    if (len - pos < 4) return false;
    *v = uint32_t(p[pos]) | uint32_t(p[pos + 1]) << 8 | uint32_t(p[pos + 2]) << 16 |
         uint32_t(p[pos + 3]) << 24;
    pos += 4;
    return true;
  }
  uint32_t word(uint64_t byte_off) const {
    uint32_t v;
    std::memcpy(&v, p + byte_off, 4);  // the host is little-endian (wordbytes.h:15-16)
    return v;
  }
};

// Visitor over one array's chunk records (container.cpp:139-165): calls
// on_chunk(body word of the payload, payload words, original length).
template <class F>
int32_t walk_records(const Reader& r, uint64_t words_at, uint32_t word_count,
                     uint32_t original_length, F&& on_chunk) {
  uint64_t remaining = original_length;
  uint64_t pos = 0;
  while (pos < word_count) {
    if (pos + 2 > word_count) return IZG_E_CT_TRUNC_RECORD;
    const uint32_t n = r.word(words_at + 4 * pos);
    const uint32_t nw = r.word(words_at + 4 * pos + 4);
    pos += 2;
    if (n == 0 || n > IZG_CHUNK_SIZE || n > remaining) return IZG_E_CT_CHUNK_LENGTH;
    if (nw > word_count - pos) return IZG_E_CT_CHUNK_WORDS;
    on_chunk(words_at + 4 * pos, nw, n);
    pos += nw;
    remaining -= n;
  }
  return remaining ? IZG_E_CT_ARRAY_LENGTH : IZG_OK;
}

// Both passes.  index == false: validate and fill *info.  index == true: the
// container is known good; write chunks / array_chunk0.
int32_t pass(const uint8_t* buf, uint64_t len, int raw, izg_container* info, bool index,
             izg_chunk* chunks, uint32_t* array_chunk0) {
  Reader r{buf, len, 0};
  // read_preamble (container.cpp:67-79)
  if (len < 8) return IZG_E_CT_TRUNCATED;
  if (std::memcmp(buf, kMagic, 8) != 0) return IZG_E_CT_MAGIC;
  r.pos = 8;
  uint32_t name_len = 0, n_arrays = 0;
  if (!r.u32(&name_len)) return IZG_E_CT_TRUNCATED;
  if (name_len == 0 || name_len > kMaxCodecNameLength) return IZG_E_CT_NAME_LENGTH;
  if (len - r.pos < name_len) return IZG_E_CT_TRUNCATED;
  const std::string_view name(reinterpret_cast<const char*>(buf + r.pos), name_len);
  r.pos += name_len;
  if (!r.u32(&n_arrays)) return IZG_E_CT_TRUNCATED;
  const bool is_raw = name == "RAW";
  if (!raw && is_raw) return IZG_E_CT_FOUND_RAW;  // container.cpp:134-135
  if (raw && !is_raw) return IZG_E_CT_NOT_RAW;    // container.cpp:95-97
  const uint64_t body = r.pos;
  if (!index) {
    std::memset(info, 0, sizeof(*info));
    std::memcpy(info->codec_name, name.data(), name_len);
    info->codec_name[name_len] = 0;
    info->n_arrays = n_arrays;
    info->body_offset = body;
  }
  uint64_t n_chunks = 0, n_values = 0;
  for (uint32_t a = 0; a < n_arrays; ++a) {
    uint32_t original_length = 0, word_count = 0;
    if (!r.u32(&original_length) || !r.u32(&word_count)) return IZG_E_CT_TRUNCATED;
    if (raw && word_count != original_length) return IZG_E_CT_RAW_COUNT;  // :104-105
    if ((len - r.pos) / 4 < word_count) return IZG_E_CT_TRUNC_PAYLOAD;    // get_words :47-48
    const uint64_t words_at = r.pos;
    if (index && array_chunk0) array_chunk0[a] = (uint32_t)n_chunks;
    if (raw) {
      if (index)
        chunks[n_chunks] = {(words_at - body) / 4, word_count, original_length, n_values};
      ++n_chunks;
      n_values += original_length;
    } else {
      const int32_t st = walk_records(r, words_at, word_count, original_length,
                                      [&](uint64_t at, uint32_t nw, uint32_t n) {
                                        if (index) chunks[n_chunks] = {(at - body) / 4, nw, n,
                                                                       n_values};
                                        ++n_chunks;
                                        n_values += n;
                                      });
      if (st) return st;
    }
    r.pos += 4ull * word_count;
  }
  if (index && array_chunk0) array_chunk0[n_arrays] = (uint32_t)n_chunks;
  if (!index) {
    if (n_chunks > UINT32_MAX) return IZG_E_CT_TRUNC_RECORD;  // cannot be indexed
    info->n_chunks = (uint32_t)n_chunks;
    info->n_values = n_values;
    info->body_words = (r.pos - body + 3) / 4;
  }
  return IZG_OK;
}

}  // namespace

extern "C" int izg_container_scan(const void* buf, uint64_t len, int raw, izg_container* info,
                                  int32_t* status) {
  if ((!buf && len) || !info || !status) return IZG_ERR_INVALID_ARGUMENT;
  *status = pass(static_cast<const uint8_t*>(buf), len, raw, info, false, nullptr, nullptr);
  return *status ? IZG_ERR_CORRUPT : IZG_SUCCESS;
}

extern "C" int izg_container_index(const void* buf, uint64_t len, const izg_container* info,
                                   izg_chunk* chunks, uint32_t* array_chunk0) {
  if (!buf || !info || (info->n_chunks && !chunks)) return IZG_ERR_INVALID_ARGUMENT;
  izg_container again;
  const int raw = std::string_view(info->codec_name) == "RAW";
  if (pass(static_cast<const uint8_t*>(buf), len, raw, &again, false, nullptr, nullptr) ||
      again.n_chunks != info->n_chunks || again.body_offset != info->body_offset)
    return IZG_ERR_INVALID_ARGUMENT;  // not the container that was scanned
  pass(static_cast<const uint8_t*>(buf), len, raw, &again, true, chunks, array_chunk0);
  return IZG_SUCCESS;
}

extern "C" int izg_container_decode_host(const void* buf, uint64_t len, uint32_t* h_out,
                                         uint64_t n_out, int32_t* ct_status,
                                         int32_t* h_status) {
  if (!buf || !ct_status) return IZG_ERR_INVALID_ARGUMENT;
  izg_container info;
  int rc = izg_container_scan(buf, len, 0, &info, ct_status);
  if (rc != IZG_SUCCESS) return rc;
  int codec = 0, delta = 0;
  if (izg_parse_codec_name(info.codec_name, &codec, &delta) != IZG_SUCCESS)
    return IZG_ERR_UNKNOWN_CODEC;
  if (info.n_values > n_out || (info.n_values && !h_out)) return IZG_ERR_INVALID_ARGUMENT;
  if (info.n_chunks == 0) return IZG_SUCCESS;
  izg_chunk* table = new (std::nothrow) izg_chunk[info.n_chunks];
  if (!table) return IZG_ERR_INVALID_ARGUMENT;
  izg_container_index(buf, len, &info, table, nullptr);
  // The body's words are read in place (pageable host memory; the copies in
  // izg_decode_host handle any host alignment).
  const uint32_t* body =
      reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(buf) + info.body_offset);
  rc = izg_decode_host(codec, delta, body, (len - info.body_offset) / 4, table, info.n_chunks,
                       h_out, n_out, h_status);
  delete[] table;
  return rc;
}
