/*
 * intzip_b200.h — C ABI of the B200-native SIMD-BP128 / SIMD-FastPFOR decoder.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `intzip` (arXiv 1209.2137): the decode side of
 *
 *   intzip::decode_array(const Codec&, std::span<const Chunk>, std::vector<uint32_t>&)
 *       /root/reference/proj/core/include/intzip/codec.h:64-71
 *       /root/reference/proj/core/src/codec.cpp:39-76
 *   intzip::Codec::decode_deltas(std::span<const uint32_t>, uint32_t*, size_t)
 *       /root/reference/proj/core/include/intzip/codec.h:36-40
 *
 * for the codecs "simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"
 * (registry: /root/reference/proj/core/src/codec.cpp:85-109).  The compressed
 * word format is the reference's, unchanged, so chunks
 * encoded by the CPU reference decode here and vice versa.
 *
 * The reference has no FFI of its own (it is a C++ library); every entry point
 * below replaces one reference call and names it.  All signatures use plain
 * pointers and sizes.  Device entry points are stream-ordered and never
 * synchronise or allocate; host entry points (suffix _host) are synchronous.
 * There is no CPU fallback: without a usable sm_100a device every compute
 * entry point returns IZG_ERR_NO_DEVICE.
 */
#ifndef INTZIP_B200_H
#define INTZIP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Chunk length cap: intzip::kChunkSize (codec.h:17). */
#define IZG_CHUNK_SIZE 65536u

/* Codec formats (codec_binpack.h:10-25, codec_patched.h:59-80).  The hot
 * path is SIMD-BP128 and SIMD-FastPFOR; BP32, FastPFOR (scalar groups) and
 * SimplePFOR (Simple-8b exception highs) are the same page framework with
 * scalar 32-integer groups: decode only. */
typedef enum izg_codec {
  IZG_SIMDBP128 = 0,
  IZG_SIMDFASTPFOR = 1,
  IZG_BP32 = 2,
  IZG_FASTPFOR = 3,
  IZG_SIMPLEPFOR = 4
} izg_codec;

/* Inverse differential coding fused into decode.
 *   NONE : no prefix sum; Codec::decode_deltas semantics (codec.h:36-40).
 *   D1   : DeltaMode::scalar  x_i = x_{i-1} + d_i          (delta.cpp:25-51)
 *   D4   : DeltaMode::stride4 x_i = x_{i-4} + d_i          (delta.cpp:60-75)
 *   D2, DM : EXTENSIONS, not in the reference (delta.h:22 has only scalar and
 *          stride4).  D2: x_i = x_{i-2} + d_i; DM: x_{4k+j} = x_{4k-1} + d_{4k+j}
 *          (x_{-1} = 0).  Parity unpinned.              */
typedef enum izg_delta {
  IZG_DELTA_NONE = 0,
  IZG_DELTA_D1 = 1,
  IZG_DELTA_D4 = 2,
  IZG_DELTA_D2 = 3,
  IZG_DELTA_DM = 4
} izg_delta;

/* One independently decodable chunk (intzip::Chunk, codec.h:54-57) placed in a
 * word buffer.  `n` is Chunk::original_length, `n_words` is payload.size(). */
typedef struct izg_chunk {
  uint64_t word_off; /* index of the first payload word in the word buffer */
  uint32_t n_words;  /* payload words                                     */
  uint32_t n;        /* decoded integers (1..65536 for array semantics)   */
  uint64_t out_off;  /* index of the first decoded integer in the output  */
} izg_chunk;

/* Per-chunk status.  Every nonzero code mirrors one reference throw site; a
 * host wrapper maps 1..63 to intzip::CorruptError and 64.. to
 * std::invalid_argument, as the reference would have thrown. */
typedef enum izg_status {
  IZG_OK = 0,
  /* pipeline, codec.cpp */
  IZG_E_CHUNK_LENGTH = 1,      /* codec.cpp:43-44   chunk: bad original length      */
  IZG_E_PAYLOAD_SIZE = 2,      /* codec.cpp:63-64   chunk: payload size mismatch    */
  /* Variable Byte remainder, codec_basic.cpp */
  IZG_E_VBYTE_TRUNCATED = 3,   /* codec_basic.cpp:34-35 vbyte: truncated stream     */
  IZG_E_VBYTE_OVERFLOW = 4,    /* codec_basic.cpp:38-39 vbyte: value exceeds 32 bits*/
  IZG_E_VBYTE_TOO_LONG = 5,    /* codec_basic.cpp:43-44 vbyte: longer than 5 bytes  */
  /* SIMD-BP128, codec_binpack.cpp */
  IZG_E_BP_TRUNC_DESC = 6,     /* codec_binpack.cpp:101-102 truncated descriptor    */
  IZG_E_BP_WIDTH = 7,          /* codec_binpack.cpp:110-111 width byte exceeds 32   */
  IZG_E_BP_TRUNC_PAYLOAD = 8,  /* codec_binpack.cpp:112-113 truncated payload       */
  /* SIMD-FastPFOR, codec_patched.cpp */
  IZG_E_FP_TRUNC_PAGE = 9,     /* codec_patched.cpp:298     truncated page          */
  IZG_E_FP_BA_OFFSET = 10,     /* codec_patched.cpp:300-301 bad byte-array offset   */
  IZG_E_FP_TRUNC_BA = 11,      /* codec_patched.cpp:304-305 truncated byte array    */
  IZG_E_FP_TRUNC_META = 12,    /* codec_patched.cpp:313-314,321-322 truncated block metadata */
  IZG_E_FP_WIDTHS = 13,        /* codec_patched.cpp:318-319 bad block widths        */
  IZG_E_FP_EMPTY_EXC = 14,     /* codec_patched.cpp:324     empty exception list    */
  IZG_E_FP_TRUNC_POS = 15,     /* codec_patched.cpp:325-326 truncated positions     */
  IZG_E_FP_POS_RANGE = 16,     /* codec_patched.cpp:328-330 position out of range   */
  IZG_E_FP_BA_LEN = 17,        /* codec_patched.cpp:335-336 byte array length mismatch */
  IZG_E_FP_NO_BITSET = 18,     /* codec_patched.cpp:347-348 missing exception bitset*/
  IZG_E_FP_TRUNC_EXC = 19,     /* codec_patched.cpp:352-353,362-363 truncated exception array */
  IZG_E_FP_OVERRUN = 20,       /* codec_patched.cpp:387-388 packed blocks overrun   */
  IZG_E_FP_EXHAUSTED = 21,     /* codec_patched.cpp:406-407 exception array exhausted */
  IZG_E_FP_PACKED_SIZE = 22,   /* codec_patched.cpp:414-415 packed area size mismatch */
  /* INTZPK01 container reader, container.cpp (one status per container) */
  IZG_E_CT_TRUNCATED = 23,     /* container.cpp:24-25,69-70,76-77 container: truncated */
  IZG_E_CT_MAGIC = 24,         /* container.cpp:71       bad magic                 */
  IZG_E_CT_NAME_LENGTH = 25,   /* container.cpp:73-74    bad codec name length     */
  IZG_E_CT_FOUND_RAW = 26,     /* container.cpp:134-135  expected encoded data, found RAW */
  IZG_E_CT_TRUNC_PAYLOAD = 27, /* container.cpp:47-48    truncated payload         */
  IZG_E_CT_TRUNC_RECORD = 28,  /* container.cpp:147-148  truncated chunk record    */
  IZG_E_CT_CHUNK_LENGTH = 29,  /* container.cpp:153-155  bad chunk length          */
  IZG_E_CT_CHUNK_WORDS = 30,   /* container.cpp:156-157  bad chunk word count      */
  IZG_E_CT_ARRAY_LENGTH = 31,  /* container.cpp:164-165  array length mismatch     */
  IZG_E_CT_NOT_RAW = 32,       /* container.cpp:95-97    expected RAW data, found codec ... */
  IZG_E_CT_RAW_COUNT = 33,     /* container.cpp:104-105  RAW word count mismatch   */
  /* BP32, codec_binpack.cpp */
  IZG_E_BP32_TRUNC_DESC = 34,  /* codec_binpack.cpp:46-47 bp32: truncated descriptor */
  IZG_E_BP32_WIDTH = 35,       /* codec_binpack.cpp:51    bp32: width byte exceeds 32 */
  IZG_E_BP32_TRUNC_PAYLOAD = 36, /* codec_binpack.cpp:52-53 bp32: truncated payload  */
  /* SimplePFOR exception highs, codec_basic.cpp */
  IZG_E_S8_EXHAUSTED = 37,     /* codec_basic.cpp:302-303 simple8b: stream exhausted before count */
  /* internal: the split decode's look-back made no progress (a bug, never
     a property of the input; reported instead of hanging the device) */
  IZG_E_SPLIT_STALL = 38,
  /* misuse -> std::invalid_argument */
  IZG_E_COUNT_MULTIPLE = 64,   /* codec_binpack.cpp:13-14, codec_patched.cpp:53-54 count % 128 != 0 */
  IZG_E_PAGE_TOO_LARGE = 65,   /* codec_patched.cpp:55-56 page exceeds 65536 integers */
  IZG_E_DECREASING = 66        /* delta.cpp:13 delta encode: input is not nondecreasing */
} izg_status;

/* API-level return codes (not per chunk). */
#define IZG_SUCCESS 0
#define IZG_ERR_INVALID_ARGUMENT (-1) /* bad enum, null pointer, misaligned buffer */
#define IZG_ERR_CUDA (-2)             /* a CUDA runtime call failed               */
#define IZG_ERR_NO_DEVICE (-3)        /* no sm_100 device: there is no CPU fallback */
#define IZG_ERR_CORRUPT (-4)          /* _host calls: some chunk had status != 0  */
#define IZG_ERR_UNKNOWN_CODEC (-5)    /* make_codec: unknown codec (codec.cpp:108) */

/* ---- library --------------------------------------------------------- */

/* Human-readable text of a per-chunk status (the reference's what()). */
const char* izg_status_string(int32_t status);

/* make_codec(name) (codec.cpp:99-109) restricted to the hot-path codecs:
 * "simdbp128" -> (IZG_SIMDBP128, D1), "simdbp128-s4" -> (.., D4), likewise
 * "simdfastpfor[-s4]".  Extension names "-d2"/"-dm" select D2/DM.  Returns
 * IZG_SUCCESS or IZG_ERR_UNKNOWN_CODEC. */
int izg_parse_codec_name(const char* name, int* codec, int* delta);

/* Word-buffer placement contract for izg_decode: the buffer is 16-byte
 * aligned, and for every chunk the 16-byte-aligned span covering its payload
 * lies inside the allocation.  izg_layout_chunks assigns word_off for chunks
 * of the given sizes (SIMD-BP128 payloads start 16-byte aligned, SIMD-FastPFOR
 * pages start at 12 mod 16 so their packed rows are 16-byte aligned) and
 * returns the total words to allocate (trailing pad included). */
uint64_t izg_layout_chunks(int codec, const uint32_t* n_words, uint32_t n_chunks,
                           uint64_t* word_off_out);

/* ---- device entry points (stream-ordered) ---------------------------- */

/* Fused decode of a batch of chunks, one kernel launch.
 *   delta == IZG_DELTA_NONE : per chunk, Codec::decode_deltas(payload, out, n)
 *                             (codec.h:36-40): n % 128 == 0 required; words
 *                             consumed go to d_consumed[i] (nullable).
 *   otherwise               : per chunk, the body of decode_array's chunk loop
 *                             (codec.cpp:50-68): core decode, Variable Byte
 *                             remainder, exact-consumption check, prefix sum.
 * d_status[i] receives the chunk's izg_status (0 = OK); after a nonzero
 * status the chunk's output is unspecified (delta.h:19-20).  d_words must
 * follow izg_layout_chunks's contract.  stream is a cudaStream_t (NULL =
 * legacy default stream).  Returns IZG_SUCCESS or an API error. */
int izg_decode(int codec, int delta, const uint32_t* d_words,
               const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
               int32_t* d_status, uint32_t* d_consumed, void* stream);

/* Bytes of device workspace izg_decode_ws can use for n_chunks chunks of
 * this codec.  SIMD-FastPFOR: the page index (a two-launch index pass +
 * table-driven decode).  Small batches of SIMD-BP128 or SIMD-FastPFOR add
 * the split decode's look-back state (several warps per chunk, decoupled
 * look-back carry; IZG_SPLIT=0/1 in the environment forces it off/on).
 * SIMD-BP128 batches of 2,432..14,208 chunks ask for the relay decode's
 * per-chunk state (64 bytes per chunk + 64: segments of a chunk claimed level
 * by level, position / carry / first error handed on in order; IZG_RELAY=0/1
 * forces it off/on): worth passing for chunks of tens of thousands of
 * integers (4-12 % faster at 65,536 per chunk); with chunks of a few thousand
 * it costs 5-15 %, so callers that know their chunks are short pass no
 * workspace for SIMD-BP128 (izg_decode_host does this itself).  0 when nothing
 * applies. */
uint64_t izg_decode_workspace_size(int codec, uint32_t n_chunks);

/* The page index alone (SIMD-FastPFOR; 0 otherwise): a workspace of exactly
 * this size selects the one-warp-per-page indexed decode even for small
 * batches. */
uint64_t izg_decode_index_workspace_size(int codec, uint32_t n_chunks);

/* izg_decode with a caller-owned device workspace (16-byte aligned, at least
 * izg_decode_workspace_size bytes; otherwise this is exactly izg_decode).
 * SIMD-FastPFOR then runs as two stream-ordered launches: a page index pass
 * (one warp per page parses the byte array and the exception directory and
 * makes every metadata check of codec_patched.cpp:292-416) and the decode
 * reading per-block records.  Small batches run the split decode (several
 * warps per chunk with a decoupled look-back carry).  Results and statuses
 * are identical to izg_decode's; the workspace must stay untouched until the
 * decode completes on `stream`. */
int izg_decode_ws(int codec, int delta, const uint32_t* d_words,
                  const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
                  int32_t* d_status, uint32_t* d_consumed, void* d_workspace,
                  uint64_t workspace_bytes, void* stream);

/* izg_decode_ws in two stream-ordered halves, so the SIMD-FastPFOR page
 * index pass can run on another stream while other work runs (e.g. a
 * SIMD-BP128 decode of the same step):
 *   phase 1: the page index pass alone (fills the workspace);
 *   phase 2: the decode alone, from a workspace phase 1 filled for the same
 *            words and table (order the two with events/streams);
 *   phase 0: both (= izg_decode_ws).
 * On batches and codecs without the two-launch indexed path, phase 1 does
 * nothing and phase 2 is the whole decode.  Results equal izg_decode_ws's. */
int izg_decode_ws_phase(int codec, int delta, const uint32_t* d_words,
                        const izg_chunk* d_chunks, uint32_t n_chunks, uint32_t* d_out,
                        int32_t* d_status, uint32_t* d_consumed, void* d_workspace,
                        uint64_t workspace_bytes, int phase, void* stream);

/* Order-sensitive checksum of n words: sum over i of (w_i + 1) * (2i + 1)
 * mod 2^64 (xor of all words in d_result[1]).  Used for whole-box parity with
 * an NCCL reduction; not part of the reference. */
int izg_checksum(const uint32_t* d_data, uint64_t n, uint64_t* d_result,
                 void* stream);

/* Fused encode of a batch of chunks, one kernel launch (secondary path;
 * encode_array's chunk body, codec.cpp:21-35, or Codec::encode_deltas when
 * delta == IZG_DELTA_NONE).  Per chunk i, d_chunks[i] is read as
 *   out_off = index of the chunk's first input value in d_values,
 *   n       = values (1..65536; a multiple of 128 for IZG_DELTA_NONE),
 *   word_off= where its payload starts in d_words, with room for
 *             izg_encode_bound(codec, n) words,
 * and the kernel writes d_chunks[i].n_words.  Output words are identical to
 * the reference encoder's.  allow_wrap != 0 takes differences mod 2^32
 * instead of rejecting a decreasing input (IZG_E_DECREASING). */
int izg_encode(int codec, int delta, const uint32_t* d_values, izg_chunk* d_chunks,
               uint32_t n_chunks, uint32_t* d_words, int32_t* d_status, int allow_wrap,
               void* stream);

/* Words one chunk of n values can need (exact upper bound of the format). */
uint64_t izg_encode_bound(int codec, uint32_t n);

/* ---- consumer: intersection of decoded arrays ------- */
/* Sorted intersection of two nondecreasing uint32 arrays in device memory
 * (e.g. two posting lists decoded by izg_decode): the distinct values present
 * in both, ascending (numpy.intersect1d semantics; the reference has no
 * intersection API, PAPER.md:1697-1719 motivates it).  d_out holds
 * min(n_a, n_b) words; *d_count (device) receives the number written.
 * Stream-ordered; workspace of izg_intersect_workspace_size bytes. */
uint64_t izg_intersect_workspace_size(uint64_t n_a, uint64_t n_b);
int izg_intersect_sorted(const uint32_t* d_a, uint64_t n_a, const uint32_t* d_b,
                         uint64_t n_b, uint32_t* d_out, uint64_t* d_count,
                         void* d_workspace, uint64_t workspace_bytes, void* stream);

/* Fused decode -> intersect: decodes the chunks (codec as izg_decode, delta
 * IZG_DELTA_D1 or IZG_DELTA_D4, array mode) and intersects the decoded
 * values with the nondecreasing device list d_s WITHOUT writing the decoded
 * integers anywhere: each decoded tile is merged against d_s in shared
 * memory.  d_out (n_s words) receives the distinct values present both in
 * d_s and in the decoded chunks, ascending; *d_count (device) their number.
 * Each chunk's decoded values must be nondecreasing (sorted lists, as D1/D4
 * encode them); chunks may come from one array or several.  d_status gets
 * the per-chunk statuses izg_decode would give; the result is meaningful
 * only when all are IZG_OK.  chunk.out_off is ignored.  Stream-ordered;
 * workspace of izg_decode_intersect_workspace_size(n_s) bytes. */
uint64_t izg_decode_intersect_workspace_size(uint64_t n_s);
int izg_decode_intersect(int codec, int delta, const uint32_t* d_words,
                         const izg_chunk* d_chunks, uint32_t n_chunks, const uint32_t* d_s,
                         uint64_t n_s, uint32_t* d_out, uint64_t* d_count, int32_t* d_status,
                         void* d_workspace, uint64_t workspace_bytes, void* stream);

/* ---- host entry points (synchronous, host buffers) -------------------- */

/* decode_array over a batch of chunks held in HOST memory: copies the words
 * and chunk table to the device, decodes, copies the integers back.  h_status
 * (nullable, n_chunks entries) receives per-chunk statuses; returns
 * IZG_ERR_CORRUPT if any chunk failed.  Device scratch is cached per thread
 * and grown on demand. */
int izg_decode_host(int codec, int delta, const uint32_t* h_words,
                    uint64_t n_words, const izg_chunk* h_chunks,
                    uint32_t n_chunks, uint32_t* h_out, uint64_t n_out,
                    int32_t* h_status);

/* Release the per-thread device scratch used by the _host entry points. */
void izg_release_host_scratch(void);

/* ---- INTZPK01 container ingest (host) --------------------------------- */
/* The reference's on-disk container (container.h:14-26) read from a host
 * buffer instead of a std::istream, without copying payloads: chunk records
 * are indexed in place, so the container body can be copied to the device
 * as one block and decoded where it lies. */
typedef struct izg_container {
  char codec_name[260]; /* NUL-terminated; "RAW" for raw containers         */
  uint32_t n_arrays;
  uint32_t n_chunks;    /* chunk records (RAW: one per array)               */
  uint64_t n_values;    /* sum of the arrays' lengths                       */
  uint64_t body_offset; /* byte offset of the first array record            */
  uint64_t body_words;  /* 32-bit words from body_offset through the last array */
} izg_container;

/* container_read_encoded (raw == 0, container.cpp:132-169) or
 * container_read_raw (raw != 0, container.cpp:93-110) validation of
 * buf[0, len): IZG_SUCCESS and *info, or IZG_ERR_CORRUPT with *status = the
 * IZG_E_CT_* code of the reference's first CorruptError.  Trailing bytes
 * after the last array are ignored, as by the reference. */
int izg_container_scan(const void* buf, uint64_t len, int raw, izg_container* info,
                       int32_t* status);

/* Chunk table of a scanned container: chunks[k].word_off = index of chunk k's
 * first payload word counted from body word 0 (the word at buf +
 * info->body_offset), out_off consecutive over all arrays in order, so the
 * arrays decode back to back.  array_chunk0 (nullable, n_arrays + 1 entries)
 * receives each array's first chunk index.  RAW: one record per array
 * covering its values. */
int izg_container_index(const void* buf, uint64_t len, const izg_container* info,
                        izg_chunk* chunks, uint32_t* array_chunk0);

/* Read + decode a whole encoded container held in host memory: scan, index,
 * then izg_decode_host of the body into h_out (n_values integers, arrays back
 * to back).  *ct_status = container status (0 = OK); h_status (nullable,
 * n_chunks entries) = per-chunk decode statuses.  Returns IZG_ERR_CORRUPT on
 * any container or chunk error, IZG_ERR_UNKNOWN_CODEC for a codec without a
 * device decoder (make_codec, codec.cpp:108). */
int izg_container_decode_host(const void* buf, uint64_t len, uint32_t* h_out, uint64_t n_out,
                              int32_t* ct_status, int32_t* h_status);

#ifdef __cplusplus
}
#endif

#endif /* INTZIP_B200_H */
