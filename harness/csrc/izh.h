// izh.h — bench/test HARNESS library (libizh.so): seeded synthetic inputs
// for the BASELINE.json configs and a host encoder for the hot-path codecs.
//
// Not product code: libintzip_b200.so (the decoder, include/intzip_b200.h)
// neither contains nor links any of this.  bench.py's GPU arm and the tests
// use libizh.so to make inputs; the reference arm gets the same generator
// compiled into oracle/_ref/libintzip_ref.so (oracle/Makefile), so both arms
// decode the same arrays without the reference arm loading any repo library.
#pragma once
#include <cstdint>

#include "../../include/intzip_b200.h"

extern "C" {

// Seeded generators, one array per index i with std::mt19937_64(seed + i).
//   model 0 UNIFORM   : n distinct sorted values from [0, 2^d)
//   model 1 CLUSTER   : BASELINE.json ClusterData recipe over [0, 2^d)
//   model 2 GEOMETRIC : gaps ~ Geometric(mean 8) on {1,2,..}; with
//                       probability rate_ppm/1e6 a gap is replaced by
//                       U[2^12, 2^24); prefix sums wrap mod 2^32
//   model 3 RAW       : n values uniform in [0, 2^d) (unsorted)
// d is drawn per array uniformly from [d_lo, d_hi] with the array's rng
// (only when d_lo != d_hi) and stored in d_out (nullable).
// Returns 0, or -1 on bad arguments.
int izh_gen_arrays(int model, uint32_t count, uint32_t n, uint32_t d_lo, uint32_t d_hi,
                   uint64_t seed, uint32_t rate_ppm, int threads, uint32_t* out,
                   uint32_t* d_out);

// The per-array width d of izh_gen_arrays for arrays [0, count), without
// generating them (bench.py balances shards by the compressed bytes d
// implies).
int izh_array_widths(uint32_t count, uint32_t d_lo, uint32_t d_hi, uint64_t seed, int threads,
                     uint32_t* d_out);

// Order-sensitive checksum of values whose first element has global index
// `base` (the device izg_checksum's definition): out[0] = sum (v+1)(2i+1)
// mod 2^64, out[1] = xor of v.
int izh_checksum_host(const uint32_t* v, uint64_t n, uint64_t base, int threads,
                      uint64_t* out);

// Host encoder: encode_array (codec.cpp:14-37) over n_chunks independent
// chunks, chunk i = values[value_off[i] .. + counts[i]).  delta ==
// IZG_DELTA_NONE encodes raw deltas (Codec::encode_deltas).  allow_wrap takes
// differences mod 2^32 instead of rejecting a decrease (delta.cpp:13).
// Payloads are placed like izg_layout_chunks.
struct izh_encoded;
izh_encoded* izh_encode_batch(int codec, int delta, const uint32_t* values,
                              const uint64_t* value_off, const uint32_t* counts,
                              uint32_t n_chunks, int allow_wrap, int threads, int* status);
uint64_t izh_encoded_words(const izh_encoded* e);
int izh_encoded_copy(const izh_encoded* e, uint32_t* words, izg_chunk* table, int threads);
void izh_encoded_free(izh_encoded* e);
}
