// intzip_b200_host.h — host-side helpers of libintzip_b200 that are not on
// the decode path: the host encoder (encode_array mirror) and the seeded
// synthetic-input generators used by bench.py and the tests.  Declared with
// C linkage so ctypes can bind them; see include/intzip_b200.h for the
// decode ABI.
#pragma once
#include <cstdint>

#include "../../include/intzip_b200.h"

extern "C" {

struct izg_encoded;

// encode_array (codec.cpp:14-37) over n_chunks independent chunks, chunk i
// being values[value_off[i] .. + counts[i]).  delta == IZG_DELTA_NONE encodes
// raw deltas (Codec::encode_deltas, codec.h:31-34).  allow_wrap takes
// differences mod 2^32 instead of rejecting a decrease (delta.cpp:13).
// Returns an opaque result (null + *status on error); the payloads are laid
// out by izg_layout_chunks.
izg_encoded* izg_encode_batch_host(int codec, int delta, const uint32_t* values,
                                   const uint64_t* value_off, const uint32_t* counts,
                                   uint32_t n_chunks, int allow_wrap, int threads, int* status);
uint64_t izg_encoded_words(const izg_encoded* e);
int izg_encoded_copy(const izg_encoded* e, uint32_t* words, izg_chunk* table, int threads);
void izg_encoded_free(izg_encoded* e);

// Seeded generators, one array per index i with std::mt19937_64(seed + i)
// (the reference's seeding convention, datagen.h:27 / datagen.cpp:129-134).
//   model 0 UNIFORM   : n distinct sorted values from [0, 2^d)
//   model 1 CLUSTER   : BASELINE.json ClusterData recipe over [0, 2^d)
//   model 2 GEOMETRIC : gaps ~ Geometric(mean 8) on {1,2,..}; with
//                       probability rate_ppm/1e6 a gap is replaced by
//                       U[2^12, 2^24); prefix sums wrap mod 2^32
//   model 3 RAW       : n values uniform in [0, 2^d) (unsorted; rng() & mask)
// d is drawn per array uniformly from [d_lo, d_hi] with the array's rng
// (only when d_lo != d_hi) and stored in d_out (nullable).
int izg_checksum_host(const uint32_t* v, uint64_t n, uint64_t base, int threads,
                      uint64_t* out);
int izg_gen_arrays(int model, uint32_t count, uint32_t n, uint32_t d_lo, uint32_t d_hi,
                   uint64_t seed, uint32_t rate_ppm, int threads, uint32_t* out,
                   uint32_t* d_out);
}
