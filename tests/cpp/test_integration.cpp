// test_integration.cpp — compiles INTEGRATION.md's C++ binding
// (integration/intzip/gpu_decode.h) against the reference's own headers and
// library (oracle/_ref, built from /root/reference/proj/core/src) and holds
// intzip::decode_array_b200 to intzip::decode_array:
//   * same output on arrays encoded by intzip::encode_array (every hot-path
//     codec name, ragged lengths, multi-chunk arrays, VByte remainders);
//   * on corrupted chunks, the same outcome: both succeed with the same
//     output, or both throw the same exception type with the same what().
// TEST INFRASTRUCTURE (built by oracle/Makefile, run by
// tests/test_gpu_integration.py on the GPU box).  Exit code 0 = pass.
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "intzip/codec.h"
#include "intzip/errors.h"
#include "intzip/gpu_decode.h"

namespace {

struct Outcome {
  int kind = 0;  // 0 ok, 1 CorruptError, 2 invalid_argument, 3 other
  std::string what;
  std::vector<uint32_t> out;
};

template <class F>
Outcome run(F&& f) {
  Outcome o;
  try {
    f(o.out);
  } catch (const intzip::CorruptError& e) {
    o.kind = 1;
    o.what = e.what();
  } catch (const std::invalid_argument& e) {
    o.kind = 2;
    o.what = e.what();
  } catch (const std::exception& e) {
    o.kind = 3;
    o.what = e.what();
  }
  return o;
}

std::vector<uint32_t> sorted_array(std::mt19937_64& rng, size_t n, uint32_t max_gap) {
  std::vector<uint32_t> v(n);
  uint64_t x = 0;
  for (auto& e : v) {
    x += rng() % (uint64_t(max_gap) + 1);
    e = static_cast<uint32_t>(std::min<uint64_t>(x, 0xFFFFFFFFu));
  }
  return v;
}

}  // namespace

int main() {
  const char* names[] = {"simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"};
  const size_t lens[] = {1, 5, 127, 128, 129, 2048, 2049, 65535, 65536, 65537, 200000};
  std::mt19937_64 rng(2012);
  int checked = 0, failures = 0, corrupt_agree = 0, corrupt_thrown = 0;
  for (const char* name : names) {
    const auto codec = intzip::make_codec(name);
    for (size_t n : lens) {
      for (uint32_t gap : {1u, 100u, 1u << 20}) {
        const auto values = sorted_array(rng, n, gap);
        const auto chunks = intzip::encode_array(*codec, values);
        const Outcome cpu = run([&](auto& out) { intzip::decode_array(*codec, chunks, out); });
        const Outcome gpu =
            run([&](auto& out) { intzip::decode_array_b200(*codec, chunks, out); });
        ++checked;
        if (cpu.kind || gpu.kind || cpu.out != gpu.out || gpu.out != values) {
          std::printf("MISMATCH %s n=%zu gap=%u cpu=%d gpu=%d %s\n", name, n, gap, cpu.kind,
                      gpu.kind, gpu.what.c_str());
          ++failures;
        }
        // corruption: flip bits / truncate / change the length of one chunk
        for (int trial = 0; trial < 12; ++trial) {
          auto bad = chunks;
          auto& ch = bad[rng() % bad.size()];
          const int kind = trial % 4;
          if (kind == 0 && !ch.payload.empty()) {
            ch.payload[rng() % ch.payload.size()] ^= 1u << (rng() % 32);
          } else if (kind == 1 && !ch.payload.empty()) {
            ch.payload.resize(rng() % ch.payload.size());
          } else if (kind == 2) {
            ch.payload.push_back(static_cast<uint32_t>(rng()));
          } else {
            ch.original_length = static_cast<uint32_t>(rng() % 70000);
          }
          const Outcome c2 = run([&](auto& out) { intzip::decode_array(*codec, bad, out); });
          const Outcome g2 = run([&](auto& out) { intzip::decode_array_b200(*codec, bad, out); });
          const bool same = c2.kind == g2.kind && c2.what == g2.what &&
                            (c2.kind != 0 || c2.out == g2.out);
          if (!same) {
            std::printf("CORRUPT MISMATCH %s n=%zu trial=%d cpu=%d '%s' gpu=%d '%s'\n", name, n,
                        trial, c2.kind, c2.what.c_str(), g2.kind, g2.what.c_str());
            ++failures;
          } else {
            ++corrupt_agree;
            corrupt_thrown += c2.kind != 0;
          }
        }
      }
    }
  }
  std::printf("checked %d arrays, %d corruptions agree (%d thrown), %d failures\n", checked,
              corrupt_agree, corrupt_thrown, failures);
  return failures ? 1 : 0;
}
