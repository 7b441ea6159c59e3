// datagen.cpp — seeded synthetic inputs for the BASELINE.json configs
// (bench/test HARNESS; see izh.h).  Written for this repo from the recipes
// in BASELINE.json (DESIGN.md §6 records the interpretation choices); the
// paper's datasets are synthetic.  The only convention
// shared with the reference generator is the per-array seeding
// std::mt19937_64(seed + i) (datagen.h:27).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "izh.h"

namespace {

using Rng = std::mt19937_64;

// Uniform integer in [0, bound), bound >= 1: draw the low bit_width(bound-1)
// bits and retry until the draw falls below bound (< 2 draws on average).
inline uint64_t below(Rng& rng, uint64_t bound) {
  if (bound <= 1) return 0;
  const uint64_t mask = ~uint64_t{0} >> __builtin_clzll(bound - 1);
  for (;;) {
    const uint64_t x = rng() & mask;
    if (x < bound) return x;
  }
}

// n distinct values of [lo, lo + range) in ascending order, written to out.
//   range <= 4n : selection sampling (Knuth's Algorithm S) — walk the
//                 candidates once and keep each with probability
//                 still_needed / still_left, so the output is born sorted;
//   otherwise   : draw n, sort, drop duplicates, draw the shortfall again.
void uniform_set(uint64_t n, uint64_t lo, uint64_t range, Rng& rng, uint32_t*& out) {
  if (n == 0) return;
  if (range <= 4 * n) {
    uint64_t need = n;
    for (uint64_t t = 0; need; ++t) {
      if (below(rng, range - t) < need) {
        *out++ = static_cast<uint32_t>(lo + t);
        --need;
      }
    }
    return;
  }
  std::vector<uint32_t> vals;
  vals.reserve(n + 16);
  while (vals.size() < n) {
    for (uint64_t k = n - vals.size(); k; --k)
      vals.push_back(static_cast<uint32_t>(lo + below(rng, range)));
    std::sort(vals.begin(), vals.end());
    vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
  }
  std::copy(vals.begin(), vals.begin() + n, out);
  out += n;
}

// BASELINE.json ClusterData: split the interval at a uniform point, give a
// uniform random (feasible) share of the count to each side, and sample
// uniformly without replacement once the count is <= 32 or the interval is
// small (range <= 2n).
void cluster_set(uint64_t n, uint64_t lo, uint64_t range, Rng& rng, uint32_t*& out) {
  if (n == 0) return;
  if (n <= 32 || range <= 2 * n) {
    uniform_set(n, lo, range, rng, out);
    return;
  }
  const uint64_t left = 1 + below(rng, range - 1);  // split point in (lo, lo + range)
  const uint64_t right = range - left;
  const uint64_t k_min = n > right ? n - right : 0;  // the right side holds <= right
  const uint64_t k_max = std::min(n, left);
  const uint64_t k = k_min + below(rng, k_max - k_min + 1);
  cluster_set(k, lo, left, rng, out);
  cluster_set(n - k, lo + left, right, rng, out);
}

// Geometric(p = 1/8) on {1, 2, ...} (mean 8): count 3-bit trials until one
// is zero; 21 trials per 64-bit draw.
struct Geometric8 {
  uint64_t bits = 0;
  int left = 0;
  uint32_t draw(Rng& rng) {
    for (uint32_t k = 1;; ++k) {
      if (!left) {
        bits = rng();
        left = 21;
      }
      const bool hit = (bits & 7u) == 0;
      bits >>= 3;
      --left;
      if (hit) return k;
    }
  }
};

void gen_one(int model, uint32_t n, uint32_t d, uint32_t rate_ppm, Rng& rng, uint32_t* out) {
  switch (model) {
    case 0:
      uniform_set(n, 0, uint64_t{1} << d, rng, out);
      break;
    case 1:
      cluster_set(n, 0, uint64_t{1} << d, rng, out);
      break;
    case 2: {  // C4: geometric gaps with outliers; x wraps mod 2^32
      Geometric8 geo;
      uint32_t x = 0;
      for (uint32_t i = 0; i < n; ++i) {
        const bool outlier = below(rng, 1000000) < rate_ppm;
        x += outlier ? 4096u + static_cast<uint32_t>(below(rng, (1u << 24) - 4096u))
                     : geo.draw(rng);
        out[i] = x;
      }
      break;
    }
    case 3: {  // C2: raw values of width <= d
      const uint64_t m = d >= 32 ? 0xFFFFFFFFull : (uint64_t{1} << d) - 1;
      for (uint32_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(rng() & m);
      break;
    }
  }
}

template <class F>
void parallel_ranges(uint64_t count, int threads, F&& f) {
  threads = std::max(1, static_cast<int>(std::min<uint64_t>(threads, std::max<uint64_t>(count, 1))));
  if (threads == 1) {
    f(0, count, 0);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const uint64_t a = count * t / threads, b = count * (t + 1) / threads;
    if (a < b) pool.emplace_back(f, a, b, t);
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" int izh_checksum_host(const uint32_t* v, uint64_t n, uint64_t base, int threads,
                                 uint64_t* out) {
  threads = std::max(1, threads);
  std::vector<uint64_t> s(threads, 0), x(threads, 0);
  parallel_ranges(n, threads, [&](uint64_t a, uint64_t b, int t) {
    uint64_t ss = 0, xx = 0;
    for (uint64_t i = a; i < b; ++i) {
      ss += (uint64_t(v[i]) + 1) * (2 * (base + i) + 1);
      xx ^= v[i];
    }
    s[t] = ss;
    x[t] = xx;
  });
  out[0] = out[1] = 0;
  for (int t = 0; t < threads; ++t) {
    out[0] += s[t];
    out[1] ^= x[t];
  }
  return 0;
}

// The width d of arrays [0, count) without generating them (the first draw
// of each array's rng, exactly as izh_gen_arrays makes it).
extern "C" int izh_array_widths(uint32_t count, uint32_t d_lo, uint32_t d_hi, uint64_t seed,
                                int threads, uint32_t* d_out) {
  if (d_lo > d_hi || d_hi > 32) return -1;
  parallel_ranges(count, threads, [&](uint64_t a, uint64_t b, int) {
    for (uint64_t i = a; i < b; ++i) {
      Rng rng(seed + i);
      d_out[i] = d_lo == d_hi ? d_lo : d_lo + static_cast<uint32_t>(below(rng, d_hi - d_lo + 1));
    }
  });
  return 0;
}

extern "C" int izh_gen_arrays(int model, uint32_t count, uint32_t n, uint32_t d_lo,
                              uint32_t d_hi, uint64_t seed, uint32_t rate_ppm, int threads,
                              uint32_t* out, uint32_t* d_out) {
  if (model < 0 || model > 3 || d_lo > d_hi || d_hi > 32) return -1;
  if (model <= 1 && (uint64_t)n > (uint64_t{1} << d_lo)) return -1;
  parallel_ranges(count, threads, [&](uint64_t a, uint64_t b, int) {
    for (uint64_t i = a; i < b; ++i) {
      Rng rng(seed + i);
      const uint32_t d = d_lo == d_hi ? d_lo : d_lo + static_cast<uint32_t>(below(rng, d_hi - d_lo + 1));
      if (d_out) d_out[i] = d;
      gen_one(model, n, d, rate_ppm, rng, out + i * n);
    }
  });
  return 0;
}
