// host_datagen.cpp — seeded synthetic inputs for the BASELINE.json configs
// (bench.py and tests).  Not on the decode path; no reference code involved.
// The paper's datasets are synthetic; BASELINE.json
// restates their recipes, and DESIGN.md §6 records the interpretation choices.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "intzip_b200_host.h"

namespace {

using Rng = std::mt19937_64;

// Exactly uniform draw from [0, bound) by 128-bit multiply-shift with
// rejection (implementation-independent, like datagen.cpp:16-28).
inline uint64_t bounded(Rng& rng, uint64_t bound) {
  unsigned __int128 m = (unsigned __int128)rng() * bound;
  uint64_t low = (uint64_t)m;
  if (low < bound) {
    const uint64_t threshold = (0 - bound) % bound;
    while (low < threshold) {
      m = (unsigned __int128)rng() * bound;
      low = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

// n distinct values from [lo, lo + range), appended in ascending order.
void uniform_into(uint64_t n, uint64_t lo, uint64_t range, Rng& rng, uint32_t*& out) {
  if (n == 0) return;
  if (range <= 32 * n) {
    // dense: bitmap rejection (complement when more than half is requested)
    const bool invert = n > range / 2;
    const uint64_t draws = invert ? range - n : n;
    const uint64_t nbw = (range + 63) / 64;
    uint64_t small[64];
    std::vector<uint64_t> big;
    uint64_t* bits = small;
    if (nbw > 64) {
      big.assign(nbw, 0);
      bits = big.data();
    } else {
      std::memset(small, 0, sizeof(uint64_t) * nbw);
    }
    for (uint64_t k = 0; k < draws;) {
      const uint64_t v = bounded(rng, range);
      uint64_t& w = bits[v >> 6];
      const uint64_t b = uint64_t{1} << (v & 63);
      if (w & b) continue;
      w |= b;
      ++k;
    }
    for (uint64_t wi = 0; wi < nbw; ++wi) {
      uint64_t w = invert ? ~bits[wi] : bits[wi];
      if (invert && wi == nbw - 1 && range % 64) w &= (uint64_t{1} << (range % 64)) - 1;
      while (w) {
        *out++ = (uint32_t)(lo + wi * 64 + (uint64_t)__builtin_ctzll(w));
        w &= w - 1;
      }
    }
    return;
  }
  if (n <= 64) {
    // sparse and small: draw, sort, drop duplicates, top up
    uint32_t buf[64];
    uint32_t have = 0;
    while (have < n) {
      for (uint32_t k = have; k < n; ++k) buf[k] = (uint32_t)(lo + bounded(rng, range));
      std::sort(buf, buf + n);
      have = (uint32_t)(std::unique(buf, buf + n) - buf);
    }
    std::memcpy(out, buf, n * 4);
    out += n;
    return;
  }
  // sparse and large: draw, sort, deduplicate, top up until n remain
  std::vector<uint32_t> vals;
  vals.reserve(n + n / 8);
  while (vals.size() < n) {
    const uint64_t need = n - vals.size();
    for (uint64_t k = 0; k < need; ++k) vals.push_back((uint32_t)(lo + bounded(rng, range)));
    std::sort(vals.begin(), vals.end());
    vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
  }
  std::memcpy(out, vals.data(), n * 4);
  out += n;
}

// BASELINE.json ClusterData: split the interval at a uniform point, give a
// uniform random (feasible) share of the count to each side, and sample
// uniformly without replacement once the count is <= 32 or the interval is
// small (range <= 2n).
void cluster_into(uint64_t n, uint64_t lo, uint64_t range, Rng& rng, uint32_t*& out) {
  if (n == 0) return;
  if (n <= 32 || range <= 2 * n) {
    uniform_into(n, lo, range, rng, out);
    return;
  }
  const uint64_t left = 1 + bounded(rng, range - 1);  // split point in (lo, lo+range)
  const uint64_t right = range - left;
  const uint64_t k_lo = n > right ? n - right : 0;
  const uint64_t k_hi = std::min(n, left);
  const uint64_t k = k_lo + bounded(rng, k_hi - k_lo + 1);
  cluster_into(k, lo, left, rng, out);
  cluster_into(n - k, lo + left, right, rng, out);
}

// Geometric(p = 1/8) on {1, 2, ...} (mean 8) from 3-bit Bernoulli trials.
struct Geo {
  uint64_t buf = 0;
  int left = 0;
  uint32_t draw(Rng& rng) {
    uint32_t k = 1;
    for (;;) {
      if (left == 0) {
        buf = rng();
        left = 21;
      }
      const uint32_t t = buf & 7;
      buf >>= 3;
      --left;
      if (t == 0) return k;
      ++k;
    }
  }
};

void gen_one(int model, uint32_t n, uint32_t d, uint32_t rate_ppm, Rng& rng, uint32_t* out) {
  switch (model) {
    case 0:
      uniform_into(n, 0, uint64_t{1} << d, rng, out);
      break;
    case 1:
      cluster_into(n, 0, uint64_t{1} << d, rng, out);
      break;
    case 2: {
      Geo geo;
      uint32_t x = 0;
      for (uint32_t i = 0; i < n; ++i) {
        uint32_t gap;
        if (bounded(rng, 1000000) < rate_ppm)
          gap = 4096u + (uint32_t)bounded(rng, (1u << 24) - 4096u);
        else
          gap = geo.draw(rng);
        x += gap;  // wraps mod 2^32
        out[i] = x;
      }
      break;
    }
    case 3: {
      const uint64_t m = d >= 32 ? 0xFFFFFFFFull : (uint64_t{1} << d) - 1;
      for (uint32_t i = 0; i < n; ++i) out[i] = (uint32_t)(rng() & m);
      break;
    }
  }
}

}  // namespace

// izg_checksum on the host over values whose first element has global index
// base: out[0] = sum (w+1)(2i+1) mod 2^64, out[1] = xor.
extern "C" int izg_checksum_host(const uint32_t* v, uint64_t n, uint64_t base, int threads,
                                 uint64_t* out) {
  threads = std::max(1, threads);
  std::vector<uint64_t> s(threads, 0), x(threads, 0);
  auto work = [&](int t) {
    const uint64_t a = n * t / threads, b = n * (t + 1) / threads;
    uint64_t ss = 0, xx = 0;
    for (uint64_t i = a; i < b; ++i) {
      ss += (uint64_t(v[i]) + 1) * (2 * (base + i) + 1);
      xx ^= v[i];
    }
    s[t] = ss;
    x[t] = xx;
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
  out[0] = out[1] = 0;
  for (int t = 0; t < threads; ++t) {
    out[0] += s[t];
    out[1] ^= x[t];
  }
  return IZG_SUCCESS;
}

extern "C" int izg_gen_arrays(int model, uint32_t count, uint32_t n, uint32_t d_lo,
                              uint32_t d_hi, uint64_t seed, uint32_t rate_ppm, int threads,
                              uint32_t* out, uint32_t* d_out) {
  if (model < 0 || model > 3 || d_lo > d_hi || d_hi > 32) return IZG_ERR_INVALID_ARGUMENT;
  if (model <= 1 && (uint64_t)n > (uint64_t{1} << d_lo)) return IZG_ERR_INVALID_ARGUMENT;
  if (model <= 1 && d_hi > 32) return IZG_ERR_INVALID_ARGUMENT;
  auto work = [&](uint32_t a, uint32_t b) {
    for (uint32_t i = a; i < b; ++i) {
      Rng rng(seed + i);
      const uint32_t d = d_lo == d_hi ? d_lo : d_lo + (uint32_t)bounded(rng, d_hi - d_lo + 1);
      if (d_out) d_out[i] = d;
      gen_one(model, n, d, rate_ppm, rng, out + (uint64_t)i * n);
    }
  };
  threads = std::max(1, std::min<int>(threads, (int)std::max<uint32_t>(count, 1)));
  std::vector<std::thread> pool;
  const uint32_t per = (count + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const uint32_t a = std::min<uint32_t>(count, per * t), b = std::min<uint32_t>(count, per * (t + 1));
    if (a < b) pool.emplace_back(work, a, b);
  }
  for (auto& th : pool) th.join();
  return IZG_SUCCESS;
}
