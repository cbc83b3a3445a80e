// rng.cuh -- the channel / construction random streams, usable on host and
// device so that device-generated LLRs reproduce the host (reference) stream.
//
// Algorithms restated from the reference's published choices
// (proj/include/ldpc/rng.hpp): SplitMix64 seeding (:10-15), the two-stream
// seed mix (:19-25), xoshiro256++ (:36-46), the (0,1] double draw (:49),
// Box-Muller with cos-then-cached-sin (:52-64), rejection next_below
// (:67-73) and back-to-front Fisher-Yates (:75-82).
#pragma once
#include <cstdint>
#include <cmath>

#ifdef __CUDACC__
#define LDPCB_HD __host__ __device__ __forceinline__
#else
#define LDPCB_HD inline
#endif

namespace ldpcb {

LDPCB_HD uint64_t splitmix_next(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Independent sub-stream seed for (seed, stream): frames, iterations, ...
LDPCB_HD uint64_t stream_seed(uint64_t seed, uint64_t stream) {
  uint64_t st = seed;
  uint64_t a = splitmix_next(st);
  st ^= 0xd1342543de82ef95ull * (stream + 1);
  return a ^ splitmix_next(st);
}

struct Stream {
  uint64_t w0, w1, w2, w3;
  double cached;
  bool have_cached;

  LDPCB_HD explicit Stream(uint64_t seed) : cached(0.0), have_cached(false) {
    uint64_t st = seed;
    w0 = splitmix_next(st);
    w1 = splitmix_next(st);
    w2 = splitmix_next(st);
    w3 = splitmix_next(st);
  }

  static LDPCB_HD uint64_t rol(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

  LDPCB_HD uint64_t u64() {
    const uint64_t out = rol(w0 + w3, 23) + w0;
    const uint64_t t = w1 << 17;
    w2 ^= w0;
    w3 ^= w1;
    w1 ^= w2;
    w0 ^= w3;
    w2 ^= t;
    w3 = rol(w3, 45);
    return out;
  }

  // (0, 1]: 53 random bits, never 0
  LDPCB_HD double unit() { return static_cast<double>((u64() >> 11) + 1) * 0x1.0p-53; }

  LDPCB_HD double normal() {
    if (have_cached) {
      have_cached = false;
      return cached;
    }
    const double a = unit();
    const double b = unit();
    const double r = sqrt(-2.0 * log(a));
    const double t = 6.283185307179586476925286766559 * b;
    cached = r * sin(t);
    have_cached = true;
    return r * cos(t);
  }

  LDPCB_HD uint64_t below(uint64_t n) {
    const uint64_t lim = (0 - n) % n;
    for (;;) {
      const uint64_t x = u64();
      if (x >= lim) return x % n;
    }
  }

  template <class T>
  LDPCB_HD void permute(T* a, uint64_t n) {
    for (uint64_t i = n; i > 1; --i) {
      const uint64_t j = below(i);
      T tmp = a[i - 1];
      a[i - 1] = a[j];
      a[j] = tmp;
    }
  }
};

// BI-AWGN noise variance for information-bit SNR (channel.hpp:21-24)
inline double awgn_sigma2(double ebn0_db, double rate) {
  return 1.0 / (2.0 * rate * std::pow(10.0, ebn0_db / 10.0));
}

}  // namespace ldpcb
