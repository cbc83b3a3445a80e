// host_rng.cpp -- jump-ahead for the channel stream (xoshiro256, rng.hpp:36-46).
//
// The xoshiro256 state transition is linear over GF(2), so advancing a state
// by d draws is multiplication by M^d, and M^d = r(M) with r(x) = x^d mod p(x),
// p the characteristic polynomial of M (Cayley-Hamilton). p is recovered once
// with Berlekamp-Massey from one state bit; r is a square-and-multiply over
// GF(2)[x]. Applying r to a state is the loop of the published jump()
// functions: for each set coefficient i (lowest first), xor the state into an
// accumulator, then step. The device channel uses this to start one thread
// per segment of a frame's noise stream (decoder.cu channel_seg_kernel).
#include <array>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "host.hpp"
#include "rng.cuh"

namespace ldpcb {
namespace {

constexpr int kDeg = 256;
constexpr int kWords = 9;  // up to degree 2*256 - 2 in products, plus slack

using Poly = std::array<uint64_t, kWords>;  // bit i = coefficient of x^i

bool bit(const Poly& a, int i) { return (a[i >> 6] >> (i & 63)) & 1u; }
void set_bit(Poly& a, int i) { a[i >> 6] |= 1ull << (i & 63); }

int degree(const Poly& a) {
  for (int w = kWords - 1; w >= 0; --w)
    if (a[w]) return 64 * w + 63 - __builtin_clzll(a[w]);
  return -1;
}

// characteristic polynomial of the xoshiro256 transition (degree 256)
Poly char_poly() {
  // 2 * 256 consecutive values of one state bit (bit 0 of w0) from an
  // arbitrary nonzero state
  Stream st(0x243f6a8885a308d3ull);
  std::vector<int> s(2 * kDeg);
  for (int t = 0; t < 2 * kDeg; ++t) {
    s[t] = static_cast<int>(st.w0 & 1u);
    st.u64();
  }
  // Berlekamp-Massey over GF(2): connection polynomial C(x) = 1 + c1 x + ...
  std::vector<int> C(2 * kDeg + 1, 0), B(2 * kDeg + 1, 0), T;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  for (int nn = 0; nn < 2 * kDeg; ++nn) {
    int d = s[nn];
    for (int i = 1; i <= L; ++i) d ^= C[i] & s[nn - i];
    if (d == 0) {
      ++m;
    } else if (2 * L <= nn) {
      T = C;
      for (int i = 0; i + m <= 2 * kDeg; ++i) C[i + m] ^= B[i];
      L = nn + 1 - L;
      B = T;
      m = 1;
    } else {
      for (int i = 0; i + m <= 2 * kDeg; ++i) C[i + m] ^= B[i];
      ++m;
    }
  }
  if (L != kDeg) throw std::runtime_error("xoshiro256 characteristic polynomial: unexpected linear complexity");
  // p(x) = x^L C(1/x)
  Poly p{};
  for (int i = 0; i <= L; ++i)
    if (C[i]) set_bit(p, L - i);
  return p;
}

const Poly& poly_p() {
  static const Poly p = char_poly();
  return p;
}

// a * b mod p, deg a, deg b < 256
Poly mulmod(const Poly& a, const Poly& b) {
  Poly r{};
  for (int i = 0; i < kDeg; ++i) {
    if (!bit(a, i)) continue;
    // r ^= b << i
    const int ws = i >> 6, bs = i & 63;
    for (int w = kWords - 1; w >= 0; --w) {
      uint64_t v = 0;
      if (w - ws >= 0) v = b[w - ws] << bs;
      if (bs && w - ws - 1 >= 0) v |= b[w - ws - 1] >> (64 - bs);
      r[w] ^= v;
    }
  }
  const Poly& p = poly_p();
  for (int dgr = degree(r); dgr >= kDeg; dgr = degree(r)) {
    const int sh = dgr - kDeg, ws = sh >> 6, bs = sh & 63;
    for (int w = kWords - 1; w >= 0; --w) {
      uint64_t v = 0;
      if (w - ws >= 0) v = p[w - ws] << bs;
      if (bs && w - ws - 1 >= 0) v |= p[w - ws - 1] >> (64 - bs);
      r[w] ^= v;
    }
  }
  return r;
}

}  // namespace

std::array<uint64_t, 4> stream_jump_poly(uint64_t draws) {
  Poly r{}, x{};
  set_bit(r, 0);  // 1
  set_bit(x, 1);  // x
  for (uint64_t d = draws; d; d >>= 1) {
    if (d & 1u) r = mulmod(r, x);
    x = mulmod(x, x);
  }
  return {r[0], r[1], r[2], r[3]};
}

void stream_jump(Stream& st, const std::array<uint64_t, 4>& poly) {
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int w = 0; w < 4; ++w)
    for (int b = 0; b < 64; ++b) {
      if ((poly[w] >> b) & 1u) {
        a0 ^= st.w0;
        a1 ^= st.w1;
        a2 ^= st.w2;
        a3 ^= st.w3;
      }
      st.u64();
    }
  st.w0 = a0;
  st.w1 = a1;
  st.w2 = a2;
  st.w3 = a3;
}

}  // namespace ldpcb
