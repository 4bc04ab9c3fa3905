// mt_jump.cpp -- jump-ahead polynomials for std::mt19937_64 (host, GF(2)).
//
// The reference's Rng is std::mt19937_64 (proj/include/cnmf/rng.hpp:13-60),
// a linear recurrence over GF(2) with a primitive characteristic polynomial
// phi of degree 19937.  Advancing the raw word sequence by J positions is
// the linear map T^J = p(T) with p = x^J mod phi (Cayley-Hamilton), so the
// 312 state words at position s + J are XORs of the words at positions
// s + i, s + i + 1, ... over the set bits i of p.  This file computes phi
// once per process (Berlekamp-Massey on the low bit of the raw words) and
// the polynomials x^(k J) mod phi for the segment starts k J the device
// generator needs (carry-less products, Barrett reduction), cached per J.
// None of this depends on the seed.
#include <immintrin.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <vector>

#include "kernels.h"

namespace cnmf {
namespace {

constexpr int kDeg = 19937;
constexpr int kPolyWords = (kDeg + 64) / 64;  // 312: bits [0, kDeg)
using Poly = std::vector<uint64_t>;

// The raw (untempered) mt19937_64 words x_0, x_1, ... for a seed.
std::vector<uint64_t> raw_words(uint64_t seed, size_t count) {
  const int n = 312, m = 156;
  std::vector<uint64_t> x(count + n);
  x[0] = seed;
  for (int i = 1; i < n; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
  for (size_t i = 0; i + n < x.size(); ++i) {
    const uint64_t y = (x[i] & 0xFFFFFFFF80000000ULL) | (x[i + 1] & 0x7FFFFFFFULL);
    x[i + n] = x[i + m] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0ULL);
  }
  return x;
}

inline int deg_of(const Poly& p) {
  for (int w = (int)p.size() - 1; w >= 0; --w)
    if (p[w]) return 64 * w + 63 - __builtin_clzll(p[w]);
  return -1;
}

// Berlekamp-Massey over GF(2): connection polynomial of the bit sequence.
// The discrepancy s_n + sum_{i=1..L} c_i s_{n-i} is a word-parallel dot
// product of C with the bit-reversed sequence R (R_j = s_{N-1-j}, so
// s_{n-i} = R_{N-1-n+i}: a contiguous run of R starting at N-1-n).
Poly berlekamp_massey(const std::vector<uint8_t>& s) {
  const size_t N = s.size(), W = (N + 64) / 64;
  std::vector<uint64_t> C(W, 0), B(W, 0), T;
  std::vector<uint64_t> R(W + 2, 0);
  for (size_t j = 0; j < N; ++j)
    if (s[N - 1 - j]) R[j >> 6] |= 1ULL << (j & 63);
  auto rbits = [&](size_t pos) -> uint64_t {  // 64 bits of R starting at pos
    const size_t w = pos >> 6, b = pos & 63;
    uint64_t v = w < R.size() ? R[w] >> b : 0;
    if (b && w + 1 < R.size()) v |= R[w + 1] << (64 - b);
    return v;
  };
  C[0] = B[0] = 1;
  size_t L = 0;
  long m = 1;
  for (size_t n = 0; n < N; ++n) {
    const size_t base = N - 1 - n;  // bit i of (R >> base) is s_{n-i}
    uint64_t acc = 0;
    const size_t words = (L >> 6) + 1;
    for (size_t w = 0; w < words; ++w) acc ^= C[w] & rbits(base + 64 * w);
    // acc bit 0 is c_0 s_n = s_n; bits i <= L are c_i s_{n-i}; bits > L are 0 in C
    const uint8_t dbit = (uint8_t)(__builtin_popcountll(acc) & 1);
    if (!dbit) {
      ++m;
      continue;
    }
    T = C;
    // C ^= B << m
    const size_t ws = m >> 6, bs = m & 63;
    for (size_t i = W; i-- > 0;) {
      uint64_t v = 0;
      if (i >= ws) {
        v = B[i - ws] << bs;
        if (bs && i >= ws + 1) v |= B[i - ws - 1] >> (64 - bs);
      }
      C[i] ^= v;
    }
    if (2 * L <= n) {
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      ++m;
    }
  }
  // connection polynomial C(x) = 1 + c1 x + ... + cL x^L; the characteristic
  // polynomial is its reciprocal x^L C(1/x)
  Poly phi(kPolyWords + 1, 0);
  for (size_t i = 0; i <= L; ++i)
    if ((C[i >> 6] >> (i & 63)) & 1) {
      const size_t j = L - i;
      phi[j >> 6] |= 1ULL << (j & 63);
    }
  return phi;
}

// Carry-less product (PCLMULQDQ) of two polynomials of kPolyWords words.
void clmul(const uint64_t* a, int na, const uint64_t* b, int nb, uint64_t* out) {
  std::memset(out, 0, sizeof(uint64_t) * (na + nb));
  for (int i = 0; i < na; ++i) {
    if (!a[i]) continue;
    const __m128i ai = _mm_set_epi64x(0, (long long)a[i]);
    for (int j = 0; j < nb; ++j) {
      if (!b[j]) continue;
      const __m128i r = _mm_clmulepi64_si128(ai, _mm_set_epi64x(0, (long long)b[j]), 0x00);
      out[i + j] ^= (uint64_t)_mm_cvtsi128_si64(r);
      out[i + j + 1] ^= (uint64_t)_mm_extract_epi64(r, 1);
    }
  }
}

struct Field {
  Poly phi;   // degree kDeg
  Poly mu;    // floor(x^(2 kDeg) / phi), degree kDeg (Barrett)
  bool ok = false;

  // r = p mod phi for p of degree < 2 kDeg (array of 2 kPolyWords words).
  Poly reduce(const std::vector<uint64_t>& p) const {
    // q = floor(floor(p / x^kDeg) * mu / x^kDeg);  r = p - q phi
    const int W = 2 * kPolyWords + 2;
    std::vector<uint64_t> hi(kPolyWords + 1, 0), t(W + 2, 0), q(kPolyWords + 1, 0), qp(W + 2, 0);
    for (int i = 0; i < kPolyWords + 1; ++i) {
      const int bit = kDeg + 64 * i;
      const int w = bit >> 6, s = bit & 63;
      uint64_t v = w < (int)p.size() ? p[w] >> s : 0;
      if (s && w + 1 < (int)p.size()) v |= p[w + 1] << (64 - s);
      hi[i] = v;
    }
    clmul(hi.data(), kPolyWords + 1, mu.data(), kPolyWords + 1, t.data());
    for (int i = 0; i < kPolyWords + 1; ++i) {
      const int bit = kDeg + 64 * i;
      const int w = bit >> 6, s = bit & 63;
      uint64_t v = w < (int)t.size() ? t[w] >> s : 0;
      if (s && w + 1 < (int)t.size()) v |= t[w + 1] << (64 - s);
      q[i] = v;
    }
    clmul(q.data(), kPolyWords + 1, phi.data(), kPolyWords + 1, qp.data());
    Poly r(kPolyWords + 1, 0);
    for (int i = 0; i < kPolyWords + 1; ++i) r[i] = (i < (int)p.size() ? p[i] : 0) ^ qp[i];
    // at most one more subtraction of phi (Barrett error <= 1 multiple)
    if (deg_of(r) >= kDeg) {
      for (int i = 0; i < kPolyWords + 1; ++i) r[i] ^= phi[i];
    }
    return r;
  }
  Poly mulmod(const Poly& a, const Poly& b) const {
    std::vector<uint64_t> p(2 * kPolyWords + 4, 0);
    clmul(a.data(), kPolyWords + 1, b.data(), kPolyWords + 1, p.data());
    return reduce(p);
  }
};

const Field& field() {
  static Field f = [] {
    Field F;
    // phi from the low bit of raw words x_312 .. (generated words only)
    const std::vector<uint64_t> x = raw_words(5489u, 2 * kDeg + 400);
    std::vector<uint8_t> bits(2 * kDeg + 64);
    for (size_t i = 0; i < bits.size(); ++i) bits[i] = (uint8_t)(x[312 + i] & 1u);
    F.phi = berlekamp_massey(bits);
    if (deg_of(F.phi) != kDeg) return F;
    // mu = floor(x^(2 kDeg) / phi) by bit-serial long division
    std::vector<uint64_t> num(2 * kPolyWords + 2, 0);
    num[(2 * kDeg) >> 6] |= 1ULL << ((2 * kDeg) & 63);
    Poly q(kPolyWords + 2, 0);
    for (int b = 2 * kDeg; b >= kDeg; --b) {
      if (!((num[b >> 6] >> (b & 63)) & 1)) continue;
      const int sh = b - kDeg;
      q[sh >> 6] |= 1ULL << (sh & 63);
      const int ws = sh >> 6, bs = sh & 63;
      for (int i = 0; i < kPolyWords + 1; ++i) {
        const uint64_t v = F.phi[i];
        if (!v) continue;
        num[i + ws] ^= v << bs;
        if (bs) num[i + ws + 1] ^= v >> (64 - bs);
      }
    }
    F.mu.assign(q.begin(), q.begin() + kPolyWords + 1);
    F.ok = true;
    return F;
  }();
  return f;
}

Poly x_pow(uint64_t e) {  // x^e mod phi by square-and-multiply
  const Field& F = field();
  Poly r(kPolyWords + 1, 0), base(kPolyWords + 1, 0);
  r[0] = 1;
  base[0] = 2;  // x
  while (e) {
    if (e & 1) r = F.mulmod(r, base);
    e >>= 1;
    if (e) base = F.mulmod(base, base);
  }
  return r;
}

std::mutex g_mu;
std::map<uint64_t, std::vector<Poly>> g_cache;  // J -> [x^(kJ) mod phi, k = 0, 1, ...]

}  // namespace

bool mt_jump_available() { return field().ok; }

// x^(k J) mod phi for k = 0 .. K-1 as K x 312 words (bit i of word i/64 is
// the coefficient of x^i).  Cached per J; grows lazily.
bool mt_jump_polys(uint64_t J, int K, std::vector<uint64_t>& out) {
  const Field& F = field();
  if (!F.ok) return false;
  std::lock_guard<std::mutex> lock(g_mu);
  std::vector<Poly>& v = g_cache[J];
  if (v.empty()) {
    Poly one(kPolyWords + 1, 0);
    one[0] = 1;
    v.push_back(one);
  }
  if ((int)v.size() < K) {
    const Poly step = x_pow(J);
    while ((int)v.size() < K) v.push_back(F.mulmod(v.back(), step));
  }
  out.assign((size_t)K * kPolyWords, 0);
  for (int k = 0; k < K; ++k)
    std::memcpy(out.data() + (size_t)k * kPolyWords, v[k].data(), sizeof(uint64_t) * kPolyWords);
  return true;
}

}  // namespace cnmf
