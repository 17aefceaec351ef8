#include "mt64.hpp"

#include <immintrin.h>

#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

namespace se {

namespace {

constexpr std::uint64_t kUM = 0xFFFFFFFF80000000ULL;  // upper 33 bits
constexpr std::uint64_t kLM = 0x7FFFFFFFULL;          // lower 31 bits
constexpr std::uint64_t kA = 0xB5026F5AA96619E9ULL;   // twist matrix row

inline std::uint64_t twist(std::uint64_t a, std::uint64_t b) {
  const std::uint64_t y = (a & kUM) | (b & kLM);
  return (y >> 1) ^ ((y & 1u) ? kA : 0u);
}

// x[312 + i] = x[156 + i] ^ twist(x[i], x[i + 1]), i = 0..311, in order (the std in-place twist)
inline void extend(std::uint64_t* x) {
  for (int i = 0; i < Mt64::kN; ++i) x[Mt64::kN + i] = x[Mt64::kM + i] ^ twist(x[i], x[i + 1]);
}

// ---- GF(2) polynomials: little-endian 64-bit words ------------------------------------------
using Poly = std::vector<std::uint64_t>;

inline void clmul_soft(std::uint64_t a, std::uint64_t b, std::uint64_t& lo, std::uint64_t& hi) {
  lo = hi = 0;
  for (int i = 0; i < 64; ++i)
    if ((b >> i) & 1u) {
      lo ^= a << i;
      if (i) hi ^= a >> (64 - i);
    }
}

__attribute__((target("pclmul,sse4.1"))) void mul_words_hw(const std::uint64_t* a, int na,
                                                          const std::uint64_t* b, int nb,
                                                          std::uint64_t* r) {
  for (int i = 0; i < na; ++i) {
    if (!a[i]) continue;
    const __m128i av = _mm_set_epi64x(0, (long long)a[i]);
    for (int j = 0; j < nb; ++j) {
      const __m128i p = _mm_clmulepi64_si128(av, _mm_set_epi64x(0, (long long)b[j]), 0x00);
      r[i + j] ^= (std::uint64_t)_mm_cvtsi128_si64(p);
      r[i + j + 1] ^= (std::uint64_t)_mm_extract_epi64(p, 1);
    }
  }
}

void mul_words(const std::uint64_t* a, int na, const std::uint64_t* b, int nb, std::uint64_t* r) {
  static const bool hw = __builtin_cpu_supports("pclmul") && __builtin_cpu_supports("sse4.1");
  if (hw) return mul_words_hw(a, na, b, nb, r);
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < nb; ++j) {
      std::uint64_t lo, hi;
      clmul_soft(a[i], b[j], lo, hi);
      r[i + j] ^= lo;
      r[i + j + 1] ^= hi;
    }
}

inline bool bit(const Poly& p, long i) { return (p[(size_t)(i >> 6)] >> (i & 63)) & 1u; }

struct Phi {
  int L = 0;       // degree
  int W = 0;       // words of a reduced polynomial (degree < L)
  Poly phi;        // monic, degree L
  std::vector<Poly> sh;  // phi << s, s = 0..63
};

// Berlekamp-Massey over GF(2) on the low output bit; phi = reciprocal of the connection poly.
Phi make_phi() {
  constexpr int kExpect = 19937;
  const int N = 2 * kExpect + 128;
  Mt64 g(5489u);
  const int NW = (N + 63) / 64 + 2;
  Poly rev((size_t)NW + 2, 0);  // rev bit k = s_{N-1-k}
  for (int q = 0; q < N; ++q)
    if (g() & 1u) {
      const int k = N - 1 - q;
      rev[(size_t)(k >> 6)] |= 1ULL << (k & 63);
    }
  const int CW = NW + 2;
  Poly C((size_t)CW, 0), B((size_t)CW, 0), T;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  auto window = [&](int off, int w) -> std::uint64_t {  // rev bits [off + 64 w, ...)
    const long b0 = (long)off + 64L * w;
    const size_t wi = (size_t)(b0 >> 6);
    const int s = (int)(b0 & 63);
    std::uint64_t v = wi < rev.size() ? rev[wi] >> s : 0;
    if (s && wi + 1 < rev.size()) v |= rev[wi + 1] << (64 - s);
    return v;
  };
  for (int n = 0; n < N; ++n) {
    // d = sum_{i=0..L} C_i s_{n-i}; s_{n-i} = rev bit (N-1-n+i)
    const int off = N - 1 - n;
    std::uint64_t acc = 0;
    const int words = L / 64 + 1;
    for (int w = 0; w < words; ++w) {
      std::uint64_t cw = C[(size_t)w];
      if (w == words - 1) {
        const int top = L - 64 * w;  // bits 0..top valid
        if (top < 63) cw &= (2ULL << top) - 1;
      }
      acc ^= cw & window(off, w);
    }
    if (!(__builtin_popcountll(acc) & 1)) {
      ++m;
      continue;
    }
    // C ^= B << m
    auto add_shift = [&](Poly& dst, const Poly& src, int sh) {
      const int ws = sh >> 6, bs = sh & 63;
      for (int w = CW - 1; w >= 0; --w) {
        const int s0 = w - ws;
        if (s0 < 0) break;
        std::uint64_t v = src[(size_t)s0] << bs;
        if (bs && s0 >= 1) v |= src[(size_t)s0 - 1] >> (64 - bs);
        dst[(size_t)w] ^= v;
      }
    };
    if (2 * L <= n) {
      T = C;
      add_shift(C, B, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      add_shift(C, B, m);
      ++m;
    }
  }
  if (L != kExpect) throw std::runtime_error("mt64: unexpected characteristic polynomial degree");
  Phi p;
  p.L = L;
  p.W = (L + 63) / 64;
  p.phi.assign((size_t)p.W + 1, 0);
  for (int k = 0; k <= L; ++k)  // phi_k = C_{L-k}
    if (bit(C, L - k)) p.phi[(size_t)(k >> 6)] |= 1ULL << (k & 63);
  p.sh.resize(64);
  for (int s = 0; s < 64; ++s) {
    Poly q((size_t)p.W + 2, 0);
    for (int w = 0; w <= p.W; ++w) {
      q[(size_t)w] ^= p.phi[(size_t)w] << s;
      if (s) q[(size_t)w + 1] ^= p.phi[(size_t)w] >> (64 - s);
    }
    p.sh[(size_t)s] = std::move(q);
  }
  return p;
}

const Phi& phi() {
  static const Phi p = make_phi();
  return p;
}

// reduce r (any length) mod phi in place; returns W words
Poly reduce(Poly r) {
  const Phi& P = phi();
  const long top = (long)r.size() * 64 - 1;
  r.resize(r.size() + P.W + 3, 0);
  for (long t = top; t >= P.L; --t) {
    if (!bit(r, t)) continue;
    const long off = t - P.L;
    const size_t ws = (size_t)(off >> 6);
    const Poly& s = P.sh[(size_t)(off & 63)];
    for (size_t w = 0; w < s.size(); ++w) r[ws + w] ^= s[w];
  }
  r.resize((size_t)P.W);
  return r;
}

}  // namespace

Poly poly_mulmod(const Poly& a, const Poly& b) {
  Poly r(a.size() + b.size() + 1, 0);
  mul_words(a.data(), (int)a.size(), b.data(), (int)b.size(), r.data());
  return reduce(std::move(r));
}

int mt64_phi_degree() { return phi().L; }

const Poly& jump_poly(std::uint64_t j) {
  static std::mutex mu;
  static std::map<std::uint64_t, Poly> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(j);
    if (it != cache.end()) return it->second;
  }
  const Phi& P = phi();
  Poly r((size_t)P.W, 0);
  r[0] = 1;
  for (int b = 63; b >= 0; --b) {
    const bool any = (j >> b) != 0;
    if (!any) continue;
    r = poly_mulmod(r, r);
    if ((j >> b) & 1u) {  // r *= x
      std::uint64_t carry = 0;
      for (size_t w = 0; w < r.size(); ++w) {
        const std::uint64_t nc = r[w] >> 63;
        r[w] = (r[w] << 1) | carry;
        carry = nc;
      }
      Poly t = r;
      t.push_back(carry);
      r = reduce(std::move(t));
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  return cache.emplace(j, std::move(r)).first->second;
}

Mt64::Mt64(std::uint64_t seed) {
  x_[0] = seed;
  for (int i = 1; i < kN; ++i) x_[i] = 6364136223846793005ULL * (x_[i - 1] ^ (x_[i - 1] >> 62)) + (std::uint64_t)i;
  extend(x_);
  pos_ = 0;
}

void Mt64::refill() {
  std::memmove(x_, x_ + pos_, sizeof(std::uint64_t) * kN);
  extend(x_);
  pos_ = 0;
}

void Mt64::jump(const Poly& g) {
  // Horner on the window: acc = g(F) W, F = shift the window by one generated word
  std::uint64_t w0[kN], c[kN];
  std::memcpy(w0, x_ + pos_, sizeof(w0));
  std::memset(c, 0, sizeof(c));
  int s = 0;  // logical index 0 of c at physical s
  long deg = (long)g.size() * 64 - 1;
  while (deg >= 0 && !bit(g, deg)) --deg;
  for (long i = deg; i >= 0; --i) {
    // F: new = c[156] ^ twist(c[0], c[1]) replaces logical 0
    const std::uint64_t a = c[s], b = c[s + 1 < kN ? s + 1 : s + 1 - kN];
    const int m = s + kM < kN ? s + kM : s + kM - kN;
    c[s] = c[m] ^ twist(a, b);
    s = s + 1 < kN ? s + 1 : 0;
    if (bit(g, i)) {
      const int h = kN - s;  // logical j < h at physical s + j
      for (int j = 0; j < h; ++j) c[s + j] ^= w0[j];
      for (int j = h; j < kN; ++j) c[j - h] ^= w0[j];
    }
  }
  for (int j = 0; j < kN; ++j) x_[j] = c[(s + j) % kN];
  extend(x_);
  pos_ = 0;
}

void Mt64::discard(std::uint64_t j) {
  if (j < (1ULL << 24)) {
    for (std::uint64_t q = 0; q < j; ++q) (*this)();
    return;
  }
  jump(jump_poly(j));
}

}  // namespace se
