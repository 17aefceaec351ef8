// MT19937-64 with jump-ahead, output-compatible with std::mt19937_64 (the engine behind the
// reference's Rng, rng.hpp:15-61).  The probe streams of kpm_dos / lan_dos (dos.hpp:96-110) are
// draws [l n, (l+1) n) of ONE stream; jump-ahead lets several host threads (or ranks) start
// their share of that stream directly instead of drawing everything before it.
//
// Jumps use the characteristic polynomial phi (degree 19937) of the generator's linear state
// transition F, found once per process by Berlekamp-Massey on an output bit sequence; advancing
// J outputs applies g(F) with g = x^J mod phi (Horner, 19937 window shifts).
#pragma once

#include <cstdint>
#include <vector>

namespace se {

class Mt64 {
 public:
  static constexpr int kN = 312, kM = 156;
  explicit Mt64(std::uint64_t seed = 5489u);
  std::uint64_t operator()() {
    if (pos_ >= kN) refill();
    return temper(x_[kN + pos_++]);
  }
  // Advance by J outputs (J >= 0) using g = x^J mod phi (from jump_poly(J)).
  void jump(const std::vector<std::uint64_t>& g);
  void discard(std::uint64_t j);  // jump_poly(j) + jump for large j, else stepping

  static std::uint64_t temper(std::uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
  }

 private:
  void refill();  // window x_[pos_ .. pos_+311] -> x_[0..311], recompute x_[312..623]
  // x_[pos_ .. pos_ + 311]: the 312 raw words preceding the next output word x_[312 + pos_]
  std::uint64_t x_[2 * kN];
  int pos_ = 0;
};

// x^J mod phi as 312 little-endian words (bit i = coefficient of x^i); cached per J.
const std::vector<std::uint64_t>& jump_poly(std::uint64_t j);
// (a * b) mod phi
std::vector<std::uint64_t> poly_mulmod(const std::vector<std::uint64_t>& a,
                                       const std::vector<std::uint64_t>& b);
int mt64_phi_degree();  // 19937 (sanity)

}  // namespace se
