// helix/modmath.hpp -- 64-bit prime-field scalars on the host (API of the
// reference's include/helix/modmath.hpp:21-152: Modulus, shoup_precompute,
// mul_shoup, is_prime_u64, find_ntt_primes).
//
// Host-side setup arithmetic only (parameter validation, root search,
// constants); every bulk operation on polynomials runs on the B200 through
// libhx_b200.  Unlike the reference, Modulus::mul is exact for all
// a, b < q < 2^63: the reference seeds its Barrett constant with `rem = 0`
// (modmath.hpp:30), which makes every product >= 2^64 wrong;
// here the product is reduced from its full 128 bits.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace helix {

using u64 = std::uint64_t;
using u128 = unsigned __int128;

struct Modulus {
  u64 q = 0;

  Modulus() = default;
  explicit Modulus(u64 value) : q(value) {
    if (q < 2) throw std::invalid_argument("Modulus: q < 2");
    if (q >> 63) throw std::invalid_argument("Modulus: q >= 2^63");
  }

  u64 add(u64 a, u64 b) const {
    const u64 s = a + b;
    return s >= q ? s - q : s;
  }
  u64 sub(u64 a, u64 b) const { return a >= b ? a - b : a + (q - b); }
  u64 neg(u64 a) const { return a ? q - a : 0; }
  u64 mul(u64 a, u64 b) const { return (u64)(((u128)a * b) % q); }
  u64 pow(u64 base, u64 exp) const {
    u64 r = 1 % q, b = base % q;
    for (; exp; exp >>= 1) {
      if (exp & 1) r = mul(r, b);
      b = mul(b, b);
    }
    return r;
  }
  // a^-1 for prime q (Fermat)
  u64 inv(u64 a) const {
    if (a % q == 0) throw std::invalid_argument("Modulus::inv(0)");
    return pow(a, q - 2);
  }
  // representative in (-q/2, q/2]
  std::int64_t centered(u64 a) const { return a > q / 2 ? (std::int64_t)a - (std::int64_t)q : (std::int64_t)a; }
  u64 reduce_i64(std::int64_t v) const {
    const std::int64_t m = v % (std::int64_t)q;
    return (u64)(m < 0 ? m + (std::int64_t)q : m);
  }
};

// Shoup companion floor(w 2^64 / q) of a fixed operand w < q, and a w mod q
// from it (result in [0, q))
inline u64 shoup_precompute(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
inline u64 mul_shoup(u64 a, u64 w, u64 wp, u64 q) {
  const u64 qt = (u64)(((u128)a * wp) >> 64);
  const u64 r = a * w - qt * q;
  return r >= q ? r - q : r;
}

// deterministic Miller-Rabin for 64-bit n
bool is_prime_u64(u64 n);
// first `count` primes p = 1 (mod two_n) at or above `start`, skipping `exclude`
std::vector<u64> find_ntt_primes(u64 start, std::size_t count, u64 two_n, const std::vector<u64>& exclude = {});

}  // namespace helix
