// helix/ntt.hpp -- negacyclic NTT tables (API of the reference's
// include/helix/ntt.hpp:19-52), executed on the B200.
//
// NttTables keeps the reference's contract: forward() leaves the bit-reversed
// layout out[k] = a(psi^(2 brv(k) + 1)) with the reference's psi (the root
// search of ntt.cpp:23-32, repeated here on the host), inverse() restores
// natural order and applies 1/n.  The transforms themselves run in
// libhx_b200 (hx_ntt_fwd / hx_ntt_inv on a one-prime device context created
// on first use); there is no host NTT.  n must be a power of two in
// [2^8, 2^16] (the device kernels' range).
#pragma once

#include <cstddef>
#include <memory>
#include <span>
#include <vector>

#include "helix/modmath.hpp"

namespace helix {

namespace detail {
struct DeviceNtt;  // lazily created one-prime hx_ctx + staging buffer
}

class NttTables {
 public:
  NttTables() = default;
  // q prime, q = 1 (mod 2n); n a power of two in [2^8, 2^16]
  NttTables(Modulus modulus, std::size_t n);

  std::size_t n() const { return n_; }
  const Modulus& modulus() const { return mod_; }
  u64 psi() const { return psi_; }

  // in place, a.size() == n (std::invalid_argument otherwise)
  void forward(std::span<u64> a) const;
  void inverse(std::span<u64> a) const;

  // c = a * b mod (X^n + 1, q), coefficient (natural) order
  std::vector<u64> negacyclic_mul(std::span<const u64> a, std::span<const u64> b) const;

 private:
  Modulus mod_;
  std::size_t n_ = 0;
  u64 psi_ = 0;
  mutable std::shared_ptr<detail::DeviceNtt> dev_;  // created on first transform, shared by later copies
};

// psi of the reference's root search (ntt.cpp:23-32): g = smallest integer >= 2
// with (g^((q-1)/2n))^n = -1, psi = g^((q-1)/2n)
u64 find_psi(const Modulus& q, std::size_t n);

// O(n^2) schoolbook product mod (X^n + 1, q) -- the reference's test oracle
// (ntt.cpp:109-125, "used by tests"); host code by definition, never on the
// product path.
std::vector<u64> schoolbook_negacyclic_mul(std::span<const u64> a, std::span<const u64> b, const Modulus& mod);

}  // namespace helix
