// helix/params.hpp -- CKKS parameter set (API of the reference's
// include/helix/params.hpp:14-51), extended for hybrid key switching:
// any number of special primes and a digit size `alpha` (limbs per gadget
// digit; the reference spec's key switch is alpha = 1 with one special prime,
// SPEC.md:229).  BackendKind::Lattice selects the B200 lattice backend
// (helix::GpuLatticeBackend).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "helix/modmath.hpp"
#include "helix/scale.hpp"

namespace helix {

enum class BackendKind { Reference, Lattice };

struct CkksParams {
  std::uint64_t ring_degree = 0;  // N (power of two)
  int max_level = 0;              // L
  int delta_log2 = 0;             // Delta = 2^delta_log2
  std::vector<std::uint64_t> moduli;          // q_0 .. q_L
  std::vector<std::uint64_t> special_primes;  // p_0 .. p_{K-1}
  BackendKind backend = BackendKind::Reference;
  bool mock_bootstrap = true;
  bool insecure_toy = false;
  // GPU backend: store key-switching keys compressed (b halves only, the
  // uniform halves regenerated from a seed in the inner product; half the key
  // memory, slower key switches on B200 -- DESIGN.md 5).  Not part of the
  // reference's parameter set (an extension key of this implementation).
  bool compress_keys = false;
  int bootstrap_level = -1;  // L_boot, -1 = L
  int digit_size = 1;        // alpha (hybrid key switching), new

  std::uint64_t slot_count() const { return ring_degree / 2; }
  Scale delta() const { return Scale::pow2(delta_log2); }
  int l_boot() const { return bootstrap_level < 0 ? max_level : bootstrap_level; }

  // std::invalid_argument on: N not a power of two, L < 1, |moduli| != L+1,
  // a modulus not prime or != 1 mod 2N, L_boot > L, digit_size < 1.
  void validate() const;

  std::string to_json() const;
  static CkksParams from_json(const std::string& text);
  static CkksParams load(const std::string& path);
  void save(const std::string& path) const;

  static CkksParams toy_lattice();
  static CkksParams reference_default(std::uint64_t ring_degree = 1ull << 16, int max_level = 20);
  // BASELINE.json configs[0] / configs[1..4] parameter shapes
  static CkksParams config1();
  static CkksParams config2(std::uint64_t ring_degree = 1ull << 16, int chain_primes = 24);
};

// find_ntt_primes / is_prime_u64: helix/modmath.hpp (as in the reference)

}  // namespace helix
