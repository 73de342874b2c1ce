// helix/encoder.hpp -- canonical CKKS slot encoding on the host (API shape of
// the reference's include/helix/encoder.hpp:20-53).
//
// Slot j <-> zeta^(5^j mod 2N).  encode: conjugate-symmetric evaluation
// vector -> inverse FFT -> untwist by zeta^-t -> x scale -> llround, exactly
// the operation order of encoder.cpp:45-117 (so the integer coefficients are
// bit-identical to the reference's).  The RNS reduction and NTT happen on the
// device (hx_from_i64 + hx_ntt_fwd); decode takes RNS limbs back from the
// device and reconstructs centred integers with a Garner mixed-radix CRT
// (no GMP) before the forward FFT.
#pragma once

#include <complex>
#include <cstdint>
#include <span>
#include <vector>

#include "helix/params.hpp"
#include "helix/rns_poly.hpp"

namespace helix {

class CkksEncoder {
 public:
  explicit CkksEncoder(const CkksParams& params);
  // the reference's constructor (encoder.hpp:22): encode() then returns RNS
  // limbs lifted on the context's device (LatticeContext::from_i64)
  explicit CkksEncoder(const LatticeContext& ctx);

  // the reference's encode / decode (encoder.cpp:97-159): coefficient-domain
  // RnsPoly over q_0..q_level; decode needs a coefficient-domain poly without
  // the special limb (std::invalid_argument otherwise)
  RnsPoly encode(std::span<const double> m, int level, double scale) const;
  std::vector<double> decode(const RnsPoly& pt, double scale) const;

  // round(scale * inverse-embedding(m)), m zero-padded to n slots.
  // std::invalid_argument: |m| > n, scale <= 0, level out of range;
  // std::overflow_error: a coefficient exceeds the level's modulus capacity.
  std::vector<std::int64_t> encode_coeffs(std::span<const double> m, int level, double scale) const;

  // limbs: coefficient-domain residues [n_limbs][N] over q_0..q_{n_limbs-1}
  std::vector<double> decode_coeffs(std::span<const std::uint64_t> limbs, int n_limbs,
                                    double scale) const;

  struct Embedding {
    std::vector<double> coefficients;
    double max_imag_residue;
  };
  Embedding embed_real(std::span<const double> m) const;

  // Tables of the device encoder (hx_encoder_create, include/hx_b200.h), all
  // computed here on the host with the same libm calls and recurrences as
  // encode_coeffs so the device result is bit-identical:
  //   perm[i]     = slot j whose value lands at position i after the FFT's bit
  //                 reversal, | 1<<31 when it is the conjugate mirror;
  //   stage_tw    = for len = 2, 4, ..., N the len/2 inverse-FFT twiddles
  //                 (w_0 = 1, w_{j+1} = w_j * wn), interleaved re/im;
  //   zeta        = zeta^t, t < N, interleaved re/im.
  void device_tables(std::vector<std::int32_t>& perm, std::vector<double>& stage_tw,
                     std::vector<double>& zeta) const;
  // log2(Q_level / 2): the capacity bound of encode_coeffs
  double capacity_log2(int level) const;

  std::size_t slot_count() const { return n_slots_; }
  std::size_t ring_degree() const { return n_; }

 private:
  void fft(std::vector<std::complex<double>>& v, bool inverse) const;
  std::vector<std::complex<double>> embed(std::span<const double> m) const;

  CkksParams params_;
  const LatticeContext* ctx_ = nullptr;
  std::size_t n_, n_slots_;
  int log_n_ = 0;
  std::vector<std::size_t> slot_to_eval_;
  std::vector<std::complex<double>> zeta_;
  std::vector<std::size_t> bitrev_;
  // Garner constants: inv_[j][k] = q_j^-1 mod q_k (j < k)
  std::vector<std::vector<std::uint64_t>> inv_;
};

}  // namespace helix
