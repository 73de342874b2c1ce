// clear_backend.hpp -- TEST INFRASTRUCTURE: the semantic oracle for the
// SlotOps kernels.  A cleartext SlotBackend restating the reference's
// ReferenceBackend (reference_backend.hpp:17-48, reference_backend.cpp:18-139):
// payloads are double slot vectors, level / scale / rotation-key bookkeeping
// and OpTrace records follow the reference exactly.  Used only by the C++ test
// driver tests/cpp/test_linalg_clear.cpp; never linked into the product.
#pragma once

#include "helix/backend.hpp"

namespace helix_oracle {

class ClearBackend final : public helix::SlotBackend {
 public:
  explicit ClearBackend(helix::CkksParams p);

  const helix::CkksParams& params() const override { return params_; }
  helix::OpTrace& trace() override { return trace_; }
  const helix::RotationKeySet& rotation_keys() const override { return keys_; }
  void generate_rotation_keys(std::span<const std::int64_t> amounts) override;

  helix::Plaintext encode(std::span<const double> m, int level, const helix::Scale& scale) override;
  std::vector<double> decode(const helix::Plaintext& pt) override;
  helix::Ciphertext encrypt(const helix::Plaintext& pt) override;
  std::vector<double> decrypt(const helix::Ciphertext& ct) override;

  helix::Ciphertext add(const helix::Ciphertext& a, const helix::Ciphertext& b) override;
  helix::Ciphertext add_plain(const helix::Ciphertext& a, const helix::Plaintext& b) override;
  helix::Ciphertext mul(const helix::Ciphertext& a, const helix::Ciphertext& b) override;
  helix::Ciphertext mul_plain(const helix::Ciphertext& a, const helix::Plaintext& b) override;
  helix::Ciphertext rotate(const helix::Ciphertext& a, std::int64_t k) override;
  helix::Ciphertext rescale(const helix::Ciphertext& a) override;
  helix::Ciphertext mod_down(const helix::Ciphertext& a, int target_level) override;
  helix::Ciphertext bootstrap(const helix::Ciphertext& a) override;

 private:
  struct Slots;
  const std::vector<double>& of(const helix::Ciphertext& c) const;
  const std::vector<double>& ofp(const helix::Plaintext& p) const;
  helix::Ciphertext make(std::vector<double> v, int level, helix::Scale s) const;

  helix::CkksParams params_;
  helix::OpTrace trace_;
  helix::RotationKeySet keys_;
};

}  // namespace helix_oracle
