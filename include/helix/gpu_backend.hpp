// helix/gpu_backend.hpp -- the B200 lattice backend: a helix::SlotBackend whose
// ciphertexts and plaintexts live in HBM and whose operations call the
// sm_100a kernels of libhx_b200.so through the C-ABI (include/hx_b200.h).
//
// It implements the lattice backend the reference specifies but does not ship
// (proj/CMakeLists.txt:20 lists the missing
// src/lattice_backend.cpp) with hybrid key switching (alpha-limb digits, K
// special primes).  Level / scale / key bookkeeping and the OpTrace records
// are those of the reference backend (reference_backend.cpp:63-139), so every
// kernel written against SlotOps runs unchanged and reports identical counts.
//
// Beyond SlotOps it exposes the fused device pipelines the linear-transform
// entry points use (helix/linalg.hpp): hoisted multi-rotation, batched
// per-key rotation and the BSGS diagonal multiply-accumulate.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <vector>

#include "helix/backend.hpp"
#include "helix/encoder.hpp"

struct hx_ctx;
struct hx_encoder;

namespace helix {

// RAII device allocation (stream-ordered malloc/free on the backend stream)
struct DeviceBuffer {
  std::uint64_t* ptr = nullptr;
  std::size_t words = 0;
  // allocated and freed in the order of the CUDA stream of the backend whose
  // operation created it (null: the legacy default stream); the reference
  // keeps that stream alive while any of its buffers lives
  void* stream = nullptr;
  std::shared_ptr<void> stream_ref;
  // derived device representations of the (immutable) words, e.g. the
  // tensor-core operand tiles of a BSGS matrix's diagonals (hx_bsgs_tc_pack),
  // keyed by a signature of the shape and the diagonal offsets; they live
  // and die with this buffer
  std::mutex derived_mu;
  std::vector<std::pair<std::uint64_t, std::shared_ptr<DeviceBuffer>>> derived;
  explicit DeviceBuffer(std::size_t words);
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

// Ciphertext payload: [2][n_q][N] NTT-domain words at buf->ptr + offset.
struct GpuCiphertext final : CiphertextPayload {
  std::shared_ptr<DeviceBuffer> buf;
  std::size_t offset = 0;
  int n_q = 0;
  std::uint64_t* data() const { return buf->ptr + offset; }
};

// Plaintext payload: [n_q][N] NTT-domain words (a slice of a shared buffer
// when encoded in bulk with encode_many).
struct GpuPlaintext final : PlaintextPayload {
  std::shared_ptr<DeviceBuffer> buf;
  std::size_t offset = 0;
  int n_q = 0;
  std::uint64_t* data() const { return buf->ptr + offset; }
};

class GpuLatticeBackend final : public SlotBackend {
 public:
  explicit GpuLatticeBackend(CkksParams params, std::uint64_t seed = 0x48454c4958ull);
  ~GpuLatticeBackend() override;
  GpuLatticeBackend(const GpuLatticeBackend&) = delete;
  GpuLatticeBackend& operator=(const GpuLatticeBackend&) = delete;

  // ---- SlotOps / SlotBackend ----
  const CkksParams& params() const override { return params_; }
  OpTrace& trace() override { return trace_; }
  const RotationKeySet& rotation_keys() const override { return rot_set_; }
  void generate_rotation_keys(std::span<const std::int64_t> amounts) override;

  Plaintext encode(std::span<const double> m, int level, const Scale& scale) override;
  std::vector<double> decode(const Plaintext& pt) override;
  Ciphertext encrypt(const Plaintext& pt) override;
  std::vector<double> decrypt(const Ciphertext& ct) override;

  Ciphertext add(const Ciphertext& a, const Ciphertext& b) override;
  Ciphertext add_plain(const Ciphertext& a, const Plaintext& b) override;
  Ciphertext mul(const Ciphertext& a, const Ciphertext& b) override;
  Ciphertext mul_plain(const Ciphertext& a, const Plaintext& b) override;
  Ciphertext rotate(const Ciphertext& a, std::int64_t k) override;
  Ciphertext rescale(const Ciphertext& a) override;
  Ciphertext mod_down(const Ciphertext& a, int target_level) override;
  Ciphertext bootstrap(const Ciphertext& a) override;

  // ---- fused device pipelines (same trace records as the SlotOps form) ----
  // Encode many slot vectors into ONE contiguous device buffer; entries that
  // are empty vectors become null-payload plaintexts (exact zeros, skipped by
  // the BSGS MAC).
  std::vector<Plaintext> encode_many(const std::vector<std::vector<double>>& msgs, int level,
                                     const Scale& scale);
  // Rotations of one ciphertext sharing one ModUp (hoisting).  Output k is
  // Rot(a, amounts[k]); records one Rotate per nonzero amount.
  std::vector<Ciphertext> rotate_many(const Ciphertext& a, std::span<const std::int64_t> amounts);
  // BSGS block: y = sum_j Rot_{n1 j}(sum_k diag[j n1 + k] (.) baby_k), with
  // baby_k = Rot_k(x) for k < n1 (baby[0] = x).  Null-payload diagonals are
  // zero.  No rescale.  Records PtMul / CtAdd / Rotate exactly as
  // linalg.cpp's generic matvec_bsgs.
  Ciphertext bsgs_block(const std::vector<Ciphertext>& baby, const std::vector<Plaintext>& diags,
                        int n1, int n2);
  // All row blocks of a tiled matrix at once (diags: blocks x n1 n2 payloads):
  // per-block MAC launches write inner sums in [n2][blocks] order, then giant
  // step j of every block is rotated with one read of key n1 j
  // (hx_rotate_grouped) and summed in one pass.  Same trace as per-block.
  // The giant rotations share one ModDown per output (double hoisting,
  // hx_rotate_grouped_sum).  allow_empty (giant-step shards, linalg.hpp
  // BsgsShard): a block without live diagonals is no error, and each output
  // is a PQ-BASIS PARTIAL -- its buffer holds T ([2][n_q][N], the ciphertext
  // words the handle shows) followed by S ([2][n_q + K][N], the unreduced
  // key-switch sum); ranks sum both, then shard_finish() applies the ModDown.
  std::vector<Ciphertext> bsgs_blocks(const std::vector<Ciphertext>& baby,
                                      const std::vector<Plaintext>& diags, int n1, int n2, int blocks,
                                      bool allow_empty = false);
  // Token batch (SURVEY §8(d) config 3, T tokens through one matrix): baby
  // sets of T ciphertexts, MACs per (token, block), and giant step j of every
  // (token, block) pair rotated with ONE read of key n1 j (hx_rotate_grouped
  // over T x blocks elements).  Outputs [token][block]; trace = T single runs.
  std::vector<std::vector<Ciphertext>> bsgs_blocks_tokens(const std::vector<std::vector<Ciphertext>>& babies,
                                                          const std::vector<Plaintext>& diags, int n1, int n2,
                                                          int blocks, bool allow_empty = false);
  // hoisted rotations of T ciphertexts in one launch sequence (ModUp of all
  // T, then every amount): out[t][i] = Rot(xs[t], amounts[i])
  std::vector<std::vector<Ciphertext>> rotate_many_tokens(const std::vector<Ciphertext>& xs,
                                                          std::span<const std::int64_t> amounts);

  // ct x ct matmul (linalg.hpp matmul_ctct) with every step
  // batched over the d column / row extractions: 2 encode_many of the masks,
  // one mask product + rescale launch per operand, one multi-key rotation
  // (Rot_j / Rot_dj), log2(d) rounds of one shared-key rotation + add per
  // operand, d ct-ct products + relinearisation in one launch, one strided sum
  // and the final rescale.  Same trace records as the SlotOps form.
  Ciphertext matmul(const Ciphertext& A, const Ciphertext& B, int d);
  // H independent products (config 4's attention heads) in one schedule:
  // each rotation / relinearisation launch covers every head, so a key is
  // read once per H heads.  outs[h] = matmul(As[h], Bs[h], d) word for word.
  std::vector<Ciphertext> matmul_heads(const std::vector<Ciphertext>& As, const std::vector<Ciphertext>& Bs, int d);

  // y = T + (ModDown(S_0), ModDown(S_1)) of a summed PQ partial (words =
  // [T][S] as bsgs_blocks(allow_empty) lays them out), at like's level / scale
  Ciphertext shard_finish(const Ciphertext& like, const std::uint64_t* words);
  std::size_t shard_partial_words(int level) const {
    return (std::size_t)2 * (2 * nq(level) + params_.special_primes.size()) * params_.ring_degree;
  }

  // ---- raw access ----
  hx_ctx* device_context() const { return ctx_; }
  // release the device scratch arena and the pool's cached blocks (between
  // workloads of different shapes); serialised with the backend's operations
  void trim();
  const CkksEncoder& encoder() const { return enc_; }
  static const GpuCiphertext& payload(const Ciphertext& ct);
  static const GpuPlaintext& payload(const Plaintext& pt);
  Ciphertext wrap(std::shared_ptr<DeviceBuffer> buf, std::size_t offset, int level,
                  const Scale& scale) const;
  // full [dnum][2][full][N] words of a compressed key (rotation_key /
  // relin_key_words pointers) into device memory `full` -- for oracles
  void expand_key(const std::uint64_t* ckey, std::uint64_t* full) const;
  // device word pointer of the (compressed) rotation-layout key for amount k (mod n), or null
  const std::uint64_t* rotation_key(std::int64_t amount_mod_n) const;
  // secret key s over the full basis (NTT) and the relinearisation key --
  // exported for the parity tests (the oracle recomputes with the same words)
  const std::uint64_t* secret_key_words() const { return s_full_->ptr; }
  const std::uint64_t* relin_key_words() const { return rlk_->ptr; }

 private:
  std::uint64_t galois(std::int64_t amount_mod_n) const;
  std::uint64_t next_u64();
  void sample_uniform(std::vector<std::uint64_t>& out, int limbs_chain, int limbs_special, int copies);
  void sample_error(std::vector<std::int64_t>& out, int copies);
  std::shared_ptr<DeviceBuffer> make_key(const std::shared_ptr<DeviceBuffer>& sprime_or_null,
                                         std::uint64_t galois_elt);
  int nq(int level) const { return level + 1; }
  // device encoder (hx_encode): n messages -> NTT-domain plaintext words at out
  void encode_device(const std::vector<const std::vector<double>*>& msgs, int level, const Scale& scale,
                     std::uint64_t* out);

  // Concurrency model: every public operation holds mu_
  // (operations on one backend serialise; handles stay value-like) and
  // issues its work on this backend's own CUDA stream (blocking w.r.t. the
  // legacy default stream, so callers that use it stay ordered), so
  // operations of distinct backends run concurrently on the device
  struct DeviceScope;
  friend struct DeviceScope;
  mutable std::recursive_mutex mu_;
  std::shared_ptr<void> stream_;

  CkksParams params_;
  CkksEncoder enc_;
  OpTrace trace_;
  RotationKeySet rot_set_;
  hx_ctx* ctx_ = nullptr;
  hx_encoder* henc_ = nullptr;  // created on first encode
  // matmul extraction masks per (d, level): immutable plaintexts, encoded once
  std::map<std::pair<int, int>, std::pair<std::vector<Plaintext>, std::vector<Plaintext>>> matmul_masks_;
  std::uint64_t rng_[4];
  std::shared_ptr<DeviceBuffer> s_full_;  // [n_chain + K][N], NTT
  std::shared_ptr<DeviceBuffer> rlk_;     // relinearisation key (standard layout)
  std::map<std::int64_t, std::shared_ptr<DeviceBuffer>> rot_keys_;  // rotation layout
};

}  // namespace helix
