// helix/linalg.hpp -- encrypted linear-algebra entry points (
// the reference's src/kernels.cpp is listed in proj/CMakeLists.txt:22 but
// absent).  Written against SlotOps only, so they run on any backend; on the
// B200 backend (GpuLatticeBackend) matvec_bsgs dispatches to the fused device
// pipeline (hoisted baby steps, one streaming diagonal-MAC launch, batched
// giant-step rotations) while recording exactly the same OpTrace counts.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "helix/backend.hpp"
#include "helix/packing.hpp"

namespace helix {

// SPEC.md:353-356
struct KernelReport {
  std::uint64_t rotations = 0, pt_muls = 0, ct_muls = 0, adds = 0;
  int levels_consumed = 0;
  Scale output_scale;
  std::string to_json() const;
};

// Plaintext payloads of a PackedMatrix encoded at one level (encode once,
// apply many times).  Diagonal layouts are encoded at scale q_level so that
// the kernel's final rescale restores the input scale.
struct EncodedMatrix {
  PackedMatrix meta;  // layout / dims (payload vectors dropped)
  int level = 0;
  std::vector<Plaintext> pts;  // null payload = zero
};

EncodedMatrix encode_matrix(SlotOps& ops, const PackedMatrix& M, int level);

// Giant-step shard of a BSGS transform (multi-GPU): only the
// diagonals of giant groups j in [giant_begin, giant_end) are encoded /
// applied; `rescale = false` returns the pre-rescale partial sum so that the
// shards' partials can be added exactly (NCCL uint64 sum + hx_reduce_mod_q)
// before the single final rescale.
struct BsgsShard {
  int giant_begin = 0;
  int giant_end = -1;  // -1: n2
  bool rescale = true;
};
EncodedMatrix encode_matrix(SlotOps& ops, const PackedMatrix& M, int level, const BsgsShard& shard);
// the shard of giant groups owned by `rank` of `world` (contiguous split)
BsgsShard bsgs_shard(const BsgsPlan& plan, int rank, int world);

// log2(span) rotate-adds at strides stride * 2^i
Ciphertext rotate_and_sum(SlotOps& ops, const Ciphertext& ct, std::size_t span, std::size_t stride,
                          KernelReport* report = nullptr);

// Rotation count the kernel records for a DENSE rows x cols matrix at `slots`
// slots, from the packing alone (no ciphertext work): the counters-only form
// of SPEC acceptance criterion 4.  Row: groups log2(pad_cols) +
// rows with a nonzero assembly shift; diag: d - 1; BSGS: (n1 - 1) +
// blocks (n2 - 1).
std::int64_t predicted_rotations(Layout layout, int rows, int cols, std::size_t slots);

// Matrix-vector products; x replicated at period d (packing.hpp).  One output
// ciphertext per row block (one for a single-block matrix).
struct MatvecResult {
  std::vector<Ciphertext> outputs;
  KernelReport report;
};
MatvecResult matvec_bsgs(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x);
MatvecResult matvec_bsgs(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x, const BsgsShard& shard);
// T input ciphertexts (tokens) through one BSGS matrix; on the GPU backend the
// key switches of all tokens are batched (hoisted baby steps over T inputs,
// giant steps grouped by key over T x blocks).  Same outputs and trace as T
// separate matvec_bsgs calls.
std::vector<MatvecResult> matvec_bsgs_tokens(SlotOps& ops, const EncodedMatrix& M, const std::vector<Ciphertext>& xs);
MatvecResult matvec_diag(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x);
// packed-row method: y in the first R slots; 2 levels
MatvecResult matvec_row(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x);

// SPEC signatures (single output block)
std::pair<Ciphertext, KernelReport> matvec_bsgs(SlotOps& ops, const PackedMatrix& M, const Ciphertext& x,
                                                const BsgsPlan& plan);
std::pair<Ciphertext, KernelReport> matvec_diag(SlotOps& ops, const PackedMatrix& M, const Ciphertext& x);
std::pair<Ciphertext, KernelReport> matvec_row(SlotOps& ops, const PackedMatrix& M, const Ciphertext& x);

// ct-ct matmul of row-major d x d operands: 2d pt-muls,
// d ct-muls, 2d(1 + log2 d) - 2 rotations, 2 levels.
std::pair<Ciphertext, KernelReport> matmul_ctct(SlotOps& ops, const Ciphertext& A, const Ciphertext& B,
                                                int d);

// rotation amounts each method needs
std::vector<std::int64_t> bsgs_rotations(const BsgsPlan& plan);
std::vector<std::int64_t> diag_rotations(int d);
std::vector<std::int64_t> row_rotations(const PackedMatrix& M);
std::vector<std::int64_t> matmul_rotations(int d, std::size_t slots);

// polyeval: slot-wise p(x) = sum_i c_i x^i (Power) or
// sum_i c_i T_i(y), y = (2x - (a + b)) / (b - a) (Chebyshev on [a, b]).
// Depth-optimal baby-step / giant-step split p = lo + X_h hi, h = 2^(m-1),
// X_h = x^h (Power) or T_h(y) (Chebyshev, division by T_h via
// T_h T_j = (T_(h+j) + T_|h-j|) / 2).  Every coefficient multiplication is a
// plaintext product whose encoding scale is chosen so that each partial
// result lands on an exact target scale: the output scale is exactly Delta.
// Levels consumed: ceil(log2(#coeffs)) (min 1), +1 for the Chebyshev domain
// map.  LevelUnderflowError when the input level is too low.
enum class PolyBasis { Power, Chebyshev };
Ciphertext polyeval(SlotOps& ops, const Ciphertext& x, const std::vector<double>& coeffs, PolyBasis basis,
                    double a = -1.0, double b = 1.0, KernelReport* report = nullptr);
// levels polyeval consumes for `n_coeffs` coefficients
int polyeval_depth(std::size_t n_coeffs, PolyBasis basis);

}  // namespace helix
