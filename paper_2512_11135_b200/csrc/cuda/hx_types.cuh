// hx_types.cuh -- argument structs shared between translation units.
#pragma once

#include "hx_common.cuh"

namespace hx {

// Shoup constant pair
struct SC {
  u64 w, wp;
};

// ------------------------------------------------------------ BSGS MAC
// inner_j = sum_k diag[j n1 + k] (.) baby_k for both ciphertext polys
// (the mul_acc loop of matvec_bsgs).  A CTA owns a tile of
// TT coefficients of one limb; the n1 baby-step words (2 polys) of the tile
// are staged in shared memory once and every diagonal word is streamed from
// HBM exactly once, accumulated lazily in 128 bits, reduced once per output.
struct MacArgs {
  u64* inner;        // [n2][2][n_q][N]
  const u64* baby;   // [n1][2][n_q][N]
  const u64* diags;  // [n2*n1][n_q][N]
  const PrimeConst* pc;
  int n1, n2, n_q, logn;
  long long diag_stride;  // words between consecutive diagonals
};

void launch_bsgs_mac(const MacArgs& A, long long N, cudaStream_t s);

}  // namespace hx
