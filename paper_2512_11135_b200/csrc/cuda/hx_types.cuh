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
  long long out_jstride;  // words between inner_j and inner_{j+1} (2 n_q N when packed)
  const int* limbs;       // device limb list for blockIdx.y (null: identity)
  // token batch: `tokens` baby sets at baby + t baby_tstride, inner sums at
  // inner + t inner_tstride; the token index varies fastest along blockIdx.x
  // (blocks of one coefficient tile and limb run back to back, so every
  // diagonal word comes from HBM once and from L2 for the other tokens)
  int tokens;
  long long baby_tstride, inner_tstride;
  // diagonals between giant groups j and j+1 (n1 for a whole block; larger when
  // the baby steps of a block are processed in chunks of at most 64)
  int diag_jstride;
};

// Sparse (pruned) BSGS MAC: the live diagonals of one row block as an index
// list grouped by giant step (CSR: group j owns entries [gptr[j], gptr[j+1])),
// entry e = baby index ks[e] and the device address dptr[e] of its [n_q][N]
// words.  inner_j is written for live groups only (dead ones keep the
// caller's zeros).
struct SparseMacArgs {
  u64* inner;
  const u64* baby;
  const int* gptr;
  const int* ks;
  const u64* const* dptr;
  const PrimeConst* pc;
  int n1, n2, n_q, logn, tokens;
  long long out_jstride, baby_tstride, inner_tstride;
};

// out = sum_{r < terms} in + r * term_stride, per (poly, limb) of `polys`
// polys of n_q limbs (ciphertext sums of the BSGS giant steps)
struct SumArgs {
  u64* out;
  const u64* in;
  const PrimeConst* pc;
  int terms, n_q, logn;
  long long term_stride, in_poly_stride, out_poly_stride;
};
void launch_sum(const SumArgs& A, int polys, long long N, cudaStream_t s);

// d_f64_limbs / d_int_limbs: device lists of the limbs (of 0..n_q-1) whose
// primes take the FP64 k-split kernel (q < 2^43) / the integer kernel
void launch_bsgs_mac(const MacArgs& A, long long N, cudaStream_t s, const int* d_f64_limbs, int n_f64,
                     const int* d_int_limbs, int n_int);

// ------------------------------------------------- packed (5-byte) BSGS MAC
// (hx_bsgs_p40.cu): limbs with q < 2^40 of one contiguous block of
// diagonals, packed once into the P40 layout, streamed by cp.async.bulk
constexpr int kP40MaxStages = 8;
struct P40Args {
  u64* inner;                   // inner_j at inner + j out_jstride ([2][n_q][N])
  const u64* baby;              // [n1][2][n_q][N]
  const unsigned char* packed;  // P40 layout [n_p40][N / 32][n2][5 n1 32 bytes]
  const int* limbs;             // P40 limb list (p -> chain limb i)
  const PrimeConst* pc;
  long long out_jstride;
  // rows r < n2 are (row block r / rpb, giant step r % rpb): inner sum at
  // inner + (r % rpb) out_jstride + (r / rpb) out_bstride (one block: rpb = n2)
  long long out_bstride;
  int rpb;
  int n1, n2, n_q, logn, stages;
};
int p40_stages(int n1);
void launch_bsgs_mac_p40(const P40Args& A, int n_p40, cudaStream_t s);
void launch_p40_pack(unsigned char* dst, const u64* diags, long long diag_stride, const int* limbs, int n_p40,
                     int n1, int n2, int dj, int logn, cudaStream_t s);

// ------------------------------------------------- tensor-core BSGS MAC
// (hx_bsgs_tc.cu): the TC-class limbs (q < 2^40) of up to 128 rows r = (block,
// giant step) per launch, T in {1, 2, 4, 8} tokens
constexpr int kTcMaxTokens = 8;
struct TcArgs {
  u64* inner;
  const long long* row_off;  // [R] word offset of row r's inner sum (j jstride + b bstride)
  long long tstride, L;      // token stride of the inner sums; words per poly (n_q N)
  const u64* baby;           // transposed baby words [n_tc][N][n1][2][T] (launch_tc_baby)
  const unsigned char* packed;  // TC section [n_tc][N][RG][KC][128]
  const int* limbs;             // TC-class limb list (li -> chain limb i)
  const PrimeConst* pc;
  const u32* mu;  // [n_tc][2]: floor(2^56 / q), floor(2^48 / q) (Barrett estimates)
  int rows, n1, n_tc, logn, KC, RG;
};
int tc_max_tokens();
void launch_tc_baby(u64* out, const u64* baby, long long btstride, long long L, const int* limbs, int n_tc, int n1,
                    int T, int logn, cudaStream_t s);
void launch_bsgs_mac_tc(const TcArgs& A, int tokens, int sms, cudaStream_t s);
void launch_tc_pack(unsigned char* dst, const u64* const* dptr, const int* tc_limbs, int n_tc, const int* wide_limbs,
                    int n_wide, int rows, int n1, int KC, int RG, int logn, size_t tc_bytes, cudaStream_t s);

}  // namespace hx
