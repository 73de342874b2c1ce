/*
 * helix_c.h -- C-ABI over the helix C++ host API (include/helix/ headers) as
 * implemented on B200 by libhelix_b200.so (GpuLatticeBackend + linalg).
 *
 * This is the reference-facing plugin boundary for non-C++ callers (the
 * ctypes stubs in INTEGRATION.md, the tests and bench.py): it exposes
 * exactly the SlotBackend / SPEC kernel entry points of the reference,
 *   SlotBackend::{encrypt, decrypt, generate_rotation_keys, rotate, add, mul,
 *                 mul_plain, rescale}            backend.hpp:90-138
 *   matvec_row / matvec_diag / matvec_bsgs
 *   matmul_ctct
 *   rotate_and_sum
 *   OpTrace::to_json                             trace.cpp:24-32
 * with host double vectors in and out; ciphertexts stay in HBM behind
 * opaque handles.  Errors: NULL / negative return + hxc_last_error().
 */
#ifndef HELIX_C_H
#define HELIX_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hxc_backend hxc_backend;
typedef struct hxc_ct hxc_ct;
typedef struct hxc_mat hxc_mat;

typedef struct {
  uint64_t rotations, pt_muls, ct_muls, adds;
  int64_t levels_consumed;
  double output_scale_log2;
} hxc_report;

/* HXC_BSGS_STACKED: row blocks stacked in one set of full-length diagonals
 * (helix::pack_bsgs_stacked); one output ciphertext, y[row] in slot `row` */
enum { HXC_ROW = 0, HXC_DIAG = 1, HXC_BSGS = 2, HXC_BSGS_STACKED = 3 };

const char* hxc_last_error(void);

/* CkksParams JSON (reference params.cpp:53-96 keys + "alpha") */
hxc_backend* hxc_backend_create(const char* params_json, uint64_t seed);
void hxc_backend_destroy(hxc_backend* b);
int64_t hxc_slots(hxc_backend* b);
int hxc_max_level(hxc_backend* b);
/* the underlying hx_ctx* (libhx_b200 C-ABI) for device-level pipelines */
void* hxc_device_context(hxc_backend* b);
/* release the device scratch arena and the stream-ordered pool's cached
   memory (hx_ctx_trim); call between workloads of different shapes */
int hxc_trim(hxc_backend* b);
int hxc_gen_rotation_keys(hxc_backend* b, const int64_t* amounts, int count);

/* encode(m, level, Delta) + encrypt; m has len <= slots entries (zero-padded) */
hxc_ct* hxc_encrypt(hxc_backend* b, const double* m, int len, int level);
/* decrypt + decode: writes slots() doubles */
int hxc_decrypt(hxc_backend* b, const hxc_ct* ct, double* out);
void hxc_ct_free(hxc_ct* ct);
int hxc_ct_level(const hxc_ct* ct);
double hxc_ct_scale_log2(const hxc_ct* ct);
/* device pointer to the ciphertext words [2][level+1][N] */
uint64_t* hxc_ct_device_ptr(const hxc_ct* ct);

hxc_ct* hxc_add(hxc_backend* b, const hxc_ct* x, const hxc_ct* y);
hxc_ct* hxc_mul(hxc_backend* b, const hxc_ct* x, const hxc_ct* y);
/* x (.) encode(m, x.level, scale_log2 == 0 ? q_level : 2^scale_log2) */
hxc_ct* hxc_mul_plain(hxc_backend* b, const hxc_ct* x, const double* m, int len);
hxc_ct* hxc_rotate(hxc_backend* b, const hxc_ct* x, int64_t k);
hxc_ct* hxc_rescale(hxc_backend* b, const hxc_ct* x);
hxc_ct* hxc_mod_down(hxc_backend* b, const hxc_ct* x, int level);
hxc_ct* hxc_rotate_and_sum(hxc_backend* b, const hxc_ct* x, int64_t span, int64_t stride,
                           hxc_report* rep);

/* Pack (method HXC_ROW / HXC_DIAG / HXC_BSGS, default BSGS plan) and encode a
 * rows x cols row-major matrix at `level` (encoding is not part of a matvec). */
hxc_mat* hxc_matrix_prepare(hxc_backend* b, int method, const double* A, int rows, int cols,
                            int level);
/* The same with an explicit BSGS split (helix::pack_bsgs(A, plan, n),
 * linalg.hpp:82): n1 = 0 the SPEC default (BsgsPlan::for_dim), n1 > 0 that
 * baby-step count (a power of two <= d, n2 = d / n1), n1 < 0 the
 * cost-tuned split BsgsPlan::for_cost(d, row_blocks). */
hxc_mat* hxc_matrix_prepare_plan(hxc_backend* b, int method, const double* A, int rows, int cols,
                                 int level, int n1);
void hxc_matrix_free(hxc_mat* m);
/* d, n1, n2, row_blocks, nonzero payloads */
int hxc_matrix_info(const hxc_mat* m, int* d, int* n1, int* n2, int* blocks, int* nonzero);
/* rotation amounts the method needs; returns the count (writes <= cap) */
int hxc_matrix_rotations(const hxc_mat* m, int64_t* out, int cap);
/* y = M x; writes up to cap output handles (one per row block); returns count */
int hxc_matvec(hxc_backend* b, const hxc_mat* m, const hxc_ct* x, hxc_ct** out, int cap,
               hxc_report* rep);
/* T ciphertexts (tokens) through one BSGS matrix with every key switch batched
 * over the tokens (helix::matvec_bsgs_tokens); out receives T x blocks handles
 * token-major; returns that count (or -1); rep = per-token counters. */
int hxc_matvec_tokens(hxc_backend* b, const hxc_mat* m, const hxc_ct* const* xs, int T, hxc_ct** out, int cap,
                      hxc_report* rep);

/* ---- giant-step sharding of BSGS (multi-GPU, one process per GPU) ----
 * rank r of world G encodes only its giant groups (helix::bsgs_shard) and
 * returns PQ-BASIS PARTIAL outputs (double-hoisted giant steps: the ModDown
 * waits for the sum of all ranks): each handle's device buffer holds
 * hxc_shard_partial_words() words, T [2][n_q][N] then S [2][n_q + K][N].  The
 * caller sums the partial words of all ranks (NCCL all-reduce of int64 =
 * wrapping uint64 sum), reduces T and S mod q (hx_reduce_mod_q with n_p = 0 /
 * K), finishes with hxc_shard_finish (T + ModDown(S)) and rescales once. */
hxc_mat* hxc_matrix_prepare_shard(hxc_backend* b, const double* A, int rows, int cols, int level,
                                  int rank, int world, int stacked);
int hxc_matvec_shard(hxc_backend* b, const hxc_mat* m, const hxc_ct* x, hxc_ct** out, int cap,
                     hxc_report* rep);
/* a new ciphertext with the level / scale of `like` and words copied from the
 * device buffer `words` ([2][level+1][N]) */
hxc_ct* hxc_ct_like(hxc_backend* b, const hxc_ct* like, const uint64_t* words);
/* words of one shard partial (T and S) at like's level */
long long hxc_shard_partial_words(hxc_backend* b, const hxc_ct* like);
/* the pre-rescale output T + (ModDown(S_0), ModDown(S_1)) of a summed, reduced
 * partial (device words laid out as hxc_matvec_shard returns them) */
hxc_ct* hxc_shard_finish(hxc_backend* b, const hxc_ct* like, const uint64_t* words);

/* ct-ct matmul of row-major d x d operands */
hxc_ct* hxc_matmul(hxc_backend* b, const hxc_ct* A, const hxc_ct* B, int d, hxc_report* rep);
/* H heads in one batched schedule (keys read once per H heads); out[h] gets
 * matmul(As[h], Bs[h]); rep = per-head counters; returns H or -1 */
int hxc_matmul_heads(hxc_backend* b, const hxc_ct* const* As, const hxc_ct* const* Bs, int H, int d, hxc_ct** out,
                     hxc_report* rep);
/* rotation count a dense rows x cols matvec records at `slots` slots (counters
 * only, no device work; helix::predicted_rotations; SPEC criterion 4) */
long long hxc_predicted_rotations(int method, int rows, int cols, int64_t slots);
/* polyeval: n coefficients, power basis (chebyshev = 0) or
 * Chebyshev on [lo, hi]; output scale exactly Delta (helix::polyeval) */
hxc_ct* hxc_polyeval(hxc_backend* b, const hxc_ct* x, const double* coeffs, int n, int chebyshev, double lo,
                     double hi, hxc_report* rep);
int hxc_matmul_rotations(int d, int64_t* out, int cap);

/* ---- raw device words, for the bit-exact parity tests ----
 * secret key [n_chain+K][N] (NTT), relinearisation key (standard layout),
 * rotation key for amount k (rotation layout, NULL if absent), payload i of an
 * encoded matrix [level+1][N] (NULL for an all-zero payload) */
const uint64_t* hxc_secret_key_ptr(hxc_backend* b);
const uint64_t* hxc_relin_key_ptr(hxc_backend* b);
const uint64_t* hxc_rotation_key_ptr(hxc_backend* b, int64_t k);
/* the backend stores compressed keys (hx_keygen_*_c): full [dnum][2][n_chain+K][N]
 * words of a key pointer (hxc_rotation_key_ptr / hxc_relin_key_ptr) into
 * device memory full_dev (hx_key_words words) */
int hxc_key_expand(hxc_backend* b, const uint64_t* ckey, uint64_t* full_dev);
const uint64_t* hxc_matrix_payload_ptr(const hxc_mat* m, int i);
int hxc_matrix_payload_count(const hxc_mat* m);
/* host-only: CkksEncoder::encode_coeffs for a CkksParams JSON (no device) */
/* device encode (GpuLatticeBackend::encode: hx_encode + RNS lift + NTT) of m at
 * `level` with a raw double scale; out: host [level+1][N] NTT-domain words.
 * -1 with hxc_last_error() on error (std::overflow_error text on capacity). */
int hxc_encode_words(hxc_backend* b, const double* m, int len, int level, double scale, uint64_t* out);
int hxc_encode_coeffs(const char* params_json, const double* m, int len, int level, double scale,
                      int64_t* out);
/* host-only: CkksEncoder::decode_coeffs (encoder.cpp:119-159 restated with a
 * Garner CRT): coefficient-domain limbs [n_limbs][N] -> N/2 slots */
int hxc_decode_coeffs(const char* params_json, const uint64_t* limbs, int n_limbs, double scale, double* out);

/* OpTrace JSON (canonical names ct_add ... bootstrap); returns length */
int hxc_trace_json(hxc_backend* b, char* buf, int cap);
void hxc_trace_reset(hxc_backend* b);
int hxc_sync(void);

#ifdef __cplusplus
}
#endif
#endif
