/*
 * hx_b200.h -- C-ABI of the B200 (sm_100a) CKKS hot-path library libhx_b200.so.
 *
 * This is the device boundary below the C++ helix API (include/helix/): the
 * GPU SlotBackend (helix::GpuLatticeBackend) and the linear-transform entry
 * points call only these functions.  Plain pointers and sizes, no torch or
 * C++ types.  Every entry point replaces a reference routine of
 * /root/reference/proj (cited per function); the ones marked SPEC have no
 * reference code (the lattice backend and kernels are missing from the
 * reference tree, proj/CMakeLists.txt:20-26) and follow SPEC.md.
 *
 * Conventions (pinned):
 *  - A poly is u64 [limbs][N]; limb k < n_q is chain prime q_k, limb
 *    n_q + k is special prime p_k.  Residues in [0, q).  Batches are
 *    contiguous: [batch][limbs][N].  Ciphertexts are [2][n_q][N] (c0, c1),
 *    NTT domain (the reference's bit-reversed NttTables::forward layout).
 *  - A switching key is [dnum_max][2][n_chain + K][N] over the full basis
 *    (dnum_max = ceil(n_chain / alpha)); hx_key_words() gives its size.
 *  - Rotation by k slots (left) uses Galois element g = 5^k mod 2N.
 *  - All device pointers are device memory; `stream` is a cudaStream_t
 *    (NULL = legacy default stream).  Calls are asynchronous on `stream`
 *    unless stated otherwise and reentrant for distinct buffers.
 *  - Errors: every int-returning call returns HX_OK (0) or an HX_ERR_*
 *    code and records a message readable with hx_last_error() (thread-local).
 *    There is no CPU fallback: without a usable sm_100 device every compute
 *    call fails with HX_ERR_CUDA.
 */
#ifndef HX_B200_H
#define HX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HX_OK 0
#define HX_ERR_INVALID 1
#define HX_ERR_CUDA 2
#define HX_ERR_UNSUPPORTED 3
#define HX_ERR_OVERFLOW 4  /* encode: a coefficient exceeds the level's capacity */

typedef struct hx_ctx hx_ctx;

const char* hx_last_error(void);
const char* hx_version(void);

/* ---- context ------------------------------------------------------------
 * Replaces LatticeContext(const CkksParams&) (rns_poly.cpp:11-22) and the
 * NttTables ctor (ntt.cpp:36-55): per-prime psi (reference root search,
 * ntt.cpp:23-32), twiddle tables with Shoup companions, Barrett/Shoup
 * constants, ModUp/ModDown/rescale basis-conversion constants.  Unlike the
 * reference (one special prime, rns_poly.cpp:14-15) any K >= 1 special primes
 * and digit size alpha >= 1 are accepted.  logn in [8, 16]. */
hx_ctx* hx_ctx_create(int logn, const uint64_t* chain, int n_chain, const uint64_t* special,
                      int n_special, int alpha);
void hx_ctx_destroy(hx_ctx* ctx);
int hx_ctx_dnum(const hx_ctx* ctx, int n_q);
uint64_t hx_ctx_psi(const hx_ctx* ctx, int prime_index);
size_t hx_key_words(const hx_ctx* ctx);
/* release the context's scratch arena (the high-water mark of its calls) and
 * the device pool's idle memory; the next call regrows it */
int hx_ctx_trim(hx_ctx* ctx);
/* number of kernels this context has launched so far (bench evidence) */
unsigned long long hx_ctx_launches(const hx_ctx* ctx);

/* live per-kernel timing for the roofline of a timed step: while `name` is
 * set ("modup_col_kernel", "moddown_col_kernel", "ks_row_inner_f64_kernel",
 * "ntt_pass_kernel", "ntt_row_combine_kernel"; NULL or "" = off) every launch
 * of that kernel family records a CUDA event pair on its launching stream;
 * hx_ctx_kernel_time synchronises them and returns the summed device time
 * and the launch count since the last call (and clears them). */
int hx_ctx_time_kernel(hx_ctx* ctx, const char* name);
int hx_ctx_kernel_time(hx_ctx* ctx, double* total_ms, long long* launches);

/* ---- memory / streams ---- */
int hx_malloc(void** ptr, size_t bytes);
int hx_free(void* ptr);
int hx_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int hx_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int hx_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);
int hx_stream_sync(void* stream);
int hx_device_sync(void);

/* ---- RNS arithmetic ------------------------------------------------------ */
/* NttTables::forward / inverse per limb = LatticeContext::to_ntt / to_coeff
 * (ntt.cpp:57-96, rns_poly.cpp:42-54), in place over [batch][n_q+n_p][N]. */
int hx_ntt_fwd(hx_ctx* ctx, uint64_t* data, int batch, int n_q, int n_p, void* stream);
int hx_ntt_inv(hx_ctx* ctx, uint64_t* data, int batch, int n_q, int n_p, void* stream);
/* LatticeContext::add / sub / negate / mul / mul_acc (rns_poly.cpp:62-110) */
int hx_add(hx_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int batch, int n_q,
           int n_p, void* stream);
int hx_sub(hx_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int batch, int n_q,
           int n_p, void* stream);
int hx_neg(hx_ctx* ctx, uint64_t* out, const uint64_t* a, int batch, int n_q, int n_p,
           void* stream);
int hx_mul(hx_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int batch, int n_q,
           int n_p, void* stream);
int hx_mul_acc(hx_ctx* ctx, uint64_t* acc, const uint64_t* a, const uint64_t* b, int batch,
               int n_q, int n_p, void* stream);
/* broadcast product over [batch][n_q][N] polys: out[i] = a[a_mod ? i % a_mod : i]
 * (.) b[i / b_div] -- e.g. d masks applied to every poly of H ciphertexts
 * (a_mod = 2H, b_div = 2H) without replicating either operand */
int hx_mul_bcast(hx_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int batch, int a_mod,
                 int b_div, int n_q, void* stream);
/* LatticeContext::automorphism (rns_poly.cpp:124-142), X -> X^g, applied in
 * the NTT domain as a permutation. */
int hx_automorphism(hx_ctx* ctx, uint64_t* out, const uint64_t* in, int batch, int n_q, int n_p,
                    uint64_t galois, void* stream);
/* LatticeContext::from_i64 (rns_poly.cpp:218-227): v is device int64 [batch][N] */
int hx_from_i64(hx_ctx* ctx, uint64_t* out, const int64_t* v, int batch, int n_q, int n_p,
                void* stream);
/* LatticeContext::rescale_drop_last (rns_poly.cpp:144-162) on NTT-domain
 * polys: in [batch][n_q][N] -> out [batch][n_q-1][N] (centred lift). */
int hx_rescale(hx_ctx* ctx, uint64_t* out, const uint64_t* in, int batch, int n_q, void* stream);
/* x mod q per limb for words < 2^64 (after an NCCL uint64 sum of partials) */
int hx_reduce_mod_q(hx_ctx* ctx, uint64_t* data, int batch, int n_q, int n_p, void* stream);

/* ---- hybrid key switching -------------------- */
/* ModUp: c1 [batch][n_q][N] (NTT) -> digits [batch][dnum][n_q+K][N] (NTT) */
int hx_modup(hx_ctx* ctx, uint64_t* digits, const uint64_t* c1, int batch, int n_q, void* stream);
/* u [batch][2][n_q+K][N] = sum_d tau_g(D_d) (.) key_d ; galois 1 = none */
int hx_ks_inner(hx_ctx* ctx, uint64_t* u, const uint64_t* digits, const uint64_t* key, int batch,
                int n_q, uint64_t galois, void* stream);
/* centred ModDown (K = 1: LatticeContext::moddown_special, rns_poly.cpp:164-180):
 * u [polys][n_q+K][N] (NTT) -> out [polys][n_q][N] (NTT) */
int hx_moddown(hx_ctx* ctx, uint64_t* out, const uint64_t* u, int polys, int n_q, void* stream);
/* out [batch][2][n_q][N] with out0 + out1*s ~= in * s' (key for s') */
int hx_keyswitch(hx_ctx* ctx, uint64_t* out, const uint64_t* in, const uint64_t* key, int batch,
                 int n_q, void* stream);
/* galois_rotate: out = (tau(c0) + u0, u1), u = KS(tau(c1)),
 * ModUp hoisted before the automorphism.  in/out [batch][2][n_q][N].
 * `key` must be in ROTATION LAYOUT (hx_ksk_to_rotation_layout /
 * hx_keygen_rotation): the automorphism is applied once to the output instead
 * of to every ModUp digit; results are bit-identical to the standard-layout
 * definition. */
int hx_rotate(hx_ctx* ctx, uint64_t* out, const uint64_t* in, const uint64_t* key, int batch,
              int n_q, uint64_t galois, void* stream);
/* R rotations of each ciphertext sharing one ModUp.  keys: host array of R
 * device key pointers (rotation layout); galois: host array of R elements.
 * out [batch][R][2][n_q][N]. */
int hx_rotate_hoisted(hx_ctx* ctx, uint64_t* out, const uint64_t* in,
                      const uint64_t* const* keys, const uint64_t* galois, int R, int batch,
                      int n_q, void* stream);
/* batch of independent rotations with per-element keys (BSGS giant steps):
 * element b of in [batch][2][n_q][N] is rotated by galois[b] with keys[b]
 * (rotation layout); one batched ModUp. */
int hx_rotate_multi(hx_ctx* ctx, uint64_t* out, const uint64_t* in, const uint64_t* const* keys,
                    const uint64_t* galois, int batch, int n_q, void* stream);
/* rotations grouped by key: in [R][E][2][n_q][N]; ciphertexts r*E .. r*E+E-1
 * are rotated by galois[r] with keys[r] (rotation layout), each key word read
 * once for its E ciphertexts (BSGS giant step j of every row block).
 * out [R][E][2][n_q][N]. */
int hx_rotate_grouped(hx_ctx* ctx, uint64_t* out, const uint64_t* in, const uint64_t* const* keys,
                      const uint64_t* galois, int R, int E, int n_q, void* stream);
/* Double-hoisted giant-step sum (BSGS):
 *   out[e] = base[e] + sum_{r < R} Rot_{g_r}(in[r][e])
 * with ONE ModDown per output e instead of one per rotation: the key-switch
 * products tau_r(U_r) are summed in the PQ basis (S_e = sum_r tau_r(U_r),
 * [E][2][n_q + K][N]) together with T_e = base[e] + (sum_r tau_r(c0_r), 0),
 * then out[e] = T_e + (ModDown(S_e,0), ModDown(S_e,1)).  in [R][E][2][n_q][N],
 * base [E][2][n_q][N] or NULL, keys[r] rotation layout.  pq_partial != NULL:
 * stop before the ModDown -- write S to pq_partial and T to out (the partial
 * a giant-step shard exchanges; finish with hx_moddown_add after the sum of
 * the ranks' S and T, each reduced mod q). */
int hx_rotate_grouped_sum(hx_ctx* ctx, uint64_t* out, uint64_t* pq_partial, const uint64_t* in,
                          const uint64_t* base, const uint64_t* const* keys, const uint64_t* galois, int R, int E,
                          int n_q, void* stream);
/* out[e] = add[e] + (ModDown(pq[e][0]), ModDown(pq[e][1])); pq [E][2][n_q+K][N],
 * add [E][2][n_q][N] or NULL */
int hx_moddown_add(hx_ctx* ctx, uint64_t* out, const uint64_t* pq, const uint64_t* add, int E, int n_q,
                   void* stream);
/* tensor (LatticeContext::mul x4): a, b [batch][2][n_q][N] -> [batch][3][n_q][N] */
int hx_tensor(hx_ctx* ctx, uint64_t* out3, const uint64_t* a, const uint64_t* b, int batch,
              int n_q, void* stream);
/* ct x ct with relinearisation: tensor + KS(d2) with the key for s^2 */
int hx_mul_relin(hx_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b,
                 const uint64_t* rlk, int batch, int n_q, void* stream);

/* ---- BSGS linear transform ------------------------------ */
/* inner [n2][2][n_q][N]: inner_j = sum_k diags[j*n1+k] (.) baby[k];
 * baby [n1][2][n_q][N]; diags [n2*n1][diag_limbs][N] (first n_q limbs used). */
/* as hx_bsgs_mac with inner_j written at inner + j * inner_jstride words (e.g.
 * [n2][blocks][2][n_q][N] so the giant steps of all row blocks are grouped) */
int hx_bsgs_mac_ex(hx_ctx* ctx, uint64_t* inner, long long inner_jstride, const uint64_t* baby,
                   const uint64_t* diags, int diag_limbs, int n1, int n2, int n_q, void* stream);
/* out[p] = sum_{r < terms} in[r * term_stride + p * in_poly_stride] (mod q per
 * limb) for polys p of n_q limbs -- the giant-step sum */
int hx_sum_strided(hx_ctx* ctx, uint64_t* out, const uint64_t* in, int terms, long long term_stride,
                   int polys, long long in_poly_stride, long long out_poly_stride, int n_q,
                   void* stream);
/* token batch: `tokens` baby sets at baby + t baby_tstride words, inner sums at
 * inner + t inner_tstride; one launch, the blocks of one (coefficient tile,
 * limb) for all tokens run back to back so each diagonal word is read from
 * HBM once (L2 for the other tokens) -- config 3 with T tokens per matrix */
int hx_bsgs_mac_tokens(hx_ctx* ctx, uint64_t* inner, long long inner_jstride, long long inner_tstride,
                       const uint64_t* baby, long long baby_tstride, const uint64_t* diags, int diag_limbs, int n1,
                       int n2, int n_q, int tokens, int diag_jstride, void* stream);
/* (diag_jstride: diagonals between giant groups j and j + 1; 0 = n1.  A block
 * with more than 64 baby steps is multiplied in chunks of <= 64 of them, each
 * chunk a launch with n1 = chunk and diag_jstride = the block's n1.) */
int hx_bsgs_mac(hx_ctx* ctx, uint64_t* inner, const uint64_t* baby, const uint64_t* diags,
                int diag_limbs, int n1, int n2, int n_q, void* stream);
/* pruned matrices: the live diagonals of one row block as an index list --
 * group j owns entries [group_ptr[j], group_ptr[j+1]) (host ints, n2 + 1),
 * entry e multiplies baby step ks[e] (host ints) by the [n_q][N] words at
 * the DEVICE address diags[e] (a host array of device pointers); inner_j is
 * written only for groups with entries.  n1 <= 128; T tokens as
 * hx_bsgs_mac_tokens.  No gathers: diagonals and baby steps are read in place. */
int hx_bsgs_mac_sparse(hx_ctx* ctx, uint64_t* inner, long long inner_jstride, long long inner_tstride,
                       const uint64_t* baby, long long baby_tstride, const int* group_ptr, const int* ks,
                       const uint64_t* const* diags, int n1, int n2, int n_q, int tokens, void* stream);

/* Packed single-token BSGS MAC (hx_bsgs_p40.cu): the diagonals of one block
 * (n2 giant rows, n1 baby steps, diagonal (j, k) at diags + (j diag_jstride +
 * k) diag_limbs N words, diag_jstride 0 = n1) are packed once into 5-byte words
 * for the limbs with q < 2^40 (hx_bsgs_p40_bytes bytes, -1 = unsupported
 * shape or no such limb); the MAC streams them with bulk copies and runs the
 * remaining (wide, e.g. 60-bit q_0) limbs on the integer MAC over the u64
 * words at `diags`.  n1 in {32, 64}.  Same words as hx_bsgs_mac_ex. */
long long hx_bsgs_p40_bytes(hx_ctx* ctx, int n1, int n2, int n_q);
int hx_bsgs_p40_pack(hx_ctx* ctx, void* packed, const uint64_t* diags, int diag_limbs, int n1, int n2,
                     int diag_jstride, int n_q, void* stream);
int hx_bsgs_mac_p40(hx_ctx* ctx, uint64_t* inner, long long inner_jstride, const uint64_t* baby, const void* packed,
                    const uint64_t* diags, int diag_limbs, int n1, int n2, int diag_jstride, int n_q, void* stream);
/* The same over `blocks` row blocks in one launch (the baby steps are read and
 * split once for all of them): the diagonals of block b follow those of block
 * b - 1 (diagonal (b, j, k) at diags + ((b n2 + j) n1 + k) diag_limbs N),
 * `packed` was made by hx_bsgs_p40_pack with n2 * blocks rows, and the inner
 * sum of (b, j) is written at inner + j inner_jstride + b inner_bstride. */
int hx_bsgs_mac_p40_blocks(hx_ctx* ctx, uint64_t* inner, long long inner_jstride, long long inner_bstride,
                           const uint64_t* baby, const void* packed, const uint64_t* diags, int diag_limbs, int n1,
                           int n2, int blocks, int diag_jstride, int n_q, void* stream);

/* Tensor-core BSGS MAC (tcgen05.mma kind::i8 on byte-sliced words, TMEM
 * accumulators, bulk-copy-streamed diagonals; hx_bsgs_tc.cu).  The diagonals of
 * up to 128 rows r = b * n2 + j (row block b, giant step j) are packed once into
 * a device buffer of hx_bsgs_tc_bytes bytes: limbs with q < 2^40 as 5-byte
 * sliced tcgen05 operand tiles (37.5 % fewer bytes than u64 words), wider limbs
 * (q_0) as u64 copies.  diag_ptrs: host array [rows * n1] of DEVICE addresses of
 * [>= n_q][N] plaintext words (NULL = zero diagonal).  n1 % 8 == 0, n1 <= 64,
 * N >= 128.  Returns -1 on a bad shape. */
long long hx_bsgs_tc_bytes(hx_ctx* ctx, int rows, int n1, int n_q);
int hx_bsgs_tc_pack(hx_ctx* ctx, void* packed, const uint64_t* const* diag_ptrs, int rows, int n1, int n_q,
                    void* stream);
/* inner sums of all rows from one packed matrix: row (b, j) of token t at
 * inner + j inner_jstride + b inner_bstride + t inner_tstride words ([2][n_q][N]);
 * baby sets [n1][2][n_q][N] at baby + t baby_tstride.  Same words as
 * hx_bsgs_mac_tokens over the unpacked diagonals. */
int hx_bsgs_mac_tc(hx_ctx* ctx, uint64_t* inner, long long inner_jstride, long long inner_bstride,
                   long long inner_tstride, const uint64_t* baby, long long baby_tstride, const void* packed,
                   int blocks, int n2, int n1, int n_q, int tokens, void* stream);

/* ---- keys / encryption ------------------------ */
/* Device samplers (counter-based: splitmix64 of (seed, index)), used for key
 * material so that key generation needs no host RNG stream or H2D copy:
 * out [copies][n_c + n_s][N] uniform in [0, q) per limb (128-bit multiply-high
 * reduction, bias < 2^-64); e [count] centred binomial (k = 21) int64. */
int hx_sample_uniform(hx_ctx* ctx, uint64_t* out, int n_c, int n_s, int copies, uint64_t seed, void* stream);
int hx_sample_cbd(hx_ctx* ctx, int64_t* e, long long count, uint64_t seed, void* stream);
/* ksk_d = (-a_d s + e_d + [P]_{q_i} s' on the chain limbs of digit d, a_d).
 * s_full, sp_full [n_chain+K][N] NTT; a_full [dnum_max][n_chain+K][N];
 * e [dnum_max][N] int64; all device. */
int hx_keygen_ksk(hx_ctx* ctx, uint64_t* key, const uint64_t* s_full, const uint64_t* sp_full,
                  const uint64_t* a_full, const int64_t* e, void* stream);
/* rotation-layout key for galois element g from a standard-layout key:
 * out = tau_{g^-1}(in) limb-wise (out != in) */
int hx_ksk_to_rotation_layout(hx_ctx* ctx, uint64_t* out, const uint64_t* in, uint64_t galois,
                              void* stream);
/* ---- compressed keys (seeded key compression) ----
 * Only the b half of every digit is stored ([dnum_max][n_chain+K][N] words,
 * hx_ckey_words: half of hx_key_words); the uniform half a is the counter
 * stream of `seed` (hx_sample_uniform) and is regenerated inside the key
 * inner product.  The context remembers (seed, layout) per compressed key
 * pointer: pass the pointer wherever a key is taken (hx_rotate*, hx_keyswitch,
 * hx_mul_relin, hx_ks_inner); hx_key_release forgets it before it is freed.
 * hx_key_expand writes the full key (e.g. for an oracle). */
size_t hx_ckey_words(const hx_ctx* ctx);
int hx_keygen_ksk_c(hx_ctx* ctx, uint64_t* ckey, const uint64_t* s_full, const uint64_t* sp_full, uint64_t seed,
                    const int64_t* e, void* stream);
int hx_keygen_rotation_c(hx_ctx* ctx, uint64_t* ckey, const uint64_t* s_full, uint64_t galois, uint64_t seed,
                         const int64_t* e, void* stream);
int hx_key_expand(hx_ctx* ctx, uint64_t* full, const uint64_t* ckey, void* stream);
int hx_key_release(hx_ctx* ctx, const uint64_t* ckey);
/* rotation key for tau_g (s' = tau_g(s)) directly in rotation layout */
int hx_keygen_rotation(hx_ctx* ctx, uint64_t* key, const uint64_t* s_full, uint64_t galois,
                       const uint64_t* a_full, const int64_t* e, void* stream);
/* ct = (m - a s + e, a), m/a [n_q][N] NTT, e [N] int64 (device) */
int hx_encrypt_sk(hx_ctx* ctx, uint64_t* ct, const uint64_t* m, const uint64_t* s_full,
                  const uint64_t* a, const int64_t* e, int n_q, void* stream);
/* m = c0 + c1 s (NTT), ct [batch][2][n_q][N] -> m [batch][n_q][N] */
int hx_decrypt(hx_ctx* ctx, uint64_t* m, const uint64_t* ct, const uint64_t* s_full, int batch,
               int n_q, void* stream);

/* ---- end-to-end entry points over HOST buffers ----------------------------
 * The reference-facing calls a CPU caller makes: host (ideally pinned) input
 * ciphertexts are copied in, processed with device-resident keys, and copied
 * back, all on `stream`; the call returns after the result is in host memory. */
int hx_rotate_host(hx_ctx* ctx, uint64_t* out_host, const uint64_t* in_host, const uint64_t* key,
                   int batch, int n_q, uint64_t galois, void* stream);
int hx_mul_relin_host(hx_ctx* ctx, uint64_t* out_host, const uint64_t* a_host,
                      const uint64_t* b_host, const uint64_t* rlk, int batch, int n_q,
                      void* stream);

/* ---- CKKS encoder on the device ----
 * Replaces CkksEncoder::encode (reference encoder.cpp:69-117) for batches of
 * real slot vectors: int64 coefficients bit-identical to the host encoder.
 * Tables come from the host (helix::CkksEncoder::device_tables): perm [N]
 * int32, stage_tw [N-1] complex (re, im interleaved), zeta [N] complex. */
typedef struct hx_encoder hx_encoder;
hx_encoder* hx_encoder_create(hx_ctx* ctx, const int32_t* perm, const double* stage_tw, const double* zeta);
void hx_encoder_destroy(hx_encoder* enc);
/* coeffs (device) [batch][N] int64 <- round(scale * embed^-1(m_b)), m (device)
 * [batch] vectors of len_m <= N/2 doubles at stride m_stride (zero padded).
 * HX_ERR_OVERFLOW when some |coefficient| >= 2^62 or log2(|c| + 1) >= cap_log2
 * (log2(Q_level / 2), CkksEncoder::capacity_log2).  Synchronises `stream`. */
int hx_encode(hx_encoder* enc, int64_t* coeffs, const double* m, int len_m, long long m_stride, int batch,
              double scale, double cap_log2, void* stream);

#ifdef __cplusplus
}
#endif
#endif
