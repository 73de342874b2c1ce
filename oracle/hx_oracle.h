/*
 * hx_oracle.h -- CPU ORACLE for the CKKS linear-transform hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2512_11135_b200/,
 * include/) links, loads or calls this library.  It is imported only by
 * tests/, by __graft_entry__.smoke() (as the checker) and by bench.py's
 * cpu_baseline / --impl reference legs.
 *
 * It is a plain-C restatement of the reference algorithms in
 * /root/reference/proj (file:line cited per function in hx_oracle.c) plus the
 * SPEC-only pieces (hybrid key switch, rotation, hoisting, relinearisation,
 * BSGS diagonal MAC) under the conventions pinned in DESIGN.md §3:
 *
 *   - NTT layout: forward leaves bit-reversed order, out[k] = a(psi^(2 brv(k)+1)),
 *     psi from the reference's root search (ntt.cpp:23-32).
 *   - Rotation k <-> Galois element g = 5^k mod 2N, left shift.
 *   - ModUp: non-centred FastBConv per alpha-limb digit.
 *   - ModDown / rescale: CENTRED FastBConv (K = 1 reduces exactly to the
 *     reference's moddown_special / rescale_drop_last).
 *   - Hoisting: ModUp(c1) once, automorphism on the NTT-form digits, inner
 *     product, ModDown per rotation.
 *
 * Poly layout: u64 [limbs][N], limb k is chain prime k for k < n_q and special
 * prime (k - n_q) for n_q <= k < n_q + n_p.  Ciphertexts are [2][limbs][N].
 * Keys are [dnum_max][2][n_chain + K][N] over the FULL basis.
 */
#ifndef HX_ORACLE_H
#define HX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HXO_MAX_PRIMES 64

typedef struct hxo_ctx hxo_ctx;

/* ---- scalar modmath (modmath.hpp) ---- */
uint64_t hxo_mulmod(uint64_t a, uint64_t b, uint64_t q);
uint64_t hxo_powmod(uint64_t a, uint64_t e, uint64_t q);
uint64_t hxo_invmod(uint64_t a, uint64_t q);
int hxo_is_prime(uint64_t n);
/* first `count` primes p = 1 mod two_n at or above start, skipping `exclude` */
int hxo_find_ntt_primes(uint64_t start, int count, uint64_t two_n, const uint64_t* exclude,
                        int n_exclude, uint64_t* out);
uint64_t hxo_find_psi(uint64_t q, uint64_t n);

/* ---- single-limb NTT (ntt.cpp) ---- */
void hxo_ntt_forward_limb(uint64_t q, uint64_t psi, int logn, uint64_t* a);
void hxo_ntt_inverse_limb(uint64_t q, uint64_t psi, int logn, uint64_t* a);
void hxo_schoolbook_negacyclic(uint64_t q, uint64_t n, const uint64_t* a, const uint64_t* b,
                               uint64_t* out);

/* ---- context ---- */
hxo_ctx* hxo_ctx_create(int logn, const uint64_t* chain, int n_chain, const uint64_t* special,
                        int n_special, int alpha);
void hxo_ctx_destroy(hxo_ctx* c);
uint64_t hxo_ctx_psi(const hxo_ctx* c, int prime_index);
int hxo_ctx_dnum(const hxo_ctx* c, int n_q);
void hxo_set_threads(int n);

/* ---- poly ops ([limbs][N]) ---- */
void hxo_ntt_fwd(const hxo_ctx* c, uint64_t* p, int n_q, int n_p);
void hxo_ntt_inv(const hxo_ctx* c, uint64_t* p, int n_q, int n_p);
void hxo_add(const hxo_ctx* c, uint64_t* o, const uint64_t* a, const uint64_t* b, int n_q, int n_p);
void hxo_sub(const hxo_ctx* c, uint64_t* o, const uint64_t* a, const uint64_t* b, int n_q, int n_p);
void hxo_neg(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q, int n_p);
void hxo_mul(const hxo_ctx* c, uint64_t* o, const uint64_t* a, const uint64_t* b, int n_q, int n_p);
void hxo_mul_acc(const hxo_ctx* c, uint64_t* acc, const uint64_t* a, const uint64_t* b, int n_q,
                 int n_p);
void hxo_automorphism_coeff(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q, int n_p,
                            uint64_t g);
void hxo_automorphism_ntt(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q, int n_p,
                          uint64_t g);
/* coefficient domain, reference rescale_drop_last: n_q -> n_q - 1 limbs */
void hxo_rescale_coeff(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q);
/* NTT domain wrapper (INTT, rescale_coeff, NTT) */
void hxo_rescale_ntt(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q);
/* centred FastBConv ModDown, coefficient domain: (n_q + K) -> n_q limbs */
void hxo_moddown_coeff(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q);
/* reduce small signed integers into every limb (rns_poly.cpp:218-227) */
void hxo_from_i64(const hxo_ctx* c, uint64_t* o, const int64_t* v, int n_q, int n_p);

/* ---- key switching ---- */
/* c1 in NTT form [n_q][N] -> digits [dnum][n_q + K][N] in NTT form */
void hxo_modup(const hxo_ctx* c, uint64_t* digits, const uint64_t* c1_ntt, int n_q);
/* U[2][n_q+K][N] = sum_d tau_g(D_d) * key_d ; g = 1 means no automorphism */
void hxo_ks_inner(const hxo_ctx* c, uint64_t* u, const uint64_t* digits, const uint64_t* key,
                  int n_q, uint64_t g);
/* NTT-domain ModDown of a PQ-basis poly pair: u[2][n_q+K][N] -> o[2][n_q][N] */
void hxo_moddown_ntt(const hxo_ctx* c, uint64_t* o, const uint64_t* u, int n_q, int n_polys);
/* out[2][n_q][N] (NTT) with out0 + out1*s ~= in * s' */
void hxo_keyswitch(const hxo_ctx* c, uint64_t* out, const uint64_t* in_ntt, const uint64_t* key,
                   int n_q);
/* Rot_k: out = (tau(c0) + u0, u1), u = KS(tau(c1)) [hoisting convention] */
void hxo_rotate(const hxo_ctx* c, uint64_t* out_ct, const uint64_t* in_ct, const uint64_t* key,
                int n_q, uint64_t g);
/* R rotations of one ciphertext sharing one ModUp; keys[r] points at key r */
void hxo_rotate_hoisted(const hxo_ctx* c, uint64_t* out_cts, const uint64_t* in_ct,
                        const uint64_t* const* keys, const uint64_t* gs, int R, int n_q);
/* (a0,a1) x (b0,b1) -> (d0,d1,d2), NTT domain */
void hxo_tensor(const hxo_ctx* c, uint64_t* out3, const uint64_t* a, const uint64_t* b, int n_q);
/* tensor + relinearise with key for s^2 */
void hxo_mul_relin(const hxo_ctx* c, uint64_t* out_ct, const uint64_t* a, const uint64_t* b,
                   const uint64_t* rlk, int n_q);
/* inner_j = sum_k diag[j*n1+k] (.) baby_k, both ciphertext polys; NTT domain */
void hxo_bsgs_mac(const hxo_ctx* c, uint64_t* inner, const uint64_t* baby, const uint64_t* diags,
                  int n1, int n2, int n_q);

/* ---- linear-algebra drivers ----
 * keys: indexed by rotation amount r in [0, N/2) -> standard-layout key
 * (NULL where unused).  Plaintexts are NTT-form [n_q][N] words. */
/* BSGS matvec: baby steps hoisted; per row block b the inner sums over the
 * NON-NULL diagonals diags[b n1 n2 + j n1 + k]; giant groups j in
 * [giant_begin, giant_end) (giant_end < 0: n2) rotated by n1 j and summed.
 * lazy = 1: double hoisting -- the giant rotations' key-switch products are
 * summed in the PQ basis and ModDown runs once per output.
 * out [blocks][2][n_q - rescale][N].  partial = 1 (giant-step shard, implies
 * lazy, no rescale): out [blocks][T 2 n_q + S 2 (n_q + K)][N], the PQ-basis
 * partial before the ModDown. */
void hxo_matvec_bsgs(const hxo_ctx* c, uint64_t* out, const uint64_t* x, int n_q, int n1, int n2, int blocks,
                     const uint64_t* const* diags, const uint64_t* const* keys, int giant_begin, int giant_end,
                     int rescale, int lazy, int partial);
/* packed-row matvec; rows_pts [groups] at n_q limbs, masks [p] at n_q - 1 limbs;
 * out [2][n_q - 2][N] */
void hxo_matvec_row(const hxo_ctx* c, uint64_t* out, const uint64_t* x, int n_q, int groups, int p, int rows,
                    int pad_cols, const uint64_t* const* rows_pts, const uint64_t* const* masks,
                    const uint64_t* const* keys);
/* ct-ct matmul of d x d row-major operands; masks [d] at n_q limbs;
 * rlk standard layout; out [2][n_q - 2][N] */
void hxo_matmul_ctct(const hxo_ctx* c, uint64_t* out, const uint64_t* A, const uint64_t* B, int n_q, int d,
                     const uint64_t* const* colmask, const uint64_t* const* rowmask, const uint64_t* rlk,
                     const uint64_t* const* keys);

/* ---- keys / encryption ---- */
/* s_full, sp_full: NTT form over the full basis (n_chain + K limbs);
 * a_full: [dnum_max][n_chain+K][N] uniform residues (used as NTT-form values);
 * e: [dnum_max][N] small signed coefficients. */
void hxo_keygen_ksk(const hxo_ctx* c, uint64_t* key, const uint64_t* s_full,
                    const uint64_t* sp_full, const uint64_t* a_full, const int64_t* e);
/* plaintext poly m (NTT, n_q limbs) -> m + c1*s */
void hxo_decrypt(const hxo_ctx* c, uint64_t* m_out, const uint64_t* ct, const uint64_t* s_full,
                 int n_q);
/* out = (m - a*s + e, a); a NTT-form uniform [n_q][N], e coeffs [N] */
void hxo_encrypt_sk(const hxo_ctx* c, uint64_t* ct, const uint64_t* m_ntt, const uint64_t* s_full,
                    const uint64_t* a, const int64_t* e, int n_q);

#ifdef __cplusplus
}
#endif
#endif
