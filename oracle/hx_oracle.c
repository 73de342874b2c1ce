/*
 * hx_oracle.c -- CPU ORACLE (test infrastructure; see hx_oracle.h).
 *
 * Plain-C restatement of the reference CKKS primitives of
 * /root/reference/proj (arXiv 2512.11135 "Helix" C++ reference) and of the
 * SPEC-only key-switching / linear-transform pieces.  Every function cites the
 * reference file:line (or SPEC.md line) it follows.  Modular products use an
 * exact 128-bit remainder, i.e. the reference algorithms with a CORRECT
 * Modulus::mul (the shipped one is broken, modmath.hpp:30 -- see DESIGN.md).
 */
#include "hx_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* scalar modular arithmetic                              modmath.hpp:21-152 */
/* ------------------------------------------------------------------------ */

/* Modulus::mul (modmath.hpp:49-63) -- exact a*b mod q */
uint64_t hxo_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (u64)(((u128)a * b) % q); }

static inline u64 addm(u64 a, u64 b, u64 q) { /* modmath.hpp:41-44 */
  u64 s = a + b;
  return s >= q ? s - q : s;
}
static inline u64 subm(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; } /* :45 */
static inline u64 negm(u64 a, u64 q) { return a == 0 ? 0 : q - a; }               /* :46 */

/* Modulus::pow (modmath.hpp:65-75) */
uint64_t hxo_powmod(uint64_t a, uint64_t e, uint64_t q) {
  u64 r = 1 % q, b = a % q;
  while (e) {
    if (e & 1) r = hxo_mulmod(r, b, q);
    b = hxo_mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}

/* Modulus::inv (modmath.hpp:77-81), Fermat */
uint64_t hxo_invmod(uint64_t a, uint64_t q) { return hxo_powmod(a % q, q - 2, q); }

/* Modulus::centered (modmath.hpp:83-86): representative in (-q/2, q/2] */
static inline int64_t centered(u64 a, u64 q) {
  return a > q / 2 ? (int64_t)a - (int64_t)q : (int64_t)a;
}
/* Modulus::reduce_i64 (modmath.hpp:88-91) */
static inline u64 reduce_i64(int64_t v, u64 q) {
  int64_t m = v % (int64_t)q;
  if (m < 0) m += (int64_t)q;
  return (u64)m;
}

/* shoup_precompute / mul_shoup (modmath.hpp:97-105) */
static inline u64 shoup_pre(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static inline u64 mul_shoup(u64 a, u64 w, u64 wp, u64 q) {
  u64 hi = (u64)(((u128)a * wp) >> 64);
  u64 r = a * w - hi * q;
  return r >= q ? r - q : r;
}

/* is_prime_u64 (modmath.hpp:107-134): trial division + MR, fixed witnesses */
int hxo_is_prime(uint64_t n) {
  static const u64 small[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (n % small[i] == 0) return n == small[i];
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (int i = 0; i < 12; ++i) {
    u64 x = hxo_powmod(small[i] % n, d, n);
    if (x == 1 || x == n - 1) continue;
    int composite = 1;
    for (int k = 1; k < r; ++k) {
      x = hxo_mulmod(x, x, n);
      if (x == n - 1) {
        composite = 0;
        break;
      }
    }
    if (composite) return 0;
  }
  return 1;
}

/* find_ntt_primes (modmath.hpp:138-152) */
int hxo_find_ntt_primes(uint64_t start, int count, uint64_t two_n, const uint64_t* exclude,
                        int n_exclude, uint64_t* out) {
  u64 p = ((start + two_n - 1) / two_n) * two_n + 1;
  int got = 0;
  while (got < count) {
    int skip = 0;
    for (int e = 0; e < n_exclude; ++e)
      if (exclude[e] == p) skip = 1;
    if (!skip && hxo_is_prime(p)) out[got++] = p;
    p += two_n;
    if (p < two_n) return -1;
  }
  return 0;
}

/* find_primitive_root (ntt.cpp:23-32): smallest g >= 2 whose
 * c = g^((q-1)/2n) satisfies c^n = -1; psi = c (NOT the minimal root). */
uint64_t hxo_find_psi(uint64_t q, uint64_t n) {
  const u64 order = 2 * n;
  if ((q - 1) % order != 0) return 0;
  for (u64 g = 2; g < q; ++g) {
    u64 c = hxo_powmod(g, (q - 1) / order, q);
    if (hxo_powmod(c, n, q) == q - 1) return c;
  }
  return 0;
}

/* bit_reverse (ntt.cpp:12-19) */
static u64 bitrev(u64 x, int bits) {
  u64 r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

/* ------------------------------------------------------------------------ */
/* NTT tables + transforms                                     ntt.cpp:36-96 */
/* ------------------------------------------------------------------------ */

typedef struct {
  u64 q, psi, ninv, ninvp;
  int logn;
  u64 *fwd, *fwdp, *inv, *invp;
} tables_t;

/* NttTables ctor (ntt.cpp:36-55): fwd[i] = psi^brv(i), inv[i] = psi^-brv(i) */
static void tables_init(tables_t* t, u64 q, u64 psi, int logn) {
  const u64 n = 1ull << logn;
  t->q = q;
  t->psi = psi;
  t->logn = logn;
  t->fwd = (u64*)malloc(n * 8);
  t->fwdp = (u64*)malloc(n * 8);
  t->inv = (u64*)malloc(n * 8);
  t->invp = (u64*)malloc(n * 8);
  const u64 psi_inv = hxo_invmod(psi, q);
  /* powers by repeated multiplication, then scattered through brv -- same
   * values as Modulus::pow(psi, brv(i)) since results mod q are unique */
  u64 pw = 1, pwi = 1;
  for (u64 e = 0; e < n; ++e) {
    const u64 i = bitrev(e, logn);
    t->fwd[i] = pw;
    t->inv[i] = pwi;
    pw = hxo_mulmod(pw, psi, q);
    pwi = hxo_mulmod(pwi, psi_inv, q);
  }
  for (u64 i = 0; i < n; ++i) {
    t->fwdp[i] = shoup_pre(t->fwd[i], q);
    t->invp[i] = shoup_pre(t->inv[i], q);
  }
  t->ninv = hxo_invmod(n % q, q);
  t->ninvp = shoup_pre(t->ninv, q);
}

static void tables_free(tables_t* t) {
  free(t->fwd);
  free(t->fwdp);
  free(t->inv);
  free(t->invp);
}

/* NttTables::forward (ntt.cpp:57-74): Cooley-Tukey, natural -> bit-reversed */
static void ntt_fwd_t(const tables_t* tb, u64* a) {
  const u64 q = tb->q, n = 1ull << tb->logn;
  u64 t = n;
  for (u64 m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (u64 i = 0; i < m; ++i) {
      const u64 w = tb->fwd[m + i], wp = tb->fwdp[m + i];
      const u64 j1 = 2 * i * t;
      for (u64 j = j1; j < j1 + t; ++j) {
        const u64 u = a[j];
        const u64 v = mul_shoup(a[j + t], w, wp, q);
        a[j] = addm(u, v, q);
        a[j + t] = subm(u, v, q);
      }
    }
  }
}

/* NttTables::inverse (ntt.cpp:76-96): Gentleman-Sande, bit-reversed -> natural, x n^-1 */
static void ntt_inv_t(const tables_t* tb, u64* a) {
  const u64 q = tb->q, n = 1ull << tb->logn;
  u64 t = 1;
  for (u64 m = n; m > 1; m >>= 1) {
    const u64 h = m >> 1;
    u64 j1 = 0;
    for (u64 i = 0; i < h; ++i) {
      const u64 w = tb->inv[h + i], wp = tb->invp[h + i];
      for (u64 j = j1; j < j1 + t; ++j) {
        const u64 u = a[j], v = a[j + t];
        a[j] = addm(u, v, q);
        a[j + t] = mul_shoup(subm(u, v, q), w, wp, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (u64 j = 0; j < n; ++j) a[j] = mul_shoup(a[j], tb->ninv, tb->ninvp, q);
}

void hxo_ntt_forward_limb(uint64_t q, uint64_t psi, int logn, uint64_t* a) {
  tables_t t;
  tables_init(&t, q, psi, logn);
  ntt_fwd_t(&t, a);
  tables_free(&t);
}

void hxo_ntt_inverse_limb(uint64_t q, uint64_t psi, int logn, uint64_t* a) {
  tables_t t;
  tables_init(&t, q, psi, logn);
  ntt_inv_t(&t, a);
  tables_free(&t);
}

/* schoolbook_negacyclic_mul (ntt.cpp:109-125) */
void hxo_schoolbook_negacyclic(uint64_t q, uint64_t n, const uint64_t* a, const uint64_t* b,
                               uint64_t* out) {
  memset(out, 0, n * 8);
  for (u64 i = 0; i < n; ++i)
    for (u64 j = 0; j < n; ++j) {
      const u64 p = hxo_mulmod(a[i], b[j], q);
      const u64 k = i + j;
      if (k < n)
        out[k] = addm(out[k], p, q);
      else
        out[k - n] = subm(out[k - n], p, q);
    }
}

/* ------------------------------------------------------------------------ */
/* context                                                 rns_poly.cpp:11-22 */
/* ------------------------------------------------------------------------ */

struct hxo_ctx {
  int logn;
  u64 n;
  int n_chain, n_special, alpha;
  u64 primes[HXO_MAX_PRIMES]; /* chain primes, then special primes */
  tables_t tb[HXO_MAX_PRIMES];
};

hxo_ctx* hxo_ctx_create(int logn, const uint64_t* chain, int n_chain, const uint64_t* special,
                        int n_special, int alpha) {
  if (n_chain + n_special > HXO_MAX_PRIMES || n_chain < 1 || alpha < 1) return NULL;
  hxo_ctx* c = (hxo_ctx*)calloc(1, sizeof(hxo_ctx));
  c->logn = logn;
  c->n = 1ull << logn;
  c->n_chain = n_chain;
  c->n_special = n_special;
  c->alpha = alpha;
  for (int i = 0; i < n_chain; ++i) c->primes[i] = chain[i];
  for (int k = 0; k < n_special; ++k) c->primes[n_chain + k] = special[k];
  const int total = n_chain + n_special;
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < total; ++i) {
    const u64 psi = hxo_find_psi(c->primes[i], c->n);
    tables_init(&c->tb[i], c->primes[i], psi, logn);
  }
  return c;
}

void hxo_ctx_destroy(hxo_ctx* c) {
  if (!c) return;
  for (int i = 0; i < c->n_chain + c->n_special; ++i) tables_free(&c->tb[i]);
  free(c);
}

uint64_t hxo_ctx_psi(const hxo_ctx* c, int i) { return c->tb[i].psi; }

int hxo_ctx_dnum(const hxo_ctx* c, int n_q) { return (n_q + c->alpha - 1) / c->alpha; }

void hxo_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* prime index of limb k of a poly with n_q chain limbs (then specials) --
 * LatticeContext::limb_modulus (rns_poly.cpp:24-27) generalised to K limbs */
static inline int pidx(const hxo_ctx* c, int k, int n_q) {
  return k < n_q ? k : c->n_chain + (k - n_q);
}

/* ------------------------------------------------------------------------ */
/* RNS poly ops                                           rns_poly.cpp:42-227 */
/* ------------------------------------------------------------------------ */

/* to_ntt (rns_poly.cpp:42-47) */
void hxo_ntt_fwd(const hxo_ctx* c, uint64_t* p, int n_q, int n_p) {
#pragma omp parallel for schedule(dynamic)
  for (int k = 0; k < n_q + n_p; ++k) ntt_fwd_t(&c->tb[pidx(c, k, n_q)], p + (u64)k * c->n);
}

/* to_coeff (rns_poly.cpp:49-54) */
void hxo_ntt_inv(const hxo_ctx* c, uint64_t* p, int n_q, int n_p) {
#pragma omp parallel for schedule(dynamic)
  for (int k = 0; k < n_q + n_p; ++k) ntt_inv_t(&c->tb[pidx(c, k, n_q)], p + (u64)k * c->n);
}

/* add (rns_poly.cpp:62-70) */
void hxo_add(const hxo_ctx* c, uint64_t* o, const uint64_t* a, const uint64_t* b, int n_q, int n_p) {
  const u64 n = c->n;
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t) o[k * n + t] = addm(a[k * n + t], b[k * n + t], q);
  }
}

/* sub (rns_poly.cpp:72-80) */
void hxo_sub(const hxo_ctx* c, uint64_t* o, const uint64_t* a, const uint64_t* b, int n_q, int n_p) {
  const u64 n = c->n;
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t) o[k * n + t] = subm(a[k * n + t], b[k * n + t], q);
  }
}

/* negate (rns_poly.cpp:82-89) */
void hxo_neg(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q, int n_p) {
  const u64 n = c->n;
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t) o[k * n + t] = negm(a[k * n + t], q);
  }
}

/* mul (rns_poly.cpp:91-100): pointwise, NTT domain */
void hxo_mul(const hxo_ctx* c, uint64_t* o, const uint64_t* a, const uint64_t* b, int n_q, int n_p) {
  const u64 n = c->n;
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t) o[k * n + t] = hxo_mulmod(a[k * n + t], b[k * n + t], q);
  }
}

/* mul_acc (rns_poly.cpp:102-110): acc += a (.) b */
void hxo_mul_acc(const hxo_ctx* c, uint64_t* acc, const uint64_t* a, const uint64_t* b, int n_q,
                 int n_p) {
  const u64 n = c->n;
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t)
      acc[k * n + t] = addm(acc[k * n + t], hxo_mulmod(a[k * n + t], b[k * n + t], q), q);
  }
}

/* automorphism (rns_poly.cpp:124-142): X^t -> X^(t g mod 2N), coefficient domain */
void hxo_automorphism_coeff(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q, int n_p,
                            uint64_t g) {
  const u64 n = c->n, two_n = 2 * n;
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t) {
      const u64 j = (u64)(((u128)t * g) % two_n);
      const u64 v = a[k * n + t];
      if (j < n)
        o[k * n + j] = v;
      else
        o[k * n + j - n] = negm(v, q);
    }
  }
}

/* NTT-domain form of the same map.  With NTT(a)[k] = a(psi^(2 brv(k)+1)):
 * NTT(tau_g a)[k] = NTT(a)[brv(((g (2 brv(k)+1)) mod 2N - 1) / 2)]. */
static inline u64 ntt_perm(u64 k, u64 g, int logn) {
  const u64 two_n = 2ull << logn;
  const u64 e = 2 * bitrev(k, logn) + 1;
  const u64 m = (u64)(((u128)g * e) % two_n);
  return bitrev((m - 1) >> 1, logn);
}

void hxo_automorphism_ntt(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q, int n_p,
                          uint64_t g) {
  const u64 n = c->n;
  u64* perm = (u64*)malloc(n * 8);
  for (u64 t = 0; t < n; ++t) perm[t] = ntt_perm(t, g, c->logn);
#pragma omp parallel for
  for (int k = 0; k < n_q + n_p; ++k)
    for (u64 t = 0; t < n; ++t) o[k * n + t] = a[k * n + perm[t]];
  free(perm);
}

/* rescale_drop_last (rns_poly.cpp:144-162): centred lift of the last limb,
 * out_i = (a_i - [c]_{q_i}) * q_last^-1 mod q_i; coefficient domain. */
void hxo_rescale_coeff(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q) {
  const u64 n = c->n;
  const u64 ql = c->primes[n_q - 1];
  const u64* last = a + (u64)(n_q - 1) * n;
#pragma omp parallel for
  for (int i = 0; i < n_q - 1; ++i) {
    const u64 q = c->primes[i];
    const u64 qinv = hxo_invmod(ql % q, q);
    for (u64 t = 0; t < n; ++t) {
      const u64 diff = subm(a[i * n + t], reduce_i64(centered(last[t], ql), q), q);
      o[i * n + t] = hxo_mulmod(diff, qinv, q);
    }
  }
}

void hxo_rescale_ntt(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q) {
  const u64 n = c->n;
  u64* tmp = (u64*)malloc((u64)n_q * n * 8);
  memcpy(tmp, a, (u64)n_q * n * 8);
  hxo_ntt_inv(c, tmp, n_q, 0);
  hxo_rescale_coeff(c, o, tmp, n_q);
  hxo_ntt_fwd(c, o, n_q - 1, 0);
  free(tmp);
}

/* Centred FastBConv ModDown over the K special primes (generalises
 * moddown_special, rns_poly.cpp:164-180, which is the K = 1 case):
 *   x_k = [a_{p_k} * (P/p_k)^-1]_{p_k},  v = sum_k centred(x_k) * (P/p_k)
 *   out_i = (a_i - [v]_{q_i}) * P^-1 mod q_i
 * coefficient domain; a has n_q + K limbs. */
void hxo_moddown_coeff(const hxo_ctx* c, uint64_t* o, const uint64_t* a, int n_q) {
  const u64 n = c->n;
  const int K = c->n_special;
  const u64* sp = a + (u64)n_q * n;
  u64 phat_inv[HXO_MAX_PRIMES];
  for (int k = 0; k < K; ++k) {
    const u64 pk = c->primes[c->n_chain + k];
    u64 prod = 1;
    for (int k2 = 0; k2 < K; ++k2)
      if (k2 != k) prod = hxo_mulmod(prod, c->primes[c->n_chain + k2] % pk, pk);
    phat_inv[k] = hxo_invmod(prod, pk);
  }
  u64* x = (u64*)malloc((u64)K * n * 8);
  for (int k = 0; k < K; ++k) {
    const u64 pk = c->primes[c->n_chain + k];
    for (u64 t = 0; t < n; ++t) x[k * n + t] = hxo_mulmod(sp[k * n + t], phat_inv[k], pk);
  }
#pragma omp parallel for
  for (int i = 0; i < n_q; ++i) {
    const u64 q = c->primes[i];
    u64 phat_q[HXO_MAX_PRIMES];
    u64 P_q = 1;
    for (int k = 0; k < K; ++k) {
      u64 prod = 1;
      for (int k2 = 0; k2 < K; ++k2)
        if (k2 != k) prod = hxo_mulmod(prod, c->primes[c->n_chain + k2] % q, q);
      phat_q[k] = prod;
      P_q = hxo_mulmod(P_q, c->primes[c->n_chain + k] % q, q);
    }
    const u64 pinv = hxo_invmod(P_q, q);
    for (u64 t = 0; t < n; ++t) {
      u64 v = 0;
      for (int k = 0; k < K; ++k) {
        const u64 pk = c->primes[c->n_chain + k];
        const u64 xr = reduce_i64(centered(x[k * n + t], pk), q);
        v = addm(v, hxo_mulmod(xr, phat_q[k], q), q);
      }
      o[i * n + t] = hxo_mulmod(subm(a[i * n + t], v, q), pinv, q);
    }
  }
  free(x);
}

/* from_i64 (rns_poly.cpp:218-227) */
void hxo_from_i64(const hxo_ctx* c, uint64_t* o, const int64_t* v, int n_q, int n_p) {
  const u64 n = c->n;
  for (int k = 0; k < n_q + n_p; ++k) {
    const u64 q = c->primes[pidx(c, k, n_q)];
    for (u64 t = 0; t < n; ++t) o[k * n + t] = reduce_i64(v[t], q);
  }
}

/* ------------------------------------------------------------------------ */
/* hybrid key switching  (K > 1 / alpha > 1 is the  */
/* builder's restatement -- no reference code exists for it)                 */
/* ------------------------------------------------------------------------ */

/* ModUp: digit d = limbs [d*alpha, min((d+1)*alpha, n_q)); non-centred
 * FastBConv y_j = sum_{i in d} [x_i (Qhat_i)^-1]_{q_i} [Qhat_i]_{p_j} to every
 * other chain limb and every special limb, then NTT.  The digit's own limbs
 * are the input limbs (unchanged, already NTT form). */
void hxo_modup(const hxo_ctx* c, uint64_t* digits, const uint64_t* c1_ntt, int n_q) {
  const u64 n = c->n;
  const int K = c->n_special, ext = n_q + K;
  const int dnum = hxo_ctx_dnum(c, n_q);
  u64* coef = (u64*)malloc((u64)n_q * n * 8);
  memcpy(coef, c1_ntt, (u64)n_q * n * 8);
  hxo_ntt_inv(c, coef, n_q, 0);
  for (int d = 0; d < dnum; ++d) {
    const int lo = d * c->alpha;
    const int hi = (lo + c->alpha < n_q) ? lo + c->alpha : n_q;
    u64* out = digits + (u64)d * ext * n;
    u64 qhat_inv[HXO_MAX_PRIMES];
    for (int i = lo; i < hi; ++i) {
      const u64 q = c->primes[i];
      u64 prod = 1;
      for (int i2 = lo; i2 < hi; ++i2)
        if (i2 != i) prod = hxo_mulmod(prod, c->primes[i2] % q, q);
      qhat_inv[i - lo] = hxo_invmod(prod, q);
    }
    /* x_i = [a_i * qhat_inv_i]_{q_i} */
    u64* x = (u64*)malloc((u64)(hi - lo) * n * 8);
    for (int i = lo; i < hi; ++i)
      for (u64 t = 0; t < n; ++t)
        x[(i - lo) * n + t] = hxo_mulmod(coef[i * n + t], qhat_inv[i - lo], c->primes[i]);
#pragma omp parallel for schedule(dynamic)
    for (int j = 0; j < ext; ++j) {
      u64* dst = out + (u64)j * n;
      if (j >= lo && j < hi) {
        memcpy(dst, c1_ntt + (u64)j * n, n * 8);
        continue;
      }
      const int pj = pidx(c, j, n_q);
      const u64 p = c->primes[pj];
      u64 qhat_p[HXO_MAX_PRIMES];
      for (int i = lo; i < hi; ++i) {
        u64 prod = 1;
        for (int i2 = lo; i2 < hi; ++i2)
          if (i2 != i) prod = hxo_mulmod(prod, c->primes[i2] % p, p);
        qhat_p[i - lo] = prod;
      }
      for (u64 t = 0; t < n; ++t) {
        u64 y = 0;
        for (int i = lo; i < hi; ++i) y = addm(y, hxo_mulmod(x[(i - lo) * n + t], qhat_p[i - lo], p), p);
        dst[t] = y;
      }
      ntt_fwd_t(&c->tb[pj], dst);
    }
    free(x);
  }
  free(coef);
}

/* U_c[j] = sum_d tau_g(D_d)[j] (.) key_{d,c}[j]  (mul_acc, rns_poly.cpp:102-110,
 * with the NTT-domain automorphism folded into the digit read). */
void hxo_ks_inner(const hxo_ctx* c, uint64_t* u, const uint64_t* digits, const uint64_t* key,
                  int n_q, uint64_t g) {
  const u64 n = c->n;
  const int K = c->n_special, ext = n_q + K, full = c->n_chain + K;
  const int dnum = hxo_ctx_dnum(c, n_q);
  u64* perm = (u64*)malloc(n * 8);
  for (u64 t = 0; t < n; ++t) perm[t] = (g == 1) ? t : ntt_perm(t, g, c->logn);
#pragma omp parallel for schedule(dynamic)
  for (int cj = 0; cj < 2 * ext; ++cj) {
    const int cc = cj / ext, j = cj % ext;
    const int kl = pidx(c, j, n_q); /* key limb index over the full basis */
    const u64 p = c->primes[kl];
    u64* dst = u + ((u64)cc * ext + j) * n;
    for (u64 t = 0; t < n; ++t) dst[t] = 0;
    for (int d = 0; d < dnum; ++d) {
      const u64* D = digits + ((u64)d * ext + j) * n;
      const u64* kk = key + (((u64)d * 2 + cc) * full + kl) * n;
      for (u64 t = 0; t < n; ++t) dst[t] = addm(dst[t], hxo_mulmod(D[perm[t]], kk[t], p), p);
    }
  }
  free(perm);
}

/* NTT-domain ModDown of n_polys PQ-basis polys (INTT, centred ModDown, NTT) */
void hxo_moddown_ntt(const hxo_ctx* c, uint64_t* o, const uint64_t* u, int n_q, int n_polys) {
  const u64 n = c->n;
  const int ext = n_q + c->n_special;
  u64* tmp = (u64*)malloc((u64)ext * n * 8);
  for (int pl = 0; pl < n_polys; ++pl) {
    memcpy(tmp, u + (u64)pl * ext * n, (u64)ext * n * 8);
    hxo_ntt_inv(c, tmp, n_q, c->n_special);
    hxo_moddown_coeff(c, o + (u64)pl * n_q * n, tmp, n_q);
    hxo_ntt_fwd(c, o + (u64)pl * n_q * n, n_q, 0);
  }
  free(tmp);
}

void hxo_keyswitch(const hxo_ctx* c, uint64_t* out, const uint64_t* in_ntt, const uint64_t* key,
                   int n_q) {
  const u64 n = c->n;
  const int ext = n_q + c->n_special, dnum = hxo_ctx_dnum(c, n_q);
  u64* D = (u64*)malloc((u64)dnum * ext * n * 8);
  u64* U = (u64*)malloc((u64)2 * ext * n * 8);
  hxo_modup(c, D, in_ntt, n_q);
  hxo_ks_inner(c, U, D, key, n_q, 1);
  hxo_moddown_ntt(c, out, U, n_q, 2);
  free(D);
  free(U);
}

static void rotate_from_digits(const hxo_ctx* c, uint64_t* out_ct, const uint64_t* in_ct,
                               const uint64_t* D, const uint64_t* key, int n_q, uint64_t g) {
  const u64 n = c->n;
  const int ext = n_q + c->n_special;
  u64* U = (u64*)malloc((u64)2 * ext * n * 8);
  u64* V = (u64*)malloc((u64)2 * n_q * n * 8);
  u64* r0 = (u64*)malloc((u64)n_q * n * 8);
  hxo_ks_inner(c, U, D, key, n_q, g);
  hxo_moddown_ntt(c, V, U, n_q, 2);
  hxo_automorphism_ntt(c, r0, in_ct, n_q, 0, g);
  hxo_add(c, out_ct, r0, V, n_q, 0);
  memcpy(out_ct + (u64)n_q * n, V + (u64)n_q * n, (u64)n_q * n * 8);
  free(U);
  free(V);
  free(r0);
}

/* galois_rotate under the hoisting convention */
void hxo_rotate(const hxo_ctx* c, uint64_t* out_ct, const uint64_t* in_ct, const uint64_t* key,
                int n_q, uint64_t g) {
  const u64 n = c->n;
  const int ext = n_q + c->n_special, dnum = hxo_ctx_dnum(c, n_q);
  u64* D = (u64*)malloc((u64)dnum * ext * n * 8);
  hxo_modup(c, D, in_ct + (u64)n_q * n, n_q);
  rotate_from_digits(c, out_ct, in_ct, D, key, n_q, g);
  free(D);
}

void hxo_rotate_hoisted(const hxo_ctx* c, uint64_t* out_cts, const uint64_t* in_ct,
                        const uint64_t* const* keys, const uint64_t* gs, int R, int n_q) {
  const u64 n = c->n;
  const int ext = n_q + c->n_special, dnum = hxo_ctx_dnum(c, n_q);
  u64* D = (u64*)malloc((u64)dnum * ext * n * 8);
  hxo_modup(c, D, in_ct + (u64)n_q * n, n_q);
  for (int r = 0; r < R; ++r)
    rotate_from_digits(c, out_cts + (u64)r * 2 * n_q * n, in_ct, D, keys[r], n_q, gs[r]);
  free(D);
}

/* tensor: LatticeContext::mul x4 (rns_poly.cpp:91-100) */
void hxo_tensor(const hxo_ctx* c, uint64_t* out3, const uint64_t* a, const uint64_t* b, int n_q) {
  const u64 L = (u64)n_q * c->n;
  hxo_mul(c, out3, a, b, n_q, 0);
  hxo_mul(c, out3 + L, a, b + L, n_q, 0);
  hxo_mul_acc(c, out3 + L, a + L, b, n_q, 0);
  hxo_mul(c, out3 + 2 * L, a + L, b + L, n_q, 0);
}

void hxo_mul_relin(const hxo_ctx* c, uint64_t* out_ct, const uint64_t* a, const uint64_t* b,
                   const uint64_t* rlk, int n_q) {
  const u64 L = (u64)n_q * c->n;
  u64* d = (u64*)malloc(3 * L * 8);
  u64* u = (u64*)malloc(2 * L * 8);
  hxo_tensor(c, d, a, b, n_q);
  hxo_keyswitch(c, u, d + 2 * L, rlk, n_q);
  hxo_add(c, out_ct, d, u, n_q, 0);
  hxo_add(c, out_ct + L, d + L, u + L, n_q, 0);
  free(d);
  free(u);
}

/* BSGS inner sums: inner_j = sum_k diag'_{n1 j + k} (.) Rot_k(x) */
void hxo_bsgs_mac(const hxo_ctx* c, uint64_t* inner, const uint64_t* baby, const uint64_t* diags,
                  int n1, int n2, int n_q) {
  const u64 n = c->n, L = (u64)n_q * n;
#pragma omp parallel for schedule(dynamic)
  for (int ji = 0; ji < n2 * n_q; ++ji) {
    const int j = ji / n_q, i = ji % n_q;
    const u64 q = c->primes[i];
    for (int cc = 0; cc < 2; ++cc) {
      u64* dst = inner + ((u64)j * 2 + cc) * L + (u64)i * n;
      for (u64 t = 0; t < n; ++t) dst[t] = 0;
      for (int k = 0; k < n1; ++k) {
        const u64* dg = diags + (u64)(j * n1 + k) * L + (u64)i * n;
        const u64* bb = baby + ((u64)k * 2 + cc) * L + (u64)i * n;
        for (u64 t = 0; t < n; ++t) dst[t] = addm(dst[t], hxo_mulmod(dg[t], bb[t], q), q);
      }
    }
  }
}

/* ------------------------------------------------------------------------ */
/* keys and encryption                            */
/* ------------------------------------------------------------------------ */

/* ksk_d = (-a_d s + e_d + [P]_{q_i} s' on chain limbs i of digit d, a_d) */
void hxo_keygen_ksk(const hxo_ctx* c, uint64_t* key, const uint64_t* s_full,
                    const uint64_t* sp_full, const uint64_t* a_full, const int64_t* e) {
  const u64 n = c->n;
  const int K = c->n_special, full = c->n_chain + K;
  const int dnum = hxo_ctx_dnum(c, c->n_chain);
  u64* en = (u64*)malloc((u64)full * n * 8);
  for (int d = 0; d < dnum; ++d) {
    const int lo = d * c->alpha;
    const int hi = (lo + c->alpha < c->n_chain) ? lo + c->alpha : c->n_chain;
    hxo_from_i64(c, en, e + (u64)d * n, c->n_chain, K);
    hxo_ntt_fwd(c, en, c->n_chain, K);
    u64* b = key + ((u64)d * 2 + 0) * full * n;
    u64* a = key + ((u64)d * 2 + 1) * full * n;
    const u64* ad = a_full + (u64)d * full * n;
    for (int l = 0; l < full; ++l) {
      const u64 q = c->primes[l];
      u64 Pq = 0;
      if (l >= lo && l < hi) {
        Pq = 1;
        for (int k = 0; k < K; ++k) Pq = hxo_mulmod(Pq, c->primes[c->n_chain + k] % q, q);
      }
      for (u64 t = 0; t < n; ++t) {
        const u64 as = hxo_mulmod(ad[l * n + t], s_full[l * n + t], q);
        u64 v = subm(en[l * n + t], as, q);
        if (Pq) v = addm(v, hxo_mulmod(Pq, sp_full[l * n + t], q), q);
        b[l * n + t] = v;
        a[l * n + t] = ad[l * n + t];
      }
    }
  }
  free(en);
}

void hxo_decrypt(const hxo_ctx* c, uint64_t* m_out, const uint64_t* ct, const uint64_t* s_full,
                 int n_q) {
  const u64 L = (u64)n_q * c->n;
  memcpy(m_out, ct, L * 8);
  hxo_mul_acc(c, m_out, ct + L, s_full, n_q, 0);
}

void hxo_encrypt_sk(const hxo_ctx* c, uint64_t* ct, const uint64_t* m_ntt, const uint64_t* s_full,
                    const uint64_t* a, const int64_t* e, int n_q) {
  const u64 n = c->n, L = (u64)n_q * n;
  u64* en = (u64*)malloc(L * 8);
  hxo_from_i64(c, en, e, n_q, 0);
  hxo_ntt_fwd(c, en, n_q, 0);
  for (int i = 0; i < n_q; ++i) {
    const u64 q = c->primes[i];
    for (u64 t = 0; t < n; ++t) {
      const u64 idx = (u64)i * n + t;
      u64 v = subm(addm(m_ntt[idx], en[idx], q), hxo_mulmod(a[idx], s_full[idx], q), q);
      ct[idx] = v;
      ct[L + idx] = a[idx];
    }
  }
  free(en);
}

/* ------------------------------------------------------------------------ */
/* linear-algebra drivers (reference kernels.cpp is missing, */
/* proj/CMakeLists.txt:22) -- the schedules the product runs                 */
/* (paper_2512_11135_b200/csrc/host/linalg.cpp, gpu_backend.cpp), restated   */
/* over the primitives above.  Modular sums are order independent, so only   */
/* the set of terms, the rotations and the rescale / ModDown placement pin    */
/* the output words.                                                          */
/* ------------------------------------------------------------------------ */

static u64 reduce_amount(int64_t r, u64 slots) {
  const int64_t s = (int64_t)slots;
  return (u64)(((r % s) + s) % s);
}

/* Rot_r(ct) with the standard-layout key keys[r]; r == 0 copies */
static void rot_by(const hxo_ctx* c, u64* out, const u64* ct, int64_t amount, const uint64_t* const* keys,
                   int n_q) {
  const u64 slots = c->n / 2, r = reduce_amount(amount, slots);
  if (r == 0) {
    memcpy(out, ct, (u64)2 * n_q * c->n * 8);
    return;
  }
  u64 g = 1;
  for (u64 i = 0; i < r; ++i) g = (g * 5) % (2 * c->n);
  hxo_rotate(c, out, ct, keys[r], n_q, g);
}

static void ct_add(const hxo_ctx* c, u64* acc, const u64* x, int n_q) {
  hxo_add(c, acc, acc, x, n_q, 0);
  hxo_add(c, acc + (u64)n_q * c->n, acc + (u64)n_q * c->n, x + (u64)n_q * c->n, n_q, 0);
}

static void ct_mul_plain(const hxo_ctx* c, u64* out, const u64* x, const u64* pt, int n_q) {
  hxo_mul(c, out, x, pt, n_q, 0);
  hxo_mul(c, out + (u64)n_q * c->n, x + (u64)n_q * c->n, pt, n_q, 0);
}

static void ct_rescale(const hxo_ctx* c, u64* out, const u64* x, int n_q) {
  hxo_rescale_ntt(c, out, x, n_q);
  hxo_rescale_ntt(c, out + (u64)(n_q - 1) * c->n, x + (u64)n_q * c->n, n_q);
}

static u64 galois_of(const hxo_ctx* c, u64 r) {
  u64 g = 1;
  for (u64 i = 0; i < r; ++i) g = (g * 5) % (2 * c->n);
  return g;
}

void hxo_matvec_bsgs(const hxo_ctx* c, uint64_t* out, const uint64_t* x, int n_q, int n1, int n2, int blocks,
                     const uint64_t* const* diags, const uint64_t* const* keys, int giant_begin, int giant_end,
                     int rescale, int lazy, int partial) {
  const u64 n = c->n, L = (u64)n_q * n, ct = 2 * L;
  if (partial) {
    lazy = 1;
    rescale = 0;
  }
  const int K = c->n_special, ext = n_q + K;
  const int gb = giant_begin, ge = giant_end < 0 ? n2 : giant_end;
  /* baby steps Rot_k(x), k < n1: one ModUp shared by all (hoisting convention) */
  u64* baby = (u64*)malloc((u64)n1 * ct * 8);
  memcpy(baby, x, ct * 8);
  if (n1 > 1) {
    const uint64_t** kk = (const uint64_t**)malloc(sizeof(void*) * (n1 - 1));
    u64* gs = (u64*)malloc(8 * (n1 - 1));
    for (int k = 1; k < n1; ++k) {
      kk[k - 1] = keys[k];
      gs[k - 1] = galois_of(c, (u64)k);
    }
    hxo_rotate_hoisted(c, baby + ct, x, kk, gs, n1 - 1, n_q);
    free(kk);
    free(gs);
  }
  u64* inner = (u64*)malloc(ct * 8);
  u64* acc = (u64*)malloc(ct * 8);
  u64* tmp = (u64*)malloc(ct * 8);
  u64* S = (u64*)malloc((u64)2 * ext * n * 8);
  u64* U = (u64*)malloc((u64)2 * ext * n * 8);
  u64* D = (u64*)malloc((u64)hxo_ctx_dnum(c, n_q) * ext * n * 8);
  const u64 slots = n / 2;
  for (int b = 0; b < blocks; ++b) {
    memset(acc, 0, ct * 8);
    memset(S, 0, (u64)2 * ext * n * 8);
    int any_giant = 0;
    for (int j = gb; j < ge; ++j) {
      int live = 0;
      memset(inner, 0, ct * 8);
      for (int k = 0; k < n1; ++k) {
        const uint64_t* dg = diags[(u64)b * n1 * n2 + (u64)j * n1 + k];
        if (!dg) continue;
        live = 1;
        hxo_mul_acc(c, inner, baby + (u64)k * ct, dg, n_q, 0);
        hxo_mul_acc(c, inner + L, baby + (u64)k * ct + L, dg, n_q, 0);
      }
      if (!live) continue;
      if (j == 0) {
        ct_add(c, acc, inner, n_q);
      } else if (!lazy) {
        rot_by(c, tmp, inner, (int64_t)n1 * j, keys, n_q);
        ct_add(c, acc, tmp, n_q);
      } else { /* double hoisting: tau_j(c0) into acc, the PQ-basis key-switch sum into S */
        const u64 r = reduce_amount((int64_t)n1 * j, slots), g = galois_of(c, r);
        hxo_modup(c, D, inner + L, n_q);
        hxo_ks_inner(c, U, D, keys[r], n_q, g);
        hxo_add(c, S, S, U, n_q, K);
        hxo_add(c, S + (u64)ext * n, S + (u64)ext * n, U + (u64)ext * n, n_q, K);
        hxo_automorphism_ntt(c, tmp, inner, n_q, 0, g);
        hxo_add(c, acc, acc, tmp, n_q, 0);
        any_giant = 1;
      }
    }
    if (partial) { /* giant-step shard: [T][S], the ModDown after the ranks' sum */
      u64* o = out + (u64)b * (ct + (u64)2 * ext * n);
      memcpy(o, acc, ct * 8);
      memcpy(o + ct, S, (u64)2 * ext * n * 8);
      continue;
    }
    if (any_giant) { /* one ModDown per output */
      hxo_moddown_ntt(c, tmp, S, n_q, 2);
      ct_add(c, acc, tmp, n_q);
    }
    if (rescale)
      ct_rescale(c, out + (u64)b * 2 * (n_q - 1) * n, acc, n_q);
    else
      memcpy(out + (u64)b * ct, acc, ct * 8);
  }
  free(baby);
  free(inner);
  free(acc);
  free(tmp);
  free(S);
  free(U);
  free(D);
}

/* packed-row matvec with the assembly of DESIGN.md s3.9
 * (SPEC.md:422 leaves it unpinned): per payload g, t = rescale(x (.) rows_g),
 * t += Rot(t, s) for s = 1, 2, .., pad_cols / 2; for r < p (row = g p + r <
 * rows): u = t (.) mask_r, u = Rot(u, r pad_cols - row) unless that is 0 mod
 * slots, acc += u; out = rescale(acc). */
void hxo_matvec_row(const hxo_ctx* c, uint64_t* out, const uint64_t* x, int n_q, int groups, int p, int rows,
                    int pad_cols, const uint64_t* const* rows_pts, const uint64_t* const* masks,
                    const uint64_t* const* keys) {
  const u64 n = c->n, slots = n / 2;
  const int n1q = n_q - 1;
  const u64 ct = 2 * (u64)n_q * n, ct1 = 2 * (u64)n1q * n;
  u64* m = (u64*)malloc(ct * 8);
  u64* t = (u64*)malloc(ct1 * 8);
  u64* r1 = (u64*)malloc(ct1 * 8);
  u64* u = (u64*)malloc(ct1 * 8);
  u64* acc = (u64*)calloc(ct1, 8);
  for (int g = 0; g < groups; ++g) {
    ct_mul_plain(c, m, x, rows_pts[g], n_q);
    ct_rescale(c, t, m, n_q);
    for (int s = 1; s < pad_cols; s <<= 1) {
      rot_by(c, r1, t, s, keys, n1q);
      ct_add(c, t, r1, n1q);
    }
    for (int r = 0; r < p; ++r) {
      const int row = g * p + r;
      if (row >= rows) break;
      ct_mul_plain(c, u, t, masks[r], n1q);
      const int64_t shift = (int64_t)r * pad_cols - row;
      if (reduce_amount(shift, slots) != 0) {
        rot_by(c, r1, u, shift, keys, n1q);
        ct_add(c, acc, r1, n1q);
      } else {
        ct_add(c, acc, u, n1q);
      }
    }
  }
  ct_rescale(c, out, acc, n1q);
  free(m);
  free(t);
  free(r1);
  free(u);
  free(acc);
}

/* ct-ct matmul as DESIGN.md s3.10 schedules
 * it: a_j = rescale(A (.) colmask_j), b_j = rescale(B (.) rowmask_j), a_j =
 * Rot(a_j, j), b_j = Rot(b_j, d j) for j >= 1; a_j += Rot(a_j, -2^i), b_j +=
 * Rot(b_j, -d 2^i) for i < log2 d; out = rescale(sum_j mul_relin(a_j, b_j)). */
void hxo_matmul_ctct(const hxo_ctx* c, uint64_t* out, const uint64_t* A, const uint64_t* B, int n_q, int d,
                     const uint64_t* const* colmask, const uint64_t* const* rowmask, const uint64_t* rlk,
                     const uint64_t* const* keys) {
  const u64 n = c->n;
  const int nb = n_q - 1;
  const u64 ct = 2 * (u64)n_q * n, cb = 2 * (u64)nb * n;
  int lg = 0;
  while ((1 << lg) < d) ++lg;
  u64* m = (u64*)malloc(ct * 8);
  u64* a = (u64*)malloc(cb * 8);
  u64* bb = (u64*)malloc(cb * 8);
  u64* t = (u64*)malloc(cb * 8);
  u64* pr = (u64*)malloc(cb * 8);
  u64* C = (u64*)calloc(cb, 8);
  for (int j = 0; j < d; ++j) {
    ct_mul_plain(c, m, A, colmask[j], n_q);
    ct_rescale(c, a, m, n_q);
    ct_mul_plain(c, m, B, rowmask[j], n_q);
    ct_rescale(c, bb, m, n_q);
    if (j) {
      rot_by(c, t, a, j, keys, nb);
      memcpy(a, t, cb * 8);
      rot_by(c, t, bb, (int64_t)d * j, keys, nb);
      memcpy(bb, t, cb * 8);
    }
    for (int i = 0; i < lg; ++i) {
      rot_by(c, t, a, -((int64_t)1 << i), keys, nb);
      ct_add(c, a, t, nb);
    }
    for (int i = 0; i < lg; ++i) {
      rot_by(c, t, bb, -((int64_t)d << i), keys, nb);
      ct_add(c, bb, t, nb);
    }
    hxo_mul_relin(c, pr, a, bb, rlk, nb);
    ct_add(c, C, pr, nb);
  }
  ct_rescale(c, out, C, nb);
  free(m);
  free(a);
  free(bb);
  free(t);
  free(pr);
  free(C);
}
