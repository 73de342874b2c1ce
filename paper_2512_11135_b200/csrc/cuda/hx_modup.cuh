// hx_modup.cuh -- ModUp basis conversion fused into the first (COL) pass of
// the forward NTT of the extended limbs.
//
// Replaces, for every digit d of c1 (coefficient domain after the INTT),
//   bconv -> [P_d]-basis limb j (coefficient domain)      (FastBConv, non-centred:
//            the hybrid ModUp of the SPEC key switch, SPEC.md:193-201 / :229 --
//            the reference has no ModUp code; K = 1 lifts per limb, rns_poly.cpp:218-227)
//   NTT COL pass on limb j                                 (ntt.cpp:57-74, first stages)
// with one kernel: a CTA owns one COL tile (2^OB adjacent columns x 2^S rows)
// of one digit of one ciphertext.  It loads the digit's alpha source limbs of
// the tile once, forms x_i = [a_i (Qhat_i)^-1]_{q_i} into shared memory, then
// loops over the digit's target limbs of one prime class: the conversion of a
// target word is computed straight into the butterfly registers, the COL
// stages run, and the tile is stored.  The extended limbs therefore never
// exist in HBM in the coefficient domain (saves one write + one read of
// 8 x 24 limbs per ciphertext at config 2) and the conversion's FP64 work
// overlaps the NTT's.  The ROW pass of those limbs is the ordinary ROW launch.
//
// Exactness: FP64-class targets (p < 2^47): x_i < 2^47 sources enter as exact
// doubles, each product by mulmod_f64 (exact); a 60-bit source (q_0, the
// ModDown specials) either by an integer Shoup product in [0, 2p) converted
// exactly (HX_WIDE_INT, every third wide source: all of them on the integer
// pipe measured slower, 5.23 vs 5.05 ms for ModDown's conversion) or as
// x = xh 2^30 + xl, two exact doubles and the constant [2^30 Qhat_i]_p; the sum kept lazily in (-(2 alpha + K) p,
// 2 alpha p): the forward FP64 NTT grows values by < p per stage, so
// |v| < (2 alpha + K + logn) p < 2^52 and |v w| < 2^99.  Integer
// targets (60-bit q_0 and special primes): Shoup products, sum in [0, 2p).
#pragma once

#include "hx_common.cuh"
#include "hx_ntt.cuh"
#include "hx_types.cuh"

namespace hx {

// conversion constant of (source limb i of the digit, target limb j):
// w = [Qhat_i]_{p_j}; FP64 form (w, w / p), (w30, w30 / p) with w30 = [2^30 w]_p;
// integer form (w, Shoup w').
// The *1 members are the same constants times the first forward twiddle
// psi^(N/2) (tw[1]) of the target prime: the words of the upper half of the
// first butterfly stage are converted with them, which IS that stage's
// twiddle product (the stage has one twiddle), so the stage multiplies nothing.
struct BconvC {
  double w, wq, w30, w30q;
  u64 sw, swp;
  double w1, w301;
  u64 sw1, swp1;
};

constexpr int kMaxDigits = 64;

struct ModUpColArgs {
  const u64* coef;        // [batch][n_q][N] coefficient-domain c1
  u64* out;               // [batch][dnum][ext][N] extended digits
  const PrimeConst* pc;
  const SC* qhinv;        // per digit at qh_off[d]: [alpha]
  const BconvC* bc;       // per digit at bc_off[d]: [ext][alpha]
  const int* tlist;       // per digit at toff[d]: tcnt[d] target limbs j (this class)
  long long qh_off[kMaxDigits], bc_off[kMaxDigits];
  // per digit: tcnt[d] FP64-class targets (conversion + COL pass) followed by
  // icnt[d] integer-class targets (conversion only, coefficient domain out)
  int toff[kMaxDigits], tcnt[kMaxDigits], icnt[kMaxDigits];
  int alpha, n_q, n_chain, ext, dnum, logn;
  // sources: src_n limbs per element in `coef`, digit d's limb i has prime
  // index src_pbase + d alpha + i (ModUp: n_q, 0; ModDown: K, n_chain)
  int src_n, src_pbase;
  // ModDown (centred conversion, rns_poly.cpp:164-180 with K specials):
  // subtract nneg [P]_{q_j}, nneg = #{k : x_k > p_k / 2} per word
  int centred;
  const double* pmf;  // [n_chain] [P]_{q_j} as double (FP64-class targets)
  const double* pmf1; // [n_chain] [P tw1]_{q_j} (upper half of the folded first stage)
  // joint reduction of a word's alpha products (bconv_tile_f64): 1.5 * 2^E with
  // sum_i x_i w_i < 2^(E-1); the host checks E against the rint range
  double cs_round;
  const u64* pmu;     // [n_chain] [P]_{q_j}
  // target split: blockIdx.y = element * tsplit + part; part p converts the
  // p-th share of the digit's target list (small batches still fill the GPU;
  // each part re-reads the alpha source tiles, from L2)
  int tsplit;
};

// bconv of one tile word (sources at src[i * stride]) into the working
// representation of the target class
// Source-class modes (fixed per digit, so a CTA runs one straight-line body and
// the instruction cache holds one variant): 0 every source limb < 2^47,
// 1 source 0 is the wide q_0 and the rest < 2^47 (config 2's digit 0),
// 2 any mix (runtime test per source), 3 every source wide (ModDown from
// 60-bit special primes).
template <int SRC, int MAXA>
__device__ __forceinline__ bool src_is_f64(const bool (&sf64)[MAXA], int i) {
  return SRC == 0 ? true : SRC == 1 ? (i != 0) : SRC == 3 ? false : sf64[i];
}

template <bool F64, int MAXA, int SRC = 2>
__device__ __forceinline__ u64 bconv_word(const u64* src, int stride, int cnt, const bool (&sf64)[MAXA],
                                          const BconvC* C, const PrimeConst& P) {
  if (F64) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < MAXA; ++i) {
      if (i < cnt) {
        const u64 v = src[i * stride];
        if (src_is_f64<SRC, MAXA>(sf64, i)) {
          acc = __dadd_rn(acc, mulmod_f64(__longlong_as_double((long long)v), C[i].w, C[i].wq, P.qd));
        } else {  // 60-bit source: x = xh 2^30 + xl
          const double xh = __dsub_rn(__longlong_as_double((long long)((v >> 30) | 0x4330000000000000ull)), kTwo52);
          const double xl =
              __dsub_rn(__longlong_as_double((long long)((v & 0x3FFFFFFFull) | 0x4330000000000000ull)), kTwo52);
          acc = __dadd_rn(acc, mulmod_f64(xh, C[i].w30, C[i].w30q, P.qd));
          acc = __dadd_rn(acc, mulmod_f64(xl, C[i].w, C[i].wq, P.qd));
        }
      }
    }
    return (u64)__double_as_longlong(acc);
  } else {
    u64 y = 0;
#pragma unroll
    for (int i = 0; i < MAXA; ++i) {
      if (i < cnt) {
        u64 v = src[i * stride];
        if (sf64[i])  // exact double -> integer
          v = (u64)__double_as_longlong(__dadd_rn(__longlong_as_double((long long)v), kTwo52)) & 0xFFFFFFFFFFFFFull;
        y = csub(y + shoup_lazy(v, C[i].sw, C[i].swp, P.q), P.two_q);
      }
    }
    return y;
  }
}

// bconv of the 16 words a thread owns in the first COL group (tile elements
// e_r = eb[r >> W] | (r mod 2^W) << lowbits), sources outer / words inner: the
// source tests are uniform, so the 16 products of a source are independent
// FP64 chains the scheduler interleaves (a per-word bconv_word puts a branch
// between every product and leaves one dependent chain in flight).
#ifndef HX_WIDE_INT
#define HX_WIDE_INT 1
#endif
constexpr bool kWideInt = HX_WIDE_INT != 0;
#ifndef HX_MODUP_INT0
#define HX_MODUP_INT0 0
#endif
constexpr bool kModUpInt0 = HX_MODUP_INT0 != 0;
#ifndef HX_MODUP_MINB
#define HX_MODUP_MINB 3
#endif

// Joint reduction: the alpha (or 2 alpha, wide sources) products x_i w_i of a
// word are summed EXACTLY before one reduction mod p.  A running sum S starts
// at cs = 1.5 * 2^E and stays in the binade [2^E, 2^(E+1)) (sum < 2^(E-1)), so
// every S' = fma(x, w, S) rounds x w to a multiple of G = 2^(E-52):
//   d = S' - S       (exact: same binade)     = x w rounded to a multiple of G
//   l = fma(x, w, -d)(exact: |l| <= G / 2, an integer below 2^53)
// and sum_i x_i w_i = (S_last - cs) + sum_i l_i with both parts exact.  One
// quotient, qf = rint(H / p) with H = S_last - cs (|H / p| < 2^51, checked on
// the host), leaves r = H - qf p exactly (one FMA), and the word is r + L,
// |r + L| < p + alpha G.  3 FP64 ops per product + 7 per word instead of 7
// per product (mulmod_f64 + add): 16 instead of 21 for alpha = 3.
// HB: the words r with bit WW-1 set are the lower inputs of the first
// butterfly stage; they are converted with the constants premultiplied by
// that stage's single twiddle (BconvC::w1 ...), so the stage adds / subtracts
// only (ntt_group_f64 SKIP1).
template <int WW, int MAXA, int SRC, int TILE, bool CEN>
__device__ __forceinline__ void bconv_tile_f64(u64 (&x)[16], const u64* src, const int (&eb)[16 >> WW],
                                               int lowbits, int cnt, const bool (&sf64)[MAXA],
                                               const BconvC (&C)[MAXA], const PrimeConst& P,
                                               const unsigned char* nn, double pm, double pm1, double cs) {
  constexpr int HB = 1 << (WW - 1);
  double S[16], L[16];
  bool lset = CEN;  // L holds a term already (compile-time in the fixed source modes)
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    S[r] = cs;
    L[r] = 0.0;
    if (CEN) {  // - nneg [P]_q (exact: nneg <= K, [P]_q < 2^47)
      const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);
      L[r] = -(double)nn[e] * ((r & HB) ? pm1 : pm);
    }
  }
  // no `i < cnt` test: sources i >= cnt are zero tiles with zero constants
  // (a per-source branch makes the compiler serialise the words)
#pragma unroll
  for (int i = 0; i < MAXA; ++i) {
    const u64* si = src + i * TILE;
    if (src_is_f64<SRC, MAXA>(sf64, i)) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);
        const double xv = __longlong_as_double((long long)si[e]);
        const double w = (r & HB) ? C[i].w1 : C[i].w;
        const double sn = __fma_rn(xv, w, S[r]);
        const double l = __fma_rn(xv, w, -__dsub_rn(sn, S[r]));
        L[r] = lset ? __dadd_rn(L[r], l) : l;
        S[r] = sn;
      }
      lset = true;
    } else if (kWideInt && i % 3 == 0) {  // one wide source in three: the pipes balance
      // 60-bit source on the integer pipe (idle in this FP64-bound kernel):
      // Shoup product [x w]_p in [0, 2p), exact in a double (p < 2^47)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);
        const u64 y = (r & HB) ? shoup_lazy(si[e], C[i].sw1, C[i].swp1, P.q) : shoup_lazy(si[e], C[i].sw, C[i].swp, P.q);
        const double yd = __longlong_as_double((long long)u64_to_f64bits(y));
        L[r] = lset ? __dadd_rn(L[r], yd) : yd;
      }
      lset = true;
    } else {  // 60-bit source: x = xh 2^30 + xl
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);
        const u64 v = si[e];
        const double xh = __dsub_rn(__longlong_as_double((long long)((v >> 30) | 0x4330000000000000ull)), kTwo52);
        const double xl =
            __dsub_rn(__longlong_as_double((long long)((v & 0x3FFFFFFFull) | 0x4330000000000000ull)), kTwo52);
        const double wa = (r & HB) ? C[i].w301 : C[i].w30, wb = (r & HB) ? C[i].w1 : C[i].w;
        const double s1 = __fma_rn(xh, wa, S[r]);
        const double l1 = __fma_rn(xh, wa, -__dsub_rn(s1, S[r]));
        const double s2 = __fma_rn(xl, wb, s1);
        const double l2 = __fma_rn(xl, wb, -__dsub_rn(s2, s1));
        L[r] = lset ? __dadd_rn(L[r], __dadd_rn(l1, l2)) : __dadd_rn(l1, l2);
        S[r] = s2;
      }
      lset = true;
    }
  }
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double H = __dsub_rn(S[r], cs);
    const double qf = __dsub_rn(__fma_rn(H, P.qinv_d, kRound), kRound);
    const double rr = __fma_rn(-qf, P.qd, H);
    x[r] = (u64)__double_as_longlong(__dadd_rn(rr, L[r]));
  }
}

// one target limb of the tile: conversion into registers, forward COL stages,
// store (FP64 or integer butterflies by the target's prime class)
template <int S, int OB, bool F64, int MAXA, int SRC, bool CEN = false>
__device__ __forceinline__ void modup_target(const u64* src, u64* sm, int cnt, const bool (&sf64)[MAXA],
                                             const BconvC (&C)[MAXA], const PrimeConst& P, u64* base,
                                             int tile, int logn, double cs, const unsigned char* nn = nullptr,
                                             double pm = 0.0, double pm1 = 0.0) {
  constexpr int TILE = 1 << (S + OB);
  constexpr int NG = Sched<S>::G + (Sched<S>::R ? 1 : 0);
  const int t = threadIdx.x;
  const ulonglong2* tw = P.tw_fwd;
  const double* twf = P.twf_fwd;
  u64 x[16];
  // forward COL schedule: full groups from the top, the remainder at bit 0 last
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    int W, g0;
    if (gi < Sched<S>::G) {
      W = 4;
      g0 = S - 4 * (gi + 1);
    } else {
      W = Sched<S>::R;
      g0 = 0;
    }
    const bool firstg = gi == 0, lastg = gi == NG - 1;
#define HX_MGROUP(WW)                                                                        \
  {                                                                                          \
    int eb[16 >> WW], jb[16 >> WW];                                                          \
    group_index<false, S, OB, WW>(t, g0, logn, tile, eb, jb);                                \
    const int lowbits = OB + g0;                                                             \
    _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                         \
      const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                       \
      if (!(F64 && firstg)) x[r] = firstg ? bconv_word<F64, MAXA, SRC>(src + e, TILE, cnt, sf64, C, P) \
                                          : sm[swz<false>(e)];                               \
    }                                                                                        \
    if (F64 && firstg)                                                                       \
      bconv_tile_f64<WW, MAXA, SRC, TILE, CEN>(x, src, eb, lowbits, cnt, sf64, C, P, nn, pm, pm1, cs); \
    if (F64 && firstg)                                                                       \
      ntt_group_f64<true, false, S, OB, WW, true>(x, jb, g0, logn, twf, nullptr, P, false);   \
    else if (F64)                                                                            \
      ntt_group_f64<true, false, S, OB, WW>(x, jb, g0, logn, twf, nullptr, P, false);         \
    else                                                                                     \
      ntt_group<true, false, S, WW>(x, jb, g0, logn, tw, P, false);                          \
    if (lastg) {                                                                             \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                     \
        base[tile_gofs<false, S, OB>(e, tile, logn)] = x[r];                                 \
      }                                                                                      \
    } else {                                                                                 \
      __syncthreads();                                                                       \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                     \
        sm[swz<false>(e)] = x[r];                                                            \
      }                                                                                      \
      __syncthreads();                                                                       \
    }                                                                                        \
  }
    if (W == 4) HX_MGROUP(4)
    else if (W == 3) HX_MGROUP(3)
    else if (W == 2) HX_MGROUP(2)
    else if (W == 1) HX_MGROUP(1)
#undef HX_MGROUP
  }
}

// One launch per ModUp.  FP64-class targets: conversion + COL pass (the ROW
// pass follows as an ordinary launch).  Integer-class targets (the 60-bit
// q_0 / special primes, at most alpha + 1 of the ~27 limbs): conversion only,
// written in the coefficient domain for an ordinary integer NTT -- their
// 64-bit Shoup butterflies need more registers and latency hiding than this
// kernel's occupancy (3 CTAs of 128 threads per SM) gives them.
template <int S, int OB, int MAXA, bool CEN = false>
__global__ void __launch_bounds__((1 << (S + OB)) / 16, (OB >= 3 ? HX_MODUP_MINB : 6)) modup_col_kernel(ModUpColArgs A) {
  constexpr int TILE = 1 << (S + OB);
  constexpr int T = TILE / 16;
  extern __shared__ u64 dyn_smem[];
  u64* sm = dyn_smem;            // [TILE] group exchange
  u64* src = dyn_smem + TILE;    // [alpha][TILE] x_i of the tile
  const int t = threadIdx.x;
  // digit slowest: the CTAs resident at a time run one source-class mode, so
  // the instruction cache holds one loop body (mode 1 -- config 2's digit 0
  // with the 60-bit q_0 -- is a larger body than mode 0)
  const int tile = blockIdx.x, d = blockIdx.z;
  const long long b = blockIdx.y / A.tsplit;
  const int part = blockIdx.y % A.tsplit;
  const int logn = A.logn;
  const long long N = 1ll << logn;
  const int lo = d * A.alpha, cnt = min(A.alpha, A.src_n - lo);
  const int nt_all = A.tcnt[d], ni_all = A.icnt[d], tot = nt_all + ni_all;
  // this part's slice [k_lo, k_hi) of the (FP64 targets, integer targets) list
  const int k_lo = (int)((long long)tot * part / A.tsplit), k_hi = (int)((long long)tot * (part + 1) / A.tsplit);
  if (k_lo >= k_hi) return;

  // ---- sources: x_i = [a_i Qhat_i^-1]_{q_i} (canonical); FP64-class sources
  // stored as double bits, the wide ones as integers
  bool sf64[MAXA];
  const u64* cb = A.coef + b * (long long)A.src_n * N;
  unsigned char* nn = reinterpret_cast<unsigned char*>(dyn_smem + TILE * (1 + MAXA));  // [TILE] nneg (ModDown)
  int nneg[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) nneg[r] = 0;
#pragma unroll
  for (int i = 0; i < MAXA; ++i) {
    sf64[i] = false;
    if (i < cnt) {
      const PrimeConst& Q = A.pc[A.src_pbase + lo + i];
      // HX_MODUP_INT0: source 0 of every ModUp digit kept as an integer, so its
      // products run on the integer pipe (Shoup, mode 1) beside the FP64 ones
      sf64[i] = Q.f64 && !(kModUpInt0 && !CEN && i == 0);
      const SC h = A.qhinv[A.qh_off[d] + i];
      const u64* ci = cb + (long long)(lo + i) * N;
      u64 a[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) a[r] = __ldcs(ci + tile_gofs<false, S, OB>(r * T + t, tile, logn));
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        u64 x = csub(shoup_lazy(a[r], h.w, h.wp, Q.q), Q.q);
        if (CEN) nneg[r] += x > (Q.q >> 1);
        if (sf64[i]) x = u64_to_f64bits(x);
        src[i * TILE + r * T + t] = x;
      }
    } else {  // padding source of a short last digit: zeros (bconv_tile_f64)
      sf64[i] = true;
#pragma unroll
      for (int r = 0; r < 16; ++r) src[i * TILE + r * T + t] = 0ull;
    }
  }
  if (CEN) {
#pragma unroll
    for (int r = 0; r < 16; ++r) nn[r * T + t] = (unsigned char)nneg[r];
  }
  __syncthreads();
  int mode = 0;  // source-class mode of this digit (see src_is_f64)
  {
    bool all = true, none = true, first_only = cnt > 0 && !sf64[0];
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < cnt) {
        all = all && sf64[i];
        none = none && !sf64[i];
        if (i > 0) first_only = first_only && sf64[i];
      }
    mode = all ? 0 : (CEN && none) ? 3 : first_only ? 1 : 2;
  }

  const int* tl = A.tlist + A.toff[d];
  const BconvC* bcd = A.bc + A.bc_off[d];
  const double cs = A.cs_round;
  u64* dout = A.out + (b * A.dnum + d) * (long long)A.ext * N;
#pragma unroll 1
  for (int k = k_lo; k < min(k_hi, nt_all); ++k) {
    const int j = tl[k];
    const int pj = j < A.n_q ? j : A.n_chain + (j - A.n_q);
    const PrimeConst P = A.pc[pj];
    BconvC C[MAXA];
#pragma unroll
    for (int i = 0; i < MAXA; ++i) {
      if (i < cnt)
        C[i] = bcd[(long long)j * A.alpha + i];
      else
        C[i] = BconvC{0.0, 0.0, 0.0, 0.0, 0ull, 0ull, 0.0, 0.0, 0ull, 0ull};
    }
    u64* base = dout + (long long)j * N;
    __syncthreads();  // the previous target's last exchange reads are done
    if (CEN) {  // ModDown
      const double pm = A.pmf[pj], pm1 = A.pmf1[pj];
      if (mode == 0)
        modup_target<S, OB, true, MAXA, 0, true>(src, sm, cnt, sf64, C, P, base, tile, logn, cs, nn, pm, pm1);
      else if (mode == 3)
        modup_target<S, OB, true, MAXA, 3, true>(src, sm, cnt, sf64, C, P, base, tile, logn, cs, nn, pm, pm1);
      else
        modup_target<S, OB, true, MAXA, 2, true>(src, sm, cnt, sf64, C, P, base, tile, logn, cs, nn, pm, pm1);
    } else if (mode == 0) {
      modup_target<S, OB, true, MAXA, 0>(src, sm, cnt, sf64, C, P, base, tile, logn, cs);
    } else if (mode == 1) {
      modup_target<S, OB, true, MAXA, 1>(src, sm, cnt, sf64, C, P, base, tile, logn, cs);
    } else {
      modup_target<S, OB, true, MAXA, 2>(src, sm, cnt, sf64, C, P, base, tile, logn, cs);
    }
  }
#pragma unroll 1
  for (int k = max(k_lo, nt_all); k < k_hi; ++k) {
    const int j = tl[k];
    const int pj = j < A.n_q ? j : A.n_chain + (j - A.n_q);
    const PrimeConst& P = A.pc[pj];
    BconvC C[MAXA];
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < cnt) C[i] = bcd[(long long)j * A.alpha + i];
    u64* base = dout + (long long)j * N;
    u64 y[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) y[r] = 0;
#pragma unroll
    for (int i = 0; i < MAXA; ++i) {  // sources outer (uniform tests), words inner
      if (i < cnt) {
        const bool f = sf64[i];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          u64 v = src[i * TILE + r * T + t];
          if (f)  // exact double -> integer
            v = (u64)__double_as_longlong(__dadd_rn(__longlong_as_double((long long)v), kTwo52)) & 0xFFFFFFFFFFFFFull;
          y[r] = csub(y[r] + shoup_lazy(v, C[i].sw, C[i].swp, P.q), P.two_q);
        }
      }
    }
    if (CEN) {
      const u64 pm = A.pmu[pj];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        u64 v = csub(y[r], P.q);
        const int ng = nn[r * T + t];
        for (int m = 0; m < ng; ++m) v = submod(v, pm, P.q);
        base[tile_gofs<false, S, OB>(r * T + t, tile, logn)] = v;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) base[tile_gofs<false, S, OB>(r * T + t, tile, logn)] = csub(y[r], P.q);
    }
  }
}

// data tile + alpha source tiles (+ the [TILE] nneg bytes of ModDown)
inline int modup_col_smem_bytes(int S, int OB, int alpha, bool centred = false) {
  return 8 * (1 << (S + OB)) * (1 + alpha) + (centred ? (1 << (S + OB)) : 0);
}

}  // namespace hx
