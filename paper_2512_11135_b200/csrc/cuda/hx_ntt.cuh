// hx_ntt.cuh -- batched negacyclic NTT / INTT for sm_100a.
//
// Replaces NttTables::forward / inverse (reference ntt.cpp:57-96) and
// LatticeContext::to_ntt / to_coeff (rns_poly.cpp:42-54).  Output is
// bit-identical to the reference: forward leaves the bit-reversed layout
// out[k] = a(psi^(2 brv(k) + 1)) with the reference's psi (ntt.cpp:23-32),
// inverse restores natural order and applies N^-1.
//
// Structure: N = 2^logn is split as N1 x N2 (N1 = 2^a "high" bits, N2 = 2^b
// "low" bits).  Forward runs two passes:
//   COL pass  -- the first a stages: 2^a-point sub-transforms over the high
//                bits, a CTA owns 16 adjacent columns (128-B coalesced rows);
//   ROW pass  -- the last b stages on contiguous 2^b-element rows, a CTA
//                owns 16 rows.
// The inverse runs ROW then COL (Gentleman-Sande order).  Inside a pass each
// thread holds 16 words in registers and performs radix-16 groups of 4 stages
// (Harvey lazy butterflies, values in [0,4q) / [0,2q)); groups exchange data
// through a 32 KB XOR-swizzled shared-memory tile.  Twiddles are the
// reference tables (psi^brv(i), Shoup companion) packed as ulonglong2 and read
// through the read-only path; the twiddle index of a butterfly whose lower
// element has global index j and whose pair bit is beta is (N + j) >> (beta+1)
// for both directions.
#pragma once

#include "hx_common.cuh"
#include "hx_types.cuh"

namespace hx {

// One entry per limb a launch transforms.  Instance i of a batched launch is
// (element b = i / count, entry e = i % count) at
//   data + (b * stride + off[e]) * N,  prime index prime[e].
constexpr int kMaxLimbEntries = 256;
struct LimbTable {
  int count;
  int stride;  // limbs per batch element
  unsigned short off[kMaxLimbEntries];
  unsigned char prime[kMaxLimbEntries];
};

struct NttArgs {
  u64* data;
  const PrimeConst* pc;
  LimbTable lt;
  int logn;
  long long instances;  // batch * lt.count
  long long batch;      // batch elements
  int bper;             // batch elements per CTA (the grid is pairs x chunks)
  // out-of-place first pass: read instance (b, e) from src + b src_estride +
  // off[e] N instead of `data` (null: in place)
  const u64* src = nullptr;
  long long src_estride = 0;
};

// Deposit free index f around the w group bits starting at bit lowbits.
__device__ __forceinline__ int deposit(int f, int lowbits, int w) {
  return (f & ((1 << lowbits) - 1)) | ((f >> lowbits) << (lowbits + w));
}

// Shared-memory tile swizzles (u64 words: bank pair = e mod 16).  ROW tiles:
// XOR the low 4 bits with the row index.  COL tiles of 8 columns: the last
// group's lanes read 8 consecutive words then jump 128 words, so word bit 3 is
// flipped by bit 7 -- lanes 0-15 then cover all 16 bank pairs (2 wavefronts per
// 8-byte warp access, the minimum).
template <bool ROW>
__device__ __forceinline__ int swz(int e) {
  return ROW ? (e ^ ((e >> 4) & 15)) : (e ^ (((e >> 7) & 1) << 3));
}

#ifndef HX_SHOUP_APPROX
#define HX_SHOUP_APPROX 0
#endif
constexpr bool kShoupApprox = HX_SHOUP_APPROX != 0;
__device__ __forceinline__ u64 shoup_ntt(u64 a, u64 w, u64 wp, u64 q) {
  return kShoupApprox ? shoup_lazy4(a, w, wp, q) : shoup_lazy(a, w, wp, q);
}
// [0, 8q) -> [0, q)
__device__ __forceinline__ u64 reduce8(u64 a, u64 q) { return csub(csub(csub(a, q << 2), q << 1), q); }

// One radix-2^W group over sub-bits [g0, g0+W) of the tile index.
// x[r], r = (r_out << W) | r_in ; element e_r = base[r_out] | (r_in << lowbits).
template <bool FWD, bool ROW, int S, int W>
__device__ __forceinline__ void ntt_group(u64 (&x)[16], const int (&jb)[16 >> W], int g0,
                                          int logn, const ulonglong2* __restrict__ tw,
                                          const PrimeConst& P, bool last_stage_inv) {
  constexpr int NO = 16 >> W;
  const int logb = ROW ? 0 : (logn - S);  // j-bit of sub-bit 0
  // lazy bound: products in [0, 2q) (exact Shoup) or [0, 4q) (shoup_lazy4);
  // forward values stay below 2 q2, inverse values below q2
  const u64 q = P.q, q2 = kShoupApprox ? (P.q << 2) : P.two_q;
  const u64 N = 1ull << logn;
#pragma unroll
  for (int ii = 0; ii < W; ++ii) {
    const int i = FWD ? (W - 1 - ii) : ii;  // register bit processed
    const int beta = logb + g0 + i;         // global j-bit of the pair
#pragma unroll
    for (int ro = 0; ro < NO; ++ro) {
#pragma unroll
      for (int hp = 0; hp < (1 << (W - 1 - i)); ++hp) {
        const int rb = (ro << W) | (hp << (i + 1));
        // global index of element rb: jb[ro] + (hp << (i+1)) << (logb + g0)
        const u64 j = (u64)jb[ro] + ((u64)(hp << (i + 1)) << (logb + g0));
        const bool fin = (!FWD) && last_stage_inv && (beta == logn - 1);
        ulonglong2 wt = make_ulonglong2(0, 0);
        if (!fin) wt = __ldg(tw + ((N + j) >> (beta + 1)));
#pragma unroll
        for (int lp = 0; lp < (1 << i); ++lp) {
          const int r0 = rb | lp, r1 = r0 | (1 << i);
          const u64 X = x[r0], Y = x[r1];
          if (FWD) {
            const u64 Xr = csub(X, q2);
            const u64 T = shoup_ntt(Y, wt.x, wt.y, q);
            x[r0] = Xr + T;
            x[r1] = Xr - T + q2;
          } else if (fin) {
            x[r0] = shoup_ntt(X + Y, P.ninv, P.ninvp, q);
            x[r1] = shoup_ntt(X - Y + q2, P.w1n, P.w1np, q);
          } else {
            x[r0] = csub(X + Y, q2);
            x[r1] = shoup_ntt(X - Y + q2, wt.x, wt.y, q);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- FP64 path
// For primes q < 2^47 the butterflies run on the FP64 pipe (B200: DFMA at 64
// lanes/clk/SM, twice the IMAD.WIDE rate, and a separate pipe from the
// integer multiplier).  Values are integers held exactly in doubles, lazily in
// a signed range; the modular product is exact:
//   h = fl(y w), l = y w - h (one FMA, exact), qf = rint(y (w/q)) (one FMA
//   against the 1.5*2^52 rounding constant), r = h - qf q (one FMA, exact),
//   y w mod q == r + l  with |r + l| < q.
// Forward (CT) values grow by < q per stage (< 17 q after 16 stages); inverse
// (GS) values are re-centred (|v| <= q/2) at the start of every register
// group.  The last pass normalises to [0, q) and converts back to u64, so the
// output is bit-identical to the integer path and to the reference.
constexpr double kRound = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double mulmod_f64(double y, double w, double wq, double q) {
  const double h = __dmul_rn(y, w);
  const double l = __fma_rn(y, w, -h);
  const double qf = __dsub_rn(__fma_rn(y, wq, kRound), kRound);
  const double r = __fma_rn(-qf, q, h);
  return __dadd_rn(r, l);
}

// Same product without a per-twiddle w / q: the quotient is taken from the
// rounded product, qf = rint(h / q) (|h / q - qf| <= 1/2 + 2^-7 for
// y w < 2^99), so r = h - qf q is exact in one FMA and |r + l| < q as before.
__device__ __forceinline__ double mulmod_f64h(double y, double w, double qinv, double q) {
  const double h = __dmul_rn(y, w);
  const double l = __fma_rn(y, w, -h);
  const double qf = __dsub_rn(__fma_rn(h, qinv, kRound), kRound);
  const double r = __fma_rn(-qf, q, h);
  return __dadd_rn(r, l);
}

// centre v into [-q/2 - eps, q/2 + eps]
__device__ __forceinline__ double centre_f64(double v, double q, double qinv) {
  const double qf = __dsub_rn(__fma_rn(v, qinv, kRound), kRound);
  return __fma_rn(-qf, q, v);
}

__device__ __forceinline__ u64 u64_to_f64bits(u64 x) {  // x < 2^52 -> bits of (double)x
  return (u64)__double_as_longlong(__dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), kTwo52));
}

__device__ __forceinline__ u64 f64bits_to_residue(u64 bits, double q, double qinv) {  // -> [0, q)
  double r = centre_f64(__longlong_as_double((long long)bits), q, qinv);
  r = r < 0.0 ? __dadd_rn(r, q) : r;
  return (u64)__double_as_longlong(__dadd_rn(r, kTwo52)) & 0xFFFFFFFFFFFFFull;
}

// ROW-pass twiddles of a tile staged in shared memory: for pair bit beta < S
// the tile's twiddle indices are contiguous, (N >> (beta+1)) + row0 2^(S-beta-1)
// + [0, OTH 2^(S-beta-1)); they are stored back to back, stage beta at offset
// OTH (2^S - 2^(S-beta)).  This turns the per-butterfly distinct twiddle
// loads of the last stages into one coalesced bulk load per tile.
// Each segment is padded with one double per 16 (index k stored at
// k + k / 16): the last register group reads twiddles at a lane stride of
// 2^(3 - beta) doubles, which without padding is a 16-way bank conflict.
template <int S, int OB>
__device__ __forceinline__ int row_tw_offset(int beta) {
  return 17 * ((1 << OB) * ((1 << S) - (1 << (S - beta)))) / 16;
}
__device__ __forceinline__ int row_tw_pad(int k) { return k + (k >> 4); }

// SKIP1 (forward only): the group's first stage (pair bit W-1) multiplies
// nothing -- its lower inputs arrive premultiplied by the stage's twiddle
// (the fused ModUp / ModDown conversion, hx_modup.cuh)
template <bool FWD, bool ROW, int S, int OB, int W, bool SKIP1 = false>
__device__ __forceinline__ void ntt_group_f64(u64 (&x)[16], const int (&jb)[16 >> W], int g0, int logn,
                                              const double* __restrict__ tw, const double* sm_tw,
                                              const PrimeConst& P, bool last_stage_inv) {
  constexpr int NO = 16 >> W;
  const int logb = ROW ? 0 : (logn - S);
  const double q = P.qd;
  const u64 N = 1ull << logn;
  // every twiddle of the group is fetched up front (all loads in flight
  // together, 32-bit indices) instead of one dependent load per stage
  double wts[W][8];
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const int beta = logb + g0 + i;
#pragma unroll
    for (int ro = 0; ro < NO; ++ro) {
#pragma unroll
      for (int hp = 0; hp < (1 << (W - 1 - i)); ++hp) {
        const unsigned j = (unsigned)jb[ro] + ((unsigned)(hp << (i + 1)) << (logb + g0));
        const bool fin = (!FWD) && last_stage_inv && (beta == logn - 1);
        double wt = 0.0;
        if (!fin && !(SKIP1 && i == W - 1)) {
          if (ROW)
            wt = sm_tw[row_tw_offset<S, OB>(beta) + row_tw_pad((int)((j & ((1u << (S + OB)) - 1)) >> (beta + 1)))];
          else
            wt = __ldg(tw + (((unsigned)N + j) >> (beta + 1)));
        }
        wts[i][ro * (1 << (W - 1 - i)) + hp] = wt;
      }
    }
  }
  double v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    v[r] = __longlong_as_double((long long)x[r]);
    if (!FWD) v[r] = centre_f64(v[r], q, P.qinv_d);
  }
#pragma unroll
  for (int ii = 0; ii < W; ++ii) {
    const int i = FWD ? (W - 1 - ii) : ii;
    const int beta = logb + g0 + i;
#pragma unroll
    for (int ro = 0; ro < NO; ++ro) {
#pragma unroll
      for (int hp = 0; hp < (1 << (W - 1 - i)); ++hp) {
        const int rb = (ro << W) | (hp << (i + 1));
        const bool fin = (!FWD) && last_stage_inv && (beta == logn - 1);
        const double wt = wts[i][ro * (1 << (W - 1 - i)) + hp];
#pragma unroll
        for (int lp = 0; lp < (1 << i); ++lp) {
          const int r0 = rb | lp, r1 = r0 | (1 << i);
          const double X = v[r0], Y = v[r1];
          if (FWD && SKIP1 && i == W - 1) {
            v[r0] = __dadd_rn(X, Y);
            v[r1] = __dsub_rn(X, Y);
          } else if (FWD) {
            const double T = mulmod_f64h(Y, wt, P.qinv_d, q);
            v[r0] = __dadd_rn(X, T);
            v[r1] = __dsub_rn(X, T);
          } else if (fin) {
            v[r0] = mulmod_f64(__dadd_rn(X, Y), P.ninv_d, P.ninv_q, q);
            v[r1] = mulmod_f64(__dsub_rn(X, Y), P.w1n_d, P.w1n_q, q);
          } else {
            v[r0] = __dadd_rn(X, Y);
            v[r1] = mulmod_f64h(__dsub_rn(X, Y), wt, P.qinv_d, q);
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = (u64)__double_as_longlong(v[r]);
}

// Compute, for a group at sub-bits [g0, g0+W), the tile element base index
// (r_in = 0) and the global j base for each r_out.
template <bool ROW, int S, int OB, int W>
__device__ __forceinline__ void group_index(int t, int g0, int logn, int tile,
                                           int (&eb)[16 >> W], int (&jb)[16 >> W]) {
  constexpr int T = (1 << (S + OB)) / 16;
  const int subbase = ROW ? 0 : OB;
  const int lowbits = subbase + g0;
#pragma unroll
  for (int ro = 0; ro < (16 >> W); ++ro) {
    const int f = ro * T + t;
    const int e = deposit(f, lowbits, W);
    eb[ro] = e;
    if (ROW) {
      jb[ro] = (tile << (S + OB)) + e;
    } else {
      const int logb = logn - S;
      jb[ro] = ((e >> OB) << logb) + (tile << OB) + (e & ((1 << OB) - 1));
    }
  }
}

template <bool ROW, int S, int OB>
__device__ __forceinline__ long long tile_gofs(int e, int tile, int logn) {
  if (ROW) return ((long long)tile << (S + OB)) + e;
  const int logb = logn - S;
  return ((long long)(e >> OB) << logb) + (tile << OB) + (e & ((1 << OB) - 1));
}

// Group schedule: forward processes sub-bits from the top (groups of 4, the
// remainder last); inverse from the bottom (remainder first).
template <int S>
struct Sched {
  static constexpr int R = S % 4;          // remainder width
  static constexpr int G = S / 4;          // number of full groups
};

// Key-switch combine fused into the last (ROW) pass of ModDown's forward NTT:
// for poly b, limb i of the converted ModDown term v (this transform's
// output), out = (u - v) [P^-1]_{q_i} (+ add), written at tau^-1 of the
// coefficient index when a rotation's automorphism is fused (perm).  tau maps
// aligned 2^j blocks of NTT indices onto aligned 2^j blocks, so a warp's 32
// consecutive source words land in one aligned 32-word block: the permuted
// store stays coalesced.  Same semantics as combine_kernel (hx_kernels.cuh).
struct EpiArgs {
  const u64* u;
  const u64* add;  // may be null
  u64* out;
  const SC* pinv;  // [n_chain]
  long long u_stride, out_stride, add_stride, add_every, add_period;
  u32 add_g;
  int n_q;
  int perm, per;
  long long out_rstride, out_estride;
  u32 pginv[64];  // g^-1 mod 2N per rotation r (perm)
};

#ifndef HX_COMBINE_UNROLL
#define HX_COMBINE_UNROLL 8
#endif
constexpr int kCombineUnroll = HX_COMBINE_UNROLL;  // epilogue words in flight per thread (A/B)

// combine epilogue of the forward ROW pass (see EpiArgs): the tile's
// transformed words sit in smem (ROW swizzle, residues in [0, q)); thread t
// handles tile words e = r T + t, i.e. coalesced runs of T.
template <int S, int OB, bool F64>
__device__ __forceinline__ void row_combine_epilogue(const u64* sm, int t, int tile, long long b, int i, int logn,
                                                     const PrimeConst& P, const EpiArgs& E) {
  constexpr int TILE = 1 << (S + OB);
  constexpr int T = TILE / 16;
  const long long N = 1ll << logn;
  long long ba = b / E.add_every;
  if (E.add_period) ba %= E.add_period;
  const bool do_add = E.add && (b % E.add_every) == 0;
  u32 ginv = 1;
  long long ob = b * E.out_stride;
  if (E.perm) {
    const long long qq = b >> 1;
    const long long rr = qq / E.per, e = qq % E.per;
    ginv = E.pginv[rr];
    ob = rr * E.out_rstride + e * E.out_estride + (b & 1) * (long long)E.n_q * N;
  }
  const SC c = E.pinv[i];
  const u64* ub = E.u + b * E.u_stride + (long long)i * N;
  const u64* abase = do_add ? E.add + ba * E.add_stride + (long long)i * N : nullptr;
  u64* outb = E.out + ob + (long long)i * N;
  const double wd = __longlong_as_double((long long)u64_to_f64bits(c.w));
  // words in flight: KB at a time, all their loads issued before any store
  // (the stores may alias the loads as far as the compiler knows, so a plain
  // unrolled loop keeps one load pair in flight per store)
  constexpr int KB = kCombineUnroll;
#pragma unroll 1
  for (int r0 = 0; r0 < 16; r0 += KB) {
  u64 uus[KB], ads[KB];
#pragma unroll
  for (int rr = 0; rr < KB; ++rr) {
    const int sidx = (tile << (S + OB)) + (r0 + rr) * T + t;
    const int aidx = E.perm ? sidx : (E.add_g == 1 ? sidx : (int)ntt_auto_index((u32)sidx, E.add_g, logn));
    uus[rr] = __ldcs(ub + sidx);
    ads[rr] = do_add ? __ldg(abase + aidx) : 0ull;
  }
#pragma unroll
  for (int rr = 0; rr < KB; ++rr) {
    const int r = r0 + rr;
    const int e = r * T + t;
    const int sidx = (tile << (S + OB)) + e;  // coefficient (NTT) index of the word
    const u64 v = sm[swz<true>(e)];
    // output index: tau^-1 (perm); the add operand is gathered at tau_{add_g}
    // when no permutation is fused (combine_kernel's asrc)
    const int oidx = ginv != 1 ? (int)ntt_auto_index((u32)sidx, ginv, logn) : sidx;
    const u64 uu = uus[rr];
    const u64 ad = ads[rr];
    u64 res;
    if (F64) {
      const double du = __longlong_as_double((long long)u64_to_f64bits(uu));
      const double dv = __longlong_as_double((long long)u64_to_f64bits(v));
      double w = mulmod_f64h(__dsub_rn(du, dv), wd, P.qinv_d, P.qd);
      w = __dadd_rn(w, __longlong_as_double((long long)u64_to_f64bits(ad)));
      res = f64bits_to_residue((u64)__double_as_longlong(w), P.qd, P.qinv_d);
    } else {
      res = csub(shoup_lazy(uu + P.q - v, c.w, c.wp, P.q), P.q);
      if (do_add) res = csub(res + ad, P.q);
    }
    __stcs(outb + oidx, res);
  }
  }
}

// dynamic shared memory of a pass kernel (bytes)
template <bool ROW, int S, int OB, bool F64>
constexpr int ntt_smem_bytes() {
  return 8 * ((1 << (S + OB)) + ((ROW && F64) ? 17 * (1 << OB) * ((1 << S) - 1) / 16 + 16 : 0));
}

template <bool FWD, bool ROW, int S, int OB, bool F64, bool EPI>
__device__ __forceinline__ void ntt_pass_body(const NttArgs& a, const EpiArgs* ep);

template <bool FWD, bool ROW, int S, int OB, bool F64>
__global__ void __launch_bounds__((1 << (S + OB)) / 16)
    ntt_pass_kernel(NttArgs a) {
  ntt_pass_body<FWD, ROW, S, OB, F64, false>(a, nullptr);
}

// forward ROW pass + combine epilogue (ModDown)
template <int S, int OB, bool F64>
__global__ void __launch_bounds__((1 << (S + OB)) / 16)
    ntt_row_combine_kernel(NttArgs a, EpiArgs ep) {
  ntt_pass_body<true, true, S, OB, F64, true>(a, &ep);
}

template <bool FWD, bool ROW, int S, int OB, bool F64, bool EPI>
__device__ __forceinline__ void ntt_pass_body(const NttArgs& a, const EpiArgs* ep) {
  constexpr int TILE = 1 << (S + OB);
  constexpr int T = TILE / 16;
  extern __shared__ u64 dyn_smem[];  // [TILE] data tile, then [kTw] staged twiddles
  u64* sm = dyn_smem;
  const int t = threadIdx.x;
  const int tiles = (1 << a.logn) / TILE;
  const long long inst = blockIdx.x / tiles;
  const int tile = blockIdx.x % tiles;
  const int per = a.lt.count;
  const long long bidx = inst / per;
  const int ent = (int)(inst % per);
  u64* base = a.data + ((long long)bidx * a.lt.stride + a.lt.off[ent]) * (1ll << a.logn);
  const u64* lbase = a.src ? a.src + (long long)bidx * a.src_estride + (long long)a.lt.off[ent] * (1ll << a.logn)
                           : base;  // first group's loads
  const PrimeConst P = a.pc[a.lt.prime[ent]];
  const ulonglong2* tw = FWD ? P.tw_fwd : P.tw_inv;
  const double* twf = FWD ? P.twf_fwd : P.twf_inv;
  const u64 q = P.q;
  // first pass of the transform reads residues, last pass writes residues
  constexpr bool kFirstPass = FWD ? !ROW : ROW;
  constexpr bool kLastPass = !kFirstPass;
  // FP64 ROW pass: stage the tile's twiddles (all S stages) in shared memory
  double* sm_tw = reinterpret_cast<double*>(dyn_smem + TILE);
  if (ROW && F64) {
    // all S stages' twiddles of the tile (255 x 2^OB doubles) with 8-byte
    // cp.async (LDGSTS): every thread has all its copies in flight at once and
    // they overlap the first group's data loads; waited for before group 0.
    constexpr int kTw = (1 << OB) * ((1 << S) - 1);
    const long long row0 = (long long)tile << OB;
#pragma unroll
    for (int i = 0; i < (kTw + T - 1) / T; ++i) {
      const int m = t + i * T;  // flat index, stage beta owns [2^(S+OB) - 2^(S+OB-beta), 2^(S+OB) - 2^(S+OB-beta-1))
      if (m < kTw) {
        const int beta = (S + OB - 1) - (31 - __clz((TILE - 1) - m));
        const int seg = TILE - (TILE >> beta);
        const int k = m - seg;
        const double* src = twf + ((1ll << a.logn) >> (beta + 1)) + (row0 << (S - beta - 1)) + k;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(sm_tw + 17 * seg / 16 + row_tw_pad(k));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }

  if (EPI) {  // warm L2 with the epilogue's u (and add) tile lines while the transform runs
    const long long N = 1ll << a.logn;
    const int li = a.lt.off[ent];
    const u64* ut = ep->u + bidx * ep->u_stride + (long long)li * N + ((long long)tile << (S + OB));
    for (int l = t; l < TILE / 16; l += T) asm volatile("prefetch.global.L2 [%0];" ::"l"(ut + l * 16));
    if (ep->add && (bidx % ep->add_every) == 0 && (ep->perm || ep->add_g == 1)) {
      long long ba = bidx / ep->add_every;
      if (ep->add_period) ba %= ep->add_period;
      const u64* at = ep->add + ba * ep->add_stride + (long long)li * N + ((long long)tile << (S + OB));
      for (int l = t; l < TILE / 16; l += T) asm volatile("prefetch.global.L2 [%0];" ::"l"(at + l * 16));
    }
  }
  u64 x[16];
  constexpr int NG = Sched<S>::G + (Sched<S>::R ? 1 : 0);
  // group g (in processing order) -> (g0, W)
  // forward: full groups from the top, remainder (at bit 0) last
  // inverse: remainder (at bit 0) first, then full groups upwards
  bool first = true;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    constexpr int Rm = Sched<S>::R;
    int W, g0;
    if (FWD) {
      if (gi < Sched<S>::G) {
        W = 4;
        g0 = S - 4 * (gi + 1);
      } else {
        W = Rm;
        g0 = 0;
      }
    } else {
      if (Rm && gi == 0) {
        W = Rm;
        g0 = 0;
      } else {
        W = 4;
        g0 = Rm + 4 * (gi - (Rm ? 1 : 0));
      }
    }
    const bool lastg = (gi == NG - 1);
    // W is a compile-time constant after unrolling; dispatch explicitly.
#define HX_GROUP(WW)                                                                           \
  {                                                                                            \
    int eb[16 >> WW], jb[16 >> WW];                                                            \
    group_index<ROW, S, OB, WW>(t, g0, a.logn, tile, eb, jb);                                  \
    const int lowbits = (ROW ? 0 : OB) + g0;                                                   \
    if (first) {                                                                               \
      if (FWD || !ROW) {                                                                       \
        /* direct coalesced global load */                                                     \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
          const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                     \
          x[r] = lbase[tile_gofs<ROW, S, OB>(e, tile, a.logn)];                                \
        }                                                                                      \
      } else {                                                                                 \
        /* inverse ROW pass: stage through smem for coalescing */                              \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
          const int e = r * T + t;                                                             \
          sm[swz<ROW>(e)] = lbase[tile_gofs<ROW, S, OB>(e, tile, a.logn)];                     \
        }                                                                                      \
        __syncthreads();                                                                       \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
          const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                     \
          x[r] = sm[swz<ROW>(e)];                                                              \
        }                                                                                      \
      }                                                                                        \
    } else {                                                                                   \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                         \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                       \
        x[r] = sm[swz<ROW>(e)];                                                                \
      }                                                                                        \
    }                                                                                          \
    if (ROW && F64 && first) {                                                                 \
      asm volatile("cp.async.wait_all;\n" ::: "memory");                                     \
      __syncthreads();                                                                         \
    }                                                                                          \
    if (F64 && kFirstPass && first) {                                                          \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) x[r] = u64_to_f64bits(x[r]);              \
    }                                                                                          \
    if (F64)                                                                                   \
      ntt_group_f64<FWD, ROW, S, OB, WW>(x, jb, g0, a.logn, twf, sm_tw, P, !ROW);              \
    else                                                                                       \
      ntt_group<FWD, ROW, S, WW>(x, jb, g0, a.logn, tw, P, !ROW);                              \
    if (lastg) {                                                                               \
      if (F64) {                                                                               \
        if (kLastPass) {                                                                       \
          _Pragma("unroll") for (int r = 0; r < 16; ++r) x[r] =                                \
              f64bits_to_residue(x[r], P.qd, P.qinv_d);                                        \
        }                                                                                      \
      } else {                                                                                 \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) x[r] =                                  \
            (FWD ? (ROW ? (kShoupApprox ? reduce8(x[r], q) : reduce4(x[r], q, P.two_q)) : x[r])   \
                 : (ROW ? x[r] : (kShoupApprox ? reduce4(x[r], q, P.two_q) : csub(x[r], q))));       \
      }                                                                                        \
      if (FWD && ROW) {                                                                        \
        /* stage through smem for a coalesced store */                                         \
        __syncthreads();                                                                       \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
          const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                     \
          sm[swz<ROW>(e)] = x[r];                                                              \
        }                                                                                      \
        __syncthreads();                                                                       \
        if (EPI)                                                                               \
          row_combine_epilogue<S, OB, F64>(sm, t, tile, bidx, a.lt.off[ent], a.logn, P, *ep);  \
        else                                                                                   \
          _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                     \
            const int e = r * T + t;                                                           \
            base[tile_gofs<ROW, S, OB>(e, tile, a.logn)] = sm[swz<ROW>(e)];                    \
          }                                                                                    \
      } else {                                                                                 \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                       \
          const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                     \
          base[tile_gofs<ROW, S, OB>(e, tile, a.logn)] = x[r];                                 \
        }                                                                                      \
      }                                                                                        \
    } else {                                                                                   \
      __syncthreads();                                                                         \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                         \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                       \
        sm[swz<ROW>(e)] = x[r];                                                                \
      }                                                                                        \
      __syncthreads();                                                                         \
    }                                                                                          \
  }
    if (W == 4) HX_GROUP(4)
    else if (W == 3) HX_GROUP(3)
    else if (W == 2) HX_GROUP(2)
    else if (W == 1) HX_GROUP(1)
#undef HX_GROUP
    first = false;
  }
}

}  // namespace hx
