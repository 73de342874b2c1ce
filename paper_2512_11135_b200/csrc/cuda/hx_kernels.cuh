// hx_kernels.cuh -- device kernels other than the NTT (declared for the
// launchers in hx_ops.cu).  Every kernel names the reference routine it
// replaces.  Layout: u64 [batch][limbs][N], limb k of an (n_q, n_p) poly is
// chain prime k for k < n_q, special prime k - n_q otherwise.
#pragma once

#include "hx_common.cuh"
#include "hx_ntt.cuh"
#include "hx_types.cuh"

namespace hx {

// counter-based uniform residue: word i of stream `seed`, floor(r q / 2^128)
// over 128 hashed bits r (bias < 2^-64).  hx_sample_uniform writes these;
// compressed keys (hx_keygen_*_c) regenerate their uniform half from them.
__device__ __forceinline__ u64 splitmix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ u64 uniform_word(u64 seed, u64 i, u64 q) {
  const u64 r0 = splitmix64(seed ^ splitmix64(2 * i));
  const u64 r1 = splitmix64(seed ^ splitmix64(2 * i + 1));
  const u64 t = mulhi64(r1, q);                // floor(r1 q / 2^64)
  const u64 lo = r0 * q, hi = mulhi64(r0, q);  // r0 q
  return hi + ((lo + t) < lo ? 1 : 0);         // floor((r0 2^64 + r1) q / 2^128)
}

// ------------------------------------------------------------ elementwise
enum class EwOp : int { Add = 0, Sub, Neg, Mul, MulAcc, Copy };

struct EwArgs {
  u64* out;
  const u64* a;
  const u64* b;
  const PrimeConst* pc;
  LimbTable lt;   // limbs of one batch element
  int logn;
  long long instances;
  // broadcast operands: element b reads a element (a_mod ? b % a_mod : b) and
  // b element b / b_div (a mask applied to every ciphertext poly of a batch)
  long long a_mod = 0, b_div = 1;
};

// add / sub / negate / mul / mul_acc (rns_poly.cpp:62-110), 2 words per thread
template <EwOp OP>
__global__ void ew_kernel(EwArgs A) {
  const int per_limb = (1 << A.logn) / (2 * blockDim.x);
  const long long inst = blockIdx.x / per_limb;
  const int chunk = blockIdx.x % per_limb;
  const long long b = inst / A.lt.count;
  const int e = (int)(inst % A.lt.count);
  const PrimeConst& P = A.pc[A.lt.prime[e]];
  const u64 q = P.q;
  const long long in_limb = (long long)A.lt.off[e] * (1ll << A.logn) + 2ll * (chunk * blockDim.x + threadIdx.x);
  const long long ofs = b * A.lt.stride * (1ll << A.logn) + in_limb;
  const long long ba = A.a_mod ? b % A.a_mod : b, bb = b / A.b_div;
  const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(A.a + ba * A.lt.stride * (1ll << A.logn) + in_limb);
  ulonglong2 y = make_ulonglong2(0, 0), r;
  if (OP != EwOp::Neg && OP != EwOp::Copy)
    y = *reinterpret_cast<const ulonglong2*>(A.b + bb * A.lt.stride * (1ll << A.logn) + in_limb);
  if (OP == EwOp::Add) {
    r.x = addmod(x.x, y.x, q);
    r.y = addmod(x.y, y.y, q);
  } else if (OP == EwOp::Sub) {
    r.x = submod(x.x, y.x, q);
    r.y = submod(x.y, y.y, q);
  } else if (OP == EwOp::Neg) {
    r.x = x.x ? q - x.x : 0;
    r.y = x.y ? q - x.y : 0;
  } else if (OP == EwOp::Mul) {
    r.x = mulmod(x.x, y.x, P);
    r.y = mulmod(x.y, y.y, P);
  } else if (OP == EwOp::MulAcc) {
    const ulonglong2 acc = *reinterpret_cast<const ulonglong2*>(A.out + ofs);
    U128 z0{acc.x, 0}, z1{acc.y, 0};
    mac128(z0, x.x, y.x);
    mac128(z1, x.y, y.y);
    r.x = reduce128(z0, P);
    r.y = reduce128(z1, P);
  } else {
    r = x;
  }
  *reinterpret_cast<ulonglong2*>(A.out + ofs) = r;
}

// NTT-domain automorphism (rns_poly.cpp:124-142 restated as a permutation of
// the bit-reversed evaluation vector): out[k] = in[perm_g(k)]
__global__ void automorphism_kernel(EwArgs A, u32 g) {
  const int per_limb = (1 << A.logn) / blockDim.x;
  const long long inst = blockIdx.x / per_limb;
  const int k = (blockIdx.x % per_limb) * blockDim.x + threadIdx.x;
  const long long b = inst / A.lt.count;
  const int e = (int)(inst % A.lt.count);
  const long long base = (b * A.lt.stride + A.lt.off[e]) * (1ll << A.logn);
  A.out[base + k] = __ldg(A.a + base + ntt_auto_index((u32)k, g, A.logn));
}

// out[b][l][t] = in[b][l][perm_g(t)] with independent batch strides (words):
// the output-side automorphism of the rotation pipeline and the key-layout
// conversion (tau_{g^-1}) of rotation keys.
__global__ void permute_kernel(u64* out, long long out_stride, const u64* in, long long in_stride,
                               u32 g, int logn) {
  const long long N = 1ll << logn;
  const long long b = blockIdx.z;
  const int l = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int src = g == 1 ? t : (int)ntt_auto_index((u32)t, g, logn);
  out[b * out_stride + l * N + t] = __ldg(in + b * in_stride + l * N + src);
}

// Several permutations in one launch: group r (blockIdx.z / per) applies
// galois element g[r] to `per` elements (blockIdx.z % per); element (r, e) is
// read at in + (r per + e) in_stride and written at out + r out_rstride +
// e out_estride.
struct PermuteMulti {
  u32 g[64];
  long long in_stride, out_rstride, out_estride;
  int per, logn;
};
__global__ void permute_multi_kernel(u64* out, const u64* in, PermuteMulti P) {
  const long long N = 1ll << P.logn;
  const int r = blockIdx.z / P.per, e = blockIdx.z % P.per;
  const int l = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const u32 g = P.g[r];
  const int src = g == 1 ? t : (int)ntt_auto_index((u32)t, g, P.logn);
  out[r * P.out_rstride + e * P.out_estride + l * N + t] =
      __ldg(in + ((long long)r * P.per + e) * P.in_stride + l * N + src);
}

// Permuted sum (double-hoisted BSGS giant steps): for element e and limb l
//   out[e][l][t] (+)= sum_{r < R} in[r][e][l][ntt_auto_index(t, g_r)]  mod q_l,
// i.e. sum_r tau_{g_r}(in_r) in the NTT domain.  Limb l of an element is limb
// l % lpoly of a poly whose first n_q limbs are chain primes and the rest
// special primes (PQ-basis key-switch products or Q-basis c0 polys).  Four
// terms' loads are issued before their adds (memory-level parallelism).
constexpr int kPermSumMax = 64;
struct PermSumArgs {
  u64* out;
  long long out_estride;
  const u64* in;
  long long in_rstride, in_estride;
  const PrimeConst* pc;
  int lpoly, n_q, n_chain, R, logn, accumulate;
  u32 g[kPermSumMax];
};
__global__ void __launch_bounds__(256) perm_sum_kernel(PermSumArgs A) {
  const long long N = 1ll << A.logn;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  const long long e = blockIdx.z;
  const int lp = l % A.lpoly;
  const u64 q = A.pc[lp < A.n_q ? lp : A.n_chain + (lp - A.n_q)].q;
  u64* o = A.out + e * A.out_estride + (long long)l * N + t;
  const u64* base = A.in + e * A.in_estride + (long long)l * N;
  u64 acc = A.accumulate ? *o : 0ull;
  int r = 0;
  for (; r + 8 <= A.R; r += 8) {  // 8 gathered loads in flight per thread
    u64 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const u32 g = A.g[r + k];
      const int src = g == 1 ? t : (int)ntt_auto_index((u32)t, g, A.logn);
      v[k] = __ldcs(base + (long long)(r + k) * A.in_rstride + src);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = addmod(acc, v[k], q);
  }
  for (; r < A.R; ++r) {
    const u32 g = A.g[r];
    const int src = g == 1 ? t : (int)ntt_auto_index((u32)t, g, A.logn);
    acc = addmod(acc, __ldcs(base + (long long)r * A.in_rstride + src), q);
  }
  *o = acc;
}

// from_i64 (rns_poly.cpp:218-227): small signed ints -> every limb.
// v is [batch][N] int64; out [batch][limbs][N].
__global__ void from_i64_kernel(u64* out, const long long* v, const PrimeConst* pc, LimbTable lt,
                                int logn) {
  const int per_limb = (1 << logn) / blockDim.x;
  const long long inst = blockIdx.x / per_limb;
  const int t = (blockIdx.x % per_limb) * blockDim.x + threadIdx.x;
  const long long b = inst / lt.count;
  const int e = (int)(inst % lt.count);
  const u64 q = pc[lt.prime[e]].q;
  const long long x = v[(b << logn) + t];
  u64 r;
  if (x >= 0) {
    r = (u64)x % q;
  } else {
    const u64 m = (u64)(-x) % q;
    r = m ? q - m : 0;
  }
  out[(b * lt.stride + lt.off[e]) * (1ll << logn) + t] = r;
}

// x mod q for values < 2^64 (after an NCCL uint64 sum of partial ciphertexts)
__global__ void reduce_kernel(EwArgs A) {
  const int per_limb = (1 << A.logn) / blockDim.x;
  const long long inst = blockIdx.x / per_limb;
  const int t = (blockIdx.x % per_limb) * blockDim.x + threadIdx.x;
  const long long b = inst / A.lt.count;
  const int e = (int)(inst % A.lt.count);
  const PrimeConst& P = A.pc[A.lt.prime[e]];
  const long long i = (b * A.lt.stride + A.lt.off[e]) * (1ll << A.logn) + t;
  const u64 x = A.out[i];
  A.out[i] = csub(x - mulhi64(x, P.onep) * P.q, P.q);
}

// ------------------------------------------------------------ key switching
// ModUp basis conversion for one digit (non-centred FastBConv):
//   x_i = [a_i * (Qhat_i)^-1]_{q_i},  y_j = sum_i x_i [Qhat_i]_{p_j}
// coef: [batch][n_q][N] coefficient-domain c1; out: digit block
// [batch][ext][N] (only non-digit limbs written, in coefficient domain)
struct ModUpArgs {
  const u64* coef;
  u64* out;
  const PrimeConst* pc;
  const SC* qhinv;   // [alpha] for this digit
  const SC* conv;    // [alpha][n_prime_total] indexed by prime index
  int lo, cnt;       // digit limbs [lo, lo+cnt)
  int n_q, n_chain, n_special, n_total;
  long long out_stride;  // words between batch elements of out
  int logn;
};

template <int MAXA>
__global__ void modup_bconv_kernel(ModUpArgs A) {
  const int N = 1 << A.logn;
  const long long b = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const u64* cb = A.coef + b * (long long)A.n_q * N;
  // FP64 pipe when every source prime of the digit and the target prime are
  // < 2^47 (exact double arithmetic, hx_ntt.cuh); integer Shoup otherwise
  bool src_f64 = true;
#pragma unroll
  for (int i = 0; i < MAXA; ++i)
    if (i < A.cnt) src_f64 = src_f64 && A.pc[A.lo + i].f64;
  u64 x[MAXA];
  double xd[MAXA];
#pragma unroll
  for (int i = 0; i < MAXA; ++i) {
    if (i < A.cnt) {
      const PrimeConst& P = A.pc[A.lo + i];
      const SC c = A.qhinv[i];
      const u64 a = cb[(long long)(A.lo + i) * N + t];
      if (src_f64) {
        const double w = __longlong_as_double((long long)u64_to_f64bits(c.w));
        const double v = mulmod_f64(__longlong_as_double((long long)u64_to_f64bits(a)), w,
                                    __dmul_rn(w, P.qinv_d), P.qd);
        x[i] = f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);  // canonical [0, q)
        xd[i] = __longlong_as_double((long long)u64_to_f64bits(x[i]));
      } else {
        x[i] = csub(shoup_lazy(a, c.w, c.wp, P.q), P.q);
        xd[i] = 0.0;
      }
    }
  }
  u64* ob = A.out + b * A.out_stride;
  const int ext = A.n_q + A.n_special;
  for (int j = 0; j < ext; ++j) {
    if (j >= A.lo && j < A.lo + A.cnt) continue;
    const int pj = j < A.n_q ? j : A.n_chain + (j - A.n_q);
    const PrimeConst& P = A.pc[pj];
    if (src_f64 && P.f64) {
      double acc = 0.0;  // |acc| < cnt q: exact
#pragma unroll
      for (int i = 0; i < MAXA; ++i) {
        if (i < A.cnt) {
          const double w = __longlong_as_double((long long)u64_to_f64bits(A.conv[i * A.n_total + pj].w));
          acc = __dadd_rn(acc, mulmod_f64(xd[i], w, __dmul_rn(w, P.qinv_d), P.qd));
        }
      }
      ob[(long long)j * N + t] = f64bits_to_residue((u64)__double_as_longlong(acc), P.qd, P.qinv_d);
    } else {
      u64 y = 0;
#pragma unroll
      for (int i = 0; i < MAXA; ++i) {
        if (i < A.cnt) {
          const SC c = A.conv[i * A.n_total + pj];
          y = csub(y + shoup_lazy(x[i], c.w, c.wp, P.q), P.two_q);
        }
      }
      ob[(long long)j * N + t] = csub(y, P.q);
    }
  }
}

// Key inner product with the NTT-domain automorphism folded into the digit
// read: u_c[j][t] = sum_d D_d[j][perm_g(t)] * key_{d,c}[kl(j)][t]
// (mul_acc, rns_poly.cpp:102-110, with lazy 128-bit accumulation).  The key
// words of a (j, t) are held in registers and reused across the batch.
// Several keys per launch, E = `batch` elements per key.  shared = 1: every
// key applies to the same digit elements 0..E-1 (hoisted rotations of a
// batch); shared = 0: key r applies to its own digit elements r E .. r E + E-1
// (independent rotations grouped by key, e.g. the BSGS giant step j of every
// row block).  Output element (r, e) at u + (r E + e) 2 ext N.
// blockIdx.z = r * slices + element slice.
constexpr int kMaxKeys = 64;
struct InnerArgs {
  const u64* digits;  // [elements][dnum][ext][N]
  const u64* keys[kMaxKeys];  // [dnum_max][2][full][N] each
  int n_keys, shared, slices;
  u64* u;             // [n_keys][E][2][ext][N]
  const PrimeConst* pc;
  int n_q, n_chain, n_special, dnum, batch;
  u32 g;  // 1 = identity (input-side automorphism of the digits)
  int logn;
  // own limbs: when c1 is set, digit d's own chain limbs j in [d alpha,
  // d alpha + alpha) are read from the ModUp input c1 (element stride
  // c1_stride words) -- ModUp then skips copying them into the digit buffer
  const u64* c1;
  long long c1_stride;
  int alpha;
  // compressed keys (hx_keygen_*_c): bit r of cmask set -> keys[r] holds only
  // the b half, [dnum_max][full][N]; the uniform half is regenerated:
  // a[d][kl][t] = uniform_word(kseed[r], (d full + kl) N + tau(t)), tau the
  // key's layout permutation (kg[r] = g^-1 for rotation layout, 1 standard)
  unsigned long long cmask;
  u64 kseed[kMaxKeys];
  u32 kg[kMaxKeys];
};

// FP64 variant for limbs with q < 2^43: the key words are split once into
// 20-bit halves held as doubles, every digit word is split on load, and the
// dnum-term inner product is accumulated exactly as S11 2^40 + S10 2^20 + S00
// (see the BSGS MAC in hx_bsgs.cu for the bounds) on the FP64 pipe; one exact
// modular combine per output word.  `limbs` lists the limbs j of this class.
__device__ __forceinline__ void split20_d(u64 v, double& hi, double& lo) {
  hi = __dsub_rn(__longlong_as_double((long long)((v >> 20) | 0x4330000000000000ull)), kTwo52);
  lo = __dsub_rn(__longlong_as_double((long long)((v & 0xFFFFFull) | 0x4330000000000000ull)), kTwo52);
}

__device__ __forceinline__ u64 combine_split(const double (&s)[3], const PrimeConst& P) {
  const double v = __dadd_rn(__dadd_rn(mulmod_f64(s[0], P.r40_d, P.r40_q, P.qd),
                                       mulmod_f64(s[1], P.r20_d, P.r20_q, P.qd)),
                             centre_f64(s[2], P.qd, P.qinv_d));
  return f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);
}

// 24-bit split for the key inner product (q < 2^47, dnum <= 8): with
// x = xh 2^24 + xl (xh < 2^23), S_hh < 8 2^46, S_hl < 8 2^48, S_ll < 8 2^48 --
// every sum below 2^52, exact; value = S_hh 2^48 + S_hl 2^24 + S_ll mod q.
__device__ __forceinline__ void split24_d(u64 v, double& hi, double& lo) {
  hi = __dsub_rn(__longlong_as_double((long long)((v >> 24) | 0x4330000000000000ull)), kTwo52);
  lo = __dsub_rn(__longlong_as_double((long long)((v & 0xFFFFFFull) | 0x4330000000000000ull)), kTwo52);
}

__device__ __forceinline__ u64 combine_split24(const double (&s)[3], const PrimeConst& P) {
  const double v = __dadd_rn(__dadd_rn(mulmod_f64(s[0], P.r48_d, P.r48_q, P.qd),
                                       mulmod_f64(s[1], P.r24_d, P.r24_q, P.qd)),
                             centre_f64(s[2], P.qd, P.qinv_d));
  return f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);
}

#ifndef HX_KSF_MINB
#define HX_KSF_MINB 2
#endif
#ifndef HX_KSI_MINB
#define HX_KSI_MINB 2
#endif
template <int MAXD>
__global__ void __launch_bounds__(256, HX_KSF_MINB) ks_inner_f64_kernel(InnerArgs A, const int* limbs) {
  const int N = 1 << A.logn;
  const int ext = A.n_q + A.n_special, full = A.n_chain + A.n_special;
  // (key x slice) fastest, coefficient tile slowest: the CTAs in flight share one
  // (limb, tile).  With hoisted rotations (shared digits, many keys) every key
  // otherwise re-reads the chunk's digit limbs from HBM -- 58 GB of digit words
  // against 7 GB of keys per 16-ciphertext chunk of the hoisted-32 batch; now
  // the keys of a (limb, tile) run together and find the digits in L2 (default
  // load policy when the digits are shared, evict-first when read once).
  const int j = limbs[blockIdx.y];
  const int t = blockIdx.z * blockDim.x + threadIdx.x;
  const int kl = j < A.n_q ? j : A.n_chain + (j - A.n_q);
  const int r = blockIdx.x / A.slices, slice = blockIdx.x % A.slices;
  const u64* key = A.keys[r];
  const int E = A.batch;
  const PrimeConst& P = A.pc[kl];
  const bool comp = (A.cmask >> r) & 1ull;
  const bool reuse = A.shared && A.n_keys > 1;
  const u64 ta = (!comp || A.kg[r] <= 1) ? (u64)t : (u64)ntt_auto_index((u32)t, A.kg[r], A.logn);
#ifndef HX_KSF_SPLIT
#define HX_KSF_SPLIT 1  // 1: the 24-bit split MAC (3 exact partial sums, one reduction per output)
#endif
  // HX_KSF_SPLIT=0: products by one exact mulmod_f64h each instead (what the
  // one-element kernel uses).  With the key split held in registers over the
  // batch slice the split MAC is the faster one here: hoisted-32 743 vs 762 ms.
  double kh[MAXD][2], klo[MAXD][2];
#pragma unroll
  for (int d = 0; d < MAXD; ++d)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      u64 kw = 0;
      if (d < A.dnum) kw = comp ? (c == 0 ? __ldg(key + ((long long)d * full + kl) * N + t)
                                           : uniform_word(A.kseed[r], ((u64)d * full + kl) * N + ta, P.q))
                                : __ldg(key + (((long long)d * 2 + c) * full + kl) * N + t);
      if (HX_KSF_SPLIT) {
        split24_d(kw, kh[d][c], klo[d][c]);
      } else {
        kh[d][c] = __longlong_as_double((long long)u64_to_f64bits(kw));
        klo[d][c] = 0.0;
      }
    }
  const int src = (A.g == 1) ? t : (int)ntt_auto_index((u32)t, A.g, A.logn);
  const int per = (E + A.slices - 1) / A.slices;
  const int b_lo = slice * per, b_hi = min(E, b_lo + per);
  const long long dstride = (long long)A.dnum * ext * N;
  const long long ebase = A.shared ? 0 : (long long)r * E;
  u64* ubase = A.u + (long long)r * E * 2 * ext * N;
  const int down = (A.c1 && j < A.n_q) ? j / A.alpha : -1;  // digit owning limb j
  // software pipeline over the batch slice: element b + 1's digit words are
  // in flight while element b's products run (HBM latency x bandwidth needs
  // more bytes in flight per SM than one element's 8 words per thread)
  u64 vn[MAXD];
  auto load = [&](int b, u64 (&v)[MAXD]) {
    const u64* Db = A.digits + (ebase + b) * dstride + (long long)j * N + src;
    const u64* Cb = down >= 0 ? A.c1 + (ebase + b) * A.c1_stride + (long long)j * N + src : nullptr;
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      v[d] = d < A.dnum ? (reuse ? __ldg(d == down ? Cb : Db + (long long)d * ext * N)
                                 : __ldcs(d == down ? Cb : Db + (long long)d * ext * N))
                        : 0ull;
  };
  if (b_lo < b_hi) load(b_lo, vn);
  for (int b = b_lo; b < b_hi; ++b) {
    u64 v[MAXD];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) v[d] = vn[d];
    if (b + 1 < b_hi) load(b + 1, vn);
    u64* ub = ubase + (long long)b * 2 * ext * N + (long long)j * N + t;
    if (HX_KSF_SPLIT) {
      double s[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        double xh, xl;
        split24_d(v[d], xh, xl);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          s[c][0] = __fma_rn(xh, kh[d][c], s[c][0]);
          s[c][1] = __fma_rn(xh, klo[d][c], s[c][1]);
          s[c][1] = __fma_rn(xl, kh[d][c], s[c][1]);
          s[c][2] = __fma_rn(xl, klo[d][c], s[c][2]);
        }
      }
      ub[0] = combine_split24(s[0], P);
      ub[(long long)ext * N] = combine_split24(s[1], P);
    } else {
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        if (d < A.dnum) {
          const double y = __longlong_as_double((long long)u64_to_f64bits(v[d]));
          acc0 = __dadd_rn(acc0, mulmod_f64h(y, kh[d][0], P.qinv_d, P.qd));
          acc1 = __dadd_rn(acc1, mulmod_f64h(y, kh[d][1], P.qinv_d, P.qd));
        }
      }
      ub[0] = f64bits_to_residue((u64)__double_as_longlong(acc0), P.qd, P.qinv_d);
      ub[(long long)ext * N] = f64bits_to_residue((u64)__double_as_longlong(acc1), P.qd, P.qinv_d);
    }
  }
}

// One element per block row (E <= 2, e.g. BSGS giant steps of a single
// ciphertext): no key reuse to amortise, so nothing is held across elements --
// the digit and key words of a (limb, coefficient) are all loaded up front
// (3 dnum loads in flight per thread) and consumed at once, with the register
// budget of 3 CTAs / SM instead of 2.
// Grid: (key x element) runs FASTEST (blockIdx.x), the coefficient tile slowest
// (blockIdx.z): the CTAs in flight then share one (limb, tile) digit slice --
// with the tile fastest every key re-read all dnum digit limbs from HBM (ncu on
// the 63 hoisted baby steps of a W1 matvec: 18.2 GB read for 12.2 GB of keys,
// L2 hit rate 0.01 %).  The digits are loaded with the default policy, the
// key words (used once) evict-first.
template <int MAXD>
__global__ void __launch_bounds__(256, 3) ks_inner_f64_one_kernel(InnerArgs A, const int* limbs) {
  const int N = 1 << A.logn;
  const int ext = A.n_q + A.n_special, full = A.n_chain + A.n_special;
  const int j = limbs[blockIdx.y];
  const int t = blockIdx.z * blockDim.x + threadIdx.x;
  const int kl = j < A.n_q ? j : A.n_chain + (j - A.n_q);
  const int E = A.batch;
  const int r = blockIdx.x / E, b = blockIdx.x % E;
  const u64* key = A.keys[r];
  const PrimeConst& P = A.pc[kl];
  const bool comp = (A.cmask >> r) & 1ull;
  const u64 ta = (!comp || A.kg[r] <= 1) ? (u64)t : (u64)ntt_auto_index((u32)t, A.kg[r], A.logn);
  const int src = (A.g == 1) ? t : (int)ntt_auto_index((u32)t, A.g, A.logn);
  const long long dstride = (long long)A.dnum * ext * N;
  const long long e = (A.shared ? 0 : (long long)r * E) + b;
  const int down = (A.c1 && j < A.n_q) ? j / A.alpha : -1;
  const u64* Db = A.digits + e * dstride + (long long)j * N + src;
  const u64* Cb = down >= 0 ? A.c1 + e * A.c1_stride + (long long)j * N + src : nullptr;
  u64 v[MAXD], k0[MAXD], k1[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d < A.dnum) {
      v[d] = __ldg(d == down ? Cb : Db + (long long)d * ext * N);
      if (comp) {
        k0[d] = __ldcs(key + ((long long)d * full + kl) * N + t);
        k1[d] = uniform_word(A.kseed[r], ((u64)d * full + kl) * N + ta, P.q);
      } else {
        k0[d] = __ldcs(key + (((long long)d * 2 + 0) * full + kl) * N + t);
        k1[d] = __ldcs(key + (((long long)d * 2 + 1) * full + kl) * N + t);
      }
    } else {
      v[d] = k0[d] = k1[d] = 0;
    }
  }
  // one exact modular product per (digit, poly) (mulmod_f64h: 6 FP64
  // instructions, no integer split) summed lazily (|acc| < dnum q) and
  // normalised once -- as in ks_row_inner_f64_kernel.  With nothing to amortise
  // over elements the 24-bit split MAC spent more instructions on splitting the
  // 3 dnum words of every element (shift / mask / convert, 6 per word) than on
  // its products: ncu showed the kernel issue-bound (70 % issue, DRAM 54 %).
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d < A.dnum) {
      const double y = __longlong_as_double((long long)u64_to_f64bits(v[d]));
      const double w0 = __longlong_as_double((long long)u64_to_f64bits(k0[d]));
      const double w1 = __longlong_as_double((long long)u64_to_f64bits(k1[d]));
      acc0 = __dadd_rn(acc0, mulmod_f64h(y, w0, P.qinv_d, P.qd));
      acc1 = __dadd_rn(acc1, mulmod_f64h(y, w1, P.qinv_d, P.qd));
    }
  }
  u64* ub = A.u + ((long long)r * E + b) * 2 * ext * N + (long long)j * N + t;
  ub[0] = f64bits_to_residue((u64)__double_as_longlong(acc0), P.qd, P.qinv_d);
  ub[(long long)ext * N] = f64bits_to_residue((u64)__double_as_longlong(acc1), P.qd, P.qinv_d);
}

template <int MAXD>
__global__ void __launch_bounds__(256, HX_KSI_MINB) ks_inner_kernel(InnerArgs A, const int* limbs) {
  const int N = 1 << A.logn;
  const int ext = A.n_q + A.n_special, full = A.n_chain + A.n_special;
  // (key x slice) fastest, coefficient tile slowest: the CTAs in flight share one
  // (limb, tile) -- its key words across the slices of a batch, its digit words
  // across the keys of hoisted rotations (kept in L2: default load policy then)
  const int j = limbs ? limbs[blockIdx.y] : blockIdx.y;
  const int t = blockIdx.z * blockDim.x + threadIdx.x;
  const int kl = j < A.n_q ? j : A.n_chain + (j - A.n_q);
  const int r = blockIdx.x / A.slices, slice = blockIdx.x % A.slices;
  const u64* key = A.keys[r];
  const int E = A.batch;
  const PrimeConst& P = A.pc[kl];
  const bool comp = (A.cmask >> r) & 1ull;
  const bool reuse = A.shared && A.n_keys > 1;  // every key reads the same digits
  const u64 ta = (!comp || A.kg[r] <= 1) ? (u64)t : (u64)ntt_auto_index((u32)t, A.kg[r], A.logn);
  u64 k0[MAXD], k1[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d < A.dnum) {
      if (comp) {
        k0[d] = __ldg(key + ((long long)d * full + kl) * N + t);
        k1[d] = uniform_word(A.kseed[r], ((u64)d * full + kl) * N + ta, P.q);
      } else {
        k0[d] = __ldg(key + (((long long)d * 2 + 0) * full + kl) * N + t);
        k1[d] = __ldg(key + (((long long)d * 2 + 1) * full + kl) * N + t);
      }
    }
  }
  const int src = (A.g == 1) ? t : (int)ntt_auto_index((u32)t, A.g, A.logn);
  // this CTA's slice of the elements; BB ciphertexts per iteration so that
  // MAXD x BB (8-16) independent digit loads are in flight per thread -- at
  // the low levels of the ct-ct matmul (dnum = 1 or 2) that is 8 / 4
  // ciphertexts per iteration
  constexpr int BB = MAXD <= 1 ? 8 : MAXD <= 2 ? 4 : MAXD <= 8 ? 2 : 1;
  const int per = (E + A.slices - 1) / A.slices;
  const int b_lo = slice * per, b_hi = min(E, b_lo + per);
  const long long dstride = (long long)A.dnum * ext * N;
  const long long ebase = A.shared ? 0 : (long long)r * E;  // digit element of e = 0
  u64* ubase = A.u + (long long)r * E * 2 * ext * N;
  const int down = (A.c1 && j < A.n_q) ? j / A.alpha : -1;  // digit owning limb j
  for (int b0 = b_lo; b0 < b_hi; b0 += BB) {
    u64 v[BB][MAXD];
#pragma unroll
    for (int bb = 0; bb < BB; ++bb) {
      const u64* Db = A.digits + (ebase + b0 + bb) * dstride + (long long)j * N + src;
      const u64* Cb = down >= 0 ? A.c1 + (ebase + b0 + bb) * A.c1_stride + (long long)j * N + src : nullptr;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        v[bb][d] = (d < A.dnum && b0 + bb < b_hi)
                       ? (reuse ? __ldg(d == down ? Cb : Db + (long long)d * ext * N)
                                : __ldcs(d == down ? Cb : Db + (long long)d * ext * N))
                       : 0ull;
    }
#pragma unroll
    for (int bb = 0; bb < BB; ++bb) {
      if (b0 + bb >= b_hi) break;
      U128 z0{0, 0}, z1{0, 0};
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        if (d < A.dnum) {
          mac128(z0, v[bb][d], k0[d]);
          mac128(z1, v[bb][d], k1[d]);
        }
      }
      u64* ub = ubase + (long long)(b0 + bb) * 2 * ext * N + (long long)j * N + t;
      ub[0] = reduce128(z0, P);
      ub[(long long)ext * N] = reduce128(z1, P);
    }
  }
}

// ModDown basis conversion P -> Q (centred FastBConv; K = 1 is
// moddown_special, rns_poly.cpp:164-180):
//   x_k = [s_k * (P/p_k)^-1]_{p_k};  v_i = sum_k x_k [P/p_k]_{q_i} - #neg * [P]_{q_i}
// sp: [bp][K][N] coefficient-domain special limbs; conv out: [bp][n_q][N]
struct ModDownArgs {
  const u64* sp;
  u64* conv;
  const PrimeConst* pc;
  const SC* phinv;   // [K]
  const SC* pconv;   // [K][n_chain]  ([P/p_k]_{q_i})
  const double* pconvf;  // [K][n_chain][4] FP64 form for q_i < 2^47 targets
  const u64* pmodq;  // [n_chain]     ([P]_{q_i})
  int n_q, n_chain, n_special, logn;
};

constexpr int kModDownEpt = 2;  // coefficient positions per thread

// per-target constants staged in shared memory once per block: for target i,
// [k][w, w/q, w30, w30/q] (FP64 form), then q, 1/q, [P]_q as doubles (q = 0
// marks an integer-class target)
inline int moddown_smem_bytes(int n_q, int K) { return 8 * n_q * (4 * K + 3); }

template <int MAXK>
__global__ void __launch_bounds__(256) moddown_bconv_kernel(ModDownArgs A) {
  extern __shared__ double mds[];
  const int N = 1 << A.logn;
  const long long b = blockIdx.y;
  const int K = A.n_special, stride = 4 * K + 3;
  for (int idx = threadIdx.x; idx < A.n_q * stride; idx += blockDim.x) {
    const int i = idx / stride, m = idx % stride;
    const PrimeConst& P = A.pc[i];
    double v;
    if (m < 4 * K)
      v = P.f64 ? A.pconvf[((long long)(m >> 2) * A.n_chain + i) * 4 + (m & 3)] : 0.0;
    else if (m == 4 * K)
      v = P.f64 ? P.qd : 0.0;
    else if (m == 4 * K + 1)
      v = P.qinv_d;
    else
      v = P.f64 ? __longlong_as_double((long long)u64_to_f64bits(A.pmodq[i])) : 0.0;
    mds[idx] = v;
  }
  __syncthreads();
  const int t0 = blockIdx.x * blockDim.x * kModDownEpt + threadIdx.x;
  u64 x[kModDownEpt][MAXK];
  int nneg[kModDownEpt];
  double xh[kModDownEpt][MAXK], xl[kModDownEpt][MAXK];
#pragma unroll
  for (int e = 0; e < kModDownEpt; ++e) {
    const int t = t0 + e * blockDim.x;
    nneg[e] = 0;
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      x[e][k] = 0;
      xh[e][k] = xl[e][k] = 0.0;
      if (k < K) {
        const PrimeConst& P = A.pc[A.n_chain + k];
        const SC c = A.phinv[k];
        x[e][k] = csub(shoup_lazy(__ldcs(A.sp + (b * K + k) * N + t), c.w, c.wp, P.q), P.q);
        nneg[e] += x[e][k] > (P.q >> 1);
        // FP64 pipe for the q_i < 2^47 targets: x_k (< 2^60) as two exact 30-bit
        // halves, v = sum_k xh_k [2^30 w_k]_q + xl_k w_k - nneg [P]_q, all exact
        xh[e][k] = __dsub_rn(__longlong_as_double((long long)((x[e][k] >> 30) | 0x4330000000000000ull)), kTwo52);
        xl[e][k] = __dsub_rn(__longlong_as_double((long long)((x[e][k] & 0x3FFFFFFFull) | 0x4330000000000000ull)), kTwo52);
      }
    }
  }
  u64* cb = A.conv + b * (long long)A.n_q * N;
  for (int i = 0; i < A.n_q; ++i) {
    const double* cst = mds + i * stride;
    const double qd = cst[4 * K];
    if (qd != 0.0) {
      const double qinv = cst[4 * K + 1], pm = cst[4 * K + 2];
      double acc[kModDownEpt];
#pragma unroll
      for (int e = 0; e < kModDownEpt; ++e) acc[e] = __fma_rn(-(double)nneg[e], pm, 0.0);
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        if (k < K) {
          const double w = cst[4 * k], wq = cst[4 * k + 1], w30 = cst[4 * k + 2], w30q = cst[4 * k + 3];
#pragma unroll
          for (int e = 0; e < kModDownEpt; ++e) {
            acc[e] = __dadd_rn(acc[e], mulmod_f64(xh[e][k], w30, w30q, qd));
            acc[e] = __dadd_rn(acc[e], mulmod_f64(xl[e][k], w, wq, qd));
          }
        }
      }
#pragma unroll
      for (int e = 0; e < kModDownEpt; ++e)
        __stcs(cb + (long long)i * N + t0 + e * blockDim.x,
               f64bits_to_residue((u64)__double_as_longlong(acc[e]), qd, qinv));
      continue;
    }
    const PrimeConst& P = A.pc[i];
#pragma unroll
    for (int e = 0; e < kModDownEpt; ++e) {
      u64 v = 0;
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        if (k < K) {
          const SC c = A.pconv[k * A.n_chain + i];
          v = csub(v + shoup_lazy(x[e][k], c.w, c.wp, P.q), P.two_q);
        }
      }
      v = csub(v, P.q);
      const u64 pm = A.pmodq[i];
      for (int m = 0; m < nneg[e]; ++m) v = submod(v, pm, P.q);
      cb[(long long)i * N + t0 + e * blockDim.x] = v;
    }
  }
}

// out_i = (u_i - conv_i) * P^-1 mod q_i   (NTT domain), optionally
// + tau_g(add)_i.  All strides in words between consecutive polys.
struct CombineArgs {
  const u64* u;
  const u64* conv;
  const u64* add;  // may be null
  u64* out;
  const PrimeConst* pc;
  const SC* pinv;  // [n_chain]
  int n_q;
  long long u_stride, conv_stride, out_stride, add_stride;
  // `add` applies to polys b with b % add_every == 0; its element is
  // (b / add_every) % add_period (add_period 0: no wrap)
  long long add_every, add_period;
  u32 add_g;  // 1 = no automorphism on `add`
  int logn;
  // Fused output automorphism (rotations): when perm != 0, poly b is poly
  // (b & 1) of ciphertext q = b / 2 = r per + e, and the result is written
  // permuted, out[r rstride + e estride + (b & 1) n_q N + i N + t] =
  // result[tau_{pg[r]}(t)] (u, conv and add gathered at the same source).
  int perm, per;
  long long out_rstride, out_estride;
  u32 pg[64];
};

constexpr int kCombineEpt = 8;  // elements per thread (amortises the per-poly setup)

__global__ void __launch_bounds__(256) combine_kernel(CombineArgs A) {
  const int N = 1 << A.logn;
  const long long b = blockIdx.z;
  long long ba = b / A.add_every;
  if (A.add_period) ba %= A.add_period;
  const bool do_add = A.add && (b % A.add_every) == 0;
  const int i = blockIdx.y;
  const PrimeConst& P = A.pc[i];
  const SC c = A.pinv[i];
  u32 g = 1;
  long long ob = b * A.out_stride;
  if (A.perm) {
    const long long q = b >> 1;
    const long long rr = q / A.per, e = q % A.per;
    g = A.pg[rr];
    ob = rr * A.out_rstride + e * A.out_estride + (b & 1) * (long long)A.n_q * N;
  }
  const u32 ag = A.perm ? g : A.add_g;
  const u64* ub = A.u + b * A.u_stride + (long long)i * N;
  const u64* cb = A.conv + b * A.conv_stride + (long long)i * N;
  const u64* abase = do_add ? A.add + ba * A.add_stride + (long long)i * N : nullptr;
  u64* outb = A.out + ob + (long long)i * N;
  const double wd = __longlong_as_double((long long)u64_to_f64bits(c.w));
  const int t0 = blockIdx.x * blockDim.x * kCombineEpt + threadIdx.x;
  u64 uu[kCombineEpt], cv[kCombineEpt], ad[kCombineEpt];
#pragma unroll
  for (int k = 0; k < kCombineEpt; ++k) {  // all loads in flight first
    const int t = t0 + k * blockDim.x;
    const int src = g != 1 ? (int)ntt_auto_index((u32)t, g, A.logn) : t;
    const int asrc = ag != 1 ? (int)ntt_auto_index((u32)t, ag, A.logn) : t;
    uu[k] = __ldg(ub + src);
    cv[k] = __ldg(cb + src);
    ad[k] = do_add ? __ldg(abase + asrc) : 0ull;
  }
#pragma unroll
  for (int k = 0; k < kCombineEpt; ++k) {
    u64 r;
    if (P.f64) {  // q < 2^47: (u - conv) P^-1 (+ add) on the FP64 pipe, exact
      const double du = __longlong_as_double((long long)u64_to_f64bits(uu[k]));
      const double dc = __longlong_as_double((long long)u64_to_f64bits(cv[k]));
      double v = mulmod_f64h(__dsub_rn(du, dc), wd, P.qinv_d, P.qd);
      v = __dadd_rn(v, __longlong_as_double((long long)u64_to_f64bits(ad[k])));  // |v| < 2q
      r = f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);
    } else {
      r = csub(shoup_lazy(uu[k] + P.q - cv[k], c.w, c.wp, P.q), P.q);
      if (do_add) r = addmod(r, ad[k], P.q);
    }
    __stcs(outb + t0 + k * blockDim.x, r);
  }
}

// Rescale helper (rns_poly.cpp:144-162): from the coefficient-domain last limb
// c, write [centred(c)]_{q_i} for every i < n_q - 1.
struct RescaleArgs {
  const u64* last;  // [bp][N]
  u64* out;         // [bp][n_q-1][N]
  const PrimeConst* pc;
  const u64* qlmod;  // [n_q-1]: [q_l]_{q_i}
  int n_q, logn;
};

__global__ void rescale_lift_kernel(RescaleArgs A) {
  const int N = 1 << A.logn;
  const long long b = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const u64 ql = A.pc[A.n_q - 1].q;
  const u64 c = A.last[b * N + t];
  const bool neg = c > (ql >> 1);
  for (int i = 0; i < A.n_q - 1; ++i) {
    const PrimeConst& P = A.pc[i];
    u64 r = csub(c - mulhi64(c, P.onep) * P.q, P.q);
    if (neg) r = submod(r, A.qlmod[i], P.q);
    A.out[(b * (A.n_q - 1) + i) * N + t] = r;
  }
}

// Tensor (LatticeContext::mul x4, rns_poly.cpp:91-100):
// d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1.  a, b: [batch][2][n_q][N],
// out: [batch][3][n_q][N]
__global__ void tensor_kernel(u64* out, const u64* a, const u64* b, const PrimeConst* pc, int n_q,
                              int logn) {
  const int N = 1 << logn;
  const long long bt = blockIdx.z;
  const int i = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst& P = pc[i];
  const long long L = (long long)n_q * N;
  const u64* ab = a + bt * 2 * L + (long long)i * N + t;
  const u64* bb = b + bt * 2 * L + (long long)i * N + t;
  const u64 a0 = ab[0], a1 = ab[L], b0 = bb[0], b1 = bb[L];
  U128 z{0, 0};
  mac128(z, a0, b1);
  mac128(z, a1, b0);
  u64* ob = out + bt * 3 * L + (long long)i * N + t;
  ob[0] = mulmod(a0, b0, P);
  ob[L] = reduce128(z, P);
  ob[2 * L] = mulmod(a1, b1, P);
}

// ------------------------------------------------------------ keys
// ksk_d over the full basis: b = e - a s + [P]_{q_l} s' on chain limbs of digit d
// ------------------------------------------------------------ samplers

// out [copies][limbs][N]: uniform mod the limb's prime, floor(r q / 2^128)
// over 128 random bits r
__global__ void sample_uniform_kernel(u64* out, const PrimeConst* pc, LimbTable lt, int logn, u64 seed) {
  const long long N = 1ll << logn;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // word index
  const long long limb = i >> logn;
  const u64 q = pc[lt.prime[limb % lt.count]].q;
  out[i] = uniform_word(seed, (u64)i, q);
  (void)N;
}

// full key words from a compressed key: out[d][0] = b[d], out[d][1] = a[d]
__global__ void key_expand_kernel(u64* out, const u64* ckey, const PrimeConst* pc, int full, int logn, u64 seed,
                                  u32 kg) {
  const long long N = 1ll << logn;
  const int d = blockIdx.z, kl = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const u64 ta = kg <= 1 ? (u64)t : (u64)ntt_auto_index((u32)t, kg, logn);
  out[(((long long)d * 2 + 0) * full + kl) * N + t] = ckey[((long long)d * full + kl) * N + t];
  out[(((long long)d * 2 + 1) * full + kl) * N + t] = uniform_word(seed, ((u64)d * full + kl) * N + ta, pc[kl].q);
}

__global__ void sample_cbd_kernel(long long* e, long long count, u64 seed) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const u64 r = splitmix64(seed ^ splitmix64((u64)i ^ 0xA5A5A5A5A5A5A5A5ull));
  e[i] = (long long)__popcll(r & 0x1fffffull) - (long long)__popcll((r >> 21) & 0x1fffffull);
}

__global__ void keygen_kernel(u64* key, const u64* en, const u64* s_full, const u64* sp_full,
                              const u64* a_full, const PrimeConst* pc, const u64* pmodq,
                              int n_chain, int n_total, int alpha, int logn) {
  const int N = 1 << logn;
  const int d = blockIdx.z, l = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst& P = pc[l];
  const long long li = (long long)l * N + t;
  const u64 a = a_full[(long long)d * n_total * N + li];
  const u64 as = mulmod(a, s_full[li], P);
  u64 v = submod(en[(long long)d * n_total * N + li], as, P.q);
  const int lo = d * alpha, hi = min(lo + alpha, n_chain);
  if (l >= lo && l < hi) v = addmod(v, mulmod(pmodq[l], sp_full[li], P), P.q);
  key[((long long)d * 2 + 0) * n_total * N + li] = v;
  key[((long long)d * 2 + 1) * n_total * N + li] = a;
}

// ct = (m + e - a s, a)
__global__ void encrypt_kernel(u64* ct, const u64* m, const u64* en, const u64* s_full,
                               const u64* a, const PrimeConst* pc, int n_q, int logn) {
  const int N = 1 << logn;
  const int i = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst& P = pc[i];
  const long long idx = (long long)i * N + t;
  const u64 as = mulmod(a[idx], s_full[idx], P);
  ct[idx] = submod(addmod(m[idx], en[idx], P.q), as, P.q);
  ct[(long long)n_q * N + idx] = a[idx];
}

// m = c0 + c1 s
__global__ void decrypt_kernel(u64* m, const u64* ct, const u64* s_full, const PrimeConst* pc,
                               int n_q, int logn) {
  const int N = 1 << logn;
  const long long b = blockIdx.z;
  const int i = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst& P = pc[i];
  const long long L = (long long)n_q * N, idx = (long long)i * N + t;
  U128 z{ct[b * 2 * L + idx], 0};
  mac128(z, ct[b * 2 * L + L + idx], s_full[idx]);
  m[b * L + idx] = reduce128(z, P);
}

}  // namespace hx
