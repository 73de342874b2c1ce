// hx_common.cuh -- 64-bit RNS modular arithmetic for sm_100a and the device
// context shared by every kernel of libhx_b200.
//
// Residues are u64 in [0, q) at every API boundary, q < 2^62.  Inside kernels
// values are kept lazily in [0, 2q) / [0, 4q) (Harvey) and products are
// accumulated unreduced in 128 bits (one reduction per output word).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hx {

using u64 = unsigned long long;
using u32 = unsigned int;

constexpr int kMaxPrimes = 64;

// Per-prime constants (device-resident array, one entry per prime; chain
// primes first, then special primes -- the LatticeContext order of
// rns_poly.cpp:11-22 generalised to K special primes).
struct PrimeConst {
  u64 q;       // modulus
  u64 two_q;   // 2q
  u64 r64;     // 2^64 mod q
  u64 r64p;    // Shoup companion of r64
  u64 onep;    // floor(2^64 / q): Shoup companion of w = 1
  u64 ninv;    // N^-1 mod q
  u64 ninvp;
  u64 w1n;     // inv-twiddle[1] * N^-1 (last INTT stage, fused scale)
  u64 w1np;
  const ulonglong2* tw_fwd;  // (psi^brv(i), shoup) i in [0, N)
  const ulonglong2* tw_inv;  // (psi^-brv(i), shoup)
  // FP64 butterfly path (q < 2^47 only; null otherwise)
  bool f64;
  double qd, qinv_d;         // q, 1/q
  double ninv_d, ninv_q;     // N^-1, N^-1 / q
  double w1n_d, w1n_q;       // last-stage twiddle * N^-1, / q
  double r20_d, r20_q;       // 2^20 mod q (and / q): 20-bit split MAC combine
  double r40_d, r40_q;       // 2^40 mod q
  double r24_d, r24_q;       // 2^24 mod q: 24-bit split key inner product (q < 2^47)
  double r48_d, r48_q;       // 2^48 mod q
  const double* twf_fwd;     // w as double (w / q formed in-kernel)
  const double* twf_inv;
};

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// a*w mod q lazily in [0, 2q) for any a < 2^64, w < q (Shoup; modmath.hpp:101-105
// without the final conditional subtraction).
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wp, u64 q) {
  return a * w - mulhi64(a, wp) * q;
}

// Same product with the Shoup quotient's lowest partial product dropped:
// hi64(a wp) ~ ah wh + hi32(ah wl) + hi32(al wh) undershoots the exact
// quotient by at most 2, so the result is in [0, 4q) (q < 2^61).  3 multiplies
// instead of the 64x64 high product's 4 plus carry chain: the integer NTT
// butterflies are IMAD-bound.
__device__ __forceinline__ u64 shoup_lazy4(u64 a, u64 w, u64 wp, u64 q) {
  const u32 al = (u32)a, ah = (u32)(a >> 32), wl = (u32)wp, wh = (u32)(wp >> 32);
  const u64 qh = (u64)ah * wh + __umulhi(ah, wl) + __umulhi(al, wh);
  return a * w - qh * q;
}

__device__ __forceinline__ u64 csub(u64 a, u64 m) { return a >= m ? a - m : a; }

// [0, 4q) -> [0, q)
__device__ __forceinline__ u64 reduce4(u64 a, u64 q, u64 two_q) { return csub(csub(a, two_q), q); }

__device__ __forceinline__ u64 addmod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// 128-bit accumulator
struct U128 {
  u64 lo, hi;
};

__device__ __forceinline__ void mac128(U128& acc, u64 a, u64 b) {
  asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\t"
      "madc.hi.u64 %1, %2, %3, %1;"
      : "+l"(acc.lo), "+l"(acc.hi)
      : "l"(a), "l"(b));
}

__device__ __forceinline__ void add128(U128& acc, u64 v) {
  asm("add.cc.u64 %0, %0, %2;\n\t"
      "addc.u64 %1, %1, 0;"
      : "+l"(acc.lo), "+l"(acc.hi)
      : "l"(v));
}

// exact (hi*2^64 + lo) mod q for any 128-bit value:
//   hi*2^64 = hi * (2^64 mod q)   (Shoup, lazy [0,2q))
//   lo      = lo * 1              (Shoup with w = 1, lazy [0,2q))
__device__ __forceinline__ u64 reduce128(const U128& z, const PrimeConst& P) {
  const u64 a = shoup_lazy(z.hi, P.r64, P.r64p, P.q);
  const u64 b = z.lo - mulhi64(z.lo, P.onep) * P.q;
  return reduce4(a + b, P.q, P.two_q);
}

__device__ __forceinline__ u64 mulmod(u64 a, u64 b, const PrimeConst& P) {
  U128 z{a * b, mulhi64(a, b)};
  return reduce128(z, P);
}

// --------------------------------------------------------- NTT automorphism
// NTT(tau_g a)[k] = NTT(a)[brv(((g (2 brv(k) + 1)) mod 2N - 1) / 2)]
// (derived from the NTT layout of ntt.cpp:57-74; verified by tests against
// LatticeContext::automorphism, rns_poly.cpp:124-142)
__device__ __forceinline__ u32 ntt_auto_index(u32 k, u32 g, int logn) {
  const u32 brk = __brev(k) >> (32 - logn);
  const u32 e = 2u * brk + 1u;
  const u32 m = (u32)(((unsigned long long)g * e) & ((2ull << logn) - 1ull));
  return __brev((m - 1u) >> 1) >> (32 - logn);
}

}  // namespace hx
