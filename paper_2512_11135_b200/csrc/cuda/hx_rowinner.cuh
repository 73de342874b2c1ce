// hx_rowinner.cuh -- ModUp's last (ROW) NTT pass fused with the key inner
// product, FP64-class limbs, one uncompressed key per group of elements.
//
// Replaces, for every FP64-class extended limb j of a key switch,
//   ntt_pass_kernel<FWD, ROW, ..., F64>  on the 8 ModUp digits of limb j
//                                        (forward NTT, last stages; ntt.cpp:57-74)
//   ks_inner_f64_kernel                  u_c[j] = sum_d D_d[j] (.) K_{d,c}[j]
//                                        (the SPEC key_switch inner product,
//                                        SPEC.md:193-201; rns_poly.cpp:102-110)
// A CTA owns one ROW tile (2^OB rows of 2^S words) of limb j of one
// ciphertext: the tile's ROW twiddles are staged in shared memory once and
// reused by all dnum digits; each digit's COL-pass output tile is loaded,
// transformed in registers (the ordinary ROW group schedule), staged through
// shared memory into the coalesced layout and multiplied straight into two
// FP64 accumulators by the key words.  The transformed digits never reach
// HBM: per ciphertext this removes one write and one read of every FP64-class
// ModUp limb (8 x ~20 limbs x 512 KB at config 2).
//
// Digit d == owner(j) (the digit limb j belongs to) is c1's own limb j, read
// in NTT form from the ModUp input (no transform).  Products are
// mulmod_f64h (exact, |y w| < 2^99: y < 17 q after the lazy forward stages,
// q < 2^47), summed lazily (|acc| < (dnum + 1) q), normalised once into
// [0, q): the output words equal ks_inner_f64_kernel's bit for bit.
// The grid runs the ciphertext index fastest, so the CTAs in flight share
// one (limb, tile) key slice through L2 and every key word comes from HBM
// about once per launch.
#pragma once

#include "hx_common.cuh"
#include "hx_ntt.cuh"

namespace hx {

#ifndef HX_ROWINNER_MINB
#define HX_ROWINNER_MINB 3
#endif
constexpr int kRowInnerMaxKeys = 64;
// HX_RI_PREFETCH: the next digit's COL-pass tile is copied into a second
// shared-memory buffer (cp.async, 16 B per copy) while the current digit is
// transformed, so the digit loop no longer waits on an HBM load per digit
#ifndef HX_RI_PREFETCH
#define HX_RI_PREFETCH 0
#endif
constexpr bool kRiPrefetch = HX_RI_PREFETCH != 0;
// HX_RI_KEYPF: at the top of a digit's iteration every thread asks L1 for one
// 128-byte line of each of the digit's two key tiles (the tile is T lines), so
// the 32 key loads at the end of the iteration -- after the ROW stages -- hit
// L1 instead of waiting on L2 / HBM; 2: also the next digit's COL-pass tile
#ifndef HX_RI_KEYPF
#define HX_RI_KEYPF 0
#endif
constexpr int kRiKeyPf = HX_RI_KEYPF;
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}
// shared memory of ks_row_inner_f64_kernel: exchange tile + ROW twiddles
// (ntt_smem_bytes<true, S, OB, true>) + two prefetch tiles
template <int S, int OB>
constexpr int row_inner_tw_words() {
  return (17 * (1 << OB) * ((1 << S) - 1) / 16 + 16 + 1) & ~1;
}
template <int S, int OB>
constexpr int row_inner_smem_bytes() {
  return 8 * ((1 << (S + OB)) + row_inner_tw_words<S, OB>() + (kRiPrefetch ? 2 * (1 << (S + OB)) : 0));
}

struct RowInnerArgs {
  const u64* digits;  // [E][dnum][ext][N]: COL-pass output (FP64 bits) of the ModUp limbs
  const u64* c1;      // own limbs, NTT form residues: element e limb j at c1 + e c1_stride + j N
  long long c1_stride;
  // element b uses keys[b / per_key] ([dnum][2][full][N]): one key over the
  // whole batch, or R keys of per_key consecutive elements each (grouped
  // rotations); the elements of one key run back to back along the grid
  const u64* keys[kRowInnerMaxKeys];
  int per_key;
  u64* u;             // [E][2][ext][N]
  const PrimeConst* pc;
  const int* limbs;   // FP64-class extended limbs j (blockIdx order)
  int n_limbs, n_q, n_chain, n_special, dnum, alpha, batch, logn;
};

template <int S, int OB, int MAXD>
__global__ void __launch_bounds__((1 << (S + OB)) / 16, HX_ROWINNER_MINB) ks_row_inner_f64_kernel(RowInnerArgs A) {
  constexpr int TILE = 1 << (S + OB);
  constexpr int T = TILE / 16;
  extern __shared__ u64 dyn_smem[];
  u64* sm = dyn_smem;
  double* sm_tw = reinterpret_cast<double*>(dyn_smem + TILE);
  const int t = threadIdx.x;
  const long long N = 1ll << A.logn;
  const int tiles = (int)(N / TILE);
  const int E = A.batch;
  const int b = (int)(blockIdx.x % (unsigned)E);
  const long long rest = blockIdx.x / (unsigned)E;
  const int tile = (int)(rest % tiles);
  const int j = A.limbs[rest / tiles];
  const int ext = A.n_q + A.n_special, full = A.n_chain + A.n_special;
  const int kl = j < A.n_q ? j : A.n_chain + (j - A.n_q);
  const PrimeConst P = A.pc[kl];
  const double* twf = P.twf_fwd;
  const long long tofs = (long long)tile * TILE;

  // the tile's ROW twiddles (all S stages), as in ntt_pass_body
  {
    constexpr int kTw = (1 << OB) * ((1 << S) - 1);
    const long long row0 = (long long)tile << OB;
#pragma unroll
    for (int i = 0; i < (kTw + T - 1) / T; ++i) {
      const int m = t + i * T;
      if (m < kTw) {
        const int beta = (S + OB - 1) - (31 - __clz((TILE - 1) - m));
        const int seg = TILE - (TILE >> beta);
        const int k = m - seg;
        const double* src = twf + (N >> (beta + 1)) + (row0 << (S - beta - 1)) + k;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(sm_tw + 17 * seg / 16 + row_tw_pad(k));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }

  const long long dstride = (long long)A.dnum * ext * N;
  const u64* Db = A.digits + (long long)b * dstride + (long long)j * N + tofs;
  const int down = j < A.n_q ? j / A.alpha : -1;
  const u64* Cb = A.c1 + (long long)b * A.c1_stride + (long long)j * N + tofs;
  const u64* K0 = A.keys[b / A.per_key] + (long long)kl * N + tofs;  // digit d, poly c at + (d 2 + c) full N

  double acc0[16], acc1[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) acc0[r] = acc1[r] = 0.0;

  u64* pbuf = dyn_smem + TILE + row_inner_tw_words<S, OB>();  // [2][TILE] (kRiPrefetch)
  auto next_digit = [&](int d) {  // first transformed digit >= d, or dnum
    while (d < A.dnum && d == down) ++d;
    return d;
  };
  auto prefetch = [&](int d, int slot) {  // one commit group per call
    if (d < A.dnum) {
      const u64* src = Db + (long long)d * ext * N;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(pbuf + slot * TILE);
#pragma unroll
      for (int i = 0; i < TILE / (2 * T); ++i) {
        const int c = t + i * T;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * c), "l"(src + 2 * c)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int slot = 0;
  if (kRiPrefetch) prefetch(next_digit(0), 0);

  bool tw_ready = false;
#pragma unroll 1
  for (int d = 0; d < MAXD; ++d) {
    if (d >= A.dnum) break;
    const u64* kd0 = K0 + (long long)(2 * d) * full * N;
    const u64* kd1 = kd0 + (long long)full * N;
    if (kRiKeyPf) {  // TILE words = T lines of 16 words: one line per thread and key poly
      prefetch_l1(kd0 + 16 * t);
      prefetch_l1(kd1 + 16 * t);
      if (kRiKeyPf > 1) {
        const int dn = next_digit(d + 1);
        if (dn < A.dnum) prefetch_l1(Db + (long long)dn * ext * N + 16 * t);
      }
    }
    if (kRiPrefetch && d != down) {
      prefetch(next_digit(d + 1), slot ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // twiddles + this digit's tile
      __syncthreads();
      tw_ready = true;
    }
    if (d == down) {  // own limb: already in NTT form (residues)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int e = r * T + t;
        const double y = __longlong_as_double((long long)u64_to_f64bits(__ldcs(Cb + e)));
        const double w0 = __longlong_as_double((long long)u64_to_f64bits(__ldg(kd0 + e)));
        const double w1 = __longlong_as_double((long long)u64_to_f64bits(__ldg(kd1 + e)));
        acc0[r] = __dadd_rn(acc0[r], mulmod_f64h(y, w0, P.qinv_d, P.qd));
        acc1[r] = __dadd_rn(acc1[r], mulmod_f64h(y, w1, P.qinv_d, P.qd));
      }
      continue;
    }
    const u64* base = Db + (long long)d * ext * N;
    u64 x[16];
    constexpr int NG = Sched<S>::G + (Sched<S>::R ? 1 : 0);
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
      const int W = gi < Sched<S>::G ? 4 : Sched<S>::R;
      const int g0 = gi < Sched<S>::G ? S - 4 * (gi + 1) : 0;
      const bool lastg = (gi == NG - 1);
#define HX_RI_GROUP(WW)                                                                     \
  {                                                                                         \
    int eb[16 >> WW], jb[16 >> WW];                                                         \
    group_index<true, S, OB, WW>(t, g0, A.logn, tile, eb, jb);                              \
    if (gi == 0) {                                                                          \
      const u64* pb = pbuf + slot * TILE;                                                   \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                      \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << g0);                         \
        x[r] = kRiPrefetch ? pb[e] : __ldcs(base + e);                                      \
      }                                                                                     \
      if (!tw_ready) {                                                                      \
        asm volatile("cp.async.wait_all;\n" ::: "memory");                                 \
        __syncthreads();                                                                    \
        tw_ready = true;                                                                    \
      }                                                                                     \
    } else {                                                                                \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                      \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << g0);                         \
        x[r] = sm[swz<true>(e)];                                                            \
      }                                                                                     \
    }                                                                                       \
    ntt_group_f64<true, true, S, OB, WW>(x, jb, g0, A.logn, twf, sm_tw, P, false);          \
    __syncthreads();                                                                        \
    _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                        \
      const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << g0);                           \
      sm[swz<true>(e)] = x[r];                                                              \
    }                                                                                       \
    __syncthreads();                                                                        \
    if (lastg) {                                                                            \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                      \
        const int e = r * T + t;                                                            \
        const double y = __longlong_as_double((long long)sm[swz<true>(e)]);                \
        const double w0 = __longlong_as_double((long long)u64_to_f64bits(__ldg(kd0 + e))); \
        const double w1 = __longlong_as_double((long long)u64_to_f64bits(__ldg(kd1 + e))); \
        acc0[r] = __dadd_rn(acc0[r], mulmod_f64h(y, w0, P.qinv_d, P.qd));                 \
        acc1[r] = __dadd_rn(acc1[r], mulmod_f64h(y, w1, P.qinv_d, P.qd));                 \
      }                                                                                     \
    }                                                                                       \
  }
      if (W == 4) HX_RI_GROUP(4)
      else if (W == 3) HX_RI_GROUP(3)
      else if (W == 2) HX_RI_GROUP(2)
      else if (W == 1) HX_RI_GROUP(1)
#undef HX_RI_GROUP
    }
    slot ^= 1;
  }
  if (!tw_ready) asm volatile("cp.async.wait_all;\n" ::: "memory");
  u64* ub = A.u + (long long)b * 2 * ext * N + (long long)j * N + tofs;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int e = r * T + t;
    ub[e] = f64bits_to_residue((u64)__double_as_longlong(acc0[r]), P.qd, P.qinv_d);
    ub[(long long)ext * N + e] = f64bits_to_residue((u64)__double_as_longlong(acc1[r]), P.qd, P.qinv_d);
  }
}

}  // namespace hx
