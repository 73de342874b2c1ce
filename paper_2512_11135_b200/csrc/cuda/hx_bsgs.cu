// hx_bsgs.cu -- fused BSGS diagonal multiply-accumulate.
//
// For every limb i and coefficient t the BSGS inner sums are a small
// matrix-vector product: inner_j[c][i][t] = sum_k diag_{j n1 + k}[i][t] *
// baby_k[c][i][t], j < n2, k < n1, c in {0, 1}.  A CTA owns TT coefficients
// of one limb: the 2 n1 baby words per coefficient are staged in shared memory
// once, then the kernel streams every diagonal word from HBM exactly once
// (evict-first loads), accumulates lazily in 128 bits (products < 2^120, so
// up to 256 terms cannot overflow) and reduces once per output word.  HBM
// traffic per launch = diagonals + baby tile + outputs = the algorithmic
// minimum.
#include "hx_internal.h"

namespace hx {

template <int TT>
__global__ void __launch_bounds__(TT) bsgs_mac_kernel(MacArgs A) {
  extern __shared__ u64 smb[];  // [n1][2][TT]
  const long long N = 1ll << A.logn;
  const int i = A.limbs ? A.limbs[blockIdx.y] : blockIdx.y;
  const int tid = threadIdx.x;
  const int tok = blockIdx.x % A.tokens;
  const long long t = (long long)(blockIdx.x / A.tokens) * TT + tid;
  const u64* baby = A.baby + tok * A.baby_tstride;
  u64* inner = A.inner + tok * A.inner_tstride;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  for (int k = 0; k < A.n1; ++k) {
    smb[(2 * k) * TT + tid] = baby[(2ll * k) * L + i * N + t];
    smb[(2 * k + 1) * TT + tid] = baby[(2ll * k + 1) * L + i * N + t];
  }
  __syncthreads();
  const u64* dg = A.diags + i * N + t;
  for (int j = 0; j < A.n2; ++j) {
    U128 z0{0, 0}, z1{0, 0};
    const u64* dj = dg + (long long)j * A.diag_jstride * A.diag_stride;
    int k = 0;
    // 16 independent diagonal loads in flight per thread (the CTA count per SM
    // is bounded by the baby tile in shared memory, so memory-level
    // parallelism has to come from each thread)
    for (; k + 16 <= A.n1; k += 16) {
      u64 d[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) d[u] = __ldcs(dj + (long long)(k + u) * A.diag_stride);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        mac128(z0, d[u], smb[(2 * (k + u)) * TT + tid]);
        mac128(z1, d[u], smb[(2 * (k + u) + 1) * TT + tid]);
      }
    }
    for (; k + 8 <= A.n1; k += 8) {
      u64 d[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = __ldcs(dj + (long long)(k + u) * A.diag_stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        mac128(z0, d[u], smb[(2 * (k + u)) * TT + tid]);
        mac128(z1, d[u], smb[(2 * (k + u) + 1) * TT + tid]);
      }
    }
    for (; k < A.n1; ++k) {
      const u64 d = __ldcs(dj + (long long)k * A.diag_stride);
      mac128(z0, d, smb[(2 * k) * TT + tid]);
      mac128(z1, d, smb[(2 * k + 1) * TT + tid]);
    }
    u64* o = inner + (long long)j * A.out_jstride + i * N + t;
    o[0] = reduce128(z0, P);
    o[L] = reduce128(z1, P);
  }
}

// ---------------------------------------------------------------------------
// FP64 k-split MAC for limbs with q < 2^43 (B200's full-rate FP64 pipe).
//
// Operands are canonical residues x, y < q; split at 20 bits,
// x = x1 2^20 + x0 (x1 < q / 2^20, x0 < 2^20), and
//   sum_k x_k y_k = S11 2^40 + S10 2^20 + S00,
//   S11 = sum x1 y1 < n1 q^2 / 2^40,  S10 = sum (x1 y0 + x0 y1) < 2 n1 q,
//   S00 = sum x0 y0 < n1 2^40,
// all integers below 2^52 for q < 2^43 and n1 <= 64, so every FMA and the
// cross-warp sums are exact in doubles.  A CTA is
// 8 warps x 32 coefficients of one limb: warp w owns baby steps
// k in [w KPT, (w+1) KPT) in registers (split into doubles once), streams its
// diagonal words (evict-first, next giant step prefetched), and the 8 warps'
// partial sums are combined through shared memory (double-buffered, one
// barrier per giant step); the combine is one exact modular reduction per
// output word.  Bit-identical to the integer kernel.
constexpr int kMacWarps = 8;

__device__ __forceinline__ void split20(u64 v, double& hi, double& lo) {
  hi = __dsub_rn(__longlong_as_double((long long)((v >> 20) | 0x4330000000000000ull)), kTwo52);
  lo = __dsub_rn(__longlong_as_double((long long)((v & 0xFFFFFull) | 0x4330000000000000ull)), kTwo52);
}

// NW warps per CTA; for KPT <= 4 at most 64 registers so that 32 warps / SM
// are resident (HBM latency x bandwidth needs that many 256-B diagonal rows
// in flight: n1 = n2 = 32 MAC 0.69 -> 0.75 of the HBM peak).  KPT = 8
// (n1 = 64) keeps 126 registers at 2 CTAs / SM: 16 warps of 4 baby steps
// each measured 2 ms slower per W2 matvec.
template <int KPT, int NW = kMacWarps>
__global__ void __launch_bounds__(32 * NW, (KPT <= 4 ? 32 / NW : 2)) bsgs_mac_f64_kernel(MacArgs A, const int* limbs) {
  constexpr int kMacWarps = NW;
  __shared__ double part[2][kMacWarps][2][3][32];  // [buf][warp][poly][S11,S10,S00][lane]
  const long long N = 1ll << A.logn;
  const int i = limbs[blockIdx.y];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tok = blockIdx.x % A.tokens;
  const long long t = (long long)(blockIdx.x / A.tokens) * 32 + lane;
  const u64* baby = A.baby + tok * A.baby_tstride;
  u64* inner = A.inner + tok * A.inner_tstride;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  // baby words of this warp's k slice, split into 20-bit halves
  double bh[KPT][2], bl[KPT][2];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) {
    const int k = w * KPT + kk;
#pragma unroll
    for (int c = 0; c < 2; ++c) split20(baby[(2ll * k + c) * L + i * N + t], bh[kk][c], bl[kk][c]);
  }
  const u64* dg = A.diags + i * N + t + (long long)(w * KPT) * A.diag_stride;
  u64 dn[KPT];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) dn[kk] = __ldcs(dg + (long long)kk * A.diag_stride);
  for (int j = 0; j < A.n2; ++j) {
    u64 d[KPT];
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) d[kk] = dn[kk];
    if (j + 1 < A.n2) {
      const u64* dj = dg + (long long)(j + 1) * A.diag_jstride * A.diag_stride;
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) dn[kk] = __ldcs(dj + (long long)kk * A.diag_stride);
    }
    double s[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) {
      double xh, xl;
      split20(d[kk], xh, xl);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        s[c][0] = __fma_rn(xh, bh[kk][c], s[c][0]);
        s[c][1] = __fma_rn(xh, bl[kk][c], s[c][1]);
        s[c][1] = __fma_rn(xl, bh[kk][c], s[c][1]);
        s[c][2] = __fma_rn(xl, bl[kk][c], s[c][2]);
      }
    }
    const int buf = j & 1;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int m = 0; m < 3; ++m) part[buf][w][c][m][lane] = s[c][m];
    __syncthreads();
    if (threadIdx.x < 64) {  // warps 0-1: (poly c, lane) reductions
      const int c = threadIdx.x >> 5;
      double S[3] = {0, 0, 0};
#pragma unroll
      for (int ww = 0; ww < kMacWarps; ++ww)
#pragma unroll
        for (int m = 0; m < 3; ++m) S[m] = __dadd_rn(S[m], part[buf][ww][c][m][lane]);
      // S11 2^40 + S10 2^20 + S00 mod q (each S exact, < 2^52)
      const double v = __dadd_rn(__dadd_rn(mulmod_f64(S[0], P.r40_d, P.r40_q, P.qd),
                                           mulmod_f64(S[1], P.r20_d, P.r20_q, P.qd)),
                                 centre_f64(S[2], P.qd, P.qinv_d));
      inner[(long long)j * A.out_jstride + c * L + i * N + t] =
          f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);
    }
  }
}

// Integer twin of the k-split kernel for the wide primes (q >= 2^43, e.g. the
// 60-bit q_0): same CTA shape and double-buffered cross-warp combine, 128-bit
// lazy accumulators (products < 2^120, n1 <= 64 terms), one reduction per output.
template <int KPT>
__global__ void __launch_bounds__(32 * kMacWarps) bsgs_mac_int_kernel(MacArgs A, const int* limbs) {
  __shared__ u64 part[2][kMacWarps][2][2][32];  // [buf][warp][poly][lo,hi][lane]
  const long long N = 1ll << A.logn;
  const int i = limbs[blockIdx.y];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tok = blockIdx.x % A.tokens;
  const long long t = (long long)(blockIdx.x / A.tokens) * 32 + lane;
  const u64* baby = A.baby + tok * A.baby_tstride;
  u64* inner = A.inner + tok * A.inner_tstride;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  u64 b[KPT][2];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) {
    const int k = w * KPT + kk;
#pragma unroll
    for (int c = 0; c < 2; ++c) b[kk][c] = baby[(2ll * k + c) * L + i * N + t];
  }
  const u64* dg = A.diags + i * N + t + (long long)(w * KPT) * A.diag_stride;
  u64 dn[KPT];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) dn[kk] = __ldcs(dg + (long long)kk * A.diag_stride);
  for (int j = 0; j < A.n2; ++j) {
    u64 d[KPT];
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) d[kk] = dn[kk];
    if (j + 1 < A.n2) {
      const u64* dj = dg + (long long)(j + 1) * A.diag_jstride * A.diag_stride;
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) dn[kk] = __ldcs(dj + (long long)kk * A.diag_stride);
    }
    U128 z[2] = {{0, 0}, {0, 0}};
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk)
#pragma unroll
      for (int c = 0; c < 2; ++c) mac128(z[c], d[kk], b[kk][c]);
    const int buf = j & 1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      part[buf][w][c][0][lane] = z[c].lo;
      part[buf][w][c][1][lane] = z[c].hi;
    }
    __syncthreads();
    if (threadIdx.x < 64) {
      const int c = threadIdx.x >> 5;
      U128 S{0, 0};
#pragma unroll
      for (int ww = 0; ww < kMacWarps; ++ww) {
        asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;"
            : "+l"(S.lo), "+l"(S.hi)
            : "l"(part[buf][ww][c][0][lane]), "l"(part[buf][ww][c][1][lane]));
      }
      inner[(long long)j * A.out_jstride + c * L + i * N + t] = reduce128(S, P);
    }
  }
}

// Sparse index-list MAC (pruned matrices): a CTA owns TT coefficients of one
// limb for one token; the baby tile [n1][2][TT] is staged in shared memory
// once, then the live (j, k) entries of the block are streamed group by
// group straight from their plaintexts (no gather copies of diagonals or
// baby steps), each diagonal word read once per token tile, 128-bit lazy
// accumulation, one reduction per live output word.
template <int TT>
__global__ void __launch_bounds__(TT) bsgs_mac_sparse_kernel(SparseMacArgs A) {
  extern __shared__ u64 smb[];  // [n1][2][TT]
  const long long N = 1ll << A.logn;
  const int i = blockIdx.y;
  const int tid = threadIdx.x;
  const int tok = blockIdx.x % A.tokens;
  const long long t = (long long)(blockIdx.x / A.tokens) * TT + tid;
  const u64* baby = A.baby + tok * A.baby_tstride;
  u64* inner = A.inner + tok * A.inner_tstride;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  for (int k = 0; k < A.n1; ++k) {
    smb[(2 * k) * TT + tid] = __ldg(baby + (2ll * k) * L + i * N + t);
    smb[(2 * k + 1) * TT + tid] = __ldg(baby + (2ll * k + 1) * L + i * N + t);
  }
  __syncthreads();
  const long long off = i * N + t;
  for (int j = 0; j < A.n2; ++j) {
    const int e0 = A.gptr[j], e1 = A.gptr[j + 1];
    if (e0 == e1) continue;
    U128 z0{0, 0}, z1{0, 0};
    int e = e0;
    for (; e + 4 <= e1; e += 4) {
      u64 d[4];
      int k[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        d[u] = __ldcs(A.dptr[e + u] + off);
        k[u] = A.ks[e + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mac128(z0, d[u], smb[(2 * k[u]) * TT + tid]);
        mac128(z1, d[u], smb[(2 * k[u] + 1) * TT + tid]);
      }
    }
    for (; e < e1; ++e) {
      const u64 d = __ldcs(A.dptr[e] + off);
      const int k = A.ks[e];
      mac128(z0, d, smb[(2 * k) * TT + tid]);
      mac128(z1, d, smb[(2 * k + 1) * TT + tid]);
    }
    u64* o = inner + (long long)j * A.out_jstride + off;
    o[0] = reduce128(z0, P);
    o[L] = reduce128(z1, P);
  }
}

void launch_bsgs_mac_sparse(const SparseMacArgs& A, long long N, cudaStream_t s) {
  constexpr int TT = 64;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(bsgs_mac_sparse_kernel<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         128 * 2 * TT * (int)sizeof(u64));
    configured = true;
  }
  const size_t smem = (size_t)A.n1 * 2 * TT * sizeof(u64);
  dim3 grid((unsigned)(N / TT * A.tokens), (unsigned)A.n_q);
  bsgs_mac_sparse_kernel<TT><<<grid, TT, smem, s>>>(A);
}

namespace {
template <class K>
void set_max_smem(K kernel, int bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
}  // namespace

void launch_bsgs_mac(const MacArgs& A, long long N, cudaStream_t s, const int* d_f64_limbs, int n_f64,
                     const int* d_int_limbs, int n_int) {
  constexpr int TT = 128;
  static bool configured = false;
  if (!configured) {
    set_max_smem(bsgs_mac_kernel<TT>, 64 * 2 * TT * (int)sizeof(u64));
    configured = true;
  }
  const int kpt = A.n1 / kMacWarps;
  const bool ksplit = N >= 32 && A.n1 % kMacWarps == 0 && (kpt == 1 || kpt == 2 || kpt == 4 || kpt == 8);
  if (ksplit && n_f64 > 0) {
    dim3 grid((unsigned)(N / 32 * A.tokens), (unsigned)n_f64);
    switch (kpt) {
      case 1: bsgs_mac_f64_kernel<1><<<grid, 32 * kMacWarps, 0, s>>>(A, d_f64_limbs); break;
      case 2: bsgs_mac_f64_kernel<2><<<grid, 32 * kMacWarps, 0, s>>>(A, d_f64_limbs); break;
      case 4: bsgs_mac_f64_kernel<4><<<grid, 32 * kMacWarps, 0, s>>>(A, d_f64_limbs); break;
      case 8: bsgs_mac_f64_kernel<8><<<grid, 32 * kMacWarps, 0, s>>>(A, d_f64_limbs); break;
    }
  }
  // integer k-split kernel for the wide primes
  if (ksplit && n_int > 0) {
    dim3 grid((unsigned)(N / 32 * A.tokens), (unsigned)n_int);
    switch (kpt) {
      case 1: bsgs_mac_int_kernel<1><<<grid, 32 * kMacWarps, 0, s>>>(A, d_int_limbs); break;
      case 2: bsgs_mac_int_kernel<2><<<grid, 32 * kMacWarps, 0, s>>>(A, d_int_limbs); break;
      case 4: bsgs_mac_int_kernel<4><<<grid, 32 * kMacWarps, 0, s>>>(A, d_int_limbs); break;
      case 8: bsgs_mac_int_kernel<8><<<grid, 32 * kMacWarps, 0, s>>>(A, d_int_limbs); break;
    }
  }
  if (ksplit) return;
  // generic smem-tile kernel (n1 not a multiple of 8, tiny N): all limbs
  const int* il = nullptr;
  const int ni = A.n_q;
  if (ni > 0) {
    const size_t smem = (size_t)A.n1 * 2 * TT * sizeof(u64);
    MacArgs B = A;
    B.limbs = il;
    dim3 grid((unsigned)(N / TT * A.tokens), (unsigned)ni);
    bsgs_mac_kernel<TT><<<grid, TT, smem, s>>>(B);
  }
}

// out[p][i][t] = sum_r in[r][p][i][t] mod q_i
__global__ void sum_kernel(SumArgs A) {
  const long long N = 1ll << A.logn;
  const int p = blockIdx.z, i = blockIdx.y;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = A.pc[i].q;
  const u64* src = A.in + p * A.in_poly_stride + i * N + t;
  u64 acc = 0;
  int r = 0;
  for (; r + 8 <= A.terms; r += 8) {  // 8 loads in flight per thread
    u64 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(src + (r + k) * A.term_stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = addmod(acc, v[k], q);
  }
  for (; r < A.terms; ++r) acc = addmod(acc, __ldcs(src + r * A.term_stride), q);
  A.out[p * A.out_poly_stride + i * N + t] = acc;
}

void launch_sum(const SumArgs& A, int polys, long long N, cudaStream_t s) {
  const int th = (int)(N < 256 ? N : 256);
  sum_kernel<<<dim3((unsigned)(N / th), (unsigned)A.n_q, (unsigned)polys), th, 0, s>>>(A);
}

}  // namespace hx
