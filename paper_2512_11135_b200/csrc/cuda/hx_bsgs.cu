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
  const int i = blockIdx.y;
  const int tid = threadIdx.x;
  const long long t = (long long)blockIdx.x * TT + tid;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  for (int k = 0; k < A.n1; ++k) {
    smb[(2 * k) * TT + tid] = A.baby[(2ll * k) * L + i * N + t];
    smb[(2 * k + 1) * TT + tid] = A.baby[(2ll * k + 1) * L + i * N + t];
  }
  __syncthreads();
  const u64* dg = A.diags + i * N + t;
  for (int j = 0; j < A.n2; ++j) {
    U128 z0{0, 0}, z1{0, 0};
    const u64* dj = dg + (long long)j * A.n1 * A.diag_stride;
    int k = 0;
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
    u64* o = A.inner + (long long)j * A.out_jstride + i * N + t;
    o[0] = reduce128(z0, P);
    o[L] = reduce128(z1, P);
  }
}

void launch_bsgs_mac(const MacArgs& A, long long N, cudaStream_t s) {
  constexpr int TT = 128;
  const int tt = (int)(N < TT ? N : TT);
  const size_t smem = (size_t)A.n1 * 2 * TT * sizeof(u64);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(bsgs_mac_kernel<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         64 * 2 * TT * (int)sizeof(u64));
    configured = true;
  }
  (void)tt;
  dim3 grid((unsigned)(N / TT), (unsigned)A.n_q);
  bsgs_mac_kernel<TT><<<grid, TT, smem, s>>>(A);
}

// out[p][i][t] = sum_r in[r][p][i][t] mod q_i
__global__ void sum_kernel(SumArgs A) {
  const long long N = 1ll << A.logn;
  const int p = blockIdx.z, i = blockIdx.y;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = A.pc[i].q;
  const u64* src = A.in + p * A.in_poly_stride + i * N + t;
  u64 acc = 0;
  for (int r = 0; r < A.terms; ++r) acc = addmod(acc, __ldcs(src + r * A.term_stride), q);
  A.out[p * A.out_poly_stride + i * N + t] = acc;
}

void launch_sum(const SumArgs& A, int polys, long long N, cudaStream_t s) {
  const int th = (int)(N < 256 ? N : 256);
  sum_kernel<<<dim3((unsigned)(N / th), (unsigned)A.n_q, (unsigned)polys), th, 0, s>>>(A);
}

}  // namespace hx
