// Compute ceiling of the FP64 radix-16 NTT group (hx_ntt.cuh ntt_group_f64)
// without global memory: every thread keeps its 16 words in registers and runs
// `reps` COL-pass groups back to back (twiddles from a small L1-resident
// table).  Reports butterflies/s and the implied FP64 pipe use (8 FP64 ops per
// butterfly), to separate the group's own instruction ceiling from the
// memory / exchange structure of the pass kernels.
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2512_11135_b200/csrc/cuda/hx_ntt.cuh"

using namespace hx;

template <bool XCH>
__global__ void __launch_bounds__(128) k_groups(u64* out, const PrimeConst* pc, int reps, int logn) {
  const PrimeConst P = pc[0];
  u64 x[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = u64_to_f64bits((threadIdx.x * 16 + r) % 1000003);
  int eb[1], jb[1];
  group_index<false, 8, 3, 4>(threadIdx.x, 4, logn, blockIdx.x & 31, eb, jb);
  __shared__ u64 sm[2048];
  for (int it = 0; it < reps; ++it) {
    ntt_group_f64<true, false, 8, 3, 4>(x, jb, 4, logn, P.twf_fwd, nullptr, P, false);
    if (XCH) {  // the pass kernels' group exchange: sync, 16 STS, sync, 16 LDS (transposed)
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 16; ++r) sm[swz<false>(r * 128 + threadIdx.x)] = x[r];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 16; ++r) x[r] = sm[swz<false>((threadIdx.x & 7) | ((threadIdx.x >> 3) << 7) | (r << 3))];
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {  // keep values bounded (as the pass's normalisation would)
      double v = __longlong_as_double((long long)x[r]);
      v = centre_f64(v, P.qd, P.qinv_d);
      x[r] = (u64)__double_as_longlong(v);
    }
  }
  u64 s = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) s ^= x[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int logn = 16;
  const long long N = 1ll << logn;
  const unsigned long long q = 549756026881ull;  // 40-bit NTT prime (config 1 chain)
  double* twf;
  cudaMalloc(&twf, N * 8);
  double* h = new double[N];
  for (long long i = 0; i < N; ++i) h[i] = (double)((i * 7919 + 13) % q);
  cudaMemcpy(twf, h, N * 8, cudaMemcpyHostToDevice);
  PrimeConst P{};
  P.q = q;
  P.qd = (double)q;
  P.qinv_d = 1.0 / (double)q;
  P.twf_fwd = twf;
  P.f64 = true;
  PrimeConst* dpc;
  cudaMalloc(&dpc, sizeof(P));
  cudaMemcpy(dpc, &P, sizeof(P), cudaMemcpyHostToDevice);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  u64* out;
  cudaMalloc(&out, (size_t)sms * 64 * 128 * 8);
  for (int xch = 0; xch < 2; ++xch)
  for (int ctas : {4, 7, 12}) {
    const int reps = 200, blocks = sms * ctas;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto kk = xch ? k_groups<true> : k_groups<false>;
    kk<<<blocks, 128>>>(out, dpc, reps, logn);
    cudaEventRecord(a);
    kk<<<blocks, 128>>>(out, dpc, reps, logn);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bfly = (double)blocks * 128 * reps * 32;  // 4 stages x 8 butterflies per thread per group
    const double fp64_ops = bfly * 8 + (double)blocks * 128 * reps * 16 * 2;  // + centring
    printf("xch %d CTAs/SM %2d: %.3f ms  %.2f Gbfly/s  FP64 %.1f lanes/clk/SM\n", xch, ctas, ms, bfly / ms / 1e6,
           fp64_ops / (ms * 1e-3) / sms / (clk * 1e3));
    (void)0;
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
