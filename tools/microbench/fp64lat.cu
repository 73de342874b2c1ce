// FP64 pipe occupancy sweep (B200): DFMA throughput vs resident warps/SM and
// per-thread ILP; and the dependent-chain latency.  Decides how many
// independent butterflies a warp needs to keep the FP64 pipe busy.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_dfma(double* out, double a, double b, int iters) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
void run(int warps_per_sm, int sms, int clk_khz, double* buf) {
  const int iters = 4096;
  const int threads = 32 * warps_per_sm;  // one CTA per SM
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<ILP><<<sms, threads>>>(buf, 1.0000001, 1e-9, iters);
  cudaEventRecord(e0);
  k_dfma<ILP><<<sms, threads>>>(buf, 1.0000001, 1e-9, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)sms * threads * iters * ILP;
  const double lanes = ops / (ms * 1e-3) / sms / (clk_khz * 1e3);
  const double cyc = (ms * 1e-3) * clk_khz * 1e3 / iters;  // cycles per iteration
  printf("warps/SM %3d ILP %2d: %6.1f lanes/clk/SM  (%.1f cycles per dependent step)\n", warps_per_sm, ILP, lanes, cyc);
}

int main() {
  int clk_khz = 0, sms = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, (size_t)sms * 1024 * 8);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w, sms, clk_khz, buf);
    run<2>(w, sms, clk_khz, buf);
    run<4>(w, sms, clk_khz, buf);
    run<8>(w, sms, clk_khz, buf);
  }
  return 0;
}
