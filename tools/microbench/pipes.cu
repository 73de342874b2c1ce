// Pipe-throughput microbenchmark (B200): DFMA (fp64 pipe), IMAD.WIDE.U32
// (fmaheavy), IMAD (32-bit), IADD3 (alu), FFMA; reports lanes/clk/SM using
// the measured SM clock.  Used to choose between integer Shoup and FP64
// modular arithmetic for the 40-bit limbs.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_imad_wide(unsigned long long* out, unsigned a) {
  unsigned long long x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = (unsigned long long)(unsigned)x0 * a + (x0 >> 32);
    x1 = (unsigned long long)(unsigned)x1 * a + (x1 >> 32);
    x2 = (unsigned long long)(unsigned)x2 * a + (x2 >> 32);
    x3 = (unsigned long long)(unsigned)x3 * a + (x3 >> 32);
    x4 = (unsigned long long)(unsigned)x4 * a + (x4 >> 32);
    x5 = (unsigned long long)(unsigned)x5 * a + (x5 >> 32);
    x6 = (unsigned long long)(unsigned)x6 * a + (x6 >> 32);
    x7 = (unsigned long long)(unsigned)x7 * a + (x7 >> 32);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_imad(unsigned* out, unsigned a, unsigned b) {
  unsigned x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
    x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_iadd3(unsigned* out, unsigned a, unsigned b) {
  unsigned x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = x0 + a + b ^ x1; x1 = x1 + a + b ^ x2; x2 = x2 + a + b ^ x3; x3 = x3 + a + b ^ x4;
    x4 = x4 + a + b ^ x5; x5 = x5 + a + b ^ x6; x6 = x6 + a + b ^ x7; x7 = x7 + a + b ^ x0;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// half the warps on the FP64 pipe, half on 32-bit IMAD / IMAD.WIDE: if the
// pipes are independent the mixed kernel takes ~half the single-pipe time.
template <int KIND>
__global__ void k_mix(unsigned long long* out, double a, double b, unsigned ia) {
  if ((threadIdx.x >> 5) & 1) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = __double_as_longlong(x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7);
  } else if (KIND == 0) {
    unsigned x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
      x0 = x0 * ia + 7; x1 = x1 * ia + 7; x2 = x2 * ia + 7; x3 = x3 * ia + 7;
      x4 = x4 * ia + 7; x5 = x5 * ia + 7; x6 = x6 * ia + 7; x7 = x7 * ia + 7;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  } else {
    unsigned long long x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
      x0 = (unsigned long long)(unsigned)x0 * ia + (x0 >> 32);
      x1 = (unsigned long long)(unsigned)x1 * ia + (x1 >> 32);
      x2 = (unsigned long long)(unsigned)x2 * ia + (x2 >> 32);
      x3 = (unsigned long long)(unsigned)x3 * ia + (x3 >> 32);
      x4 = (unsigned long long)(unsigned)x4 * ia + (x4 >> 32);
      x5 = (unsigned long long)(unsigned)x5 * ia + (x5 >> 32);
      x6 = (unsigned long long)(unsigned)x6 * ia + (x6 >> 32);
      x7 = (unsigned long long)(unsigned)x7 * ia + (x7 >> 32);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  }
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  int clk_khz = 0, sms = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  const double ops = (double)blocks * threads * ITERS * 8;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  auto report = [&](const char* name, float ms, double per_op_instr) {
    const double lanes = ops * per_op_instr / (ms * 1e-3) / sms / (clk_khz * 1e3);
    printf("%-28s %8.3f ms  %7.1f lanes/clk/SM (at max clock %d MHz)\n", name, ms, lanes, clk_khz / 1000);
  };
  report("DFMA", timeit([&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0000001, 1e-9); }), 1);
  report("FFMA", timeit([&] { k_ffma<<<blocks, threads>>>((float*)buf, 1.0001f, 1e-3f); }), 1);
  report("IMAD.WIDE.U32 (+shift/add)", timeit([&] { k_imad_wide<<<blocks, threads>>>((unsigned long long*)buf, 2654435761u); }), 1);
  report("IMAD (32-bit)", timeit([&] { k_imad<<<blocks, threads>>>((unsigned*)buf, 2654435761u, 7); }), 1);
  report("IADD3+LOP3", timeit([&] { k_iadd3<<<blocks, threads>>>((unsigned*)buf, 3, 7); }), 1);
  // mixed: each half does the same per-thread work as above, so 'lanes' counts all lanes
  report("MIX DFMA | IMAD", timeit([&] { k_mix<0><<<blocks, threads>>>((unsigned long long*)buf, 1.0000001, 1e-9, 2654435761u); }), 1);
  report("MIX DFMA | IMAD.WIDE", timeit([&] { k_mix<1><<<blocks, threads>>>((unsigned long long*)buf, 1.0000001, 1e-9, 2654435761u); }), 1);
  cudaDeviceSynchronize();
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
