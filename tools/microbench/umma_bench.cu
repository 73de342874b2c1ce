// tcgen05.mma throughput microbenchmark (B200, one CTA per SM): cycles per
// u8 x u8 -> s32 MMA (kind::i8, M = 128, K = 32) for several N, K-major
// SWIZZLE_NONE operands (the tensor-core BSGS MAC's layout), vs kind::f16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench umma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned u32;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 desc(u32 a, u32 lbo, u32 sbo, u32 layout) {
  return (u64)((a >> 4) & 0x3FFF) | ((u64)((lbo >> 4) & 0x3FFF) << 16) | ((u64)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | ((u64)layout << 61);
}
template <int KIND>
__device__ __forceinline__ void mma(u32 d, u64 a, u64 b, u32 id, u32 acc) {
  if (KIND == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

template <int KIND>
__global__ void bench(int N, int reps, int kbytes, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ u64 bar;
  __shared__ u32 tslot;
  unsigned char* sA = sm;              // 128 rows x kbytes
  unsigned char* sB = sm + 128 * kbytes;  // N rows x kbytes
  for (int i = threadIdx.x; i < (128 + N) * kbytes / 4; i += blockDim.x) ((u32*)sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const u32 tmem = tslot;
  if (threadIdx.x == 0) {
    const int KB = kbytes / 16 * 128;  // bytes per 8-row group
    u32 id;
    int ksteps;
    if (KIND == 0) {
      id = (2u << 4) | ((u32)(N >> 3) << 17) | ((u32)(128 >> 4) << 24);
      ksteps = kbytes / 32;
    } else {
      id = (1u << 4) | (1u << 7) | (1u << 10) | ((u32)(N >> 3) << 17) | ((u32)(128 >> 4) << 24);  // bf16 -> f32
      ksteps = kbytes / 32;  // K = 16 elements = 32 bytes per MMA
    }
    const u32 a0 = smem_u32(sA), b0 = smem_u32(sB);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < ksteps; ++k)
        mma<KIND>(tmem + (r & 1) * 256, desc(a0 + k * 256, 128, KB, 0), desc(b0 + k * 256, 128, KB, 0), id, k > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
        smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int reps = 200;
  for (int kind = 0; kind < 2; ++kind)
    for (int N : {16, 32, 64, 80, 128, 160, 256}) {
      for (int kbytes : {160, 320}) {
        const int smem = (128 + N) * kbytes;
        if (kind == 0) {
          cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          bench<0><<<148, 128, smem>>>(N, reps, kbytes, d);
        } else {
          cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          bench<1><<<148, 128, smem>>>(N, reps, kbytes, d);
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        const double mmas = (double)reps * (kbytes / 32);
        const double cyc = h[0] / mmas;
        const double macs = 128.0 * N * (kind == 0 ? 32 : 16) / cyc;
        printf("%s N=%3d K'=%3d B: %7.1f cycles/MMA  %7.0f MAC/clk/SM\n", kind == 0 ? "i8 " : "f16", N, kbytes, cyc, macs);
      }
    }
  return 0;
}
