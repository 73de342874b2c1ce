// hx_bsgs_p40.cu -- BSGS diagonal multiply-accumulate over 5-byte packed
// diagonals, streamed into shared memory by the bulk-copy engine.
//
// The single-token MAC of matvec_bsgs (the mul_acc loop over
// rns_poly.cpp:102-110) is HBM-bound: every diagonal word is read once and
// used for two products.  A diagonal word of a limb with q < 2^40 needs 5
// bytes, not 8, so the matrix is packed once ("P40 layout") and the MAC
// streams 37.5 % fewer bytes.  The arithmetic is the FP64 k-split MAC of
// hx_bsgs.cu (20-bit halves, exact FMAs, one reduction per output): the
// output words are identical to bsgs_mac_f64_kernel's.
//
// P40 layout of one block (n2 giant rows j, n1 baby steps k, diagonal
// (j, k) = j dj + k of a contiguous [n_diag][diag_limbs][N] buffer), for each
// P40 limb p (q < 2^40, in limb order) and tile of 32 coefficients:
//   stage (p, tile, j) = lo32[k / 2][32][2] (u32, bits 0-31 of the word)
//                        | hi8[k / 4][32][4] (u8, bits 32-39),   5 n1 32 bytes,
// (one 8-byte and half a 4-byte shared load per lane for 2 words, both
// conflict-free),
// stages of one (p, tile) back to back, tiles of one limb back to back.  A
// CTA owns one (p, tile): thread 0 keeps S stages in flight with
// cp.async.bulk (one copy per stage, mbarrier with expect-tx), the 8 warps
// (warp w: baby steps [w KPT, (w+1) KPT), lane = coefficient) read their
// words from shared memory, and the per-stage barrier of the cross-warp
// combine also releases the stage slot for the next copy.  Bytes in flight
// come from shared memory, not registers, so the kernel keeps the 64-register
// budget of 32 resident warps.
#include <cstdlib>

#include "hx_internal.h"

namespace hx {

namespace {

__device__ __forceinline__ u32 p40_smem(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void p40_bar_init(u64* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(p40_smem(bar)));
}
__device__ __forceinline__ void p40_expect(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(p40_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void p40_wait(u64* bar, u32 parity) {
  u32 ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(p40_smem(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void p40_copy(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   p40_smem(dst)),
               "l"(src), "r"(bytes), "r"(p40_smem(bar))
               : "memory");
}

__device__ __forceinline__ double p40_dbl(u32 v) {  // exact (double) of a < 2^32 integer
  return __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ull | v)), kTwo52);
}

constexpr int kP40Warps = 8;
constexpr int kP40TT = 32;  // coefficients per CTA (one per lane)

}  // namespace

template <int KPT>
__global__ void __launch_bounds__(32 * kP40Warps, (KPT <= 4 ? 4 : 2)) bsgs_mac_p40_kernel(P40Args A) {
  __shared__ double part[2][kP40Warps][2][3][32];  // [buf][warp][poly][S11,S10,S00][lane]
  __shared__ u64 full[kP40MaxStages];
  extern __shared__ __align__(128) unsigned char stages[];
  const long long N = 1ll << A.logn;
  const int tile = blockIdx.x, p = blockIdx.y;
  const int i = A.limbs[p];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const long long t = (long long)tile * kP40TT + lane;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  const u32 SB = 5u * A.n1 * kP40TT;  // bytes of one stage
  const int S = A.stages, n2 = A.n2;
  const unsigned char* src = A.packed + (((size_t)p * (size_t)(N / kP40TT) + tile) * n2) * SB;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) p40_bar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < S && s < n2; ++s) {
      p40_expect(&full[s], SB);
      p40_copy(stages + (size_t)s * SB, src + (size_t)s * SB, SB, &full[s]);
    }
  }
  // baby words of this warp's k slice, split into 20-bit halves (hx_bsgs.cu)
  double bh[KPT][2], bl[KPT][2];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) {
    const int k = w * KPT + kk;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const u64 v = A.baby[(2ll * k + c) * L + i * N + t];
      bh[kk][c] = p40_dbl((u32)(v >> 20));
      bl[kk][c] = p40_dbl((u32)(v & 0xFFFFFull));
    }
  }
  int jj = 0;           // row j = (block jb, giant step jj), tracked without a division
  long long boff = 0;   // jb out_bstride
  for (int j = 0; j < n2; ++j) {
    const int slot = j % S;
    p40_wait(&full[slot], (u32)((j / S) & 1));
    const unsigned char* st = stages + (size_t)slot * SB;
    const uint2* lo = reinterpret_cast<const uint2*>(st);
    const u32* hi = reinterpret_cast<const u32*>(st + 4 * A.n1 * kP40TT);
    u32 lw[KPT], hw[KPT / 4];
#pragma unroll
    for (int q = 0; q < KPT / 2; ++q) {
      const uint2 v = lo[(w * KPT / 2 + q) * kP40TT + lane];
      lw[2 * q] = v.x;
      lw[2 * q + 1] = v.y;
    }
#pragma unroll
    for (int q = 0; q < KPT / 4; ++q) hw[q] = hi[(w * KPT / 4 + q) * kP40TT + lane];
    double s[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) {
      const u32 l = lw[kk], h = (hw[kk >> 2] >> (8 * (kk & 3))) & 0xFFu;
      const double xh = p40_dbl((l >> 20) | (h << 12)), xl = p40_dbl(l & 0xFFFFFu);
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
    __syncthreads();  // every warp is done with stage j: its slot takes stage j + S
    if (tid == 0 && j + S < n2) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      p40_expect(&full[slot], SB);
      p40_copy(stages + (size_t)slot * SB, src + (size_t)(j + S) * SB, SB, &full[slot]);
    }
    if (tid < 64) {  // warps 0-1: (poly c, lane) reductions
      const int c = tid >> 5;
      double Sm[3] = {0, 0, 0};
#pragma unroll
      for (int ww = 0; ww < kP40Warps; ++ww)
#pragma unroll
        for (int m = 0; m < 3; ++m) Sm[m] = __dadd_rn(Sm[m], part[buf][ww][c][m][lane]);
      const double v = __dadd_rn(__dadd_rn(mulmod_f64(Sm[0], P.r40_d, P.r40_q, P.qd),
                                           mulmod_f64(Sm[1], P.r20_d, P.r20_q, P.qd)),
                                 centre_f64(Sm[2], P.qd, P.qinv_d));
      A.inner[(long long)jj * A.out_jstride + boff + c * L + i * N + t] =
          f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);
    }
    if (++jj == A.rpb) {
      jj = 0;
      boff += A.out_bstride;
    }
  }
}

// RPS giant rows per step.  The per-row cross-warp combine of the kernel above
// is its critical path (ncu: "barrier" is the top stall -- warps 0-1 reduce
// every row on top of their own products while the other six wait at the next
// row's barrier).  With RPS rows per barrier 2 RPS warps reduce one (row,
// poly) each, so the combine costs every reducing warp one reduction per RPS
// rows of products.  A stage is RPS consecutive rows (they are contiguous in
// the P40 layout: one bulk copy), the partial sums live in dynamic shared
// memory behind the stage ring.  Rows of one step never straddle row blocks
// (host: rows per block % RPS == 0).  NW warps split the n1 baby steps (KPT
// each): n1 = 64 runs 8 warps x 8, n1 = 32 runs 4 warps x 8 so that with two
// rows per step every warp reduces one (row, poly) -- the combine is then
// balanced over the CTA.  Same words as the kernel above.
template <int KPT, int RPS, int NW>
__global__ void __launch_bounds__(32 * NW, (NW <= 4 ? 4 : 2)) bsgs_mac_p40x_kernel(P40Args A) {
  __shared__ u64 full[kP40MaxStages];
  extern __shared__ __align__(128) unsigned char stages[];
  const long long N = 1ll << A.logn;
  const int tile = blockIdx.x, p = blockIdx.y;
  const int i = A.limbs[p];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const long long t = (long long)tile * kP40TT + lane;
  const PrimeConst& P = A.pc[i];
  const long long L = (long long)A.n_q * N;
  const u32 SB = 5u * A.n1 * kP40TT;  // bytes of one row
  const u32 SS = RPS * SB;            // bytes of one stage
  const int S = A.stages, steps = A.n2 / RPS;
  // [buf][warp][row][poly][S11,S10,S00][lane]
  double(*part)[NW][RPS][2][3][32] =
      reinterpret_cast<double(*)[NW][RPS][2][3][32]>(stages + (size_t)S * SS);
  const unsigned char* src = A.packed + (((size_t)p * (size_t)(N / kP40TT) + tile) * A.n2) * SB;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) p40_bar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < S && s < steps; ++s) {
      p40_expect(&full[s], SS);
      p40_copy(stages + (size_t)s * SS, src + (size_t)s * SS, SS, &full[s]);
    }
  }
  double bh[KPT][2], bl[KPT][2];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) {
    const int k = w * KPT + kk;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const u64 v = A.baby[(2ll * k + c) * L + i * N + t];
      bh[kk][c] = p40_dbl((u32)(v >> 20));
      bl[kk][c] = p40_dbl((u32)(v & 0xFFFFFull));
    }
  }
  int jj = 0;          // giant step of the step's first row inside its row block
  long long boff = 0;  // that block's output offset
  for (int js = 0; js < steps; ++js) {
    const int slot = js % S;
    p40_wait(&full[slot], (u32)((js / S) & 1));
    const int buf = js & 1;
#pragma unroll
    for (int rr = 0; rr < RPS; ++rr) {
      const unsigned char* st = stages + (size_t)slot * SS + (size_t)rr * SB;
      const uint2* lo = reinterpret_cast<const uint2*>(st);
      const u32* hi = reinterpret_cast<const u32*>(st + 4 * A.n1 * kP40TT);
      u32 lw[KPT], hw[KPT / 4];
#pragma unroll
      for (int q = 0; q < KPT / 2; ++q) {
        const uint2 v = lo[(w * KPT / 2 + q) * kP40TT + lane];
        lw[2 * q] = v.x;
        lw[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int q = 0; q < KPT / 4; ++q) hw[q] = hi[(w * KPT / 4 + q) * kP40TT + lane];
      double s[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) {
        const u32 l = lw[kk], h = (hw[kk >> 2] >> (8 * (kk & 3))) & 0xFFu;
        const double xh = p40_dbl((l >> 20) | (h << 12)), xl = p40_dbl(l & 0xFFFFFu);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          s[c][0] = __fma_rn(xh, bh[kk][c], s[c][0]);
          s[c][1] = __fma_rn(xh, bl[kk][c], s[c][1]);
          s[c][1] = __fma_rn(xl, bh[kk][c], s[c][1]);
          s[c][2] = __fma_rn(xl, bl[kk][c], s[c][2]);
        }
      }
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int m = 0; m < 3; ++m) part[buf][w][rr][c][m][lane] = s[c][m];
    }
    __syncthreads();  // every warp is done with stage js: its slot takes stage js + S
    if (tid == 0 && js + S < steps) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      p40_expect(&full[slot], SS);
      p40_copy(stages + (size_t)slot * SS, src + (size_t)(js + S) * SS, SS, &full[slot]);
    }
    static_assert(2 * RPS <= NW, "one reducing warp per (row, poly)");
    if (tid < 64 * RPS) {  // warps 0 .. 2 RPS - 1: one (row, poly) each
      const int rr = tid >> 6, c = (tid >> 5) & 1;
      double Sm[3] = {0, 0, 0};
#pragma unroll
      for (int ww = 0; ww < NW; ++ww)
#pragma unroll
        for (int m = 0; m < 3; ++m) Sm[m] = __dadd_rn(Sm[m], part[buf][ww][rr][c][m][lane]);
      const double v = __dadd_rn(__dadd_rn(mulmod_f64(Sm[0], P.r40_d, P.r40_q, P.qd),
                                           mulmod_f64(Sm[1], P.r20_d, P.r20_q, P.qd)),
                                 centre_f64(Sm[2], P.qd, P.qinv_d));
      A.inner[(long long)(jj + rr) * A.out_jstride + boff + c * L + i * N + t] =
          f64bits_to_residue((u64)__double_as_longlong(v), P.qd, P.qinv_d);
    }
    jj += RPS;
    if (jj == A.rpb) {
      jj = 0;
      boff += A.out_bstride;
    }
  }
}

// P40 packing: thread (lane = coefficient, k slice) of block (tile, j, p)
__global__ void p40_pack_kernel(unsigned char* dst, const u64* diags, long long diag_stride, const int* limbs,
                                int n1, int n2, int dj, int logn) {
  const long long N = 1ll << logn;
  const int tile = blockIdx.x, j = blockIdx.y, p = blockIdx.z;
  const int i = limbs[p];
  const int lane = threadIdx.x & 31;
  const long long t = (long long)tile * kP40TT + lane;
  const size_t SB = (size_t)5 * n1 * kP40TT;
  unsigned char* st = dst + (((size_t)p * (size_t)(N / kP40TT) + tile) * n2 + j) * SB;
  u32* lo = reinterpret_cast<u32*>(st);
  unsigned char* hi = st + 4 * n1 * kP40TT;
  for (int k = threadIdx.x >> 5; k < n1; k += blockDim.x >> 5) {
    const u64 v = __ldg(diags + (long long)(j * dj + k) * diag_stride + i * N + t);
    lo[((k >> 1) * kP40TT + lane) * 2 + (k & 1)] = (u32)v;
    hi[((k >> 2) * kP40TT + lane) * 4 + (k & 3)] = (unsigned char)(v >> 32);
  }
}

void launch_p40_pack(unsigned char* dst, const u64* diags, long long diag_stride, const int* limbs, int n_p40,
                     int n1, int n2, int dj, int logn, cudaStream_t s) {
  const long long N = 1ll << logn;
  dim3 grid((unsigned)(N / kP40TT), (unsigned)n2, (unsigned)n_p40);
  p40_pack_kernel<<<grid, 256, 0, s>>>(dst, diags, diag_stride, limbs, n1, n2, dj, logn);
}

int p40_stages(int n1) { return n1 <= 32 ? 6 : 8; }

void launch_bsgs_mac_p40(const P40Args& A0, int n_p40, cudaStream_t s) {
  P40Args A = A0;
  const long long N = 1ll << A.logn;
  const int kpt = A.n1 / kP40Warps;
  dim3 grid((unsigned)(N / kP40TT), (unsigned)n_p40);
  // two giant rows per step (bsgs_mac_p40x_kernel) whenever the rows per block
  // are even: 9.24 -> 7.72 ms at n1 = n2 = 64, 2.78 -> 2.61 ms at 32 (measured);
  // HX_P40_RPS=1 / HX_P40_RPS4=1: the one-row kernel for n1 = 64 / 32 (A/B)
  static const int rps_env = [] {
    const char* e = getenv("HX_P40_RPS");
    return e ? atoi(e) : 2;
  }();
  static const int rps4_env = [] {
    const char* e = getenv("HX_P40_RPS4");
    return e ? atoi(e) : 2;
  }();
  const int rps = kpt == 8 ? rps_env : rps4_env;
  if (rps == 2 && A.rpb % 2 == 0) {
    constexpr int RPS = 2;
    A.stages = 3;  // 3 x 2 rows in flight
    auto gox = [&](auto kern, int nw) {
      const size_t smem = (size_t)A.stages * RPS * 5 * A.n1 * kP40TT + sizeof(double) * 2 * nw * RPS * 2 * 3 * 32;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, 32 * nw, smem, s>>>(A);
    };
    if (kpt == 8) {
      gox(bsgs_mac_p40x_kernel<8, RPS, 8>, 8);
      return;
    }
    if (kpt == 4) {  // n1 = 32
      static const int nw4 = [] {  // HX_P40_NW4=8: 8 warps x 4 baby steps (A/B)
        const char* e = getenv("HX_P40_NW4");
        return e ? atoi(e) : 4;
      }();
      if (nw4 == 4)
        gox(bsgs_mac_p40x_kernel<8, RPS, 4>, 4);
      else
        gox(bsgs_mac_p40x_kernel<4, RPS, 8>, 8);
      return;
    }
  }
  const size_t smem = (size_t)A.stages * 5 * A.n1 * kP40TT;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * kP40Warps, smem, s>>>(A);
  };
  switch (kpt) {
    case 4: go(bsgs_mac_p40_kernel<4>); break;
    case 8: go(bsgs_mac_p40_kernel<8>); break;
    default: break;
  }
}

}  // namespace hx
