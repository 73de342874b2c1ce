// hx_bsgs_tc.cu -- BSGS diagonal multiply-accumulate on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM, diagonals streamed
// into shared memory by the bulk-copy engine).
//
// The MAC of matvec_bsgs (the mul_acc loop over
// rns_poly.cpp:102-110) is, for every limb i and coefficient t, a small
// modular matrix product
//     Y[r][(c, tok)] = sum_k D_r,k[i][t] * B_tok,k,c[i][t]  mod q_i,
// r = (row block b, giant step j) < R <= 128, k < n1 baby steps, c the
// ciphertext poly, tok the token.  It is a dense contraction, so it runs on
// the INT8 tensor cores, exactly, through byte slicing:
//   * D (a plaintext diagonal word, q < 2^40) is split into 5 bytes D_a;
//   * the baby word B is pre-multiplied per plane, B^(a) = B 2^(8a) mod q, and
//     split into 5 bytes B^(a)_b;
//   * Y = sum_b 2^(8b) sum_(a,k) D_a[r][k] B^(a)_b[k][(c,tok)]  (mod q):
//     ONE u8 x u8 -> s32 GEMM per coefficient with K' = 5 n1 (a, k) and
//     N' = 5 * 2T (b, c, tok); every s32 sum is < 5 n1 255^2 < 2^24 (n1 <= 64),
//     and the 5 planes recombine exactly in 64 bits (< 2^56) before one
//     reduction mod q.  Bit-identical to the integer / FP64 MAC kernels.
//
// HBM layout of the packed diagonals ("TC layout", built once per matrix by
// tc_pack_kernel): per TC-class limb li and coefficient t, the R_pad x K'_pad
// byte matrix A_t in the tcgen05 K-major SWIZZLE_NONE canonical form (8-row
// x 16-byte core matrices; core matrices adjacent in K 128 B apart, 8-row
// groups KC * 128 B apart) -- one bulk copy lands it ready for the MMA.
// 5 bytes per diagonal word instead of 8: the dominant HBM stream of the
// matvec shrinks by 37.5 %.  Limbs with q >= 2^40 (the 60-bit q_0) keep u64
// words ([li][r][k][N]) and the integer MAC kernel.
//
// Kernel (persistent, 2 CTAs / SM, 4 warps): per work item = (limb, group of
// G consecutive coefficients):
//   1. thread 0: expect-tx + G bulk copies of A_t (cp.async.bulk, mbarrier);
//   2. all threads: build B'_t (K-major, same canonical form) from the baby
//      words (4 consecutive k packed into one 32-bit st.shared per plane byte);
//   3. thread 0: G x KC/2 tcgen05.mma (M = 128, N = N', K = 32) into TMEM
//      columns [g N', (g+1) N'), tcgen05.commit -> mbarrier;
//   4. 4 warps: tcgen05.ld their 32 TMEM lanes (= rows), recombine the planes,
//      reduce mod q, store the G coefficients of each output as one vector.
#include <cstdint>
#include <vector>

#include "hx_internal.h"

namespace hx {



__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(u64* bar, u32 parity) {
  u32 ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait with a short sleep between polls: a spinning warp would take issue
// slots from the builder / epilogue warps of its SM sub-partition
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  if (mbar_try(bar, parity)) return;
  u32 ns = 32;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ns);
    if (ns < 256) ns *= 2;
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, SWIZZLE_NONE shared-memory matrix descriptor (tcgen05): start
// address, leading byte offset (core matrices adjacent in K), stride byte
// offset (adjacent 8-row groups), version 1
__device__ __forceinline__ u64 umma_desc(u32 saddr, u32 lbo, u32 sbo) {
  return (u64)((saddr >> 4) & 0x3FFF) | ((u64)((lbo >> 4) & 0x3FFF) << 16) | ((u64)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46);
}

// instruction descriptor: u8 x u8 -> s32, both K-major, M x N
__host__ __device__ constexpr u32 idesc_i8(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((u32)(N >> 3) << 17) | ((u32)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 16 consecutive TMEM columns of the warp's 32 lanes (one row per thread)
__device__ __forceinline__ void tmem_ld16(u32 taddr, u32 (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld1(u32 taddr, u32& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Barrett with a 32-bit quotient estimate, q in (2^39, 2^40): for v < 2^(32+s),
// qt = (floor(v / 2^s) mu) >> 32 with mu = floor(2^(32+s) / q) is within 2 of
// floor(v / q), so v - qt q < 3q and two conditional subtractions finish it
__device__ __forceinline__ u64 barrett_small(u64 v, int s, u32 mu, u64 q) {
  const u64 qt = ((u64)(u32)(v >> s) * mu) >> 32;
  u64 r = v - qt * q;
  r = r >= q ? r - q : r;
  return r >= q ? r - q : r;
}

__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on `bar` once all prior cp.async of this thread have landed (counts as an arrival)
__device__ __forceinline__ void cp_async_arrive(u64* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// warp roles of the persistent CTA (one per SM)
constexpr int kTcProducerWarp = 0;  // bulk copies of A tiles, cp.async of baby words
constexpr int kTcMmaWarp = 1;       // one lane issues tcgen05.mma
constexpr int kTcBuildWarp0 = 2, kTcBuildWarps = 6;   // B' tiles
constexpr int kTcEpiWarp0 = 8, kTcEpiWarps = 8;       // TMEM -> reduce -> store (2 per TMEM sub-partition)
constexpr int kTcWarps = kTcEpiWarp0 + kTcEpiWarps;

#ifdef HX_TC_TRACE
// per-item role timeline of CTA 0 (clock64), read by hx_tc_trace_get (trace builds only)
__device__ unsigned long long hx_tc_trace[16][64];
#define TC_TRACE(ev, n)                                                                        \
  do {                                                                                         \
    if (blockIdx.x == 0 && (n) < 64) hx_tc_trace[ev][n] = (unsigned long long)clock64();       \
  } while (0)
#else
#define TC_TRACE(ev, n) \
  do {                  \
  } while (0)
#endif
constexpr int kTcThreads = 32 * kTcWarps;
constexpr int kTcCols = 512;  // TMEM: two accumulator sets of 256 columns
constexpr int kTcMaxStages = 4;  // A / baby / B' ring depth: as many as fit (>= 2)
constexpr size_t kTcSmemMax = 225 * 1024;

template <int T>
struct TcShape {
  static constexpr int NC = 10 * T;               // used accumulator columns: n = (c T + tok) 5 + b
  static constexpr int NP = (NC + 15) / 16 * 16;  // MMA N (multiple of 16 for M = 128)
};

// shared-memory plan: S stages of (A tiles, B' tiles, baby words) + barriers
struct TcSmem {
  size_t a, bp, bb, stage;
  int stages;
  __host__ __device__ TcSmem(int G, int NP, int KC, int T, int n1) {
    a = (size_t)G * 16 * KC * 128;
    bp = (size_t)G * (NP / 8) * KC * 128;
    bb = (size_t)G * n1 * 2 * T * 8;
    stage = a + bp + bb;
    stages = (int)((kTcSmemMax - 256) / stage);
    if (stages > kTcMaxStages) stages = kTcMaxStages;
  }
  __host__ __device__ size_t total() const { return stages * stage + 256; }
};

// TMEM columns [c0, c0 + n) of this warp's 32 lanes, n in {1, 2, 4, 8, 16, 32} chunks
template <int NCOL>
__device__ __forceinline__ void tmem_ld_cols(u32 taddr, u32* v) {
  int c = 0;
#pragma unroll
  for (; c + 16 <= NCOL; c += 16) {
    u32 p[16];
    tmem_ld16(taddr + c, p);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[c + e] = p[e];
  }
#pragma unroll
  for (; c < NCOL; ++c) tmem_ld1(taddr + c, v[c]);
}

template <int T, int G>
__global__ void __launch_bounds__(kTcThreads, 1) bsgs_mac_tc_kernel(TcArgs A) {
  constexpr int NP = TcShape<T>::NP;

  static_assert(G * NP <= kTcCols / 2, "TMEM columns");
  extern __shared__ __align__(128) unsigned char sm[];
  const TcSmem plan(G, NP, A.KC, T, A.n1);
  const int S = plan.stages;
  const int KB = A.KC * 128;  // bytes of one 8-row group (all K chunks)
  // stage s: A tiles [G][16 groups][KC][128] | B' tiles [G][NP/8 groups][KC][128] | baby [g][k][c][tok]
  auto sA = [&](int s) { return sm + s * plan.stage; };
  auto sBp = [&](int s) { return sm + s * plan.stage + plan.a; };
  auto sBb = [&](int s) { return (u64*)(sm + s * plan.stage + plan.a + plan.bp); };
  u64* bar = (u64*)(sm + S * plan.stage);
  u64* full_a = bar;             // [S] A tiles landed (expect-tx)
  u64* full_b = bar + S;         // [S] baby words landed (expect-tx)
  u64* bp_full = bar + 2 * S;    // [S] B' built (builder threads)
  u64* slot_free = bar + 3 * S;  // [S] MMA done reading stage s
  u64* acc_full = bar + 4 * S;   // [2] accumulator set ready
  u64* acc_free = bar + 4 * S + 2;  // [2] accumulator set drained (epilogue threads)
  u32* tslot = (u32*)(bar + 4 * S + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long N = 1ll << A.logn;
  const int n1 = A.n1;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(kTcCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&full_b[s], 1);
      mbar_init(&bp_full[s], 32 * kTcBuildWarps);
      mbar_init(&slot_free[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&acc_full[x], 1);
      mbar_init(&acc_free[x], 32 * kTcEpiWarps);
    }
  }
  // rows >= 8 RG of every A slot stay zero (the bulk copies never touch them)
  for (int s = 0; s < S; ++s)
    for (int g = 0; g < G; ++g) {
      unsigned char* z = sA(s) + (size_t)g * 16 * KB + (size_t)A.RG * KB;
      const int nz = (16 - A.RG) * KB / 16;
      for (int e = tid; e < nz; e += kTcThreads) reinterpret_cast<uint4*>(z)[e] = make_uint4(0, 0, 0, 0);
    }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const u32 tmem = *tslot;
  const long long groups = N / G;
  const long long items = (long long)A.n_tc * groups;
  // a contiguous range of items per CTA: consecutive coefficients of one limb
  // (the output rows of neighbouring items share L2 lines; the A tiles and
  // staged baby words of the range are one sequential stream)
  const long long per = items / gridDim.x, extra = items % gridDim.x;
  const long long first = blockIdx.x * per + (blockIdx.x < extra ? blockIdx.x : extra);
  const long long my_items = per + (blockIdx.x < extra ? 1 : 0);
  auto item_of = [&](long long n, int& li, long long& t0) {
    const long long item = first + n;
    li = (int)(item / groups);
    t0 = (item % groups) * G;
  };

  if (warp == kTcProducerWarp) {
    const u32 abytes = (u32)A.RG * KB;
    for (long long n = 0; n < my_items; ++n) {
      const int s = (int)(n % S);
      if (n >= S) mbar_wait(&slot_free[s], (u32)((n / S - 1) & 1));
      if (lane == 0) TC_TRACE(0, n);
      int li;
      long long t0;
      item_of(n, li, t0);
      if (lane == 0) {
        mbar_expect_tx(&full_a[s], abytes * G);
        const unsigned char* src = A.packed + ((size_t)li * N + t0) * abytes;
#pragma unroll
        for (int g = 0; g < G; ++g) bulk_g2s(sA(s) + (size_t)g * 16 * KB, src + (size_t)g * abytes, abytes, &full_a[s]);
      }
      if (lane == 0) {
        // transposed baby words [li][t][k][c][tok]: the G coefficients of the item are contiguous
        const u32 bbytes = (u32)(G * n1 * 2 * T * 8);
        mbar_expect_tx(&full_b[s], bbytes);
        bulk_g2s(sBb(s), A.baby + ((size_t)li * N + t0) * n1 * 2 * T, bbytes, &full_b[s]);
      }
    }
  } else if (warp == kTcMmaWarp) {
    if (lane == 0) {
      const u32 idesc = idesc_i8(128, NP);
      const int KS = A.KC / 2;  // MMA K steps of 32 bytes
      for (long long n = 0; n < my_items; ++n) {
        const int s = (int)(n % S), x = (int)(n & 1);
        TC_TRACE(13, n);
        if (n >= 2) mbar_wait(&acc_free[x], (u32)(((n >> 1) - 1) & 1));
        TC_TRACE(4, n);
        mbar_wait(&full_a[s], (u32)((n / S) & 1));
        TC_TRACE(5, n);
        mbar_wait(&bp_full[s], (u32)((n / S) & 1));
        TC_TRACE(6, n);
        tc_fence_after();
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const u32 a0 = smem_u32(sA(s) + (size_t)g * 16 * KB), b0 = smem_u32(sBp(s) + (size_t)g * (NP / 8) * KB);
          for (int k = 0; k < KS; ++k)
            mma_i8(tmem + (u32)(x * (kTcCols / 2) + g * NP), umma_desc(a0 + k * 256, 128, KB),
                   umma_desc(b0 + k * 256, 128, KB), idesc, k > 0 ? 1u : 0u);
        }
        TC_TRACE(11, n);
        mma_commit(&slot_free[s]);
        mma_commit(&acc_full[x]);
        TC_TRACE(12, n);
      }
    }
  } else if (warp < kTcEpiWarp0) {
    // ---- B' builders: unit = (tok, poly c, coefficient g, quad kq), tok fastest
    const int bt = tid - 32 * kTcBuildWarp0;
    const int nkq = n1 / 4;
    const int units = G * T * 2 * nkq;
    for (long long n = 0; n < my_items; ++n) {
      const int s = (int)(n % S);
      int li;
      long long t0;
      item_of(n, li, t0);
      const int i = A.limbs[li];
      const u64 q = A.pc[i].q;
      const u32 mu48 = A.mu[2 * li + 1];
      mbar_wait(&full_b[s], (u32)((n / S) & 1));
      if (bt == 0) TC_TRACE(1, n);
      if (n >= S) mbar_wait(&slot_free[s], (u32)((n / S - 1) & 1));
      if (bt == 0) TC_TRACE(2, n);
      const u64* bb = sBb(s);
      for (int u = bt; u < units; u += 32 * kTcBuildWarps) {
        // lane order (tok, kq mod 4, c, g, kq / 4): the 32 stores of a warp
        // land on distinct (row nn mod 8, 4-byte column kq mod 4) words of
        // the 128-byte core matrices -- one shared-memory wavefront each for
        // T >= 4 (tok fastest alone put 4 lanes on every bank)
        const int tok = u % T;
        int rest = u / T;
        int kq, c, g;
        if ((nkq & 3) == 0) {
          const int klo = rest & 3;
          rest >>= 2;
          c = rest & 1;
          rest >>= 1;
          g = rest % G;
          kq = klo + 4 * (rest / G);
        } else {
          c = rest & 1;
          rest >>= 1;
          g = rest % G;
          kq = rest / G;
        }
        u64 w[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) w[m] = bb[((size_t)(g * n1 + 4 * kq + m) * 2 + c) * T + tok];
        unsigned char* bg = sBp(s) + (size_t)g * (NP / 8) * KB;
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          const int kp = a * n1 + 4 * kq;
          unsigned char* col = bg + (kp >> 4) * 128 + (kp & 15);
          u32 wl[4], wh[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            wl[m] = (u32)w[m];
            wh[m] = (u32)(w[m] >> 32);
          }
#pragma unroll
          for (int b = 0; b < 5; ++b) {
            const int nn = (c * T + tok) * 5 + b;
            // byte b of w[0..3] -> bytes 0..3 of one word (bytes 0-3 from the low halves, 4 from the high)
            const u32 sel = b < 4 ? (u32)(b | ((4 + b) << 4)) : 0x40u;
            const u32 p01 = __byte_perm(b < 4 ? wl[0] : wh[0], b < 4 ? wl[1] : wh[1], sel);
            const u32 p23 = __byte_perm(b < 4 ? wl[2] : wh[2], b < 4 ? wl[3] : wh[3], sel);
            *reinterpret_cast<u32*>(col + (nn >> 3) * KB + (nn & 7) * 16) = __byte_perm(p01, p23, 0x5410);
          }
          if (a < 4) {
#pragma unroll
            for (int m = 0; m < 4; ++m) w[m] = barrett_small(w[m] << 8, 16, mu48, q);
          }
        }
      }
      fence_async_smem();
      if (bt == 0) TC_TRACE(3, n);
      if (bt == 32 * kTcBuildWarps - 1) TC_TRACE(10, n);
      mbar_arrive(&bp_full[s]);
    }
  } else {
    // ---- epilogue: warp = (TMEM sub-partition sp, poly c); thread = row r
    const int ew = warp - kTcEpiWarp0;
    const int sp = warp & 3, c = ew >> 2;
    const int r = sp * 32 + lane;
    const long long roff = r < A.rows ? A.row_off[r] : 0;
    constexpr int P = 4 / G;  // items per 32-byte output group
    u64 grp[4][T];
    for (long long n = 0; n < my_items; ++n) {
      const int x = (int)(n & 1);
      int li;
      long long t0;
      item_of(n, li, t0);
      const int i = A.limbs[li];
      const u64 q = A.pc[i].q;
      const u32 mu56 = A.mu[2 * li];
      mbar_wait(&acc_full[x], (u32)((n >> 1) & 1));
      if (ew == 0 && lane == 0) TC_TRACE(7, n);
      tc_fence_after();
      const u32 tbase = tmem + ((u32)(sp * 32) << 16) + (u32)(x * (kTcCols / 2) + c * T * 5);
      // slot of this item in its aligned group of 4 coefficients (one 32-byte
      // sector per output row): the group is written once, whole -- partial
      // sector writes cost a DRAM read-modify-write each
      const int p = (int)((t0 & 3) / G);
      const bool whole = n - p >= 0 && n - p + P - 1 < my_items;
      const bool live = sp * 32 < A.rows;  // sub-partitions without rows only release the accumulator
#pragma unroll
      for (int g = 0; g < (live ? G : 0); ++g) {
        u32 v[5 * T];
        tmem_ld_cols<5 * T>(tbase + (u32)(g * NP), v);
        tmem_wait_ld();
#pragma unroll
        for (int tok = 0; tok < T; ++tok) {
          const u32* y = v + 5 * tok;
          const u64 V = (u64)y[0] + (u64)y[1] * 256u + (u64)y[2] * 65536u + (u64)y[3] * 16777216u + ((u64)y[4] << 32);
          const u64 val = barrett_small(V, 24, mu56, q);
#pragma unroll
          for (int pp = 0; pp < P; ++pp)
            if (pp == p) grp[pp * G + g][tok] = val;
        }
      }
      tc_fence_before();
      if (ew == 0 && lane == 0) TC_TRACE(8, n);
      if (ew == 4 && lane == 0) TC_TRACE(14, n);
      if (ew == 3 && lane == 0) TC_TRACE(15, n);
      mbar_arrive(&acc_free[x]);
      if (r < A.rows) {
#pragma unroll
        for (int tok = 0; tok < T; ++tok) {
          u64* o = A.inner + roff + tok * A.tstride + c * A.L + (long long)i * N + (t0 & ~3ll);
          if (whole) {
            if (p == P - 1)
              asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(o), "l"(grp[0][tok]), "l"(grp[1][tok]),
                           "l"(grp[2][tok]), "l"(grp[3][tok])
                           : "memory");
          } else {  // group split between two CTAs' ranges: this item's words alone
#pragma unroll
            for (int pp = 0; pp < P; ++pp)
              if (pp == p)
#pragma unroll
                for (int g = 0; g < G; ++g) o[pp * G + g] = grp[pp * G + g][tok];
          }
        }
      }
      if (ew == 0 && lane == 0) TC_TRACE(9, n);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcCols));
}

// ------------------------------------------------------ baby transposition
// baby steps [tok][k][c][n_q][N] (hoisted-rotation output) -> [li][t][k][c][tok]
// for the TC-class limbs: the words one MAC work item needs become one
// contiguous run (one bulk copy).  Tile of 8 coefficients x all (k, c, tok)
// rows through shared memory: 64-byte reads, contiguous n1 2 T-word writes.
__global__ void tc_baby_kernel(u64* out, const u64* baby, long long btstride, long long L, const int* limbs,
                               int n1, int T, int logn) {
  extern __shared__ u64 tile[];  // [rows][8]
  const long long N = 1ll << logn;
  const int li = blockIdx.y, i = limbs[li];
  const long long t0 = (long long)blockIdx.x * 8;
  const int rows = n1 * 2 * T;
  for (int e = threadIdx.x; e < rows * 8; e += blockDim.x) {
    const int row = e >> 3, tt = e & 7;
    const int tok = row % T, c = (row / T) & 1, k = row / (2 * T);
    tile[e] = __ldcs(baby + tok * btstride + (2ll * k + c) * L + (long long)i * N + t0 + tt);
  }
  __syncthreads();
  u64* o = out + ((size_t)li * N + t0) * rows;
  for (int e = threadIdx.x; e < rows * 8; e += blockDim.x) {
    const int tt = e / rows, row = e % rows;
    o[e] = tile[row * 8 + tt];
  }
}

// ---------------------------------------------------------------- packing
// TC section: thread per (limb li, coefficient t, row r, K chunk kc) writes the
// 16 bytes k' in [16 kc, 16 kc + 16) of row r: byte a of diagonal (r, k) at
// k' = a n1 + k (zero past 5 n1, for rows >= R and for absent diagonals).
__global__ void tc_pack_kernel(unsigned char* dst, const u64* const* dptr, const int* limbs, int rows, int n1,
                               int KC, int RG, int logn) {
  const long long N = 1ll << logn;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int kc = blockIdx.y % KC, r = blockIdx.y / KC;
  const int li = blockIdx.z;
  const int i = limbs[li];
  u32 out[4] = {0, 0, 0, 0};
  if (r < rows) {
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const int kp = kc * 16 + p;
      if (kp < 5 * n1) {
        const int a = kp / n1, k = kp % n1;
        const u64* d = dptr[(size_t)r * n1 + k];
        const u32 byte = d ? (u32)((__ldg(d + (long long)i * N + t) >> (8 * a)) & 0xff) : 0u;
        out[p >> 2] |= byte << (8 * (p & 3));
      }
    }
  }
  const size_t KB = (size_t)KC * 128;
  unsigned char* o = dst + ((size_t)li * N + t) * RG * KB + (size_t)(r >> 3) * KB + (size_t)kc * 128 + (r & 7) * 16;
  *reinterpret_cast<uint4*>(o) = make_uint4(out[0], out[1], out[2], out[3]);
}

// wide section: [w][r][k][N] u64 copies of the limbs with q >= 2^40
__global__ void tc_pack_wide_kernel(u64* dst, const u64* const* dptr, const int* limbs, int rows, int n1, int logn) {
  const long long N = 1ll << logn;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int rk = blockIdx.y, w = blockIdx.z;
  const int i = limbs[w];
  const u64* d = dptr[rk];
  dst[((size_t)w * rows * n1 + rk) * N + t] = d ? __ldg(d + (long long)i * N + t) : 0ull;
}

// ------------------------------------------------------------- launchers
namespace {

template <int T, int G>
void launch_tc(const TcArgs& A, int sms, cudaStream_t s) {
  constexpr int NP = TcShape<T>::NP;
  const size_t smem = TcSmem(G, NP, A.KC, T, A.n1).total();
  cudaFuncSetAttribute(bsgs_mac_tc_kernel<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long items = (long long)A.n_tc * ((1ll << A.logn) / G);
  const int grid = (int)(items < sms ? items : sms);
  bsgs_mac_tc_kernel<T, G><<<grid, kTcThreads, smem, s>>>(A);
}

// largest coefficient group G in {4, 2, 1} whose accumulators (G N' TMEM
// columns, double-buffered) and shared memory fit one CTA per SM
template <int T>
void dispatch_g(const TcArgs& A, int sms, cudaStream_t s) {
  constexpr int NP = TcShape<T>::NP;
  auto fits = [&](int G) { return G * NP <= kTcCols / 2 && TcSmem(G, NP, A.KC, T, A.n1).stages >= 3; };
  if constexpr (4 * NP <= kTcCols / 2) {
    if (fits(4)) return launch_tc<T, 4>(A, sms, s);
  }
  if constexpr (2 * NP <= kTcCols / 2) {
    if (fits(2)) return launch_tc<T, 2>(A, sms, s);
  }
  launch_tc<T, 1>(A, sms, s);
}

}  // namespace

int tc_max_tokens() { return kTcMaxTokens; }

#ifdef HX_TC_TRACE
extern "C" int hx_tc_trace_get(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, hx_tc_trace, sizeof(hx_tc_trace)) == cudaSuccess ? 0 : 1;
}
#endif

void launch_tc_baby(u64* out, const u64* baby, long long btstride, long long L, const int* limbs, int n_tc, int n1,
                    int T, int logn, cudaStream_t s) {
  const int smem = n1 * 2 * T * 8 * 8;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tc_baby_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 2 * kTcMaxTokens * 64);
    configured = true;
  }
  tc_baby_kernel<<<dim3((unsigned)((1ll << logn) / 8), (unsigned)n_tc), 256, smem, s>>>(out, baby, btstride, L, limbs,
                                                                                       n1, T, logn);
}

void launch_bsgs_mac_tc(const TcArgs& A, int tokens, int sms, cudaStream_t s) {
  switch (tokens) {
    case 1: return dispatch_g<1>(A, sms, s);
    case 2: return dispatch_g<2>(A, sms, s);
    case 4: return dispatch_g<4>(A, sms, s);
    case 8: return dispatch_g<8>(A, sms, s);
    default: break;
  }
}

void launch_tc_pack(unsigned char* dst, const u64* const* dptr, const int* tc_limbs, int n_tc, const int* wide_limbs,
                    int n_wide, int rows, int n1, int KC, int RG, int logn, size_t tc_bytes, cudaStream_t s) {
  const long long N = 1ll << logn;
  const int th = 128;
  if (n_tc)
    tc_pack_kernel<<<dim3((unsigned)(N / th), (unsigned)(RG * 8 * KC), (unsigned)n_tc), th, 0, s>>>(
        dst, dptr, tc_limbs, rows, n1, KC, RG, logn);
  if (n_wide)
    tc_pack_wide_kernel<<<dim3((unsigned)(N / th), (unsigned)(rows * n1), (unsigned)n_wide), th, 0, s>>>(
        reinterpret_cast<u64*>(dst + tc_bytes), dptr, wide_limbs, rows, n1, logn);
}

}  // namespace hx
