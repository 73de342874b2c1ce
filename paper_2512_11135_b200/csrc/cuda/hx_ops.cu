// hx_ops.cu -- context construction, launchers and the C-ABI of libhx_b200.
//
// Host-side precomputation mirrors the reference constructors:
//   psi search            ntt.cpp:23-32   (smallest g with (g^((q-1)/2N))^N = -1)
//   twiddle tables        ntt.cpp:36-55   (psi^brv(i), psi^-brv(i), Shoup)
//   rescale constants     rns_poly.cpp:144-162
//   moddown constants     rns_poly.cpp:164-180 (generalised to K primes)
// and the SPEC-only hybrid key-switch constants (ModUp FastBConv per digit).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../../../include/hx_b200.h"
#include "hx_internal.h"
#include "hx_kernels.cuh"
#include "hx_modup.cuh"
#include "hx_rowinner.cuh"

using hx::LimbTable;
using hx::PrimeConst;
using hx::SC;
using hx::u64;
using u128 = unsigned __int128;

namespace {

thread_local std::string g_last_error;

struct HxError : std::runtime_error {
  int code;
  HxError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HX_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) throw HxError(HX_ERR_INVALID, msg); \
  } while (0)

// element counts: negative is an error, zero a no-op (no zero-sized launches)
#define HX_COUNT(n)                                   \
  do {                                                \
    HX_REQUIRE((n) >= 0, "negative element count");   \
    if ((n) == 0) return;                              \
  } while (0)

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw HxError(HX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void launched(hx_ctx* c, const char* what, int n = 1) {
  c->launches += n;
  cuda_ok(cudaGetLastError(), what);
}

template <class F>
int guarded(F f) {
  try {
    f();
    return HX_OK;
  } catch (const HxError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HX_ERR_INVALID;
  }
}

// ---- host modular arithmetic (setup only) ----
u64 hmul(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
u64 hpow(u64 a, u64 e, u64 q) {
  u64 r = 1 % q, b = a % q;
  while (e) {
    if (e & 1) r = hmul(r, b, q);
    b = hmul(b, b, q);
    e >>= 1;
  }
  return r;
}
u64 hinv(u64 a, u64 q) { return hpow(a % q, q - 2, q); }
u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
SC sc(u64 w, u64 q) { return SC{w % q, shoup(w % q, q)}; }
u64 brv(u64 x, int bits) {
  u64 r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}
bool is_prime(u64 n) {
  static const u64 sm[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 p : sm)
    if (n % p == 0) return n == p;
  u64 d = n - 1;
  int r = 0;
  while (!(d & 1)) {
    d >>= 1;
    ++r;
  }
  for (u64 a : sm) {
    u64 x = hpow(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < r; ++i) {
      x = hmul(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}
// ntt.cpp:23-32
u64 find_psi(u64 q, u64 n) {
  const u64 order = 2 * n;
  for (u64 g = 2; g < q; ++g) {
    const u64 c = hpow(g, (q - 1) / order, q);
    if (hpow(c, n, q) == q - 1) return c;
  }
  throw HxError(HX_ERR_INVALID, "no primitive 2N-th root");
}

// An allocation that failed may succeed once the stream-ordered pool has
// returned its cached (freed) blocks to the device: sync, trim, retry once.
void trim_pool() {
  cudaGetLastError();
  if (getenv("HX_ALLOC_TRACE")) fprintf(stderr, "[hx] pool trim + retry\n");
  cuda_ok(cudaDeviceSynchronize(), "sync");
  int dev = 0;
  cudaMemPool_t pool;
  cuda_ok(cudaGetDevice(&dev), "device");
  cuda_ok(cudaDeviceGetDefaultMemPool(&pool, dev), "mem pool");
  cuda_ok(cudaMemPoolTrimTo(pool, 0), "mem pool trim");
}

// ---- stream-ordered scratch buffer ----
// Scoped device temporary: from the context arena (HxArena, hx_internal.h)
// when a context is given, else from the stream-ordered pool.
struct DBuf {
  u64* p = nullptr;
  cudaStream_t s = nullptr;
  hx_ctx* c = nullptr;
  size_t bytes = 0;
  bool from_arena = false;
  DBuf(size_t words, cudaStream_t st, hx_ctx* ctx = nullptr) : s(st), c(ctx), bytes(((words * 8) + 255) & ~size_t(255)) {
    if (!words) return;
    static const bool no_arena = getenv("HX_NO_ARENA") != nullptr;  // debugging: pool allocations only
    if (no_arena) c = nullptr;
    if (c) {
      HxArena& A = c->arena;
      if (A.stream_set && A.stream != st) {  // hand the arena over to stream st
        if (!A.ev) cuda_ok(cudaEventCreateWithFlags(&A.ev, cudaEventDisableTiming), "event");
        cuda_ok(cudaEventRecord(A.ev, A.stream), "event record");
        cuda_ok(cudaStreamWaitEvent(st, A.ev, 0), "stream wait");
      }
      A.stream = st;
      A.stream_set = true;
      if (A.depth == 0 && A.high > A.cap) {  // regrow to the high-water mark
        // the arena is a plain cudaMalloc block outside the stream-ordered pool:
        // freeing it returns the memory to the device at once (the pool keeps
        // what it frees), and the pool's cached blocks stay untouched
        if (A.base) {
          cuda_ok(cudaStreamSynchronize(st), "sync");
          cuda_ok(cudaFree(A.base), "cudaFree(arena)");
        }
        A.base = nullptr;
        if (cudaMalloc((void**)&A.base, A.high) != cudaSuccess) {
          A.base = nullptr;
          trim_pool();
          cuda_ok(cudaMalloc((void**)&A.base, A.high), "cudaMalloc(arena)");
        }
        A.cap = A.high;
        if (getenv("HX_ALLOC_TRACE")) fprintf(stderr, "[hx] arena regrown to %.2f GB\n", A.cap * 1e-9);
      }
      A.depth++;
      A.high = std::max(A.high, A.top + bytes);
      if (A.base && A.top + bytes <= A.cap) {
        p = (u64*)(A.base + A.top);
        A.top += bytes;
        from_arena = true;
        return;
      }
      A.top += bytes;  // keeps the LIFO accounting; memory from the pool
    }
    if (cudaMallocAsync((void**)&p, words * 8, st) != cudaSuccess) {
      p = nullptr;
      trim_pool();
      cuda_ok(cudaMallocAsync((void**)&p, words * 8, st), "cudaMallocAsync");
    }
  }
  ~DBuf() {
    if (!p) return;
    if (c) {
      c->arena.top -= bytes;
      c->arena.depth--;
    }
    if (!from_arena) cudaFreeAsync(p, s);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

template <class T>
T* upload(const std::vector<T>& v) {
  T* d = nullptr;
  if (v.empty()) return nullptr;
  cuda_ok(cudaMalloc((void**)&d, v.size() * sizeof(T)), "cudaMalloc(const)");
  cuda_ok(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
  return d;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void check_ctx(const hx_ctx* c) { HX_REQUIRE(c != nullptr, "null hx_ctx"); }
void check_nq(const hx_ctx* c, int n_q) {
  HX_REQUIRE(n_q >= 1 && n_q <= c->n_chain, "n_q out of range");
}

// strided 2-D device copy: rows of `width` words, pitches in words
void copy2d(u64* dst, long long dpitch, const u64* src, long long spitch, long long width,
            long long rows, cudaStream_t s) {
  if (rows <= 0 || width <= 0) return;
  cuda_ok(cudaMemcpy2DAsync(dst, dpitch * 8, src, spitch * 8, width * 8, rows,
                            cudaMemcpyDeviceToDevice, s),
          "cudaMemcpy2DAsync");
}

int ew_threads(const hx_ctx* c) { return (int)std::min<long long>(256, c->N() / 2); }
int pt_threads(const hx_ctx* c) { return (int)std::min<long long>(256, c->N()); }
// combine_kernel: kCombineEpt elements per thread (N >= kCombineEpt)
int combine_threads(const hx_ctx* c) { return (int)std::min<long long>(256, c->N() / hx::kCombineEpt); }

template <hx::EwOp OP>
void ew(hx_ctx* c, u64* out, const u64* a, const u64* b, long long batch, const LimbTable& lt,
        cudaStream_t s, long long a_mod = 0, long long b_div = 1) {
  hx::EwArgs A{out, a, b, c->d_pc, lt, c->logn, batch * lt.count};
  A.a_mod = a_mod;
  A.b_div = b_div;
  const int th = ew_threads(c);
  const long long blocks = A.instances * (c->N() / (2 * th));
  if (blocks <= 0) return;
  hx::ew_kernel<OP><<<(unsigned)blocks, th, 0, s>>>(A);
  launched(c, "ew_kernel");
}

void automorphism(hx_ctx* c, u64* out, const u64* in, long long batch, const LimbTable& lt,
                  u64 g, cudaStream_t s) {
  hx::EwArgs A{out, in, nullptr, c->d_pc, lt, c->logn, batch * lt.count};
  const int th = pt_threads(c);
  const long long blocks = A.instances * (c->N() / th);
  if (blocks <= 0) return;
  hx::automorphism_kernel<<<(unsigned)blocks, th, 0, s>>>(A, (hx::u32)g);
  launched(c, "automorphism_kernel");
}

// ---- key-switch building blocks ----

// ---- fused ModUp bconv + forward COL pass (hx_modup.cuh) ----
template <int S, int MAXA, bool CEN>
void launch_modup_col_t(hx_ctx* c, const hx::ModUpColArgs& A, long long batch, cudaStream_t s) {
  constexpr int OB = 3, TILE = 1 << (S + OB);
  auto kern = hx::modup_col_kernel<S, OB, MAXA, CEN>;
  const int smem = hx::modup_col_smem_bytes(S, OB, MAXA, CEN);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  // enough CTAs for ~3 waves of resident CTAs even for one ciphertext
  hx::ModUpColArgs B = A;
  const long long base = (c->N() / TILE) * (long long)A.dnum * batch;
  int maxt = 1;
  for (int d = 0; d < A.dnum; ++d) maxt = std::max(maxt, A.tcnt[d] + A.icnt[d]);
  B.tsplit = (int)std::max(1ll, std::min<long long>(maxt, (148ll * 3 * 3 + base - 1) / base));
  HX_REQUIRE(batch * B.tsplit <= 65535, "modup_col: batch too large for one launch");
  dim3 grid((unsigned)(c->N() / TILE), (unsigned)(batch * B.tsplit), (unsigned)A.dnum);
  {
    hx::KTimer kt(c, A.centred ? "moddown_col_kernel" : "modup_col_kernel", s);
    kern<<<grid, TILE / 16, smem, s>>>(B);
  }
  launched(c, "modup_col_kernel");
}

template <int S, bool CEN>
bool launch_modup_col_a(hx_ctx* c, const hx::ModUpColArgs& A, long long batch, cudaStream_t s) {
  switch (A.alpha) {
    case 1: launch_modup_col_t<S, 1, CEN>(c, A, batch, s); return true;
    case 2: launch_modup_col_t<S, 2, CEN>(c, A, batch, s); return true;
    case 3: launch_modup_col_t<S, 3, CEN>(c, A, batch, s); return true;
    case 4: launch_modup_col_t<S, 4, CEN>(c, A, batch, s); return true;
    default: return false;
  }
}

template <bool CEN>
bool launch_modup_col_c(hx_ctx* c, const hx::ModUpColArgs& A, long long batch, cudaStream_t s) {
  switch (hx::ntt_split_a(c->logn)) {
    case 5: return launch_modup_col_a<5, CEN>(c, A, batch, s);
    case 6: return launch_modup_col_a<6, CEN>(c, A, batch, s);
    case 7: return launch_modup_col_a<7, CEN>(c, A, batch, s);
    case 8: return launch_modup_col_a<8, CEN>(c, A, batch, s);
    default: return false;
  }
}

// A.centred selects the ModDown instantiation (its own kernel, so ModUp's
// loop body and shared-memory footprint are untouched)
bool launch_modup_col(hx_ctx* c, const hx::ModUpColArgs& A, long long batch, cudaStream_t s) {
  return A.centred ? launch_modup_col_c<true>(c, A, batch, s) : launch_modup_col_c<false>(c, A, batch, s);
}

// Rounding constant 1.5 * 2^E of the fused conversion's joint reduction
// (hx_modup.cuh bconv_tile_f64) for source primes `sr` and FP64-class target
// primes `tg` (prime indices), `cen` centred-correction terms of up to p each;
// 0.0 when an exactness bound fails (the caller then takes the unfused path):
//   sum of the products  < 2^(E-1)           (the running sum keeps its binade)
//   |H / p| < 2^50                            (the rint range of the one quotient)
//   low parts + integer-pipe terms + centred terms, and the NTT's lazy growth
//   on top of the converted words, stay below 2^52
double bconv_round(const hx_ctx* c, const std::vector<int>& sr, const std::vector<int>& tg, int cen) {
  long double pmax = 0, pmin = 0, per_p = 0;
  int nprod = 0, nwide = 0;
  for (int j : tg) {
    const long double p = (long double)c->primes[j];
    pmax = std::max(pmax, p);
    pmin = pmin == 0 ? p : std::min(pmin, p);
  }
  for (int i : sr) {
    if (c->f64[i]) {
      per_p += (long double)c->primes[i];
      nprod += 1;
    } else {  // x = xh 2^30 + xl, q < 2^62 (or one Shoup product in [0, 2p) on the integer pipe)
      per_p += 4294967296.0L + 1073741824.0L;
      nprod += 2;
      nwide += 1;
    }
  }
  int E = 0;
  std::frexp((double)(per_p * pmax), &E);  // per_p pmax < 2^E
  E += 1;
  int lmin = 0;
  std::frexp((double)pmin, &lmin);         // pmin >= 2^(lmin - 1)
  if (E - 1 - (lmin - 1) > 50 || E > 1000) return 0.0;
  const long double lb = (long double)nprod * std::ldexp(1.0L, E - 53) + (2.0L * nwide + cen) * pmax;
  const long double word = pmax + lb;  // |r| < p
  if (2.0L * word + (long double)c->logn * pmax >= std::ldexp(1.0L, 52)) return 0.0;
  return std::ldexp(1.5, E);
}

bool modup_fused_ok(const hx_ctx* c, int n_q) {
  static const bool off = getenv("HX_MODUP_UNFUSED") != nullptr;
  const int a = hx::ntt_split_a(c->logn);
  return !off && a >= 5 && a <= 8 && c->alpha <= 4 && c->dnum(n_q) <= hx::kMaxDigits && c->cs_up[n_q] != 0.0;
}

// c1: [batch] polys of n_q limbs at stride c1_stride words.
// copy_own = false: the digits' own limbs are left out of `digits` (the key
// inner product reads them from c1, InnerArgs::c1)
// defer_rows: the FP64-class limbs are left after their COL pass (the fused
// ROW + inner-product kernel finishes them, ks_inner_multi rows_deferred);
// only valid when modup_fused_ok
bool side_stream_on() {
  static const bool on = getenv("HX_KS_SIDE") && atoi(getenv("HX_KS_SIDE")) != 0;
  return on;
}
// s -> c->side: the side stream starts after everything issued on s so far
void fork_side(hx_ctx* c, cudaStream_t s) {
  if (!c->side) {
    cuda_ok(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
    cuda_ok(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "side event");
    cuda_ok(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "side event");
  }
  cuda_ok(cudaEventRecord(c->ev_fork, s), "fork");
  cuda_ok(cudaStreamWaitEvent(c->side, c->ev_fork, 0), "fork");
  c->side_open = true;
}
// c->side -> s: work issued on s from now on waits for the side stream
void join_side(hx_ctx* c, cudaStream_t s) {
  if (!c->side_open) return;
  cuda_ok(cudaEventRecord(c->ev_join, c->side), "join");
  cuda_ok(cudaStreamWaitEvent(s, c->ev_join, 0), "join");
  c->side_open = false;
}

void modup(hx_ctx* c, u64* digits, const u64* c1, long long c1_stride, long long batch, int n_q,
           cudaStream_t s, bool copy_own = true, bool defer_rows = false) {
  const long long N = c->N();
  const int K = c->n_special, ext = n_q + K, dnum = c->dnum(n_q);
  DBuf coef(batch * n_q * N, s, c);
  hx::ntt_inverse(c, coef.p, batch, hx::make_table(c, n_q, 0), s, c1, c1_stride);  // out of place
  if (modup_fused_ok(c, n_q)) {
    // conversion fused into the COL pass (one launch per prime class), the
    // digits' own limbs copied from the NTT-domain input, then the ROW pass
    hx::ModUpColArgs A{};
    A.coef = coef.p;
    A.out = digits;
    A.pc = c->d_pc;
    A.qhinv = c->d_modup;
    A.bc = c->d_bconv;
    A.tlist = c->d_tlist;
    A.alpha = c->alpha;
    A.n_q = n_q;
    A.n_chain = c->n_chain;
    A.ext = ext;
    A.dnum = dnum;
    A.logn = c->logn;
    A.src_n = n_q;
    A.src_pbase = 0;
    A.centred = 0;
    A.cs_round = c->cs_up[n_q];
    LimbTable lt{};
    lt.stride = dnum * ext;
    for (int d = 0; d < dnum; ++d) {
      A.qh_off[d] = c->modup_qh_off[n_q][d];
      A.bc_off[d] = c->bc_off[n_q][d];
      const int lo = d * c->alpha, cnt = std::min(c->alpha, n_q - lo);
      if (copy_own)
        copy2d(digits + ((long long)d * ext + lo) * N, (long long)dnum * ext * N, c1 + (long long)lo * N, c1_stride,
               (long long)cnt * N, batch, s);
      for (int j = 0; j < ext; ++j) {
        if (j >= lo && j < lo + cnt) continue;
        HX_REQUIRE(lt.count < hx::kMaxLimbEntries, "modup: too many limbs for one launch");
        lt.off[lt.count] = (unsigned short)(d * ext + j);
        lt.prime[lt.count] = (unsigned char)c->pidx(j, n_q);
        ++lt.count;
      }
    }
    int total = 0;
    for (int d = 0; d < dnum; ++d) {
      A.toff[d] = c->tl_off[n_q][d];
      A.tcnt[d] = c->tl_cnt[n_q][d];
      A.icnt[d] = c->tl_icnt[n_q][d];
      total += A.tcnt[d] + A.icnt[d];
    }
    if (total) HX_REQUIRE(launch_modup_col(c, A, batch, s), "modup: fused path unavailable");
    // integer-class limbs: full forward NTT; FP64-class limbs: ROW pass only
    LimbTable li{}, lf{};
    li.stride = lf.stride = lt.stride;
    for (int e = 0; e < lt.count; ++e) {
      LimbTable& x = c->f64[lt.prime[e]] ? lf : li;
      x.off[x.count] = lt.off[e];
      x.prime[x.count] = lt.prime[e];
      ++x.count;
    }
    if (li.count && defer_rows && side_stream_on()) {
      // the integer-class limbs (NTT here, inner product in ks_inner_multi)
      // on the side stream, beside the fused FP64 ROW + inner kernel
      fork_side(c, s);
      hx::ntt_forward(c, digits, batch, li, c->side);
    } else if (li.count) {
      hx::ntt_forward(c, digits, batch, li, s);
    }
    if (lf.count && !defer_rows) hx::ntt_forward_rows(c, digits, batch, lf, s);
    return;
  }
  HX_REQUIRE(!defer_rows, "modup: deferred ROW pass needs the fused path");
  // basis conversion per digit (coefficient domain), own limbs copied (NTT)
  LimbTable lt{};
  lt.stride = dnum * ext;
  lt.count = 0;
  const long long out_stride = (long long)dnum * ext * N;
  for (int d = 0; d < dnum; ++d) {
    const int lo = d * c->alpha, cnt = std::min(c->alpha, n_q - lo);
    hx::ModUpArgs A;
    A.coef = coef.p;
    A.out = digits + (long long)d * ext * N;
    A.pc = c->d_pc;
    A.qhinv = c->d_modup + c->modup_qh_off[n_q][d];
    A.conv = c->d_modup + c->modup_cv_off[n_q][d];
    A.lo = lo;
    A.cnt = cnt;
    A.n_q = n_q;
    A.n_chain = c->n_chain;
    A.n_special = K;
    A.n_total = c->n_total();
    A.out_stride = out_stride;
    A.logn = c->logn;
    const int th = pt_threads(c);
    dim3 grid((unsigned)(N / th), (unsigned)batch);
    if (c->alpha <= 1)
      hx::modup_bconv_kernel<1><<<grid, th, 0, s>>>(A);
    else if (c->alpha <= 2)
      hx::modup_bconv_kernel<2><<<grid, th, 0, s>>>(A);
    else if (c->alpha <= 4)
      hx::modup_bconv_kernel<4><<<grid, th, 0, s>>>(A);
    else
      hx::modup_bconv_kernel<8><<<grid, th, 0, s>>>(A);
    launched(c, "modup_bconv_kernel");
    copy2d(digits + ((long long)d * ext + lo) * N, out_stride, c1 + (long long)lo * N, c1_stride,
           (long long)cnt * N, batch, s);
    for (int j = 0; j < ext; ++j) {
      if (j >= lo && j < lo + cnt) continue;
      HX_REQUIRE(lt.count < hx::kMaxLimbEntries, "modup: too many limbs for one launch");
      lt.off[lt.count] = (unsigned short)(d * ext + j);
      lt.prime[lt.count] = (unsigned char)c->pidx(j, n_q);
      ++lt.count;
    }
  }
  if (lt.count) hx::ntt_forward(c, digits, batch, lt, s);
}

// Key inner products for R keys, E elements per key, one launch:
//   shared: keys[r] applies to digit elements 0..E-1 (hoisting);
//   !shared: keys[r] applies to digit elements r E .. r E + E - 1.
// Output element (r, e) at u + (r E + e) 2 ext N.
template <int S>
void launch_row_inner_t(hx_ctx* c, const hx::RowInnerArgs& A, cudaStream_t s) {
  constexpr int OB = 3, TILE = 1 << (S + OB);  // the ROW tile of hx_ntt.cu (HX_NTT_OB)
  auto kern = hx::ks_row_inner_f64_kernel<S, OB, 8>;
  // HX_RI_2CTA=1: request enough shared memory that only 2 CTAs fit an SM,
  // leaving registers for the side stream's integer kernels (HX_KS_SIDE)
  static const bool two = getenv("HX_RI_2CTA") && atoi(getenv("HX_RI_2CTA")) != 0;
  const int smem = two ? std::max(hx::row_inner_smem_bytes<S, OB>(), 78 * 1024) : hx::row_inner_smem_bytes<S, OB>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  const long long blocks = (long long)A.batch * (c->N() / TILE) * A.n_limbs;
  if (blocks <= 0) return;
  {
    hx::KTimer kt(c, "ks_row_inner_f64_kernel", s);
    kern<<<(unsigned)blocks, TILE / 16, smem, s>>>(A);
  }
  launched(c, "ks_row_inner_f64_kernel");
}

void launch_row_inner(hx_ctx* c, const hx::RowInnerArgs& A, cudaStream_t s) {
  switch (c->logn - hx::ntt_split_a(c->logn)) {
    case 3: launch_row_inner_t<3>(c, A, s); break;
    case 4: launch_row_inner_t<4>(c, A, s); break;
    case 5: launch_row_inner_t<5>(c, A, s); break;
    case 6: launch_row_inner_t<6>(c, A, s); break;
    case 7: launch_row_inner_t<7>(c, A, s); break;
    case 8: launch_row_inner_t<8>(c, A, s); break;
    default: throw std::runtime_error("row_inner: unsupported sub-transform size");
  }
}

// The fused ModUp ROW pass + key inner product applies to one uncompressed
// key on the FP64-class limbs (hx_rowinner.cuh); HX_ROWINNER_OFF=1 disables it.
bool row_inner_ok(const hx_ctx* c, int n_q, const std::vector<const u64*>& keys) {
  static const bool off = getenv("HX_ROWINNER_OFF") && atoi(getenv("HX_ROWINNER_OFF")) != 0;
  if (off || !modup_fused_ok(c, n_q) || c->dnum(n_q) > 8 || c->ks_nf64[n_q] == 0) return false;
  for (const u64* k : keys)
    if (c->ckeys.find(k) != c->ckeys.end()) return false;
  return true;
}
bool row_inner_ok(const hx_ctx* c, int n_q, const u64* key) {
  return row_inner_ok(c, n_q, std::vector<const u64*>{key});
}

// rows_deferred: `digits` holds the FP64-class ModUp limbs after their COL
// pass only (modup defer_rows); one key over the batch or one key per E
// elements (!shared), uncompressed keys, identity g, own limbs from c1.
void ks_inner_multi(hx_ctx* c, u64* u, const u64* digits, const std::vector<const u64*>& keys,
                    bool shared, long long E, int n_q, u64 g, cudaStream_t s_main, const u64* c1 = nullptr,
                    long long c1_stride = 0, bool rows_deferred = false) {
  const cudaStream_t s = s_main;
  HX_REQUIRE(!keys.empty() && (int)keys.size() <= hx::kMaxKeys, "ks_inner: 1..64 keys per launch");
  hx::InnerArgs A;
  A.digits = digits;
  A.cmask = 0;
  for (std::size_t r = 0; r < keys.size(); ++r) {
    A.keys[r] = keys[r];
    const auto it = c->ckeys.find(keys[r]);
    A.kseed[r] = 0;
    A.kg[r] = 1;
    if (it != c->ckeys.end()) {
      A.cmask |= 1ull << r;
      A.kseed[r] = it->second.seed;
      A.kg[r] = it->second.kg;
    }
  }
  A.n_keys = (int)keys.size();
  A.shared = shared ? 1 : 0;
  const long long batch = E;
  A.u = u;
  A.pc = c->d_pc;
  A.n_q = n_q;
  A.n_chain = c->n_chain;
  A.n_special = c->n_special;
  A.dnum = c->dnum(n_q);
  A.batch = (int)batch;
  A.g = (hx::u32)g;
  A.logn = c->logn;
  A.c1 = c1;
  A.c1_stride = c1_stride;
  A.alpha = c->alpha;
  const int th = pt_threads(c);
  // split each key's elements over slices: more CTAs in flight, the key words
  // of a (limb, coefficient) are re-read only once per slice
  A.slices = (int)std::max<long long>(1, std::min<long long>(E / 16, 8));
  const unsigned gz = (unsigned)(A.n_keys * A.slices);
  // limbs with q < 2^43 take the FP64 split-MAC kernel (dnum <= 8), the rest
  // (60-bit q_0 and special primes) the 128-bit integer kernel
  const int* lists = c->d_kslimbs + (size_t)n_q * 2 * c->n_total();
  const int nf = A.dnum <= 8 ? c->ks_nf64[n_q] : 0;
  const int ni = A.dnum <= 8 ? c->ks_nint[n_q] : n_q + c->n_special;
  const int* il = A.dnum <= 8 ? lists + c->n_total() : nullptr;
  static const bool one_off = getenv("HX_KS_ONE") && atoi(getenv("HX_KS_ONE")) == 0;
  if (rows_deferred) {
    static_assert(hx::kRowInnerMaxKeys == hx::kMaxKeys, "key table sizes");
    HX_REQUIRE((A.n_keys == 1 || !shared) && A.cmask == 0 && g == 1 && c1 && A.dnum <= 8 && nf > 0,
               "ks_inner: deferred ROW pass needs unshared uncompressed keys, g = 1, own limbs from c1");
    hx::RowInnerArgs R;
    R.digits = digits;
    R.c1 = c1;
    R.c1_stride = c1_stride;
    for (int r = 0; r < A.n_keys; ++r) R.keys[r] = keys[r];
    R.per_key = (int)E;
    R.u = u;
    R.pc = c->d_pc;
    R.limbs = lists;
    R.n_limbs = nf;
    R.n_q = n_q;
    R.n_chain = c->n_chain;
    R.n_special = c->n_special;
    R.dnum = A.dnum;
    R.alpha = c->alpha;
    R.batch = (int)(E * (shared ? 1 : A.n_keys));
    R.logn = c->logn;
    launch_row_inner(c, R, s);
  } else if (nf > 0 && E <= 2 && !one_off) {  // no key reuse across elements: one element per block row
    dim3 grid((unsigned)(A.n_keys * E), (unsigned)nf, (unsigned)(c->N() / th));  // keys fastest, tiles slowest
    if (A.dnum <= 4)
      hx::ks_inner_f64_one_kernel<4><<<grid, th, 0, s>>>(A, lists);
    else
      hx::ks_inner_f64_one_kernel<8><<<grid, th, 0, s>>>(A, lists);
    launched(c, "ks_inner_f64_one_kernel");
  } else if (nf > 0) {
    dim3 grid(gz, (unsigned)nf, (unsigned)(c->N() / th));  // (key, slice) fastest, tiles slowest
    if (A.dnum <= 4)
      hx::ks_inner_f64_kernel<4><<<grid, th, 0, s>>>(A, lists);
    else
      hx::ks_inner_f64_kernel<8><<<grid, th, 0, s>>>(A, lists);
    launched(c, "ks_inner_f64_kernel");
  }
  if (ni > 0) {
    // integer-class limbs: on the side stream when modup forked it
    const cudaStream_t s = rows_deferred && c->side_open ? c->side : s_main;
    dim3 grid(gz, (unsigned)ni, (unsigned)(c->N() / th));  // (key, slice) fastest, tiles slowest
    if (A.dnum <= 1)
      hx::ks_inner_kernel<1><<<grid, th, 0, s>>>(A, il);
    else if (A.dnum <= 2)
      hx::ks_inner_kernel<2><<<grid, th, 0, s>>>(A, il);
    else if (A.dnum <= 4)
      hx::ks_inner_kernel<4><<<grid, th, 0, s>>>(A, il);
    else if (A.dnum <= 8)
      hx::ks_inner_kernel<8><<<grid, th, 0, s>>>(A, il);
    else if (A.dnum <= 16)
      hx::ks_inner_kernel<16><<<grid, th, 0, s>>>(A, il);
    else if (A.dnum <= 32)
      hx::ks_inner_kernel<32><<<grid, th, 0, s>>>(A, il);
    else
      hx::ks_inner_kernel<64><<<grid, th, 0, s>>>(A, il);
    launched(c, "ks_inner_kernel");
  }
  join_side(c, s_main);
}

void ks_inner(hx_ctx* c, u64* u, const u64* digits, const u64* key, long long batch, int n_q,
              u64 g, cudaStream_t s, const u64* c1 = nullptr, long long c1_stride = 0,
              bool rows_deferred = false) {
  ks_inner_multi(c, u, digits, {key}, true, batch, n_q, g, s, c1, c1_stride, rows_deferred);
}

// Centred ModDown of `polys` PQ-basis polys u (stride u_stride words) into
// out (stride out_stride words).  Optionally adds tau_g(add) to the polys with
// index % add_every == 0, using add element (index / add_every) % add_period.
// Output permutation fused into the ModDown combine (rotations): see
// CombineArgs::perm.  g[r] for the r-th group of `per` ciphertexts.
struct OutPerm {
  std::vector<u64> g;
  int per = 1;
  long long rstride = 0, estride = 0;
};

void moddown(hx_ctx* c, u64* out, long long out_stride, const u64* u, long long u_stride,
             long long polys, int n_q, const u64* add, long long add_stride, u64 add_g,
             cudaStream_t s, long long add_every = 1, long long add_period = 0,
             const OutPerm* perm = nullptr) {
  const long long N = c->N();
  const int K = c->n_special;
  DBuf sp(polys * K * N, s, c), conv(polys * n_q * N, s, c);
  hx::ntt_inverse(c, sp.p, polys, hx::make_table(c, 0, K), s, u + (long long)n_q * N, u_stride);  // out of place
  static const bool unfused = getenv("HX_MODDOWN_UNFUSED") != nullptr;
  static const bool col_off = getenv("HX_MODDOWN_COL_OFF") != nullptr;
  const int sa = hx::ntt_split_a(c->logn);
  bool col_done = false;
  if (!unfused && !col_off && K >= 1 && K <= 4 && sa >= 5 && sa <= 8 && c->cs_down[n_q] != 0.0) {
    // conversion P -> Q fused into the forward COL pass of the FP64-class
    // targets (modup_col_kernel, centred mode); integer-class targets are
    // written in the coefficient domain for their ordinary passes
    hx::ModUpColArgs A{};
    A.coef = sp.p;
    A.out = conv.p;
    A.pc = c->d_pc;
    A.qhinv = c->d_phinv;
    A.bc = c->d_mdbc;
    A.tlist = c->d_mdtl;
    A.qh_off[0] = 0;
    A.bc_off[0] = 0;
    A.toff[0] = c->md_tl_off[n_q];
    A.tcnt[0] = c->md_tl_cnt[n_q];
    A.icnt[0] = c->md_tl_icnt[n_q];
    A.alpha = K;
    A.n_q = n_q;
    A.n_chain = c->n_chain;
    A.ext = n_q;
    A.dnum = 1;
    A.logn = c->logn;
    A.src_n = K;
    A.src_pbase = c->n_chain;
    A.centred = 1;
    A.pmf = c->d_pmodqf;
    A.pmf1 = c->d_pmodqf1;
    A.cs_round = c->cs_down[n_q];
    A.pmu = c->d_pmodq;
    HX_REQUIRE(launch_modup_col(c, A, polys, s), "moddown: fused conversion unavailable");
    col_done = true;
  }
  if (!col_done) {
  hx::ModDownArgs M;
  M.sp = sp.p;
  M.conv = conv.p;
  M.pc = c->d_pc;
  M.phinv = c->d_phinv;
  M.pconv = c->d_pconv;
  M.pconvf = c->d_pconvf;
  M.pmodq = c->d_pmodq;
  M.n_q = n_q;
  M.n_chain = c->n_chain;
  M.n_special = K;
  M.logn = c->logn;
  const int th = (int)std::min<long long>(256, N / hx::kModDownEpt);
  dim3 grid((unsigned)(N / th / hx::kModDownEpt), (unsigned)polys);
  const int smem = hx::moddown_smem_bytes(n_q, K);
  HX_REQUIRE(smem <= 48 * 1024, "moddown: too many limbs for the constant stage");
  if (K <= 1)
    hx::moddown_bconv_kernel<1><<<grid, th, smem, s>>>(M);
  else if (K <= 4)
    hx::moddown_bconv_kernel<4><<<grid, th, smem, s>>>(M);
  else
    hx::moddown_bconv_kernel<8><<<grid, th, smem, s>>>(M);
  launched(c, "moddown_bconv_kernel");
  }
  if (!unfused) {  // combine in the ROW pass epilogue of the conversion's NTT
    hx::EpiArgs E{};
    E.u = u;
    E.add = add;
    E.out = out;
    E.pinv = c->d_pinv;
    E.u_stride = u_stride;
    E.out_stride = out_stride;
    E.add_stride = add_stride;
    E.add_every = add_every;
    E.add_period = add_period;
    E.add_g = (hx::u32)add_g;
    E.n_q = n_q;
    E.perm = 0;
    if (perm) {
      HX_REQUIRE(perm->g.size() <= 64 && add_g == 1 && add_every == 2, "fused output permutation");
      E.perm = 1;
      E.per = perm->per;
      E.out_rstride = perm->rstride;
      E.out_estride = perm->estride;
      const u64 two_n = 2 * (u64)N;
      for (std::size_t r = 0; r < perm->g.size(); ++r) {  // g^-1 mod 2N = g^(N-1) (g odd, |Z_2N^*| = N)
        u64 g = perm->g[r] % two_n, inv = 1, e = (u64)N - 1;
        while (e) {
          if (e & 1) inv = inv * g % two_n;
          g = g * g % two_n;
          e >>= 1;
        }
        E.pginv[r] = (hx::u32)inv;
      }
    }
    hx::ntt_forward_combine(c, conv.p, polys, hx::make_table(c, n_q, 0), E, s, col_done);
    return;
  }
  hx::ntt_forward(c, conv.p, polys, hx::make_table(c, n_q, 0), s);
  hx::CombineArgs C;
  C.u = u;
  C.conv = conv.p;
  C.add = add;
  C.out = out;
  C.pc = c->d_pc;
  C.pinv = c->d_pinv;
  C.n_q = n_q;
  C.u_stride = u_stride;
  C.conv_stride = (long long)n_q * N;
  C.out_stride = out_stride;
  C.add_stride = add_stride;
  C.add_every = add_every;
  C.add_period = add_period;
  C.add_g = (hx::u32)add_g;
  C.logn = c->logn;
  C.perm = 0;
  if (perm) {
    HX_REQUIRE(perm->g.size() <= 64 && add_g == 1 && add_every == 2, "fused output permutation");
    C.perm = 1;
    C.per = perm->per;
    C.out_rstride = perm->rstride;
    C.out_estride = perm->estride;
    for (std::size_t r = 0; r < perm->g.size(); ++r) C.pg[r] = (hx::u32)perm->g[r];
  }
  const int cth = combine_threads(c);
  dim3 g3((unsigned)(N / cth / hx::kCombineEpt), (unsigned)n_q, (unsigned)polys);
  hx::combine_kernel<<<g3, cth, 0, s>>>(C);
  launched(c, "combine_kernel");
}

void rescale(hx_ctx* c, u64* out, const u64* in, long long polys, int n_q, cudaStream_t s) {
  const long long N = c->N();
  DBuf last(polys * N, s, c), lift(polys * (n_q - 1) * N, s, c);
  LimbTable lt{};
  lt.count = 1;
  lt.stride = 1;
  lt.off[0] = 0;
  lt.prime[0] = (unsigned char)(n_q - 1);
  hx::ntt_inverse(c, last.p, polys, lt, s, in + (long long)(n_q - 1) * N, (long long)n_q * N);  // out of place
  hx::RescaleArgs R;
  R.last = last.p;
  R.out = lift.p;
  R.pc = c->d_pc;
  R.qlmod = c->d_qlmod + (long long)(n_q - 1) * c->n_chain;
  R.n_q = n_q;
  R.logn = c->logn;
  const int th = pt_threads(c);
  hx::rescale_lift_kernel<<<dim3((unsigned)(N / th), (unsigned)polys), th, 0, s>>>(R);
  launched(c, "rescale_lift_kernel");
  hx::ntt_forward(c, lift.p, polys, hx::make_table(c, n_q - 1, 0), s);
  hx::CombineArgs C;
  C.u = in;
  C.conv = lift.p;
  C.add = nullptr;
  C.out = out;
  C.pc = c->d_pc;
  C.pinv = c->d_qlinv + (long long)(n_q - 1) * c->n_chain;
  C.n_q = n_q - 1;
  C.u_stride = (long long)n_q * N;
  C.conv_stride = (long long)(n_q - 1) * N;
  C.out_stride = (long long)(n_q - 1) * N;
  C.add_stride = 0;
  C.add_every = 1;
  C.add_period = 0;
  C.add_g = 1;
  C.logn = c->logn;
  const int cth = combine_threads(c);
  hx::combine_kernel<<<dim3((unsigned)(N / cth / hx::kCombineEpt), (unsigned)(n_q - 1), (unsigned)polys), cth, 0,
                       s>>>(C);
  launched(c, "combine_kernel");
}

void permute(hx_ctx* c, u64* out, long long out_stride, const u64* in, long long in_stride,
             int limbs, long long batch, u64 g, cudaStream_t s) {
  const int th = pt_threads(c);
  hx::permute_kernel<<<dim3((unsigned)(c->N() / th), (unsigned)limbs, (unsigned)batch), th, 0, s>>>(
      out, out_stride, in, in_stride, (hx::u32)g, c->logn);
  launched(c, "permute_kernel");
}

u64 galois_inverse(u64 g, u64 two_n) {
  // g odd, 2N a power of two: g^-1 = g^(N/2 - 1) (the unit group has exponent N/2)
  u64 r = 1, b = g % two_n, e = two_n / 4 - 1;
  while (e) {
    if (e & 1) r = (u64)(((u128)r * b) % two_n);
    b = (u64)(((u128)b * b) % two_n);
    e >>= 1;
  }
  return r;
}

// Rotations from precomputed ModUp digits with rotation-layout keys
// K' = tau^-1(K):  U' = sum_d D_d (.) K'_d,  W = (c0 + ModDown(U'_0),
// ModDown(U'_1)),  out = tau_g(W) -- bit-identical to (tau(c0) +
// ModDown(sum_d tau(D_d) (.) K_d), ...) because the centred ModDown commutes
// with tau.  R keys at once, E ciphertexts per key:
//   shared (hoisting): every key applies to input cts 0..E-1;
//     output ct (e, r) at out + (e R + r) ct.
//   !shared (independent rotations grouped by key, e.g. the BSGS giant step j
//     of every row block): key r applies to input cts r E .. r E + E - 1;
//     output (r, e) at out + (r E + e) ct.
// One inner-product launch, one ModDown (both ciphertext polys of every
// output), one permutation launch (per 64 keys).
void rotate_batch_from_digits(hx_ctx* c, u64* out, const u64* in, const u64* digits,
                              const std::vector<const u64*>& keys, const std::vector<u64>& galois,
                              bool shared, long long E, int n_q, cudaStream_t s,
                              bool rows_deferred = false) {
  const long long N = c->N(), ct = 2ll * n_q * N;
  HX_REQUIRE(!rows_deferred || !shared || keys.size() == 1, "rotate: deferred ROW pass with shared digits needs one key");
  const int ext = n_q + c->n_special;
  const long long R = (long long)keys.size();
  const long long dstride = (long long)c->dnum(n_q) * ext * N;
  DBuf U(R * E * 2 * ext * N, s, c);
  for (long long r0 = 0; r0 < R; r0 += hx::kMaxKeys) {
    const long long nr = std::min<long long>(hx::kMaxKeys, R - r0);
    const std::vector<const u64*> kk(keys.begin() + r0, keys.begin() + r0 + nr);
    const u64* dg = shared ? digits : digits + r0 * E * dstride;
    const u64* c1 = (shared ? in : in + r0 * E * ct) + (long long)n_q * N;  // own limbs (not copied by ModUp)
    ks_inner_multi(c, U.p + r0 * E * 2 * ext * N, dg, kk, shared, E, n_q, 1, s, c1, ct, rows_deferred);
  }
  // polys p = (r E + e) 2 + c; the c0 polys add input ct (shared ? e : r E + e);
  // the output automorphism tau_{g_r} is fused into the combine (64 keys per call)
  const long long out_rstride = shared ? ct : E * ct, out_estride = shared ? R * ct : ct;
  for (long long r0 = 0; r0 < R; r0 += 64) {
    const long long nr = std::min<long long>(64, R - r0);
    OutPerm P;
    P.g.assign(galois.begin() + r0, galois.begin() + r0 + nr);
    P.per = (int)E;
    P.rstride = out_rstride;
    P.estride = out_estride;
    moddown(c, out + r0 * out_rstride, (long long)n_q * N, U.p + r0 * E * 2 * ext * N, (long long)ext * N,
            nr * E * 2, n_q, shared ? in : in + r0 * E * ct, ct, 1, s, 2, shared ? E : 0, &P);
  }
}

// sum_r tau_{g_r}(in_r) into out (accumulate: out += ...), elements e < E
// of `limbs` limbs (polys of lpoly limbs, the first n_q chain primes)
void perm_sum(hx_ctx* c, u64* out, long long out_estride, const u64* in, long long in_rstride,
              long long in_estride, const std::vector<u64>& g, long long E, int limbs, int lpoly, int n_q,
              bool accumulate, cudaStream_t s) {
  const int th = pt_threads(c);
  for (std::size_t r0 = 0; r0 < g.size(); r0 += hx::kPermSumMax) {
    const int nr = (int)std::min<std::size_t>(hx::kPermSumMax, g.size() - r0);
    hx::PermSumArgs A;
    A.out = out;
    A.out_estride = out_estride;
    A.in = in + (long long)r0 * in_rstride;
    A.in_rstride = in_rstride;
    A.in_estride = in_estride;
    A.pc = c->d_pc;
    A.lpoly = lpoly;
    A.n_q = n_q;
    A.n_chain = c->n_chain;
    A.R = nr;
    A.logn = c->logn;
    A.accumulate = (accumulate || r0) ? 1 : 0;
    for (int r = 0; r < nr; ++r) A.g[r] = (hx::u32)g[r0 + r];
    for (long long e0 = 0; e0 < E; e0 += 65535) {
      const long long ne = std::min<long long>(65535, E - e0);
      hx::PermSumArgs B = A;
      B.out += e0 * out_estride;
      B.in += e0 * in_estride;
      hx::perm_sum_kernel<<<dim3((unsigned)(c->N() / th), (unsigned)limbs, (unsigned)ne), th, 0, s>>>(B);
      launched(c, "perm_sum_kernel");
    }
  }
}

// Host-buffer round trip, pipelined: the batch is cut into chunks; chunk i's
// host->device copy (stream h), compute (stream s) and device->host copy
// (stream d) overlap with chunks i-1 / i+1 on double-buffered device slots.
// Host buffers should be pinned for the copies to run asynchronously.
template <class F>
void pipelined_host(hx_ctx* c, int batch, std::vector<const uint64_t*> in_host,
                    std::vector<long long> in_words, uint64_t* out_host, long long out_words,
                    cudaStream_t s, F compute) {
  // chunks of 8 ciphertexts in a ring of 3 device slots: H2D of chunk i + 2,
  // compute of i + 1 and D2H of i run at once, and pipeline fill / drain is one
  // small chunk (PCIe, ~55 GB/s each way, is the bound of this path)
  static const int chunk_env = [] {
    const char* e = getenv("HX_PIPE_CHUNK");
    return e ? atoi(e) : 0;
  }();
  constexpr int NS = 3;
  const int chunk = std::max(1, std::min(batch, chunk_env > 0 ? chunk_env : 8));
  const int nchunks = (batch + chunk - 1) / chunk;
  // streams, events and the arena slots live in one guard: on every exit path
  // (including a throw from `compute` after copies were queued) all three
  // streams are drained BEFORE the slots return to the arena and the streams /
  // events are destroyed, so no in-flight copy can land in reused memory
  struct Pipe {
    hx_ctx* c;
    cudaStream_t s, h = nullptr, d = nullptr;
    cudaEvent_t ev_in[NS] = {}, ev_cmp[NS] = {}, ev_out[NS] = {};
    std::vector<std::unique_ptr<DBuf>> slots;
    explicit Pipe(hx_ctx* c_, cudaStream_t s_) : c(c_), s(s_) {}
    ~Pipe() {
      if (h) cudaStreamSynchronize(h);
      if (d) cudaStreamSynchronize(d);
      cudaStreamSynchronize(s);
      while (!slots.empty()) slots.pop_back();
      for (int k = 0; k < NS; ++k) {
        if (ev_in[k]) cudaEventDestroy(ev_in[k]);
        if (ev_cmp[k]) cudaEventDestroy(ev_cmp[k]);
        if (ev_out[k]) cudaEventDestroy(ev_out[k]);
      }
      if (h) cudaStreamDestroy(h);
      if (d) cudaStreamDestroy(d);
    }
  } P(c, s);
  cuda_ok(cudaStreamCreateWithFlags(&P.h, cudaStreamNonBlocking), "stream");
  cuda_ok(cudaStreamCreateWithFlags(&P.d, cudaStreamNonBlocking), "stream");
  for (int k = 0; k < NS; ++k) {
    cuda_ok(cudaEventCreateWithFlags(&P.ev_in[k], cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&P.ev_cmp[k], cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&P.ev_out[k], cudaEventDisableTiming), "event");
  }
  cudaStream_t h = P.h, d = P.d;
  // chunk slots from the context arena (released in reverse order by the guard)
  std::vector<u64*> din[NS];
  u64* dout[NS] = {};
  for (int k = 0; k < NS && k < nchunks; ++k) {
    for (long long w : in_words) {
      P.slots.push_back(std::make_unique<DBuf>((size_t)w * chunk, s, c));
      din[k].push_back(P.slots.back()->p);
    }
    P.slots.push_back(std::make_unique<DBuf>((size_t)out_words * chunk, s, c));
    dout[k] = P.slots.back()->p;
  }
  cuda_ok(cudaStreamSynchronize(s), "sync");
  for (int i = 0; i < nchunks; ++i) {
    const int k = i % NS, b0 = i * chunk, n = std::min(chunk, batch - b0);
    if (i >= NS) cuda_ok(cudaStreamWaitEvent(h, P.ev_cmp[k], 0), "wait");  // input slot consumed
    for (std::size_t a = 0; a < in_host.size(); ++a)
      cuda_ok(cudaMemcpyAsync(din[k][a], in_host[a] + (long long)b0 * in_words[a], (size_t)n * in_words[a] * 8,
                              cudaMemcpyHostToDevice, h), "h2d");
    cuda_ok(cudaEventRecord(P.ev_in[k], h), "event record");
    cuda_ok(cudaStreamWaitEvent(s, P.ev_in[k], 0), "wait");
    if (i >= NS) cuda_ok(cudaStreamWaitEvent(s, P.ev_out[k], 0), "wait");  // output slot drained
    compute(dout[k], din[k], n, s);
    cuda_ok(cudaEventRecord(P.ev_cmp[k], s), "event record");
    cuda_ok(cudaStreamWaitEvent(d, P.ev_cmp[k], 0), "wait");
    cuda_ok(cudaMemcpyAsync(out_host + (long long)b0 * out_words, dout[k], (size_t)n * out_words * 8,
                            cudaMemcpyDeviceToHost, d), "d2h");
    cuda_ok(cudaEventRecord(P.ev_out[k], d), "event record");
  }
  cuda_ok(cudaStreamSynchronize(d), "sync");
  cuda_ok(cudaStreamSynchronize(s), "sync");
}

}  // namespace

namespace hx {

void set_error(const std::string& msg) { throw HxError(HX_ERR_UNSUPPORTED, msg); }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

LimbTable make_table(const hx_ctx* c, int n_q, int n_p, int stride, int first) {
  LimbTable lt{};
  lt.count = n_q + n_p;
  lt.stride = stride < 0 ? lt.count : stride;
  HX_REQUIRE(lt.count <= kMaxLimbEntries, "too many limbs");
  for (int k = 0; k < lt.count; ++k) {
    lt.off[k] = (unsigned short)(first + k);
    lt.prime[k] = (unsigned char)c->pidx(k, n_q);
  }
  return lt;
}

}  // namespace hx

// =============================================================================
// C-ABI
// =============================================================================
extern "C" {

const char* hx_last_error(void) { return g_last_error.c_str(); }
const char* hx_version(void) { return "libhx_b200 0.1 (sm_100a)"; }

hx_ctx* hx_ctx_create(int logn, const uint64_t* chain, int n_chain, const uint64_t* special,
                      int n_special, int alpha) {
  hx_ctx* out = nullptr;
  const int rc = guarded([&] {
    HX_REQUIRE(logn >= 8 && logn <= 16, "logn must be in [8, 16]");
    HX_REQUIRE(n_chain >= 1 && n_special >= 1 && n_chain + n_special <= hx::kMaxPrimes,
               "prime counts out of range");
    HX_REQUIRE(alpha >= 1 && alpha <= 8, "alpha must be in [1, 8]");
    int ndev = 0;
    cuda_ok(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    HX_REQUIRE(ndev > 0, "no CUDA device");
    auto c = std::make_unique<hx_ctx>();
    c->logn = logn;
    c->n_chain = n_chain;
    c->n_special = n_special;
    c->alpha = alpha;
    cuda_ok(cudaGetDevice(&c->device), "cudaGetDevice");
    // keep stream-ordered scratch (ModUp digits, ModDown temporaries) cached
    // in the device pool instead of returning it to the OS at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    c->primes.assign(chain, chain + n_chain);
    c->primes.insert(c->primes.end(), special, special + n_special);
    const u64 N = 1ull << logn;
    const int T = c->n_total();
    for (int i = 0; i < T; ++i) {
      const u64 q = c->primes[i];
      HX_REQUIRE(q < (1ull << 62) && q % (2 * N) == 1 && is_prime(q),
                 "modulus must be prime, < 2^62 and = 1 mod 2N");
      for (int j = 0; j < i; ++j) HX_REQUIRE(c->primes[j] != q, "duplicate modulus");
    }
    // twiddles + per-prime constants
    std::vector<ulonglong2> tw((size_t)T * 2 * N);
    std::vector<double> twf((size_t)T * 2 * N, 0.0);
    std::vector<PrimeConst> pc(T);
    const char* force_int = std::getenv("HX_NTT_INT");
    c->allow_f64 = !(force_int && force_int[0] == '1');
    cuda_ok(cudaMalloc((void**)&c->d_tw, tw.size() * sizeof(ulonglong2)), "cudaMalloc(tw)");
    cuda_ok(cudaMalloc((void**)&c->d_twf, twf.size() * sizeof(double)), "cudaMalloc(twf)");
    for (int i = 0; i < T; ++i) {
      const u64 q = c->primes[i];
      const u64 psi = find_psi(q, N), psi_inv = hinv(psi, q);
      c->psi.push_back(psi);
      ulonglong2* f = tw.data() + (size_t)i * 2 * N;
      ulonglong2* g = f + N;
      u64 pw = 1, pwi = 1;
      for (u64 e = 0; e < N; ++e) {
        const u64 k = brv(e, logn);
        f[k] = make_ulonglong2(pw, shoup(pw, q));
        g[k] = make_ulonglong2(pwi, shoup(pwi, q));
        pw = hmul(pw, psi, q);
        pwi = hmul(pwi, psi_inv, q);
      }
      PrimeConst& P = pc[i];
      P.q = q;
      P.two_q = 2 * q;
      P.r64 = (u64)(((u128)1 << 64) % q);
      P.r64p = shoup(P.r64, q);
      P.onep = (u64)(((u128)1 << 64) / q);
      P.ninv = hinv(N % q, q);
      P.ninvp = shoup(P.ninv, q);
      P.w1n = hmul(g[1].x, P.ninv, q);
      P.w1np = shoup(P.w1n, q);
      P.tw_fwd = c->d_tw + (size_t)i * 2 * N;
      P.tw_inv = c->d_tw + (size_t)i * 2 * N + N;
      // FP64 butterfly path for q < 2^47 (exactness bounds in hx_ntt.cuh)
      P.f64 = c->allow_f64 && q < (1ull << 47);
      c->f64.push_back(P.f64 ? 1 : 0);
      const double qd = (double)q;
      P.qd = qd;
      P.qinv_d = 1.0 / qd;
      P.ninv_d = (double)P.ninv;
      P.ninv_q = (double)P.ninv / qd;
      P.w1n_d = (double)P.w1n;
      P.w1n_q = (double)P.w1n / qd;
      P.r20_d = (double)((1ull << 20) % q);
      P.r20_q = P.r20_d / qd;
      P.r40_d = (double)((1ull << 40) % q);
      P.r40_q = P.r40_d / qd;
      P.r24_d = (double)((1ull << 24) % q);
      P.r24_q = P.r24_d / qd;
      P.r48_d = (double)((1ull << 48) % q);
      P.r48_q = P.r48_d / qd;
      double* ff = twf.data() + (size_t)i * 2 * N;
      if (P.f64)
        for (u64 k = 0; k < 2 * N; ++k) ff[k] = (double)(k < N ? f[k] : g[k - N]).x;
      P.twf_fwd = c->d_twf + (size_t)i * 2 * N;
      P.twf_inv = c->d_twf + (size_t)i * 2 * N + N;
    }
    cuda_ok(cudaMemcpy(c->d_tw, tw.data(), tw.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice),
            "upload tw");
    cuda_ok(cudaMemcpy(c->d_twf, twf.data(), twf.size() * sizeof(double), cudaMemcpyHostToDevice),
            "upload twf");
    c->d_pc = upload(pc);
    // ModUp constants per (n_q, digit)
    std::vector<SC> mu;
    c->modup_qh_off.assign(n_chain + 1, {});
    c->modup_cv_off.assign(n_chain + 1, {});
    for (int nq = 1; nq <= n_chain; ++nq) {
      const int dn = c->dnum(nq);
      for (int d = 0; d < dn; ++d) {
        const int lo = d * alpha, cnt = std::min(alpha, nq - lo);
        c->modup_qh_off[nq].push_back((long long)mu.size());
        for (int i = lo; i < lo + cnt; ++i) {
          const u64 q = c->primes[i];
          u64 prod = 1;
          for (int i2 = lo; i2 < lo + cnt; ++i2)
            if (i2 != i) prod = hmul(prod, c->primes[i2] % q, q);
          mu.push_back(sc(hinv(prod, q), q));
        }
        c->modup_cv_off[nq].push_back((long long)mu.size());
        for (int i = lo; i < lo + cnt; ++i) {
          for (int p = 0; p < T; ++p) {
            const u64 m = c->primes[p];
            u64 prod = 1;
            for (int i2 = lo; i2 < lo + cnt; ++i2)
              if (i2 != i) prod = hmul(prod, c->primes[i2] % m, m);
            mu.push_back(sc(prod, m));
          }
        }
      }
    }
    c->d_modup = upload(mu);
    // Fused ModUp (hx_modup.cuh): conversion constants per (n_q, digit) as
    // [ext][alpha] BconvC and per-class target limb lists per (n_q, digit)
    {
      std::vector<hx::BconvC> bc;
      std::vector<int> tl;
      c->bc_off.assign(n_chain + 1, {});
      c->tl_off.assign(n_chain + 1, {});
      c->tl_cnt.assign(n_chain + 1, {});
      c->tl_icnt.assign(n_chain + 1, {});
      for (int nq = 1; nq <= n_chain; ++nq) {
        const int dn = c->dnum(nq), ext = nq + n_special;
        for (int d = 0; d < dn; ++d) {
          const int lo = d * alpha, cnt = std::min(alpha, nq - lo);
          c->bc_off[nq].push_back((long long)bc.size());
          for (int j = 0; j < ext; ++j) {
            const int pj = c->pidx(j, nq);
            const u64 m = c->primes[pj];
            for (int ii = 0; ii < alpha; ++ii) {
              hx::BconvC e{};
              if (ii < cnt) {
                const int i = lo + ii;
                u64 prod = 1;
                for (int i2 = lo; i2 < lo + cnt; ++i2)
                  if (i2 != i) prod = hmul(prod, c->primes[i2] % m, m);
                const SC w = sc(prod, m);
                const u64 w30 = hmul(prod, (1ull << 30) % m, m);
                e.w = (double)prod;
                e.wq = (double)prod / (double)m;
                e.w30 = (double)w30;
                e.w30q = (double)w30 / (double)m;
                e.sw = w.w;
                e.swp = w.wp;
                // premultiplied by the target's first forward twiddle psi^(N/2)
                const u64 tw1 = hpow(c->psi[pj], N / 2, m);
                const SC w1 = sc(hmul(prod, tw1, m), m);
                e.w1 = (double)w1.w;
                e.w301 = (double)hmul(w30, tw1, m);
                e.sw1 = w1.w;
                e.swp1 = w1.wp;
              }
              bc.push_back(e);
            }
          }
          c->tl_off[nq].push_back((int)tl.size());
          for (int cls = 0; cls < 2; ++cls) {  // FP64-class targets first, then integer ones
            int n = 0;
            for (int j = 0; j < ext; ++j) {
              if (j >= lo && j < lo + cnt) continue;
              if ((c->f64[c->pidx(j, nq)] != 0) != (cls == 0)) continue;
              tl.push_back(j);
              ++n;
            }
            (cls == 0 ? c->tl_cnt : c->tl_icnt)[nq].push_back(n);
          }
        }
      }
      c->d_bconv = upload(bc);
      c->d_tlist = upload(tl);
    }
    // ModDown constants
    std::vector<SC> phinv(n_special), pconv((size_t)n_special * n_chain), pinv(n_chain);
    std::vector<u64> pmodq(n_chain);
    for (int k = 0; k < n_special; ++k) {
      const u64 pk = c->primes[n_chain + k];
      u64 prod = 1;
      for (int k2 = 0; k2 < n_special; ++k2)
        if (k2 != k) prod = hmul(prod, c->primes[n_chain + k2] % pk, pk);
      phinv[k] = sc(hinv(prod, pk), pk);
      for (int i = 0; i < n_chain; ++i) {
        const u64 q = c->primes[i];
        u64 pr = 1;
        for (int k2 = 0; k2 < n_special; ++k2)
          if (k2 != k) pr = hmul(pr, c->primes[n_chain + k2] % q, q);
        pconv[(size_t)k * n_chain + i] = sc(pr, q);
      }
    }
    for (int i = 0; i < n_chain; ++i) {
      const u64 q = c->primes[i];
      u64 P = 1;
      for (int k = 0; k < n_special; ++k) P = hmul(P, c->primes[n_chain + k] % q, q);
      pmodq[i] = P;
      pinv[i] = sc(hinv(P, q), q);
    }
    c->d_phinv = upload(phinv);
    c->d_pconv = upload(pconv);
    c->d_pmodq = upload(pmodq);
    // FP64 form of the P -> Q conversion constants: [k][i] -> (w, w/q, w30, w30/q)
    {
      std::vector<double> pf((size_t)n_special * n_chain * 4);
      for (int k = 0; k < n_special; ++k)
        for (int i = 0; i < n_chain; ++i) {
          const u64 q = c->primes[i], w = pconv[(size_t)k * n_chain + i].w;
          const u64 w30 = hmul(w, (1ull << 30) % q, q);
          double* e = pf.data() + ((size_t)k * n_chain + i) * 4;
          e[0] = (double)w;
          e[1] = (double)w / (double)q;
          e[2] = (double)w30;
          e[3] = (double)w30 / (double)q;
        }
      c->d_pconvf = upload(pf);
    }
    {  // fused ModDown conversion + COL pass tables (modup_col_kernel, centred)
      std::vector<hx::BconvC> mb((size_t)n_chain * n_special);
      std::vector<double> pmf(n_chain), pmf1(n_chain);
      for (int j = 0; j < n_chain; ++j) {
        const u64 q = c->primes[j];
        pmf[j] = (double)pmodq[j];
        const u64 tw1 = hpow(c->psi[j], N / 2, q);  // first forward twiddle
        pmf1[j] = (double)hmul(pmodq[j], tw1, q);
        for (int k = 0; k < n_special; ++k) {
          const SC w = pconv[(size_t)k * n_chain + j];
          const u64 w30 = hmul(w.w, (1ull << 30) % q, q);
          hx::BconvC& e = mb[(size_t)j * n_special + k];
          e.w = (double)w.w;
          e.wq = (double)w.w / (double)q;
          e.w30 = (double)w30;
          e.w30q = (double)w30 / (double)q;
          e.sw = w.w;
          e.swp = w.wp;
          const SC w1 = sc(hmul(w.w, tw1, q), q);
          e.w1 = (double)w1.w;
          e.w301 = (double)hmul(w30, tw1, q);
          e.sw1 = w1.w;
          e.swp1 = w1.wp;
        }
      }
      std::vector<int> tl;
      c->md_tl_off.assign(n_chain + 1, 0);
      c->md_tl_cnt.assign(n_chain + 1, 0);
      c->md_tl_icnt.assign(n_chain + 1, 0);
      for (int nq = 1; nq <= n_chain; ++nq) {
        c->md_tl_off[nq] = (int)tl.size();
        for (int cls = 0; cls < 2; ++cls)
          for (int j = 0; j < nq; ++j) {
            if ((c->f64[j] != 0) != (cls == 0)) continue;
            tl.push_back(j);
            ++(cls == 0 ? c->md_tl_cnt : c->md_tl_icnt)[nq];
          }
      }
      c->d_mdbc = upload(mb);
      c->d_mdtl = upload(tl);
      c->d_pmodqf = upload(pmf);
      c->d_pmodqf1 = upload(pmf1);
      // rounding constants of the joint conversion (hx_modup.cuh bconv_tile_f64)
      c->cs_up.assign(n_chain + 1, 0.0);
      c->cs_down.assign(n_chain + 1, 0.0);
      for (int nq = 1; nq <= n_chain; ++nq) {
        std::vector<int> tg, sr;
        const int dn = c->dnum(nq);
        double up = -1.0;
        for (int d = 0; d < dn && up != 0.0; ++d) {
          const int lo = d * alpha, cnt = std::min(alpha, nq - lo);
          tg.clear();
          sr.clear();
          for (int i = lo; i < lo + cnt; ++i) sr.push_back(i);
          for (int j = 0; j < nq + n_special; ++j)
            if (!(j >= lo && j < lo + cnt) && c->f64[c->pidx(j, nq)]) tg.push_back(c->pidx(j, nq));
          if (tg.empty()) continue;
          const double r = bconv_round(c.get(), sr, tg, 0);
          up = (r == 0.0) ? 0.0 : std::max(up, r);
        }
        c->cs_up[nq] = up < 0.0 ? 1.0 : up;  // no FP64-class target at all: unused
        tg.clear();
        sr.clear();
        for (int k = 0; k < n_special; ++k) sr.push_back(n_chain + k);
        for (int j = 0; j < nq; ++j)
          if (c->f64[j]) tg.push_back(j);
        c->cs_down[nq] = tg.empty() ? 1.0 : bconv_round(c.get(), sr, tg, n_special);
      }
    }
    c->d_pinv = upload(pinv);
    // Rescale constants
    std::vector<SC> qlinv((size_t)n_chain * n_chain, SC{0, 0});
    std::vector<u64> qlmod((size_t)n_chain * n_chain, 0);
    for (int l = 1; l < n_chain; ++l)
      for (int i = 0; i < l; ++i) {
        const u64 q = c->primes[i], ql = c->primes[l];
        qlinv[(size_t)l * n_chain + i] = sc(hinv(ql % q, q), q);
        qlmod[(size_t)l * n_chain + i] = ql % q;
      }
    c->d_qlinv = upload(qlinv);
    c->d_qlmod = upload(qlmod);
    // BSGS MAC limb classes: FP64 k-split kernel for q < 2^43, integer otherwise
    std::vector<int> ml((size_t)(n_chain + 1) * 2 * n_chain, 0);
    c->mac_nf64.assign(n_chain + 1, 0);
    c->mac_nint.assign(n_chain + 1, 0);
    for (int nq = 1; nq <= n_chain; ++nq) {
      int* f = ml.data() + (size_t)nq * 2 * n_chain;
      int* g = f + n_chain;
      for (int i = 0; i < nq; ++i) {
        if (c->allow_f64 && c->primes[i] < (1ull << 43))
          f[c->mac_nf64[nq]++] = i;
        else
          g[c->mac_nint[nq]++] = i;
      }
    }
    c->d_maclimbs = upload(ml);
    std::vector<int> kl((size_t)(n_chain + 1) * 2 * T, 0);
    c->ks_nf64.assign(n_chain + 1, 0);
    c->ks_nint.assign(n_chain + 1, 0);
    for (int nq = 1; nq <= n_chain; ++nq) {
      int* f = kl.data() + (size_t)nq * 2 * T;
      int* g = f + T;
      for (int j = 0; j < nq + n_special; ++j) {
        if (c->allow_f64 && c->primes[c->pidx(j, nq)] < (1ull << 47))  // 24-bit split inner product
          f[c->ks_nf64[nq]++] = j;
        else
          g[c->ks_nint[nq]++] = j;
      }
    }
    c->d_kslimbs = upload(kl);
    out = c.release();
  });
  return rc == HX_OK ? out : nullptr;
}

void hx_ctx_destroy(hx_ctx* c) {
  if (!c) return;
  for (void* p : {(void*)c->d_pc, (void*)c->d_tw, (void*)c->d_twf, (void*)c->d_modup, (void*)c->d_phinv,
                  (void*)c->d_pconvf,
                  (void*)c->d_pconv, (void*)c->d_pmodq, (void*)c->d_pinv, (void*)c->d_qlinv,
                  (void*)c->d_qlmod, (void*)c->d_maclimbs, (void*)c->d_kslimbs, (void*)c->d_bconv,
                  (void*)c->d_tlist, (void*)c->d_mdbc, (void*)c->d_mdtl, (void*)c->d_pmodqf,
                  (void*)c->d_pmodqf1})
    if (p) cudaFree(p);
  if (c->arena.base) {
    cudaDeviceSynchronize();
    cudaFree(c->arena.base);
  }
  if (c->arena.ev) cudaEventDestroy(c->arena.ev);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
  }
  delete c;
}

int hx_ctx_trim(hx_ctx* c) {
  return guarded([&] {
    check_ctx(c);
    HxArena& A = c->arena;
    HX_REQUIRE(A.depth == 0, "hx_ctx_trim: scratch in use");
    cuda_ok(cudaDeviceSynchronize(), "sync");
    if (A.base) cuda_ok(cudaFree(A.base), "cudaFree(arena)");
    A.base = nullptr;
    A.cap = A.high = A.top = 0;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  });
}

int hx_ctx_dnum(const hx_ctx* c, int n_q) { return c ? c->dnum(n_q) : -1; }
uint64_t hx_ctx_psi(const hx_ctx* c, int i) {
  return (c && i >= 0 && i < c->n_total()) ? c->psi[i] : 0;
}
size_t hx_key_words(const hx_ctx* c) {
  return c ? (size_t)c->dnum(c->n_chain) * 2 * c->n_total() * c->N() : 0;
}
unsigned long long hx_ctx_launches(const hx_ctx* c) { return c ? c->launches : 0; }

int hx_malloc(void** p, size_t bytes) {
  return guarded([&] { cuda_ok(cudaMalloc(p, bytes), "cudaMalloc"); });
}
int hx_free(void* p) {
  return guarded([&] { cuda_ok(cudaFree(p), "cudaFree"); });
}
int hx_memcpy_h2d(void* dst, const void* src, size_t bytes, void* s) {
  return guarded(
      [&] { cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(s)), "h2d"); });
}
int hx_memcpy_d2h(void* dst, const void* src, size_t bytes, void* s) {
  return guarded(
      [&] { cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(s)), "d2h"); });
}
int hx_memcpy_d2d(void* dst, const void* src, size_t bytes, void* s) {
  return guarded(
      [&] { cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(s)), "d2d"); });
}
int hx_stream_sync(void* s) {
  return guarded([&] { cuda_ok(cudaStreamSynchronize(S(s)), "cudaStreamSynchronize"); });
}
int hx_device_sync(void) {
  return guarded([&] { cuda_ok(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); });
}

int hx_ntt_fwd(hx_ctx* c, uint64_t* data, int batch, int n_q, int n_p, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    HX_REQUIRE(n_q >= 0 && n_q <= c->n_chain && n_p >= 0 && n_p <= c->n_special && n_q + n_p >= 1, "limbs");
    hx::ntt_forward(c, (u64*)data, batch, hx::make_table(c, n_q, n_p), S(s));
    cuda_ok(cudaGetLastError(), "ntt_forward");
  });
}

int hx_ntt_inv(hx_ctx* c, uint64_t* data, int batch, int n_q, int n_p, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    HX_REQUIRE(n_q >= 0 && n_q <= c->n_chain && n_p >= 0 && n_p <= c->n_special && n_q + n_p >= 1, "limbs");
    hx::ntt_inverse(c, (u64*)data, batch, hx::make_table(c, n_q, n_p), S(s));
    cuda_ok(cudaGetLastError(), "ntt_inverse");
  });
}

#define HX_EW_ENTRY(NAME, OP)                                                                 \
  int NAME(hx_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, int batch, int n_q, \
           int n_p, void* s) {                                                                \
    return guarded([&] {                                                                      \
      check_ctx(c);                                                                           \
      HX_COUNT(batch);                                                                        \
      ew<OP>(c, (u64*)out, (const u64*)a, (const u64*)b, batch, hx::make_table(c, n_q, n_p),   \
             S(s));                                                                           \
    });                                                                                       \
  }
HX_EW_ENTRY(hx_add, hx::EwOp::Add)
HX_EW_ENTRY(hx_sub, hx::EwOp::Sub)
HX_EW_ENTRY(hx_mul, hx::EwOp::Mul)
#undef HX_EW_ENTRY

int hx_mul_bcast(hx_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, int batch, int a_mod,
                 int b_div, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    HX_REQUIRE(a_mod >= 0 && b_div >= 1, "mul_bcast: a_mod >= 0, b_div >= 1");
    ew<hx::EwOp::Mul>(c, (u64*)out, (const u64*)a, (const u64*)b, batch, hx::make_table(c, n_q, 0), S(s), a_mod,
                      b_div);
  });
}

int hx_mul_acc(hx_ctx* c, uint64_t* acc, const uint64_t* a, const uint64_t* b, int batch, int n_q,
               int n_p, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    ew<hx::EwOp::MulAcc>(c, (u64*)acc, (const u64*)a, (const u64*)b, batch,
                         hx::make_table(c, n_q, n_p), S(s));
  });
}

int hx_neg(hx_ctx* c, uint64_t* out, const uint64_t* a, int batch, int n_q, int n_p, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    ew<hx::EwOp::Neg>(c, (u64*)out, (const u64*)a, nullptr, batch, hx::make_table(c, n_q, n_p),
                      S(s));
  });
}

int hx_automorphism(hx_ctx* c, uint64_t* out, const uint64_t* in, int batch, int n_q, int n_p,
                    uint64_t g, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element must be odd and < 2N");
    HX_REQUIRE(out != in, "automorphism cannot run in place");
    automorphism(c, (u64*)out, (const u64*)in, batch, hx::make_table(c, n_q, n_p), g, S(s));
  });
}

int hx_from_i64(hx_ctx* c, uint64_t* out, const int64_t* v, int batch, int n_q, int n_p,
                void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    const LimbTable lt = hx::make_table(c, n_q, n_p);
    const int th = pt_threads(c);
    const long long blocks = (long long)batch * lt.count * (c->N() / th);
    if (blocks <= 0) return;
    hx::from_i64_kernel<<<(unsigned)blocks, th, 0, S(s)>>>((u64*)out, (const long long*)v,
                                                            c->d_pc, lt, c->logn);
    launched(c, "from_i64_kernel");
  });
}

int hx_reduce_mod_q(hx_ctx* c, uint64_t* data, int batch, int n_q, int n_p, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    hx::EwArgs A{(u64*)data, nullptr, nullptr, c->d_pc, hx::make_table(c, n_q, n_p), c->logn, 0};
    A.instances = (long long)batch * A.lt.count;
    const int th = pt_threads(c);
    const long long blocks = A.instances * (c->N() / th);
    if (blocks <= 0) return;
    hx::reduce_kernel<<<(unsigned)blocks, th, 0, S(s)>>>(A);
    launched(c, "reduce_kernel");
  });
}

int hx_rescale(hx_ctx* c, uint64_t* out, const uint64_t* in, int batch, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    HX_REQUIRE(n_q >= 2, "rescale: no limb to drop");
    rescale(c, (u64*)out, (const u64*)in, batch, n_q, S(s));
  });
}

int hx_modup(hx_ctx* c, uint64_t* digits, const uint64_t* c1, int batch, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    modup(c, (u64*)digits, (const u64*)c1, (long long)n_q * c->N(), batch, n_q, S(s));
  });
}

int hx_ks_inner(hx_ctx* c, uint64_t* u, const uint64_t* digits, const uint64_t* key, int batch,
                int n_q, uint64_t g, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element must be odd and < 2N");
    ks_inner(c, (u64*)u, (const u64*)digits, (const u64*)key, batch, n_q, g, S(s));
  });
}

int hx_moddown(hx_ctx* c, uint64_t* out, const uint64_t* u, int polys, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(polys);
    check_nq(c, n_q);
    const long long N = c->N();
    moddown(c, (u64*)out, (long long)n_q * N, (const u64*)u, (long long)(n_q + c->n_special) * N,
            polys, n_q, nullptr, 0, 1, S(s));
  });
}

int hx_keyswitch(hx_ctx* c, uint64_t* out, const uint64_t* in, const uint64_t* key, int batch,
                 int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    const long long N = c->N();
    const int ext = n_q + c->n_special;
    DBuf D((long long)batch * c->dnum(n_q) * ext * N, S(s), c), U((long long)batch * 2 * ext * N, S(s), c);
    const bool fuse = row_inner_ok(c, n_q, (const u64*)key);
    modup(c, D.p, (const u64*)in, (long long)n_q * N, batch, n_q, S(s), false, fuse);
    ks_inner(c, U.p, D.p, (const u64*)key, batch, n_q, 1, S(s), (const u64*)in, (long long)n_q * N, fuse);
    moddown(c, (u64*)out, (long long)n_q * N, U.p, (long long)ext * N, 2ll * batch, n_q, nullptr,
            0, 1, S(s));
  });
}

int hx_rotate(hx_ctx* c, uint64_t* out, const uint64_t* in, const uint64_t* key, int batch,
              int n_q, uint64_t g, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element must be odd and < 2N");
    HX_REQUIRE(out != in, "rotate cannot run in place");
    const long long N = c->N();
    const int ext = n_q + c->n_special;
    DBuf D((long long)batch * c->dnum(n_q) * ext * N, S(s), c);
    const bool fuse = row_inner_ok(c, n_q, (const u64*)key);
    modup(c, D.p, (const u64*)in + (long long)n_q * N, 2ll * n_q * N, batch, n_q, S(s), false, fuse);
    rotate_batch_from_digits(c, (u64*)out, (const u64*)in, D.p, {(const u64*)key}, {g}, true, batch,
                             n_q, S(s), fuse);
  });
}

int hx_rotate_hoisted(hx_ctx* c, uint64_t* out, const uint64_t* in, const uint64_t* const* keys,
                      const uint64_t* galois, int R, int batch, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    HX_REQUIRE(R >= 1, "R >= 1");
    const long long N = c->N();
    const int ext = n_q + c->n_special;
    DBuf D((long long)batch * c->dnum(n_q) * ext * N, S(s), c);
    modup(c, D.p, (const u64*)in + (long long)n_q * N, 2ll * n_q * N, batch, n_q, S(s), false);
    std::vector<const u64*> kk;
    std::vector<u64> gg;
    for (int r = 0; r < R; ++r) {
      HX_REQUIRE((galois[r] & 1) && galois[r] < 2 * (u64)N, "galois element");
      kk.push_back((const u64*)keys[r]);
      gg.push_back(galois[r]);
    }
    rotate_batch_from_digits(c, (u64*)out, (const u64*)in, D.p, kk, gg, true, batch, n_q, S(s));
  });
}

int hx_rotate_multi(hx_ctx* c, uint64_t* out, const uint64_t* in, const uint64_t* const* keys,
                    const uint64_t* galois, int batch, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    const long long N = c->N(), ct = 2ll * n_q * N;
    const int ext = n_q + c->n_special;
    const long long dstride = (long long)c->dnum(n_q) * ext * N;
    for (int b = 0; b < batch; ++b)
      HX_REQUIRE((galois[b] & 1) && galois[b] < 2 * (u64)N, "galois element");
    DBuf D((long long)batch * dstride, S(s), c);
    std::vector<const u64*> kk;
    std::vector<u64> gg;
    for (int b = 0; b < batch; ++b) {
      kk.push_back((const u64*)keys[b]);
      gg.push_back((u64)galois[b]);
    }
    const bool fuse = batch > 0 && row_inner_ok(c, n_q, kk);
    modup(c, D.p, (const u64*)in + (long long)n_q * N, ct, batch, n_q, S(s), false, fuse);
    rotate_batch_from_digits(c, (u64*)out, (const u64*)in, D.p, kk, gg, false, 1, n_q, S(s), fuse);
  });
}

int hx_rotate_grouped(hx_ctx* c, uint64_t* out, const uint64_t* in, const uint64_t* const* keys,
                      const uint64_t* galois, int R, int E, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(R);
    HX_COUNT(E);
    check_nq(c, n_q);
    HX_REQUIRE(R >= 1 && E >= 1, "R, E >= 1");
    const long long N = c->N(), ct = 2ll * n_q * N;
    const int ext = n_q + c->n_special;
    std::vector<const u64*> kk;
    std::vector<u64> gg;
    for (int r = 0; r < R; ++r) {
      HX_REQUIRE((galois[r] & 1) && galois[r] < 2 * (u64)N, "galois element");
      kk.push_back((const u64*)keys[r]);
      gg.push_back((u64)galois[r]);
    }
    // keys in chunks so the ModUp digits + inner products of a chunk stay
    // within ~16 GB (T tokens x blocks elements per key multiply them)
    const long long per_key = (long long)E * (c->dnum(n_q) + 2) * ext * N * 8;
    const int Rc = (int)std::max(1ll, std::min<long long>(R, (16ll << 30) / per_key));
    for (int r0 = 0; r0 < R; r0 += Rc) {
      const int nr = std::min(Rc, R - r0);
      const u64* ip = (const u64*)in + (long long)r0 * E * ct;
      DBuf D((long long)nr * E * c->dnum(n_q) * ext * N, S(s), c);
      const std::vector<const u64*> kc(kk.begin() + r0, kk.begin() + r0 + nr);
      const std::vector<u64> gc(gg.begin() + r0, gg.begin() + r0 + nr);
      const bool fuse = row_inner_ok(c, n_q, kc);
      modup(c, D.p, ip + (long long)n_q * N, ct, (long long)nr * E, n_q, S(s), false, fuse);
      rotate_batch_from_digits(c, (u64*)out + (long long)r0 * E * ct, ip, D.p, kc, gc, false, E, n_q, S(s),
                               fuse);
    }
  });
}

int hx_rotate_grouped_sum(hx_ctx* c, uint64_t* out, uint64_t* pq_partial, const uint64_t* in,
                          const uint64_t* base, const uint64_t* const* keys, const uint64_t* galois, int R, int E,
                          int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(R);
    HX_COUNT(E);
    check_nq(c, n_q);
    HX_REQUIRE(R >= 0 && E >= 1, "R >= 0, E >= 1");
    const long long N = c->N(), ct = 2ll * n_q * N;
    const int K = c->n_special, ext = n_q + K;
    const long long uw = 2ll * ext * N;  // one PQ-basis key-switch product (2 polys)
    for (int r = 0; r < R; ++r)
      HX_REQUIRE((galois[r] & 1) && galois[r] < 2 * (u64)N, "galois element");
    // T = base + sum_r tau_r(c0_r) (c1 part: base's), S = sum_r tau_r(U'_r)
    DBuf Tb(pq_partial ? 0 : E * ct, S(s), c), Sb(pq_partial ? 0 : E * uw, S(s), c);
    u64* T = pq_partial ? (u64*)out : Tb.p;
    u64* Sp = pq_partial ? (u64*)pq_partial : Sb.p;
    if (base)
      cuda_ok(cudaMemcpyAsync(T, base, (size_t)(E * ct) * 8, cudaMemcpyDeviceToDevice, S(s)), "d2d");
    else
      cuda_ok(cudaMemsetAsync(T, 0, (size_t)(E * ct) * 8, S(s)), "memset");
    cuda_ok(cudaMemsetAsync(Sp, 0, (size_t)(E * uw) * 8, S(s)), "memset");
    // keys in chunks so the ModUp digits + products of a chunk stay within ~16 GB
    const long long per_key = (long long)E * (c->dnum(n_q) + 2) * ext * N * 8;
    const int Rc = (int)std::max(1ll, std::min<long long>(std::max(R, 1), (16ll << 30) / per_key));
    for (int r0 = 0; r0 < R; r0 += Rc) {
      const int nr = std::min(Rc, R - r0);
      const u64* ip = (const u64*)in + (long long)r0 * E * ct;
      std::vector<const u64*> kc;
      std::vector<u64> gc;
      for (int r = r0; r < r0 + nr; ++r) {
        kc.push_back((const u64*)keys[r]);
        gc.push_back((u64)galois[r]);
      }
      DBuf D((long long)nr * E * c->dnum(n_q) * ext * N, S(s), c);
      DBuf U((long long)nr * E * uw, S(s), c);
      const bool fuse = row_inner_ok(c, n_q, kc);
      modup(c, D.p, ip + (long long)n_q * N, ct, (long long)nr * E, n_q, S(s), false, fuse);
      const long long dstride = (long long)c->dnum(n_q) * ext * N;
      for (int k0 = 0; k0 < nr; k0 += hx::kMaxKeys) {
        const int nk = std::min(hx::kMaxKeys, nr - k0);
        const std::vector<const u64*> kk(kc.begin() + k0, kc.begin() + k0 + nk);
        ks_inner_multi(c, U.p + (long long)k0 * E * uw, D.p + (long long)k0 * E * dstride, kk, false, E, n_q, 1,
                       S(s), ip + (long long)k0 * E * ct + (long long)n_q * N, ct, fuse);
      }
      // rotation-layout keys: U' = tau_r^-1(U_r), so tau_r(U'_r) is the product of the rotation
      perm_sum(c, Sp, uw, U.p, E * uw, uw, gc, E, 2 * ext, ext, n_q, true, S(s));
      perm_sum(c, T, ct, ip, E * ct, ct, gc, E, n_q, n_q, n_q, true, S(s));
    }
    if (pq_partial) return;
    // one ModDown per output ciphertext: out = T + (ModDown(S_0), ModDown(S_1))
    moddown(c, (u64*)out, (long long)n_q * N, Sp, (long long)ext * N, 2 * E, n_q, T, (long long)n_q * N, 1,
            S(s), 1, 0, nullptr);
  });
}

int hx_moddown_add(hx_ctx* c, uint64_t* out, const uint64_t* pq, const uint64_t* add, int E, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(E);
    check_nq(c, n_q);
    if (!E) return;
    const long long N = c->N();
    const int ext = n_q + c->n_special;
    moddown(c, (u64*)out, (long long)n_q * N, (const u64*)pq, (long long)ext * N, 2ll * E, n_q, (const u64*)add,
            add ? (long long)n_q * N : 0, 1, S(s), 1, 0, nullptr);
  });
}

int hx_tensor(hx_ctx* c, uint64_t* out3, const uint64_t* a, const uint64_t* b, int batch, int n_q,
              void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    const int th = pt_threads(c);
    hx::tensor_kernel<<<dim3((unsigned)(c->N() / th), (unsigned)n_q, (unsigned)batch), th, 0,
                        S(s)>>>((u64*)out3, (const u64*)a, (const u64*)b, c->d_pc, n_q, c->logn);
    launched(c, "tensor_kernel");
  });
}

int hx_mul_relin(hx_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b,
                 const uint64_t* rlk, int batch, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    const long long N = c->N(), L = (long long)n_q * N;
    const int ext = n_q + c->n_special;
    DBuf d3((long long)batch * 3 * L, S(s), c), D((long long)batch * c->dnum(n_q) * ext * N, S(s), c),
        U((long long)batch * 2 * ext * N, S(s), c);
    const int th = pt_threads(c);
    hx::tensor_kernel<<<dim3((unsigned)(N / th), (unsigned)n_q, (unsigned)batch), th, 0, S(s)>>>(
        d3.p, (const u64*)a, (const u64*)b, c->d_pc, n_q, c->logn);
    launched(c, "tensor_kernel");
    const bool fuse = row_inner_ok(c, n_q, (const u64*)rlk);
    modup(c, D.p, d3.p + 2 * L, 3 * L, batch, n_q, S(s), false, fuse);
    ks_inner(c, U.p, D.p, (const u64*)rlk, batch, n_q, 1, S(s), d3.p + 2 * L, 3 * L, fuse);
    moddown(c, (u64*)out, 2 * L, U.p, 2ll * ext * N, batch, n_q, d3.p, 3 * L, 1, S(s));
    moddown(c, (u64*)out + L, 2 * L, U.p + (long long)ext * N, 2ll * ext * N, batch, n_q,
            d3.p + L, 3 * L, 1, S(s));
  });
}

int hx_bsgs_mac_tokens(hx_ctx* c, uint64_t* inner, long long inner_jstride, long long inner_tstride,
                       const uint64_t* baby, long long baby_tstride, const uint64_t* diags, int diag_limbs, int n1,
                       int n2, int n_q, int tokens, int diag_jstride, void* s) {
  return guarded([&] {
    check_ctx(c);
    check_nq(c, n_q);
    HX_REQUIRE(n1 >= 1 && n1 <= 64 && n2 >= 1 && diag_limbs >= n_q && tokens >= 1, "bsgs_mac: bad shape");
    HX_REQUIRE((long long)tokens * (c->N() / 32) < (1ll << 31), "bsgs_mac: too many tokens");
    hx::MacArgs A;
    A.inner = (u64*)inner;
    A.baby = (const u64*)baby;
    A.diags = (const u64*)diags;
    A.pc = c->d_pc;
    A.n1 = n1;
    A.n2 = n2;
    A.n_q = n_q;
    A.logn = c->logn;
    A.diag_stride = (long long)diag_limbs * c->N();
    A.out_jstride = inner_jstride;
    A.limbs = nullptr;
    A.tokens = tokens;
    A.baby_tstride = baby_tstride;
    A.inner_tstride = inner_tstride;
    HX_REQUIRE(diag_jstride == 0 || diag_jstride >= n1, "bsgs_mac: diag_jstride < n1");
    A.diag_jstride = diag_jstride ? diag_jstride : n1;
    const int* lists = c->d_maclimbs + (size_t)n_q * 2 * c->n_chain;
    hx::launch_bsgs_mac(A, c->N(), S(s), lists, c->mac_nf64[n_q], lists + c->n_chain, c->mac_nint[n_q]);
    launched(c, "bsgs_mac_kernel", 2);
  });
}

// ---- P40: 5-byte packed diagonals (limbs with q < 2^40), hx_bsgs_p40.cu
namespace {
struct P40Plan {
  std::vector<int> p40, wide;  // limbs of 0..n_q-1 with q < 2^40 / the rest
};
P40Plan p40_plan(const hx_ctx* c, int n_q) {
  P40Plan P;
  for (int i = 0; i < n_q; ++i) (c->primes[i] < (1ull << 40) && c->f64[i] ? P.p40 : P.wide).push_back(i);
  return P;
}
bool p40_shape_ok(const hx_ctx* c, int n1, int n2, int n_q) {
  return c && (n1 == 32 || n1 == 64) && n2 >= 1 && n_q >= 1 && n_q <= c->n_chain && c->N() >= 32;
}
}  // namespace

long long hx_bsgs_p40_bytes(hx_ctx* c, int n1, int n2, int n_q) {
  if (!p40_shape_ok(c, n1, n2, n_q)) return -1;
  const P40Plan P = p40_plan(c, n_q);
  if (P.p40.empty()) return -1;
  return (long long)P.p40.size() * c->N() * n2 * n1 * 5;
}

int hx_bsgs_p40_pack(hx_ctx* c, void* packed, const uint64_t* diags, int diag_limbs, int n1, int n2,
                     int diag_jstride, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_REQUIRE(p40_shape_ok(c, n1, n2, n_q) && diag_limbs >= n_q, "bsgs_p40_pack: bad shape (n1 in {32, 64})");
    HX_REQUIRE(packed && diags, "bsgs_p40_pack: null buffer");
    const int dj = diag_jstride ? diag_jstride : n1;
    HX_REQUIRE(dj >= n1, "bsgs_p40_pack: diag_jstride < n1");
    const P40Plan P = p40_plan(c, n_q);
    HX_REQUIRE(!P.p40.empty(), "bsgs_p40_pack: no limb with q < 2^40");
    DBuf tab((P.p40.size() * sizeof(int) + 7) / 8, S(s), c);
    cuda_ok(cudaMemcpyAsync(tab.p, P.p40.data(), P.p40.size() * sizeof(int), cudaMemcpyHostToDevice, S(s)), "h2d");
    hx::launch_p40_pack(static_cast<unsigned char*>(packed), (const u64*)diags, (long long)diag_limbs * c->N(),
                        reinterpret_cast<const int*>(tab.p), (int)P.p40.size(), n1, n2, dj, c->logn, S(s));
    launched(c, "p40_pack_kernel");
  });
}

int hx_bsgs_mac_p40(hx_ctx* c, uint64_t* inner, long long inner_jstride, const uint64_t* baby, const void* packed,
                    const uint64_t* diags, int diag_limbs, int n1, int n2, int diag_jstride, int n_q, void* s) {
  return hx_bsgs_mac_p40_blocks(c, inner, inner_jstride, 0, baby, packed, diags, diag_limbs, n1, n2, 1, diag_jstride,
                                n_q, s);
}

int hx_bsgs_mac_p40_blocks(hx_ctx* c, uint64_t* inner, long long inner_jstride, long long inner_bstride,
                           const uint64_t* baby, const void* packed, const uint64_t* diags, int diag_limbs, int n1,
                           int n2, int blocks, int diag_jstride, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    check_nq(c, n_q);
    HX_REQUIRE(blocks >= 1 && (blocks == 1 || diag_jstride == 0 || diag_jstride == n1),
               "bsgs_mac_p40: several blocks need contiguous diagonals (diag_jstride = n1)");
    HX_REQUIRE(p40_shape_ok(c, n1, n2, n_q) && diag_limbs >= n_q, "bsgs_mac_p40: bad shape (n1 in {32, 64})");
    HX_REQUIRE(inner && baby && packed && diags, "bsgs_mac_p40: null buffer");
    const int dj = diag_jstride ? diag_jstride : n1;
    HX_REQUIRE(dj >= n1, "bsgs_mac_p40: diag_jstride < n1");
    const P40Plan P = p40_plan(c, n_q);
    HX_REQUIRE(!P.p40.empty(), "bsgs_mac_p40: no limb with q < 2^40");
    std::vector<int> lists(P.p40);
    lists.insert(lists.end(), P.wide.begin(), P.wide.end());
    DBuf tab((lists.size() * sizeof(int) + 7) / 8, S(s), c);
    cuda_ok(cudaMemcpyAsync(tab.p, lists.data(), lists.size() * sizeof(int), cudaMemcpyHostToDevice, S(s)), "h2d");
    const int* dl = reinterpret_cast<const int*>(tab.p);
    hx::P40Args A;
    A.inner = (u64*)inner;
    A.baby = (const u64*)baby;
    A.packed = static_cast<const unsigned char*>(packed);
    A.limbs = dl;
    A.pc = c->d_pc;
    A.out_jstride = inner_jstride;
    A.out_bstride = inner_bstride;
    A.rpb = n2;
    A.n1 = n1;
    A.n2 = n2 * blocks;  // rows of one launch: every block's giant steps
    A.n_q = n_q;
    A.logn = c->logn;
    A.stages = hx::p40_stages(n1);
    {
      hx::KTimer kt(c, "bsgs_mac_p40_kernel", S(s));
      hx::launch_bsgs_mac_p40(A, (int)P.p40.size(), S(s));
    }
    launched(c, "bsgs_mac_p40_kernel");
    for (int b = 0; b < blocks && !P.wide.empty(); ++b) {  // the wide limbs (60-bit q_0): 128-bit integer MAC over the u64 words
      hx::MacArgs M;
      M.inner = (u64*)inner + (long long)b * inner_bstride;
      M.baby = (const u64*)baby;
      M.diags = (const u64*)diags + (long long)b * n2 * dj * diag_limbs * c->N();
      M.pc = c->d_pc;
      M.n1 = n1;
      M.n2 = n2;
      M.n_q = n_q;
      M.logn = c->logn;
      M.diag_stride = (long long)diag_limbs * c->N();
      M.out_jstride = inner_jstride;
      M.limbs = nullptr;
      M.tokens = 1;
      M.baby_tstride = 0;
      M.inner_tstride = 0;
      M.diag_jstride = dj;
      hx::launch_bsgs_mac(M, c->N(), S(s), nullptr, 0, dl + P.p40.size(), (int)P.wide.size());
      launched(c, "bsgs_mac_int_kernel");
    }
  });
}

int hx_bsgs_mac_sparse(hx_ctx* c, uint64_t* inner, long long inner_jstride, long long inner_tstride,
                       const uint64_t* baby, long long baby_tstride, const int* group_ptr, const int* ks,
                       const uint64_t* const* diags, int n1, int n2, int n_q, int tokens, void* s) {
  return guarded([&] {
    check_ctx(c);
    check_nq(c, n_q);
    HX_REQUIRE(n1 >= 1 && n1 <= 128 && n2 >= 1 && tokens >= 1, "bsgs_mac_sparse: bad shape");
    HX_REQUIRE(c->N() >= 64 && (long long)tokens * (c->N() / 64) < (1ll << 31), "bsgs_mac_sparse: shape");
    HX_REQUIRE(group_ptr[0] == 0, "bsgs_mac_sparse: group_ptr[0] != 0");
    for (int j = 0; j < n2; ++j) HX_REQUIRE(group_ptr[j + 1] >= group_ptr[j], "bsgs_mac_sparse: group_ptr not monotone");
    const int nnz = group_ptr[n2];
    if (nnz <= 0) return;
    for (int e = 0; e < nnz; ++e) HX_REQUIRE(ks[e] >= 0 && ks[e] < n1 && diags[e], "bsgs_mac_sparse: bad entry");
    // one device table: gptr [n2 + 1] | ks [nnz] (ints) | dptr [nnz] (pointers)
    const size_t ib = ((size_t)(n2 + 1 + nnz) * sizeof(int) + 15) & ~(size_t)15;
    std::vector<char> host(ib + (size_t)nnz * sizeof(void*));
    std::memcpy(host.data(), group_ptr, (size_t)(n2 + 1) * sizeof(int));
    std::memcpy(host.data() + (size_t)(n2 + 1) * sizeof(int), ks, (size_t)nnz * sizeof(int));
    std::memcpy(host.data() + ib, diags, (size_t)nnz * sizeof(void*));
    DBuf tab((host.size() + 7) / 8, S(s), c);
    cuda_ok(cudaMemcpyAsync(tab.p, host.data(), host.size(), cudaMemcpyHostToDevice, S(s)), "h2d");
    hx::SparseMacArgs A;
    A.inner = (u64*)inner;
    A.baby = (const u64*)baby;
    A.gptr = (const int*)tab.p;
    A.ks = A.gptr + (n2 + 1);
    A.dptr = (const u64* const*)((const char*)tab.p + ib);
    A.pc = c->d_pc;
    A.n1 = n1;
    A.n2 = n2;
    A.n_q = n_q;
    A.logn = c->logn;
    A.tokens = tokens;
    A.out_jstride = inner_jstride;
    A.baby_tstride = baby_tstride;
    A.inner_tstride = inner_tstride;
    hx::launch_bsgs_mac_sparse(A, c->N(), S(s));
    launched(c, "bsgs_mac_sparse_kernel");  // (pageable H2D: `host` may go once the call returns)
  });
}

namespace {
struct TcPlan {
  int KC, RG;
  std::vector<int> tc, wide;  // limb lists (q < 2^40: sliced operand tiles; else u64 copies)
  size_t tc_bytes, wide_bytes;
};
bool tc_shape_ok(const hx_ctx* c, int rows, int n1, int n_q) {
  return c && rows >= 1 && rows <= 128 && n1 >= 8 && n1 <= 64 && n1 % 8 == 0 && n_q >= 1 && n_q <= c->n_chain &&
         c->N() >= 128;
}
TcPlan tc_plan(const hx_ctx* c, int rows, int n1, int n_q) {
  TcPlan P;
  P.KC = (5 * n1 + 31) / 32 * 2;
  P.RG = (rows + 7) / 8;
  for (int i = 0; i < n_q; ++i) (c->primes[i] < (1ull << 40) ? P.tc : P.wide).push_back(i);
  P.tc_bytes = P.tc.size() * (size_t)c->N() * P.RG * P.KC * 128;
  P.wide_bytes = P.wide.size() * (size_t)rows * n1 * c->N() * 8;
  return P;
}
int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}
}  // namespace

long long hx_bsgs_tc_bytes(hx_ctx* c, int rows, int n1, int n_q) {
  if (!tc_shape_ok(c, rows, n1, n_q)) return -1;
  const TcPlan P = tc_plan(c, rows, n1, n_q);
  return (long long)(P.tc_bytes + P.wide_bytes);
}

int hx_bsgs_tc_pack(hx_ctx* c, void* packed, const uint64_t* const* diag_ptrs, int rows, int n1, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_REQUIRE(tc_shape_ok(c, rows, n1, n_q), "bsgs_tc_pack: bad shape (rows <= 128, n1 % 8 == 0, n1 <= 64, N >= 128)");
    HX_REQUIRE(packed && diag_ptrs, "bsgs_tc_pack: null buffer");
    const TcPlan P = tc_plan(c, rows, n1, n_q);
    const size_t np = (size_t)rows * n1;
    const size_t pb = np * sizeof(void*);
    std::vector<char> host(pb + (P.tc.size() + P.wide.size()) * sizeof(int));
    std::memcpy(host.data(), diag_ptrs, pb);
    int* hl = reinterpret_cast<int*>(host.data() + pb);
    std::copy(P.tc.begin(), P.tc.end(), hl);
    std::copy(P.wide.begin(), P.wide.end(), hl + P.tc.size());
    DBuf tab((host.size() + 7) / 8, S(s), c);
    cuda_ok(cudaMemcpyAsync(tab.p, host.data(), host.size(), cudaMemcpyHostToDevice, S(s)), "h2d");
    const int* dl = reinterpret_cast<const int*>(reinterpret_cast<const char*>(tab.p) + pb);
    hx::launch_tc_pack(static_cast<unsigned char*>(packed), reinterpret_cast<const u64* const*>(tab.p), dl,
                       (int)P.tc.size(), dl + P.tc.size(), (int)P.wide.size(), rows, n1, P.KC, P.RG, c->logn,
                       P.tc_bytes, S(s));
    launched(c, "tc_pack_kernel", (P.tc.empty() ? 0 : 1) + (P.wide.empty() ? 0 : 1));
  });
}

int hx_bsgs_mac_tc(hx_ctx* c, uint64_t* inner, long long inner_jstride, long long inner_bstride,
                   long long inner_tstride, const uint64_t* baby, long long baby_tstride, const void* packed,
                   int blocks, int n2, int n1, int n_q, int tokens, void* s) {
  return guarded([&] {
    check_ctx(c);
    check_nq(c, n_q);
    HX_REQUIRE(blocks >= 1 && n2 >= 1 && tokens >= 1, "bsgs_mac_tc: bad shape");
    const int rows = blocks * n2;
    HX_REQUIRE(tc_shape_ok(c, rows, n1, n_q), "bsgs_mac_tc: bad shape (rows <= 128, n1 % 8 == 0, n1 <= 64)");
    HX_REQUIRE(inner && baby && packed, "bsgs_mac_tc: null buffer");
    HX_REQUIRE((reinterpret_cast<uintptr_t>(inner) & 31) == 0 && inner_jstride % 4 == 0 && inner_bstride % 4 == 0 &&
                   inner_tstride % 4 == 0,
               "bsgs_mac_tc: inner sums must be 32-byte aligned (whole-sector stores)");
    const TcPlan P = tc_plan(c, rows, n1, n_q);
    const long long N = c->N();
    // device table: row offsets [rows] | TC limbs | wide limbs | Barrett constants [n_tc][2]
    const size_t lb = (size_t)rows * 8 + (P.tc.size() + P.wide.size()) * sizeof(int);
    std::vector<char> host(lb + P.tc.size() * 2 * sizeof(hx::u32));
    hx::u32* mu = reinterpret_cast<hx::u32*>(host.data() + lb);
    for (size_t e = 0; e < P.tc.size(); ++e) {
      const u64 q = c->primes[P.tc[e]];
      mu[2 * e] = (hx::u32)((((unsigned __int128)1) << 56) / q);
      mu[2 * e + 1] = (hx::u32)((1ull << 48) / q);
    }
    long long* ro = reinterpret_cast<long long*>(host.data());
    for (int b = 0; b < blocks; ++b)
      for (int j = 0; j < n2; ++j) ro[b * n2 + j] = j * inner_jstride + b * inner_bstride;
    int* hl = reinterpret_cast<int*>(host.data() + (size_t)rows * 8);
    std::copy(P.tc.begin(), P.tc.end(), hl);
    std::copy(P.wide.begin(), P.wide.end(), hl + P.tc.size());
    DBuf tab((host.size() + 7) / 8, S(s), c);
    cuda_ok(cudaMemcpyAsync(tab.p, host.data(), host.size(), cudaMemcpyHostToDevice, S(s)), "h2d");
    const int* dl = reinterpret_cast<const int*>(reinterpret_cast<const char*>(tab.p) + (size_t)rows * 8);
    const long long L = (long long)n_q * N;
    int launches = 0;
    if (!P.tc.empty()) {
      hx::TcArgs A;
      A.row_off = reinterpret_cast<const long long*>(tab.p);
      A.L = L;
      A.packed = static_cast<const unsigned char*>(packed);
      A.limbs = dl;
      A.pc = c->d_pc;
      A.mu = reinterpret_cast<const hx::u32*>(reinterpret_cast<const char*>(tab.p) + lb);
      A.rows = rows;
      A.n1 = n1;
      A.n_tc = (int)P.tc.size();
      A.logn = c->logn;
      A.KC = P.KC;
      A.RG = P.RG;
      A.tstride = inner_tstride;
      DBuf bt((size_t)std::min(tokens, hx::kTcMaxTokens) * n1 * 2 * P.tc.size() * N, S(s), c);
      for (int t0 = 0; t0 < tokens;) {
        int T = hx::kTcMaxTokens;
        while (T > tokens - t0) T /= 2;
        hx::launch_tc_baby(bt.p, (const u64*)baby + t0 * baby_tstride, baby_tstride, L, dl, (int)P.tc.size(), n1, T,
                           c->logn, S(s));
        A.inner = (u64*)inner + t0 * inner_tstride;
        A.baby = bt.p;
        hx::KTimer kt(c, "bsgs_mac_tc_kernel", S(s));
        hx::launch_bsgs_mac_tc(A, T, sm_count(), S(s));
        launches += 2;
        t0 += T;
      }
    }
    // limbs with q >= 2^40: the integer k-split MAC over the u64 copies
    // ([w][r][k][N]; the kernel indexes diags + i N + (j n1 + k) N)
    const u64* wide = reinterpret_cast<const u64*>(static_cast<const char*>(packed) + P.tc_bytes);
    for (size_t w = 0; w < P.wide.size(); ++w) {
      const int i = P.wide[w];
      for (int b = 0; b < blocks; ++b) {
        hx::MacArgs A;
        A.inner = (u64*)inner + b * inner_bstride;
        A.baby = (const u64*)baby;
        A.diags = wide + ((long long)w * rows + (long long)b * n2) * n1 * N - (long long)i * N;
        A.pc = c->d_pc;
        A.n1 = n1;
        A.n2 = n2;
        A.n_q = n_q;
        A.logn = c->logn;
        A.diag_stride = N;
        A.out_jstride = inner_jstride;
        A.limbs = nullptr;
        A.tokens = tokens;
        A.baby_tstride = baby_tstride;
        A.inner_tstride = inner_tstride;
        A.diag_jstride = n1;
        hx::launch_bsgs_mac(A, N, S(s), nullptr, 0, dl + P.tc.size() + w, 1);
        ++launches;
      }
    }
    launched(c, "bsgs_mac_tc_kernel", launches);
  });
}

int hx_bsgs_mac_ex(hx_ctx* c, uint64_t* inner, long long inner_jstride, const uint64_t* baby,
                   const uint64_t* diags, int diag_limbs, int n1, int n2, int n_q, void* s) {
  return hx_bsgs_mac_tokens(c, inner, inner_jstride, 0, baby, 0, diags, diag_limbs, n1, n2, n_q, 1, 0, s);
}

int hx_bsgs_mac(hx_ctx* c, uint64_t* inner, const uint64_t* baby, const uint64_t* diags,
                int diag_limbs, int n1, int n2, int n_q, void* s) {
  return hx_bsgs_mac_ex(c, inner, 2ll * n_q * (c ? c->N() : 0), baby, diags, diag_limbs, n1, n2, n_q, s);
}

int hx_sum_strided(hx_ctx* c, uint64_t* out, const uint64_t* in, int terms, long long term_stride,
                   int polys, long long in_poly_stride, long long out_poly_stride, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(polys);
    check_nq(c, n_q);
    HX_REQUIRE(terms >= 1 && polys >= 1, "sum: terms, polys >= 1");
    hx::SumArgs A;
    A.out = (u64*)out;
    A.in = (const u64*)in;
    A.pc = c->d_pc;
    A.terms = terms;
    A.n_q = n_q;
    A.logn = c->logn;
    A.term_stride = term_stride;
    A.in_poly_stride = in_poly_stride;
    A.out_poly_stride = out_poly_stride;
    hx::launch_sum(A, polys, c->N(), S(s));
    launched(c, "sum_kernel");
  });
}

int hx_ctx_time_kernel(hx_ctx* c, const char* name) {
  return guarded([&] {
    check_ctx(c);
    for (auto& e : c->ktime_ev) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    c->ktime_ev.clear();
    c->ktime_on = name && *name;
    c->ktime_name = name ? name : "";
  });
}

int hx_ctx_kernel_time(hx_ctx* c, double* total_ms, long long* launches) {
  return guarded([&] {
    check_ctx(c);
    double tot = 0.0;
    for (auto& e : c->ktime_ev) {
      cuda_ok(cudaEventSynchronize(e.second), "event sync");
      float ms = 0.f;
      cuda_ok(cudaEventElapsedTime(&ms, e.first, e.second), "event elapsed");
      tot += ms;
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    if (launches) *launches = (long long)c->ktime_ev.size();
    if (total_ms) *total_ms = tot;
    c->ktime_ev.clear();
  });
}

int hx_sample_uniform(hx_ctx* c, uint64_t* out, int n_c, int n_s, int copies, uint64_t seed, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(copies);
    HX_REQUIRE(n_c >= 0 && n_c <= c->n_chain && n_s >= 0 && n_s <= c->n_special && copies >= 0, "sample_uniform");
    const long long words = (long long)copies * (n_c + n_s) * c->N();
    if (!words) return;
    const LimbTable lt = hx::make_table(c, n_c, n_s);
    hx::sample_uniform_kernel<<<(unsigned)(words / 256), 256, 0, S(s)>>>((u64*)out, c->d_pc, lt, c->logn, seed);
    launched(c, "sample_uniform_kernel");
  });
}

int hx_sample_cbd(hx_ctx* c, int64_t* e, long long count, uint64_t seed, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(count);
    HX_REQUIRE(count >= 0, "sample_cbd");
    if (!count) return;
    hx::sample_cbd_kernel<<<(unsigned)((count + 255) / 256), 256, 0, S(s)>>>((long long*)e, count, seed);
    launched(c, "sample_cbd_kernel");
  });
}

int hx_keygen_ksk(hx_ctx* c, uint64_t* key, const uint64_t* s_full, const uint64_t* sp_full,
                  const uint64_t* a_full, const int64_t* e, void* s) {
  return guarded([&] {
    check_ctx(c);
    const long long N = c->N();
    const int T = c->n_total(), dn = c->dnum(c->n_chain);
    DBuf en((long long)dn * T * N, S(s), c);
    const LimbTable lt = hx::make_table(c, c->n_chain, c->n_special);
    const int th = pt_threads(c);
    hx::from_i64_kernel<<<(unsigned)((long long)dn * T * (N / th)), th, 0, S(s)>>>(
        en.p, (const long long*)e, c->d_pc, lt, c->logn);
    launched(c, "from_i64_kernel");
    hx::ntt_forward(c, en.p, dn, lt, S(s));
    hx::keygen_kernel<<<dim3((unsigned)(N / th), (unsigned)T, (unsigned)dn), th, 0, S(s)>>>(
        (u64*)key, en.p, (const u64*)s_full, (const u64*)sp_full, (const u64*)a_full, c->d_pc,
        c->d_pmodq, c->n_chain, T, c->alpha, c->logn);
    launched(c, "keygen_kernel");
  });
}

size_t hx_ckey_words(const hx_ctx* c) {
  return c ? (size_t)c->dnum(c->n_chain) * c->n_total() * c->N() : 0;
}

// b half of a full key [dnum][2][full][N] -> compressed [dnum][full][N]
static void take_b(hx_ctx* c, u64* ckey, const u64* full, cudaStream_t s) {
  const long long w = (long long)c->n_total() * c->N();
  copy2d(ckey, w, full, 2 * w, w, c->dnum(c->n_chain), s);
}

int hx_keygen_ksk_c(hx_ctx* c, uint64_t* ckey, const uint64_t* s_full, const uint64_t* sp_full, uint64_t seed,
                    const int64_t* e, void* s) {
  return guarded([&] {
    check_ctx(c);
    const int dn = c->dnum(c->n_chain);
    DBuf a((long long)dn * c->n_total() * c->N(), S(s), c), full((long long)hx_key_words(c), S(s), c);
    int rc = hx_sample_uniform(c, (uint64_t*)a.p, c->n_chain, c->n_special, dn, seed, s);
    if (rc == HX_OK) rc = hx_keygen_ksk(c, (uint64_t*)full.p, s_full, sp_full, (const uint64_t*)a.p, e, s);
    if (rc != HX_OK) throw HxError(rc, g_last_error);
    take_b(c, (u64*)ckey, full.p, S(s));
    c->ckeys[ckey] = hx_ckey{seed, 1u};
  });
}

int hx_keygen_rotation_c(hx_ctx* c, uint64_t* ckey, const uint64_t* s_full, uint64_t g, uint64_t seed,
                         const int64_t* e, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element must be odd and < 2N");
    const int dn = c->dnum(c->n_chain);
    DBuf a((long long)dn * c->n_total() * c->N(), S(s), c), full((long long)hx_key_words(c), S(s), c);
    int rc = hx_sample_uniform(c, (uint64_t*)a.p, c->n_chain, c->n_special, dn, seed, s);
    if (rc == HX_OK) rc = hx_keygen_rotation(c, (uint64_t*)full.p, s_full, g, (const uint64_t*)a.p, e, s);
    if (rc != HX_OK) throw HxError(rc, g_last_error);
    // rotation layout: full = tau_{g^-1}(standard), its uniform half is the
    // seed's stream read at ntt_auto_index(t, g^-1)
    take_b(c, (u64*)ckey, full.p, S(s));
    c->ckeys[ckey] = hx_ckey{seed, (hx::u32)galois_inverse(g, 2 * (u64)c->N())};
  });
}

int hx_key_expand(hx_ctx* c, uint64_t* full, const uint64_t* ckey, void* s) {
  return guarded([&] {
    check_ctx(c);
    const auto it = c->ckeys.find(ckey);
    HX_REQUIRE(it != c->ckeys.end(), "hx_key_expand: not a compressed key of this context");
    const int th = pt_threads(c);
    hx::key_expand_kernel<<<dim3((unsigned)(c->N() / th), (unsigned)c->n_total(), (unsigned)c->dnum(c->n_chain)), th, 0,
                            S(s)>>>((u64*)full, (const u64*)ckey, c->d_pc, c->n_total(), c->logn, it->second.seed,
                                    it->second.kg);
    launched(c, "key_expand_kernel");
  });
}

int hx_key_release(hx_ctx* c, const uint64_t* ckey) {
  return guarded([&] {
    check_ctx(c);
    c->ckeys.erase(ckey);
  });
}

int hx_ksk_to_rotation_layout(hx_ctx* c, uint64_t* out, const uint64_t* in, uint64_t g,
                              void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element must be odd and < 2N");
    HX_REQUIRE(out != in, "key layout conversion cannot run in place");
    const int limbs = c->dnum(c->n_chain) * 2 * c->n_total();
    permute(c, (u64*)out, 0, (const u64*)in, 0, limbs, 1, galois_inverse(g, 2 * c->N()), S(s));
  });
}

int hx_keygen_rotation(hx_ctx* c, uint64_t* key, const uint64_t* s_full, uint64_t g,
                       const uint64_t* a_full, const int64_t* e, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element must be odd and < 2N");
    const long long N = c->N();
    const int T = c->n_total();
    DBuf sp((long long)T * N, S(s), c), std_key((long long)hx_key_words(c), S(s), c);
    permute(c, sp.p, 0, (const u64*)s_full, 0, T, 1, g, S(s));  // s' = tau_g(s)
    int rc = hx_keygen_ksk(c, (uint64_t*)std_key.p, s_full, (const uint64_t*)sp.p, a_full, e, s);
    if (rc != HX_OK) throw HxError(rc, g_last_error);
    rc = hx_ksk_to_rotation_layout(c, key, (const uint64_t*)std_key.p, g, s);
    if (rc != HX_OK) throw HxError(rc, g_last_error);
  });
}

int hx_encrypt_sk(hx_ctx* c, uint64_t* ct, const uint64_t* m, const uint64_t* s_full,
                  const uint64_t* a, const int64_t* e, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    check_nq(c, n_q);
    const long long N = c->N();
    DBuf en((long long)n_q * N, S(s), c);
    const LimbTable lt = hx::make_table(c, n_q, 0);
    const int th = pt_threads(c);
    hx::from_i64_kernel<<<(unsigned)((long long)n_q * (N / th)), th, 0, S(s)>>>(
        en.p, (const long long*)e, c->d_pc, lt, c->logn);
    launched(c, "from_i64_kernel");
    hx::ntt_forward(c, en.p, 1, lt, S(s));
    hx::encrypt_kernel<<<dim3((unsigned)(N / th), (unsigned)n_q), th, 0, S(s)>>>(
        (u64*)ct, (const u64*)m, en.p, (const u64*)s_full, (const u64*)a, c->d_pc, n_q, c->logn);
    launched(c, "encrypt_kernel");
  });
}

int hx_decrypt(hx_ctx* c, uint64_t* m, const uint64_t* ct, const uint64_t* s_full, int batch,
               int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    const int th = pt_threads(c);
    hx::decrypt_kernel<<<dim3((unsigned)(c->N() / th), (unsigned)n_q, (unsigned)batch), th, 0,
                         S(s)>>>((u64*)m, (const u64*)ct, (const u64*)s_full, c->d_pc, n_q,
                                 c->logn);
    launched(c, "decrypt_kernel");
  });
}

int hx_rotate_host(hx_ctx* c, uint64_t* out_host, const uint64_t* in_host, const uint64_t* key,
                   int batch, int n_q, uint64_t g, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    HX_REQUIRE((g & 1) && g < 2 * (u64)c->N(), "galois element");  // before any copy is queued
    HX_REQUIRE(key != nullptr && in_host != nullptr && out_host != nullptr, "null buffer");
    const long long ct = 2ll * n_q * c->N();
    pipelined_host(c, batch, {in_host}, {ct}, out_host, ct, S(s),
                   [&](u64* out, const std::vector<u64*>& in, int n, cudaStream_t st) {
                     const int rc = hx_rotate(c, (uint64_t*)out, (const uint64_t*)in[0], key, n, n_q, g, st);
                     if (rc != HX_OK) throw HxError(rc, g_last_error);
                   });
  });
}

int hx_mul_relin_host(hx_ctx* c, uint64_t* out_host, const uint64_t* a_host,
                      const uint64_t* b_host, const uint64_t* rlk, int batch, int n_q, void* s) {
  return guarded([&] {
    check_ctx(c);
    HX_COUNT(batch);
    check_nq(c, n_q);
    HX_REQUIRE(rlk != nullptr && a_host != nullptr && b_host != nullptr && out_host != nullptr, "null buffer");
    const long long ct = 2ll * n_q * c->N();
    pipelined_host(c, batch, {a_host, b_host}, {ct, ct}, out_host, ct, S(s),
                   [&](u64* out, const std::vector<u64*>& in, int n, cudaStream_t st) {
                     const int rc = hx_mul_relin(c, (uint64_t*)out, (const uint64_t*)in[0],
                                                 (const uint64_t*)in[1], rlk, n, n_q, st);
                     if (rc != HX_OK) throw HxError(rc, g_last_error);
                   });
  });
}

}  // extern "C"
