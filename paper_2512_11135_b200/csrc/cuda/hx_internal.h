// hx_internal.h -- host-side context and launcher prototypes shared by the
// translation units of libhx_b200.so (not part of the public C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "hx_common.cuh"
#include "hx_types.cuh"
#include "hx_ntt.cuh"
#include "hx_modup.cuh"

// Scratch arena of a context: one device block handed out as a LIFO stack to
// the scoped temporaries of the C-ABI calls (DBuf), so the steady state makes
// no allocator calls at all (mapping fresh pool memory costs ~0.1 s per
// 5 GB and would land inside timed steps).  Requests that do not fit fall
// back to the stream-ordered pool and raise the high-water mark; the block is
// regrown to the mark when the stack is next empty.  Stream safety: the arena
// follows one stream at a time; a call on another stream first waits for the
// previous stream's work (event), so reuse never races.
struct HxArena {
  char* base = nullptr;
  size_t cap = 0, top = 0, high = 0;
  int depth = 0;
  cudaStream_t stream = nullptr;
  bool stream_set = false;
  cudaEvent_t ev = nullptr;
};

struct hx_ckey {
  hx::u64 seed;
  hx::u32 kg;  // layout permutation of the uniform half: g^-1 (rotation layout) or 1
};

struct hx_ctx {
  HxArena arena;
  // compressed keys created by this context (b half only; see hx_keygen_*_c)
  std::unordered_map<const void*, hx_ckey> ckeys;
  int logn = 0;
  int n_chain = 0, n_special = 0, alpha = 1;
  int device = 0;
  std::vector<hx::u64> primes;  // chain then special
  std::vector<hx::u64> psi;
  // device memory
  hx::PrimeConst* d_pc = nullptr;
  ulonglong2* d_tw = nullptr;  // [n_total][2][N]
  double* d_twf = nullptr;     // FP64-path twiddles [n_total][2][N] (w as double)
  std::vector<char> f64;       // prime index -> NTT on the FP64 pipe (q < 2^47)
  bool allow_f64 = true;       // HX_NTT_INT=1 forces the integer path (A/B tests)
  // BSGS MAC limb lists per n_q: [n_q][2][n_chain] ints (FP64 list, integer list)
  int* d_maclimbs = nullptr;
  std::vector<int> mac_nf64, mac_nint;
  // key inner-product limb lists over the n_q + K limbs: [n_q][2][n_total]
  int* d_kslimbs = nullptr;
  std::vector<int> ks_nf64, ks_nint;
  // ModUp constants: for each n_q in [1, n_chain] and digit d < dnum(n_q):
  // qhinv [alpha] and conv [alpha][n_total]; offsets in units of SC.
  hx::SC* d_modup = nullptr;
  std::vector<std::vector<long long>> modup_qh_off, modup_cv_off;  // [n_q][d]
  // fused ModUp: BconvC table offsets [n_q][d]; target lists [n_q][d] into
  // d_tlist (FP64-class limbs first, then integer-class)
  hx::BconvC* d_bconv = nullptr;
  int* d_tlist = nullptr;
  std::vector<std::vector<long long>> bc_off;
  std::vector<std::vector<int>> tl_off, tl_cnt, tl_icnt;
  // ModDown constants
  hx::SC* d_phinv = nullptr;   // [K]
  hx::SC* d_pconv = nullptr;   // [K][n_chain]
  double* d_pconvf = nullptr;  // [K][n_chain][4]: FP64 form (w, w/q, [2^30 w]_q, /q)
  // ModDown through modup_col_kernel (centred): BconvC [n_chain][K] with
  // w = [P / p_k]_{q_j}; target lists per n_q (FP64 class first); [P]_{q_j}
  // as double
  hx::BconvC* d_mdbc = nullptr;
  int* d_mdtl = nullptr;
  std::vector<int> md_tl_off, md_tl_cnt, md_tl_icnt;
  double* d_pmodqf = nullptr;
  double* d_pmodqf1 = nullptr;  // [P psi^(N/2)]_{q_j}: the folded first stage
  // joint-reduction rounding constants per n_q (0: bounds fail, unfused path)
  std::vector<double> cs_up, cs_down;
  hx::u64* d_pmodq = nullptr;  // [n_chain]
  hx::SC* d_pinv = nullptr;    // [n_chain]
  // Rescale constants: [l][i] for i < l
  hx::SC* d_qlinv = nullptr;   // [n_chain][n_chain]
  hx::u64* d_qlmod = nullptr;  // [n_chain][n_chain]
  // side stream of the key switch (HX_KS_SIDE=1): the integer-class ModUp
  // limbs (NTT + key inner product) run beside the FP64 ROW + inner kernel;
  // fork / join events, `side_open` between the fork in modup and the join
  // in the inner product
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool side_open = false;
  // launch counter (kernels issued through this context)
  unsigned long long launches = 0;
  // live per-kernel timing (hx_ctx_time_kernel): CUDA events recorded on the
  // launching stream around every launch of the kernel family `ktime_name`
  bool ktime_on = false;
  std::string ktime_name;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ktime_ev;

  int n_total() const { return n_chain + n_special; }
  long long N() const { return 1ll << logn; }
  int dnum(int n_q) const { return (n_q + alpha - 1) / alpha; }
  int pidx(int k, int n_q) const { return k < n_q ? k : n_chain + (k - n_q); }
};

namespace hx {

// RAII: events around one launch when its kernel family is being timed
struct KTimer {
  hx_ctx* c;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  KTimer(hx_ctx* c_, const char* name, cudaStream_t s_) : c(c_), s(s_) {
    if (c->ktime_on && c->ktime_name == name && cudaEventCreate(&a) == cudaSuccess) cudaEventRecord(a, s);
  }
  ~KTimer() {
    cudaEvent_t b = nullptr;
    if (a && cudaEventCreate(&b) == cudaSuccess) {
      cudaEventRecord(b, s);
      c->ktime_ev.emplace_back(a, b);
    }
  }
  KTimer(const KTimer&) = delete;
  KTimer& operator=(const KTimer&) = delete;
};

// limb table for an (n_q chain, n_p special) poly batch element with `stride`
// limbs per element starting at limb offset `first`
LimbTable make_table(const hx_ctx* c, int n_q, int n_p, int stride = -1, int first = 0);

// NTT launchers (hx_ntt.cu)
void ntt_forward(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s);
// src: read the input from src (element b, limb entry e at src + b src_estride
// + off[e] N) and leave the result in data -- an out-of-place transform
void ntt_inverse(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s,
                 const u64* src = nullptr, long long src_estride = 0);
// forward ROW pass only (the COL pass done by a fused producer, hx_modup.cuh)
// f64_col_done: the FP64-class limbs already had their COL pass (fused ModDown
// conversion); the integer-class limbs still get theirs
void ntt_forward_combine(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, const EpiArgs& ep,
                         cudaStream_t s, bool f64_col_done = false);
void ntt_forward_rows(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s);
int ntt_split_a(int logn);

void launch_bsgs_mac_sparse(const SparseMacArgs& A, long long N, cudaStream_t s);

void set_error(const std::string& msg);
// record `msg` as hx_last_error() and return `code` (C-ABI entry points outside hx_ops.cu)
int fail(int code, const std::string& msg);

}  // namespace hx
