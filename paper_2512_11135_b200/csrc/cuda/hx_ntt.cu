// hx_ntt.cu -- NTT pass instantiations and launchers (see hx_ntt.cuh).
//
// A launch's limb table is split by prime class: primes q < 2^47 run the
// FP64-pipe butterflies, wider primes (the 60-bit q_0 and special primes of
// config 2, the 50-bit special of config 1) the integer Shoup butterflies.
// Both classes are issued on the same stream in pass order, so every limb
// sees its COL pass before its ROW pass (forward) and vice versa (inverse).
#include <algorithm>
#include <cstdlib>

#include "hx_internal.h"
#include "hx_ntt_cluster.cuh"

#ifndef HX_NTT_OB
#define HX_NTT_OB 3
#endif

namespace hx {

namespace {

template <bool FWD, bool ROW, int S, bool F64>
void launch_pass(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s,
                 const u64* src = nullptr, long long src_estride = 0) {
  constexpr int OB = HX_NTT_OB;
  constexpr int TILE = 1 << (S + OB);
  NttArgs a;
  a.data = data;
  a.pc = c->d_pc;
  a.lt = lt;
  a.logn = c->logn;
  a.instances = batch * lt.count;
  a.batch = batch;
  a.bper = 1;
  a.src = src;
  a.src_estride = src_estride;
  const long long tiles = c->N() / TILE;
  const long long blocks = a.instances * tiles;
  if (blocks <= 0) return;
  constexpr int smem = ntt_smem_bytes<ROW, S, OB, F64>();
  static bool configured = false;  // opt in to > 48 KB once per instantiation
  if (!configured) {
    cudaFuncSetAttribute(ntt_pass_kernel<FWD, ROW, S, OB, F64>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  KTimer kt(c, "ntt_pass_kernel", s);
  ntt_pass_kernel<FWD, ROW, S, OB, F64><<<(unsigned)blocks, TILE / 16, smem, s>>>(a);
  ++c->launches;
}

template <int S, bool F64>
void launch_row_combine(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, const EpiArgs& ep,
                        cudaStream_t s) {
  constexpr int OB = HX_NTT_OB;
  constexpr int TILE = 1 << (S + OB);
  NttArgs a;
  a.data = data;
  a.pc = c->d_pc;
  a.lt = lt;
  a.logn = c->logn;
  a.instances = batch * lt.count;
  a.batch = batch;
  a.bper = 1;
  const long long blocks = a.instances * (c->N() / TILE);
  if (blocks <= 0) return;
  constexpr int smem = ntt_smem_bytes<true, S, OB, F64>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ntt_row_combine_kernel<S, OB, F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  KTimer kt(c, "ntt_row_combine_kernel", s);
  ntt_row_combine_kernel<S, OB, F64><<<(unsigned)blocks, TILE / 16, smem, s>>>(a, ep);
  ++c->launches;
}

template <bool F64>
void dispatch_row_combine(hx_ctx* c, int S, u64* data, long long batch, const LimbTable& lt, const EpiArgs& ep,
                          cudaStream_t s) {
  switch (S) {
    case 3: launch_row_combine<3, F64>(c, data, batch, lt, ep, s); break;
    case 4: launch_row_combine<4, F64>(c, data, batch, lt, ep, s); break;
    case 5: launch_row_combine<5, F64>(c, data, batch, lt, ep, s); break;
    case 6: launch_row_combine<6, F64>(c, data, batch, lt, ep, s); break;
    case 7: launch_row_combine<7, F64>(c, data, batch, lt, ep, s); break;
    case 8: launch_row_combine<8, F64>(c, data, batch, lt, ep, s); break;
    default: set_error("ntt: unsupported sub-transform size");
  }
}

template <bool FWD, bool ROW, bool F64>
void dispatch(hx_ctx* c, int S, u64* data, long long batch, const LimbTable& lt, cudaStream_t s,
              const u64* src = nullptr, long long src_estride = 0) {
  switch (S) {
    case 3: launch_pass<FWD, ROW, 3, F64>(c, data, batch, lt, s, src, src_estride); break;
    case 4: launch_pass<FWD, ROW, 4, F64>(c, data, batch, lt, s, src, src_estride); break;
    case 5: launch_pass<FWD, ROW, 5, F64>(c, data, batch, lt, s, src, src_estride); break;
    case 6: launch_pass<FWD, ROW, 6, F64>(c, data, batch, lt, s, src, src_estride); break;
    case 7: launch_pass<FWD, ROW, 7, F64>(c, data, batch, lt, s, src, src_estride); break;
    case 8: launch_pass<FWD, ROW, 8, F64>(c, data, batch, lt, s, src, src_estride); break;
    default: set_error("ntt: unsupported sub-transform size");
  }
}

// Single-pass FP64-class transform of N = 2^16 limbs, one limb per cluster of
// 16 CTAs (hx_ntt_cluster.cuh).  Opt-in (HX_NTT_CLUSTER=1): measured slower
// than the two passes on B200 (1.31 M vs 2.09 M limb-NTT/s; 52.3 vs 50.1 ms
// per 256 key switches) -- each CTA runs load / transform / cluster barrier /
// DSMEM gather / transform / store in lockstep with its cluster, so nothing
// overlaps the phases.  false when not selected or unavailable (other N, no
// cluster of that shape fits the device).
template <bool FWD>
bool launch_cluster(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s,
                    const u64* src = nullptr, long long src_estride = 0) {
  constexpr int S = 8, OB = 4, TILE = 1 << (S + OB), C = 1 << (S - OB);
  static const bool off = !(getenv("HX_NTT_CLUSTER") && atoi(getenv("HX_NTT_CLUSTER")) == 1);
  if (off || c->logn != 2 * S || lt.count == 0) return false;
  auto kern = ntt_cluster_kernel<FWD, S, OB>;
  constexpr int smem = ntt_cluster_smem_bytes<S, OB>();
  static int ok = -1;
  if (ok < 0) {
    ok = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C * 64);
      cfg.blockDim = dim3(TILE / 16);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) ok = 1;
      if (getenv("HX_ALLOC_TRACE")) fprintf(stderr, "[hx] ntt cluster kernel: %d active clusters\n", n);
    }
    cudaGetLastError();
  }
  if (!ok) return false;
  NttArgs a;
  a.data = data;
  a.pc = c->d_pc;
  a.lt = lt;
  a.logn = c->logn;
  a.instances = batch * lt.count;
  a.batch = batch;
  a.bper = 1;
  a.src = src;
  a.src_estride = src_estride;
  const long long blocks = a.instances * C;
  if (blocks <= 0) return true;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(TILE / 16);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) {
    set_error("ntt: cluster launch failed");
    return true;
  }
  ++c->launches;
  return true;
}

// N = 2^a (column / high bits) x 2^b (row / low bits), a = ceil(logn/2)
inline int split_a(int logn) { return (logn + 1) / 2; }

void split(const hx_ctx* c, const LimbTable& lt, LimbTable& ti, LimbTable& tf) {
  ti = LimbTable{};
  tf = LimbTable{};
  ti.stride = tf.stride = lt.stride;
  for (int e = 0; e < lt.count; ++e) {
    LimbTable& t = c->f64[lt.prime[e]] ? tf : ti;
    t.off[t.count] = lt.off[e];
    t.prime[t.count] = lt.prime[e];
    ++t.count;
  }
}

}  // namespace

void ntt_forward(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s) {
  const int a = split_a(c->logn), b = c->logn - a;
  LimbTable ti, tf;
  split(c, lt, ti, tf);
  const bool one = tf.count && launch_cluster<true>(c, data, batch, tf, s);  // FP64 limbs in one pass
  if (ti.count) dispatch<true, false, false>(c, a, data, batch, ti, s);  // first a stages (COL)
  if (tf.count && !one) dispatch<true, false, true>(c, a, data, batch, tf, s);
  if (ti.count) dispatch<true, true, false>(c, b, data, batch, ti, s);   // last b stages (ROW)
  if (tf.count && !one) dispatch<true, true, true>(c, b, data, batch, tf, s);
}

// forward NTT of ModDown's converted term whose ROW pass writes the key-switch
// combine instead of the transform (EpiArgs); `data` is left after the COL pass
void ntt_forward_combine(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, const EpiArgs& ep,
                         cudaStream_t s, bool f64_col_done) {
  const int a = split_a(c->logn), b = c->logn - a;
  LimbTable ti, tf;
  split(c, lt, ti, tf);
  if (ti.count) dispatch<true, false, false>(c, a, data, batch, ti, s);
  if (tf.count && !f64_col_done) dispatch<true, false, true>(c, a, data, batch, tf, s);
  if (ti.count) dispatch_row_combine<false>(c, b, data, batch, ti, ep, s);
  if (tf.count) dispatch_row_combine<true>(c, b, data, batch, tf, ep, s);
}

void ntt_forward_rows(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s) {
  const int a = split_a(c->logn), b = c->logn - a;
  LimbTable ti, tf;
  split(c, lt, ti, tf);
  if (ti.count) dispatch<true, true, false>(c, b, data, batch, ti, s);
  if (tf.count) dispatch<true, true, true>(c, b, data, batch, tf, s);
}

int ntt_split_a(int logn) { return split_a(logn); }

void ntt_inverse(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s, const u64* src,
                 long long src_estride) {
  const int a = split_a(c->logn), b = c->logn - a;
  LimbTable ti, tf;
  split(c, lt, ti, tf);
  // FP64 limbs in one pass (cluster kernel) when available
  const bool one = tf.count && launch_cluster<false>(c, data, batch, tf, s, src, src_estride);
  // low-bit stages (ROW); with src, out of place (saves copying the input first)
  if (ti.count) dispatch<false, true, false>(c, b, data, batch, ti, s, src, src_estride);
  if (tf.count && !one) dispatch<false, true, true>(c, b, data, batch, tf, s, src, src_estride);
  if (ti.count) dispatch<false, false, false>(c, a, data, batch, ti, s);  // high-bit stages (COL), x N^-1
  if (tf.count && !one) dispatch<false, false, true>(c, a, data, batch, tf, s);
}

}  // namespace hx
