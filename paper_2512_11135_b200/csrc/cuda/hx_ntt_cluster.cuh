// hx_ntt_cluster.cuh -- single-pass FP64-class NTT / INTT of one limb per
// thread-block cluster (N = 2^(2 S), sm_100a distributed shared memory).
//
// Same transform as the two-pass ntt_pass_kernel pair (hx_ntt.cuh; reference
// NttTables::forward / inverse, ntt.cpp:57-96) and bit-identical output (the
// same butterflies in the same order; only where the intermediate lives
// changes): the 2^S x 2^S limb is split over a cluster of C = 2^(S - OB)
// CTAs.  Phase A: CTA k runs the first pass on its tile (forward: COL tile k
// = 2^OB adjacent columns; inverse: ROW tile k = 2^OB adjacent rows) from HBM
// and leaves the result in its own shared memory.  cluster barrier.  Phase B:
// CTA k gathers its second-pass tile (forward: ROW tile k; inverse: COL tile
// k) straight from the other CTAs' shared memory (ld.shared::cluster), runs
// the second pass and writes the limb to HBM.  Every limb is read once and
// written once (the two-pass kernels move it twice), and the ROW-pass
// twiddles are staged with cp.async while phase A runs.
#pragma once

#include <cooperative_groups.h>

#include "hx_common.cuh"
#include "hx_ntt.cuh"

namespace hx {

// Generic pass over one tile, data already in the thread's first-group
// layout is produced by `load(e)`; the last group hands its words to
// `store(e, word)`.  FIRST: convert residues to FP64 bits on load; LAST:
// normalise to [0, q) before the store.
template <bool FWD, bool ROW, int S, int OB, bool FIRST, bool LAST, class Load, class Store>
__device__ __forceinline__ void cl_pass(u64* sm, const double* sm_tw, const double* twf, const PrimeConst& P,
                                        int tile, int logn, Load load, Store store) {
  const int t = threadIdx.x;
  u64 x[16];
  constexpr int NG = Sched<S>::G + (Sched<S>::R ? 1 : 0);
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    constexpr int Rm = Sched<S>::R;
    int W, g0;
    if (FWD) {
      if (gi < Sched<S>::G) {
        W = 4;
        g0 = S - 4 * (gi + 1);
      } else {
        W = Rm;
        g0 = 0;
      }
    } else {
      if (Rm && gi == 0) {
        W = Rm;
        g0 = 0;
      } else {
        W = 4;
        g0 = Rm + 4 * (gi - (Rm ? 1 : 0));
      }
    }
    const bool lastg = (gi == NG - 1);
#define HX_CL_GROUP(WW)                                                                   \
  {                                                                                       \
    int eb[16 >> WW], jb[16 >> WW];                                                       \
    group_index<ROW, S, OB, WW>(t, g0, logn, tile, eb, jb);                               \
    const int lowbits = (ROW ? 0 : OB) + g0;                                              \
    if (gi == 0) {                                                                        \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                    \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                  \
        x[r] = load(e);                                                                   \
        if (FIRST) x[r] = u64_to_f64bits(x[r]);                                           \
      }                                                                                   \
    } else {                                                                              \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                    \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                  \
        x[r] = sm[swz<ROW>(e)];                                                           \
      }                                                                                   \
    }                                                                                     \
    if (gi == 0) load.done();                                                             \
    ntt_group_f64<FWD, ROW, S, OB, WW>(x, jb, g0, logn, twf, sm_tw, P, !ROW);             \
    if (lastg) {                                                                          \
      if (LAST) {                                                                         \
        _Pragma("unroll") for (int r = 0; r < 16; ++r) x[r] =                             \
            f64bits_to_residue(x[r], P.qd, P.qinv_d);                                     \
      }                                                                                   \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                    \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                  \
        store.put(r, e, x[r]);                                                            \
      }                                                                                   \
    } else {                                                                              \
      __syncthreads();                                                                    \
      _Pragma("unroll") for (int r = 0; r < 16; ++r) {                                    \
        const int e = eb[r >> WW] | ((r & ((1 << WW) - 1)) << lowbits);                  \
        sm[swz<ROW>(e)] = x[r];                                                           \
      }                                                                                   \
      __syncthreads();                                                                    \
    }                                                                                     \
  }
    if (W == 4) HX_CL_GROUP(4)
    else if (W == 3) HX_CL_GROUP(3)
    else if (W == 2) HX_CL_GROUP(2)
    else if (W == 1) HX_CL_GROUP(1)
#undef HX_CL_GROUP
  }
}

// shared memory: [TILE] data tile, then the ROW twiddles of the CTA's ROW tile
template <int S, int OB>
constexpr int ntt_cluster_smem_bytes() {
  return ntt_smem_bytes<true, S, OB, true>();
}

// One limb instance per cluster of 2^(S - OB) CTAs (blockIdx.x / C).  The
// limb table, src / data addressing and the FP64 class are those of NttArgs.
template <bool FWD, int S, int OB>
__global__ void __launch_bounds__((1 << (S + OB)) / 16, 2) ntt_cluster_kernel(NttArgs a) {
  namespace cg = cooperative_groups;
  constexpr int TILE = 1 << (S + OB);
  constexpr int T = TILE / 16;
  constexpr int C = 1 << (S - OB);
  extern __shared__ u64 dyn_smem[];
  u64* sm = dyn_smem;
  double* sm_tw = reinterpret_cast<double*>(dyn_smem + TILE);
  cg::cluster_group cl = cg::this_cluster();
  const int t = threadIdx.x;
  const int rank = (int)cl.block_rank();  // == blockIdx.x % C (1-D clusters)
  const long long inst = blockIdx.x / C;
  const int per = a.lt.count;
  const long long bidx = inst / per;
  const int ent = (int)(inst % per);
  const int logn = a.logn;  // == 2 S
  const long long N = 1ll << logn;
  u64* base = a.data + ((long long)bidx * a.lt.stride + a.lt.off[ent]) * N;
  const u64* lbase = a.src ? a.src + (long long)bidx * a.src_estride + (long long)a.lt.off[ent] * N : base;
  const PrimeConst P = a.pc[a.lt.prime[ent]];
  const double* twf = FWD ? P.twf_fwd : P.twf_inv;

  // ROW twiddles of ROW tile `rank` (all S stages), cp.async, as ntt_pass_body
  {
    constexpr int kTw = (1 << OB) * ((1 << S) - 1);
    const long long row0 = (long long)rank << OB;
#pragma unroll
    for (int i = 0; i < (kTw + T - 1) / T; ++i) {
      const int m = t + i * T;
      if (m < kTw) {
        const int beta = (S + OB - 1) - (31 - __clz((TILE - 1) - m));
        const int seg = TILE - (TILE >> beta);
        const int k = m - seg;
        const double* srcp = twf + (N >> (beta + 1)) + (row0 << (S - beta - 1)) + k;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(sm_tw + 17 * seg / 16 + row_tw_pad(k));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(srcp) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }

  struct NoDone {
    __device__ void done() const {}
  };
  // phase-A result stays in this CTA's shared memory (swizzled as phase A's layout)
  struct SmStore {
    u64* sm;
    bool row;
    __device__ void put(int r, int e, u64 v) const {
      if (r == 0) __syncthreads();  // the last group's exchange reads are done
      sm[row ? swz<true>(e) : swz<false>(e)] = v;
    }
  };

  if constexpr (FWD) {
    // phase A: COL tile `rank` from HBM (direct coalesced loads)
    struct GLoad : NoDone {
      const u64* p;
      int tile, logn;
      __device__ u64 operator()(int e) const { return p[tile_gofs<false, S, OB>(e, tile, logn)]; }
    } ld{{}, lbase, rank, logn};
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();  // twiddles visible (phase B's ROW pass reads them)
    cl_pass<true, false, S, OB, true, false>(sm, sm_tw, twf, P, rank, logn, ld, SmStore{sm, false});
  } else {
    // phase A: ROW tile `rank` from HBM, staged through sm for coalescing
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int e = r * T + t;
      sm[swz<true>(e)] = lbase[tile_gofs<true, S, OB>(e, rank, logn)];
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    struct SLoad : NoDone {
      const u64* sm;
      __device__ u64 operator()(int e) const { return sm[swz<true>(e)]; }
    } ld{{}, sm};
    cl_pass<false, true, S, OB, true, false>(sm, sm_tw, twf, P, rank, logn, ld, SmStore{sm, true});
  }
  // (cl_pass's last group wrote sm without a trailing barrier; the cluster
  // barrier orders every CTA's phase-A stores before any phase-B remote load)
  cl.sync();

  // phase B: gather this CTA's second-pass tile from the cluster
  struct RLoad {
    cg::cluster_group* cl;
    u64* sm;
    int tile, logn;
    __device__ u64 operator()(int e) const {
      // global index of element e of the phase-B tile, then its phase-A owner
      long long j;
      int owner, eo;
      if constexpr (FWD) {  // phase B = ROW tile `tile`; phase A = COL tiles of 2^OB columns
        j = ((long long)tile << (S + OB)) + e;
        const int row = (int)(j >> S), col = (int)(j & ((1 << S) - 1));
        owner = col >> OB;
        eo = (row << OB) | (col & ((1 << OB) - 1));
        return cl->map_shared_rank(sm, owner)[swz<false>(eo)];
      } else {  // phase B = COL tile `tile`; phase A = ROW tiles of 2^OB rows
        j = tile_gofs<false, S, OB>(e, tile, logn);
        owner = (int)(j >> (S + OB));
        eo = (int)(j & ((1 << (S + OB)) - 1));
        return cl->map_shared_rank(sm, owner)[swz<true>(eo)];
      }
    }
    // every CTA has its words in registers before any CTA reuses its sm
    __device__ void done() const { cl->sync(); }
  } rl{&cl, sm, rank, logn};

  if constexpr (FWD) {
    // ROW pass, last: stage through sm for a coalesced store
    struct RowStore {
      u64* sm;
      u64* base;
      int tile;
      __device__ void put(int r, int e, u64 v) const {
        if (r == 0) __syncthreads();
        sm[swz<true>(e)] = v;
        if (r == 15) {
          __syncthreads();
#pragma unroll
          for (int rr = 0; rr < 16; ++rr) {
            const int ee = rr * T + (int)threadIdx.x;
            base[tile_gofs<true, S, OB>(ee, tile, 2 * S)] = sm[swz<true>(ee)];
          }
        }
      }
    };
    cl_pass<true, true, S, OB, false, true>(sm, sm_tw, twf, P, rank, logn, rl, RowStore{sm, base, rank});
  } else {
    struct ColStore {
      u64* base;
      int tile;
      __device__ void put(int, int e, u64 v) const { base[tile_gofs<false, S, OB>(e, tile, 2 * S)] = v; }
    };
    cl_pass<false, false, S, OB, false, true>(sm, sm_tw, twf, P, rank, logn, rl, ColStore{base, rank});
  }
}

}  // namespace hx
