// hx_ntt.cu -- NTT pass instantiations and launchers (see hx_ntt.cuh).
#include "hx_internal.h"

namespace hx {

namespace {

template <bool FWD, bool ROW, int S>
void launch_pass(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s) {
  constexpr int OB = 4;
  constexpr int TILE = 1 << (S + OB);
  NttArgs a;
  a.data = data;
  a.pc = c->d_pc;
  a.lt = lt;
  a.logn = c->logn;
  a.instances = batch * lt.count;
  const long long tiles = c->N() / TILE;
  const long long blocks = a.instances * tiles;
  if (blocks <= 0) return;
  ntt_pass_kernel<FWD, ROW, S, OB><<<(unsigned)blocks, TILE / 16, 0, s>>>(a);
  ++c->launches;
}

template <bool FWD, bool ROW>
void dispatch(hx_ctx* c, int S, u64* data, long long batch, const LimbTable& lt, cudaStream_t s) {
  switch (S) {
    case 3: launch_pass<FWD, ROW, 3>(c, data, batch, lt, s); break;
    case 4: launch_pass<FWD, ROW, 4>(c, data, batch, lt, s); break;
    case 5: launch_pass<FWD, ROW, 5>(c, data, batch, lt, s); break;
    case 6: launch_pass<FWD, ROW, 6>(c, data, batch, lt, s); break;
    case 7: launch_pass<FWD, ROW, 7>(c, data, batch, lt, s); break;
    case 8: launch_pass<FWD, ROW, 8>(c, data, batch, lt, s); break;
    default: set_error("ntt: unsupported sub-transform size");
  }
}

// N = 2^a (column / high bits) x 2^b (row / low bits), a = ceil(logn/2)
inline int split_a(int logn) { return (logn + 1) / 2; }

}  // namespace

void ntt_forward(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s) {
  const int a = split_a(c->logn), b = c->logn - a;
  dispatch<true, false>(c, a, data, batch, lt, s);  // first a stages (COL)
  dispatch<true, true>(c, b, data, batch, lt, s);   // last b stages (ROW)
}

void ntt_inverse(hx_ctx* c, u64* data, long long batch, const LimbTable& lt, cudaStream_t s) {
  const int a = split_a(c->logn), b = c->logn - a;
  dispatch<false, true>(c, b, data, batch, lt, s);   // low-bit stages (ROW)
  dispatch<false, false>(c, a, data, batch, lt, s);  // high-bit stages (COL), x N^-1
}

}  // namespace hx
