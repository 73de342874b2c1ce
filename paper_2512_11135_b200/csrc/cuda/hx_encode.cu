// hx_encode.cu -- CKKS slot encoding on the device.
//
// Restates CkksEncoder::encode_coeffs (the reference's encoder.cpp:45-117, and
// our host restatement csrc/host/encoder.cpp) operation for operation, so the
// int64 coefficients are bit-identical to the host's:
//   v[k] = (x_j, +0), v[N-1-k] = (x_j, -0)        k = (5^j mod 2N - 1) / 2
//   bit reversal, radix-2 inverse FFT stages len = 2 .. N with the host's
//   w_{j+1} = w_j * wn twiddle sequence (table from the host: the libm values
//   are the host's), complex products as (ac - bd, ad + bc) with separate
//   roundings (__dmul_rn / __dsub_rn / __dadd_rn: no FMA contraction),
//   x (1/N), x conj(zeta^t), real part x scale, llround (half away from 0),
//   capacity check |s| < 2^62 and log2(|s| + 1) < log2(Q_l / 2).
// Layout: stages len <= 2048 run in shared memory on 2048-element tiles (one
// CTA per tile), the remaining log2(N / 2048) stages are one launch each over
// all batch elements; the last one fuses the scale / untwist / rounding and
// writes the coefficients.  The RNS lift and NTT follow (hx_from_i64,
// hx_ntt_fwd).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>

#include "../../../include/hx_b200.h"
#include "hx_internal.h"

struct hx_encoder {
  hx_ctx* ctx = nullptr;
  int logn = 0;
  int* perm = nullptr;        // [N]
  double2* stage_tw = nullptr;  // [N - 1]: stage len at offset len/2 - 1
  double2* zeta = nullptr;    // [N]
  int* flag = nullptr;        // capacity violation
};

namespace {

using hx::u64;
constexpr int kTile = 2048;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {  // (a.x + i a.y)(b.x + i b.y)
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// embedding + bit reversal + stages len = 2 .. min(N, kTile) in shared memory
__global__ void __launch_bounds__(256) enc_tile_kernel(double2* v, const double* m, int len_m, long long m_stride,
                                                       const int* perm, const double2* stage_tw, int logn) {
  __shared__ double2 s[kTile];
  const int N = 1 << logn;
  const int T = min(N, kTile);
  const long long b = blockIdx.y;
  const int base = blockIdx.x * T;
  const double* mb = m + b * m_stride;
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    const int p = perm[base + i];
    const int j = p & 0x7FFFFFFF;
    const double x = j < len_m ? mb[j] : 0.0;
    s[i] = make_double2(x, p < 0 ? -0.0 : 0.0);
  }
  __syncthreads();
  for (int len = 2; len <= T; len <<= 1) {
    const int half = len >> 1;
    const double2* w = stage_tw + (half - 1);
    for (int k = threadIdx.x; k < T / 2; k += blockDim.x) {
      const int blk = k / half, j = k % half;
      const int i0 = blk * len + j, i1 = i0 + half;
      const double2 u = s[i0];
      const double2 t = cmul(w[j], s[i1]);
      s[i0] = make_double2(__dadd_rn(u.x, t.x), __dadd_rn(u.y, t.y));
      s[i1] = make_double2(__dsub_rn(u.x, t.x), __dsub_rn(u.y, t.y));
    }
    __syncthreads();
  }
  double2* vb = v + b * (long long)N + base;
  for (int i = threadIdx.x; i < T; i += blockDim.x) vb[i] = s[i];
}

// one global stage (len > kTile); the last stage (len == N) finishes the encode
__device__ __forceinline__ void finish(double2 x, int t, const double2* zeta, double inv_n, double scale,
                                       double cap, long long* out, int* flag) {
  x = make_double2(__dmul_rn(x.x, inv_n), __dmul_rn(x.y, inv_n));
  const double2 z = zeta[t];
  const double re = __dsub_rn(__dmul_rn(x.x, z.x), __dmul_rn(x.y, -z.y));  // real of x * conj(z)
  const double sc = __dmul_rn(re, scale);
  const double a = fabs(sc);
  if (a >= 4611686018427387904.0 || log2(a + 1.0) >= cap) atomicOr(flag, 1);
  out[t] = llround(sc);
}

__global__ void enc_stage_kernel(double2* v, int len, const double2* stage_tw, int logn, long long* out,
                                 const double2* zeta, double scale, double cap, int* flag) {
  const int N = 1 << logn;
  const long long b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // butterfly index < N / 2
  const int half = len >> 1;
  const int blk = k / half, j = k % half;
  const int i0 = blk * len + j, i1 = i0 + half;
  double2* vb = v + b * (long long)N;
  const double2 u = vb[i0];
  const double2 t = cmul(stage_tw[half - 1 + j], vb[i1]);
  const double2 y0 = make_double2(__dadd_rn(u.x, t.x), __dadd_rn(u.y, t.y));
  const double2 y1 = make_double2(__dsub_rn(u.x, t.x), __dsub_rn(u.y, t.y));
  if (len == N) {
    const double inv_n = 1.0 / (double)N;
    long long* ob = out + b * (long long)N;
    finish(y0, i0, zeta, inv_n, scale, cap, ob, flag);
    finish(y1, i1, zeta, inv_n, scale, cap, ob, flag);
  } else {
    vb[i0] = y0;
    vb[i1] = y1;
  }
}

// N <= kTile: the whole transform ran in the tile kernel; finish per element
__global__ void enc_finish_kernel(const double2* v, int logn, long long* out, const double2* zeta, double scale,
                                  double cap, int* flag) {
  const int N = 1 << logn;
  const long long b = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  finish(v[b * (long long)N + t], t, zeta, 1.0 / (double)N, scale, cap, out + b * (long long)N, flag);
}

template <class F>
int guard_enc(F f) {
  try {
    f();
    return HX_OK;
  } catch (const std::overflow_error& e) {
    return hx::fail(HX_ERR_OVERFLOW, e.what());
  } catch (const std::invalid_argument& e) {
    return hx::fail(HX_ERR_INVALID, e.what());
  } catch (const std::exception& e) {
    return hx::fail(HX_ERR_CUDA, e.what());
  }
}

}  // namespace

extern "C" {

hx_encoder* hx_encoder_create(hx_ctx* c, const int32_t* perm, const double* stage_tw, const double* zeta) {
  if (!c || !perm || !stage_tw || !zeta) return nullptr;
  auto* e = new hx_encoder;
  e->ctx = c;
  e->logn = c->logn;
  const size_t N = (size_t)1 << c->logn;
  bool ok = cudaMalloc((void**)&e->perm, N * 4) == cudaSuccess &&
            cudaMalloc((void**)&e->stage_tw, (N - 1) * 16) == cudaSuccess &&
            cudaMalloc((void**)&e->zeta, N * 16) == cudaSuccess && cudaMalloc((void**)&e->flag, 4) == cudaSuccess;
  ok = ok && cudaMemcpy(e->perm, perm, N * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(e->stage_tw, stage_tw, (N - 1) * 16, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(e->zeta, zeta, N * 16, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    hx_encoder_destroy(e);
    return nullptr;
  }
  return e;
}

void hx_encoder_destroy(hx_encoder* e) {
  if (!e) return;
  for (void* p : {(void*)e->perm, (void*)e->stage_tw, (void*)e->zeta, (void*)e->flag})
    if (p) cudaFree(p);
  delete e;
}

int hx_encode(hx_encoder* e, int64_t* coeffs, const double* m, int len_m, long long m_stride, int batch,
              double scale, double cap_log2, void* stream) {
  return guard_enc([&] {
    if (!e || !coeffs || !m || batch < 0 || len_m < 0) throw std::invalid_argument("hx_encode: bad arguments");
    if (!(scale > 0.0)) throw std::invalid_argument("encode: non-positive scale");
    if (batch == 0) return;
    cudaStream_t s = (cudaStream_t)stream;
    const int N = 1 << e->logn;
    double2* v = nullptr;
    if (cudaMallocAsync((void**)&v, (size_t)batch * N * 16, s) != cudaSuccess)
      throw std::runtime_error("hx_encode: out of device memory");
    cudaMemsetAsync(e->flag, 0, 4, s);
    const int T = std::min(N, kTile);
    enc_tile_kernel<<<dim3((unsigned)(N / T), (unsigned)batch), 256, 0, s>>>(v, m, len_m, m_stride, e->perm,
                                                                             e->stage_tw, e->logn);
    e->ctx->launches++;
    if (N <= kTile) {
      enc_finish_kernel<<<dim3((unsigned)((N + 255) / 256), (unsigned)batch), 256, 0, s>>>(
          v, e->logn, (long long*)coeffs, e->zeta, scale, cap_log2, e->flag);
      e->ctx->launches++;
    } else {
      for (int len = 2 * kTile; len <= N; len <<= 1) {
        enc_stage_kernel<<<dim3((unsigned)(N / 2 / 256), (unsigned)batch), 256, 0, s>>>(
            v, len, e->stage_tw, e->logn, (long long*)coeffs, e->zeta, scale, cap_log2, e->flag);
        e->ctx->launches++;
      }
    }
    int flag = 0;
    cudaMemcpyAsync(&flag, e->flag, 4, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(v, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) throw std::runtime_error("hx_encode: device error");
    if (flag) throw std::overflow_error("encode: coefficient exceeds modulus capacity");
  });
}

}  // extern "C"
