// gpu_backend.cpp -- helix::GpuLatticeBackend over libhx_b200 (see header).
//
// Bookkeeping mirrors reference_backend.cpp:63-139 (level/scale checks,
// trace records, rotation-key checks); the arithmetic is the lattice backend
// of SPEC.md:143-245 with hybrid key switching.  Randomness: xoshiro256**
// seeded by splitmix64 (secret key ternary, uniform `a`, centred-binomial
// errors with k = 21, sigma ~ 3.24 ~ the spec's 3.2).  INSECURE TOY
// PARAMETERS: requires params.insecure_toy.
#include "helix/gpu_backend.hpp"
#include "helix/packing.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

#include "hx_b200.h"

namespace helix {

namespace {
using u64 = std::uint64_t;

void ck(int rc, const char* what) {
  if (rc != HX_OK) throw std::runtime_error(std::string(what) + ": " + hx_last_error());
}
void cuda_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
u64 splitmix(u64& x) {
  u64 z = (x += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
u64 rotl(u64 x, int k) { return (x << k) | (x >> (64 - k)); }
}  // namespace

// xoshiro256**
std::uint64_t GpuLatticeBackend::next_u64() {
  const u64 r = rotl(rng_[1] * 5, 7) * 9;
  const u64 t = rng_[1] << 17;
  rng_[2] ^= rng_[0];
  rng_[3] ^= rng_[1];
  rng_[1] ^= rng_[2];
  rng_[0] ^= rng_[3];
  rng_[2] ^= t;
  rng_[3] = rotl(rng_[3], 45);
  return r;
}

// ------------------------------------------------- backend stream / lock
namespace {
// the stream (and its owner) of the backend operation running on this thread
thread_local cudaStream_t tl_stream = nullptr;
thread_local const std::shared_ptr<void>* tl_owner = nullptr;
cudaStream_t cur() { return tl_stream; }
}  // namespace

struct GpuLatticeBackend::DeviceScope {
  std::unique_lock<std::recursive_mutex> lk;
  cudaStream_t prev_s;
  const std::shared_ptr<void>* prev_o;
  explicit DeviceScope(const GpuLatticeBackend& b) : lk(b.mu_), prev_s(tl_stream), prev_o(tl_owner) {
    tl_stream = static_cast<cudaStream_t>(b.stream_.get());
    tl_owner = &b.stream_;
  }
  ~DeviceScope() {
    tl_stream = prev_s;
    tl_owner = prev_o;
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

// ------------------------------------------------------------- DeviceBuffer
DeviceBuffer::DeviceBuffer(std::size_t w) : words(w) {
  if (!w) return;
  stream = cur();
  if (tl_owner) stream_ref = *tl_owner;
  if (cudaMallocAsync((void**)&ptr, w * 8, cur()) == cudaSuccess) return;
  // the pool may hold freed blocks too small for this request (e.g. the
  // packed forms of a matrix swapped for one another): release them to the
  // device and try once more
  cudaGetLastError();
  ptr = nullptr;
  if (getenv("HX_ALLOC_TRACE")) fprintf(stderr, "[helix] pool trim + retry for %.2f GB\n", w * 8e-9);
  cuda_ck(cudaDeviceSynchronize(), "sync");
  int dev = 0;
  cudaMemPool_t pool;
  cuda_ck(cudaGetDevice(&dev), "device");
  cuda_ck(cudaDeviceGetDefaultMemPool(&pool, dev), "mem pool");
  cuda_ck(cudaMemPoolTrimTo(pool, 0), "mem pool trim");
  cuda_ck(cudaMallocAsync((void**)&ptr, w * 8, cur()), "cudaMallocAsync");
}
DeviceBuffer::~DeviceBuffer() {
  if (ptr) cudaFreeAsync(ptr, static_cast<cudaStream_t>(stream));
}

static std::shared_ptr<DeviceBuffer> dev(std::size_t words) {
  return std::make_shared<DeviceBuffer>(words);
}

// ------------------------------------------------------------- construction
GpuLatticeBackend::GpuLatticeBackend(CkksParams params, std::uint64_t seed)
    : params_(std::move(params)), enc_(params_) {
  params_.validate();
  if (!params_.insecure_toy)
    throw std::invalid_argument("GpuLatticeBackend: parameters must set insecure_toy (toy CKKS)");
  if (params_.special_primes.empty())
    throw std::invalid_argument("GpuLatticeBackend: at least one special prime required");
  int logn = 0;
  while ((1ull << logn) < params_.ring_degree) ++logn;
  ctx_ = hx_ctx_create(logn, params_.moduli.data(), (int)params_.moduli.size(),
                       params_.special_primes.data(), (int)params_.special_primes.size(),
                       params_.digit_size);
  if (!ctx_) throw std::runtime_error(std::string("hx_ctx_create: ") + hx_last_error());
  cudaStream_t st = nullptr;
  cuda_ck(cudaStreamCreate(&st), "backend stream");
  stream_ = std::shared_ptr<void>(st, [](void* p) {
    cudaStreamSynchronize(static_cast<cudaStream_t>(p));
    cudaStreamDestroy(static_cast<cudaStream_t>(p));
  });
  DeviceScope ds(*this);
  u64 sm = seed;
  for (auto& w : rng_) w = splitmix(sm);
  const std::size_t N = params_.ring_degree;
  const int nc = (int)params_.moduli.size(), K = (int)params_.special_primes.size();
  // secret key: ternary, NTT form over the full basis
  std::vector<std::int64_t> s(N);
  for (auto& c : s) {
    u64 r;
    do r = next_u64() & 3;
    while (r == 3);
    c = (std::int64_t)r - 1;
  }
  DeviceBuffer sv(N);
  cuda_ck(cudaMemcpyAsync(sv.ptr, s.data(), N * 8, cudaMemcpyHostToDevice, cur()), "h2d");
  s_full_ = dev((std::size_t)(nc + K) * N);
  ck(hx_from_i64(ctx_, s_full_->ptr, (const int64_t*)sv.ptr, 1, nc, K, cur()), "from_i64");
  ck(hx_ntt_fwd(ctx_, s_full_->ptr, 1, nc, K, cur()), "ntt");
  // relinearisation key (s' = s^2)
  auto s2 = dev((std::size_t)(nc + K) * N);
  ck(hx_mul(ctx_, s2->ptr, s_full_->ptr, s_full_->ptr, 1, nc, K, cur()), "mul");
  rlk_ = make_key(s2, 0);
  cuda_ck(cudaStreamSynchronize(cur()), "sync");
}

GpuLatticeBackend::~GpuLatticeBackend() {
  rot_keys_.clear();
  rlk_.reset();
  s_full_.reset();
  matmul_masks_.clear();
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream_.get()));
  hx_encoder_destroy(henc_);
  hx_ctx_destroy(ctx_);  // forgets the compressed keys with the context
}

void GpuLatticeBackend::sample_uniform(std::vector<u64>& out, int lc, int ls, int copies) {
  const std::size_t N = params_.ring_degree;
  out.resize((std::size_t)copies * (lc + ls) * N);
  auto next = [&]() { return next_u64(); };
  std::size_t o = 0;
  for (int c = 0; c < copies; ++c)
    for (int l = 0; l < lc + ls; ++l) {
      const u64 q = l < lc ? params_.moduli[l] : params_.special_primes[l - lc];
      int bits = 64 - __builtin_clzll(q);
      const u64 mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
      for (std::size_t t = 0; t < N; ++t) {
        u64 v;
        do v = next() & mask;
        while (v >= q);
        out[o++] = v;
      }
    }
}

void GpuLatticeBackend::sample_error(std::vector<std::int64_t>& out, int copies) {
  const std::size_t N = params_.ring_degree;
  out.resize((std::size_t)copies * N);
  for (auto& e : out) {
    const u64 r = next_u64();
    // centred binomial, k = 21: popcount(21 bits) - popcount(21 bits)
    e = (std::int64_t)__builtin_popcountll(r & 0x1fffff) - (std::int64_t)__builtin_popcountll((r >> 21) & 0x1fffff);
  }
}

std::shared_ptr<DeviceBuffer> GpuLatticeBackend::make_key(const std::shared_ptr<DeviceBuffer>& sp,
                                                          std::uint64_t g) {
  // Key material from two seeds of the backend's stream: the uniform halves
  // are the counter stream of the first (hx_sample_uniform), the CBD errors of
  // the second.  compress_keys: store only the b halves and
  // regenerate the uniform halves inside the key inner product (half the key
  // bytes; the same key words either way).
  const int nc = (int)params_.moduli.size();
  const int dn = hx_ctx_dnum(ctx_, nc);
  const std::size_t N = params_.ring_degree;
  DeviceBuffer de((std::size_t)dn * N);
  const std::uint64_t seed = next_u64();
  ck(hx_sample_cbd(ctx_, (int64_t*)de.ptr, (long long)dn * N, next_u64(), cur()), "sample_cbd");
  std::shared_ptr<DeviceBuffer> key;
  if (params_.compress_keys) {
    key = dev(hx_ckey_words(ctx_));
    if (g == 0)
      ck(hx_keygen_ksk_c(ctx_, key->ptr, s_full_->ptr, sp->ptr, seed, (const int64_t*)de.ptr, cur()), "keygen");
    else
      ck(hx_keygen_rotation_c(ctx_, key->ptr, s_full_->ptr, g, seed, (const int64_t*)de.ptr, cur()),
         "keygen_rotation");
  } else {  // full keys: the same words, the uniform halves materialised
    const int K = (int)params_.special_primes.size();
    DeviceBuffer da((std::size_t)dn * (nc + K) * N);
    ck(hx_sample_uniform(ctx_, da.ptr, nc, K, dn, seed, cur()), "sample_uniform");
    key = dev(hx_key_words(ctx_));
    if (g == 0)
      ck(hx_keygen_ksk(ctx_, key->ptr, s_full_->ptr, sp->ptr, da.ptr, (const int64_t*)de.ptr, cur()), "keygen");
    else
      ck(hx_keygen_rotation(ctx_, key->ptr, s_full_->ptr, g, da.ptr, (const int64_t*)de.ptr, cur()),
         "keygen_rotation");
  }
  cuda_ck(cudaStreamSynchronize(cur()), "sync");  // da / de die here
  return key;
}

void GpuLatticeBackend::expand_key(const std::uint64_t* key, std::uint64_t* full) const {
  DeviceScope ds(*this);
  if (params_.compress_keys)
    ck(hx_key_expand(ctx_, full, key, cur()), "key_expand");
  else
    cuda_ck(cudaMemcpyAsync(full, key, hx_key_words(ctx_) * 8, cudaMemcpyDeviceToDevice, cur()), "d2d");
  cuda_ck(cudaStreamSynchronize(cur()), "sync");
}

std::uint64_t GpuLatticeBackend::galois(std::int64_t r) const {
  const u64 two_n = 2 * params_.ring_degree;
  u64 g = 1, b = 5;
  for (u64 e = (u64)r; e; e >>= 1) {
    if (e & 1) g = g * b % two_n;
    b = b * b % two_n;
  }
  return g;
}

void GpuLatticeBackend::generate_rotation_keys(std::span<const std::int64_t> amounts) {
  DeviceScope ds(*this);
  const auto n = (std::int64_t)slots();
  for (std::int64_t a : amounts) {
    const std::int64_t r = detail::reduce_amount(a, n);
    rot_set_.insert(r);
    if (r == 0 || rot_keys_.count(r)) continue;
    rot_keys_[r] = make_key(nullptr, galois(r));
  }
}

const std::uint64_t* GpuLatticeBackend::rotation_key(std::int64_t r) const {
  DeviceScope ds(*this);
  auto it = rot_keys_.find(r);
  return it == rot_keys_.end() ? nullptr : it->second->ptr;
}

void GpuLatticeBackend::trim() {
  DeviceScope ds(*this);
  cuda_ck(cudaStreamSynchronize(cur()), "sync");
  ck(hx_ctx_trim(ctx_), "trim");
}

const GpuCiphertext& GpuLatticeBackend::payload(const Ciphertext& ct) {
  auto* p = dynamic_cast<const GpuCiphertext*>(ct.payload.get());
  if (!p) throw std::invalid_argument("ciphertext does not belong to the GPU backend");
  return *p;
}
const GpuPlaintext& GpuLatticeBackend::payload(const Plaintext& pt) {
  auto* p = dynamic_cast<const GpuPlaintext*>(pt.payload.get());
  if (!p) throw std::invalid_argument("plaintext does not belong to the GPU backend");
  return *p;
}

Ciphertext GpuLatticeBackend::wrap(std::shared_ptr<DeviceBuffer> buf, std::size_t offset, int level,
                                   const Scale& scale) const {
  auto p = std::make_shared<GpuCiphertext>();
  p->buf = std::move(buf);
  p->offset = offset;
  p->n_q = level + 1;
  Ciphertext ct;
  ct.payload = std::move(p);
  ct.level = level;
  ct.scale = scale;
  ct.slot_count = slots();
  ct.id = next_handle_id();
  return ct;
}

// ------------------------------------------------------------- encode / decode
// Encoding runs on the device (hx_encode, bit-identical to CkksEncoder::
// encode_coeffs), then the RNS lift and NTT; messages go in chunks of 1024.
void GpuLatticeBackend::encode_device(const std::vector<const std::vector<double>*>& msgs, int level,
                                      const Scale& scale, std::uint64_t* out) {
  if (!scale.is_positive()) throw std::invalid_argument("encode: non-positive scale");
  if (level < 0 || level > params_.max_level) throw std::invalid_argument("encode: level out of range");
  const std::size_t N = params_.ring_degree, S = slots();
  for (const auto* m : msgs)
    if (m->size() > S) throw std::invalid_argument("encode: vector longer than slot count");
  if (!henc_) {
    std::vector<std::int32_t> perm;
    std::vector<double> tw, zeta;
    enc_.device_tables(perm, tw, zeta);
    henc_ = hx_encoder_create(ctx_, perm.data(), tw.data(), zeta.data());
    if (!henc_) throw std::runtime_error("hx_encoder_create failed");
  }
  const int n = nq(level);
  const double cap = enc_.capacity_log2(level);
  const std::size_t chunk = std::min<std::size_t>(msgs.size(), 1024);
  std::size_t width = 1;
  for (const auto* m : msgs) width = std::max(width, m->size());
  std::vector<double> host(chunk * width);
  DeviceBuffer dm(chunk * width), dc(chunk * N);
  for (std::size_t c0 = 0; c0 < msgs.size(); c0 += chunk) {
    const std::size_t k = std::min(chunk, msgs.size() - c0);
    std::fill(host.begin(), host.end(), 0.0);
    for (std::size_t i = 0; i < k; ++i)
      std::memcpy(host.data() + i * width, msgs[c0 + i]->data(), msgs[c0 + i]->size() * 8);
    cuda_ck(cudaMemcpy(dm.ptr, host.data(), k * width * 8, cudaMemcpyHostToDevice), "h2d");
    const int rc = hx_encode(henc_, (int64_t*)dc.ptr, (const double*)dm.ptr, (int)width, (long long)width, (int)k,
                             scale.to_double(), cap, cur());
    if (rc == HX_ERR_OVERFLOW) throw std::overflow_error(hx_last_error());
    ck(rc, "encode");
    std::uint64_t* o = out + c0 * n * N;
    ck(hx_from_i64(ctx_, o, (const int64_t*)dc.ptr, (int)k, n, 0, cur()), "from_i64");
    ck(hx_ntt_fwd(ctx_, o, (int)k, n, 0, cur()), "ntt");
  }
  cuda_ck(cudaStreamSynchronize(cur()), "sync");
}

Plaintext GpuLatticeBackend::encode(std::span<const double> m, int level, const Scale& scale) {
  DeviceScope ds(*this);
  if (m.size() > slots()) throw std::invalid_argument("encode: vector longer than slot count");
  if (!scale.is_positive()) throw std::invalid_argument("encode: non-positive scale");
  if (level < 0 || level > params_.max_level) throw std::invalid_argument("encode: level out of range");
  const std::vector<double> v(m.begin(), m.end());
  auto buf = dev((std::size_t)nq(level) * params_.ring_degree);
  encode_device({&v}, level, scale, buf->ptr);
  auto p = std::make_shared<GpuPlaintext>();
  p->buf = buf;
  p->n_q = nq(level);
  Plaintext pt;
  pt.payload = p;
  pt.level = level;
  pt.scale = scale;
  pt.slot_count = slots();
  return pt;
}

std::vector<Plaintext> GpuLatticeBackend::encode_many(const std::vector<std::vector<double>>& msgs,
                                                      int level, const Scale& scale) {
  DeviceScope ds(*this);
  if (level < 0 || level > params_.max_level) throw std::invalid_argument("encode: level out of range");
  const std::size_t N = params_.ring_degree;
  const int n = nq(level);
  std::vector<const std::vector<double>*> src;  // non-empty messages
  for (const auto& m : msgs)
    if (!m.empty()) src.push_back(&m);
  std::vector<Plaintext> out(msgs.size());
  for (auto& pt : out) {
    pt.level = level;
    pt.scale = scale;
    pt.slot_count = slots();
  }
  if (src.empty()) return out;
  auto buf = dev(src.size() * n * N);
  encode_device(src, level, scale, buf->ptr);
  std::size_t idx = 0;
  for (std::size_t i = 0; i < msgs.size(); ++i) {
    if (msgs[i].empty()) continue;
    auto p = std::make_shared<GpuPlaintext>();
    p->buf = buf;
    p->offset = idx * n * N;
    p->n_q = n;
    out[i].payload = p;
    ++idx;
  }
  return out;
}

std::vector<double> GpuLatticeBackend::decode(const Plaintext& pt) {
  DeviceScope ds(*this);
  const std::size_t N = params_.ring_degree;
  const int n = nq(pt.level);
  if (!pt.payload) return std::vector<double>(slots(), 0.0);
  const auto& p = payload(pt);
  DeviceBuffer tmp((std::size_t)n * N);
  cuda_ck(cudaMemcpyAsync(tmp.ptr, p.data(), (std::size_t)n * N * 8, cudaMemcpyDeviceToDevice, cur()), "d2d");
  ck(hx_ntt_inv(ctx_, tmp.ptr, 1, n, 0, cur()), "intt");
  std::vector<u64> limbs((std::size_t)n * N);
  cuda_ck(cudaMemcpyAsync(limbs.data(), tmp.ptr, limbs.size() * 8, cudaMemcpyDeviceToHost, cur()), "d2h");
  cuda_ck(cudaStreamSynchronize(cur()), "sync");
  return enc_.decode_coeffs(limbs, n, pt.scale.to_double());
}

// ------------------------------------------------------------- encrypt / decrypt
Ciphertext GpuLatticeBackend::encrypt(const Plaintext& pt) {
  DeviceScope ds(*this);
  const std::size_t N = params_.ring_degree;
  const int n = nq(pt.level);
  std::vector<u64> a;
  std::vector<std::int64_t> e;
  sample_uniform(a, n, 0, 1);
  sample_error(e, 1);
  DeviceBuffer da(a.size()), de(e.size());
  cuda_ck(cudaMemcpyAsync(da.ptr, a.data(), a.size() * 8, cudaMemcpyHostToDevice, cur()), "h2d");
  cuda_ck(cudaMemcpyAsync(de.ptr, e.data(), e.size() * 8, cudaMemcpyHostToDevice, cur()), "h2d");
  std::shared_ptr<DeviceBuffer> zero;
  const u64* m;
  if (pt.payload) {
    m = payload(pt).data();
  } else {
    zero = dev((std::size_t)n * N);
    cuda_ck(cudaMemsetAsync(zero->ptr, 0, (std::size_t)n * N * 8, cur()), "memset");
    m = zero->ptr;
  }
  auto buf = dev((std::size_t)2 * n * N);
  ck(hx_encrypt_sk(ctx_, buf->ptr, m, s_full_->ptr, da.ptr, (const int64_t*)de.ptr, n, cur()), "encrypt");
  cuda_ck(cudaStreamSynchronize(cur()), "sync");
  return wrap(buf, 0, pt.level, pt.scale);
}

std::vector<double> GpuLatticeBackend::decrypt(const Ciphertext& ct) {
  DeviceScope ds(*this);
  const std::size_t N = params_.ring_degree;
  const int n = nq(ct.level);
  auto buf = dev((std::size_t)n * N);
  ck(hx_decrypt(ctx_, buf->ptr, payload(ct).data(), s_full_->ptr, 1, n, cur()), "decrypt");
  auto p = std::make_shared<GpuPlaintext>();
  p->buf = buf;
  p->n_q = n;
  Plaintext pt;
  pt.payload = p;
  pt.level = ct.level;
  pt.scale = ct.scale;
  pt.slot_count = slots();
  return decode(pt);
}

// ------------------------------------------------------------- SlotOps
Ciphertext GpuLatticeBackend::add(const Ciphertext& a, const Ciphertext& b) {
  DeviceScope ds(*this);
  detail::require_same_level(a.level, b.level, "add");
  detail::require_same_scale(a.scale, b.scale, "add");
  const int n = nq(a.level);
  auto buf = dev((std::size_t)2 * n * params_.ring_degree);
  ck(hx_add(ctx_, buf->ptr, payload(a).data(), payload(b).data(), 2, n, 0, cur()), "add");
  trace_.record(OpKind::CtAdd, a.level);
  return wrap(buf, 0, a.level, a.scale);
}

Ciphertext GpuLatticeBackend::add_plain(const Ciphertext& a, const Plaintext& b) {
  DeviceScope ds(*this);
  detail::require_same_level(a.level, b.level, "add_plain");
  detail::require_same_scale(a.scale, b.scale, "add_plain");
  const std::size_t N = params_.ring_degree;
  const int n = nq(a.level);
  auto buf = dev((std::size_t)2 * n * N);
  const u64* ad = payload(a).data();
  if (b.payload)
    ck(hx_add(ctx_, buf->ptr, ad, payload(b).data(), 1, n, 0, cur()), "add");
  else
    cuda_ck(cudaMemcpyAsync(buf->ptr, ad, (std::size_t)n * N * 8, cudaMemcpyDeviceToDevice, cur()), "d2d");
  cuda_ck(cudaMemcpyAsync(buf->ptr + (std::size_t)n * N, ad + (std::size_t)n * N, (std::size_t)n * N * 8,
                          cudaMemcpyDeviceToDevice, cur()), "d2d");
  trace_.record(OpKind::PtAdd, a.level);
  return wrap(buf, 0, a.level, a.scale);
}

Ciphertext GpuLatticeBackend::mul(const Ciphertext& a, const Ciphertext& b) {
  DeviceScope ds(*this);
  detail::require_same_level(a.level, b.level, "mul");
  if (a.level < 1) throw LevelUnderflowError("mul: no level left for a following rescale");
  const int n = nq(a.level);
  auto buf = dev((std::size_t)2 * n * params_.ring_degree);
  ck(hx_mul_relin(ctx_, buf->ptr, payload(a).data(), payload(b).data(), rlk_->ptr, 1, n, cur()), "mul_relin");
  trace_.record(OpKind::CtMul, a.level);
  return wrap(buf, 0, a.level, a.scale * b.scale);
}

Ciphertext GpuLatticeBackend::mul_plain(const Ciphertext& a, const Plaintext& b) {
  DeviceScope ds(*this);
  detail::require_same_level(a.level, b.level, "mul_plain");
  if (a.level < 1) throw LevelUnderflowError("mul_plain: no level left for a following rescale");
  const std::size_t N = params_.ring_degree;
  const int n = nq(a.level);
  auto buf = dev((std::size_t)2 * n * N);
  if (!b.payload) {
    cuda_ck(cudaMemsetAsync(buf->ptr, 0, (std::size_t)2 * n * N * 8, cur()), "memset");
  } else {
    const u64* ad = payload(a).data();
    const u64* bd = payload(b).data();
    ck(hx_mul(ctx_, buf->ptr, ad, bd, 1, n, 0, cur()), "mul");
    ck(hx_mul(ctx_, buf->ptr + (std::size_t)n * N, ad + (std::size_t)n * N, bd, 1, n, 0, cur()), "mul");
  }
  trace_.record(OpKind::PtMul, a.level);
  return wrap(buf, 0, a.level, a.scale * b.scale);
}

Ciphertext GpuLatticeBackend::rotate(const Ciphertext& a, std::int64_t k) {
  DeviceScope ds(*this);
  const auto n = (std::int64_t)slots();
  const std::int64_t r = detail::reduce_amount(k, n);
  const std::size_t N = params_.ring_degree;
  const int nqv = nq(a.level);
  if (r == 0) {
    auto buf = dev((std::size_t)2 * nqv * N);
    cuda_ck(cudaMemcpyAsync(buf->ptr, payload(a).data(), (std::size_t)2 * nqv * N * 8,
                            cudaMemcpyDeviceToDevice, cur()), "d2d");
    return wrap(buf, 0, a.level, a.scale);
  }
  const u64* key = rotation_key(r);
  if (!rot_set_.contains(r) || !key) throw MissingRotationKeyError("rotate: no key for amount " + std::to_string(r));
  auto buf = dev((std::size_t)2 * nqv * N);
  ck(hx_rotate(ctx_, buf->ptr, payload(a).data(), key, 1, nqv, galois(r), cur()), "rotate");
  trace_.record(OpKind::Rotate, a.level);
  return wrap(buf, 0, a.level, a.scale);
}

Ciphertext GpuLatticeBackend::rescale(const Ciphertext& a) {
  DeviceScope ds(*this);
  if (a.level < 1) throw LevelUnderflowError("rescale: no levels remain");
  if (!(a.scale.log2() > params_.delta().log2()))
    throw std::invalid_argument("rescale: scale not above Delta (no multiplication preceded)");
  const int n = nq(a.level);
  auto buf = dev((std::size_t)2 * (n - 1) * params_.ring_degree);
  ck(hx_rescale(ctx_, buf->ptr, payload(a).data(), 2, n, cur()), "rescale");
  trace_.record(OpKind::Rescale, a.level);
  return wrap(buf, 0, a.level - 1, a.scale / Scale::prime(modulus_at(a.level)));
}

Ciphertext GpuLatticeBackend::mod_down(const Ciphertext& a, int target) {
  DeviceScope ds(*this);
  if (target > a.level) throw std::invalid_argument("mod_down: target level above current level");
  if (target < 0) throw std::invalid_argument("mod_down: negative target level");
  const std::size_t N = params_.ring_degree;
  const int n = nq(a.level), t = nq(target);
  auto buf = dev((std::size_t)2 * t * N);
  cuda_ck(cudaMemcpy2DAsync(buf->ptr, (std::size_t)t * N * 8, payload(a).data(), (std::size_t)n * N * 8,
                            (std::size_t)t * N * 8, 2, cudaMemcpyDeviceToDevice, cur()),
          "memcpy2d");
  if (target != a.level) trace_.record(OpKind::ModDown, a.level);
  return wrap(buf, 0, target, a.scale);
}

Ciphertext GpuLatticeBackend::bootstrap(const Ciphertext& a) {
  DeviceScope ds(*this);
  if (!params_.mock_bootstrap)
    throw std::runtime_error("bootstrap: only the insecure mock refresh is implemented (mock_bootstrap=false)");
  trace_.record(OpKind::Bootstrap, a.level);
  const auto v = decrypt(a);
  return encrypt(encode(v, params_.l_boot(), params_.delta()));
}

// ------------------------------------------------------------- fused pipelines
std::vector<Ciphertext> GpuLatticeBackend::rotate_many(const Ciphertext& a,
                                                       std::span<const std::int64_t> amounts) {
  DeviceScope ds(*this);
  const auto n = (std::int64_t)slots();
  const std::size_t N = params_.ring_degree;
  const int nqv = nq(a.level);
  const std::size_t ctw = (std::size_t)2 * nqv * N;
  std::vector<const u64*> keys;
  std::vector<u64> gs;
  std::vector<std::size_t> which;
  for (std::size_t i = 0; i < amounts.size(); ++i) {
    const std::int64_t r = detail::reduce_amount(amounts[i], n);
    if (r == 0) continue;
    const u64* key = rotation_key(r);
    if (!rot_set_.contains(r) || !key) throw MissingRotationKeyError("rotate: no key for amount " + std::to_string(r));
    keys.push_back(key);
    gs.push_back(galois(r));
    which.push_back(i);
  }
  auto buf = dev(amounts.size() * ctw);
  if (!keys.empty()) {
    // hoisted outputs land contiguously; identity rotations are copied after
    auto tmp = dev(keys.size() * ctw);
    ck(hx_rotate_hoisted(ctx_, tmp->ptr, payload(a).data(), keys.data(), gs.data(), (int)keys.size(), 1,
                         nqv, cur()), "rotate_hoisted");
    for (std::size_t j = 0; j < which.size(); ++j)
      cuda_ck(cudaMemcpyAsync(buf->ptr + which[j] * ctw, tmp->ptr + j * ctw, ctw * 8, cudaMemcpyDeviceToDevice,
                              cur()), "d2d");
    trace_.record(OpKind::Rotate, a.level, keys.size());
  }
  std::vector<Ciphertext> out;
  for (std::size_t i = 0; i < amounts.size(); ++i) {
    if (detail::reduce_amount(amounts[i], n) == 0)
      cuda_ck(cudaMemcpyAsync(buf->ptr + i * ctw, payload(a).data(), ctw * 8, cudaMemcpyDeviceToDevice, cur()),
              "d2d");
    out.push_back(wrap(buf, i * ctw, a.level, a.scale));
  }
  return out;
}

Ciphertext GpuLatticeBackend::matmul(const Ciphertext& A, const Ciphertext& B, int d) {
  DeviceScope ds(*this);
  return matmul_heads({A}, {B}, d).front();
}

// H independent products (attention heads) through one schedule: every
// buffer is laid out [j][h][ct], so each rotation launch covers all heads and
// reads its key once (the multi-key rotation groups the H heads of column j
// under key j), the d x H ct-ct products share one relinearisation-key read,
// and the d masks are applied by broadcast (hx_mul_bcast) without replicas.
// Heads are processed in chunks bounded by device memory.
std::vector<Ciphertext> GpuLatticeBackend::matmul_heads(const std::vector<Ciphertext>& As,
                                                        const std::vector<Ciphertext>& Bs, int d) {
  DeviceScope ds(*this);
  const std::size_t N = params_.ring_degree, n = slots();
  if (As.empty() || As.size() != Bs.size()) throw std::invalid_argument("matmul_heads: operand count");
  const Ciphertext& A0 = As[0];
  for (std::size_t h = 0; h < As.size(); ++h) {
    detail::require_same_level(As[h].level, Bs[h].level, "matmul_ctct");
    detail::require_same_level(As[h].level, A0.level, "matmul_heads");
    if (As[h].scale != A0.scale || Bs[h].scale != Bs[0].scale) throw ScaleMismatchError("matmul_heads: scales differ");
  }
  if (A0.level < 2) throw LevelUnderflowError("matmul_ctct: requires a multiplicative level of 2");
  const int lv = A0.level, nqa = nq(lv), nqb = nqa - 1, lg = __builtin_ctz((unsigned)d);
  const std::size_t cw = (std::size_t)2 * nqa * N, cwb = (std::size_t)2 * nqb * N;
  const Scale ms = Scale::prime(modulus_at(lv));
  const Scale ms_b = ms * Scale::prime(modulus_at(lv - 1)) / params_.delta();
  const auto need = [&](std::int64_t k) {
    const std::int64_t r = detail::reduce_amount(k, (std::int64_t)n);
    const u64* key = rotation_key(r);
    if (!rot_set_.contains(r) || !key) throw MissingRotationKeyError("rotate: no key for amount " + std::to_string(r));
    return std::pair<const u64*, u64>{key, galois(r)};
  };
  // the d column / row extraction masks, encoded once per (d, level) and cached
  auto it = matmul_masks_.find({d, lv});
  if (it == matmul_masks_.end()) {
    std::vector<std::vector<double>> cmv, rmv;
    for (int j = 0; j < d; ++j) {
      cmv.push_back(make_mask(MaskKind::ColumnExtractor, j, d, n));
      rmv.push_back(make_mask(MaskKind::RowExtractor, j, d, n));
    }
    it = matmul_masks_.emplace(std::make_pair(d, lv), std::make_pair(encode_many(cmv, lv, ms), encode_many(rmv, lv, ms_b)))
             .first;
  }
  const auto& cm = it->second.first;
  const auto& rm = it->second.second;
  // heads per chunk: ~6 buffers of d x (level ct) plus the rotations' ModUp digits
  const int H_all = (int)As.size();
  const std::size_t dnum = (std::size_t)hx_ctx_dnum(ctx_, nqb), ext = nqb + params_.special_primes.size();
  const std::size_t per_head = (std::size_t)d * 8 * (3 * cw + 4 * cwb + dnum * ext * N);
  std::size_t free_b = 0, total_b = 0;
  cuda_ck(cudaMemGetInfo(&free_b, &total_b), "mem info");
  const int Hc = (int)std::max<std::size_t>(1, std::min<std::size_t>(H_all, (free_b * 6 / 10) / std::max<std::size_t>(per_head, 1)));
  std::vector<Ciphertext> outs;
  for (int h0 = 0; h0 < H_all; h0 += Hc) {
    const int H = std::min(Hc, H_all - h0);
    auto in = dev((std::size_t)H * cw), prod = dev((std::size_t)d * H * cw);
    auto sa = dev((std::size_t)d * H * cwb), sb = dev((std::size_t)d * H * cwb), tmp = dev((std::size_t)d * H * cwb);
    const auto side = [&](const std::vector<Ciphertext>& X, const std::vector<Plaintext>& masks,
                          const std::shared_ptr<DeviceBuffer>& out, std::int64_t unit) {
      for (int h = 0; h < H; ++h)
        cuda_ck(cudaMemcpyAsync(in->ptr + h * cw, payload(X[h0 + h]).data(), cw * 8, cudaMemcpyDeviceToDevice,
                                cur()), "d2d");
      // prod[j][h][c] = X_h[c] (.) mask_j  (encode_many: masks contiguous [d][nqa][N])
      ck(hx_mul_bcast(ctx_, prod->ptr, in->ptr, payload(masks[0]).data(), 2 * d * H, 2 * H, 2 * H, nqa, cur()),
         "mul_bcast");
      ck(hx_rescale(ctx_, out->ptr, prod->ptr, 2 * d * H, nqa, cur()), "rescale");
      // column / row j -> 0 for j >= 1: key j applied to the H heads of column j
      if (d > 1) {
        std::vector<const u64*> keys;
        std::vector<u64> gal;
        for (int j = 1; j < d; ++j) {
          const auto kg = need(unit * j);
          keys.push_back(kg.first);
          gal.push_back(kg.second);
        }
        ck(hx_rotate_grouped(ctx_, tmp->ptr, out->ptr + (std::size_t)H * cwb, keys.data(), gal.data(), d - 1, H, nqb,
                             cur()),
           "rotate_grouped");
        cuda_ck(cudaMemcpyAsync(out->ptr + (std::size_t)H * cwb, tmp->ptr, (std::size_t)(d - 1) * H * cwb * 8,
                                cudaMemcpyDeviceToDevice, cur()), "d2d");
      }
      // replicate: x += Rot_{-unit 2^i}(x), i < log2 d, all d x H at once (one key read)
      for (int i = 0; i < lg; ++i) {
        const auto kg = need(-(unit << i));
        ck(hx_rotate(ctx_, tmp->ptr, out->ptr, kg.first, d * H, nqb, kg.second, cur()), "rotate");
        ck(hx_add(ctx_, out->ptr, out->ptr, tmp->ptr, 2 * d * H, nqb, 0, cur()), "add");
      }
    };
    side(As, cm, sa, 1);
    side(Bs, rm, sb, d);
    // d x H ct-ct products + relinearisation, summed over j per head, one rescale
    ck(hx_mul_relin(ctx_, tmp->ptr, sa->ptr, sb->ptr, rlk_->ptr, d * H, nqb, cur()), "mul_relin");
    auto acc = dev((std::size_t)H * cwb);
    ck(hx_sum_strided(ctx_, acc->ptr, tmp->ptr, d, (long long)H * cwb, 2 * H, (long long)nqb * N, (long long)nqb * N,
                      nqb, cur()),
       "sum");
    auto outb = dev((std::size_t)H * 2 * (nqb - 1) * N);
    ck(hx_rescale(ctx_, outb->ptr, acc->ptr, 2 * H, nqb, cur()), "rescale");
    cuda_ck(cudaStreamSynchronize(cur()), "sync");
    for (int h = 0; h < H; ++h) {
      const Ciphertext& A = As[h0 + h];
      const Ciphertext& B = Bs[h0 + h];
      // trace: exactly the SlotOps schedule of linalg.cpp matmul_ctct, per head
      trace_.record(OpKind::PtMul, lv, 2 * d);
      trace_.record(OpKind::Rescale, lv, 2 * d);
      trace_.record(OpKind::Rotate, lv - 1, 2 * (d - 1) + 2 * (std::size_t)d * lg);
      trace_.record(OpKind::CtAdd, lv - 1, 2 * (std::size_t)d * lg + (d - 1));
      trace_.record(OpKind::CtMul, lv - 1, d);
      trace_.record(OpKind::Rescale, lv - 1);
      const Scale s_a = A.scale * ms / Scale::prime(modulus_at(lv));
      const Scale s_b = B.scale * ms_b / Scale::prime(modulus_at(lv));
      outs.push_back(wrap(outb, (std::size_t)h * 2 * (nqb - 1) * N, lv - 2, s_a * s_b / Scale::prime(modulus_at(lv - 1))));
    }
  }
  return outs;
}

Ciphertext GpuLatticeBackend::bsgs_block(const std::vector<Ciphertext>& baby,
                                         const std::vector<Plaintext>& diags, int n1, int n2) {
  DeviceScope ds(*this);
  return bsgs_blocks(baby, diags, n1, n2, 1).front();
}

std::vector<Ciphertext> GpuLatticeBackend::bsgs_blocks(const std::vector<Ciphertext>& baby,
                                                       const std::vector<Plaintext>& diags, int n1, int n2,
                                                       int blocks, bool allow_empty) {
  DeviceScope ds(*this);
  return bsgs_blocks_tokens({baby}, diags, n1, n2, blocks, allow_empty).front();
}

// inner[off + j jstride + t tstride] = sum_{k < n1} diag[j dj + k] (.) baby_t,k
// for T tokens at a uniform baby stride.  n1 > 64 (the MAC kernels' limit) is
// split into chunks of 64 baby steps; chunks >= 1 go to a zeroed copy of the
// whole inner buffer (inner_polys polys) that is then added into it.
static void mac_chunked(hx_ctx* ctx, std::uint64_t* inner, std::size_t inner_polys, std::size_t off,
                        long long jstride, long long tstride, const std::uint64_t* baby, long long btstride,
                        std::size_t ctw, const std::uint64_t* diags, std::size_t ptw, int nqv, int n1, int n2, int dj,
                        int T) {
  constexpr int kMax = 64;
  std::unique_ptr<DeviceBuffer> tmp;
  for (int k0 = 0; k0 < n1; k0 += kMax) {
    const int kc = std::min(kMax, n1 - k0);
    std::uint64_t* dst = inner;
    if (k0) {
      if (!tmp) tmp = std::make_unique<DeviceBuffer>(inner_polys * ptw);
      cuda_ck(cudaMemsetAsync(tmp->ptr, 0, inner_polys * ptw * 8, cur()), "memset");
      dst = tmp->ptr;
    }
    ck(hx_bsgs_mac_tokens(ctx, dst + off, jstride, tstride, baby + (std::size_t)k0 * ctw, btstride,
                          diags + (std::size_t)k0 * ptw, nqv, kc, n2, nqv, T, dj, cur()),
       "bsgs_mac");
    if (k0) ck(hx_add(ctx, inner, inner, dst, (int)inner_polys, nqv, 0, cur()), "add");
  }
}

// Tensor-core operand tiles of the diagonals of rows r = (block b, giant
// step j) < rows (hx_bsgs_tc_pack), made once and attached to the buffer that
// holds the diagonals (every live diagonal must sit in `buf`).  Key: shape and
// the offsets of all rows x n1 diagonals (-1 = absent).
static std::shared_ptr<DeviceBuffer> tc_pack(hx_ctx* ctx, const std::shared_ptr<DeviceBuffer>& buf,
                                             const std::vector<const u64*>& ptrs, int rows, int n1, int nqv) {
  u64 sig = 0xcbf29ce484222325ull;
  auto mix = [&](u64 v) {
    sig ^= v;
    sig *= 0x100000001b3ull;
  };
  mix((u64)rows);
  mix((u64)n1);
  mix((u64)nqv);
  for (const u64* q : ptrs) mix(q ? (u64)(q - buf->ptr) : ~0ull);
  sig &= ~1ull;  // low bit 0: tensor-core tiles, 1: P40 packs
  std::lock_guard<std::mutex> g(buf->derived_mu);
  for (const auto& e : buf->derived)
    if (e.first == sig) return e.second;
  // one packed form per matrix at a time (the P40 packs of single-token
  // matvecs go when the token batches need tiles): u64 + one pack fits HBM
  std::erase_if(buf->derived, [](const auto& e) { return (e.first & 1) != 0; });
  const long long bytes = hx_bsgs_tc_bytes(ctx, rows, n1, nqv);
  if (bytes < 0) throw std::invalid_argument("bsgs: tensor-core shape");
  auto pk = dev(((std::size_t)bytes + 7) / 8);
  ck(hx_bsgs_tc_pack(ctx, pk->ptr, ptrs.data(), rows, n1, nqv, cur()), "bsgs_tc_pack");
  buf->derived.emplace_back(sig, pk);
  return pk;
}

// 5-byte packed diagonals (hx_bsgs_p40_pack) of n2 giant groups x n1 baby
// steps starting at `diags` (group stride dj diagonals) inside `buf`, made
// once and attached to the buffer; null when the shape / primes do not allow it
static bool p40_mac_enabled() {
  static const bool on = [] {
    const char* e = getenv("HX_MAC_P40");
    return !e || atoi(e) != 0;
  }();
  return on;
}
static std::shared_ptr<DeviceBuffer> p40_pack(hx_ctx* ctx, const std::shared_ptr<DeviceBuffer>& buf,
                                              const u64* diags, int n1, int n2, int dj, int nqv) {
  if (!p40_mac_enabled()) return nullptr;
  const long long bytes = hx_bsgs_p40_bytes(ctx, n1, n2, nqv);
  if (bytes < 0) return nullptr;
  u64 sig = 0x9e3779b97f4a7c15ull;
  const u64 key[] = {(u64)(diags - buf->ptr), (u64)n1, (u64)n2, (u64)dj, (u64)nqv, 0x7034300000000000ull};
  for (u64 v : key) {
    sig ^= v;
    sig *= 0x100000001b3ull;
  }
  sig |= 1ull;
  std::lock_guard<std::mutex> g(buf->derived_mu);
  for (const auto& e : buf->derived)
    if (e.first == sig) return e.second;
  std::erase_if(buf->derived, [](const auto& e) { return (e.first & 1) == 0; });  // tensor-core tiles
  auto pk = dev(((std::size_t)bytes + 7) / 8);
  ck(hx_bsgs_p40_pack(ctx, pk->ptr, diags, nqv, n1, n2, dj, nqv, cur()), "bsgs_p40_pack");
  buf->derived.emplace_back(sig, pk);
  return pk;
}

static bool tc_mac_enabled() {
  static const bool on = [] {
    const char* e = getenv("HX_MAC_TC");
    return !e || atoi(e) != 0;
  }();
  return on;
}

std::vector<std::vector<Ciphertext>> GpuLatticeBackend::bsgs_blocks_tokens(
    const std::vector<std::vector<Ciphertext>>& babies, const std::vector<Plaintext>& diags, int n1, int n2,
    int blocks, bool allow_empty) {
  DeviceScope ds(*this);
  const int T = (int)babies.size();
  if (T < 1) throw std::invalid_argument("bsgs_blocks: no tokens");
  for (const auto& bb : babies)
    if ((int)bb.size() < n1) throw std::invalid_argument("bsgs_blocks: shape");
  if ((long long)diags.size() < (long long)n1 * n2 * blocks) throw std::invalid_argument("bsgs_blocks: shape");
  const Ciphertext& x = babies[0][0];
  const int level = x.level, nqv = nq(level);
  const std::size_t N = params_.ring_degree, ctw = (std::size_t)2 * nqv * N, ptw = (std::size_t)nqv * N;
  const std::size_t d = (std::size_t)n1 * n2;
  const auto n = (std::int64_t)slots();
  for (const auto& bb : babies)
    if (bb[0].level != level || bb[0].scale != x.scale) throw LevelMismatchError("bsgs: token level/scale mismatch");
  // baby steps of token t contiguous [n1][2][n_q][N]
  std::vector<std::shared_ptr<DeviceBuffer>> keep;
  std::vector<const u64*> baby_ptr(T);
  for (int t = 0; t < T; ++t) {
    const auto& p0 = payload(babies[t][0]);
    bool contiguous = true;
    for (int k = 1; k < n1 && contiguous; ++k) {
      const auto& pk = payload(babies[t][k]);
      contiguous = pk.buf == p0.buf && pk.offset == p0.offset + k * ctw;
    }
    if (contiguous) {
      baby_ptr[t] = p0.data();
    } else {
      auto bb = dev(n1 * ctw);
      for (int k = 0; k < n1; ++k)
        cuda_ck(cudaMemcpyAsync(bb->ptr + k * ctw, payload(babies[t][k]).data(), ctw * 8, cudaMemcpyDeviceToDevice,
                                cur()), "d2d");
      baby_ptr[t] = bb->ptr;
      keep.push_back(bb);
    }
  }
  // inner sums, layout [n2][T][blocks][2][n_q][N]: giant step j of every
  // (token, block) is one contiguous group (one key read for all of them);
  // dead groups stay 0
  const int E = T * blocks;
  const std::size_t jstride = (std::size_t)E * ctw;
  auto inner = dev((std::size_t)n2 * jstride);
  const std::size_t inner_polys = (std::size_t)n2 * E * 2;
  cuda_ck(cudaMemsetAsync(inner->ptr, 0, inner->words * 8, cur()), "memset");
  Scale dscale;
  bool have_scale = false;
  std::vector<std::vector<char>> live(blocks, std::vector<char>(n2, 0));
  // ---- tensor-core MAC: every row block at once (tiles of <= 128 rows), the
  // diagonals as byte-sliced operand tiles made once per matrix; dense or
  // mostly dense blocks whose diagonals share one buffer
  bool tc_done = false;
  {
    const long long bst = T > 1 ? (long long)(baby_ptr[1] - baby_ptr[0]) : 0;
    bool ok = tc_mac_enabled() && n1 % 8 == 0 && n1 <= 64 && n2 <= 128 && N >= 128;
    for (int t = 1; t < T && ok; ++t) ok = (long long)(baby_ptr[t] - baby_ptr[t - 1]) == bst;
    std::shared_ptr<DeviceBuffer> src;
    std::size_t nlive = 0;
    for (std::size_t e = 0; e < (std::size_t)blocks * d && ok; ++e) {
      const Plaintext& pt = diags[e];
      if (!pt.payload) continue;
      const auto& pl = payload(pt);
      if (!src) src = pl.buf;
      ok = pl.buf == src && pt.level == level && (!have_scale || pt.scale == dscale);
      dscale = pt.scale;
      have_scale = true;
      ++nlive;
    }
    ok = ok && src && 2 * nlive >= (std::size_t)blocks * d;  // sparse matrices: the index-list MAC
    // one token: the packed (P40) MAC wherever it applies (n1 = 32 / 64; two rows
    // per step, all row blocks in one launch: W1's 96 rows x n1 = 32 take 25.1 ms
    // per matvec against 27.1 on the tensor cores), else the tensor cores from 96
    // rows (below that the streaming CUDA-core MAC is faster)
    static const int tc_min_rows = [] {
      const char* e = getenv("HX_TC_MIN_ROWS");  // A/B switch for the T = 1 threshold
      return e ? atoi(e) : 96;
    }();
    static const bool tc_over_p40 = getenv("HX_TC_OVER_P40") != nullptr;  // A/B: the round-2 choice
    const bool p40_shape = p40_mac_enabled() && (n1 == 32 || n1 == 64) && !tc_over_p40;
    ok = ok && (T >= 2 || (blocks * n2 >= tc_min_rows && !p40_shape));
    if (ok) {
      const int bpt = std::max(1, 128 / n2);
      for (int b0 = 0; b0 < blocks; b0 += bpt) {
        const int nb = std::min(bpt, blocks - b0);
        std::vector<const u64*> ptrs((std::size_t)nb * d, nullptr);
        for (std::size_t e = 0; e < ptrs.size(); ++e) {
          const Plaintext& pt = diags[(std::size_t)b0 * d + e];
          if (pt.payload) ptrs[e] = payload(pt).data();
        }
        const auto pk = tc_pack(ctx_, src, ptrs, nb * n2, n1, nqv);
        ck(hx_bsgs_mac_tc(ctx_, inner->ptr + (std::size_t)b0 * ctw, (long long)jstride, (long long)ctw,
                          (long long)(blocks * ctw), baby_ptr[0], bst, pk->ptr, nb, n2, n1, nqv, T, cur()),
           "bsgs_mac_tc");
      }
      for (int b = 0; b < blocks; ++b) {
        std::uint64_t ptmuls = 0, adds = 0;
        for (int j = 0; j < n2; ++j) {
          int cnt = 0;
          for (int k = 0; k < n1; ++k) cnt += diags[(std::size_t)b * d + (std::size_t)j * n1 + k].payload != nullptr;
          if (cnt) {
            ptmuls += cnt;
            adds += cnt - 1;
            live[b][j] = 1;
          }
        }
        if (!ptmuls && !allow_empty) throw std::invalid_argument("matvec_bsgs: block has no non-zero diagonal");
        if (ptmuls) trace_.record(OpKind::PtMul, level, ptmuls * T);
        if (adds) trace_.record(OpKind::CtAdd, level, adds * T);
      }
      tc_done = true;
    } else {
      have_scale = false;
    }
  }
  // ---- one token, several dense row blocks whose diagonals follow one another
  // in one buffer: ONE packed (P40) MAC launch over all blocks x n2 rows -- the
  // baby steps are loaded and split once for every block and a CTA streams
  // blocks x n2 stages instead of n2 (the cost-tuned W1 split has n2 = 16)
  bool p40_merged = false;
  if (!tc_done && T == 1 && blocks > 1 && n1 <= 64 && diags[0].payload) {
    static const bool merge = [] {
      const char* e = getenv("HX_P40_MERGE");
      return !e || atoi(e) != 0;
    }();
    const GpuPlaintext* q0 = &payload(diags[0]);
    bool ok = merge;
    for (std::size_t i = 0; i < (std::size_t)blocks * d && ok; ++i) {
      if (!diags[i].payload) {
        ok = false;
        break;
      }
      const auto& pi = payload(diags[i]);
      ok = pi.buf == q0->buf && pi.offset == q0->offset + i * ptw && diags[i].level == level &&
           diags[i].scale == diags[0].scale;
    }
    if (ok) {
      if (auto pk = p40_pack(ctx_, q0->buf, q0->data(), n1, blocks * n2, n1, nqv)) {
        ck(hx_bsgs_mac_p40_blocks(ctx_, inner->ptr, (long long)jstride, (long long)ctw, baby_ptr[0], pk->ptr,
                                  q0->data(), nqv, n1, n2, blocks, n1, nqv, cur()),
           "bsgs_mac_p40_blocks");
        p40_merged = true;
      }
    }
  }
  for (int b = 0; b < blocks && !tc_done; ++b) {
    const Plaintext* D = diags.data() + (std::size_t)b * d;
    std::uint64_t ptmuls = 0, adds = 0;
    // fast path: the whole block dense and contiguous (encode_many) -> one MAC launch per token
    bool all_contig = D[0].payload != nullptr;
    const GpuPlaintext* p0 = all_contig ? &payload(D[0]) : nullptr;
    for (std::size_t i = 0; i < d && all_contig; ++i) {
      if (!D[i].payload) {
        all_contig = false;
        break;
      }
      const auto& pi = payload(D[i]);
      all_contig = pi.buf == p0->buf && pi.offset == p0->offset + i * ptw && D[i].level == level &&
                   D[i].scale == D[0].scale;
    }
    if (all_contig) {
      if (have_scale && D[0].scale != dscale) throw ScaleMismatchError("bsgs: diagonal scales differ");
      dscale = D[0].scale;
      have_scale = true;
      // one launch over the tokens when their baby sets sit at a uniform stride
      static const bool tok_mac = [] {
        const char* e = getenv("HX_MAC_TOKENS");
        return !e || atoi(e) != 0;
      }();
      bool uniform = tok_mac;
      const long long bstride = T > 1 ? (long long)(baby_ptr[1] - baby_ptr[0]) : 0;
      for (int t = 1; t < T && uniform; ++t) uniform = (long long)(baby_ptr[t] - baby_ptr[t - 1]) == bstride;
      std::shared_ptr<DeviceBuffer> pk;
      if (T == 1 && n1 <= 64 && !p40_merged) pk = p40_pack(ctx_, p0->buf, p0->data(), n1, n2, n1, nqv);
      if (p40_merged) {
        // this block's inner sums came from the merged launch above
      } else if (pk) {
        ck(hx_bsgs_mac_p40(ctx_, inner->ptr + (std::size_t)b * ctw, (long long)jstride, baby_ptr[0], pk->ptr,
                           p0->data(), nqv, n1, n2, n1, nqv, cur()),
           "bsgs_mac_p40");
      } else if (uniform) {
        mac_chunked(ctx_, inner->ptr, inner_polys, (std::size_t)b * ctw, (long long)jstride, (long long)(blocks * ctw),
                    baby_ptr[0], bstride, ctw, p0->data(), ptw, nqv, n1, n2, n1, T);
      } else {
        for (int t = 0; t < T; ++t)
          mac_chunked(ctx_, inner->ptr, inner_polys, ((std::size_t)t * blocks + b) * ctw, (long long)jstride, 0,
                      baby_ptr[t], 0, ctw, p0->data(), ptw, nqv, n1, n2, n1, 1);
      }
      ptmuls = d;
      adds = (std::uint64_t)(n1 - 1) * n2;
      for (int j = 0; j < n2; ++j) live[b][j] = 1;
    } else if (n1 <= 128) {
      // pruned / scattered block: one index-list MAC over its live (j, k)
      // entries for all tokens, plaintexts and baby steps read in place
      std::vector<int> gptr(n2 + 1, 0), ks;
      std::vector<const u64*> dp;
      for (int j = 0; j < n2; ++j) {
        for (int k = 0; k < n1; ++k) {
          const Plaintext& pt = D[(std::size_t)j * n1 + k];
          if (!pt.payload) continue;
          if (pt.level != level) throw LevelMismatchError("bsgs: diagonal level mismatch");
          if (!have_scale) {
            dscale = pt.scale;
            have_scale = true;
          } else if (pt.scale != dscale) {
            throw ScaleMismatchError("bsgs: diagonal scales differ");
          }
          ks.push_back(k);
          dp.push_back(payload(pt).data());
        }
        gptr[j + 1] = (int)ks.size();
        const int cnt = gptr[j + 1] - gptr[j];
        if (cnt) {
          ptmuls += cnt;
          adds += cnt - 1;
          live[b][j] = 1;
        }
      }
      bool uniform = true;
      const long long bstride = T > 1 ? (long long)(baby_ptr[1] - baby_ptr[0]) : 0;
      for (int t = 1; t < T && uniform; ++t) uniform = (long long)(baby_ptr[t] - baby_ptr[t - 1]) == bstride;
      // runs of consecutive groups whose n1 diagonals are all live and contiguous
      // (mostly-dense matrices) take the streaming dense MAC; the rest the index list
      const auto dense_at = [&](int j) {
        if (gptr[j + 1] - gptr[j] != n1) return false;
        for (int k = 1; k < n1; ++k)
          if (dp[gptr[j] + k] != dp[gptr[j]] + (std::size_t)k * ptw) return false;
        return true;
      };
      std::vector<int> sgptr(n2 + 1, 0), sks;
      std::vector<const u64*> sdp;
      for (int j = 0; j < n2;) {
        if (dense_at(j)) {
          int j1 = j + 1;
          while (j1 < n2 && dense_at(j1) && dp[gptr[j1]] == dp[gptr[j1 - 1]] + (std::size_t)n1 * ptw) ++j1;
          const std::size_t off = (std::size_t)j * jstride + (std::size_t)b * ctw;
          std::shared_ptr<DeviceBuffer> pk;
          if (T == 1 && n1 <= 64) {
            const Plaintext& p0 = D[(std::size_t)j * n1];
            pk = p40_pack(ctx_, payload(p0).buf, dp[gptr[j]], n1, j1 - j, n1, nqv);
          }
          if (pk) {
            ck(hx_bsgs_mac_p40(ctx_, inner->ptr + off, (long long)jstride, baby_ptr[0], pk->ptr, dp[gptr[j]], nqv, n1,
                               j1 - j, n1, nqv, cur()),
               "bsgs_mac_p40");
          } else if (uniform) {
            mac_chunked(ctx_, inner->ptr, inner_polys, off, (long long)jstride, (long long)(blocks * ctw), baby_ptr[0],
                        bstride, ctw, dp[gptr[j]], ptw, nqv, n1, j1 - j, n1, T);
          } else {
            for (int t = 0; t < T; ++t)
              mac_chunked(ctx_, inner->ptr, inner_polys, off + (std::size_t)t * blocks * ctw, (long long)jstride, 0,
                          baby_ptr[t], 0, ctw, dp[gptr[j]], ptw, nqv, n1, j1 - j, n1, 1);
          }
          for (int jj = j; jj < j1; ++jj) sgptr[jj + 1] = (int)sks.size();
          j = j1;
          continue;
        }
        for (int e = gptr[j]; e < gptr[j + 1]; ++e) {
          sks.push_back(ks[e]);
          sdp.push_back(dp[e]);
        }
        sgptr[j + 1] = (int)sks.size();
        ++j;
      }
      gptr.swap(sgptr);
      ks.swap(sks);
      dp.swap(sdp);
      if (!ks.empty()) {
        if (uniform) {
          ck(hx_bsgs_mac_sparse(ctx_, inner->ptr + (std::size_t)b * ctw, (long long)jstride, (long long)(blocks * ctw),
                                baby_ptr[0], bstride, gptr.data(), ks.data(), dp.data(), n1, n2, nqv, T, cur()),
             "bsgs_mac_sparse");
        } else {
          for (int t = 0; t < T; ++t)
            ck(hx_bsgs_mac_sparse(ctx_, inner->ptr + ((std::size_t)t * blocks + b) * ctw, (long long)jstride, 0,
                                  baby_ptr[t], 0, gptr.data(), ks.data(), dp.data(), n1, n2, nqv, 1, cur()),
               "bsgs_mac_sparse");
        }
      }
    } else {
      for (int j = 0; j < n2; ++j) {
        std::vector<int> ks;
        for (int k = 0; k < n1; ++k) {
          const Plaintext& pt = D[(std::size_t)j * n1 + k];
          if (!pt.payload) continue;
          if (pt.level != level) throw LevelMismatchError("bsgs: diagonal level mismatch");
          if (!have_scale) {
            dscale = pt.scale;
            have_scale = true;
          } else if (pt.scale != dscale) {
            throw ScaleMismatchError("bsgs: diagonal scales differ");
          }
          ks.push_back(k);
        }
        if (ks.empty()) continue;
        ptmuls += ks.size();
        adds += ks.size() - 1;
        const auto& q0 = payload(D[(std::size_t)j * n1 + ks[0]]);
        bool dense = (int)ks.size() == n1;
        for (int k = 1; k < n1 && dense; ++k) {
          const auto& pk = payload(D[(std::size_t)j * n1 + k]);
          dense = pk.buf == q0.buf && pk.offset == q0.offset + k * ptw;
        }
        std::unique_ptr<DeviceBuffer> dg;
        if (!dense) {  // sparse group: gather its diagonals once for all tokens
          dg = std::make_unique<DeviceBuffer>(ks.size() * ptw);
          for (std::size_t i = 0; i < ks.size(); ++i)
            cuda_ck(cudaMemcpyAsync(dg->ptr + i * ptw, payload(D[(std::size_t)j * n1 + ks[i]]).data(), ptw * 8,
                                    cudaMemcpyDeviceToDevice, cur()), "d2d");
        }
        for (int t = 0; t < T; ++t) {
          const std::size_t off = j * jstride + ((std::size_t)t * blocks + b) * ctw;
          if (dense) {
            mac_chunked(ctx_, inner->ptr, inner_polys, off, (long long)ctw, 0, baby_ptr[t], 0, ctw, q0.data(), ptw,
                        nqv, n1, 1, n1, 1);
          } else {  // ... and the matching baby steps of the token
            DeviceBuffer bs(ks.size() * ctw);
            for (std::size_t i = 0; i < ks.size(); ++i)
              cuda_ck(cudaMemcpyAsync(bs.ptr + i * ctw, baby_ptr[t] + ks[i] * ctw, ctw * 8, cudaMemcpyDeviceToDevice,
                                      cur()), "d2d");
            mac_chunked(ctx_, inner->ptr, inner_polys, off, (long long)ctw, 0, bs.ptr, 0, ctw, dg->ptr, ptw, nqv,
                        (int)ks.size(), 1, (int)ks.size(), 1);
          }
        }
        live[b][j] = 1;
      }
    }
    bool any = false;
    for (int j = 0; j < n2; ++j) any |= live[b][j] != 0;
    if (!any && !allow_empty) throw std::invalid_argument("matvec_bsgs: block has no non-zero diagonal");
    if (ptmuls) trace_.record(OpKind::PtMul, level, ptmuls * T);
    if (adds) trace_.record(OpKind::CtAdd, level, adds * T);
  }
  if (!have_scale) dscale = Scale::prime(modulus_at(level));  // empty shard: the diagonal scale
  const Scale out_scale = x.scale * dscale;
  // giant steps j >= 1: rotate group j of every (token, block) by n1 j with one key
  std::vector<const u64*> keys;
  std::vector<u64> gs;
  std::vector<int> J;
  for (int j = 1; j < n2; ++j) {
    bool any = false;
    for (int b = 0; b < blocks; ++b) any |= live[b][j] != 0;
    if (!any) continue;
    const std::int64_t r = detail::reduce_amount((std::int64_t)n1 * j, n);
    const u64* key = rotation_key(r);
    if (!rot_set_.contains(r) || !key) throw MissingRotationKeyError("rotate: no key for amount " + std::to_string(r));
    keys.push_back(key);
    gs.push_back(galois(r));
    J.push_back(j);
  }
  // y = inner_0 + sum_j Rot(inner_j) with ONE ModDown per output (double
  // hoisting): the giant rotations' key-switch products are
  // summed in the PQ basis (hx_rotate_grouped_sum).  Giant-step shards
  // (allow_empty) stop before the ModDown: each output is the PQ partial
  // [T = 2 n_q limbs][S = 2 (n_q + K) limbs] that the ranks sum (shard.py).
  const bool partial = allow_empty;
  const std::size_t uw = (std::size_t)2 * (nqv + params_.special_primes.size()) * N;
  const std::size_t pw = partial ? ctw + uw : ctw;
  auto out = dev((std::size_t)E * pw);
  if (J.empty() && !partial) {
    cuda_ck(cudaMemcpyAsync(out->ptr, inner->ptr, jstride * 8, cudaMemcpyDeviceToDevice, cur()), "d2d");
  } else {
    std::shared_ptr<DeviceBuffer> src;
    const u64* srcp = inner->ptr + jstride;  // groups 1..n2-1 are contiguous
    if (!J.empty() && (int)J.size() != n2 - 1) {
      src = dev(J.size() * jstride);
      for (std::size_t i = 0; i < J.size(); ++i)
        cuda_ck(cudaMemcpyAsync(src->ptr + i * jstride, inner->ptr + J[i] * jstride, jstride * 8,
                                cudaMemcpyDeviceToDevice, cur()), "d2d");
      srcp = src->ptr;
    }
    if (!partial) {
      ck(hx_rotate_grouped_sum(ctx_, out->ptr, nullptr, srcp, inner->ptr, keys.data(), gs.data(), (int)J.size(), E,
                               nqv, cur()),
         "rotate_grouped_sum");
    } else {
      auto tb = dev((std::size_t)E * ctw), sb = dev((std::size_t)E * uw);
      ck(hx_rotate_grouped_sum(ctx_, tb->ptr, sb->ptr, srcp, inner->ptr, keys.data(), gs.data(), (int)J.size(), E,
                               nqv, cur()),
         "rotate_grouped_sum");
      cuda_ck(cudaMemcpy2DAsync(out->ptr, pw * 8, tb->ptr, ctw * 8, ctw * 8, E, cudaMemcpyDeviceToDevice, cur()),
              "memcpy2d");
      cuda_ck(cudaMemcpy2DAsync(out->ptr + ctw, pw * 8, sb->ptr, uw * 8, uw * 8, E, cudaMemcpyDeviceToDevice, cur()),
              "memcpy2d");
    }
  }
  std::vector<std::vector<Ciphertext>> res(T);
  for (int b = 0; b < blocks; ++b) {
    std::uint64_t nl = 0, nr = 0;
    for (int j = 0; j < n2; ++j) {
      nl += live[b][j] != 0;
      nr += (j > 0 && live[b][j] != 0);
    }
    if (nr) trace_.record(OpKind::Rotate, level, nr * T);
    if (nl > 1) trace_.record(OpKind::CtAdd, level, (nl - 1) * T);
  }
  for (int t = 0; t < T; ++t)
    for (int b = 0; b < blocks; ++b)
      res[t].push_back(wrap(out, ((std::size_t)t * blocks + b) * pw, level, out_scale));
  return res;
}

Ciphertext GpuLatticeBackend::shard_finish(const Ciphertext& like, const std::uint64_t* words) {
  DeviceScope ds(*this);
  const int n = nq(like.level);
  const std::size_t N = params_.ring_degree, ctw = (std::size_t)2 * n * N;
  auto buf = dev(ctw);
  ck(hx_moddown_add(ctx_, buf->ptr, words + ctw, words, 1, n, cur()), "moddown_add");
  return wrap(buf, 0, like.level, like.scale);
}

std::vector<std::vector<Ciphertext>> GpuLatticeBackend::rotate_many_tokens(const std::vector<Ciphertext>& xs,
                                                                           std::span<const std::int64_t> amounts) {
  DeviceScope ds(*this);
  const int T = (int)xs.size();
  if (T < 1) throw std::invalid_argument("rotate_many: no ciphertexts");
  const auto n = (std::int64_t)slots();
  const std::size_t N = params_.ring_degree;
  const int level = xs[0].level, nqv = nq(level);
  const std::size_t ctw = (std::size_t)2 * nqv * N;
  const std::size_t R = amounts.size();
  // inputs contiguous [T][ct]
  auto in = dev((std::size_t)T * ctw);
  for (int t = 0; t < T; ++t) {
    if (xs[t].level != level) throw LevelMismatchError("rotate_many: token level mismatch");
    cuda_ck(cudaMemcpyAsync(in->ptr + t * ctw, payload(xs[t]).data(), ctw * 8, cudaMemcpyDeviceToDevice, cur()),
            "d2d");
  }
  std::vector<const u64*> keys;
  std::vector<u64> gs;
  std::vector<std::size_t> which;
  for (std::size_t i = 0; i < R; ++i) {
    const std::int64_t r = detail::reduce_amount(amounts[i], n);
    if (r == 0) continue;
    const u64* key = rotation_key(r);
    if (!rot_set_.contains(r) || !key) throw MissingRotationKeyError("rotate: no key for amount " + std::to_string(r));
    keys.push_back(key);
    gs.push_back(galois(r));
    which.push_back(i);
  }
  // out [T][R][ct]: hoisted rotations land at [t][1 + ...] when amounts[0] == 0
  auto buf = dev((std::size_t)T * R * ctw);
  if (!keys.empty()) {
    const bool lead_identity = detail::reduce_amount(amounts[0], n) == 0 && which.size() == R - 1;
    if (lead_identity) {  // BSGS baby steps: write rotations straight after the identity slot
      auto tmp = dev((std::size_t)T * keys.size() * ctw);
      ck(hx_rotate_hoisted(ctx_, tmp->ptr, in->ptr, keys.data(), gs.data(), (int)keys.size(), T, nqv, cur()),
         "rotate_hoisted");
      cuda_ck(cudaMemcpy2DAsync(buf->ptr + ctw, R * ctw * 8, tmp->ptr, keys.size() * ctw * 8, keys.size() * ctw * 8,
                                T, cudaMemcpyDeviceToDevice, cur()),
              "memcpy2d");
    } else {
      auto tmp = dev((std::size_t)T * keys.size() * ctw);
      ck(hx_rotate_hoisted(ctx_, tmp->ptr, in->ptr, keys.data(), gs.data(), (int)keys.size(), T, nqv, cur()),
         "rotate_hoisted");
      for (int t = 0; t < T; ++t)
        for (std::size_t j = 0; j < which.size(); ++j)
          cuda_ck(cudaMemcpyAsync(buf->ptr + (t * R + which[j]) * ctw, tmp->ptr + (t * keys.size() + j) * ctw, ctw * 8,
                                  cudaMemcpyDeviceToDevice, cur()), "d2d");
    }
    trace_.record(OpKind::Rotate, level, keys.size() * T);
  }
  std::vector<std::vector<Ciphertext>> out(T);
  for (int t = 0; t < T; ++t)
    for (std::size_t i = 0; i < R; ++i) {
      if (detail::reduce_amount(amounts[i], n) == 0)
        cuda_ck(cudaMemcpyAsync(buf->ptr + (t * R + i) * ctw, in->ptr + t * ctw, ctw * 8, cudaMemcpyDeviceToDevice,
                                cur()), "d2d");
      out[t].push_back(wrap(buf, (t * R + i) * ctw, level, xs[t].scale));
    }
  return out;
}

}  // namespace helix
