// lattice.cpp -- helix::NttTables / helix::LatticeContext over libhx_b200 (see
// include/helix/ntt.hpp, rns_poly.hpp).  Reference behaviour, file:line:
//   psi search            ntt.cpp:23-32
//   forward / inverse     ntt.cpp:57-96    -> hx_ntt_fwd / hx_ntt_inv
//   add/sub/negate/mul    rns_poly.cpp:62-100 -> hx_add / hx_sub / hx_neg / hx_mul
//   mul_acc               rns_poly.cpp:102-110 -> hx_mul_acc
//   ring_mul              rns_poly.cpp:112-122 (NTT, mul, INTT on the device)
//   automorphism          rns_poly.cpp:124-142 -> NTT, hx_automorphism, INTT (exact)
//   rescale_drop_last     rns_poly.cpp:144-162 -> NTT, hx_rescale, INTT (exact)
//   moddown_special       rns_poly.cpp:164-180 -> NTT, hx_moddown (K = 1), INTT
//   samplers / from_i64   rns_poly.cpp:191-227 (host distributions, device lift)
// Error messages and exception types are the reference's.
#include "helix/rns_poly.hpp"

#include <cuda_runtime.h>

#include <mutex>
#include <stdexcept>
#include <string>

#include "hx_b200.h"

namespace helix {

namespace {
void ck(int rc, const char* what) {
  if (rc != HX_OK) throw std::runtime_error(std::string(what) + ": " + hx_last_error());
}
void cuda_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
int log2_exact(std::size_t n) {
  int l = 0;
  while ((std::size_t(1) << l) < n) ++l;
  return l;
}
// device buffer of `words` u64 (grown on demand)
struct DevVec {
  u64* p = nullptr;
  std::size_t cap = 0;
  u64* get(std::size_t words) {
    if (words > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cuda_ck(cudaMalloc((void**)&p, words * 8), "cudaMalloc");
      cap = words;
    }
    return p;
  }
  ~DevVec() {
    if (p) cudaFree(p);
  }
};
}  // namespace

// ------------------------------------------------------------------ NTT tables
namespace detail {
struct DeviceNtt {
  hx_ctx* ctx = nullptr;
  DevVec a, b;
  std::mutex m;
  ~DeviceNtt() {
    if (ctx) hx_ctx_destroy(ctx);
  }
};
}  // namespace detail

u64 find_psi(const Modulus& q, std::size_t n) {
  const u64 e = (q.q - 1) / (2 * n);
  for (u64 g = 2; g < q.q; ++g) {
    const u64 w = q.pow(g, e);
    if (q.pow(w, n) == q.q - 1) return w;
  }
  throw std::invalid_argument("NttTables: no primitive 2n-th root");
}

NttTables::NttTables(Modulus modulus, std::size_t n) : mod_(modulus), n_(n) {
  if (n < 2 || (n & (n - 1))) throw std::invalid_argument("NttTables: n must be a power of two");
  if ((mod_.q - 1) % (2 * n) != 0) throw std::invalid_argument("NttTables: q != 1 mod 2n");
  psi_ = find_psi(mod_, n);
}

namespace {
// the one-prime device context of a table set, created on first use
detail::DeviceNtt& device_for(std::shared_ptr<detail::DeviceNtt>& d, const Modulus& q, std::size_t n) {
  if (n == 0) throw std::logic_error("NttTables: default-constructed");
  static std::mutex create_m;
  std::lock_guard<std::mutex> lk(create_m);
  if (!d) {
    const int logn = log2_exact(n);
    if (logn < 8 || logn > 16) throw std::invalid_argument("NttTables: the B200 NTT supports n in [2^8, 2^16]");
    // hx contexts carry >= 1 special prime: a companion NTT prime, unused here
    const auto sp = find_ntt_primes(std::uint64_t(1) << 40, 1, 2 * n, {q.q});
    auto dn = std::make_shared<detail::DeviceNtt>();
    dn->ctx = hx_ctx_create(logn, &q.q, 1, sp.data(), 1, 1);
    if (!dn->ctx) throw std::runtime_error(std::string("NttTables: ") + hx_last_error());
    d = dn;
  }
  return *d;
}

template <class F>
void on_device(detail::DeviceNtt& D, std::span<u64> a, std::size_t n, F f) {
  if (a.size() != n) throw std::invalid_argument("ntt: wrong length");
  std::lock_guard<std::mutex> lk(D.m);
  u64* p = D.a.get(n);
  cuda_ck(cudaMemcpy(p, a.data(), n * 8, cudaMemcpyHostToDevice), "h2d");
  f(p);
  cuda_ck(cudaMemcpy(a.data(), p, n * 8, cudaMemcpyDeviceToHost), "d2h");
}
}  // namespace

void NttTables::forward(std::span<u64> a) const {
  auto& d = device_for(dev_, mod_, n_);
  on_device(d, a, n_, [&](u64* p) { ck(hx_ntt_fwd(d.ctx, p, 1, 1, 0, nullptr), "ntt_fwd"); });
}

void NttTables::inverse(std::span<u64> a) const {
  auto& d = device_for(dev_, mod_, n_);
  on_device(d, a, n_, [&](u64* p) { ck(hx_ntt_inv(d.ctx, p, 1, 1, 0, nullptr), "ntt_inv"); });
}

std::vector<u64> NttTables::negacyclic_mul(std::span<const u64> a, std::span<const u64> b) const {
  if (a.size() != n_ || b.size() != n_) throw std::invalid_argument("negacyclic_mul: wrong length");
  auto& d = device_for(dev_, mod_, n_);
  std::vector<u64> out(a.begin(), a.end());
  std::lock_guard<std::mutex> lk(d.m);
  u64* pa = d.a.get(n_);
  u64* pb = d.b.get(n_);
  cuda_ck(cudaMemcpy(pa, a.data(), n_ * 8, cudaMemcpyHostToDevice), "h2d");
  cuda_ck(cudaMemcpy(pb, b.data(), n_ * 8, cudaMemcpyHostToDevice), "h2d");
  ck(hx_ntt_fwd(d.ctx, pa, 1, 1, 0, nullptr), "ntt_fwd");
  ck(hx_ntt_fwd(d.ctx, pb, 1, 1, 0, nullptr), "ntt_fwd");
  ck(hx_mul(d.ctx, pa, pa, pb, 1, 1, 0, nullptr), "mul");
  ck(hx_ntt_inv(d.ctx, pa, 1, 1, 0, nullptr), "ntt_inv");
  cuda_ck(cudaMemcpy(out.data(), pa, n_ * 8, cudaMemcpyDeviceToHost), "d2h");
  return out;
}

std::vector<u64> schoolbook_negacyclic_mul(std::span<const u64> a, std::span<const u64> b, const Modulus& mod) {
  if (a.size() != b.size()) throw std::invalid_argument("schoolbook: length mismatch");
  const std::size_t n = a.size();
  std::vector<u64> c(n, 0);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      const u64 p = mod.mul(a[i], b[j]);
      const std::size_t k = i + j;
      c[k % n] = k < n ? mod.add(c[k], p) : mod.sub(c[k - n], p);  // X^n = -1
    }
  return c;
}

// ------------------------------------------------------------------ lattice context
struct LatticeContext::Staging {
  std::mutex m;
  DevVec a, b, c;
};

LatticeContext::LatticeContext(const CkksParams& params) : params_(params), n_(params.ring_degree) {
  params_.validate();
  if (params_.special_primes.empty()) throw std::invalid_argument("lattice context: a special prime is required");
  for (u64 q : params_.moduli) {
    chain_.emplace_back(q);
    ntt_.emplace_back(Modulus(q), n_);
  }
  special_ = Modulus(params_.special_primes[0]);
  ntt_special_ = NttTables(special_, n_);
  ctx_ = hx_ctx_create(log2_exact(n_), params_.moduli.data(), (int)params_.moduli.size(),
                       params_.special_primes.data(), (int)params_.special_primes.size(),
                       std::max(1, params_.digit_size));
  if (!ctx_) throw std::runtime_error(std::string("lattice context: ") + hx_last_error());
  stage_ = std::make_unique<Staging>();
}

LatticeContext::~LatticeContext() {
  stage_.reset();
  if (ctx_) hx_ctx_destroy(ctx_);
}

LatticeContext::Staging& LatticeContext::stage() const { return *stage_; }

const Modulus& LatticeContext::limb_modulus(const RnsPoly& p, int limb) const {
  if (p.has_special && limb == static_cast<int>(p.limbs.size()) - 1) return special_;
  return chain_.at(limb);
}

const NttTables& LatticeContext::limb_ntt(const RnsPoly& p, int limb) const {
  if (p.has_special && limb == static_cast<int>(p.limbs.size()) - 1) return ntt_special_;
  return ntt_.at(limb);
}

RnsPoly LatticeContext::zero(int chain_limbs, bool with_special, PolyDomain domain) const {
  RnsPoly p;
  p.has_special = with_special;
  p.domain = domain;
  p.limbs.assign(chain_limbs + (with_special ? 1 : 0), std::vector<u64>(n_, 0));
  return p;
}

void LatticeContext::check_match(const RnsPoly& a, const RnsPoly& b, const char* what) const {
  if (a.limbs.size() != b.limbs.size() || a.has_special != b.has_special)
    throw std::invalid_argument(std::string(what) + ": limb-count mismatch");
  if (a.domain != b.domain) throw std::invalid_argument(std::string(what) + ": domain mismatch");
}

namespace {
void check_shape(const RnsPoly& p, std::size_t n, int n_chain) {
  for (const auto& l : p.limbs)
    if (l.size() != n) throw std::invalid_argument("RnsPoly: limb of wrong length");
  if (p.chain_limbs() < 0 || p.chain_limbs() > n_chain) throw std::invalid_argument("RnsPoly: too many limbs");
}
void upload(u64* d, const RnsPoly& p, std::size_t n) {
  for (std::size_t k = 0; k < p.limbs.size(); ++k)
    cuda_ck(cudaMemcpy(d + k * n, p.limbs[k].data(), n * 8, cudaMemcpyHostToDevice), "h2d");
}
void download(RnsPoly& p, const u64* d, std::size_t n) {
  for (std::size_t k = 0; k < p.limbs.size(); ++k)
    cuda_ck(cudaMemcpy(p.limbs[k].data(), d + k * n, n * 8, cudaMemcpyDeviceToHost), "d2h");
}
}  // namespace

void LatticeContext::to_ntt(RnsPoly& p) const {
  if (p.domain == PolyDomain::Ntt) return;
  check_shape(p, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  u64* d = stage().a.get(p.limbs.size() * n_);
  upload(d, p, n_);
  ck(hx_ntt_fwd(ctx_, d, 1, p.chain_limbs(), p.has_special ? 1 : 0, nullptr), "to_ntt");
  download(p, d, n_);
  p.domain = PolyDomain::Ntt;
}

void LatticeContext::to_coeff(RnsPoly& p) const {
  if (p.domain == PolyDomain::Coeff) return;
  check_shape(p, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  u64* d = stage().a.get(p.limbs.size() * n_);
  upload(d, p, n_);
  ck(hx_ntt_inv(ctx_, d, 1, p.chain_limbs(), p.has_special ? 1 : 0, nullptr), "to_coeff");
  download(p, d, n_);
  p.domain = PolyDomain::Coeff;
}

namespace {
template <class F>
RnsPoly binary(const LatticeContext& L, hx_ctx* ctx, std::size_t n, const RnsPoly& a, const RnsPoly* b, u64* da,
               u64* db, F f) {
  RnsPoly out = a;
  upload(da, a, n);
  if (b) upload(db, *b, n);
  ck(f(ctx, da, da, db, 1, a.chain_limbs(), a.has_special ? 1 : 0, nullptr), "elementwise");
  download(out, da, n);
  (void)L;
  return out;
}
}  // namespace

RnsPoly LatticeContext::add(const RnsPoly& a, const RnsPoly& b) const {
  check_match(a, b, "poly add");
  check_shape(a, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  const std::size_t w = a.limbs.size() * n_;
  return binary(*this, ctx_, n_, a, &b, stage().a.get(w), stage().b.get(w), hx_add);
}

RnsPoly LatticeContext::sub(const RnsPoly& a, const RnsPoly& b) const {
  check_match(a, b, "poly sub");
  check_shape(a, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  const std::size_t w = a.limbs.size() * n_;
  return binary(*this, ctx_, n_, a, &b, stage().a.get(w), stage().b.get(w), hx_sub);
}

RnsPoly LatticeContext::negate(const RnsPoly& a) const {
  check_shape(a, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  const std::size_t w = a.limbs.size() * n_;
  RnsPoly out = a;
  u64* d = stage().a.get(w);
  upload(d, a, n_);
  ck(hx_neg(ctx_, d, d, 1, a.chain_limbs(), a.has_special ? 1 : 0, nullptr), "negate");
  download(out, d, n_);
  return out;
}

RnsPoly LatticeContext::mul(const RnsPoly& a, const RnsPoly& b) const {
  check_match(a, b, "poly mul");
  if (a.domain != PolyDomain::Ntt) throw std::invalid_argument("poly mul: need NTT domain");
  check_shape(a, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  const std::size_t w = a.limbs.size() * n_;
  return binary(*this, ctx_, n_, a, &b, stage().a.get(w), stage().b.get(w), hx_mul);
}

void LatticeContext::mul_acc(const RnsPoly& a, const RnsPoly& b, RnsPoly& acc) const {
  check_match(a, b, "poly mul_acc");
  check_match(a, acc, "poly mul_acc");
  check_shape(a, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  const std::size_t w = a.limbs.size() * n_;
  u64 *da = stage().a.get(w), *db = stage().b.get(w), *dc = stage().c.get(w);
  upload(da, a, n_);
  upload(db, b, n_);
  upload(dc, acc, n_);
  ck(hx_mul_acc(ctx_, dc, da, db, 1, a.chain_limbs(), a.has_special ? 1 : 0, nullptr), "mul_acc");
  download(acc, dc, n_);
}

RnsPoly LatticeContext::ring_mul(const RnsPoly& a, const RnsPoly& b) const {
  if (a.limbs.size() != b.limbs.size() || a.has_special != b.has_special)
    throw std::invalid_argument("ring_mul: limb-count mismatch");
  RnsPoly fa = a, fb = b;
  to_ntt(fa);
  to_ntt(fb);
  RnsPoly out = mul(fa, fb);
  to_coeff(out);
  return out;
}

RnsPoly LatticeContext::automorphism(const RnsPoly& a, u64 g) const {
  if (a.domain != PolyDomain::Coeff) throw std::invalid_argument("automorphism: need coefficient domain");
  check_shape(a, n_, (int)chain_.size());
  const u64 gg = g % (2 * n_);
  if (!(gg & 1)) throw std::invalid_argument("automorphism: g must be odd");
  std::lock_guard<std::mutex> lk(stage().m);
  const std::size_t w = a.limbs.size() * n_;
  const int nq = a.chain_limbs(), np = a.has_special ? 1 : 0;
  u64 *da = stage().a.get(w), *db = stage().b.get(w);
  RnsPoly out = a;
  upload(da, a, n_);
  // NTT(tau_g a) is a permutation of NTT(a): transform, permute, transform back (exact)
  ck(hx_ntt_fwd(ctx_, da, 1, nq, np, nullptr), "automorphism");
  ck(hx_automorphism(ctx_, db, da, 1, nq, np, gg, nullptr), "automorphism");
  ck(hx_ntt_inv(ctx_, db, 1, nq, np, nullptr), "automorphism");
  download(out, db, n_);
  return out;
}

RnsPoly LatticeContext::rescale_drop_last(const RnsPoly& a) const {
  if (a.domain != PolyDomain::Coeff) throw std::invalid_argument("rescale: need coeff domain");
  if (a.has_special) throw std::invalid_argument("rescale: unexpected special limb");
  const int k = a.chain_limbs();
  if (k < 2) throw std::invalid_argument("rescale: no limb to drop");
  check_shape(a, n_, (int)chain_.size());
  std::lock_guard<std::mutex> lk(stage().m);
  u64 *da = stage().a.get((std::size_t)k * n_), *db = stage().b.get((std::size_t)k * n_);
  upload(da, a, n_);
  ck(hx_ntt_fwd(ctx_, da, 1, k, 0, nullptr), "rescale");
  ck(hx_rescale(ctx_, db, da, 1, k, nullptr), "rescale");
  ck(hx_ntt_inv(ctx_, db, 1, k - 1, 0, nullptr), "rescale");
  RnsPoly out = zero(k - 1, false, PolyDomain::Coeff);
  download(out, db, n_);
  return out;
}

RnsPoly LatticeContext::moddown_special(const RnsPoly& a) const {
  if (a.domain != PolyDomain::Coeff) throw std::invalid_argument("moddown: need coeff domain");
  if (!a.has_special) throw std::invalid_argument("moddown: no special limb");
  if (params_.special_primes.size() != 1)
    throw std::invalid_argument("moddown: RnsPoly carries one special limb; K > 1 switches keys on the device");
  check_shape(a, n_, (int)chain_.size());
  const int k = a.chain_limbs();
  std::lock_guard<std::mutex> lk(stage().m);
  u64 *da = stage().a.get((std::size_t)(k + 1) * n_), *db = stage().b.get((std::size_t)k * n_);
  upload(da, a, n_);
  ck(hx_ntt_fwd(ctx_, da, 1, k, 1, nullptr), "moddown");
  ck(hx_moddown(ctx_, db, da, 1, k, nullptr), "moddown");
  ck(hx_ntt_inv(ctx_, db, 1, k, 0, nullptr), "moddown");
  RnsPoly out = zero(k, false, PolyDomain::Coeff);
  download(out, db, n_);
  return out;
}

RnsPoly LatticeContext::drop_to_level(const RnsPoly& a, int target_level) const {
  if (a.has_special) throw std::invalid_argument("drop_to_level: unexpected special limb");
  if (target_level + 1 > a.chain_limbs()) throw std::invalid_argument("drop_to_level: target above current");
  RnsPoly out = a;
  out.limbs.resize(target_level + 1);
  return out;
}

RnsPoly LatticeContext::sample_uniform(int chain_limbs, bool with_special, PolyDomain domain,
                                       std::mt19937_64& rng) const {
  RnsPoly p = zero(chain_limbs, with_special, domain);
  for (std::size_t i = 0; i < p.limbs.size(); ++i) {
    std::uniform_int_distribution<u64> dist(0, limb_modulus(p, (int)i).q - 1);
    for (auto& x : p.limbs[i]) x = dist(rng);
  }
  return p;
}

RnsPoly LatticeContext::sample_ternary(int chain_limbs, bool with_special, std::mt19937_64& rng) const {
  std::uniform_int_distribution<int> dist(-1, 1);
  std::vector<std::int64_t> coeffs(n_);
  for (auto& c : coeffs) c = dist(rng);
  return from_i64(coeffs, chain_limbs, with_special);
}

RnsPoly LatticeContext::sample_gaussian(int chain_limbs, bool with_special, std::mt19937_64& rng) const {
  std::normal_distribution<double> dist(0.0, 3.2);
  std::vector<std::int64_t> coeffs(n_);
  for (auto& c : coeffs) c = static_cast<std::int64_t>(std::llround(dist(rng)));
  return from_i64(coeffs, chain_limbs, with_special);
}

RnsPoly LatticeContext::from_i64(const std::vector<std::int64_t>& coeffs, int chain_limbs, bool with_special) const {
  if (coeffs.size() != n_) throw std::invalid_argument("from_i64: wrong length");
  if (chain_limbs < 1 || chain_limbs > (int)chain_.size()) throw std::invalid_argument("from_i64: limb count");
  RnsPoly p = zero(chain_limbs, with_special, PolyDomain::Coeff);
  std::lock_guard<std::mutex> lk(stage().m);
  u64* dv = stage().b.get(n_);
  u64* d = stage().a.get(p.limbs.size() * n_);
  cuda_ck(cudaMemcpy(dv, coeffs.data(), n_ * 8, cudaMemcpyHostToDevice), "h2d");
  ck(hx_from_i64(ctx_, d, (const std::int64_t*)dv, 1, chain_limbs, with_special ? 1 : 0, nullptr), "from_i64");
  download(p, d, n_);
  return p;
}

}  // namespace helix
