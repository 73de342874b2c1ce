// ref_shim.cpp -- TEST INFRASTRUCTURE.  C entry points over the REFERENCE's
// own compiled primitives (/root/reference/proj/src/*.cpp, built into
// oracle/_ref/ by oracle/Makefile with the one-line modmath.hpp:30 fix applied
// to a generated overlay header -- the reference tree itself is never edited
// and no reference source is copied into this repository).
//
// Used by tests/ to pin the C oracle (hx_oracle.c) against the reference and to
// generate tests/golden/ fixtures, and by bench.py --impl reference as the CPU
// reference arm.  The key-switch / rotation drivers below are the SPEC-only
// pieces composed from the reference's NttTables::forward /
// inverse (ntt.cpp:57-96) and Modulus::mul/add/sub (modmath.hpp:41-63), with
// the same conventions as the oracle.
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <memory>
#include <thread>
#include <vector>

#include "helix/encoder.hpp"
#include "helix/modmath.hpp"
#include "helix/ntt.hpp"
#include "helix/params.hpp"
#include "helix/rns_poly.hpp"

using helix::u64;

namespace {

// Persistent worker pool (created once per context by ref_set_threads): a
// parallel_for hands out indices through an atomic counter to the parked
// workers and the calling thread; nested parallel_for calls made from inside
// a task run serially on that task's thread (the batched arm threads across
// ciphertexts, each rotation single-threaded).
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i + 1 < n; ++i) th_.emplace_back([this] { work(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  void run(int count, const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &f;
      count_ = count;
      next_.store(0);
      busy_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return busy_ == 0; });
    job_ = nullptr;
  }

 private:
  void drain() {
    in_task() = true;
    for (int i; (i = next_.fetch_add(1)) < count_;) (*job_)(i);
    in_task() = false;
  }
  void work() {
    long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      drain();
      std::lock_guard<std::mutex> lk(m_);
      if (--busy_ == 0) done_.notify_one();
    }
  }

 public:
  static bool& in_task() {
    static thread_local bool t = false;
    return t;
  }

 private:
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  std::atomic<int> next_{0};
  int count_ = 0, busy_ = 0;
  long gen_ = 0;
  bool stop_ = false;
};

struct RefCtx {
  int logn = 0;
  std::size_t n = 0;
  int n_chain = 0, n_special = 0, alpha = 1, threads = 1;
  std::unique_ptr<Pool> pool;
  std::vector<helix::Modulus> mods;   // chain then special
  std::vector<helix::NttTables> ntt;  // same order
  std::unique_ptr<helix::LatticeContext> lc;
  std::unique_ptr<helix::CkksEncoder> enc;
};

template <class F>
void parallel_for(Pool* pool, int count, F f) {
  if (!pool || pool->size() <= 1 || count <= 1 || Pool::in_task()) {
    for (int i = 0; i < count; ++i) f(i);
    return;
  }
  const std::function<void(int)> fn = f;
  pool->run(count, fn);
}

int pidx(const RefCtx* c, int k, int n_q) { return k < n_q ? k : c->n_chain + (k - n_q); }

helix::RnsPoly to_rns(const RefCtx* c, const u64* data, int n_q, bool special,
                      helix::PolyDomain dom) {
  helix::RnsPoly p;
  p.has_special = special;
  p.domain = dom;
  const int nl = n_q + (special ? 1 : 0);
  p.limbs.resize(nl);
  for (int k = 0; k < nl; ++k) p.limbs[k].assign(data + (std::size_t)k * c->n, data + (std::size_t)(k + 1) * c->n);
  return p;
}

void from_rns(const RefCtx* c, const helix::RnsPoly& p, u64* out) {
  for (std::size_t k = 0; k < p.limbs.size(); ++k)
    std::memcpy(out + k * c->n, p.limbs[k].data(), c->n * 8);
}

// ---- key switching over reference primitives -------------------------------

void modup(const RefCtx* c, u64* D, const u64* c1, int n_q) {
  const std::size_t n = c->n;
  const int K = c->n_special, ext = n_q + K, dnum = (n_q + c->alpha - 1) / c->alpha;
  std::vector<u64> coef(c1, c1 + (std::size_t)n_q * n);
  parallel_for(c->pool.get(), n_q, [&](int i) {
    c->ntt[i].inverse(std::span<u64>(coef.data() + (std::size_t)i * n, n));
  });
  for (int d = 0; d < dnum; ++d) {
    const int lo = d * c->alpha, hi = std::min(lo + c->alpha, n_q);
    std::vector<u64> x((std::size_t)(hi - lo) * n);
    parallel_for(c->pool.get(), hi - lo, [&](int ii) {
      const int i = lo + ii;
      const auto& m = c->mods[i];
      u64 prod = 1;
      for (int i2 = lo; i2 < hi; ++i2)
        if (i2 != i) prod = m.mul(prod, c->mods[i2].q % m.q);
      const u64 inv = m.inv(prod);
      for (std::size_t t = 0; t < n; ++t) x[(i - lo) * n + t] = m.mul(coef[i * n + t], inv);
    });
    u64* out = D + (std::size_t)d * ext * n;
    parallel_for(c->pool.get(), ext, [&](int j) {
      u64* dst = out + (std::size_t)j * n;
      if (j >= lo && j < hi) {
        std::memcpy(dst, c1 + (std::size_t)j * n, n * 8);
        return;
      }
      const int pj = pidx(c, j, n_q);
      const auto& m = c->mods[pj];
      std::vector<u64> qh(hi - lo);
      for (int i = lo; i < hi; ++i) {
        u64 prod = 1;
        for (int i2 = lo; i2 < hi; ++i2)
          if (i2 != i) prod = m.mul(prod, c->mods[i2].q % m.q);
        qh[i - lo] = prod;
      }
      for (std::size_t t = 0; t < n; ++t) {
        u64 y = 0;
        for (int i = lo; i < hi; ++i) y = m.add(y, m.mul(x[(i - lo) * n + t] % m.q, qh[i - lo]));
        dst[t] = y;
      }
      c->ntt[pj].forward(std::span<u64>(dst, n));
    });
  }
}

u64 bitrev(u64 x, int bits) {
  u64 r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

std::vector<u64> perm_table(const RefCtx* c, u64 g) {
  std::vector<u64> perm(c->n);
  const u64 two_n = 2 * c->n;
  for (u64 k = 0; k < c->n; ++k) {
    if (g == 1) {
      perm[k] = k;
      continue;
    }
    const u64 e = 2 * bitrev(k, c->logn) + 1;
    const u64 m = (u64)(((unsigned __int128)g * e) % two_n);
    perm[k] = bitrev((m - 1) >> 1, c->logn);
  }
  return perm;
}

void inner_(const RefCtx* c, u64* U, const u64* D, const u64* key, int n_q, u64 g) {
  const std::size_t n = c->n;
  const int K = c->n_special, ext = n_q + K, full = c->n_chain + K;
  const int dnum = (n_q + c->alpha - 1) / c->alpha;
  const auto perm = perm_table(c, g);
  parallel_for(c->pool.get(), 2 * ext, [&](int cj) {
    const int cc = cj / ext, j = cj % ext, kl = pidx(c, j, n_q);
    const auto& m = c->mods[kl];
    u64* dst = U + ((std::size_t)cc * ext + j) * n;
    std::fill(dst, dst + n, 0);
    for (int d = 0; d < dnum; ++d) {
      const u64* Dd = D + ((std::size_t)d * ext + j) * n;
      const u64* kk = key + (((std::size_t)d * 2 + cc) * full + kl) * n;
      for (std::size_t t = 0; t < n; ++t) dst[t] = m.add(dst[t], m.mul(Dd[perm[t]], kk[t]));
    }
  });
}

// centred FastBConv ModDown; K = 1 is LatticeContext::moddown_special (rns_poly.cpp:164-180)
void moddown(const RefCtx* c, u64* out, const u64* U, int n_q) {
  const std::size_t n = c->n;
  const int K = c->n_special, ext = n_q + K;
  std::vector<u64> sp(U + (std::size_t)n_q * n, U + (std::size_t)ext * n);
  std::vector<u64> x((std::size_t)K * n);
  parallel_for(c->pool.get(), K, [&](int k) {
    const auto& m = c->mods[c->n_chain + k];
    c->ntt[c->n_chain + k].inverse(std::span<u64>(sp.data() + (std::size_t)k * n, n));
    u64 prod = 1;
    for (int k2 = 0; k2 < K; ++k2)
      if (k2 != k) prod = m.mul(prod, c->mods[c->n_chain + k2].q % m.q);
    const u64 inv = m.inv(prod);
    for (std::size_t t = 0; t < n; ++t) x[k * n + t] = m.mul(sp[k * n + t], inv);
  });
  parallel_for(c->pool.get(), n_q, [&](int i) {
    const auto& m = c->mods[i];
    std::vector<u64> ph(K);
    u64 Pq = 1;
    for (int k = 0; k < K; ++k) {
      u64 prod = 1;
      for (int k2 = 0; k2 < K; ++k2)
        if (k2 != k) prod = m.mul(prod, c->mods[c->n_chain + k2].q % m.q);
      ph[k] = prod;
      Pq = m.mul(Pq, c->mods[c->n_chain + k].q % m.q);
    }
    const u64 pinv = m.inv(Pq);
    std::vector<u64> v(n);
    for (std::size_t t = 0; t < n; ++t) {
      u64 acc = 0;
      for (int k = 0; k < K; ++k) {
        const auto& pk = c->mods[c->n_chain + k];
        acc = m.add(acc, m.mul(m.reduce_i64(pk.centered(x[k * n + t])), ph[k]));
      }
      v[t] = acc;
    }
    c->ntt[i].forward(std::span<u64>(v.data(), n));
    const u64* ui = U + (std::size_t)i * n;
    u64* oi = out + (std::size_t)i * n;
    for (std::size_t t = 0; t < n; ++t) oi[t] = m.mul(m.sub(ui[t], v[t]), pinv);
  });
}

}  // namespace

extern "C" {

void* ref_ctx_create(int logn, const u64* primes, int n_chain, int n_special, int alpha,
                     int delta_log2) {
  try {
    auto* c = new RefCtx;
    c->logn = logn;
    c->n = std::size_t(1) << logn;
    c->n_chain = n_chain;
    c->n_special = n_special;
    c->alpha = alpha;
    c->threads = 1;
    for (int i = 0; i < n_chain + n_special; ++i) {
      c->mods.emplace_back(primes[i]);
      c->ntt.emplace_back(helix::Modulus(primes[i]), c->n);
    }
    if (n_special == 1 && n_chain >= 2) {
      helix::CkksParams p;
      p.ring_degree = c->n;
      p.max_level = n_chain - 1;
      p.delta_log2 = delta_log2;
      p.moduli.assign(primes, primes + n_chain);
      p.special_primes.assign(primes + n_chain, primes + n_chain + 1);
      p.backend = helix::BackendKind::Lattice;
      p.insecure_toy = true;
      c->lc = std::make_unique<helix::LatticeContext>(p);
      c->enc = std::make_unique<helix::CkksEncoder>(*c->lc);
    }
    return c;
  } catch (...) {
    return nullptr;
  }
}

void ref_ctx_destroy(void* h) {
  auto* c = static_cast<RefCtx*>(h);
  c->enc.reset();
  c->lc.reset();
  delete c;
}

void ref_set_threads(void* h, int threads) {
  auto* c = static_cast<RefCtx*>(h);
  if (threads < 1) threads = 1;
  if (c->threads == threads && (threads == 1 || c->pool)) return;
  c->pool.reset();
  c->threads = threads;
  if (threads > 1) c->pool = std::make_unique<Pool>(threads);
}

u64 ref_psi(void* h, int i) { return static_cast<RefCtx*>(h)->ntt[i].psi(); }

void ref_ntt_fwd(void* h, int i, u64* data) {
  auto* c = static_cast<RefCtx*>(h);
  c->ntt[i].forward(std::span<u64>(data, c->n));
}

void ref_ntt_inv(void* h, int i, u64* data) {
  auto* c = static_cast<RefCtx*>(h);
  c->ntt[i].inverse(std::span<u64>(data, c->n));
}

// LatticeContext (K = 1) entry points; coefficient domain unless noted.
int ref_lc_automorphism(void* h, const u64* in, u64* out, int n_q, int with_special, u64 g) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->lc) return -1;
  auto p = to_rns(c, in, n_q, with_special != 0, helix::PolyDomain::Coeff);
  from_rns(c, c->lc->automorphism(p, g), out);
  return 0;
}

int ref_lc_rescale(void* h, const u64* in, u64* out, int n_q) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->lc) return -1;
  auto p = to_rns(c, in, n_q, false, helix::PolyDomain::Coeff);
  from_rns(c, c->lc->rescale_drop_last(p), out);
  return 0;
}

int ref_lc_moddown(void* h, const u64* in, u64* out, int n_q) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->lc) return -1;
  auto p = to_rns(c, in, n_q, true, helix::PolyDomain::Coeff);
  from_rns(c, c->lc->moddown_special(p), out);
  return 0;
}

int ref_lc_ring_mul(void* h, const u64* a, const u64* b, u64* out, int n_q) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->lc) return -1;
  auto pa = to_rns(c, a, n_q, false, helix::PolyDomain::Coeff);
  auto pb = to_rns(c, b, n_q, false, helix::PolyDomain::Coeff);
  from_rns(c, c->lc->ring_mul(pa, pb), out);
  return 0;
}

int ref_lc_mul_acc(void* h, const u64* a, const u64* b, u64* acc, int n_q) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->lc) return -1;
  auto pa = to_rns(c, a, n_q, false, helix::PolyDomain::Ntt);
  auto pb = to_rns(c, b, n_q, false, helix::PolyDomain::Ntt);
  auto pc = to_rns(c, acc, n_q, false, helix::PolyDomain::Ntt);
  c->lc->mul_acc(pa, pb, pc);
  from_rns(c, pc, acc);
  return 0;
}

// CkksEncoder::encode (encoder.cpp:97-117) -> coefficient-domain RNS limbs
int ref_encode(void* h, const double* m, int len, int level, double scale, u64* out) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->enc) return -1;
  try {
    auto p = c->enc->encode(std::span<const double>(m, len), level, scale);
    from_rns(c, p, out);
    return 0;
  } catch (...) {
    return -2;
  }
}

// CkksEncoder::decode (encoder.cpp:119-159); limbs in coefficient domain
int ref_decode(void* h, const u64* limbs, int n_q, double scale, double* out) {
  auto* c = static_cast<RefCtx*>(h);
  if (!c->enc) return -1;
  auto p = to_rns(c, limbs, n_q, false, helix::PolyDomain::Coeff);
  auto v = c->enc->decode(p, scale);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return 0;
}

// SPEC-only drivers over the reference primitives (the CPU reference arm).
int ref_keyswitch(void* h, const u64* in_ntt, const u64* key, u64* out, int n_q) {
  auto* c = static_cast<RefCtx*>(h);
  const std::size_t n = c->n;
  const int ext = n_q + c->n_special, dnum = (n_q + c->alpha - 1) / c->alpha;
  std::vector<u64> D((std::size_t)dnum * ext * n), U((std::size_t)2 * ext * n);
  modup(c, D.data(), in_ntt, n_q);
  inner_(c, U.data(), D.data(), key, n_q, 1);
  moddown(c, out, U.data(), n_q);
  moddown(c, out + (std::size_t)n_q * n, U.data() + (std::size_t)ext * n, n_q);
  return 0;
}

int ref_rotate(void* h, const u64* in_ct, const u64* key, u64* out_ct, int n_q, u64 g) {
  auto* c = static_cast<RefCtx*>(h);
  const std::size_t n = c->n, L = (std::size_t)n_q * n;
  const int ext = n_q + c->n_special, dnum = (n_q + c->alpha - 1) / c->alpha;
  std::vector<u64> D((std::size_t)dnum * ext * n), U((std::size_t)2 * ext * n), V(2 * L);
  modup(c, D.data(), in_ct + L, n_q);
  inner_(c, U.data(), D.data(), key, n_q, g);
  moddown(c, V.data(), U.data(), n_q);
  moddown(c, V.data() + L, U.data() + (std::size_t)ext * n, n_q);
  const auto perm = perm_table(c, g);
  parallel_for(c->pool.get(), n_q, [&](int i) {
    const auto& m = c->mods[i];
    for (std::size_t t = 0; t < n; ++t)
      out_ct[i * n + t] = m.add(in_ct[i * n + perm[t]], V[i * n + t]);
  });
  std::memcpy(out_ct + L, V.data() + L, L * 8);
  return 0;
}

// ---- BSGS matvec over the reference primitives (the matvec CPU arm) --------
// The same schedule as hxo_matvec_bsgs (lazy = 1, the product's double-hoisted
// giant steps): hoisted baby steps, the diagonal MAC with Modulus::mul/add
// (LatticeContext::mul_acc, rns_poly.cpp:102-110), giant key-switch products
// summed in the PQ basis with one ModDown per output, then the rescale of
// rns_poly.cpp:144-162 in the NTT domain (NttTables::inverse/forward).
// Limb loops run on the context's pool.
static u64 galois_of(const RefCtx* c, u64 r) {
  u64 g = 1;
  for (u64 i = 0; i < r; ++i) g = (g * 5) % (2 * c->n);
  return g;
}

static void ref_rescale_ntt(RefCtx* c, u64* out, const u64* in, int n_q) {
  const std::size_t n = c->n;
  std::vector<u64> last(in + (std::size_t)(n_q - 1) * n, in + (std::size_t)n_q * n);
  c->ntt[n_q - 1].inverse(std::span<u64>(last.data(), n));
  const auto& ql = c->mods[n_q - 1];
  parallel_for(c->pool.get(), n_q - 1, [&](int i) {
    const auto& m = c->mods[i];
    const u64 qinv = m.inv(ql.q % m.q);
    std::vector<u64> v(in + (std::size_t)i * n, in + (std::size_t)(i + 1) * n);
    c->ntt[i].inverse(std::span<u64>(v.data(), n));
    for (std::size_t t = 0; t < n; ++t) v[t] = m.mul(m.sub(v[t], m.reduce_i64(ql.centered(last[t]))), qinv);
    c->ntt[i].forward(std::span<u64>(v.data(), n));
    std::memcpy(out + (std::size_t)i * n, v.data(), n * 8);
  });
}

extern "C" int ref_matvec_bsgs(void* h, u64* out, const u64* x, int n_q, int n1, int n2, int blocks,
                               const u64* const* diags, const u64* const* keys, int gb, int ge, int rescale) {
  auto* c = static_cast<RefCtx*>(h);
  const std::size_t n = c->n, L = (std::size_t)n_q * n, ct = 2 * L;
  const int K = c->n_special, ext = n_q + K, dnum = (n_q + c->alpha - 1) / c->alpha;
  const u64 slots = n / 2;
  if (ge < 0) ge = n2;
  std::vector<u64> baby((std::size_t)n1 * ct), D((std::size_t)dnum * ext * n), U((std::size_t)2 * ext * n),
      S((std::size_t)2 * ext * n), V(ct), inner(ct), acc(ct);
  std::memcpy(baby.data(), x, ct * 8);
  if (n1 > 1) modup(c, D.data(), x + L, n_q);  // hoisted: one ModUp for every baby step
  for (int k = 1; k < n1; ++k) {
    const u64 g = galois_of(c, (u64)k);
    inner_(c, U.data(), D.data(), keys[k], n_q, g);
    moddown(c, V.data(), U.data(), n_q);
    moddown(c, V.data() + L, U.data() + (std::size_t)ext * n, n_q);
    const auto perm = perm_table(c, g);
    u64* bk = baby.data() + (std::size_t)k * ct;
    parallel_for(c->pool.get(), n_q, [&](int i) {
      const auto& m = c->mods[i];
      for (std::size_t t = 0; t < n; ++t) bk[i * n + t] = m.add(x[i * n + perm[t]], V[i * n + t]);
    });
    std::memcpy(bk + L, V.data() + L, L * 8);
  }
  for (int b = 0; b < blocks; ++b) {
    std::fill(acc.begin(), acc.end(), 0);
    std::fill(S.begin(), S.end(), 0);
    bool any_giant = false;
    for (int j = gb; j < ge; ++j) {
      bool live = false;
      std::fill(inner.begin(), inner.end(), 0);
      for (int k = 0; k < n1; ++k) {
        const u64* dg = diags[(std::size_t)b * n1 * n2 + (std::size_t)j * n1 + k];
        if (!dg) continue;
        live = true;
        const u64* bk = baby.data() + (std::size_t)k * ct;
        parallel_for(c->pool.get(), 2 * n_q, [&](int ci) {
          const int cc = ci / n_q, i = ci % n_q;
          const auto& m = c->mods[i];
          u64* o = inner.data() + cc * L + (std::size_t)i * n;
          const u64* a = bk + cc * L + (std::size_t)i * n;
          const u64* d = dg + (std::size_t)i * n;
          for (std::size_t t = 0; t < n; ++t) o[t] = m.add(o[t], m.mul(a[t], d[t]));
        });
      }
      if (!live) continue;
      if (j == 0) {
        parallel_for(c->pool.get(), 2 * n_q, [&](int ci) {
          const auto& m = c->mods[ci % n_q];
          for (std::size_t t = 0; t < n; ++t) acc[ci * n + t] = m.add(acc[ci * n + t], inner[ci * n + t]);
        });
        continue;
      }
      const u64 r = (u64)(((long long)n1 * j) % (long long)slots), g = galois_of(c, r);
      modup(c, D.data(), inner.data() + L, n_q);
      inner_(c, U.data(), D.data(), keys[r], n_q, g);
      const auto perm = perm_table(c, g);
      parallel_for(c->pool.get(), 2 * ext, [&](int cj) {
        const int j2 = cj % ext;
        const auto& m = c->mods[pidx(c, j2, n_q)];
        for (std::size_t t = 0; t < n; ++t) S[cj * n + t] = m.add(S[cj * n + t], U[cj * n + t]);
      });
      parallel_for(c->pool.get(), n_q, [&](int i) {
        const auto& m = c->mods[i];
        for (std::size_t t = 0; t < n; ++t) acc[i * n + t] = m.add(acc[i * n + t], inner[i * n + perm[t]]);
      });
      any_giant = true;
    }
    if (any_giant) {
      moddown(c, V.data(), S.data(), n_q);
      moddown(c, V.data() + L, S.data() + (std::size_t)ext * n, n_q);
      parallel_for(c->pool.get(), 2 * n_q, [&](int ci) {
        const auto& m = c->mods[ci % n_q];
        for (std::size_t t = 0; t < n; ++t) acc[ci * n + t] = m.add(acc[ci * n + t], V[ci * n + t]);
      });
    }
    if (rescale) {
      u64* o = out + (std::size_t)b * 2 * (n_q - 1) * n;
      ref_rescale_ntt(c, o, acc.data(), n_q);
      ref_rescale_ntt(c, o + (std::size_t)(n_q - 1) * n, acc.data() + L, n_q);
    } else {
      std::memcpy(out + (std::size_t)b * ct, acc.data(), ct * 8);
    }
  }
  return 0;
}

// The CPU reference arm over a batch: ciphertexts spread over the context's
// persistent pool, one whole (single-threaded) rotation per task -- the
// parallel axis BASELINE.md section 3 plans (independent ciphertexts).
int ref_rotate_batch(void* h, const u64* in_cts, const u64* key, u64* out_cts, int batch, int n_q, u64 g) {
  auto* c = static_cast<RefCtx*>(h);
  const std::size_t ct = (std::size_t)2 * n_q * c->n;
  if (batch == 1) return ref_rotate(h, in_cts, key, out_cts, n_q, g);
  parallel_for(c->pool.get(), batch, [&](int b) { ref_rotate(h, in_cts + b * ct, key, out_cts + b * ct, n_q, g); });
  return 0;
}

}  // extern "C"
