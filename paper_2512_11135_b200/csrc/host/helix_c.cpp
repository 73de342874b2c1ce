// helix_c.cpp -- C-ABI over GpuLatticeBackend + linalg (include/helix_c.h).
#include "helix_c.h"

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "helix/gpu_backend.hpp"
#include "hx_b200.h"
#include "helix/linalg.hpp"

using namespace helix;

struct hxc_backend {
  std::unique_ptr<GpuLatticeBackend> b;
};
struct hxc_ct {
  Ciphertext c;
};
struct hxc_mat {
  EncodedMatrix m;
  int method;
  BsgsShard shard;
};

namespace {
thread_local std::string g_err;

template <class T, class F>
T guard(T fail, F f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return fail;
  }
}

hxc_ct* wrap(Ciphertext c) { return new hxc_ct{std::move(c)}; }

void fill(hxc_report* r, const KernelReport& k) {
  if (!r) return;
  r->rotations = k.rotations;
  r->pt_muls = k.pt_muls;
  r->ct_muls = k.ct_muls;
  r->adds = k.adds;
  r->levels_consumed = k.levels_consumed;
  r->output_scale_log2 = k.output_scale.log2();
}
}  // namespace

extern "C" {

const char* hxc_last_error(void) { return g_err.c_str(); }

hxc_backend* hxc_backend_create(const char* json, uint64_t seed) {
  return guard<hxc_backend*>(nullptr, [&] {
    auto p = CkksParams::from_json(json);
    auto* h = new hxc_backend;
    h->b = std::make_unique<GpuLatticeBackend>(p, seed);
    return h;
  });
}

void hxc_backend_destroy(hxc_backend* b) { delete b; }
int64_t hxc_slots(hxc_backend* b) { return (int64_t)b->b->slots(); }
int hxc_max_level(hxc_backend* b) { return b->b->params().max_level; }
void* hxc_device_context(hxc_backend* b) { return b->b->device_context(); }

int hxc_trim(hxc_backend* b) {
  return guard(-1, [&] {
    b->b->trim();
    return 0;
  });
}

int hxc_gen_rotation_keys(hxc_backend* b, const int64_t* a, int n) {
  return guard(-1, [&] {
    b->b->generate_rotation_keys(std::span<const std::int64_t>(a, n));
    return 0;
  });
}

hxc_ct* hxc_encrypt(hxc_backend* b, const double* m, int len, int level) {
  return guard<hxc_ct*>(nullptr, [&] {
    auto& be = *b->b;
    return wrap(be.encrypt(be.encode(std::span<const double>(m, len), level, be.params().delta())));
  });
}

int hxc_decrypt(hxc_backend* b, const hxc_ct* ct, double* out) {
  return guard(-1, [&] {
    const auto v = b->b->decrypt(ct->c);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  });
}

void hxc_ct_free(hxc_ct* ct) { delete ct; }
int hxc_ct_level(const hxc_ct* ct) { return ct->c.level; }
double hxc_ct_scale_log2(const hxc_ct* ct) { return ct->c.scale.log2(); }
uint64_t* hxc_ct_device_ptr(const hxc_ct* ct) { return GpuLatticeBackend::payload(ct->c).data(); }

hxc_ct* hxc_add(hxc_backend* b, const hxc_ct* x, const hxc_ct* y) {
  return guard<hxc_ct*>(nullptr, [&] { return wrap(b->b->add(x->c, y->c)); });
}
hxc_ct* hxc_mul(hxc_backend* b, const hxc_ct* x, const hxc_ct* y) {
  return guard<hxc_ct*>(nullptr, [&] { return wrap(b->b->mul(x->c, y->c)); });
}
hxc_ct* hxc_mul_plain(hxc_backend* b, const hxc_ct* x, const double* m, int len) {
  return guard<hxc_ct*>(nullptr, [&] {
    auto& be = *b->b;
    const auto pt = be.encode(std::span<const double>(m, len), x->c.level, Scale::prime(be.modulus_at(x->c.level)));
    return wrap(be.mul_plain(x->c, pt));
  });
}
hxc_ct* hxc_rotate(hxc_backend* b, const hxc_ct* x, int64_t k) {
  return guard<hxc_ct*>(nullptr, [&] { return wrap(b->b->rotate(x->c, k)); });
}
hxc_ct* hxc_rescale(hxc_backend* b, const hxc_ct* x) {
  return guard<hxc_ct*>(nullptr, [&] { return wrap(b->b->rescale(x->c)); });
}
hxc_ct* hxc_mod_down(hxc_backend* b, const hxc_ct* x, int level) {
  return guard<hxc_ct*>(nullptr, [&] { return wrap(b->b->mod_down(x->c, level)); });
}
hxc_ct* hxc_rotate_and_sum(hxc_backend* b, const hxc_ct* x, int64_t span, int64_t stride, hxc_report* rep) {
  return guard<hxc_ct*>(nullptr, [&] {
    KernelReport k;
    auto c = rotate_and_sum(*b->b, x->c, (std::size_t)span, (std::size_t)stride, &k);
    fill(rep, k);
    return wrap(c);
  });
}

hxc_mat* hxc_matrix_prepare(hxc_backend* b, int method, const double* A, int rows, int cols, int level) {
  return hxc_matrix_prepare_plan(b, method, A, rows, cols, level, 0);
}

hxc_mat* hxc_matrix_prepare_plan(hxc_backend* b, int method, const double* A, int rows, int cols, int level,
                                 int n1) {
  return guard<hxc_mat*>(nullptr, [&] {
    Matrix M(rows, cols);
    std::memcpy(M.data.data(), A, sizeof(double) * (std::size_t)rows * cols);
    const std::size_t n = b->b->slots();
    static const bool trace = getenv("HX_PREP_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const bool bsgs = method == HXC_BSGS || method == HXC_BSGS_STACKED;
    if (n1 != 0 && !bsgs) throw std::invalid_argument("hxc_matrix_prepare_plan: n1 applies to the BSGS methods");
    BsgsPlan plan;
    if (bsgs) {
      const int d = next_pow2(std::max(cols, 1));
      const int blocks = method == HXC_BSGS_STACKED ? 1 : std::max(1, (rows + d - 1) / d);
      if (n1 == 0) {
        plan = BsgsPlan::for_dim(d);
      } else if (n1 < 0) {
        plan = BsgsPlan::for_cost(d, blocks);
      } else {
        if ((n1 & (n1 - 1)) || n1 > d) throw std::invalid_argument("hxc_matrix_prepare_plan: n1 must be a power of two <= d");
        plan.n1 = n1;
        plan.n2 = d / n1;
      }
    }
    PackedMatrix P = method == HXC_ROW              ? pack_rows(M, n)
                     : method == HXC_DIAG           ? pack_diagonals(M, n)
                     : method == HXC_BSGS_STACKED   ? pack_bsgs_stacked(M, plan, n)
                                                    : pack_bsgs(M, plan, n);
    const auto t1 = std::chrono::steady_clock::now();
    auto* h = new hxc_mat;
    h->method = method;
    h->m = encode_matrix(*b->b, P, level);
    if (trace) {
      const auto t2 = std::chrono::steady_clock::now();
      fprintf(stderr, "[prep] pack %.3f s, encode %.3f s\n", std::chrono::duration<double>(t1 - t0).count(),
              std::chrono::duration<double>(t2 - t1).count());
    }
    return h;
  });
}

void hxc_matrix_free(hxc_mat* m) { delete m; }

int hxc_matrix_info(const hxc_mat* m, int* d, int* n1, int* n2, int* blocks, int* nonzero) {
  if (d) *d = m->m.meta.d;
  if (n1) *n1 = m->m.meta.plan.n1;
  if (n2) *n2 = m->m.meta.plan.n2;
  if (blocks) *blocks = m->m.meta.row_blocks;
  if (nonzero) {
    int c = 0;
    for (const auto& p : m->m.pts) c += p.payload != nullptr;
    *nonzero = c;
  }
  return 0;
}

int hxc_matrix_rotations(const hxc_mat* m, int64_t* out, int cap) {
  std::vector<std::int64_t> r = m->method == HXC_ROW    ? row_rotations(m->m.meta)
                                : m->method == HXC_DIAG ? diag_rotations(m->m.meta.d)
                                                        : bsgs_rotations(m->m.meta.plan);
  for (int i = 0; i < (int)r.size() && i < cap; ++i) out[i] = r[i];
  return (int)r.size();
}

int hxc_matvec(hxc_backend* b, const hxc_mat* m, const hxc_ct* x, hxc_ct** out, int cap, hxc_report* rep) {
  return guard(-1, [&] {
    MatvecResult r = m->method == HXC_ROW    ? matvec_row(*b->b, m->m, x->c)
                     : m->method == HXC_DIAG ? matvec_diag(*b->b, m->m, x->c)
                                             : matvec_bsgs(*b->b, m->m, x->c);
    fill(rep, r.report);
    int k = 0;
    for (; k < (int)r.outputs.size() && k < cap; ++k) out[k] = wrap(r.outputs[k]);
    return (int)r.outputs.size();
  });
}

int hxc_matvec_tokens(hxc_backend* b, const hxc_mat* m, const hxc_ct* const* xs, int T, hxc_ct** out, int cap,
                      hxc_report* rep) {
  return guard(-1, [&] {
    if (m->method != HXC_BSGS && m->method != HXC_BSGS_STACKED)
      throw std::invalid_argument("hxc_matvec_tokens: BSGS matrices only");
    std::vector<Ciphertext> in;
    for (int t = 0; t < T; ++t) in.push_back(xs[t]->c);
    const auto rs = matvec_bsgs_tokens(*b->b, m->m, in);
    int k = 0;
    for (const auto& r : rs)
      for (const auto& c : r.outputs) {
        if (k < cap) out[k] = wrap(c);
        ++k;
      }
    if (!rs.empty()) fill(rep, rs.front().report);
    return k;
  });
}

hxc_mat* hxc_matrix_prepare_shard(hxc_backend* b, const double* A, int rows, int cols, int level, int rank,
                                  int world, int stacked) {
  return guard<hxc_mat*>(nullptr, [&] {
    Matrix M(rows, cols);
    std::memcpy(M.data.data(), A, sizeof(double) * (std::size_t)rows * cols);
    const PackedMatrix P = stacked ? pack_bsgs_stacked(M, b->b->slots()) : pack_bsgs(M, b->b->slots());
    auto* h = new hxc_mat;
    h->method = stacked ? HXC_BSGS_STACKED : HXC_BSGS;
    h->shard = bsgs_shard(P.plan, rank, world);
    h->m = encode_matrix(*b->b, P, level, h->shard);
    return h;
  });
}

int hxc_matvec_shard(hxc_backend* b, const hxc_mat* m, const hxc_ct* x, hxc_ct** out, int cap, hxc_report* rep) {
  return guard(-1, [&] {
    BsgsShard s = m->shard;
    s.rescale = false;
    MatvecResult r = matvec_bsgs(*b->b, m->m, x->c, s);
    fill(rep, r.report);
    int k = 0;
    for (; k < (int)r.outputs.size() && k < cap; ++k) out[k] = wrap(r.outputs[k]);
    return (int)r.outputs.size();
  });
}

hxc_ct* hxc_ct_like(hxc_backend* b, const hxc_ct* like, const uint64_t* words) {
  return guard<hxc_ct*>(nullptr, [&] {
    const std::size_t w = (std::size_t)2 * (like->c.level + 1) * b->b->params().ring_degree;
    auto buf = std::make_shared<DeviceBuffer>(w);
    if (cudaMemcpyAsync(buf->ptr, words, w * 8, cudaMemcpyDeviceToDevice, nullptr) != cudaSuccess)
      throw std::runtime_error("hxc_ct_like: copy failed");
    return wrap(b->b->wrap(buf, 0, like->c.level, like->c.scale));
  });
}

long long hxc_shard_partial_words(hxc_backend* b, const hxc_ct* like) {
  return (long long)b->b->shard_partial_words(like->c.level);
}

hxc_ct* hxc_shard_finish(hxc_backend* b, const hxc_ct* like, const uint64_t* words) {
  return guard<hxc_ct*>(nullptr, [&] { return wrap(b->b->shard_finish(like->c, words)); });
}

hxc_ct* hxc_matmul(hxc_backend* b, const hxc_ct* A, const hxc_ct* B, int d, hxc_report* rep) {
  return guard<hxc_ct*>(nullptr, [&] {
    auto r = matmul_ctct(*b->b, A->c, B->c, d);
    fill(rep, r.second);
    return wrap(r.first);
  });
}

int hxc_matmul_heads(hxc_backend* b, const hxc_ct* const* As, const hxc_ct* const* Bs, int H, int d, hxc_ct** out,
                     hxc_report* rep) {
  return guard(-1, [&] {
    auto* g = b->b.get();
    std::vector<Ciphertext> A, B;
    for (int h = 0; h < H; ++h) {
      A.push_back(As[h]->c);
      B.push_back(Bs[h]->c);
    }
    const auto snap = TraceSnapshot::take(g->trace());
    const auto outs = g->matmul_heads(A, B, d);
    KernelReport r;
    r.rotations = snap.delta(g->trace(), OpKind::Rotate) / (std::uint64_t)H;
    r.pt_muls = snap.delta(g->trace(), OpKind::PtMul) / (std::uint64_t)H;
    r.ct_muls = snap.delta(g->trace(), OpKind::CtMul) / (std::uint64_t)H;
    r.adds = snap.delta(g->trace(), OpKind::CtAdd) / (std::uint64_t)H;
    r.levels_consumed = A[0].level - outs[0].level;
    r.output_scale = outs[0].scale;
    fill(rep, r);
    for (int h = 0; h < H; ++h) out[h] = wrap(outs[h]);
    return H;
  });
}

long long hxc_predicted_rotations(int method, int rows, int cols, int64_t slots) {
  return guard<long long>(-1, [&] {
    const Layout l = method == HXC_ROW    ? Layout::PackedRow
                     : method == HXC_DIAG ? Layout::Diagonal
                     : method == HXC_BSGS_STACKED ? Layout::BsgsStacked
                                                  : Layout::BsgsDiagonal;
    return (long long)predicted_rotations(l, rows, cols, (std::size_t)slots);
  });
}

hxc_ct* hxc_polyeval(hxc_backend* b, const hxc_ct* x, const double* coeffs, int n, int chebyshev, double lo,
                     double hi, hxc_report* rep) {
  return guard<hxc_ct*>(nullptr, [&] {
    KernelReport k;
    auto c = polyeval(*b->b, x->c, std::vector<double>(coeffs, coeffs + n),
                      chebyshev ? PolyBasis::Chebyshev : PolyBasis::Power, lo, hi, &k);
    fill(rep, k);
    return wrap(c);
  });
}

int hxc_matmul_rotations(int d, int64_t* out, int cap) {
  const auto r = matmul_rotations(d, 0);
  for (int i = 0; i < (int)r.size() && i < cap; ++i) out[i] = r[i];
  return (int)r.size();
}

const uint64_t* hxc_secret_key_ptr(hxc_backend* b) { return b->b->secret_key_words(); }
const uint64_t* hxc_relin_key_ptr(hxc_backend* b) { return b->b->relin_key_words(); }
const uint64_t* hxc_rotation_key_ptr(hxc_backend* b, int64_t k) {
  return b->b->rotation_key(detail::reduce_amount(k, (std::int64_t)b->b->slots()));
}
int hxc_key_expand(hxc_backend* b, const uint64_t* ckey, uint64_t* full_dev) {
  return guard(-1, [&] {
    b->b->expand_key(ckey, full_dev);
    return 0;
  });
}

const uint64_t* hxc_matrix_payload_ptr(const hxc_mat* m, int i) {
  if (i < 0 || i >= (int)m->m.pts.size() || !m->m.pts[i].payload) return nullptr;
  return GpuLatticeBackend::payload(m->m.pts[i]).data();
}
int hxc_matrix_payload_count(const hxc_mat* m) { return (int)m->m.pts.size(); }

int hxc_encode_words(hxc_backend* b, const double* m, int len, int level, double scale, uint64_t* out) {
  return guard(-1, [&] {
    auto& be = *b->b;
    const auto pt = be.encode(std::span<const double>(m, len), level, Scale::raw(scale));
    const std::size_t w = (std::size_t)(level + 1) * be.params().ring_degree;
    if (cudaMemcpy(out, GpuLatticeBackend::payload(pt).data(), w * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("hxc_encode_words: copy failed");
    return 0;
  });
}

int hxc_encode_coeffs(const char* json, const double* m, int len, int level, double scale, int64_t* out) {
  return guard(-1, [&] {
    const CkksEncoder enc(CkksParams::from_json(json));
    const auto c = enc.encode_coeffs(std::span<const double>(m, len), level, scale);
    std::memcpy(out, c.data(), c.size() * 8);
    return 0;
  });
}

int hxc_decode_coeffs(const char* json, const uint64_t* limbs, int n_limbs, double scale, double* out) {
  return guard(-1, [&] {
    const CkksEncoder enc(CkksParams::from_json(json));
    const std::size_t n = enc.ring_degree();
    const auto v = enc.decode_coeffs(std::span<const std::uint64_t>(limbs, (std::size_t)n_limbs * n), n_limbs, scale);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  });
}

int hxc_trace_json(hxc_backend* b, char* buf, int cap) {
  const auto s = b->b->trace().to_json();
  if (buf && cap > 0) {
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return (int)s.size();
}

void hxc_trace_reset(hxc_backend* b) { b->b->trace().reset(); }

int hxc_sync(void) { return cudaDeviceSynchronize() == cudaSuccess ? 0 : -1; }

}  // extern "C"
