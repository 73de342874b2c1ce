// linalg.cpp -- encrypted linear algebra over SlotOps.
#include "helix/linalg.hpp"

#include <map>
#include <optional>
#include <sstream>

#ifndef HELIX_NO_GPU
#include "helix/gpu_backend.hpp"
#endif

namespace helix {

namespace {

int ilog2(std::size_t v) {
  int l = 0;
  while ((std::size_t(1) << l) < v) ++l;
  return l;
}

KernelReport report_since(OpTrace& t, const TraceSnapshot& s, int in_level, const Ciphertext& out) {
  KernelReport r;
  r.rotations = s.delta(t, OpKind::Rotate);
  r.pt_muls = s.delta(t, OpKind::PtMul);
  r.ct_muls = s.delta(t, OpKind::CtMul);
  r.adds = s.delta(t, OpKind::CtAdd) + s.delta(t, OpKind::PtAdd);
  r.levels_consumed = in_level - out.level;
  r.output_scale = out.scale;
  return r;
}

Ciphertext add_opt(SlotOps& ops, std::optional<Ciphertext>& acc, const Ciphertext& t) {
  acc = acc ? ops.add(*acc, t) : t;
  return *acc;
}

void require_matvec_input(const EncodedMatrix& M, const Ciphertext& x, Layout want) {
  const bool ok = M.meta.layout == want || (want == Layout::BsgsDiagonal && M.meta.layout == Layout::BsgsStacked);
  if (!ok) throw std::invalid_argument("matvec: wrong matrix layout");
  detail::require_same_level(x.level, M.level, "matvec");
  if (x.level < 1) throw LevelUnderflowError("matvec: level budget < 1");
}

}  // namespace

std::string KernelReport::to_json() const {
  std::ostringstream o;
  o << "{\"rotations\": " << rotations << ", \"pt_muls\": " << pt_muls << ", \"ct_muls\": " << ct_muls
    << ", \"adds\": " << adds << ", \"levels_consumed\": " << levels_consumed << ", \"output_scale_log2\": "
    << output_scale.log2() << "}";
  return o.str();
}

EncodedMatrix encode_matrix(SlotOps& ops, const PackedMatrix& M, int level) {
  EncodedMatrix E;
  E.meta = M;
  E.meta.payloads.clear();
  E.level = level;
  if (M.layout == Layout::RowMajor) throw std::invalid_argument("encode_matrix: RowMajor operands are ciphertexts");
  const Scale s = Scale::prime(ops.modulus_at(level));
#ifndef HELIX_NO_GPU
  if (auto* g = dynamic_cast<GpuLatticeBackend*>(&ops)) {
    E.pts = g->encode_many(M.payloads, level, s);
    return E;
  }
#endif
  {
    for (const auto& p : M.payloads) {
      if (p.empty()) {
        Plaintext z;
        z.level = level;
        z.scale = s;
        z.slot_count = ops.slots();
        E.pts.push_back(z);
      } else {
        E.pts.push_back(ops.encode(p, level, s));
      }
    }
  }
  return E;
}

Ciphertext rotate_and_sum(SlotOps& ops, const Ciphertext& ct, std::size_t span, std::size_t stride,
                          KernelReport* report) {
  if (span == 0 || (span & (span - 1))) throw std::invalid_argument("rotate_and_sum: span must be a power of two");
  const auto snap = TraceSnapshot::take(ops.trace());
  Ciphertext acc = ct;
  for (std::size_t s = 1; s < span; s <<= 1) acc = ops.add(acc, ops.rotate(acc, (std::int64_t)(stride * s)));
  if (report) *report = report_since(ops.trace(), snap, ct.level, acc);
  return acc;
}

// ------------------------------------------------------------------- BSGS
MatvecResult matvec_bsgs(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x) {
  return matvec_bsgs(ops, M, x, BsgsShard{});
}

BsgsShard bsgs_shard(const BsgsPlan& plan, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bsgs_shard: bad rank/world");
  BsgsShard s;
  s.giant_begin = (int)((long long)plan.n2 * rank / world);
  s.giant_end = (int)((long long)plan.n2 * (rank + 1) / world);
  s.rescale = world == 1;
  return s;
}

EncodedMatrix encode_matrix(SlotOps& ops, const PackedMatrix& M, int level, const BsgsShard& shard) {
  if (M.layout != Layout::BsgsDiagonal && M.layout != Layout::BsgsStacked)
    throw std::invalid_argument("encode_matrix: shards apply to BSGS layouts");
  PackedMatrix S = M;
  const int n1 = M.plan.n1, ge = shard.giant_end < 0 ? M.plan.n2 : shard.giant_end;
  for (int b = 0; b < M.row_blocks; ++b)
    for (int i = 0; i < M.d; ++i) {
      const int j = i / n1;
      if (j < shard.giant_begin || j >= ge) S.payloads[(std::size_t)b * M.d + i].clear();
    }
  return encode_matrix(ops, S, level);
}

MatvecResult matvec_bsgs(SlotOps& ops, const EncodedMatrix& Min, const Ciphertext& x, const BsgsShard& shard) {
  require_matvec_input(Min, x, Layout::BsgsDiagonal);
  const auto snap = TraceSnapshot::take(ops.trace());
  const int d = Min.meta.d, n1 = Min.meta.plan.n1, n2 = Min.meta.plan.n2;
  const int gb = shard.giant_begin, ge = shard.giant_end < 0 ? n2 : shard.giant_end;
  const bool sharded = gb > 0 || ge < n2;
  // groups outside the shard are treated as zero
  EncodedMatrix Msh;
  if (sharded) {
    Msh.meta = Min.meta;
    Msh.level = Min.level;
    Msh.pts = Min.pts;
    for (std::size_t i = 0; i < Msh.pts.size(); ++i) {
      const int j = (int)(i % (std::size_t)d) / n1;
      if (j < gb || j >= ge) Msh.pts[i].payload.reset();
    }
  }
  const EncodedMatrix& M = sharded ? Msh : Min;
  auto finish = [&](const Ciphertext& acc) { return shard.rescale ? ops.rescale(acc) : acc; };
  MatvecResult R;
#ifndef HELIX_NO_GPU
  auto* gpu = dynamic_cast<GpuLatticeBackend*>(&ops);
#endif
  // baby steps Rot(x, k), k < n1, shared by every row block
  std::vector<Ciphertext> baby;
#ifndef HELIX_NO_GPU
  if (gpu) {
    std::vector<std::int64_t> ks(n1);
    for (int k = 0; k < n1; ++k) ks[k] = k;
    baby = gpu->rotate_many(x, ks);  // one ModUp for all n1 - 1 rotations
  } else
#endif
  {
    baby.push_back(x);
    for (int k = 1; k < n1; ++k) baby.push_back(ops.rotate(x, k));
  }
#ifndef HELIX_NO_GPU
  if (gpu) {
    for (const auto& acc : gpu->bsgs_blocks(baby, M.pts, n1, n2, M.meta.row_blocks, sharded))
      R.outputs.push_back(finish(acc));
    R.report = report_since(ops.trace(), snap, x.level, R.outputs.front());
    return R;
  }
#endif
  for (int b = 0; b < M.meta.row_blocks; ++b) {
    const std::vector<Plaintext> diags(M.pts.begin() + (std::ptrdiff_t)b * d,
                                       M.pts.begin() + (std::ptrdiff_t)(b + 1) * d);
    Ciphertext acc;
    {
      std::optional<Ciphertext> sum;
      for (int j = 0; j < n2; ++j) {
        std::optional<Ciphertext> inner;
        for (int k = 0; k < n1; ++k) {
          const Plaintext& pt = diags[(std::size_t)j * n1 + k];
          if (!pt.payload) continue;
          add_opt(ops, inner, ops.mul_plain(baby[k], pt));
        }
        if (!inner) continue;
        add_opt(ops, sum, j ? ops.rotate(*inner, (std::int64_t)n1 * j) : *inner);
      }
      if (!sum) throw std::invalid_argument("matvec_bsgs: block has no non-zero diagonal");
      acc = *sum;
    }
    R.outputs.push_back(finish(acc));
  }
  R.report = report_since(ops.trace(), snap, x.level, R.outputs.front());
  return R;
}

std::vector<MatvecResult> matvec_bsgs_tokens(SlotOps& ops, const EncodedMatrix& M, const std::vector<Ciphertext>& xs) {
  std::vector<MatvecResult> out;
  if (xs.empty()) return out;
#ifndef HELIX_NO_GPU
  if (auto* gpu = dynamic_cast<GpuLatticeBackend*>(&ops)) {
    for (const auto& x : xs) require_matvec_input(M, x, Layout::BsgsDiagonal);
    const int n1 = M.meta.plan.n1, n2 = M.meta.plan.n2;
    std::vector<std::int64_t> ks(n1);
    for (int k = 0; k < n1; ++k) ks[k] = k;
    const auto snap = TraceSnapshot::take(ops.trace());
    const auto babies = gpu->rotate_many_tokens(xs, ks);
    const auto accs = gpu->bsgs_blocks_tokens(babies, M.pts, n1, n2, M.meta.row_blocks);
    for (const auto& per : accs) {
      MatvecResult R;
      for (const auto& a : per) R.outputs.push_back(ops.rescale(a));
      out.push_back(std::move(R));
    }
    // the batch's counters, reported per token (identical for every token)
    KernelReport rep = report_since(ops.trace(), snap, xs[0].level, out[0].outputs.front());
    const auto T = (std::uint64_t)xs.size();
    rep.rotations /= T;
    rep.pt_muls /= T;
    rep.ct_muls /= T;
    rep.adds /= T;
    for (auto& r : out) r.report = rep;
    return out;
  }
#endif
  for (const auto& x : xs) out.push_back(matvec_bsgs(ops, M, x));
  return out;
}

// ------------------------------------------------------------------- diagonal
MatvecResult matvec_diag(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x) {
  require_matvec_input(M, x, Layout::Diagonal);
  const auto snap = TraceSnapshot::take(ops.trace());
  const int d = M.meta.d;
  std::vector<bool> need(d, false);
  for (int b = 0; b < M.meta.row_blocks; ++b)
    for (int i = 0; i < d; ++i) need[i] = need[i] || M.pts[(std::size_t)b * d + i].payload != nullptr;
  std::map<int, Ciphertext> rot;
#ifndef HELIX_NO_GPU
  if (auto* gpu = dynamic_cast<GpuLatticeBackend*>(&ops)) {
    std::vector<std::int64_t> ks;
    for (int i = 0; i < d; ++i)
      if (need[i]) ks.push_back(i);
    const auto r = gpu->rotate_many(x, ks);
    for (std::size_t j = 0; j < ks.size(); ++j) rot.emplace((int)ks[j], r[j]);
  } else
#endif
  {
    for (int i = 0; i < d; ++i)
      if (need[i]) rot.emplace(i, i ? ops.rotate(x, i) : x);
  }
  MatvecResult R;
  for (int b = 0; b < M.meta.row_blocks; ++b) {
    std::optional<Ciphertext> acc;
    for (int i = 0; i < d; ++i) {
      const Plaintext& pt = M.pts[(std::size_t)b * d + i];
      if (pt.payload) add_opt(ops, acc, ops.mul_plain(rot.at(i), pt));
    }
    if (!acc) throw std::invalid_argument("matvec_diag: block has no non-zero diagonal");
    R.outputs.push_back(ops.rescale(*acc));
  }
  R.report = report_since(ops.trace(), snap, x.level, R.outputs.front());
  return R;
}

// ------------------------------------------------------------------- packed rows
// Per payload g: t = rescale(x (.) rows_g); rotate_and_sum(t, pad_cols, 1)
// leaves row r's dot product in slots [r pc, (r+1) pc).  Assembly
// (SPEC.md:422): mask slot r pc (second level), rotate left by
// r pc - (g p + r) so it lands in slot g p + r, sum, rescale.
MatvecResult matvec_row(SlotOps& ops, const EncodedMatrix& M, const Ciphertext& x) {
  if (M.meta.layout != Layout::PackedRow) throw std::invalid_argument("matvec_row: wrong layout");
  detail::require_same_level(x.level, M.level, "matvec_row");
  if (x.level < 2) throw LevelUnderflowError("matvec_row: level budget < 2");
  const auto snap = TraceSnapshot::take(ops.trace());
  const int pc = M.meta.pad_cols, p = M.meta.rows_per_payload, R = M.meta.rows;
  const std::size_t n = ops.slots();
  const int lvl1 = x.level - 1;
  const Scale mscale = Scale::prime(ops.modulus_at(lvl1));
  std::map<int, Plaintext> masks;
  std::optional<Ciphertext> acc;
  for (std::size_t g = 0; g < M.pts.size(); ++g) {
    Ciphertext t = ops.rescale(ops.mul_plain(x, M.pts[g]));
    t = rotate_and_sum(ops, t, (std::size_t)pc, 1);
    for (int r = 0; r < p; ++r) {
      const int row = (int)g * p + r;
      if (row >= R) break;
      auto it = masks.find(r);
      if (it == masks.end()) {
        std::vector<double> m(n, 0.0);
        m[(std::size_t)r * pc] = 1.0;
        it = masks.emplace(r, ops.encode(m, lvl1, mscale)).first;
      }
      Ciphertext u = ops.mul_plain(t, it->second);
      const std::int64_t shift = (std::int64_t)r * pc - row;
      if (detail::reduce_amount(shift, (std::int64_t)n) != 0) u = ops.rotate(u, shift);
      add_opt(ops, acc, u);
    }
  }
  MatvecResult Rz;
  Rz.outputs.push_back(ops.rescale(*acc));
  Rz.report = report_since(ops.trace(), snap, x.level, Rz.outputs.front());
  return Rz;
}

// ------------------------------------------------------------------- SPEC forms
static std::pair<Ciphertext, KernelReport> single(MatvecResult r) {
  if (r.outputs.size() != 1) throw std::invalid_argument("matvec: matrix has several row blocks; use the EncodedMatrix form");
  return {r.outputs.front(), r.report};
}

std::pair<Ciphertext, KernelReport> matvec_bsgs(SlotOps& ops, const PackedMatrix& M, const Ciphertext& x,
                                                const BsgsPlan& plan) {
  if (plan.n1 != M.plan.n1 || plan.n2 != M.plan.n2) throw std::invalid_argument("matvec_bsgs: plan mismatch");
  return single(matvec_bsgs(ops, encode_matrix(ops, M, x.level), x));
}
std::pair<Ciphertext, KernelReport> matvec_diag(SlotOps& ops, const PackedMatrix& M, const Ciphertext& x) {
  return single(matvec_diag(ops, encode_matrix(ops, M, x.level), x));
}
std::pair<Ciphertext, KernelReport> matvec_row(SlotOps& ops, const PackedMatrix& M, const Ciphertext& x) {
  return single(matvec_row(ops, encode_matrix(ops, M, x.level), x));
}

// ------------------------------------------------------------------- matmul
std::pair<Ciphertext, KernelReport> matmul_ctct(SlotOps& ops, const Ciphertext& A, const Ciphertext& B,
                                                int d) {
  if (d < 1 || (d & (d - 1))) throw std::invalid_argument("matmul_ctct: d must be a power of two");
  const std::size_t n = ops.slots();
  if ((std::size_t)d * d > n) throw std::invalid_argument("matmul_ctct: d^2 > n");
  detail::require_same_level(A.level, B.level, "matmul_ctct");
  if (A.level < 2) throw LevelUnderflowError("matmul_ctct: requires a multiplicative level of 2");
  const auto snap = TraceSnapshot::take(ops.trace());
#ifndef HELIX_NO_GPU
  if (auto* g = dynamic_cast<GpuLatticeBackend*>(&ops)) {  // batched device pipeline
    const Ciphertext out = g->matmul(A, B, d);
    return {out, report_since(ops.trace(), snap, A.level, out)};
  }
#endif
  const int lv = A.level, lg = ilog2((std::size_t)d);
  // A's column mask at scale q_l (A_col keeps Delta); B's row mask at scale
  // q_l q_{l-1} / Delta so that the ct-ct product has scale Delta q_{l-1} and
  // the final rescale by q_{l-1} restores exactly Delta (SPEC.md:417 invariant)
  const Scale ms = Scale::prime(ops.modulus_at(lv));
  const Scale ms_b = ms * Scale::prime(ops.modulus_at(lv - 1)) / ops.params().delta();
  std::optional<Ciphertext> C;
  for (int j = 0; j < d; ++j) {
    const Plaintext cm = ops.encode(make_mask(MaskKind::ColumnExtractor, j, d, n), lv, ms);
    const Plaintext rm = ops.encode(make_mask(MaskKind::RowExtractor, j, d, n), lv, ms_b);
    Ciphertext a = ops.rescale(ops.mul_plain(A, cm));
    Ciphertext b = ops.rescale(ops.mul_plain(B, rm));
    if (j) {
      a = ops.rotate(a, j);                      // column j -> column 0
      b = ops.rotate(b, (std::int64_t)d * j);    // row j -> row 0
    }
    for (int i = 0; i < lg; ++i) a = ops.add(a, ops.rotate(a, -(std::int64_t(1) << i)));
    for (int i = 0; i < lg; ++i) b = ops.add(b, ops.rotate(b, -((std::int64_t)d << i)));
    add_opt(ops, C, ops.mul(a, b));
  }
  const Ciphertext out = ops.rescale(*C);
  return {out, report_since(ops.trace(), snap, A.level, out)};
}

std::int64_t predicted_rotations(Layout layout, int rows, int cols, std::size_t slots) {
  if (rows < 1 || cols < 1) throw std::invalid_argument("predicted_rotations: empty matrix");
  int pc = 1;
  while (pc < cols) pc <<= 1;
  if ((std::size_t)pc > slots) throw std::invalid_argument("predicted_rotations: input dimension exceeds the slot count");
  const int lg = ilog2((std::size_t)pc);
  switch (layout) {
    case Layout::PackedRow: {
      const int p = std::max(1, std::min((int)(slots / pc), rows));
      const std::int64_t groups = (rows + p - 1) / p;
      std::int64_t r = groups * lg;
      for (int row = 0; row < rows; ++row)
        if (detail::reduce_amount((std::int64_t)(row % p) * pc - row, (std::int64_t)slots) != 0) ++r;
      return r;
    }
    case Layout::Diagonal:
      return pc - 1;
    case Layout::BsgsDiagonal: {
      const BsgsPlan plan = BsgsPlan::for_dim(pc);
      const std::int64_t blocks = (rows + pc - 1) / pc;
      return (plan.n1 - 1) + blocks * (plan.n2 - 1);
    }
    case Layout::BsgsStacked: {
      const BsgsPlan plan = BsgsPlan::for_dim(pc);
      return (plan.n1 - 1) + (plan.n2 - 1);
    }
    default:
      throw std::invalid_argument("predicted_rotations: not a matvec layout");
  }
}

// ------------------------------------------------------------------- polyeval
int polyeval_depth(std::size_t n, PolyBasis basis) {
  int m = 0;
  while ((std::size_t(1) << m) < n) ++m;
  return std::max(1, m) + (basis == PolyBasis::Chebyshev ? 1 : 0);
}

namespace {
struct PolyCtx {
  SlotOps& ops;
  PolyBasis basis;
  Ciphertext x;                      // the variable (y for Chebyshev), level L0
  std::vector<Ciphertext> pw;        // pw[k] = X_{2^k}
  std::vector<double> constv(double c) const { return std::vector<double>(ops.slots(), c); }

  // X_{2^k}: x^(2^k) by squaring, or T_(2^k) = 2 T_(2^(k-1))^2 - 1
  const Ciphertext& power(int k) {
    while ((int)pw.size() <= k) {
      const Ciphertext& p = pw.back();
      Ciphertext sq = ops.rescale(ops.mul(p, p));
      if (basis == PolyBasis::Chebyshev) {
        sq = ops.add(sq, sq);
        sq = ops.add_plain(sq, ops.encode(constv(-1.0), sq.level, sq.scale));
      }
      pw.push_back(sq);
    }
    return pw[k];
  }

  // c[0..n) evaluated to (level, scale) exactly; level <= L0 - depth(n)
  Ciphertext eval(const std::vector<double>& c, int level, const Scale& target) {
    const std::size_t n = c.size();
    if (n <= 2) {  // c0 + c1 X: one plaintext product at level + 1, scale chosen to land on `target`
      const int l1 = level + 1;
      const Ciphertext xl = x.level == l1 ? x : ops.mod_down(x, l1);
      const Scale s = target * Scale::prime(ops.modulus_at(l1)) / x.scale;
      Ciphertext y = ops.rescale(ops.mul_plain(xl, ops.encode(constv(n > 1 ? c[1] : 0.0), l1, s)));
      if (c[0] != 0.0) y = ops.add_plain(y, ops.encode(constv(c[0]), level, target));
      return y;
    }
    int m = 0;
    while ((std::size_t(1) << m) < n) ++m;
    const std::size_t h = std::size_t(1) << (m - 1);
    std::vector<double> lo(c.begin(), c.begin() + (std::ptrdiff_t)h), hi(c.begin() + (std::ptrdiff_t)h, c.end());
    if (basis == PolyBasis::Chebyshev) {  // p = lo + T_h hi (Chebyshev division by T_h)
      for (std::size_t j = 1; j < hi.size(); ++j) {
        lo[h - j] -= c[h + j];
        hi[j] = 2.0 * c[h + j];
      }
    }
    const Ciphertext& P = power(m - 1);
    const int lp = P.level;
    // hi at (lp, T q_lp / S_P): the product's rescale lands exactly on `target`
    const Scale th = target * Scale::prime(ops.modulus_at(lp)) / P.scale;
    Ciphertext prod;
    if (hi.size() == 1) {  // constant quotient: a plaintext product instead of a ciphertext one
      prod = ops.rescale(ops.mul_plain(P, ops.encode(constv(hi[0]), lp, th)));
    } else {
      prod = ops.rescale(ops.mul(P, eval(hi, lp, th)));
    }
    if (prod.level != level) prod = ops.mod_down(prod, level);
    return ops.add(eval(lo, level, target), prod);
  }
};
}  // namespace

Ciphertext polyeval(SlotOps& ops, const Ciphertext& x, const std::vector<double>& coeffs, PolyBasis basis,
                    double a, double b, KernelReport* report) {
  if (coeffs.empty()) throw std::invalid_argument("polyeval: no coefficients");
  if (basis == PolyBasis::Chebyshev && !(b > a)) throw std::invalid_argument("polyeval: empty interval");
  const int depth = polyeval_depth(coeffs.size(), basis);
  if (x.level < depth) throw LevelUnderflowError("polyeval: insufficient level");
  const auto snap = TraceSnapshot::take(ops.trace());
  Ciphertext v = x;
  if (basis == PolyBasis::Chebyshev) {  // y = alpha x + beta at level L - 1, scale Delta
    const double alpha = 2.0 / (b - a), beta = -(a + b) / (b - a);
    const Scale s = ops.params().delta() * Scale::prime(ops.modulus_at(x.level)) / x.scale;
    v = ops.rescale(ops.mul_plain(x, ops.encode(std::vector<double>(ops.slots(), alpha), x.level, s)));
    if (beta != 0.0) v = ops.add_plain(v, ops.encode(std::vector<double>(ops.slots(), beta), v.level, v.scale));
  }
  PolyCtx P{ops, basis, v, {v}};
  const int out_level = v.level - polyeval_depth(coeffs.size(), PolyBasis::Power);
  Ciphertext out = P.eval(coeffs, out_level, ops.params().delta());
  if (report) *report = report_since(ops.trace(), snap, x.level, out);
  return out;
}

// ------------------------------------------------------------------- keys
std::vector<std::int64_t> bsgs_rotations(const BsgsPlan& plan) {
  std::vector<std::int64_t> r;
  for (int k = 1; k < plan.n1; ++k) r.push_back(k);
  for (int j = 1; j < plan.n2; ++j) r.push_back((std::int64_t)plan.n1 * j);
  return r;
}
std::vector<std::int64_t> diag_rotations(int d) {
  std::vector<std::int64_t> r;
  for (int i = 1; i < d; ++i) r.push_back(i);
  return r;
}
std::vector<std::int64_t> row_rotations(const PackedMatrix& M) {
  std::vector<std::int64_t> r;
  for (int s = 1; s < M.pad_cols; s <<= 1) r.push_back(s);
  const int p = M.rows_per_payload;
  for (int row = 0; row < M.rows; ++row) {
    const std::int64_t shift = (std::int64_t)(row % p) * M.pad_cols - row;
    if (shift) r.push_back(shift);
  }
  return r;
}
std::vector<std::int64_t> matmul_rotations(int d, std::size_t) {
  std::vector<std::int64_t> r;
  for (int s = 1; s < d; s <<= 1) {
    r.push_back(-s);
    r.push_back(-(std::int64_t)d * s);
  }
  for (int j = 1; j < d; ++j) {
    r.push_back(j);
    r.push_back((std::int64_t)d * j);
  }
  return r;
}

}  // namespace helix
