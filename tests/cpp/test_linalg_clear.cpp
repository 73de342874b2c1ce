// test_linalg_clear.cpp -- SPEC acceptance tests for the linear-algebra entry
// points (helix/linalg.hpp, helix/packing.hpp) on the REFERENCE's own
// cleartext backend: helix::ReferenceBackend compiled from
// /root/reference/proj/src/reference_backend.cpp against this repository's
// API-compatible headers (Makefile `testbin`; test infrastructure, built only
// where the reference tree is present).  Known answers are the SPEC's own examples
// (acceptance criteria :674-682).  Run by
// tests/test_linalg_cpu.py; exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "helix/linalg.hpp"
#include "helix/reference_backend.hpp"
#include "helix/packing.hpp"

using namespace helix;
using helix::ReferenceBackend;

static int g_checks = 0;
#define CHECK(cond, msg)                                                                  \
  do {                                                                                    \
    ++g_checks;                                                                           \
    if (!(cond)) {                                                                        \
      std::fprintf(stderr, "FAIL %s:%d: %s  [%s]\n", __FILE__, __LINE__, #cond, msg);     \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)

template <class E, class F>
bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static CkksParams params(std::uint64_t N, int L) { return CkksParams::reference_default(N, L); }

static Matrix from_rows(std::vector<std::vector<double>> r) {
  Matrix A((int)r.size(), (int)r[0].size());
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j) A.at(i, j) = r[i][j];
  return A;
}

static Matrix random_matrix(std::mt19937_64& g, int R, int C) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  Matrix A(R, C);
  for (auto& v : A.data) v = u(g);
  return A;
}

static std::vector<double> cleartext(const Matrix& A, const std::vector<double>& x) {
  std::vector<double> y(A.rows, 0.0);
  for (int r = 0; r < A.rows; ++r)
    for (int c = 0; c < A.cols; ++c) y[r] += A.at(r, c) * x[c];
  return y;
}

static double maxdiff(const std::vector<double>& a, const std::vector<double>& b, std::size_t n) {
  double m = 0;
  for (std::size_t i = 0; i < n; ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

// output slot of row r for each method (row: slot r; diag/bsgs: block r/d, slot r%d)
static std::vector<double> matvec_result(ReferenceBackend& be, const MatvecResult& R, const PackedMatrix& M) {
  std::vector<double> y(M.rows);
  if (M.layout == Layout::PackedRow) {
    const auto v = be.decrypt(R.outputs[0]);
    for (int r = 0; r < M.rows; ++r) y[r] = v[r];
  } else {
    for (int r = 0; r < M.rows; ++r) y[r] = be.decrypt(R.outputs[r / M.d])[r % M.d];
  }
  return y;
}

static MatvecResult run(ReferenceBackend& be, const PackedMatrix& M, const std::vector<double>& x, int level) {
  std::vector<std::int64_t> keys = M.layout == Layout::PackedRow ? row_rotations(M)
                                   : M.layout == Layout::Diagonal ? diag_rotations(M.d)
                                                                  : bsgs_rotations(M.plan);
  be.generate_rotation_keys(keys);
  const auto xs = replicate(x, M.d, be.params().slot_count());
  const auto ct = be.encrypt(be.encode(xs, level, be.params().delta()));
  const auto E = encode_matrix(be, M, level);
  return M.layout == Layout::PackedRow ? matvec_row(be, E, ct)
         : M.layout == Layout::Diagonal ? matvec_diag(be, E, ct)
                                        : matvec_bsgs(be, E, ct);
}

// --------------------------------------------------------------- counting backend
// payload-free SlotBackend (bookkeeping + trace only) for the Llama-scale
// rotation-count comparison ("counters only, no lattice ops").
class CountingBackend final : public SlotBackend {
 public:
  explicit CountingBackend(CkksParams p) : p_(std::move(p)) {}
  const CkksParams& params() const override { return p_; }
  OpTrace& trace() override { return t_; }
  const RotationKeySet& rotation_keys() const override { return k_; }
  void generate_rotation_keys(std::span<const std::int64_t> a) override {
    for (auto v : a) k_.insert(detail::reduce_amount(v, (std::int64_t)slots()));
  }
  Plaintext encode(std::span<const double>, int level, const Scale& s) override {
    Plaintext pt;
    pt.payload = std::make_shared<PlaintextPayload>();
    pt.level = level;
    pt.scale = s;
    return pt;
  }
  std::vector<double> decode(const Plaintext&) override { return {}; }
  Ciphertext encrypt(const Plaintext& pt) override { return mk(pt.level, pt.scale); }
  std::vector<double> decrypt(const Ciphertext&) override { return {}; }
  Ciphertext add(const Ciphertext& a, const Ciphertext& b) override {
    detail::require_same_level(a.level, b.level, "add");
    detail::require_same_scale(a.scale, b.scale, "add");
    t_.record(OpKind::CtAdd, a.level);
    return mk(a.level, a.scale);
  }
  Ciphertext add_plain(const Ciphertext& a, const Plaintext&) override {
    t_.record(OpKind::PtAdd, a.level);
    return mk(a.level, a.scale);
  }
  Ciphertext mul(const Ciphertext& a, const Ciphertext& b) override {
    t_.record(OpKind::CtMul, a.level);
    return mk(a.level, a.scale * b.scale);
  }
  Ciphertext mul_plain(const Ciphertext& a, const Plaintext& b) override {
    detail::require_same_level(a.level, b.level, "mul_plain");
    t_.record(OpKind::PtMul, a.level);
    return mk(a.level, a.scale * b.scale);
  }
  Ciphertext rotate(const Ciphertext& a, std::int64_t k) override {
    const auto r = detail::reduce_amount(k, (std::int64_t)slots());
    if (r == 0) return mk(a.level, a.scale);
    if (!k_.contains(r)) throw MissingRotationKeyError("missing key");
    t_.record(OpKind::Rotate, a.level);
    return mk(a.level, a.scale);
  }
  Ciphertext rescale(const Ciphertext& a) override {
    t_.record(OpKind::Rescale, a.level);
    return mk(a.level - 1, a.scale / Scale::prime(modulus_at(a.level)));
  }
  Ciphertext mod_down(const Ciphertext& a, int l) override { return mk(l, a.scale); }
  Ciphertext bootstrap(const Ciphertext& a) override { return mk(p_.l_boot(), p_.delta()); }

 private:
  Ciphertext mk(int level, Scale s) {
    Ciphertext c;
    c.payload = std::make_shared<CiphertextPayload>();
    c.level = level;
    c.scale = std::move(s);
    c.slot_count = slots();
    return c;
  }
  CkksParams p_;
  OpTrace t_;
  RotationKeySet k_;
};

// dims-only EncodedMatrix (dense) for the counting backend
static EncodedMatrix shape_only(SlotOps& ops, Layout layout, int rows, int cols, int level) {
  EncodedMatrix E;
  E.level = level;
  PackedMatrix& M = E.meta;
  M.layout = layout;
  M.rows = rows;
  M.cols = cols;
  M.slots = ops.slots();
  const Scale s = Scale::prime(ops.modulus_at(level));
  Plaintext dense = ops.encode({}, level, s);
  if (layout == Layout::PackedRow) {
    M.pad_cols = M.d = next_pow2(cols);
    M.rows_per_payload = std::min((int)(M.slots / M.pad_cols), rows);
    const int groups = (rows + M.rows_per_payload - 1) / M.rows_per_payload;
    E.pts.assign(groups, dense);
  } else {
    M.d = M.pad_cols = next_pow2(cols);
    M.row_blocks = (rows + M.d - 1) / M.d;
    M.plan = BsgsPlan::for_dim(M.d);
    E.pts.assign((std::size_t)M.row_blocks * M.d, dense);
  }
  return E;
}

static std::uint64_t count_rotations(Layout layout, int rows, int cols) {
  CountingBackend be(params(1ull << 16, 4));
  EncodedMatrix E = shape_only(be, layout, rows, cols, 3);
  be.generate_rotation_keys(layout == Layout::PackedRow ? row_rotations(E.meta) : bsgs_rotations(E.meta.plan));
  const auto x = be.encrypt(be.encode({}, 3, be.params().delta()));
  const auto r = layout == Layout::PackedRow ? matvec_row(be, E, x) : matvec_bsgs(be, E, x);
  return r.report.rotations;
}

int main() {
  const double tol = 1e-9;
  // ---------------------------------------------------------- slot API
  {
    ReferenceBackend be(params(8, 3));  // n = 4
    be.generate_rotation_keys(std::vector<std::int64_t>{1});
    const std::vector<double> v{1, 2, 3, 4};
    const auto r = be.decrypt(be.rotate(be.encrypt(be.encode(v, 3, be.params().delta())), 1));
    CHECK((r == std::vector<double>{2, 3, 4, 1}), "Rot([1,2,3,4],1) = [2,3,4,1] (SPEC.md:86)");
    CHECK(throws<MissingRotationKeyError>([&] { be.rotate(be.encrypt(be.encode(v, 3, be.params().delta())), 2); }),
          "missing rotation key is an error");
  }
  {
    ReferenceBackend be(params(32, 3));  // n = 16
    be.generate_rotation_keys(std::vector<std::int64_t>{3, 5, 8});
    std::vector<double> v(16);
    for (int i = 0; i < 16; ++i) v[i] = i * 1.5 - 3;
    const auto c = be.encrypt(be.encode(v, 3, be.params().delta()));
    CHECK(be.decrypt(be.rotate(be.rotate(c, 3), 5)) == be.decrypt(be.rotate(c, 8)), "Rot o Rot additivity (SPEC.md:88)");
  }
  // ---------------------------------------------------------- packing
  {
    const Matrix A = from_rows({{1, 2, 3, 4}, {5, 6, 7, 8}, {9, 10, 11, 12}, {13, 14, 15, 16}});
    const auto D = pack_diagonals(A, 4);
    CHECK((D.payloads[1] == std::vector<double>{2, 7, 12, 13}), "diag[1] = [2,7,12,13] (SPEC.md:275)");
    const auto B = pack_bsgs(A, BsgsPlan{2, 2}, 4);
    CHECK(B.payloads.size() == 4, "d=4, n1=n2=2 -> 4 payloads (SPEC.md:284)");
    // cost-tuned split (an extension; the SPEC default stays for_dim)
    {
      const BsgsPlan one = BsgsPlan::for_cost(1024, 1), w1 = BsgsPlan::for_cost(1024, 3), w2 = BsgsPlan::for_cost(4096, 1);
      CHECK(one.n1 == 32 && one.n2 == 32, "for_cost: one row block keeps the square split");
      CHECK(w1.n1 == 64 && w1.n2 == 16, "for_cost: 3 row blocks sharing the baby steps -> n1 = 64, n2 = 16");
      CHECK(w2.n1 == 64 && w2.n2 == 64, "for_cost: d = 4096, one block keeps 64 x 64");
      const BsgsPlan tie = BsgsPlan::for_cost(8, 1, 1.0, 1.0), def8 = BsgsPlan::for_dim(8);
      CHECK(tie.n1 == def8.n1 && tie.n2 == def8.n2, "for_cost: ties keep the SPEC default");
      CHECK(BsgsPlan::for_cost(1024, 64, 88.0, 144.0, 64).n1 == 64, "for_cost: n1 capped at max_n1");
      bool threw = false;
      try {
        (void)BsgsPlan::for_cost(12, 1);
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      CHECK(threw, "for_cost: d must be a power of two");
      for (int B2 = 1; B2 <= 8; ++B2) {
        const BsgsPlan p = BsgsPlan::for_cost(256, B2);
        CHECK(p.n1 * p.n2 == 256, "for_cost: n1 n2 = d");
      }
    }
    CHECK(B.payloads[0] == D.payloads[0] && B.payloads[1] == D.payloads[1], "j=0 group = plain diagonals");
    // pre-rotation consistency: rotate stored payload left by n1 j -> plain diagonal
    for (int i = 2; i < 4; ++i) {
      std::vector<double> r(4);
      for (int s = 0; s < 4; ++s) r[s] = B.payloads[i][(s + 2) % 4];
      CHECK(r == D.payloads[i], "BSGS pre-rotation consistency (SPEC.md:281)");
    }
    Matrix I(4, 4);
    for (int i = 0; i < 4; ++i) I.at(i, i) = 1;
    const auto DI = pack_diagonals(I, 4);
    CHECK(DI.nonzero_payloads() == 1 && DI.payloads[0] == std::vector<double>(4, 1.0), "identity diagonals");
    const auto R1 = pack_rows(A, 4);
    CHECK(R1.rows_per_payload == 1 && R1.payloads.size() == 4, "4x4, n=4 -> 4 packed-row payloads (SPEC.md:293)");
    const auto R2 = pack_rows(from_rows({{1, 2}, {3, 4}}), 8);
    CHECK(R2.payloads.size() == 1 && (R2.payloads[0] == std::vector<double>{1, 2, 3, 4, 0, 0, 0, 0}), "2x2, n=8 packed rows");
    const auto RM = pack_rowmajor(from_rows({{1, 2}, {3, 4}}), 8);
    CHECK((RM.payloads[0] == std::vector<double>{1, 2, 3, 4, 0, 0, 0, 0}), "row-major packing");
    CHECK(throws<std::invalid_argument>([&] { pack_rowmajor(Matrix(64, 64), 2048); }), "d^2 > n rejected");
    const auto cm = make_mask(MaskKind::ColumnExtractor, 1, 2, 16);
    CHECK(cm[1] == 1 && cm[3] == 1 && std::count(cm.begin(), cm.end(), 1.0) == 2, "column-extractor(1,2) (SPEC.md:310)");
    const auto rm = make_mask(MaskKind::RowExtractor, 0, 4, 16);
    CHECK(std::count(rm.begin(), rm.begin() + 4, 1.0) == 4 && std::count(rm.begin(), rm.end(), 1.0) == 4, "row-extractor(0,4)");
    std::mt19937_64 g(11);
    for (int trial = 0; trial < 20; ++trial) {
      const int R = 1 + (int)(g() % 16), C = 1 + (int)(g() % 16);
      const Matrix X = random_matrix(g, R, C);
      for (const auto& P : {pack_diagonals(X, 64), pack_bsgs(X, 64), pack_rows(X, 64)}) {
        const Matrix U = unpack(P);
        CHECK(U.data == X.data, "unpack o pack = identity");
      }
    }
    const auto t = tile_matrix(Matrix(768, 3072), 2048, Layout::Diagonal);
    CHECK(t.block == 2048 && t.grid_cols == 2, "tile_matrix 768x3072 at n=2^11 (SPEC.md:319)");
  }
  // ---------------------------------------------------------- rotate_and_sum
  {
    ReferenceBackend be(params(8, 3));
    be.generate_rotation_keys(std::vector<std::int64_t>{1, 2});
    KernelReport rep;
    const auto c = rotate_and_sum(be, be.encrypt(be.encode(std::vector<double>{1, 2, 3, 4}, 3, be.params().delta())), 4, 1, &rep);
    CHECK((be.decrypt(c) == std::vector<double>{10, 10, 10, 10}) && rep.rotations == 2, "rotate_and_sum -> [10,10,10,10], 2 rotations (SPEC.md:365)");
    KernelReport r1;
    rotate_and_sum(be, c, 1, 1, &r1);
    CHECK(r1.rotations == 0, "span 1 -> 0 rotations");
  }
  // ---------------------------------------------------------- stacked-block BSGS
  {
    std::mt19937_64 g(21);
    for (auto [r, c] : std::vector<std::pair<int, int>>{{40, 16}, {64, 32}, {5, 8}, {48, 12}}) {
      ReferenceBackend be(params(1024, 6));
      const Matrix A = random_matrix(g, r, c);
      const PackedMatrix P = pack_bsgs_stacked(A, be.params().slot_count());
      CHECK(unpack(P).data == A.data, "unpack o pack_bsgs_stacked = identity");
      std::vector<double> x(c);
      std::uniform_real_distribution<double> U(-1, 1);
      for (auto& v : x) v = U(g);
      be.generate_rotation_keys(bsgs_rotations(P.plan));
      std::vector<double> xp((std::size_t)P.d, 0.0);
      std::copy(x.begin(), x.end(), xp.begin());
      const auto ct = be.encrypt(be.encode(replicate(xp, P.d, be.params().slot_count()), 5, be.params().delta()));
      const auto R = matvec_bsgs(be, encode_matrix(be, P, 5), ct);
      const auto y = be.decrypt(R.outputs[0]);
      double err = 0;
      for (int i = 0; i < r; ++i) {
        double acc = 0;
        for (int k = 0; k < c; ++k) acc += A.at(i, k) * x[k];
        err = std::max(err, std::abs(y[i] - acc));
      }
      CHECK(R.outputs.size() == 1 && err < 1e-9, "stacked BSGS = cleartext product, one output");
      CHECK((int64_t)R.report.rotations == predicted_rotations(Layout::BsgsStacked, r, c, be.params().slot_count()),
            "stacked BSGS rotations = (n1 - 1) + (n2 - 1)");
    }
  }
  // ---------------------------------------------------------- polyeval
  {
    ReferenceBackend be(params(1024, 8));
    std::mt19937_64 g(11);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::vector<double> xs(be.params().slot_count());
    for (auto& v : xs) v = U(g);
    const auto ct = be.encrypt(be.encode(xs, 8, be.params().delta()));
    std::vector<double> c(8);
    for (auto& v : c) v = U(g);
    KernelReport rep;
    const auto out = polyeval(be, ct, c, PolyBasis::Power, -1, 1, &rep);
    const auto y = be.decrypt(out);
    double err = 0;
    for (std::size_t i = 0; i < xs.size(); ++i) {
      double h = 0;
      for (int k = 7; k >= 0; --k) h = h * xs[i] + c[k];
      err = std::max(err, std::abs(y[i] - h));
    }
    CHECK(err < 1e-9, "polyeval degree 7 == Horner (SPEC.md:411)");
    CHECK(rep.levels_consumed == 3 && out.scale == be.params().delta(), "polyeval: 3 levels, scale exactly Delta");
    const auto sq = polyeval(be, be.encrypt(be.encode(std::vector<double>{1, 2, 3}, 8, be.params().delta())),
                             std::vector<double>{0, 0, 1}, PolyBasis::Power);
    const auto s3 = be.decrypt(sq);
    CHECK(std::abs(s3[0] - 1) + std::abs(s3[1] - 4) + std::abs(s3[2] - 9) < 1e-9, "x^2 on [1,2,3] -> [1,4,9] (SPEC.md:410)");
    // Chebyshev on [-8, 8]: T_3(y) at y = x / 8
    std::vector<double> ch{0, 0, 0, 1};
    const auto t3 = be.decrypt(polyeval(be, be.encrypt(be.encode(std::vector<double>{4.0}, 8, be.params().delta())), ch,
                                        PolyBasis::Chebyshev, -8, 8, &rep));
    CHECK(std::abs(t3[0] - (4 * 0.125 - 3 * 0.5)) < 1e-9 && rep.levels_consumed == 3, "Chebyshev T_3 + domain map level");
    CHECK(throws<LevelUnderflowError>([&] {
            polyeval(be, be.encrypt(be.encode(xs, 2, be.params().delta())), c, PolyBasis::Power);
          }),
          "polyeval: insufficient level");
  }
  // ---------------------------------------------------------- the 4x4 example
  {
    const Matrix A = from_rows({{1, 2, 3, 4}, {5, 6, 7, 8}, {9, 10, 11, 12}, {13, 14, 15, 16}});
    const std::vector<double> x{1, 2, 3, 4}, want{30, 70, 110, 150};
    for (Layout L : {Layout::PackedRow, Layout::Diagonal, Layout::BsgsDiagonal}) {
      ReferenceBackend be(params(1024, 6));
      const auto P = L == Layout::PackedRow ? pack_rows(A, be.params().slot_count())
                     : L == Layout::Diagonal ? pack_diagonals(A, be.params().slot_count())
                                             : pack_bsgs(A, BsgsPlan{2, 2}, be.params().slot_count());
      const auto R = run(be, P, x, 5);
      CHECK(maxdiff(matvec_result(be, R, P), want, 4) < tol, "4x4 matvec = [30,70,110,150] (SPEC.md:374)");
      CHECK(R.report.output_scale == be.params().delta(), "output scale exactly Delta");
      if (L == Layout::PackedRow) CHECK(R.report.levels_consumed == 2, "row method: 2 levels");
      if (L == Layout::Diagonal) CHECK(R.report.levels_consumed == 1 && R.report.rotations == 3, "diag: 3 rotations, 1 level (SPEC.md:383)");
      if (L == Layout::BsgsDiagonal) CHECK(R.report.levels_consumed == 1 && R.report.rotations == 2 && R.report.pt_muls == 4, "bsgs: 2 rotations, 1 level (SPEC.md:392)");
    }
    // bsgs 16x16 -> 6 rotations
    ReferenceBackend be(params(1024, 6));
    std::mt19937_64 g(3);
    const Matrix M = random_matrix(g, 16, 16);
    const auto R = run(be, pack_bsgs(M, be.params().slot_count()), std::vector<double>(16, 0.5), 4);
    CHECK(R.report.rotations == 6, "bsgs 16x16 -> 6 rotations");
    // 1x1 trivial plan: 0 rotations
    ReferenceBackend b1(params(1024, 6));
    const auto R1 = run(b1, pack_bsgs(from_rows({{3.0}}), b1.slots()), std::vector<double>{2.0}, 4);
    CHECK(R1.report.rotations == 0 && std::abs(b1.decrypt(R1.outputs[0])[0] - 6.0) < tol, "1x1 -> 0 rotations, pure pt-mul");
  }
  // ---------------------------------------------------------- 200 seeded instances
  {
    std::mt19937_64 g(20251211);
    const std::vector<std::pair<int, int>> dims = {{4, 4}, {8, 8}, {16, 16}, {64, 64}, {8, 32}, {32, 8}};
    int inst = 0;
    for (int rep = 0; inst < 200; ++rep)
      for (auto [R, C] : dims) {
        if (inst++ >= 200) break;
        const Matrix A = random_matrix(g, R, C);
        std::vector<double> x(C);
        std::uniform_real_distribution<double> u(-1, 1);
        for (auto& v : x) v = u(g);
        const auto want = cleartext(A, x);
        for (Layout L : {Layout::PackedRow, Layout::Diagonal, Layout::BsgsDiagonal}) {
          ReferenceBackend be(params(2048, 4));
          const auto P = L == Layout::PackedRow ? pack_rows(A, be.params().slot_count())
                         : L == Layout::Diagonal ? pack_diagonals(A, be.params().slot_count())
                                                 : pack_bsgs(A, be.params().slot_count());
          const auto Rr = run(be, P, x, 3);
          CHECK(maxdiff(matvec_result(be, Rr, P), want, R) < tol, "method equivalence vs cleartext (SPEC.md:674)");
          const int lv = L == Layout::PackedRow ? 2 : 1;
          CHECK(Rr.report.levels_consumed == lv, "level consumption row 2 / diag 1 / bsgs 1 (SPEC.md:675)");
          if (L == Layout::BsgsDiagonal) {
            const int blocks = P.row_blocks, n1 = P.plan.n1, n2 = P.plan.n2;
            CHECK(Rr.report.rotations == (std::uint64_t)((n1 - 1) + blocks * (n2 - 1)), "BSGS rotations (n1-1)+(n2-1) per block row");
          }
          if (L == Layout::PackedRow) {
            const std::uint64_t groups = P.payloads.size();
            int lg = 0;
            while ((1 << lg) < P.pad_cols) ++lg;
            CHECK(Rr.report.rotations == groups * lg + (std::uint64_t)(R - 1), "row rotations = groups log2(pc) + R - 1");
          }
        }
      }
  }
  // ---------------------------------------------------------- matmul
  {
    ReferenceBackend be(params(64, 5));  // n = 32
    be.generate_rotation_keys(matmul_rotations(2, be.params().slot_count()));
    const auto A = be.encrypt(be.encode(pack_rowmajor(from_rows({{1, 2}, {3, 4}}), be.params().slot_count()).payloads[0], 5, be.params().delta()));
    const auto B = be.encrypt(be.encode(pack_rowmajor(from_rows({{5, 6}, {7, 8}}), be.params().slot_count()).payloads[0], 5, be.params().delta()));
    const auto [Cm, rep] = matmul_ctct(be, A, B, 2);
    const auto c = be.decrypt(Cm);
    CHECK(maxdiff(c, {19, 22, 43, 50}, 4) < tol, "matmul [[1,2],[3,4]][[5,6],[7,8]] (SPEC.md:401)");
    std::printf("levels %d scale %s\n", rep.levels_consumed, rep.output_scale.str().c_str());
    CHECK(rep.levels_consumed == 2 && rep.output_scale == be.params().delta(), "matmul: 2 levels, scale Delta");
    CHECK(throws<std::invalid_argument>([&] { matmul_ctct(be, A, B, 3); }), "d = 3 rejected");
    CHECK(throws<LevelUnderflowError>([&] { matmul_ctct(be, be.mod_down(A, 1), be.mod_down(B, 1), 2); }), "level < 2 rejected");
  }
  for (int d : {2, 4, 8, 16}) {
    ReferenceBackend be(params(1024, 5));
    be.generate_rotation_keys(matmul_rotations(d, be.params().slot_count()));
    std::mt19937_64 g(d);
    const Matrix A = random_matrix(g, d, d), B = random_matrix(g, d, d), B2 = random_matrix(g, d, d);
    auto enc = [&](const Matrix& M) {
      return be.encrypt(be.encode(pack_rowmajor(M, be.params().slot_count()).payloads[0], 5, be.params().delta()));
    };
    const auto [C, rep] = matmul_ctct(be, enc(A), enc(B), d);
    const int lg = d == 2 ? 1 : d == 4 ? 2 : d == 8 ? 3 : 4;
    CHECK(rep.rotations == (std::uint64_t)(2 * d * (1 + lg) - 2), "matmul rotations 6/22/62/158 (SPEC.md:677)");
    CHECK(rep.pt_muls == (std::uint64_t)(2 * d) && rep.ct_muls == (std::uint64_t)d, "matmul 2d pt-muls, d ct-muls");
    const auto c = be.decrypt(C);
    double err = 0;
    for (int r = 0; r < d; ++r)
      for (int col = 0; col < d; ++col) {
        double s = 0;
        for (int k = 0; k < d; ++k) s += A.at(r, k) * B.at(k, col);
        err = std::max(err, std::abs(s - c[(std::size_t)r * d + col]));
      }
    CHECK(err < tol, "matmul vs cleartext");
    // bilinearity: A (B + B2) = A B + A B2
    Matrix S(d, d);
    for (std::size_t i = 0; i < S.data.size(); ++i) S.data[i] = B.data[i] + B2.data[i];
    const auto c1 = be.decrypt(matmul_ctct(be, enc(A), enc(S), d).first);
    const auto c2 = be.decrypt(be.add(C, matmul_ctct(be, enc(A), enc(B2), d).first));
    CHECK(maxdiff(c1, c2, (std::size_t)d * d) < 1e-9, "matmul bilinearity");
  }
  // ---------------------------------------------------------- row vs BSGS at scale
  {
    // M = W^T for x -> x W (768->3072, 3072->8192, 4096->14336), n = 2^15
    const std::uint64_t gb = count_rotations(Layout::BsgsDiagonal, 3072, 768),
                        gr = count_rotations(Layout::PackedRow, 3072, 768);
    const std::uint64_t pb = count_rotations(Layout::BsgsDiagonal, 8192, 3072),
                        pr = count_rotations(Layout::PackedRow, 8192, 3072);
    const std::uint64_t lb = count_rotations(Layout::BsgsDiagonal, 14336, 4096),
                        lr = count_rotations(Layout::PackedRow, 14336, 4096);
    std::printf("rotations row/bsgs: gpt2 %llu/%llu phi3 %llu/%llu llama %llu/%llu\n", (unsigned long long)gr,
                (unsigned long long)gb, (unsigned long long)pr, (unsigned long long)pb, (unsigned long long)lr,
                (unsigned long long)lb);
    CHECK(gb == 31 + 3 * 31, "GPT-2 W1 BSGS rotations (d=1024, 3 blocks)");
    CHECK(lb * 10 < lr, "Llama BSGS rotations < 10% of row-method rotations (SPEC.md:676)");
    CHECK((double)gr / gb < (double)pr / pb && (double)pr / pb < (double)lr / lb, "ratio monotone GPT-2 -> Phi-3 -> Llama");
  }
  std::printf("test_linalg_clear: %d checks passed\n", g_checks);
  return 0;
}
