// test_gpu_api.cpp -- a REFERENCE-STYLE caller compiled unchanged against this
// repository's include/helix and linked with libhelix_b200.so (the B200
// backend).  It uses only the reference's public API shapes:
//   CkksParams fields / find_ntt_primes          params.hpp:19-51, modmath.hpp:138-152
//   LatticeContext / RnsPoly ring layer          rns_poly.hpp:21-99
//   NttTables / schoolbook_negacyclic_mul        ntt.hpp:19-52
//   CkksEncoder(const LatticeContext&) encode/decode  encoder.hpp:22-38
//   SlotBackend (GpuLatticeBackend) + SPEC matvec_bsgs / matmul_ctct
//                                                backend.hpp:86-139
// and checks the reference's own known answers.  Run on a B200 by
// tests/test_gpu_cpp_api.py (pytest -m gpu); exits non-zero on the first
// failure.  Build: make testgpu.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "helix/encoder.hpp"
#include "helix/gpu_backend.hpp"
#include "helix/linalg.hpp"
#include "helix/modmath.hpp"
#include "helix/ntt.hpp"
#include "helix/packing.hpp"
#include "helix/params.hpp"
#include "helix/rns_poly.hpp"

using namespace helix;

static int g_checks = 0;
#define CHECK(cond, msg)                                                              \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s  [%s]\n", __FILE__, __LINE__, #cond, msg); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

template <class E, class F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// config 1's parameter shape, written the way a reference caller fills CkksParams
static CkksParams lattice_params(std::uint64_t N, int L) {
  CkksParams p;
  p.ring_degree = N;
  p.max_level = L;
  p.delta_log2 = 40;
  p.moduli = find_ntt_primes(std::uint64_t(1) << 39, (std::size_t)L + 1, 2 * N);
  p.special_primes = find_ntt_primes(std::uint64_t(1) << 49, 1, 2 * N);
  p.backend = BackendKind::Lattice;
  p.insecure_toy = true;
  return p;
}

static void test_modmath_and_ntt() {
  // SPEC.md:172-174 ring known answers through NttTables / LatticeContext
  const std::uint64_t N = 256;
  const auto qs = find_ntt_primes(std::uint64_t(1) << 39, 1, 2 * N);
  Modulus m(qs[0]);
  CHECK(m.mul(m.q - 1, m.q - 1) == 1, "(-1)^2 = 1 with 128-bit products");
  CHECK(m.mul(m.inv(12345), 12345) == 1, "inverse");
  NttTables t(m, N);
  CHECK(t.psi() == find_psi(m, N) && m.pow(t.psi(), 2 * N) == 1 && m.pow(t.psi(), N) == m.q - 1, "psi order 2N");
  std::mt19937_64 rng(7);
  std::uniform_int_distribution<std::uint64_t> u(0, m.q - 1);
  std::vector<std::uint64_t> a(N), b(N);
  for (auto& x : a) x = u(rng);
  for (auto& x : b) x = u(rng);
  auto fa = a;
  t.forward(fa);
  auto back = fa;
  t.inverse(back);
  CHECK(back == a, "inverse(forward(a)) == a on the device");
  // forward leaves the bit-reversed evaluation layout: out[k] = a(psi^(2 brv(k) + 1))
  auto eval = [&](std::uint64_t x) {
    std::uint64_t r = 0;
    for (std::size_t i = N; i-- > 0;) r = m.add(m.mul(r, x), a[i]);
    return r;
  };
  for (std::size_t k : {0ul, 1ul, 77ul, 255ul}) {
    std::size_t br = 0;
    for (int i = 0; i < 8; ++i) br |= ((k >> i) & 1) << (7 - i);
    CHECK(fa[k] == eval(m.pow(t.psi(), 2 * br + 1)), "NTT layout = reference forward()");
  }
  CHECK(t.negacyclic_mul(a, b) == schoolbook_negacyclic_mul(a, b, m), "NTT product == schoolbook");
  std::vector<std::uint64_t> x(N, 0), xn1(N, 0);
  x[1] = 1;
  xn1[N - 1] = 1;
  const auto r = t.negacyclic_mul(x, xn1);
  CHECK(r[0] == m.q - 1, "X * X^(N-1) = -1");
  CHECK(throws<std::invalid_argument>([&] { t.forward(std::span<std::uint64_t>(a.data(), N - 1)); }), "length");
}

static void test_lattice_context() {
  const CkksParams p = lattice_params(1 << 13, 2);
  LatticeContext ctx(p);
  CkksEncoder enc(ctx);
  const std::size_t n = enc.slot_count();
  std::vector<double> m(n);
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> ud(-1.0, 1.0);
  for (auto& v : m) v = ud(rng);
  const double delta = std::ldexp(1.0, 40);
  // SPEC.md:182 round trip < 1e-4 (encode -> RNS limbs -> decode)
  RnsPoly pt = enc.encode(m, 2, delta);
  CHECK(pt.domain == PolyDomain::Coeff && pt.chain_limbs() == 3 && !pt.has_special, "encode shape");
  auto back = enc.decode(pt, delta);
  double err = 0;
  for (std::size_t j = 0; j < n; ++j) err = std::max(err, std::abs(back[j] - m[j]));
  CHECK(err < 1e-4, "encode/decode round trip");
  // NTT round trip through the context
  RnsPoly f = pt;
  ctx.to_ntt(f);
  CHECK(f.domain == PolyDomain::Ntt, "to_ntt domain");
  ctx.to_coeff(f);
  CHECK(f.limbs == pt.limbs, "to_coeff(to_ntt(p)) == p");
  // automorphism X -> X^(5^k) rotates slots left by k (encoder.cpp:19-24 slot order)
  const std::uint64_t g = 5ull * 5ull * 5ull % (2 * p.ring_degree);
  auto rot = enc.decode(ctx.automorphism(pt, g), delta);
  err = 0;
  for (std::size_t j = 0; j < n; ++j) err = std::max(err, std::abs(rot[j] - m[(j + 3) % n]));
  CHECK(err < 1e-4, "automorphism(5^3) = left rotation by 3");
  RnsPoly fn = pt;
  ctx.to_ntt(fn);
  CHECK(throws<std::invalid_argument>([&] { ctx.automorphism(fn, g); }), "automorphism needs the coefficient domain");
  // ring_mul of two encodings = slot-wise product at scale^2; rescale drops one limb
  RnsPoly pt2 = enc.encode(m, 2, static_cast<double>(p.moduli[2]));
  RnsPoly prod = ctx.ring_mul(pt, pt2);
  RnsPoly rs = ctx.rescale_drop_last(prod);
  CHECK(rs.chain_limbs() == 2, "rescale drops a limb");
  auto sq = enc.decode(rs, delta);
  err = 0;
  for (std::size_t j = 0; j < n; ++j) err = std::max(err, std::abs(sq[j] - m[j] * m[j]));
  CHECK(err < 1e-4, "rescale(ring_mul) = slot-wise product");
  // add / sub / negate / mul / mul_acc agree with each other
  RnsPoly a = ctx.sample_uniform(3, false, PolyDomain::Ntt, rng), b = ctx.sample_uniform(3, false, PolyDomain::Ntt, rng);
  RnsPoly s = ctx.add(a, b), d = ctx.sub(s, b);
  CHECK(d.limbs == a.limbs, "(a + b) - b == a");
  CHECK(ctx.add(a, ctx.negate(a)).limbs == ctx.zero(3, false, PolyDomain::Ntt).limbs, "a + (-a) == 0");
  RnsPoly acc = ctx.zero(3, false, PolyDomain::Ntt);
  ctx.mul_acc(a, b, acc);
  CHECK(acc.limbs == ctx.mul(a, b).limbs, "mul_acc into zero == mul");
  // moddown_special divides by the special prime (rns_poly.cpp:164-180)
  RnsPoly big = ctx.from_i64(std::vector<std::int64_t>(p.ring_degree, 0), 3, true);
  const std::uint64_t P = p.special_primes[0];
  for (std::size_t i = 0; i < 3; ++i) big.limbs[i][5] = ctx.chain_modulus((int)i).mul(P % p.moduli[i], 1000);
  big.limbs[3][5] = 0;
  RnsPoly md = ctx.moddown_special(big);
  CHECK(md.limbs[0][5] == 1000 && md.limbs[2][5] == 1000 && md.limbs[1][4] == 0, "P * 1000 / P == 1000");
  CHECK(throws<std::invalid_argument>([&] { ctx.rescale_drop_last(big); }), "rescale rejects the special limb");
  CHECK(ctx.drop_to_level(pt, 0).chain_limbs() == 1, "drop_to_level");
}

static void test_backend_matvec_and_matmul() {
  CkksParams p = lattice_params(1 << 13, 2);
  p.digit_size = 1;
  GpuLatticeBackend be(p, 42);
  SlotOps& ops = be;
  const std::size_t n = be.slots();
  std::mt19937_64 rng(20251211ull * 10 + 1);
  std::uniform_real_distribution<double> ud(-1.0, 1.0);
  // BASELINE configs[0]: 64 x 64 BSGS matvec: 14 rotations, 1 level
  Matrix A(64, 64);
  for (auto& v : A.data) v = ud(rng);
  std::vector<double> x(64);
  for (auto& v : x) v = ud(rng);
  const BsgsPlan plan = BsgsPlan::for_dim(64);
  const PackedMatrix M = pack_bsgs(A, plan, n);
  be.generate_rotation_keys(bsgs_rotations(plan));
  const Ciphertext ct = be.encrypt(be.encode(replicate(x, 64, n), p.max_level, p.delta()));
  auto [y, rep] = matvec_bsgs(ops, M, ct, plan);
  CHECK(rep.rotations == 14 && rep.levels_consumed == 1 && rep.pt_muls == 64, "BSGS counts");
  CHECK(y.scale == p.delta(), "output scale exactly Delta");
  const auto yv = be.decrypt(y);
  double err = 0;
  for (int r = 0; r < 64; ++r) {
    double acc = 0;
    for (int c = 0; c < 64; ++c) acc += A.at(r, c) * x[c];
    err = std::max(err, std::abs(yv[r] - acc));
  }
  CHECK(err < 1e-4, "BSGS matvec value");
  // SPEC.md:401 matmul known answer [[1,2],[3,4]] [[5,6],[7,8]] = [[19,22],[43,50]], 6 rotations
  be.generate_rotation_keys(matmul_rotations(2, n));
  const Ciphertext a = be.encrypt(be.encode(std::vector<double>{1, 2, 3, 4}, p.max_level, p.delta()));
  const Ciphertext b = be.encrypt(be.encode(std::vector<double>{5, 6, 7, 8}, p.max_level, p.delta()));
  auto [c, mrep] = matmul_ctct(ops, a, b, 2);
  const auto cv = be.decrypt(c);
  const double exp[4] = {19, 22, 43, 50};
  for (int i = 0; i < 4; ++i) CHECK(std::abs(cv[i] - exp[i]) < 1e-3, "matmul known answer");
  CHECK(mrep.rotations == 6 && mrep.levels_consumed == 2, "matmul counts (SPEC.md:403)");
  // errors map to the reference's exception types (backend.hpp:66-81)
  CHECK(throws<MissingRotationKeyError>([&] { be.rotate(ct, 9); }), "missing key (9 is in neither key set)");
  CHECK(throws<LevelMismatchError>([&] { be.add(ct, be.mod_down(ct, 0)); }), "level mismatch");
}

int main() {
  try {
    test_modmath_and_ntt();
    test_lattice_context();
    test_backend_matvec_and_matmul();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAIL: uncaught %s\n", e.what());
    return 1;
  }
  std::printf("test_gpu_api: %d checks passed\n", g_checks);
  return 0;
}
