// cli.cpp -- `helix`, the command-line entry point of SPEC.md:600-669
// (module bench-cli; the reference's tools/ directory is listed in
// proj/CMakeLists.txt:32 but absent) over the B200 backend.
//
//   helix roofline [--profile paper|b200] [--peak-gops G --bandwidth-gbs B]
//                  [--params file] [--levels l0:l1] [--csv path] [--svg path] [--json]
//   helix matvec --method row|diag|bsgs --rows R --cols C [--seed S] [--repeats K]
//                [--params file] [--json] [--csv path]
//   helix matvec --preset gpt2|phi3|llama          (rotation counters only, no ciphertexts)
//   helix matmul --d D [--level L] [--seed S] [--repeats K] [--params file] [--json] [--csv path]
//
// Backend: `lattice` (GpuLatticeBackend on the B200, the default; insecure toy
// parameters CkksParams::toy_lattice() unless --params / HELIX_PARAMS).
// `--backend reference` is the reference's cleartext backend, not part of this
// build (exit 2).  Exit codes: 0 success, 1 correctness
// failure, 2 usage error.  Every table is also printed as JSON with --json.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"

#include "helix/gpu_backend.hpp"
#include "helix/linalg.hpp"
#include "helix/packing.hpp"
#include "helix/params.hpp"
#include "helix/roofline.hpp"

using namespace helix;
using json = nlohmann::json;

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  long num(const std::string& k, long d) const {
    if (!has(k)) return d;
    char* end = nullptr;
    const long v = std::strtol(get(k).c_str(), &end, 10);
    if (!end || *end) throw Usage("--" + k + " expects an integer");
    return v;
  }
  double real(const std::string& k, double d) const {
    if (!has(k)) return d;
    char* end = nullptr;
    const double v = std::strtod(get(k).c_str(), &end);
    if (!end || *end) throw Usage("--" + k + " expects a number");
    return v;
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw Usage("missing subcommand");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw Usage("unexpected argument " + s);
    s = s.substr(2);
    const bool flag = s == "json";
    if (flag) {
      a.kv[s] = "1";
    } else {
      if (i + 1 >= argc) throw Usage("--" + s + " needs a value");
      a.kv[s] = argv[++i];
    }
  }
  return a;
}

CkksParams load_params(const Args& a) {
  std::string path = a.get("params");
  if (path.empty() && std::getenv("HELIX_PARAMS")) path = std::getenv("HELIX_PARAMS");
  CkksParams p = path.empty() ? CkksParams::toy_lattice() : CkksParams::load(path);
  return p;
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write " + path);
  f << text;
}

void check_backend(const Args& a) {
  const std::string b = a.get("backend", "lattice");
  if (b == "reference") throw Usage("--backend reference: the reference's cleartext backend is not part of this build");
  if (b != "lattice") throw Usage("unknown backend " + b);
}

// ------------------------------------------------------------------ roofline
int cmd_roofline(const Args& a) {
  MachineProfile prof =
      a.get("profile", "paper") == "b200" ? MachineProfile::b200_measured() : MachineProfile::paper_default();
  if (a.get("profile", "paper") != "paper" && a.get("profile") != "b200") throw Usage("unknown profile");
  if (a.has("peak-gops") || a.has("bandwidth-gbs")) {
    prof.peak_gops = a.real("peak-gops", prof.peak_gops);
    prof.bandwidth_gbs = a.real("bandwidth-gbs", prof.bandwidth_gbs);
    prof.name = "custom";
  }
  try {
    prof.validate();
  } catch (const std::invalid_argument& e) {
    throw Usage(e.what());
  }
  // N = 2^16, l = 1..20 on the reference default parameter shape
  CostModel model;
  if (a.has("params")) model = CostModel::from(load_params(a));
  int l0 = 1, l1 = std::min(20, model.L);
  if (a.has("levels")) {
    const std::string s = a.get("levels");
    const auto c = s.find(':');
    if (c == std::string::npos) throw Usage("--levels l0:l1");
    l0 = std::atoi(s.substr(0, c).c_str());
    l1 = std::atoi(s.substr(c + 1).c_str());
  }
  if (l0 < 1 || l1 > model.L || l0 > l1) throw Usage("--levels outside [1, L]");
  const RooflineReport rep = RooflineReport::sweep(model, prof, l0, l1);
  if (a.has("csv")) write_file(a.get("csv"), rep.to_csv());
  if (a.has("svg")) write_file(a.get("svg"), rep.to_svg());
  if (a.has("json")) {
    std::printf("%s\n", rep.to_json().c_str());
  } else {
    std::printf("profile %s: peak %.1f GOPS, %.1f GB/s, ridge %.4f ops/B\n", prof.name.c_str(), prof.peak_gops,
                prof.bandwidth_gbs, prof.ridge_point());
    std::printf("%-8s %5s %14s %14s %10s %12s %s\n", "prim", "level", "int_ops", "bytes", "ops/B", "attain", "bound");
    for (const auto& r : rep.rows)
      std::printf("%-8s %5d %14.4g %14.4g %10.5f %12.4g %s\n", r.primitive.c_str(), r.level, r.int_ops, r.bytes,
                  r.intensity, r.attainable_gops, r.memory_bound ? "memory" : "compute");
  }
  return 0;
}

// ------------------------------------------------------------------ matvec / matmul
json report_json(const KernelReport& r) { return json::parse(r.to_json()); }

int emit(const Args& a, const json& table) {
  if (a.has("csv")) {
    std::ostringstream o;
    const auto& rows = table["rows"];
    if (!rows.empty()) {
      bool first = true;
      for (auto it = rows[0].begin(); it != rows[0].end(); ++it) {
        o << (first ? "" : ",") << it.key();
        first = false;
      }
      o << "\n";
      for (const auto& r : rows) {
        first = true;
        for (auto it = r.begin(); it != r.end(); ++it) {
          o << (first ? "" : ",") << (it->is_string() ? it->get<std::string>() : it->dump());
          first = false;
        }
        o << "\n";
      }
    }
    write_file(a.get("csv"), o.str());
  }
  if (a.has("json")) {
    std::printf("%s\n", table.dump(2).c_str());
  } else {
    for (const auto& r : table["rows"]) {
      std::ostringstream o;
      for (auto it = r.begin(); it != r.end(); ++it)
        o << it.key() << "=" << (it->is_string() ? it->get<std::string>() : it->dump()) << "  ";
      std::printf("%s\n", o.str().c_str());
    }
  }
  bool ok = true;
  for (const auto& r : table["rows"])
    if (r.contains("correct")) ok = ok && r["correct"].get<bool>();
  return ok ? 0 : 1;
}

// SPEC.md:614 model presets (attention-free FFN up-projections; counters only)
int matvec_presets(const Args& a) {
  struct P {
    const char* name;
    int rows, cols;
  };
  const P presets[] = {{"gpt2", 3072, 768}, {"phi3", 8192, 3072}, {"llama", 14336, 4096}};
  const std::string want = a.get("preset");
  const std::size_t slots = 1u << 15;
  json t;
  t["rows"] = json::array();
  bool found = false;
  for (const auto& p : presets) {
    if (want != "all" && want != p.name) continue;
    found = true;
    const auto row = predicted_rotations(Layout::PackedRow, p.rows, p.cols, slots);
    const auto bsgs = predicted_rotations(Layout::BsgsDiagonal, p.rows, p.cols, slots);
    t["rows"].push_back({{"preset", p.name},
                         {"rows", p.rows},
                         {"cols", p.cols},
                         {"row_rotations", row},
                         {"bsgs_rotations", bsgs},
                         {"ratio", (double)bsgs / (double)row}});
  }
  if (!found) throw Usage("unknown preset " + want);
  return emit(a, t);
}

int cmd_matvec(const Args& a) {
  if (a.has("preset")) return matvec_presets(a);
  check_backend(a);
  const std::string method = a.get("method", "bsgs");
  if (method != "row" && method != "diag" && method != "bsgs") throw Usage("--method row|diag|bsgs");
  const int R = (int)a.num("rows", 16), Cc = (int)a.num("cols", 16);
  const int repeats = (int)a.num("repeats", 3);
  if (R < 1 || Cc < 1 || repeats < 1) throw Usage("--rows, --cols, --repeats >= 1");
  const CkksParams p = load_params(a);
  GpuLatticeBackend be(p, (std::uint64_t)a.num("seed", 1));
  SlotOps& ops = be;
  const std::size_t n = be.slots();
  std::mt19937_64 rng((std::uint64_t)a.num("seed", 1));
  std::uniform_real_distribution<double> ud(-1.0, 1.0);
  Matrix A(R, Cc);
  for (auto& v : A.data) v = ud(rng);
  std::vector<double> x(Cc);
  for (auto& v : x) v = ud(rng);
  PackedMatrix M;
  std::vector<std::int64_t> rots;
  BsgsPlan plan;
  if (method == "bsgs") {
    M = pack_bsgs(A, n);
    plan = M.plan;
    rots = bsgs_rotations(plan);
  } else if (method == "diag") {
    M = pack_diagonals(A, n);
    rots = diag_rotations(M.d);
  } else {
    M = pack_rows(A, n);
    rots = row_rotations(M);
  }
  be.generate_rotation_keys(rots);
  const int d = method == "row" ? M.pad_cols : M.d;
  const Ciphertext ct = be.encrypt(be.encode(replicate(x, d, n), p.max_level, p.delta()));
  const EncodedMatrix E = encode_matrix(ops, M, p.max_level);
  double secs = 0;
  MatvecResult res;
  for (int r = 0; r < repeats; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    res = method == "bsgs" ? matvec_bsgs(ops, E, ct) : method == "diag" ? matvec_diag(ops, E, ct) : matvec_row(ops, E, ct);
    const auto yv = be.decrypt(res.outputs[0]);  // includes the device work
    secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  // y = A x vs the cleartext product; lattice tolerance 1e-2
  double err = 0;
  const int blk = M.d > 0 ? M.d : R;
  for (int r = 0; r < R; ++r) {
    double acc = 0;
    for (int c = 0; c < Cc; ++c) acc += A.at(r, c) * x[c];
    const auto& out = res.outputs[method == "row" ? 0 : std::min<std::size_t>(r / blk, res.outputs.size() - 1)];
    const auto yv = be.decrypt(out);
    const double got = yv[method == "row" ? r : r % blk];
    err = std::max(err, std::abs(got - acc));
  }
  json t;
  json row = {{"method", method}, {"rows", R}, {"cols", Cc}, {"backend", "lattice"},
              {"correct", err < 1e-2}, {"max_abs_err", err}, {"seconds_mean", secs / repeats}};
  const json rep = report_json(res.report);
  for (auto it = rep.begin(); it != rep.end(); ++it) row[it.key()] = it.value();
  t["rows"] = json::array({row});
  return emit(a, t);
}

int cmd_matmul(const Args& a) {
  check_backend(a);
  const int d = (int)a.num("d", 4);
  if (d < 1 || (d & (d - 1))) throw Usage("--d must be a power of two");
  const CkksParams p = load_params(a);
  const int level = (int)a.num("level", p.max_level);
  if (level < 2) throw Usage("matmul requires a multiplicative level of 2");
  if (level > p.max_level) throw Usage("--level above the parameter set's top level");
  const int repeats = (int)a.num("repeats", 3);
  GpuLatticeBackend be(p, (std::uint64_t)a.num("seed", 1));
  SlotOps& ops = be;
  const std::size_t n = be.slots();
  if ((std::size_t)d * d > n) throw Usage("d^2 must not exceed the slot count");
  std::mt19937_64 rng((std::uint64_t)a.num("seed", 1));
  std::uniform_real_distribution<double> ud(-1.0, 1.0);
  std::vector<double> Av((std::size_t)d * d), Bv((std::size_t)d * d);
  for (auto& v : Av) v = ud(rng);
  for (auto& v : Bv) v = ud(rng);
  be.generate_rotation_keys(matmul_rotations(d, n));
  const Ciphertext A = be.encrypt(be.encode(Av, level, p.delta()));
  const Ciphertext B = be.encrypt(be.encode(Bv, level, p.delta()));
  double secs = 0;
  std::pair<Ciphertext, KernelReport> res{A, {}};
  std::vector<double> cv;
  for (int r = 0; r < repeats; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    res = matmul_ctct(ops, A, B, d);
    cv = be.decrypt(res.first);
    secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  double err = 0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double acc = 0;
      for (int k = 0; k < d; ++k) acc += Av[(std::size_t)i * d + k] * Bv[(std::size_t)k * d + j];
      err = std::max(err, std::abs(cv[(std::size_t)i * d + j] - acc));
    }
  // modelled cost of the run's trace (measure_trace)
  const Cost c = measure_trace(be.trace(), CostModel::from(p));
  json row = {{"d", d},       {"level", level},      {"backend", "lattice"},          {"correct", err < 1e-2},
              {"max_abs_err", err}, {"seconds_mean", secs / repeats}, {"modeled_int_ops", c.int_ops},
              {"modeled_bytes", c.bytes}};
  const json rep = report_json(res.second);
  for (auto it = rep.begin(); it != rep.end(); ++it) row[it.key()] = it.value();
  json t;
  t["rows"] = json::array({row});
  return emit(a, t);
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "roofline") return cmd_roofline(a);
    if (a.cmd == "matvec") return cmd_matvec(a);
    if (a.cmd == "matmul") return cmd_matmul(a);
    throw Usage("unknown subcommand " + a.cmd);
  } catch (const Usage& e) {
    std::fprintf(stderr, "helix: %s\nusage: helix roofline|matvec|matmul [--flags] (see cli.cpp header)\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "helix: error: %s\n", e.what());
    return 2;
  }
}
