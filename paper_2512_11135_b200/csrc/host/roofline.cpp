// roofline.cpp -- cost model, intensity and roofline report (formula sheet in
// include/helix/roofline.hpp).
#include "helix/roofline.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include "json.hpp"

namespace helix {

void MachineProfile::validate() const {
  if (!(peak_gops > 0) || !(bandwidth_gbs > 0))
    throw std::invalid_argument("machine profile: peak_gops and bandwidth_gbs must be positive");
}

MachineProfile MachineProfile::paper_default() { return {48 * 2.4, 100.0, "paper-cpu-48x2.4GHz-100GBps"}; }

MachineProfile MachineProfile::b200_measured() { return {148 * 63.6 * 1.965, 6535.7, "b200-int-issue-hbm3e"}; }

const char* primitive_name(Primitive p) {
  switch (p) {
    case Primitive::Add: return "add";
    case Primitive::Mul: return "mul";
    case Primitive::Rotate: return "rotate";
  }
  return "?";
}

CostModel CostModel::from(const CkksParams& p) {
  CostModel m;
  m.N = p.ring_degree;
  m.L = p.max_level;
  const int a = std::max(1, p.digit_size);
  m.dnum = (p.max_level + 1 + a - 1) / a;
  m.K = std::max<int>(1, (int)p.special_primes.size());
  return m;
}

Cost CostModel::cost(Primitive p, int level) const {
  if (level < 1 || level > L) throw std::invalid_argument("model_cost: level out of range [1, L]");
  constexpr double k_add = 2, k_mul_limb = 4;
  const double n = level + 1.0, NN = (double)N;
  const double k_ntt = 1.5 * std::log2(NN);
  const double ct = 2 * n * NN * 8;
  const double key = 2.0 * dnum * (L + 2) * NN * 8;
  const double ks = n * NN * (3 * k_ntt + k_add + 1);
  switch (p) {
    case Primitive::Add: return {k_add * 2 * n * NN, 3 * ct};
    case Primitive::Rotate: return {ks, 2 * ct + key};
    case Primitive::Mul: return {ks + n * NN * (4 * k_mul_limb + k_add), 3 * ct + key};
  }
  return {};
}

double intensity(double int_ops, double bytes) {
  if (!(bytes > 0)) throw std::invalid_argument("intensity: bytes must be positive");
  return int_ops / bytes;
}

double attainable(double i, const MachineProfile& profile) {
  profile.validate();
  return std::min(profile.peak_gops, i * profile.bandwidth_gbs);
}

Cost measure_trace(const OpTrace& trace, const CostModel& model) {
  Cost total;
  for (const auto& [key, times] : trace.level_histogram()) {
    const auto [kind, level] = key;
    Primitive p;
    switch (kind) {
      case OpKind::CtAdd:
      case OpKind::PtAdd: p = Primitive::Add; break;
      case OpKind::CtMul:
      case OpKind::PtMul: p = Primitive::Mul; break;
      case OpKind::Rotate: p = Primitive::Rotate; break;
      default: continue;
    }
    if (level < 1 || level > model.L) continue;  // level-0 ops are not modelled
    const Cost c = model.cost(p, level);
    total.int_ops += c.int_ops * (double)times;
    total.bytes += c.bytes * (double)times;
  }
  return total;
}

RooflineReport RooflineReport::sweep(const CostModel& model, const MachineProfile& profile, int l0, int l1) {
  profile.validate();
  RooflineReport r;
  r.profile = profile;
  for (Primitive p : {Primitive::Add, Primitive::Mul, Primitive::Rotate})
    for (int l = l0; l <= l1; ++l) {
      const Cost c = model.cost(p, l);
      RooflineRow row;
      row.primitive = primitive_name(p);
      row.level = l;
      row.int_ops = c.int_ops;
      row.bytes = c.bytes;
      row.intensity = intensity(c.int_ops, c.bytes);
      row.attainable_gops = attainable(row.intensity, profile);
      row.memory_bound = row.intensity < profile.ridge_point();
      r.rows.push_back(row);
    }
  return r;
}

namespace {
std::string fmt(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.9g", v);
  return b;
}
}  // namespace

std::string RooflineReport::to_csv() const {
  bool meas = false;
  for (const auto& r : rows) meas |= r.measured_gbs >= 0;
  std::ostringstream o;
  o << "primitive,level,ops,bytes,intensity,attainable,bound" << (meas ? ",measured_gbs" : "") << "\n";
  for (const auto& r : rows) {
    o << r.primitive << ',' << r.level << ',' << fmt(r.int_ops) << ',' << fmt(r.bytes) << ',' << fmt(r.intensity)
      << ',' << fmt(r.attainable_gops) << ',' << (r.memory_bound ? "memory" : "compute");
    if (meas) o << ',' << (r.measured_gbs >= 0 ? fmt(r.measured_gbs) : "");
    o << "\n";
  }
  return o.str();
}

std::string RooflineReport::to_json() const {
  nlohmann::json j;
  j["profile"] = {{"name", profile.name},
                  {"peak_gops", profile.peak_gops},
                  {"bandwidth_gbs", profile.bandwidth_gbs},
                  {"ridge_point", profile.ridge_point()}};
  j["rows"] = nlohmann::json::array();
  for (const auto& r : rows) {
    nlohmann::json e = {{"primitive", r.primitive}, {"level", r.level},           {"ops", r.int_ops},
                        {"bytes", r.bytes},         {"intensity", r.intensity},   {"attainable", r.attainable_gops},
                        {"bound", r.memory_bound ? "memory" : "compute"}};
    if (r.measured_gbs >= 0) e["measured_gbs"] = r.measured_gbs;
    j["rows"].push_back(e);
  }
  return j.dump(2);
}

// log-log plot: x = intensity (ops / byte), y = attainable GOPS
std::string RooflineReport::to_svg() const {
  if (rows.empty()) throw std::invalid_argument("emit_roofline: empty report");
  profile.validate();
  const double W = 720, H = 480, ml = 70, mr = 20, mt = 30, mb = 50;
  double xmin = profile.ridge_point(), xmax = profile.ridge_point();
  for (const auto& r : rows) {
    xmin = std::min(xmin, r.intensity);
    xmax = std::max(xmax, r.intensity);
  }
  const double lx0 = std::floor(std::log10(xmin)) - 0.5, lx1 = std::ceil(std::log10(xmax)) + 0.5;
  const double ly1 = std::ceil(std::log10(profile.peak_gops)) + 0.5;
  const double ly0 = std::floor(std::log10(std::pow(10.0, lx0) * profile.bandwidth_gbs)) - 0.5;
  auto X = [&](double v) { return ml + (std::log10(v) - lx0) / (lx1 - lx0) * (W - ml - mr); };
  auto Y = [&](double v) { return H - mb - (std::log10(v) - ly0) / (ly1 - ly0) * (H - mt - mb); };
  std::ostringstream o;
  o << "<?xml version=\"1.0\" encoding=\"UTF-8\"?>\n"
    << "<svg xmlns=\"http://www.w3.org/2000/svg\" version=\"1.1\" width=\"" << W << "\" height=\"" << H << "\">\n"
    << "<title>Roofline: " << profile.name << "</title>\n"
    << "<rect x=\"0\" y=\"0\" width=\"" << W << "\" height=\"" << H << "\" fill=\"white\"/>\n"
    << "<line x1=\"" << ml << "\" y1=\"" << H - mb << "\" x2=\"" << W - mr << "\" y2=\"" << H - mb
    << "\" stroke=\"black\"/>\n"
    << "<line x1=\"" << ml << "\" y1=\"" << mt << "\" x2=\"" << ml << "\" y2=\"" << H - mb << "\" stroke=\"black\"/>\n";
  // bandwidth slope up to the ridge, then the compute peak
  const double xr = profile.ridge_point(), xa = std::pow(10.0, lx0), xb = std::pow(10.0, lx1);
  o << "<polyline fill=\"none\" stroke=\"#1f4e9c\" stroke-width=\"2\" points=\"" << fmt(X(xa)) << ','
    << fmt(Y(xa * profile.bandwidth_gbs)) << ' ' << fmt(X(xr)) << ',' << fmt(Y(profile.peak_gops)) << ' '
    << fmt(X(xb)) << ',' << fmt(Y(profile.peak_gops)) << "\"/>\n";
  o << "<text x=\"" << fmt(X(xr) + 6) << "\" y=\"" << fmt(Y(profile.peak_gops) - 6)
    << "\" font-size=\"11\">ridge " << fmt(xr) << " ops/B</text>\n";
  for (int e = (int)std::ceil(lx0); e <= (int)std::floor(lx1); ++e)
    o << "<text x=\"" << fmt(X(std::pow(10.0, e))) << "\" y=\"" << H - mb + 16 << "\" font-size=\"10\">1e" << e
      << "</text>\n";
  for (int e = (int)std::ceil(ly0); e <= (int)std::floor(ly1); ++e)
    o << "<text x=\"4\" y=\"" << fmt(Y(std::pow(10.0, e))) << "\" font-size=\"10\">1e" << e << "</text>\n";
  o << "<text x=\"" << W / 2 - 80 << "\" y=\"" << H - 8 << "\" font-size=\"12\">intensity (int ops / DRAM byte)</text>\n"
    << "<text x=\"14\" y=\"" << mt - 10 << "\" font-size=\"12\">attainable GOPS</text>\n";
  const char* colour[3] = {"#2a9d2a", "#c0392b", "#8e44ad"};
  for (const auto& r : rows) {
    const int ci = r.primitive == "add" ? 0 : r.primitive == "mul" ? 1 : 2;
    o << "<circle cx=\"" << fmt(X(r.intensity)) << "\" cy=\"" << fmt(Y(r.attainable_gops)) << "\" r=\"3\" fill=\""
      << colour[ci] << "\"><title>" << r.primitive << " l=" << r.level << "</title></circle>\n";
  }
  for (int ci = 0; ci < 3; ++ci)
    o << "<text x=\"" << W - 120 << "\" y=\"" << mt + 14 * (ci + 1) << "\" font-size=\"11\" fill=\"" << colour[ci]
      << "\">" << (ci == 0 ? "add" : ci == 1 ? "mul" : "rotate") << "</text>\n";
  o << "</svg>\n";
  return o.str();
}

}  // namespace helix
