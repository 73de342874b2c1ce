// helix/roofline.hpp -- analytic cost model of the FHE primitives, arithmetic
// intensity and roofline reports (module `roofline`; the
// reference lists src/roofline.cpp in proj/CMakeLists.txt:27 but does not ship
// it).  Besides the paper's CPU profile the same model is
// evaluated against the B200's measured integer-issue and HBM peaks
// (`helix roofline --profile b200`); a row can carry a measured bandwidth
// beside the model (measured_gbs, CSV column / JSON key when present).
//
// Formula sheet (per call at level l, n = l + 1 active limbs, N ring degree,
// L top level, dnum key digits, K special primes; counts in 64-bit integer
// operations, and DRAM bytes):
//   ct(l)      = 2 n N 8                       (one ciphertext)
//   key        = 2 dnum (L + 2) N 8            (charged in full)
//   k_add = 2, k_mul_limb = 4 ops per coefficient-limb
//   k_ntt = 3 log2(N) / 2 ops per coefficient-limb (N/2 log2 N butterflies of
//           3 ops over the N coefficients of one limb)
//   add:    ops = k_add 2 n N                  bytes = 3 ct
//   rotate: ops = n N (3 k_ntt + k_add + 1)    bytes = 2 ct + key
//           (the key switch per limb: INTT of c1, NTT of the lifted digit,
//            NTT of the ModDown result; the automorphism and the gadget
//            product amortised to one op per limb-word)
//   mul:    ops = rotate + n N (4 k_mul_limb + k_add)   bytes = 3 ct + key
//           (tensor product: 4 limb products and one add, then the
//            relinearisation key switch)
// Invariants (tests/test_roofline_cpu.py): add intensity = 1/12 exactly; all
// counts positive and monotone in l and N; with the paper profile (115.2
// GOPS, 100 GB/s) every primitive at N = 2^16, L = 20, l in [1, 20] is
// memory-bound for dnum >= 2 and lies in [0.02, 0.3] ops/byte for the
// reference parameters (dnum = L + 1); mul within 2x of rotate.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "helix/params.hpp"
#include "helix/trace.hpp"

namespace helix {

// SPEC.md:524-526
struct MachineProfile {
  double peak_gops = 0;      // 1e9 integer ops / s
  double bandwidth_gbs = 0;  // 1e9 bytes / s
  std::string name;

  double ridge_point() const { return peak_gops / bandwidth_gbs; }
  void validate() const;  // std::invalid_argument unless both positive

  // SPEC.md:584 default: 48 threads x 2.4 GHz, 100 GB/s (the paper's CPU)
  static MachineProfile paper_default();
  // B200 (this run's pool): 148 SMs x 63.6 IMAD lanes / clk x 1.965 GHz
  // integer issue, 6535.7 GB/s measured copy bandwidth (MEASURED_PEAKS.json)
  static MachineProfile b200_measured();
};

enum class Primitive { Add, Mul, Rotate };
const char* primitive_name(Primitive p);

struct Cost {
  double int_ops = 0, bytes = 0;
};

// SPEC.md:527-530
struct CostModel {
  std::uint64_t N = 1ull << 16;
  int L = 20;    // top level
  int dnum = 21; // key digits (reference key switch: one-limb digits, dnum = L + 1)
  int K = 1;     // special primes

  static CostModel from(const CkksParams& p);  // dnum = ceil((L + 1) / digit_size)
  // std::invalid_argument for level outside [1, L]
  Cost cost(Primitive p, int level) const;
};

// SPEC.md:548-556; std::invalid_argument for bytes <= 0
double intensity(double int_ops, double bytes);
double attainable(double intensity, const MachineProfile& profile);

// sum of model costs of the trace's (op, level) histogram
// (add, pt-add: Add; ct-mul, pt-mul: Mul; rotate: Rotate; others free)
Cost measure_trace(const OpTrace& trace, const CostModel& model);

struct RooflineRow {
  std::string primitive;
  int level = 0;
  double int_ops = 0, bytes = 0, intensity = 0, attainable_gops = 0;
  bool memory_bound = true;
  double measured_gbs = -1;  // optional measurement beside the model (<0: none)
};

// SPEC.md:529-532, :566-574
struct RooflineReport {
  MachineProfile profile;
  std::vector<RooflineRow> rows;

  // add / mul / rotate at every level in [l0, l1]
  static RooflineReport sweep(const CostModel& model, const MachineProfile& profile, int l0, int l1);
  // CSV: primitive,level,ops,bytes,intensity,attainable,bound[,measured_gbs]
  // (UTF-8, header row, ',' separator, '.' decimal, fixed row order)
  std::string to_csv() const;
  // SVG 1.1 log-log roofline: bandwidth slope, peak line, ridge marker and one
  // point per (primitive, level); std::invalid_argument on an empty report
  std::string to_svg() const;
  std::string to_json() const;
};

}  // namespace helix
