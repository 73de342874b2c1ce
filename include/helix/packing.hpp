// helix/packing.hpp -- cleartext matrix re-layout for the encrypted
// linear-algebra kernels (the reference's src/packing.cpp is
// listed in proj/CMakeLists.txt:21 but absent, so this follows the spec).
//
// Slot vectors are length n = N/2.  Matrices are zero-padded to powers of
// two.  For matrix-vector layouts the input vector is expected replicated
// n/d times (slot s holds x[s mod d]) so that slot rotations act cyclically on
// the d-dimensional block; every diagonal payload is replicated the same way.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace helix {

struct Matrix {
  int rows = 0, cols = 0;
  std::vector<double> data;  // row-major
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), data((std::size_t)r * c, 0.0) {}
  double& at(int r, int c) { return data[(std::size_t)r * cols + c]; }
  double at(int r, int c) const { return data[(std::size_t)r * cols + c]; }
};

enum class Layout { PackedRow, Diagonal, BsgsDiagonal, RowMajor, BsgsStacked };

// n1 * n2 = d, powers of two
struct BsgsPlan {
  int n1 = 1, n2 = 1;
  // default: n1 = n2 = sqrt(d) for an even power of two, else n1 = sqrt(2d), n2 = d / n1
  static BsgsPlan for_dim(int d);
  // Extension beyond the SPEC default: the split that minimises the key-switch
  // cost (n1 - 1) baby + row_blocks (n2 - 1) giant of a matrix with
  // `row_blocks` output blocks sharing the baby steps.  Hoisted baby steps
  // share one ModUp and pay inner product + ModDown each; double-hoisted giant
  // steps pay ModUp + inner product each, so with B > 1
  // row blocks a longer baby side wins (config 3 W1, B = 3: n1 = 64, n2 = 16
  // instead of 32 x 32).  The default cost ratio is the measured one on B200
  // (hoisted rotation 88 us, ModUp + inner product 144 us at N = 2^16, 24
  // limbs); n1 is capped at max_n1 (baby ciphertexts held in HBM at once).
  static BsgsPlan for_cost(int d, int row_blocks, double baby_cost = 88.0, double giant_cost = 144.0,
                           int max_n1 = 256);
};

struct PackedMatrix {
  Layout layout = Layout::Diagonal;
  int rows = 0, cols = 0;          // original dims (output x input for matvec layouts)
  int pad_rows = 0, pad_cols = 0;  // zero-padded powers of two
  int d = 0;                       // block dimension (matvec layouts) / matrix dim (RowMajor)
  int row_blocks = 1;              // output blocks of d rows (matvec layouts)
  int rows_per_payload = 0;        // PackedRow only
  BsgsPlan plan;                   // BsgsDiagonal / BsgsStacked
  int stacked_blocks = 0;          // BsgsStacked: row blocks stacked in the slots
  std::size_t slots = 0;
  // Diagonal / BsgsDiagonal: payloads[b * d + i] (empty vector = all-zero payload)
  // PackedRow: payloads[g]; RowMajor: payloads[0]
  std::vector<std::vector<double>> payloads;
  std::size_t nonzero_payloads() const;
};

int next_pow2(int v);

// diag[i][j] = A[j][(i + j) mod d] per d x d block
PackedMatrix pack_diagonals(const Matrix& A, std::size_t slots);
// diagonal n1 j + k stored rotated right by n1 j
PackedMatrix pack_bsgs(const Matrix& A, const BsgsPlan& plan, std::size_t slots);
PackedMatrix pack_bsgs(const Matrix& A, std::size_t slots);
// Stacked-block BSGS (an extension beyond the SPEC layouts): the row blocks of
// a tall matrix are stacked in ONE set of d full-length diagonals,
// D_i[b d + r] = A[b d + r][(r + i) mod d] for blocks b < B = ceil(rows / d)
// (B d <= n), each pre-rotated right by n1 (i / n1) over all n slots.  With x
// replicated at period d the BSGS identity holds on the whole slot vector, so
// one matvec yields every block at once -- y[row] in slot `row` -- with
// (n1 - 1) + (n2 - 1) rotations and d plaintext products instead of
// (n1 - 1) + B (n2 - 1) and B d (config 3 W1: 62 key switches instead of 124).
PackedMatrix pack_bsgs_stacked(const Matrix& A, const BsgsPlan& plan, std::size_t slots);
PackedMatrix pack_bsgs_stacked(const Matrix& A, std::size_t slots);
// rows_per_payload = min(n / pad_cols, R); payload g holds rows [g p, (g+1) p)
// at stride pad_cols
PackedMatrix pack_rows(const Matrix& A, std::size_t slots);
// slot r d + c = A[r][c], d power of two, d^2 <= n
PackedMatrix pack_rowmajor(const Matrix& A, std::size_t slots);
// exact inverse of every layout (padding excluded)
Matrix unpack(const PackedMatrix& M);

enum class MaskKind { ColumnExtractor, RowExtractor, StrideSelector };
// ColumnExtractor(i, d): 1 at {i + k d : k < d}; RowExtractor(i, d): 1 at
// [i d, (i+1) d); StrideSelector(stride = d, offset = i): 1 at {i + k d} < n.
std::vector<double> make_mask(MaskKind kind, int i, int d, std::size_t slots);

// pad-square tiling: blocks of d_b x d_b
struct Tiling {
  int block = 0, grid_rows = 0, grid_cols = 0;
};
Tiling tile_matrix(const Matrix& A, std::size_t slots, Layout layout);

// replicate a d-vector across n slots (the matvec input layout)
std::vector<double> replicate(const std::vector<double>& x, int d, std::size_t slots);

}  // namespace helix
