// packing.cpp -- matrix layouts of SPEC.md:247-346 (see helix/packing.hpp).
#include "helix/packing.hpp"

#include <algorithm>

namespace helix {

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

BsgsPlan BsgsPlan::for_dim(int d) {
  if (d < 1 || (d & (d - 1))) throw std::invalid_argument("BsgsPlan: d must be a power of two");
  int lg = 0;
  while ((1 << lg) < d) ++lg;
  BsgsPlan p;
  p.n1 = 1 << ((lg + 1) / 2);  // sqrt(d) for even lg, sqrt(2d) for odd lg
  p.n2 = d / p.n1;
  return p;
}

BsgsPlan BsgsPlan::for_cost(int d, int row_blocks, double baby_cost, double giant_cost, int max_n1) {
  if (d < 1 || (d & (d - 1))) throw std::invalid_argument("BsgsPlan: d must be a power of two");
  if (row_blocks < 1 || !(baby_cost > 0.0) || !(giant_cost > 0.0))
    throw std::invalid_argument("BsgsPlan::for_cost: row_blocks and the costs must be positive");
  BsgsPlan best = for_dim(d);
  auto cost = [&](const BsgsPlan& p) {
    return (p.n1 - 1) * baby_cost + (double)row_blocks * (p.n2 - 1) * giant_cost;
  };
  double bc = cost(best);
  for (int n1 = 1; n1 <= d && n1 <= max_n1; n1 <<= 1) {
    BsgsPlan p;
    p.n1 = n1;
    p.n2 = d / n1;
    const double c = cost(p);
    if (c < bc) {  // ties keep the SPEC default
      bc = c;
      best = p;
    }
  }
  return best;
}

std::size_t PackedMatrix::nonzero_payloads() const {
  std::size_t c = 0;
  for (const auto& p : payloads) c += !p.empty();
  return c;
}

std::vector<double> replicate(const std::vector<double>& x, int d, std::size_t n) {
  std::vector<double> out(n, 0.0);
  for (std::size_t s = 0; s < n; ++s) {
    const std::size_t i = s % (std::size_t)d;
    out[s] = i < x.size() ? x[i] : 0.0;
  }
  return out;
}

namespace {

PackedMatrix diag_common(const Matrix& A, std::size_t n, Layout layout) {
  PackedMatrix M;
  M.layout = layout;
  M.rows = A.rows;
  M.cols = A.cols;
  M.d = next_pow2(std::max(A.cols, 1));
  if ((std::size_t)M.d > n) throw std::invalid_argument("pack: input dimension exceeds the slot count");
  M.row_blocks = (A.rows + M.d - 1) / M.d;
  M.pad_cols = M.d;
  M.pad_rows = M.row_blocks * M.d;
  M.slots = n;
  return M;
}

// diag_i of block b (d entries), empty when all zero
std::vector<double> block_diag(const Matrix& A, int b, int i, int d) {
  std::vector<double> v(d, 0.0);
  bool nz = false;
  for (int j = 0; j < d; ++j) {
    const int r = b * d + j, c = (i + j) % d;
    if (r < A.rows && c < A.cols) {
      v[j] = A.at(r, c);
      nz |= v[j] != 0.0;
    }
  }
  if (!nz) v.clear();
  return v;
}

}  // namespace

PackedMatrix pack_diagonals(const Matrix& A, std::size_t n) {
  PackedMatrix M = diag_common(A, n, Layout::Diagonal);
  for (int b = 0; b < M.row_blocks; ++b)
    for (int i = 0; i < M.d; ++i) {
      const auto v = block_diag(A, b, i, M.d);
      M.payloads.push_back(v.empty() ? v : replicate(v, M.d, n));
    }
  return M;
}

PackedMatrix pack_bsgs(const Matrix& A, const BsgsPlan& plan, std::size_t n) {
  PackedMatrix M = diag_common(A, n, Layout::BsgsDiagonal);
  if (plan.n1 * plan.n2 != M.d) throw std::invalid_argument("pack_bsgs: plan inconsistent with padded dim");
  M.plan = plan;
  for (int b = 0; b < M.row_blocks; ++b)
    for (int i = 0; i < M.d; ++i) {
      auto v = block_diag(A, b, i, M.d);
      if (!v.empty()) {
        const int shift = (i / plan.n1) * plan.n1;  // pre-rotate right by n1 j
        std::vector<double> r(M.d);
        for (int s = 0; s < M.d; ++s) r[s] = v[((s - shift) % M.d + M.d) % M.d];
        v = replicate(r, M.d, n);
      }
      M.payloads.push_back(std::move(v));
    }
  return M;
}

PackedMatrix pack_bsgs(const Matrix& A, std::size_t n) {
  return pack_bsgs(A, BsgsPlan::for_dim(next_pow2(std::max(A.cols, 1))), n);
}

PackedMatrix pack_bsgs_stacked(const Matrix& A, const BsgsPlan& plan, std::size_t n) {
  PackedMatrix M = diag_common(A, n, Layout::BsgsStacked);
  if (plan.n1 * plan.n2 != M.d) throw std::invalid_argument("pack_bsgs_stacked: plan inconsistent with padded dim");
  if ((std::size_t)M.row_blocks * M.d > n) throw std::invalid_argument("pack_bsgs_stacked: blocks x d exceeds the slot count");
  M.plan = plan;
  const int B = M.row_blocks, d = M.d;
  M.row_blocks = 1;  // one stacked output ciphertext
  for (int i = 0; i < d; ++i) {
    std::vector<double> D(n, 0.0);
    bool any = false;
    for (int b = 0; b < B; ++b)
      for (int r = 0; r < d; ++r) {
        const int row = b * d + r, col = (r + i) % d;
        if (row < A.rows && col < A.cols) {
          const double v = A.at(row, col);
          D[(std::size_t)row] = v;
          any = any || v != 0.0;
        }
      }
    if (!any) {
      M.payloads.emplace_back();
      continue;
    }
    const std::size_t shift = (std::size_t)(i / plan.n1) * plan.n1;  // rotate right by n1 j over all n slots
    std::vector<double> R(n);
    for (std::size_t s = 0; s < n; ++s) R[s] = D[(s + n - shift) % n];
    M.payloads.push_back(std::move(R));
  }
  M.stacked_blocks = B;
  return M;
}

PackedMatrix pack_bsgs_stacked(const Matrix& A, std::size_t n) {
  return pack_bsgs_stacked(A, BsgsPlan::for_dim(next_pow2(std::max(A.cols, 1))), n);
}

PackedMatrix pack_rows(const Matrix& A, std::size_t n) {
  PackedMatrix M;
  M.layout = Layout::PackedRow;
  M.rows = A.rows;
  M.cols = A.cols;
  M.pad_cols = next_pow2(std::max(A.cols, 1));
  if ((std::size_t)M.pad_cols > n) throw std::invalid_argument("pack_rows: row wider than the slot count");
  M.d = M.pad_cols;
  M.rows_per_payload = std::max(1, std::min((int)(n / M.pad_cols), A.rows));
  const int groups = (A.rows + M.rows_per_payload - 1) / M.rows_per_payload;
  M.pad_rows = groups * M.rows_per_payload;
  M.slots = n;
  for (int g = 0; g < groups; ++g) {
    std::vector<double> v(n, 0.0);
    for (int r = 0; r < M.rows_per_payload; ++r) {
      const int row = g * M.rows_per_payload + r;
      if (row >= A.rows) break;
      for (int c = 0; c < A.cols; ++c) v[(std::size_t)r * M.pad_cols + c] = A.at(row, c);
    }
    M.payloads.push_back(std::move(v));
  }
  return M;
}

PackedMatrix pack_rowmajor(const Matrix& A, std::size_t n) {
  PackedMatrix M;
  M.layout = Layout::RowMajor;
  M.rows = A.rows;
  M.cols = A.cols;
  M.d = next_pow2(std::max({A.rows, A.cols, 1}));
  if ((std::size_t)M.d * M.d > n) throw std::invalid_argument("pack_rowmajor: d^2 > n");
  M.pad_rows = M.pad_cols = M.d;
  M.slots = n;
  std::vector<double> v(n, 0.0);
  for (int r = 0; r < A.rows; ++r)
    for (int c = 0; c < A.cols; ++c) v[(std::size_t)r * M.d + c] = A.at(r, c);
  M.payloads.push_back(std::move(v));
  return M;
}

Matrix unpack(const PackedMatrix& M) {
  Matrix A(M.rows, M.cols);
  switch (M.layout) {
    case Layout::Diagonal:
    case Layout::BsgsDiagonal:
      for (int b = 0; b < M.row_blocks; ++b)
        for (int i = 0; i < M.d; ++i) {
          const auto& p = M.payloads[(std::size_t)b * M.d + i];
          if (p.empty()) continue;
          const int shift = M.layout == Layout::BsgsDiagonal ? (i / M.plan.n1) * M.plan.n1 : 0;
          for (int j = 0; j < M.d; ++j) {
            const int r = b * M.d + j, c = (i + j) % M.d;
            if (r < M.rows && c < M.cols) A.at(r, c) = p[(j + shift) % M.d];
          }
        }
      break;
    case Layout::PackedRow:
      for (std::size_t g = 0; g < M.payloads.size(); ++g)
        for (int r = 0; r < M.rows_per_payload; ++r) {
          const int row = (int)g * M.rows_per_payload + r;
          if (row >= M.rows) break;
          for (int c = 0; c < M.cols; ++c) A.at(row, c) = M.payloads[g][(std::size_t)r * M.pad_cols + c];
        }
      break;
    case Layout::RowMajor:
      for (int r = 0; r < M.rows; ++r)
        for (int c = 0; c < M.cols; ++c) A.at(r, c) = M.payloads[0][(std::size_t)r * M.d + c];
      break;
    case Layout::BsgsStacked:
      for (int i = 0; i < M.d; ++i) {
        const auto& p = M.payloads[i];
        if (p.empty()) continue;
        const std::size_t shift = (std::size_t)(i / M.plan.n1) * M.plan.n1, n = p.size();
        for (int row = 0; row < M.rows; ++row) {
          const int c = (row % M.d + i) % M.d;
          if (c < M.cols) A.at(row, c) = p[((std::size_t)row + shift) % n];
        }
      }
      break;
  }
  return A;
}

std::vector<double> make_mask(MaskKind kind, int i, int d, std::size_t n) {
  if (d < 1 || i < 0 || i >= d) throw std::invalid_argument("make_mask: index out of range");
  std::vector<double> m(n, 0.0);
  switch (kind) {
    case MaskKind::ColumnExtractor:
      for (int k = 0; k < d; ++k)
        if ((std::size_t)(i + k * d) < n) m[i + (std::size_t)k * d] = 1.0;
      break;
    case MaskKind::RowExtractor:
      for (int k = 0; k < d; ++k)
        if ((std::size_t)i * d + k < n) m[(std::size_t)i * d + k] = 1.0;
      break;
    case MaskKind::StrideSelector:
      for (std::size_t s = i; s < n; s += d) m[s] = 1.0;
      break;
  }
  return m;
}

Tiling tile_matrix(const Matrix& A, std::size_t n, Layout layout) {
  Tiling t;
  const int pr = next_pow2(std::max(A.rows, 1)), pc = next_pow2(std::max(A.cols, 1));
  int b = 1;
  if (layout == Layout::RowMajor) {
    while ((std::size_t)(2 * b) * (2 * b) <= n) b <<= 1;
    b = std::min({b, std::max(pr, pc)});
  } else {
    while ((std::size_t)(2 * b) <= n) b <<= 1;
    b = std::min(b, std::max(pr, pc));
  }
  t.block = b;
  t.grid_rows = (A.rows + b - 1) / b;
  t.grid_cols = (A.cols + b - 1) / b;
  return t;
}

}  // namespace helix
