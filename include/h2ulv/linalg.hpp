// Drop-in for proj/include/h2ulv/linalg.hpp (linalg.hpp:12-104). The dense
// kernels run on the B200 through the C ABI's single-primitive entry points,
// which reproduce the reference's rounding (gemm_core's fma order, lu_factor's
// right-looking recurrences): gemm / matmul / gemm_acc -> h2g_gemm,
// lu_factor -> h2g_lu_factor, LuFactors::solve* -> h2g_lu_solve,
// qr_pivoted_members -> h2g_basis_from_members. Norms and permutations are
// host bookkeeping.
#pragma once

#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2g.h"
#include "h2ulv/matrix.hpp"

namespace h2ulv {

namespace b200 {
// Status -> the reference's exception types (invalid_argument for shapes and
// configuration, runtime_error for numerical failures).
inline void check(int rc) {
  if (rc == 0) return;
  const std::string msg = h2g_last_error();
  if (msg.rfind("config:", 0) == 0 || msg.find("must be") != std::string::npos ||
      msg.find("need N >=") != std::string::npos || msg.find("empty range") != std::string::npos)
    throw std::invalid_argument(msg);
  if (msg.find("outside cloud") != std::string::npos || msg.find("no dense block") != std::string::npos)
    throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}
}  // namespace b200

struct Permutation {
  std::vector<int64_t> forward;
  int64_t size() const { return static_cast<int64_t>(forward.size()); }
  static Permutation identity(int64_t n) {
    Permutation p;
    p.forward.resize(size_t(n));
    for (int64_t i = 0; i < n; ++i) p.forward[size_t(i)] = i;
    return p;
  }
  bool valid() const {
    std::vector<char> seen(forward.size(), 0);
    for (int64_t v : forward) {
      if (v < 0 || v >= size() || seen[size_t(v)]) return false;
      seen[size_t(v)] = 1;
    }
    return true;
  }
};

struct RankDecision {
  double tol = 1e-8;
  std::optional<int64_t> cap;
};

enum class Side { left, right };
enum class Uplo { lower, upper };

inline void require_finite(const Matrix& A, const char* what) {
  if (!A.finite()) throw std::invalid_argument(std::string("non-finite input to ") + what);
}

// C = alpha op(A) op(B) + beta C (linalg.cpp:86-116): beta C first, then the
// reference's fma chain on the device.
inline Matrix gemm(double alpha, const Matrix& A, const Matrix& B, double beta, const Matrix& C,
                   bool transA = false, bool transB = false) {
  const int64_t m = transA ? A.cols : A.rows, k = transA ? A.rows : A.cols;
  const int64_t kb = transB ? B.cols : B.rows, n = transB ? B.rows : B.cols;
  if (kb != k)
    throw std::invalid_argument("gemm: shape mismatch (" + std::to_string(m) + "x" + std::to_string(k) +
                                " * " + std::to_string(kb) + "x" + std::to_string(n) + ")");
  Matrix R(m, n);
  if (beta != 0.0) {
    if (C.rows != m || C.cols != n) throw std::invalid_argument("gemm: C shape mismatch");
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) R(i, j) = beta * C(i, j);
  }
  if (alpha != 0.0 && m > 0 && n > 0 && k > 0)
    b200::check(h2g_gemm(m, n, k, alpha, A.data(), transA ? 1 : 0, B.data(), transB ? 1 : 0, 1, R.data()));
  return R;
}
inline Matrix matmul(const Matrix& A, const Matrix& B, bool transA = false, bool transB = false,
                     double alpha = 1.0) {
  return gemm(alpha, A, B, 0.0, Matrix(), transA, transB);
}
inline void gemm_acc(Matrix& C, const Matrix& A, const Matrix& B, double alpha) {
  if (A.cols != B.rows || C.rows != A.rows || C.cols != B.cols)
    throw std::invalid_argument("gemm_acc: shape mismatch");
  if (A.rows > 0 && B.cols > 0 && A.cols > 0)
    b200::check(h2g_gemm(A.rows, B.cols, A.cols, alpha, A.data(), 0, B.data(), 0, 1, C.data()));
}

struct PivotedQr {
  Matrix Qs;
  Matrix Qr;
  int64_t rank = 0;
  Permutation perm;  // not reported by the device QR (left empty)
};

// Pivoted QR over member groups with the member-mass stopping rule
// (linalg.cpp:216-332), on the device. The device entry point applies the
// reference's member tolerance factor (0.5 tol, compression.hpp:67).
inline PivotedQr qr_pivoted_members(const Matrix& A, const RankDecision& decision,
                                    const std::vector<int64_t>& member_offsets, double member_tol) {
  if (std::fabs(member_tol - 0.5 * decision.tol) > 1e-15 * decision.tol)
    throw std::invalid_argument("qr_pivoted_members: the B200 path supports member_tol = 0.5 tol");
  Matrix sq(A.rows, A.rows);
  int64_t rank = 0;
  b200::check(h2g_basis_from_members(A.rows, A.cols, A.data(), int64_t(member_offsets.size()) - 1,
                                     member_offsets.data(), decision.tol, decision.cap.value_or(0), 0,
                                     sq.data(), &rank));
  PivotedQr out;
  out.rank = rank;
  out.Qs = sq.block(0, A.rows - rank, A.rows, rank);
  out.Qr = sq.block(0, 0, A.rows, A.rows - rank);
  return out;
}

struct LuFactors {
  Matrix lu;
  Permutation perm;
  int64_t n() const { return lu.rows; }

  void solve_in_place(Matrix& X) const { apply(X, 0); }
  void solve_right_in_place(Matrix& X) const { apply(X, 4); }
  Matrix solve(const Matrix& B) const {
    Matrix X = B;
    solve_in_place(X);
    return X;
  }
  Matrix solve_right(const Matrix& B) const {
    Matrix X = B;
    solve_right_in_place(X);
    return X;
  }
  void solve_lower_in_place(Matrix& X) const { apply(X, 1); }
  void solve_upper_in_place(Matrix& X) const { apply(X, 2); }
  void solve_upper_right_in_place(Matrix& X) const { apply(X, 5); }
  void solve_transpose_in_place(Matrix& X) const { apply(X, 3); }
  Matrix solve_transpose(const Matrix& B) const {
    Matrix X = B;
    solve_transpose_in_place(X);
    return X;
  }

 private:
  // h2g_lu_solve kinds: 0 solve, 1 lower, 2 upper, 3 transpose, 4 right, 5 upper_right
  void apply(Matrix& X, int kind) const {
    const bool right = kind == 4 || kind == 5;
    if ((right ? X.cols : X.rows) != n()) throw std::invalid_argument("LuFactors: shape mismatch");
    if (X.empty() || n() == 0) return;
    b200::check(h2g_lu_solve(n(), lu.data(), perm.forward.data(), kind, X.rows, X.cols, X.data()));
  }
};

// lu_factor (linalg.cpp:352-388) on the device; a singular pivot raises the
// reference's "singular block in LU of <what> at step k".
inline LuFactors lu_factor(const Matrix& A, double pivot_tol = 1e-14, const char* what = "block") {
  if (A.rows != A.cols) throw std::invalid_argument("lu_factor: matrix not square");
  LuFactors f;
  f.lu = Matrix(A.rows, A.rows);
  f.perm.forward.resize(size_t(A.rows));
  if (A.rows == 0) return f;
  if (h2g_lu_factor(A.rows, A.data(), pivot_tol, f.lu.data(), f.perm.forward.data()) != 0) {
    std::string msg = h2g_last_error();
    const std::string from = "LU of block";
    const size_t at = msg.find(from);
    if (at != std::string::npos) msg.replace(at, from.size(), std::string("LU of ") + what);
    throw std::runtime_error(msg);
  }
  return f;
}

inline double norm_frobenius(const Matrix& A) {
  double s = 0.0;
  for (int64_t j = 0; j < A.cols; ++j)
    for (int64_t i = 0; i < A.rows; ++i) s += A(i, j) * A(i, j);
  return std::sqrt(s);
}
inline double norm_max_abs(const Matrix& A) {
  double m = 0.0;
  for (int64_t j = 0; j < A.cols; ++j)
    for (int64_t i = 0; i < A.rows; ++i) m = std::max(m, std::fabs(A(i, j)));
  return m;
}
inline double rel_error(const Matrix& x, const Matrix& x_ref) {
  if (x.rows != x_ref.rows || x.cols != x_ref.cols) throw std::invalid_argument("rel_error: shape mismatch");
  double num = 0.0, den = 0.0;
  for (int64_t j = 0; j < x.cols; ++j)
    for (int64_t i = 0; i < x.rows; ++i) {
      const double d = x(i, j) - x_ref(i, j);
      num += d * d;
      den += x_ref(i, j) * x_ref(i, j);
    }
  if (den == 0.0) throw std::invalid_argument("rel_error: reference is zero");
  return std::sqrt(num / den);
}
inline Matrix apply_permutation_rows(const Permutation& p, const Matrix& A) {
  if (p.size() != A.rows) throw std::invalid_argument("apply_permutation_rows: size mismatch");
  Matrix B(A.rows, A.cols);
  for (int64_t j = 0; j < A.cols; ++j)
    for (int64_t i = 0; i < A.rows; ++i) B(i, j) = A(p.forward[size_t(i)], j);
  return B;
}

}  // namespace h2ulv
