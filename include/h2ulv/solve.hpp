// Drop-in for proj/include/h2ulv/solve.hpp (solve.hpp:10-22).
// solve runs the forward/backward ULV sweeps on the device (all right-hand
// sides at once, each column bit-identical to a single-column solve). The
// dense oracles keep the reference's N guard and run on the device too:
// assemble_block + gemm (== matvec_dense_oracle bit for bit) and lu_factor +
// LuFactors::solve (== dense_solve_oracle).
#pragma once

#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2ulv/ulv.hpp"

namespace h2ulv {

// solve (solve.cpp:209-224): b and the result in the original point order.
inline Matrix solve(const ULVFactors& f, const Matrix& b) {
  if (!f.b200) throw std::logic_error("solve: factors not from the B200 factorization");
  if (b.rows != f.n()) throw std::invalid_argument("solve: rhs row count mismatch");
  Matrix x(b.rows, b.cols);
  if (b.cols > 0) b200::check(h2g_solve(f.b200->handle->p, b.cols, b.data(), x.data()));
  return x;
}

inline Matrix assemble_full_matrix(const PointCloud& cloud, const KernelSpec& kernel, int64_t guard = 16384) {
  const int64_t n = cloud.size();
  if (n > guard) throw std::runtime_error("dense oracle guard exceeded: N = " + std::to_string(n));
  return assemble_block(kernel, cloud, {0, n}, {0, n});
}
inline Matrix matvec_dense_oracle(const PointCloud& cloud, const KernelSpec& kernel, const Matrix& x,
                                  int64_t guard = 16384) {
  Matrix A = assemble_full_matrix(cloud, kernel, guard);
  return matmul(A, x);
}
inline Matrix dense_solve_oracle(const PointCloud& cloud, const KernelSpec& kernel, const Matrix& b,
                                 int64_t guard = 16384) {
  Matrix A = assemble_full_matrix(cloud, kernel, guard);
  LuFactors lu = lu_factor(A, 1e-15, "dense oracle");
  return lu.solve(b);
}

// One value per line, %.17g (solve.cpp:249-268).
inline void write_vector(const Matrix& v, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("write_vector: cannot open " + path);
  char buf[64];
  for (int64_t i = 0; i < v.rows; ++i) {
    std::snprintf(buf, sizeof(buf), "%.17g\n", v(i, 0));
    f << buf;
  }
}
inline Matrix read_vector(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("read_vector: cannot open " + path);
  std::vector<double> vals;
  double x;
  while (f >> x) vals.push_back(x);
  Matrix v(static_cast<int64_t>(vals.size()), 1);
  for (size_t i = 0; i < vals.size(); ++i) v(static_cast<int64_t>(i), 0) = vals[i];
  return v;
}

}  // namespace h2ulv
