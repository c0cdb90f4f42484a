// Drop-in for proj/include/h2ulv/kernels.hpp (kernels.hpp:11-39).
// assemble_block evaluates on the B200 (h2g_assemble_block): bitwise equal to
// the reference for Laplace and Yukawa (glibc exp restated on the device).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2g.h"
#include "h2ulv/geometry.hpp"
#include "h2ulv/matrix.hpp"

namespace h2ulv {

// gaussian: the BASELINE.json configs[2] kernel (B200 extension, not in the reference).
enum class KernelKind { laplace, yukawa, gaussian };

struct KernelSpec {
  KernelKind kind = KernelKind::laplace;
  double alpha_m = 0.0;
  double permittivity_scale = 4.0 * 3.14159265358979323846;
  double eta_reg = 0.0;

  static KernelSpec laplace(double eta_reg) {
    KernelSpec k;
    k.kind = KernelKind::laplace;
    k.eta_reg = eta_reg;
    return k;
  }
  static KernelSpec yukawa(double alpha_m, double eta_reg) {
    KernelSpec k;
    k.kind = KernelKind::yukawa;
    k.alpha_m = alpha_m;
    k.eta_reg = eta_reg;
    return k;
  }
};

inline double default_eta_reg(double domain_diameter, int64_t n) {
  return 1e-3 * domain_diameter / std::cbrt(static_cast<double>(n));
}

struct IndexRange {
  int64_t begin = 0;
  int64_t end = 0;
  int64_t size() const { return end - begin; }
};

namespace b200 {
inline h2g_kernel kernel_of(const KernelSpec& k) {
  return h2g_kernel{k.kind == KernelKind::laplace ? 0 : k.kind == KernelKind::yukawa ? 1 : 2, k.alpha_m,
                    k.permittivity_scale, k.eta_reg};
}
}  // namespace b200

// Single entry (kernels.cpp:232-240), host scalar helper (not a hot path).
inline double kernel_eval(const KernelSpec& spec, const std::array<double, 3>& xi,
                          const std::array<double, 3>& xj, double qj) {
  const double dx = xi[0] - xj[0], dy = xi[1] - xj[1], dz = xi[2] - xj[2];
  if (spec.kind == KernelKind::gaussian) {
    const double r2 = std::fma(dz, dz, std::fma(dx, dx, dy * dy));
    return qj * (std::exp(-spec.alpha_m * r2) + (r2 == 0.0 ? spec.eta_reg : 0.0)) / spec.permittivity_scale;
  }
  const double r = std::sqrt(std::fma(dz, dz, std::fma(dx, dx, dy * dy)));
  const double denom = spec.permittivity_scale * (r + spec.eta_reg);
  if (denom == 0.0) throw std::runtime_error("kernel_eval: singular evaluation (r + eta_reg == 0)");
  if (spec.kind == KernelKind::laplace) return qj / denom;
  return qj * std::exp(-spec.alpha_m * r) / denom;
}

// assemble_block (kernels.cpp:242-268) on the device.
inline Matrix assemble_block(const KernelSpec& spec, const PointCloud& cloud, IndexRange rows, IndexRange cols) {
  if (rows.size() <= 0 || cols.size() <= 0) throw std::invalid_argument("assemble_block: empty range");
  if (rows.begin < 0 || cols.begin < 0 || rows.end > cloud.size() || cols.end > cloud.size())
    throw std::out_of_range("assemble_block: range outside cloud");
  std::vector<double> xyz;
  b200::aos(cloud, xyz);
  const h2g_kernel k = b200::kernel_of(spec);
  Matrix B(rows.size(), cols.size());
  b200::check(h2g_assemble_block(&k, cloud.size(), xyz.data(), cloud.charges.data(), rows.begin, rows.end,
                                 cols.begin, cols.end, B.data()));
  return B;
}

}  // namespace h2ulv
