// Shared device-side definitions for the B200 H2-ULV hot path.
//
// Every dense object is an FP64 strided view: element (i, j) lives at
// p[i * rs + j * cs]. Column-major (the reference Matrix layout,
// proj/include/h2ulv/matrix.hpp:19-20) is rs = 1, cs = ld; a transpose is a
// stride swap, so op(A) never needs a copy.
//
// Floating point: all kernels are compiled with --fmad=false and write every
// FMA the reference's GCC -O3 -mfma build contracts as an explicit fma(), in
// the reference's per-element accumulation order. That is what makes the GPU
// results bitwise equal to the reference for the Laplace kernel.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "exp_table.cuh"

namespace h2g {

struct Mat {
  double* p = nullptr;
  int rows = 0, cols = 0;
  int64_t rs = 1, cs = 0;
  __host__ __device__ double& at(int64_t i, int64_t j) const { return p[i * rs + j * cs]; }
  __host__ __device__ Mat t() const { return Mat{p, cols, rows, cs, rs}; }
  __host__ __device__ Mat sub(int r0, int c0, int nr, int nc) const {
    return Mat{p + r0 * rs + c0 * cs, nr, nc, rs, cs};
  }
  __host__ __device__ int64_t size() const { return int64_t(rows) * cols; }
};

inline Mat colmajor(double* p, int rows, int cols, int64_t ld = -1) {
  return Mat{p, rows, cols, 1, ld < 0 ? rows : ld};
}

// Kernel function parameters (kernels.hpp:15-23): 0 = Laplace, 1 = Yukawa,
// 2 = Gaussian (BASELINE configs[2]; not in the reference): q_j (exp(-alpha_m r^2)
// + [r == 0] reg) / scale, i.e. exp(-r^2/h) + sigma I with alpha_m = 1/h, reg = sigma.
struct KernelParams {
  int kind = 0;
  double alpha_m = 0.0;
  double scale = 4.0 * 3.14159265358979323846;
  double reg = 0.0;
};

// Counted flops per kernel entry (kernels.cpp:266: 9 Laplace, 11 Yukawa; the
// Gaussian is counted like Yukawa).
inline double kernel_entry_flops(int kind) { return kind == 0 ? 9.0 : 11.0; }

// Reordered cloud in SoA form on the device.
struct Cloud {
  const double* x = nullptr;
  const double* y = nullptr;
  const double* z = nullptr;
  const double* q = nullptr;
  int64_t n = 0;
};

// The double-precision exp of glibc >= 2.28 (x86-64 FMA variant, the
// algorithm of ARM optimized-routines' exp: N = 128 table, degree-5
// polynomial, its published coefficients), restated operation by operation
// with the contractions of libm's __exp_fma, so the result has the same bits
// as the std::exp the reference's Yukawa kernel calls (kernels.cpp:36,58).
// Covered bit for bit: |x| < 512 (the main path and the tiny-|x| path);
// larger |x| (over/underflow handling) falls back to CUDA exp.
static __device__ const uint64_t k_exp_tab[2 * 128] = {H2G_EXP_TABLE_INIT};

__host__ __device__ __forceinline__ double exp_glibc_core(double x, const uint64_t* tab, bool* special) {
  const double inv_ln2_n = 0x1.71547652b82fep+7, shift = 0x1.8p52;
  const double neg_ln2_hi_n = -0x1.62e42fefa0000p-8, neg_ln2_lo_n = -0x1.cf79abc9e3b3ap-47;
  const double c2 = 0x1.ffffffffffdbdp-2, c3 = 0x1.555555555543cp-3;
  const double c4 = 0x1.55555cf172b91p-5, c5 = 0x1.1111167a4d017p-7;
  uint64_t ix;
  memcpy(&ix, &x, 8);
  const int abstop = int((ix >> 52) & 0x7ff);
  *special = false;
  if (unsigned(abstop - 0x3c9) > 0x3eu) {
    if (abstop - 0x3c9 < 0) return x + 1.0;  // |x| < 2^-54
    *special = true;                         // |x| >= 512, inf, nan
    return 0.0;
  }
  const double z = fma(x, inv_ln2_n, shift);
  uint64_t ki;
  memcpy(&ki, &z, 8);
  const double kd = z - shift;
  double r = fma(kd, neg_ln2_hi_n, x);
  r = fma(kd, neg_ln2_lo_n, r);
  const int idx = int(2 * (ki & 127));
  const uint64_t top = ki << 45;
  double tail;
  memcpy(&tail, &tab[idx], 8);
  const uint64_t sbits = tab[idx + 1] + top;
  const double p23 = fma(r, c3, c2);
  const double t0 = r + tail;
  const double r2 = r * r;
  const double p45 = fma(r, c5, c4);
  const double t1 = fma(p23, r2, t0);
  const double r4 = r2 * r2;
  const double tmp = fma(r4, p45, t1);
  double scale;
  memcpy(&scale, &sbits, 8);
  return fma(scale, tmp, scale);
}

__device__ __forceinline__ double exp_glibc(double x) {
  bool special;
  const double v = exp_glibc_core(x, k_exp_tab, &special);
  return special ? exp(x) : v;
}

// kernel_eval / assemble_block entry (kernels.cpp:232-268): bitwise equal to
// the reference (r = sqrt(fma(dz,dz,fma(dx,dx,dy*dy))), IEEE sqrt and
// division, glibc's exp for Yukawa).
template <int KIND>
__device__ __forceinline__ double kernel_pair_k(const KernelParams& kp, double xi, double yi,
                                                double zi, double xj, double yj, double zj,
                                                double qj, int* singular) {
  const double dx = xi - xj, dy = yi - yj, dz = zi - zj;
  if (KIND == 2) {
    const double r2 = fma(dz, dz, fma(dx, dx, dy * dy));
    const double v = exp_glibc(-kp.alpha_m * r2) + (r2 == 0.0 ? kp.reg : 0.0);
    return qj * v / kp.scale;
  }
  const double r = sqrt(fma(dz, dz, fma(dx, dx, dy * dy)));
  const double denom = kp.scale * (r + kp.reg);
  if (denom == 0.0) {
    *singular = 1;
    return 0.0;
  }
  if (KIND == 0) return qj / denom;
  return qj * exp_glibc(-kp.alpha_m * r) / denom;
}

__device__ __forceinline__ double kernel_pair(const KernelParams& kp, double xi, double yi,
                                              double zi, double xj, double yj, double zj,
                                              double qj, int* singular) {
  if (kp.kind == 0) return kernel_pair_k<0>(kp, xi, yi, zi, xj, yj, zj, qj, singular);
  if (kp.kind == 1) return kernel_pair_k<1>(kp, xi, yi, zi, xj, yj, zj, qj, singular);
  return kernel_pair_k<2>(kp, xi, yi, zi, xj, yj, zj, qj, singular);
}

__device__ __forceinline__ double kernel_entry(const KernelParams& kp, const Cloud& c, int64_t i,
                                               int64_t j, int* singular) {
  return kernel_pair(kp, c.x[i], c.y[i], c.z[i], c.x[j], c.y[j], c.z[j], c.q[j], singular);
}

// Device-wide error word: first nonzero code wins (host reads after sync).
struct ErrWord {
  int code;   // 0 ok, 1 singular kernel evaluation, 2 singular LU pivot
  int job;    // job index within the failing batch
  int step;   // LU step
  int tag;    // caller tag (which batch)
};

__device__ __forceinline__ void raise_err(ErrWord* e, int code, int job, int step, int tag) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->job = job;
    e->step = step;
    e->tag = tag;
  }
}

}  // namespace h2g
