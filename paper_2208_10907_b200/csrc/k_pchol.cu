// Member compression for the compressed QR mode (qr_mode = 2).
//
// basis_from_members (compression.cpp:111-146) factors the concatenation
// [M_1 | M_2 | ...] of a box's members with a column-pivoted QR whose stopping
// rule is per member: every member's leftover mass ||(I - QQ^T) M_i||_F^2 must
// fall below (member_tol)^2 ||M_i||_F^2 (linalg.cpp:276-297). Both the range
// and those masses depend on M_i only through its Gram matrix G_i = M_i M_i^T,
// so any C_i with C_i C_i^T = G_i can replace M_i without changing what the
// rule measures. The exact-member scheme makes the ancestor far-field members
// O(N) wide; C_i from a diagonally pivoted Cholesky of G_i has at most
// min(dim, w_i) columns (its numerical rank, usually far fewer).
//
// pchol_kernel: one CTA per member. The lower triangle of G (dim x dim,
// column-major) is read, never written; R (dim x kmax column-major) receives the columns in pick order:
//   p_t = argmax of the unpicked remaining diagonal (lowest index on ties),
//   R(:, t) = (G(:, p_t) - R(:, 0:t) R(p_t, 0:t)^T) / sqrt(d_{p_t}),
//   d_j -= R(j, t)^2.
// It stops when the unpicked remaining trace is <= eta * trace(G) (eta is
// chosen by the host from the QR tolerance) or the diagonal is exhausted.
// The dropped mass is then <= eta * ||M_i||_F^2 by construction.
#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int NT = 256, NW = NT / 32;

struct ArgMax {
  double v;
  int i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__global__ void __launch_bounds__(NT) pchol_kernel(const PcholJob* __restrict__ jobs) {
  const PcholJob job = jobs[blockIdx.x];
  const int m = job.m;
  extern __shared__ double sm[];
  double* d = sm;            // m remaining diagonal (-1 = picked)
  double* rp = sm + m;       // kmax: row p of R
  __shared__ double red_v[NW], red_s[NW];
  __shared__ int red_i[NW];
  __shared__ double s_tr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  double tr = 0;
  for (int j = threadIdx.x; j < m; j += NT) {
    const double g = fmax(job.G[int64_t(j) * job.ldg + j], 0.0);
    d[j] = g;
    tr += g;
  }
  for (int o = 16; o; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  if (lane == 0) red_s[warp] = tr;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < NW; ++w) t += red_s[w];
    s_tr = t;
  }
  __syncthreads();
  const double stop = job.eta * s_tr;

  int t = 0;
  for (; t < job.kmax; ++t) {
    // argmax and remaining trace over the unpicked diagonal
    ArgMax am{-1.0, 0x7fffffff};
    double rem = 0;
    for (int j = threadIdx.x; j < m; j += NT) {
      const double v = d[j];
      if (v >= 0) {
        rem += v;
        am = better(am, ArgMax{v, j});
      }
    }
    for (int o = 16; o; o >>= 1) {
      rem += __shfl_xor_sync(0xffffffffu, rem, o);
      ArgMax b{__shfl_xor_sync(0xffffffffu, am.v, o), __shfl_xor_sync(0xffffffffu, am.i, o)};
      am = better(am, b);
    }
    if (lane == 0) {
      red_v[warp] = am.v;
      red_i[warp] = am.i;
      red_s[warp] = rem;
    }
    __syncthreads();
    am = ArgMax{red_v[0], red_i[0]};
    rem = red_s[0];
    for (int w = 1; w < NW; ++w) {
      am = better(am, ArgMax{red_v[w], red_i[w]});
      rem += red_s[w];
    }
    if (!(am.v > 0) || rem <= stop) break;  // uniform across the CTA
    const int p = am.i;
    // row p of R (columns 0..t-1) for the left-looking update
    for (int s = threadIdx.x; s < t; s += NT) rp[s] = job.R[int64_t(s) * job.ldr + p];
    __syncthreads();
    const double piv = sqrt(am.v);
    const double inv = 1.0 / piv;
    for (int j = threadIdx.x; j < m; j += NT) {
      double r = 0;
      if (j == p) {
        r = piv;
      } else if (d[j] >= 0) {
        // lower triangle only (the Gram GEMM skips tiles above the diagonal)
        double v = j >= p ? job.G[int64_t(p) * job.ldg + j] : job.G[int64_t(j) * job.ldg + p];
        const double* Rj = job.R + j;
        for (int s = 0; s < t; ++s) v = fma(-Rj[int64_t(s) * job.ldr], rp[s], v);
        r = v * inv;
      }
      job.R[int64_t(t) * job.ldr + j] = r;
      if (j == p)
        d[j] = -1.0;
      else if (d[j] >= 0)
        d[j] = fmax(d[j] - r * r, 0.0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) job.count[0] = t;
}

}  // namespace

void launch_pchol(const PcholJob* jobs, int njobs, int max_m, int max_k, cudaStream_t st) {
  if (njobs <= 0) return;
  const size_t smem = sizeof(double) * size_t(max_m + max_k);
  smem_attr((const void*)pchol_kernel, smem, "pchol smem attribute");
  pchol_kernel<<<njobs, NT, smem, st>>>(jobs);
}

}  // namespace h2g
