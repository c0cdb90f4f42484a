// Batched column-pivoted Householder QR with the member-mass stopping rule,
// followed by full Q formation: run_pivoted_qr + form_q (linalg.cpp:137-185,
// :216-332) as driven by basis_from_members (compression.cpp:111-146).
//
// One CTA per basis. The working copy R is row-major so that the
// thread-per-column reflector application (each column's dot product and
// update run sequentially over rows, exactly as the reference) reads and
// writes coalesced rows. Column norms, downdates, the 4e-15 tie rule, the
// member masses and the stopping tests all follow the reference's operation
// order, so ranks and Q are bitwise equal to the reference's.
#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int NT = 512;

// The reference's reductions as GCC -O3 -mavx2 -mfma compiles them
// (linalg.cpp; disassembly of oracle/_ref, verified bit-exact on random
// members in tests). In every vectorised loop the 4-wide groups round each
// product and add in order; the loops differ only in their tails:
//   H : trailing pair rounded-and-added, odd last element fused
//       (apply_reflector dot, vnormsq for tc >= 2, solve_transpose);
//   P2: tc <= 3 all fused; otherwise each remainder element fused
//       (column norms, make_reflector normsq, downdate recompute).
template <class G>
__device__ __forceinline__ double red_h(G get, int i0, int tc, double s) {
  const int v4 = tc & ~3;
  int i = 0;
  for (; i < v4; ++i) {
    double a, b;
    get(i0 + i, a, b);
    s = s + a * b;
  }
  if ((tc & 3) >= 2) {
    double a, b;
    get(i0 + i, a, b);
    s = s + a * b;
    get(i0 + i + 1, a, b);
    s = s + a * b;
    i += 2;
  }
  if (tc & 1) {
    double a, b;
    get(i0 + i, a, b);
    s = fma(a, b, s);
  }
  return s;
}

template <class G>
__device__ __forceinline__ double red_p2(G get, int i0, int tc) {
  double s = 0.0;
  if (tc <= 3) {
    for (int i = 0; i < tc; ++i) {
      double a, b;
      get(i0 + i, a, b);
      s = fma(a, b, s);
    }
    return s;
  }
  const int v4 = tc & ~3;
  int i = 0;
  for (; i < v4; ++i) {
    double a, b;
    get(i0 + i, a, b);
    s = s + a * b;
  }
  for (; i < tc; ++i) {
    double a, b;
    get(i0 + i, a, b);
    s = fma(a, b, s);
  }
  return s;
}

struct Scratch {
  double* cn2;
  double* cn2o;
  int* piv;
  int* mof;
  double* mm;
  double* mt;
  double* V;
  double* tau;
};

__host__ __device__ inline Scratch carve(double* s, int m, int n, int nmem) {
  const int kmax0 = m < n ? m : n;
  Scratch c;
  c.cn2 = s;
  c.cn2o = s + n;
  c.piv = reinterpret_cast<int*>(s + 2 * int64_t(n));
  c.mof = c.piv + n;
  c.mm = s + 3 * int64_t(n);
  c.mt = c.mm + nmem;
  c.tau = c.mt + nmem;
  c.V = c.tau + kmax0;
  return c;
}

__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < int(blockDim.x >> 5) ? red[l] : -1.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ int block_min_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_down_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < int(blockDim.x >> 5) ? red[l] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_down_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const int r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(NT) qr_kernel(const QrJob* __restrict__ jobs) {
  extern __shared__ double vsh[];  // reflector, m doubles
  __shared__ double redd[32];
  __shared__ int redi[32];
  __shared__ double sh_tau;
  const QrJob job = jobs[blockIdx.x];
  const int m = job.m, n = job.n, nmem = job.nmem;
  double* W = job.work;
  const int64_t ldw = job.ldw;
  const int tid = threadIdx.x;
  Scratch S = carve(job.scratch, m, n, nmem);
  const int kmax0 = m < n ? m : n;
  int kmax = kmax0;
  if (job.cap > 0 && job.cap < kmax) kmax = job.cap;

  // R = A (skipped when factoring in place), column norms.
  if (!(job.A.p == W && job.A.rs == ldw && job.A.cs == 1)) {
    for (int64_t e = tid; e < int64_t(m) * n; e += NT) {
      const int i = int(e / n), j = int(e % n);
      W[i * ldw + j] = job.A.at(i, j);
    }
  }
  __syncthreads();
  for (int j = tid; j < n; j += NT) {
    const double s = red_p2([&](int i, double& a, double& b) { a = b = W[i * ldw + j]; }, 0, m);
    S.cn2[j] = s;
    S.cn2o[j] = s;
    S.piv[j] = j;
  }
  __syncthreads();
  const bool members = nmem >= 1;
  if (members) {
    for (int g = tid; g < nmem; g += NT) {
      double mass = 0.0;
      for (int64_t j = job.member_off[g]; j < job.member_off[g + 1]; ++j) {
        S.mof[j] = g;
        mass += S.cn2[j];
      }
      S.mm[g] = mass;
      S.mt[g] = job.member_tol * job.member_tol * mass;
    }
  }
  __syncthreads();

  double r11 = -1.0;
  int rank = 0;
  for (int k = 0; k < kmax; ++k) {
    double mx = -1.0;
    for (int j = k + tid; j < n; j += NT) mx = fmax(mx, S.cn2[j]);
    const double best = block_max(mx, redd);
    if (best <= 0.0) break;
    const double tie = best * (1.0 - 4e-15);
    int cand = 0x7fffffff;
    for (int j = k + tid; j < n; j += NT)
      if (S.cn2[j] >= tie) cand = min(cand, S.piv[j]);
    const int sel_orig = block_min_int(cand, redi);
    // Locate the position holding original column sel_orig (unique).
    int selpos = 0x7fffffff;
    for (int j = k + tid; j < n; j += NT)
      if (S.piv[j] == sel_orig && S.cn2[j] >= tie) selpos = j;
    const int sel = block_min_int(selpos, redi);
    if (sel != k) {
      for (int i = tid; i < m; i += NT) {
        const double t = W[i * ldw + k];
        W[i * ldw + k] = W[i * ldw + sel];
        W[i * ldw + sel] = t;
      }
      if (tid == 0) {
        double t = S.cn2[k]; S.cn2[k] = S.cn2[sel]; S.cn2[sel] = t;
        t = S.cn2o[k]; S.cn2o[k] = S.cn2o[sel]; S.cn2o[sel] = t;
        int ti = S.piv[k]; S.piv[k] = S.piv[sel]; S.piv[sel] = ti;
        if (members) { ti = S.mof[k]; S.mof[k] = S.mof[sel]; S.mof[sel] = ti; }
      }
    }
    __syncthreads();
    const double pivot_norm = sqrt(fmax(0.0, S.cn2[k]));
    if (k == 0) r11 = pivot_norm;
    const bool diag_done = pivot_norm <= job.tol * r11;
    int not_done = 0;
    if (members)
      for (int g = tid; g < nmem; g += NT) not_done |= (S.mm[g] > S.mt[g]);
    const bool members_done = !__syncthreads_or(not_done);
    const bool floor_hit = pivot_norm <= 1e-15 * r11;
    if ((diag_done && members_done) || floor_hit) break;

    // make_reflector (linalg.cpp:152-178), sequential on one thread.
    double* vk = S.V + int64_t(k) * m;
    if (tid == 0) {
      const double normsq =
          red_p2([&](int i, double& a, double& b) { a = b = W[i * ldw + k]; }, k, m - k);
      const double norm = sqrt(normsq);
      for (int i = 0; i < k; ++i) vk[i] = 0.0;
      double tau = 0.0;
      if (norm == 0.0) {
        for (int i = k; i < m; ++i) vk[i] = 0.0;
      } else {
        const double a0 = W[k * ldw + k];
        const double alpha = (a0 >= 0.0) ? -norm : norm;
        vk[k] = a0 - alpha;
        double vn = vk[k] * vk[k];
        for (int i = k + 1; i < m; ++i) vk[i] = W[i * ldw + k];
        const int tcv = m - k - 1;
        if (tcv == 1) {
          vn = vn + vk[k + 1] * vk[k + 1];
        } else if (tcv > 1) {
          vn = red_h([&](int i, double& a, double& b) { a = b = vk[i]; }, k + 1, tcv, vn);
        }
        tau = (vn == 0.0) ? 0.0 : 2.0 / vn;
        W[k * ldw + k] = alpha;
        for (int i = k + 1; i < m; ++i) W[i * ldw + k] = 0.0;
      }
      S.tau[k] = tau;
      sh_tau = tau;
    }
    __syncthreads();
    for (int i = tid; i < m; i += NT) vsh[i] = vk[i];
    __syncthreads();
    const double tau = sh_tau;
    // apply_reflector to columns k+1.. (linalg.cpp:137-149) + norm downdate.
    for (int j = k + 1 + tid; j < n; j += NT) {
      if (tau != 0.0) {
        const double dot =
            red_h([&](int i, double& a, double& b) { a = vsh[i]; b = W[i * ldw + j]; }, k, m - k, 0.0);
        const double s = tau * dot;
        for (int i = k; i < m; ++i) W[i * ldw + j] = fma(-s, vsh[i], W[i * ldw + j]);
      }
      // GCC computes rkj*rkj once (rounded) for the norm and member downdates.
      const double rkj = W[k * ldw + j];
      const double sq = rkj * rkj;
      double upd = S.cn2[j] - sq;
      if (upd < 1e-8 * S.cn2o[j])
        upd = red_p2([&](int i, double& a, double& b) { a = b = W[i * ldw + j]; }, k + 1, m - k - 1);
      S.cn2[j] = fmax(0.0, upd);
    }
    __syncthreads();
    ++rank;
    if (members && tid == 0) {
      // member_mass[g] -= rkj^2 in column order (linalg.cpp:312-315).
      const double* rowk = W + k * ldw;
      for (int j = k + 1; j < n; ++j) {
        const double rkj = rowk[j];
        const int g = S.mof[j];
        const double v = S.mm[g] - rkj * rkj;
        S.mm[g] = v < 0.0 ? 0.0 : v;
      }
      const int gk = S.mof[k];
      double v = S.mm[gk] - S.cn2[k];
      S.mm[gk] = v < 0.0 ? 0.0 : v;
      S.cn2[k] = 0.0;
    }
    __syncthreads();
  }

  // form_q (linalg.cpp:181-185): Q = I, reflectors applied backward.
  double* Q = job.Q;
  for (int64_t e = tid; e < int64_t(m) * m; e += NT) Q[e] = (e / m == e % m) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = rank - 1; k >= 0; --k) {
    const double tau = S.tau[k];
    if (tau == 0.0) continue;
    const double* vk = S.V + int64_t(k) * m;
    for (int i = tid; i < m; i += NT) vsh[i] = vk[i];
    __syncthreads();
    for (int j = tid; j < m; j += NT) {
      const double dot = red_h(
          [&](int i, double& a, double& b) { a = vsh[i]; b = Q[int64_t(i) * m + j]; }, k, m - k, 0.0);
      const double s = tau * dot;
      for (int i = k; i < m; ++i) Q[int64_t(i) * m + j] = fma(-s, vsh[i], Q[int64_t(i) * m + j]);
    }
    __syncthreads();
  }
  if (tid == 0) *job.rank_out = rank;
}

}  // namespace

size_t qr_scratch_doubles(int m, int n, int nmem) {
  const size_t kmax0 = size_t(m < n ? m : n);
  return 3 * size_t(n) + 2 * size_t(nmem) + kmax0 + size_t(m) * kmax0 + 8;
}

void launch_qr(const QrJob* jobs, int njobs, int max_m, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  qr_kernel<<<njobs, NT, sizeof(double) * size_t(max_m > 0 ? max_m : 1), st>>>(jobs);
}

}  // namespace h2g
