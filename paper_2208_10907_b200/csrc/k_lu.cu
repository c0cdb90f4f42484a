// Batched LU with block-local partial pivoting and the LuFactors solve
// family. One CTA per matrix (LU) or per RHS chunk (solves). Every element
// sees the reference's exact rounding sequence (linalg.cpp:352-559), so the
// packed factors and solutions are bitwise equal to the reference.
#include <cstdio>
#include <cstdlib>

#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int NT = 512;

struct ValIdx {
  double v;
  int i;
};

// Max value; ties to the lowest index — the first strict maximum of the
// reference's ascending scan (linalg.cpp:362-370).
__device__ __forceinline__ ValIdx better(ValIdx a, ValIdx b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ ValIdx block_argmax(ValIdx x, ValIdx* red) {
  for (int o = 16; o > 0; o >>= 1) {
    ValIdx y{__shfl_down_sync(0xffffffffu, x.v, o), __shfl_down_sync(0xffffffffu, x.i, o)};
    x = better(x, y);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (w == 0) {
    x = (l < (int)(blockDim.x >> 5)) ? red[l] : ValIdx{-1.0, 0x7fffffff};
    for (int o = 16; o > 0; o >>= 1) {
      ValIdx y{__shfl_down_sync(0xffffffffu, x.v, o), __shfl_down_sync(0xffffffffu, x.i, o)};
      x = better(x, y);
    }
    if (l == 0) red[0] = x;
  }
  __syncthreads();
  ValIdx r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(NT, 2) lu_kernel(const LuJob* __restrict__ jobs, ErrWord* err,
                                                int tag) {
  __shared__ ValIdx red[32];
  extern __shared__ double lcol[];  // scaled pivot column of the current step (n doubles)
  const LuJob job = jobs[blockIdx.x];
  const Mat M = job.A;
  const int n = M.rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n; i += NT) job.perm[i] = i;
  // amax = norm_max_abs(A)
  ValIdx am{0.0, 0};
  for (int j = warp; j < n; j += NT / 32)
    for (int i = lane; i < n; i += 32) {
      const double v = fabs(M.at(i, j));
      if (v > am.v) am.v = v;
    }
  const double amax = block_argmax(am, red).v;
  for (int k = 0; k < n; ++k) {
    ValIdx best{-1.0, 0x7fffffff};
    for (int i = k + threadIdx.x; i < n; i += NT) best = better(best, ValIdx{fabs(M.at(i, k)), i});
    best = block_argmax(best, red);
    if (best.v <= job.tol * amax) {
      if (threadIdx.x == 0) raise_err(err, 2, blockIdx.x, k, tag);
      return;
    }
    const int p = best.i;
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += NT) {
        const double t = M.at(k, j);
        M.at(k, j) = M.at(p, j);
        M.at(p, j) = t;
      }
      if (threadIdx.x == 0) {
        const int64_t t = job.perm[k];
        job.perm[k] = job.perm[p];
        job.perm[p] = t;
      }
      __syncthreads();
    }
    const double inv = 1.0 / M.at(k, k);
    for (int i = k + 1 + threadIdx.x; i < n; i += NT) {
      const double l = M.at(i, k) * inv;
      M.at(i, k) = l;
      lcol[i] = l;
    }
    __syncthreads();
    // Rank-1 update of the trailing block: a warp per column (u_kj loaded
    // once), lanes down the rows (coalesced), l_ik from shared memory.
    for (int j = k + 1 + warp; j < n; j += NT / 32) {
      const double u = M.at(k, j);
      for (int i = k + 1 + lane; i < n; i += 32) M.at(i, j) = fma(-lcol[i], u, M.at(i, j));
    }
    __syncthreads();
  }
}

// ---- blocked LU inside one CTA (medium blocks) ------------------------------
// The same right-looking order as lu_kernel, with the trailing update delayed
// by panels of FNB columns (exactly the scheme of the multi-kernel blocked LU
// below, fused into one CTA per block so a batch of leaf blocks costs no extra
// launches): per panel, (A) the panel's columns are factored step by step
// (pivot search, full-row swap, scaling, rank-1 updates inside the panel),
// (B) the panel rows of the columns to the right receive the panel's
// unit-lower steps, (C) the trailing block gets its FNB updates per element
// from shared-memory copies of L21 and U12. Every element still receives
// fma(-l_ik, u_kj, a_ij) in ascending k: bitwise equal to lu_kernel. The
// trailing block is read and written once per panel instead of once per step.
constexpr int FNB = 16;
__global__ void __launch_bounds__(NT, 1) lu_fused_kernel(const LuJob* __restrict__ jobs, ErrWord* err, int tag) {
  __shared__ ValIdx red[32 + FNB];  // reduction scratch + the panel's pivots
  extern __shared__ double fsm[];
  const LuJob job = jobs[blockIdx.x];
  const Mat M = job.A;
  const int n = M.rows;
  double* lcol = fsm;                 // n
  double* Lp = lcol + n;              // FNB x n   (k-major: Lp[kk * n + i])
  double* Up = Lp + size_t(FNB) * n;  // FNB x n   (Up[kk * n + j])
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = NT / 32;
  for (int i = threadIdx.x; i < n; i += NT) job.perm[i] = i;
  ValIdx am{0.0, 0};
  for (int j = warp; j < n; j += nwarp)
    for (int i = lane; i < n; i += 32) {
      const double v = fabs(M.at(i, j));
      if (v > am.v) am.v = v;
    }
  const double amax = block_argmax(am, red).v;
  for (int kb = 0; kb < n; kb += FNB) {
    const int nb = min(FNB, n - kb);
    // (A) panel columns [kb, kb + nb), factored in shared memory: Lp holds the
    // panel's rows kb.. (column c at Lp[c * n + (i - kb)]); the row
    // interchanges are applied to the panel at once and to every other column
    // of the block after the panel (a permutation commutes with the delayed
    // updates: a row's values and multipliers still move together).
    const int pr = n - kb;
    for (int e = threadIdx.x; e < nb * pr; e += NT) {
      const int cc = e / pr, i = e % pr;
      Lp[cc * n + i] = M.at(kb + i, kb + cc);
    }
    __syncthreads();
    int* piv = reinterpret_cast<int*>(red + 32);  // FNB pivots (shared, after the reduction scratch)
    for (int k = kb; k < kb + nb; ++k) {
      const int kc = k - kb;
      double* colk = Lp + kc * n;
      ValIdx best{-1.0, 0x7fffffff};
      for (int i = kc + threadIdx.x; i < pr; i += NT) best = better(best, ValIdx{fabs(colk[i]), kb + i});
      best = block_argmax(best, red);
      if (best.v <= job.tol * amax) {
        if (threadIdx.x == 0) raise_err(err, 2, blockIdx.x, k, tag);
        return;
      }
      const int p = best.i;
      if (threadIdx.x == 0) piv[kc] = p;
      if (p != k) {
        if (threadIdx.x < nb) {
          double* cc = Lp + threadIdx.x * n;
          const double t = cc[kc];
          cc[kc] = cc[p - kb];
          cc[p - kb] = t;
        }
        if (threadIdx.x == 0) {
          const int64_t t = job.perm[k];
          job.perm[k] = job.perm[p];
          job.perm[p] = t;
        }
      }
      __syncthreads();
      const double inv = 1.0 / colk[kc];
      __syncthreads();
      for (int i = kc + 1 + threadIdx.x; i < pr; i += NT) colk[i] = colk[i] * inv;
      __syncthreads();
      for (int j = kc + 1 + warp; j < nb; j += nwarp) {
        double* colj = Lp + j * n;
        const double u = colj[kc];
        for (int i = kc + 1 + lane; i < pr; i += 32) colj[i] = fma(-colk[i], u, colj[i]);
      }
      __syncthreads();
    }
    // panel back to the block; its interchanges on every other column, in order
    for (int e = threadIdx.x; e < nb * pr; e += NT) {
      const int cc = e / pr, i = e % pr;
      M.at(kb + i, kb + cc) = Lp[cc * n + i];
    }
    for (int j = threadIdx.x; j < n; j += NT) {
      if (j >= kb && j < kb + nb) continue;
      for (int kc = 0; kc < nb; ++kc) {
        const int p = piv[kc];
        if (p != kb + kc) {
          const double t = M.at(kb + kc, j);
          M.at(kb + kc, j) = M.at(p, j);
          M.at(p, j) = t;
        }
      }
    }
    __syncthreads();
    const int c0 = kb + nb, r = n - c0;
    if (r <= 0) break;
    // (B) panel rows of the columns to the right: one thread per column, k ascending
    for (int j = c0 + threadIdx.x; j < n; j += NT) {
      double x[FNB];
#pragma unroll
      for (int i = 0; i < FNB; ++i) x[i] = i < nb ? M.at(kb + i, j) : 0.0;
#pragma unroll
      for (int kk = 0; kk < FNB; ++kk) {
        const double u = x[kk];
#pragma unroll
        for (int i = kk + 1; i < FNB; ++i)
          if (i < nb) x[i] = fma(-M.at(kb + i, kb + kk), u, x[i]);
      }
#pragma unroll
      for (int i = 0; i < FNB; ++i)
        if (i < nb) {
          M.at(kb + i, j) = x[i];
          Up[i * n + (j - c0)] = x[i];
        }
    }
    for (int e = threadIdx.x; e < nb * r; e += NT) {
      const int kk = e / r, i = e % r;
      Lp[kk * n + i] = M.at(c0 + i, kb + kk);
    }
    __syncthreads();
    // (C) trailing block: nb ordered updates per element
    for (int j = warp; j < r; j += nwarp)
      for (int i = lane; i < r; i += 32) {
        double v = M.at(c0 + i, c0 + j);
        for (int kk = 0; kk < nb; ++kk) v = fma(-Lp[kk * n + i], Up[kk * n + j], v);
        M.at(c0 + i, c0 + j) = v;
      }
    __syncthreads();
  }
}

// ---- blocked LU for large blocks (the top system) ---------------------------
// Right-looking, panels of LU_NB columns: (1) lu_panel_kernel factors columns
// [kb, kb+nb) on one CTA (pivot search, full-row swap over all n columns,
// reciprocal scaling, in-panel rank-1 updates), (2) lu_rows_kernel applies
// the panel's unit-lower steps to the panel rows of the columns to the right
// (one thread per column, k ascending), (3) a DMMA GEMM does the trailing
// update A22 = fma(L21, -U12, A22) with k ascending. Every element receives
// the reference's updates fma(-l_ik, u_kj, a_ij) in ascending k (linalg.cpp:
// 352-388): a row swap only moves a row's values and its multipliers
// together, so delaying the right-hand columns' updates to the GEMM does not
// change any element's sequence. Results equal lu_kernel's bit for bit.
__global__ void __launch_bounds__(1024) lu_panel_kernel(const LuJob* __restrict__ jobs, int kb, int nb_max,
                                                        const double* __restrict__ amax_p, ErrWord* err,
                                                        int tag) {
  const LuJob job = jobs[blockIdx.x];
  const double amax = amax_p[blockIdx.x];
  __shared__ ValIdx red[32];
  extern __shared__ double lcol[];
  const Mat M = job.A;
  const int n = M.rows;
  if (kb >= n) return;  // a smaller block of the batch: already finished
  const int nb = min(nb_max, n - kb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int k = kb; k < kb + nb; ++k) {
    ValIdx best{-1.0, 0x7fffffff};
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) best = better(best, ValIdx{fabs(M.at(i, k)), i});
    best = block_argmax(best, red);
    if (best.v <= job.tol * amax) {
      if (threadIdx.x == 0) raise_err(err, 2, int(blockIdx.x), k, tag);
      return;
    }
    const int p = best.i;
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double t = M.at(k, j);
        M.at(k, j) = M.at(p, j);
        M.at(p, j) = t;
      }
      if (threadIdx.x == 0) {
        const int64_t t = job.perm[k];
        job.perm[k] = job.perm[p];
        job.perm[p] = t;
      }
      __syncthreads();
    }
    const double inv = 1.0 / M.at(k, k);
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
      const double l = M.at(i, k) * inv;
      M.at(i, k) = l;
      lcol[i] = l;
    }
    __syncthreads();
    for (int j = k + 1 + warp; j < kb + nb; j += nwarp) {
      const double u = M.at(k, j);
      for (int i = k + 1 + lane; i < n; i += 32) M.at(i, j) = fma(-lcol[i], u, M.at(i, j));
    }
    __syncthreads();
  }
}

// Panel rows [kb, kb+nb) of the columns j >= kb + nb: a_ij -= l_ik u_kj for
// k ascending, i in (k, kb+nb). One thread per column, values in registers.
__global__ void __launch_bounds__(128) lu_rows_kernel(const LuJob* __restrict__ jobs, int kb, int nb_max) {
  __shared__ double lblk[32 * 33];
  const LuJob job = jobs[blockIdx.y];
  const Mat M = job.A;
  const int n = M.rows;
  if (kb >= n) return;
  const int nb = min(nb_max, n - kb);
  if (kb + nb + int(blockIdx.x * blockDim.x) >= n) return;  // (uniform per CTA)
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int i = e % 32, kk = e / 32;
    lblk[kk * 33 + i] = (i < nb && kk < nb) ? M.at(kb + i, kb + kk) : 0.0;
  }
  __syncthreads();
  const int j = kb + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < nb ? M.at(kb + i, j) : 0.0;
#pragma unroll
  for (int kk = 0; kk < 32; ++kk) {
    const double u = x[kk];
#pragma unroll
    for (int i = kk + 1; i < 32; ++i)
      if (i < nb) x[i] = fma(-lblk[kk * 33 + i], u, x[i]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < nb) M.at(kb + i, j) = x[i];
}

__global__ void lu_amax_kernel(const LuJob* __restrict__ jobs, double* out_all) {
  __shared__ ValIdx red[32];
  const LuJob job = jobs[blockIdx.x];
  double* out = out_all + blockIdx.x;
  const Mat M = job.A;
  const int n = M.rows;
  ValIdx am{0.0, 0};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < n; j += blockDim.x / 32)
    for (int i = lane; i < n; i += 32) {
      const double v = fabs(M.at(i, j));
      if (v > am.v) am.v = v;
    }
  am = block_argmax(am, red);
  if (threadIdx.x == 0) *out = am.v;
  for (int i = threadIdx.x; i < n; i += blockDim.x) job.perm[i] = i;
}

// Dot products of the reference's solve_transpose_in_place (linalg.cpp:487-495)
// as GCC -O3 -mavx2 -mfma vectorises them: products of each 4-wide group are
// rounded and added in order (no FMA), a trailing pair likewise, and an odd
// last element is fused (vfmadd231sd). Verified against the compiled
// reference for every trip count (tests/test_gpu_parity.py).
__device__ __forceinline__ double gcc_dot_h(const Mat& A, int i0, int col, const double* x,
                                            int tc) {
  double s = 0.0;
  const int v4 = tc & ~3;
  int i = 0;
  for (; i < v4; ++i) s = s + A.at(i0 + i, col) * x[i0 + i];
  if ((tc & 3) >= 2) {
    s = s + A.at(i0 + i, col) * x[i0 + i];
    s = s + A.at(i0 + i + 1, col) * x[i0 + i + 1];
    i += 2;
  }
  if (tc & 1) s = fma(A.at(i0 + i, col), x[i0 + i], s);
  return s;
}

// xs is chunk-local column-major: xs[c * m + i] (left) / xs[j * nr + r] (right).
__global__ void __launch_bounds__(256) solve_kernel(const SolveJob* __restrict__ jobs,
                                                    const SolveChunk* __restrict__ chunks) {
  extern __shared__ double xs[];
  const SolveChunk ch = chunks[blockIdx.x];
  const SolveJob job = jobs[ch.job];
  const Mat L = job.lu;
  const int m = L.rows;
  const int nc = ch.nc;
  const int tid = threadIdx.x, nt = blockDim.x;
  const Mat X = job.X;
  const bool right = job.kind >= SOLVE_RIGHT;

  if (!right) {
    const bool perm_in = job.kind == SOLVE_FULL || job.kind == SOLVE_LOWER;
    for (int e = tid; e < m * nc; e += nt) {
      const int i = e % m, c = e / m;
      xs[c * m + i] = X.at(perm_in ? job.perm[i] : i, ch.c0 + c);
    }
    __syncthreads();
    if (job.kind == SOLVE_TRANSPOSE) {
      // A = P^T L U: U^T w = b, L^T v = w, x = P^T v (linalg.cpp:479-503).
      for (int c = tid; c < nc; c += nt) {
        double* x = xs + c * m;
        for (int k = 0; k < m; ++k) {
          const double dot = gcc_dot_h(L, 0, k, x, k);
          x[k] = (x[k] - dot) / L.at(k, k);
        }
        for (int k = m - 1; k >= 0; --k) {
          const double dot = gcc_dot_h(L, k + 1, k, x, m - k - 1);
          x[k] = x[k] - dot;
        }
      }
      __syncthreads();
      for (int e = tid; e < m * nc; e += nt) {
        const int i = e % m, c = e / m;
        X.at(job.perm[i], ch.c0 + c) = xs[c * m + i];
      }
      return;
    }
    if (job.kind != SOLVE_UPPER) {
      // Forward, unit lower: x[i] -= L(i,k) * x[k].
      for (int k = 0; k < m - 1; ++k) {
        const int t = m - k - 1;
        for (int e = tid; e < t * nc; e += nt) {
          const int i = k + 1 + e % t, c = e / t;
          xs[c * m + i] = fma(-L.at(i, k), xs[c * m + k], xs[c * m + i]);
        }
        __syncthreads();
      }
    }
    if (job.kind != SOLVE_LOWER) {
      // Backward: x[k] /= U(k,k); x[i] -= U(i,k) * x[k] for i < k.
      for (int k = m - 1; k >= 0; --k) {
        const double ukk = L.at(k, k);
        for (int e = tid; e < (k + 1) * nc; e += nt) {
          const int i = e % (k + 1), c = e / (k + 1);
          const double xk = xs[c * m + k] / ukk;
          if (i < k) xs[c * m + i] = fma(-L.at(i, k), xk, xs[c * m + i]);
        }
        __syncthreads();
        for (int c = tid; c < nc; c += nt) xs[c * m + k] = xs[c * m + k] / ukk;
        __syncthreads();
      }
    }
    for (int e = tid; e < m * nc; e += nt) {
      const int i = e % m, c = e / m;
      X.at(i, ch.c0 + c) = xs[c * m + i];
    }
    return;
  }

  // Right solves over a chunk of X rows [c0, c0 + nc).
  const int nr = nc;
  for (int e = tid; e < m * nr; e += nt) {
    const int r = e % nr, j = e / nr;
    xs[j * nr + r] = X.at(ch.c0 + r, j);
  }
  __syncthreads();
  // X <- X U^-1 (linalg.cpp:441-451 / :547-557).
  for (int k = 0; k < m; ++k) {
    const double inv = 1.0 / L.at(k, k);
    for (int r = tid; r < nr; r += nt) xs[k * nr + r] = xs[k * nr + r] * inv;
    __syncthreads();
    const int t = m - k - 1;
    for (int e = tid; e < t * nr; e += nt) {
      const int r = e % nr, j = k + 1 + e / nr;
      const double ukj = L.at(k, j);
      if (ukj != 0.0) xs[j * nr + r] = fma(-ukj, xs[k * nr + r], xs[j * nr + r]);
    }
    __syncthreads();
  }
  if (job.kind == SOLVE_RIGHT) {
    // X <- X L^-1, then undo the row permutation on the columns.
    for (int k = m - 1; k >= 1; --k) {
      for (int e = tid; e < k * nr; e += nt) {
        const int r = e % nr, j = e / nr;
        const double lkj = L.at(k, j);
        if (lkj != 0.0) xs[j * nr + r] = fma(-lkj, xs[k * nr + r], xs[j * nr + r]);
      }
      __syncthreads();
    }
    for (int e = tid; e < m * nr; e += nt) {
      const int r = e % nr, k = e / nr;
      X.at(ch.c0 + r, job.perm[k]) = xs[k * nr + r];
    }
    return;
  }
  for (int e = tid; e < m * nr; e += nt) {
    const int r = e % nr, j = e / nr;
    X.at(ch.c0 + r, j) = xs[j * nr + r];
  }
}

// One diagonal block of a blocked left triangular solve, for every RHS
// column (one thread per column; the nb x nb factor block staged in shared
// memory). lower: unit-lower forward steps k in [kb, kb+nb); upper: divide and
// backward steps k from kb+nb-1 down to kb. Together with the GEMM updates
// between blocks (accumulated in the same k order) every element sees the
// reference's exact update sequence (linalg.cpp:404-542).
__global__ void __launch_bounds__(128) trsm_block_kernel(const TrsmBlockJob* __restrict__ jobs,
                                                         const int2* __restrict__ tiles) {
  __shared__ double blk[32 * 32];
  const int2 t = tiles[blockIdx.x];
  const TrsmBlockJob job = jobs[t.x];
  const int kb = job.kb, nb = job.nb;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, kk = e / nb;
    blk[kk * 32 + i] = job.lu.at(kb + i, kb + kk);
  }
  __syncthreads();
  const int c = t.y * blockDim.x + threadIdx.x;
  if (c >= job.X.cols) return;
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < nb ? job.X.at(kb + i, c) : 0.0;
  if (job.lower) {
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) {
      if (kk >= nb) break;
      const double xk = x[kk];
#pragma unroll
      for (int i = kk + 1; i < 32; ++i)
        if (i < nb) x[i] = fma(-blk[kk * 32 + i], xk, x[i]);
    }
  } else {
#pragma unroll
    for (int kk = 31; kk >= 0; --kk) {
      if (kk >= nb) continue;
      x[kk] = x[kk] / blk[kk * 32 + kk];
      const double xk = x[kk];
#pragma unroll
      for (int i = 0; i < kk; ++i) x[i] = fma(-blk[kk * 32 + i], xk, x[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < nb) job.X.at(kb + i, c) = x[i];
}


// Fused blocked left solve for wide right-hand sides (SOLVE_FULL / LOWER /
// UPPER): one CTA per (job, 32-column chunk of X); the chunk lives in shared
// memory for the whole solve, so X is read and written once (the previous
// path re-read the rows below / above every 32-row block from HBM through a
// GEMM launch per block). Per 32-row diagonal block: warp 0 solves the block
// with one lane per column (registers, the 32 x 32 factor block staged in
// shared memory), then every warp updates 32-row groups of the remaining rows
// with one lane per row, the row's factor segment in registers and the
// block's solved values broadcast from shared memory. Each element sees the
// reference's update sequence: forward fma(-L(i,k), x_k, x_i) for k ascending,
// backward k descending then the division (linalg.cpp:404-542) — the same
// sequence the GEMM-update path produced, so results are bitwise unchanged.
constexpr int TRSM_NC = 32;

__global__ void __launch_bounds__(256, 2) trsm_chunk_kernel(const SolveJob* __restrict__ jobs,
                                                            const int2* __restrict__ tiles) {
  extern __shared__ double xs[];  // [TRSM_NC][ldx]
  __shared__ double blk[32 * 33];
  const int2 t = tiles[blockIdx.x];
  const SolveJob job = jobs[t.x];
  const Mat L = job.lu;
  const Mat X = job.X;
  const int m = L.rows;
  const int ldx = m | 1;  // odd stride: lane-per-column accesses are conflict-free
  const int c0 = t.y * TRSM_NC;
  const int nc = min(TRSM_NC, X.cols - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool perm_in = job.kind == SOLVE_FULL || job.kind == SOLVE_LOWER;
  for (int e = threadIdx.x; e < m * TRSM_NC; e += blockDim.x) {
    const int i = e % m, c = e / m;
    xs[c * ldx + i] = c < nc ? X.at(perm_in ? job.perm[i] : i, c0 + c) : 0.0;
  }
  __syncthreads();
  const int nblk = (m + 31) / 32;
  if (job.kind != SOLVE_UPPER) {
    for (int b = 0; b < nblk; ++b) {
      const int kb = b * 32, nb = min(32, m - kb);
      for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int i = e % 32, kk = e / 32;
        blk[kk * 33 + i] = (i < nb && kk < nb) ? L.at(kb + i, kb + kk) : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        double* col = xs + lane * ldx + kb;
        double x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = i < nb ? col[i] : 0.0;
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) {
          const double xk = x[kk];
#pragma unroll
          for (int i = kk + 1; i < 32; ++i)
            if (i < nb) x[i] = fma(-blk[kk * 33 + i], xk, x[i]);  // rows/cols >= nb are zero-padded
        }
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nb) col[i] = x[i];
      }
      __syncthreads();
      // rows below the block: (32-row group, 8-column group) items round-robin
      // over the warps; a lane owns a row and runs 8 independent column chains.
      {
        const int rbeg = kb + nb, ng = (m - rbeg + 31) / 32, ncg = (nc + 7) / 8;
        for (int it = warp; it < ng * ncg; it += nw) {
          const int i = rbeg + (it / ncg) * 32 + lane, cb = (it % ncg) * 8;
          if (i < m) {
            double l[32];
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) l[kk] = kk < nb ? L.at(i, kb + kk) : 0.0;
            double acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = xs[(cb + q) * ldx + i];
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
              if (kk < nb) {
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[q] = fma(-l[kk], xs[(cb + q) * ldx + kb + kk], acc[q]);
              }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (cb + q < nc) xs[(cb + q) * ldx + i] = acc[q];
          }
        }
      }
      __syncthreads();
    }
  }
  if (job.kind != SOLVE_LOWER) {
    for (int b = nblk - 1; b >= 0; --b) {
      const int kb = b * 32, nb = min(32, m - kb);
      for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int i = e % 32, kk = e / 32;
        blk[kk * 33 + i] = (i < nb && kk < nb) ? L.at(kb + i, kb + kk) : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        double* col = xs + lane * ldx + kb;
        double x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = i < nb ? col[i] : 0.0;
#pragma unroll
        for (int kk = 31; kk >= 0; --kk) {
          if (kk < nb) {
            x[kk] = x[kk] / blk[kk * 33 + kk];
            const double xk = x[kk];
#pragma unroll
            for (int i = 0; i < kk; ++i) x[i] = fma(-blk[kk * 33 + i], xk, x[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nb) col[i] = x[i];
      }
      __syncthreads();
      // rows above the block (k descending), same work split as the forward sweep
      {
        const int ng = (kb + 31) / 32, ncg = (nc + 7) / 8;
        for (int it = warp; it < ng * ncg; it += nw) {
          const int i = (it / ncg) * 32 + lane, cb = (it % ncg) * 8;
          if (i < kb) {
            double u[32];
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) u[kk] = kk < nb ? L.at(i, kb + kk) : 0.0;
            double acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = xs[(cb + q) * ldx + i];
#pragma unroll
            for (int kk = 31; kk >= 0; --kk) {
              if (kk < nb) {
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[q] = fma(-u[kk], xs[(cb + q) * ldx + kb + kk], acc[q]);
              }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (cb + q < nc) xs[(cb + q) * ldx + i] = acc[q];
          }
        }
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < m * nc; e += blockDim.x) {
    const int i = e % m, c = e / m;
    X.at(i, c0 + c) = xs[c * ldx + i];
  }
}

__global__ void gather_rows_kernel(const GatherJob* __restrict__ jobs, const int2* __restrict__ tiles) {
  const int2 t = tiles[blockIdx.x];
  const GatherJob job = jobs[t.x];
  const int64_t e0 = int64_t(t.y) * 4096;
  const int64_t tot = int64_t(job.dst.rows) * job.dst.cols;
  for (int64_t e = e0 + threadIdx.x; e < min(tot, e0 + 4096); e += blockDim.x) {
    const int i = int(e % job.dst.rows), j = int(e / job.dst.rows);
    job.dst.at(i, j) = job.src.at(job.perm[i], j);
  }
}

}  // namespace

void launch_trsm_block(const TrsmBlockJob* jobs, const int2* tiles, int ntiles, cudaStream_t st) {
  if (ntiles > 0) trsm_block_kernel<<<ntiles, 128, 0, st>>>(jobs, tiles);
}

void launch_trsm_chunk(const SolveJob* jobs, const int2* tiles, int ntiles, int max_m, cudaStream_t st) {
  if (ntiles <= 0) return;
  const size_t smem = sizeof(double) * size_t(TRSM_NC) * size_t(max_m | 1);
  // static shared memory (blk) counts against the 48 KB default too
  smem_attr((const void*)trsm_chunk_kernel, smem, "trsm_chunk smem attribute");
  trsm_chunk_kernel<<<ntiles, 256, smem, st>>>(jobs, tiles);  // errors surface at the caller's check
}

int trsm_chunk_cols() { return TRSM_NC; }

void launch_gather_rows(const GatherJob* jobs, const int2* tiles, int ntiles, cudaStream_t st) {
  if (ntiles > 0) gather_rows_kernel<<<ntiles, 256, 0, st>>>(jobs, tiles);
}

void launch_lu_amax(const LuJob* jobs, int njobs, double* out, cudaStream_t st) {
  lu_amax_kernel<<<njobs, 1024, 0, st>>>(jobs, out);
}

void launch_lu_panel(const LuJob* jobs, int njobs, int max_n, int kb, int nb, const double* amax, ErrWord* err,
                     int tag, cudaStream_t st) {
  const size_t smem = sizeof(double) * size_t(max_n);
  smem_attr((const void*)lu_panel_kernel, smem, "lu_panel smem attribute");
  lu_panel_kernel<<<njobs, 1024, smem, st>>>(jobs, kb, nb, amax, err, tag);
}

void launch_lu_rows(const LuJob* jobs, int njobs, int max_n, int kb, int nb, cudaStream_t st) {
  const int ncols = max_n - kb - nb;
  if (ncols > 0) lu_rows_kernel<<<dim3((ncols + 127) / 128, njobs), 128, 0, st>>>(jobs, kb, nb);
}

void launch_lu(const LuJob* jobs, int njobs, int max_n, ErrWord* err, int tag, cudaStream_t st) {
  if (njobs <= 0) return;
  static const bool unfused = getenv("H2G_LU_UNFUSED") != nullptr;
  const size_t fsmem = sizeof(double) * size_t(max_n > 0 ? max_n : 1) * (1 + 2 * FNB);
  if (!unfused && max_n >= 48 && fsmem <= size_t(200) << 10) {
    smem_attr((const void*)lu_fused_kernel, fsmem, "lu_fused smem attribute");
    lu_fused_kernel<<<njobs, NT, fsmem, st>>>(jobs, err, tag);
    return;
  }
  const size_t smem = sizeof(double) * size_t(max_n > 0 ? max_n : 1);
  smem_attr((const void*)lu_kernel, smem, "lu smem attribute");
  lu_kernel<<<njobs, NT, smem, st>>>(jobs, err, tag);
}

int solve_chunk_width(int m) {
  int w = 24000 / (m > 0 ? m : 1);
  if (w > 256) w = 256;
  return w < 1 ? 1 : w;
}

void launch_solve(const SolveJob* jobs, const SolveChunk* chunks, int nchunks,
                  size_t smem_doubles, cudaStream_t st) {
  if (nchunks <= 0) return;
  const size_t smem = sizeof(double) * (smem_doubles > 0 ? smem_doubles : 1);
  smem_attr((const void*)solve_kernel, 227 * 1024, "solve smem attribute");
  solve_kernel<<<nchunks, 256, smem, st>>>(jobs, chunks);
}

}  // namespace h2g
