// Batched column-pivoted Householder QR with the member-mass stopping rule,
// followed by full Q formation: run_pivoted_qr + form_q (linalg.cpp:137-185,
// :216-332) as driven by basis_from_members (compression.cpp:111-146).
//
// One thread-block cluster per basis; the working copy R is column-major in
// HBM and streamed through shared memory once per Householder step. Each
// column's reflector dot product runs sequentially over rows in one lane,
// exactly as the reference; column norms, downdates, the 4e-15 tie rule,
// the member masses and the stopping tests all follow the reference's
// operation order, so ranks and Q are bitwise equal to the reference's.
#include <cooperative_groups.h>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace h2g {

void cuda_check(cudaError_t e, const char* what);  // batch.cu

namespace {

constexpr int NT = 128;

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
  double* sq;  // rkj^2 of the current step, by position
  int* piv;   // position -> original column
  int* grp;   // original column -> member (static)
  double* mm;
  double* mt;
  double* pn2;  // pivot column's norm^2 at each step (after the swap)
  int* swp;     // pivot position selected at each step
  double* V;
  double* tau;
};

__host__ __device__ inline Scratch carve(double* s, int m, int n, int nmem) {
  const int kmax0 = m < n ? m : n;
  Scratch c;
  c.cn2 = s;
  c.cn2o = s + n;
  c.piv = reinterpret_cast<int*>(s + 2 * int64_t(n));
  c.grp = c.piv + n;
  c.sq = s + 3 * int64_t(n);
  c.mm = s + 4 * int64_t(n);
  c.mt = c.mm + nmem;
  c.pn2 = c.mt + nmem;
  c.swp = reinterpret_cast<int*>(c.pn2 + kmax0);  // [0, kmax0): list D, [kmax0, 2 kmax0): pivots
  c.tau = c.pn2 + 2 * int64_t(kmax0);
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

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void st_global16(double* p, double x, double y) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(x), "d"(y) : "memory");
}

// red_h (above) over a shared-memory column against v, streamed as 16-byte
// pairs: element t is col[off + t] * vb[off + t], t < tc, with col and vb
// 16-byte aligned and off in {0, 1}. Every element is a rounded product
// added in order except an odd last one, which is fused.
__device__ __forceinline__ double dot_h_pairs(const double* __restrict__ col,
                                              const double* __restrict__ vb, int off, int tc) {
  double s = 0.0;
  if (tc <= 0) return s;
  const bool lastf = tc & 1;
  const int nu = lastf ? tc - 1 : tc;
  int t = 0;
  if (off == 1 && nu >= 1) {
    s = s + col[1] * vb[1];
    t = 1;
  }
  const double2* c2 = reinterpret_cast<const double2*>(col + off + t);
  const double2* v2 = reinterpret_cast<const double2*>(vb + off + t);
  const int npair = (nu - t) >> 1;
  int q = 0;
  for (; q + 4 <= npair; q += 4) {
    double2 x[4], y[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      x[w] = c2[q + w];
      y[w] = v2[q + w];
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      s = s + x[w].x * y[w].x;
      s = s + x[w].y * y[w].y;
    }
  }
  for (; q < npair; ++q) {
    const double2 x = c2[q], y = v2[q];
    s = s + x.x * y.x;
    s = s + x.y * y.y;
  }
  t += 2 * npair;
  if (t < nu) {
    s = s + col[off + t] * vb[off + t];
    ++t;
  }
  if (lastf) s = fma(col[off + t], vb[off + t], s);
  return s;
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}

// Column ownership inside a cluster: blocks of CB consecutive positions go
// round-robin to the G CTAs (owner = (j / CB) % G). A CTA walks its own
// positions through a dense local index li.
constexpr int CB = 256;
struct Own {
  int G, cr;
  __device__ __forceinline__ int l2g(int li) const {
    return ((li / CB) * G + cr) * CB + li % CB;
  }
  // Number of own positions < x.
  __device__ __forceinline__ int below(int x) const {
    const int bx = x / CB;
    int c = bx > cr ? ((bx - cr + G - 1) / G) * CB : 0;
    if (bx % G == cr) c += x % CB;
    return c;
  }
};

// Member-mass downdates of one step (linalg.cpp:312-321), lead CTA. Members
// are contiguous ranges of original columns and position j initially holds
// column j; only pivot swaps displace columns, so the positions (> s) where
// a column of another member sits form a short sorted list D (positions Dp,
// their columns' members Dg, both in shared memory). Each thread owns whole
// members and runs each member's chain over its range (skipping D) merged
// with its displaced columns, i.e. in the reference's position order; the
// range's rkj^2 are fetched eight at a time ahead of the dependent chain.
__device__ __forceinline__ double mass_sub(double val, double x) {
  const double v = val - x;
  return v < 0.0 ? 0.0 : v;
}
__device__ void member_step(const double* __restrict__ sq, int s, int nmem, const int64_t* off,
                            const int* Dp, const int* Dg, int nd, double* mmsh) {
  for (int g = threadIdx.x; g < nmem; g += NT) {
    const int a = max(s + 1, int(off[g])), b = int(off[g + 1]);
    double val = mmsh[g];
    int p = 0;
    for (; p < nd && Dp[p] < a; ++p)
      if (Dg[p] == g) val = mass_sub(val, __ldcg(&sq[Dp[p]]));
    int nextd = p < nd ? Dp[p] : 0x7fffffff;
    for (int j0 = a; j0 < b; j0 += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = j0 + u < b ? __ldcg(&sq[j0 + u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        if (j < b) {
          if (j == nextd) {
            ++p;
            nextd = p < nd ? Dp[p] : 0x7fffffff;
          } else {
            val = mass_sub(val, x[u]);
          }
        }
      }
    }
    for (; p < nd; ++p)
      if (Dp[p] >= b && Dg[p] == g) val = mass_sub(val, __ldcg(&sq[Dp[p]]));
    mmsh[g] = val;
  }
}

struct ClSlots {
  double d;
  int piv, pos;
  int flag;
};

// Cluster-split QR: the G CTAs of a thread-block cluster share one basis.
// Per Householder step: cluster-wide pivot reductions through distributed
// shared memory, the swap and the reflector by CTA 0, every CTA sweeps its
// own columns, CTA 0 runs the member-mass chains. Global data written by one
// CTA is read by the others only across cluster barriers (barrier.cluster
// release/acquire).
//
// Column sweep: each warp streams tiles of up to 32 columns through its own
// slice of shared memory. Lane c runs column c's sequential dot chain (the
// reference's rounding order), the whole warp then writes the updated
// column straight from the FMA to global memory and refills the slot with
// the next tile's column (cp.async), so loads overlap the stores.
//
// Dynamic shared memory: [ v (m) | member masses (nmem) | D (2 kmax ints) | column tiles ].
__global__ void __launch_bounds__(NT, 1) qr_kernel(const QrJob* __restrict__ jobs, int tile_doubles,
                                                   int nmem_cap, int m_cap) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double redd[32];
  __shared__ int redi[32];
  __shared__ double sh_tau;
  __shared__ int sh_nd;
  __shared__ ClSlots slot;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = int(cluster.num_blocks());
  const int cr = int(cluster.block_rank());
  const Own own{G, cr};
  const QrJob job = jobs[blockIdx.x / G];
  const int m = job.m, n = job.n, nmem = job.nmem;
  double* W = job.work;
  const int64_t ldw = job.ldw;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = NT / 32;
  const int vcap = (m_cap + 3) & ~1;  // v, plus one pad row for pair reads
  double* vsh = dsm;
  double* mmsh = dsm + vcap;
  int* Dp = reinterpret_cast<int*>(mmsh + nmem_cap);
  int* Dg = Dp + m_cap;
  double* T = dsm + ((vcap + m_cap + nmem_cap + 1) & ~1);  // 16-byte aligned tiles
  Scratch S = carve(job.scratch, m, n, nmem);
  const int kmax0 = m < n ? m : n;
  int kmax = kmax0;
  if (job.cap > 0 && job.cap < kmax) kmax = job.cap;
  const bool lead = cr == 0;
  const int nloc = own.below(n);

  // R = A (skipped when factoring in place): own columns.
  if (!(job.A.p == W && job.A.rs == 1 && job.A.cs == ldw)) {
    for (int li = 0; li < nloc; ++li) {
      const int j = own.l2g(li);
      for (int i = tid; i < m; i += NT) W[int64_t(j) * ldw + i] = job.A.at(i, j);
    }
    __syncthreads();
  }
  // Column norms of own columns (pattern P2 over all rows), tile by tile.
  {
    const int pitch = m | 1;
    const int twmax = max(1, min(NT, tile_doubles / pitch));
    for (int l0 = 0; l0 < nloc; l0 += twmax) {
      const int tw = min(twmax, nloc - l0);
      for (int c = warp; c < tw; c += NW) {
        const double* src = W + int64_t(own.l2g(l0 + c)) * ldw;
        for (int r = lane; r < m; r += 32) cp_async8(T + c * pitch + r, src + r);
      }
      cp_async_wait_all();
      __syncthreads();
      if (tid < tw) {
        const int j = own.l2g(l0 + tid);
        const double* col = T + tid * pitch;
        const double s = red_p2([&](int i, double& a, double& b) { a = b = col[i]; }, 0, m);
        S.cn2[j] = s;
        S.cn2o[j] = s;
        S.piv[j] = j;
      }
      __syncthreads();
    }
  }
  cluster.sync();
  const bool members = nmem >= 1;
  if (lead) {
    if (members) {
      for (int g = tid; g < nmem; g += NT) {
        double mass = 0.0;
        for (int64_t j = job.member_off[g]; j < job.member_off[g + 1]; ++j) {
          S.grp[j] = g;
          mass += S.cn2[j];
        }
        mmsh[g] = mass;
        S.mt[g] = job.member_tol * job.member_tol * mass;
      }
    }
    __syncthreads();
    int not_done = 0;
    if (members)
      for (int g = tid; g < nmem; g += NT) not_done |= (mmsh[g] > S.mt[g]);
    not_done = __syncthreads_or(not_done);
    if (tid == 0) slot.flag = not_done;
  }

  double r11 = -1.0;
  int rank = 0;
  int nd = 0;  // length of the displaced-position list D (lead CTA)
  long long t_piv = 0, t_refl = 0, t_tile = 0, t_mem = 0, t0c;
  long long t_w = 0, t_c = 0, t_s = 0, n_t = 0;
  for (int k = 0; k < kmax; ++k) {
    t0c = clock64();
    // Pivot: cluster-wide max of the remaining norms, then the lowest
    // original index within the 4e-15 tie band (linalg.cpp:263-274).
    const int lk = own.below(k);
    double mx = -1.0;
    for (int li = lk + tid; li < nloc; li += NT) mx = fmax(mx, S.cn2[own.l2g(li)]);
    mx = block_max(mx, redd);
    if (tid == 0) slot.d = mx;
    cluster.sync();
    double best = -1.0;
    for (int q = 0; q < G; ++q) best = fmax(best, cluster.map_shared_rank(&slot, q)->d);
    const int members_not_done = cluster.map_shared_rank(&slot, 0)->flag;
    if (best <= 0.0) break;
    const double tie = best * (1.0 - 4e-15);
    int cand = 0x7fffffff;
    for (int li = lk + tid; li < nloc; li += NT) {
      const int j = own.l2g(li);
      if (S.cn2[j] >= tie) cand = min(cand, S.piv[j]);
    }
    cand = block_min_int(cand, redi);
    int cpos = 0x7fffffff;
    for (int li = lk + tid; li < nloc; li += NT) {
      const int j = own.l2g(li);
      if (S.piv[j] == cand && S.cn2[j] >= tie) cpos = j;
    }
    cpos = block_min_int(cpos, redi);
    if (tid == 0) {
      slot.piv = cand;
      slot.pos = cpos;
    }
    cluster.sync();
    int sel_orig = 0x7fffffff, sel = 0x7fffffff;
    for (int q = 0; q < G; ++q) {
      const ClSlots* o = cluster.map_shared_rank(&slot, q);
      if (o->piv < sel_orig) {
        sel_orig = o->piv;
        sel = o->pos;
      }
    }
    if (lead && sel != k) {
      for (int i = tid; i < m; i += NT) {
        const double t = W[int64_t(k) * ldw + i];
        W[int64_t(k) * ldw + i] = W[int64_t(sel) * ldw + i];
        W[int64_t(sel) * ldw + i] = t;
      }
      if (tid == 0) {
        double t = S.cn2[k]; S.cn2[k] = S.cn2[sel]; S.cn2[sel] = t;
        t = S.cn2o[k]; S.cn2o[k] = S.cn2o[sel]; S.cn2o[sel] = t;
        int ti = S.piv[k]; S.piv[k] = S.piv[sel]; S.piv[sel] = ti;
      }
    }
    if (lead && tid == 0) {
      S.swp[kmax0 + k] = sel;
      S.pn2[k] = S.cn2[k];
    }
    cluster.sync();
    const double pivot_norm = sqrt(fmax(0.0, __ldcg(&S.cn2[k])));
    if (k == 0) r11 = pivot_norm;
    const bool diag_done = pivot_norm <= job.tol * r11;
    const bool floor_hit = pivot_norm <= 1e-15 * r11;
    if (floor_hit) break;
    if (diag_done && !members_not_done) break;

    t_piv += clock64() - t0c; t0c = clock64();
    // make_reflector (linalg.cpp:152-178), sequential on one thread of CTA 0.
    double* vk = S.V + int64_t(k) * m;
    double* wk = W + int64_t(k) * ldw;
    if (lead && tid == 0) {
      const double normsq = red_p2([&](int i, double& a, double& b) { a = b = wk[i]; }, k, m - k);
      const double norm = sqrt(normsq);
      for (int i = 0; i < k; ++i) vk[i] = 0.0;
      double tau = 0.0;
      if (norm == 0.0) {
        for (int i = k; i < m; ++i) vk[i] = 0.0;
      } else {
        const double a0 = wk[k];
        const double alpha = (a0 >= 0.0) ? -norm : norm;
        vk[k] = a0 - alpha;
        double vn = vk[k] * vk[k];
        for (int i = k + 1; i < m; ++i) vk[i] = wk[i];
        const int tcv = m - k - 1;
        if (tcv == 1) {
          vn = vn + vk[k + 1] * vk[k + 1];
        } else if (tcv > 1) {
          vn = red_h([&](int i, double& a, double& b) { a = b = vk[i]; }, k + 1, tcv, vn);
        }
        tau = (vn == 0.0) ? 0.0 : 2.0 / vn;
        wk[k] = alpha;
        for (int i = k + 1; i < m; ++i) wk[i] = 0.0;
      }
      S.tau[k] = tau;
    }
    cluster.sync();
    for (int i = tid; i < m; i += NT) vsh[i] = __ldcg(&vk[i]);
    if (tid == 0) sh_tau = __ldcg(&S.tau[k]);
    __syncthreads();
    const double tau = sh_tau;
    t_refl += clock64() - t0c; t0c = clock64();
    // apply_reflector to own columns k+1.. (linalg.cpp:137-149) + norm
    // downdates (linalg.cpp:300-311). Column segments move as 16-byte pairs
    // of rows [k0, m), k0 = k rounded down to even (ldw is even, so every
    // segment is 16-byte aligned); slot pitch P = 2 mod 4 doubles keeps the
    // per-lane 16-byte shared loads conflict-free.
    {
      const int rows = m - k;
      const int k0 = k & ~1, off = k - k0;
      const int np = (m - k0 + 1) >> 1;  // pairs per segment
      const int P = (np & 1) ? 2 * np : 2 * np + 2;
      const int per_warp = (tile_doubles / NW) & ~1;
      const int cw = max(1, min(32, per_warp / P));
      double* Tw = T + warp * per_warp;
      // Store pairs start at k1 = (k + 1) rounded down to even: row k (R's
      // final row k, never read again) may be rewritten with its own value.
      const int k1 = (k + 1) & ~1;
      const int nps = (m - k1 + 1) >> 1;
      const double* vb = vsh + k0;
      double2 vr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = lane + 32 * u;
        vr[u] = p < nps ? *reinterpret_cast<const double2*>(vsh + k1 + 2 * p) : make_double2(0.0, 0.0);
      }
      const int l0 = own.below(k + 1);
      auto load_col = [&](int slotc, int j) {
        const double* src = W + int64_t(j) * ldw + k0;
        double* dst = Tw + slotc * P;
        if (np <= 128) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int p = lane + 32 * u;
            if (p < np) cp_async16(dst + 2 * p, src + 2 * p);
          }
        } else {
          for (int p = lane; p < np; p += 32) cp_async16(dst + 2 * p, src + 2 * p);
        }
      };
      int a = l0 + warp * cw;
      if (a < nloc) {
        const int tw = min(cw, nloc - a);
        for (int c = 0; c < tw; ++c) load_col(c, own.l2g(a + c));
      }
      for (; a < nloc; a += NW * cw) {
        const int tw = min(cw, nloc - a);
        long long c0 = clock64();
        cp_async_wait_all();
        __syncwarp();
        long long c1 = clock64();
        double sc = 0.0;
        int jl = 0;
        if (lane < tw) {
          jl = own.l2g(a + lane);
          const double cn2j = S.cn2[jl], cn2oj = S.cn2o[jl];  // in flight during the chain
          const double* col = Tw + lane * P;
          if (tau != 0.0) sc = -(tau * dot_h_pairs(col, vb, off, rows));
          // GCC computes rkj*rkj once (rounded) for the norm and member downdates.
          const double rkj = tau != 0.0 ? fma(sc, vsh[k], col[off]) : col[off];
          const double sq = rkj * rkj;
          double upd = cn2j - sq;
          if (upd < 1e-8 * cn2oj)
            upd = red_p2(
                [&](int r, double& x, double& y) {
                  x = y = tau != 0.0 ? fma(sc, vsh[k + r], col[off + r]) : col[off + r];
                },
                1, rows - 1);
          S.cn2[jl] = fmax(0.0, upd);
          S.sq[jl] = sq;
        }
        __syncwarp();
        long long c2 = clock64();
        const int an = a + NW * cw;
        const int twn = an < nloc ? min(cw, nloc - an) : 0;
        for (int c = 0; c < tw; ++c) {
          const double s_c = __shfl_sync(0xffffffffu, sc, c);
          const int j = __shfl_sync(0xffffffffu, jl, c);
          const double* colc = Tw + c * P + (k1 - k0);
          if (tau != 0.0) {
            double* dst = W + int64_t(j) * ldw + k1;
            if (nps <= 128) {
              double2 x[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int p = lane + 32 * u;
                x[u] = p < nps ? *reinterpret_cast<const double2*>(colc + 2 * p) : make_double2(0.0, 0.0);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int p = lane + 32 * u;
                if (p < nps)
                  st_global16(dst + 2 * p, fma(s_c, vr[u].x, x[u].x), fma(s_c, vr[u].y, x[u].y));
              }
            } else {
              for (int p = lane; p < nps; p += 32) {
                const double2 x = *reinterpret_cast<const double2*>(colc + 2 * p);
                const double2 v = *reinterpret_cast<const double2*>(vsh + k1 + 2 * p);
                st_global16(dst + 2 * p, fma(s_c, v.x, x.x), fma(s_c, v.y, x.y));
              }
            }
          }
          if (c < twn) load_col(c, own.l2g(an + c));
        }
        for (int c = tw; c < twn; ++c) load_col(c, own.l2g(an + c));
        long long c3 = clock64();
        t_w += c1 - c0; t_c += c2 - c1; t_s += c3 - c2; ++n_t;
      }
      cp_async_wait_all();
    }
    cluster.sync();
    t_tile += clock64() - t0c; t0c = clock64();
    ++rank;
    if (lead && members) {
      // D: positions > k holding a column of another member (sorted). The
      // swap of step k moved the column from position k to position sel.
      if (tid == 0) {
        const int sel = S.swp[kmax0 + k];
        int w = 0;
        for (int q = 0; q < nd; ++q)
          if (Dp[q] > k && Dp[q] != sel) {
            Dp[w] = Dp[q];
            Dg[w] = Dg[q];
            ++w;
          }
        const int gs = S.grp[S.piv[sel]];
        if (sel > k && gs != S.grp[sel]) {
          int q = w;
          while (q > 0 && Dp[q - 1] > sel) {
            Dp[q] = Dp[q - 1];
            Dg[q] = Dg[q - 1];
            --q;
          }
          Dp[q] = sel;
          Dg[q] = gs;
          ++w;
        }
        sh_nd = w;
      }
      __syncthreads();
      nd = sh_nd;
      member_step(S.sq, k, nmem, job.member_off, Dp, Dg, nd, mmsh);
      __syncthreads();
      if (tid == 0) {
        const int gk = S.grp[S.piv[k]];
        mmsh[gk] = mass_sub(mmsh[gk], S.pn2[k]);
      }
      __syncthreads();
      int not_done = 0;
      for (int g = tid; g < nmem; g += NT) not_done |= (mmsh[g] > S.mt[g]);
      not_done = __syncthreads_or(not_done);
      if (tid == 0) slot.flag = not_done;
    }
    t_mem += clock64() - t0c;
  }
  // No CTA may leave while others can still read its slots.
  cluster.sync();
  if (!lead) return;
  if (tid == 0 && job.dbg) {
    job.dbg[0] = double(t_piv); job.dbg[1] = double(t_refl); job.dbg[2] = double(t_tile);
    job.dbg[3] = double(t_mem); job.dbg[4] = double(rank); job.dbg[5] = double(n);
    job.dbg[8] = double(t_w); job.dbg[9] = double(t_c); job.dbg[10] = double(t_s); job.dbg[11] = double(n_t);
  }
  long long tq = clock64();

  // form_q (linalg.cpp:181-185): Q = I, reflectors applied backward.
  double* Q = job.Q;
  for (int64_t e = tid; e < int64_t(m) * m; e += NT) Q[e] = (e / m == e % m) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = rank - 1; k >= 0; --k) {
    const double tau = __ldcg(&S.tau[k]);
    if (tau == 0.0) continue;
    const double* vk = S.V + int64_t(k) * m;
    for (int i = tid; i < m; i += NT) vsh[i] = __ldcg(&vk[i]);
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
  if (tid == 0 && job.dbg) job.dbg[6] = double(clock64() - tq);
}

size_t qr_fixed_doubles(int max_m, int max_nmem) {
  return size_t((((max_m + 3) & ~1) + max_m + max_nmem + 1) & ~1);
}

// Dynamic shared memory per CTA: H2G_QR_SMEM_KB (default 110, two CTAs per
// SM; the column tiles take everything past the fixed part).
size_t qr_smem_bytes(int max_m, int max_nmem, size_t* tile_doubles) {
  static const size_t budget = [] {
    const char* e = getenv("H2G_QR_SMEM_KB");
    return size_t(std::min(e ? atoi(e) : 110, 220)) * 1024;
  }();
  const size_t fixed = qr_fixed_doubles(max_m, max_nmem);
  size_t tile = budget / sizeof(double) > fixed + 1024 ? budget / sizeof(double) - fixed : 1024;
  // Every warp needs at least one column slot (pitch <= max_m + 4).
  const size_t min_tile = size_t(NT / 32) * size_t(max_m + 4);
  if (tile < min_tile) tile = min_tile;
  if (tile_doubles) *tile_doubles = tile;
  return (fixed + tile) * sizeof(double);
}

}  // namespace

size_t qr_scratch_doubles(int m, int n, int nmem) {
  const size_t kmax0 = size_t(m < n ? m : n);
  return 4 * size_t(n) + 2 * size_t(nmem) + 3 * kmax0 + size_t(m) * kmax0 + 8;
}

static void qr_attr() {
  static bool attr = false;
  if (!attr) {
    cuda_check(cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    220 * 1024),
               "qr smem attribute");
    attr = true;
  }
}

static cudaLaunchConfig_t qr_config(int njobs, int cluster, size_t smem, cudaStream_t st,
                                    cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(njobs * cluster));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(cluster);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

void launch_qr(const QrJob* jobs, int njobs, int max_m, int max_nmem, int cluster,
               cudaStream_t st) {
  if (njobs <= 0) return;
  qr_attr();
  size_t tile = 0;
  const size_t smem = qr_smem_bytes(max_m, max_nmem, &tile);
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = qr_config(njobs, cluster, smem, st, at);
  cudaLaunchKernelEx(&cfg, qr_kernel, jobs, int(tile), max_nmem, max_m);
}

int qr_cluster_size(int njobs, int min_n, int max_m, int max_nmem) {
  // A basis is a ~100-step sequential sweep, so the batch runs in waves of
  // co-resident clusters. Pick the cluster size g (CTAs per basis) that
  // minimises waves / g, using the occupancy API for how many clusters of
  // size g fit at once (GPC packing included); every CTA must own at least
  // two column blocks. Ties go to the smaller cluster.
  qr_attr();
  const size_t smem = qr_smem_bytes(max_m, max_nmem, nullptr);
  static int cache_key[9] = {0};
  static int cache_val[9] = {0};
  int best = 1;
  double best_cost = 1e30;
  for (int g = 1; g <= 8; ++g) {
    if (g > 1 && min_n < 2 * CB * g) break;
    int fit = 0;
    if (cache_key[g] == int(smem)) {
      fit = cache_val[g];
    } else {
      cudaLaunchAttribute at[1];
      cudaLaunchConfig_t cfg = qr_config(g, g, smem, nullptr, at);
      if (cudaOccupancyMaxActiveClusters(&fit, qr_kernel, &cfg) != cudaSuccess) {
        cudaGetLastError();
        fit = 0;
      }
      cache_key[g] = int(smem);
      cache_val[g] = fit;
    }
    if (fit <= 0) continue;
    const int waves = (njobs + fit - 1) / fit;
    const double cost = double(waves) / g * (1.0 + 0.02 * (g - 1));
    if (cost < best_cost) {
      best_cost = cost;
      best = g;
    }
  }
  return best;
}

}  // namespace h2g
