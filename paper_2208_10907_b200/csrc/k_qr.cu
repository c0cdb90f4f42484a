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
#include <cooperative_groups.h>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace h2g {

namespace {

constexpr int NT = 256;

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
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// red_h over a shared-memory column (stride ld) with 8-deep load prefetch:
// the dependent add chain then runs at FP64 latency, not LDS latency.
__device__ __forceinline__ double red_h_smem(const double* __restrict__ v,
                                             const double* __restrict__ col, int ld, int tc) {
  double s = 0.0;
  const int v4 = tc & ~3;
  int i = 0;
  for (; i + 8 <= v4; i += 8) {
    double p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = v[i + u] * col[(i + u) * ld];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = s + p[u];
  }
  for (; i < v4; ++i) s = s + v[i] * col[i * ld];
  if ((tc & 3) >= 2) {
    s = s + v[i] * col[i * ld];
    s = s + v[i + 1] * col[(i + 1) * ld];
    i += 2;
  }
  if (tc & 1) s = fma(v[i], col[i * ld], s);
  return s;
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity));
}
// TMA bulk copies (UBLKCP): global -> shared completing on an mbarrier, and
// shared -> global in a bulk group.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}

// Column-major panel W (element (i, j) at W[j * ldw + i]): a tile of
// whole column segments [k, m) is one contiguous HBM range, loaded with
// cp.async into shared memory at an odd pitch (conflict-free per-thread
// column walks), updated there, and written back: one read + one write of
// the trailing panel per Householder step.
// Warp w copies columns w, w + NT/32, ...; lanes walk the contiguous
// segment (no per-element index division).
__device__ __forceinline__ void load_tile(double* T, int pitch, const double* W, int64_t ldw,
                                          int k, int rows, int jt, int tw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < tw; c += NT / 32) {
    const double* src = W + int64_t(jt + c) * ldw + k;
    double* dst = T + c * pitch;
    for (int r = lane; r < rows; r += 32) cp_async8(dst + r, src + r);
  }
  cp_async_wait_all();
}

__device__ __forceinline__ void store_tile(const double* T, int pitch, double* W, int64_t ldw,
                                           int k, int rows, int jt, int tw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < tw; c += NT / 32) {
    double* dst = W + int64_t(jt + c) * ldw + k;
    const double* src = T + c * pitch;
    for (int r = lane; r < rows; r += 32) dst[r] = src[r];
  }
}

// Cluster-split QR: the G CTAs of a thread-block cluster share one basis;
// column blocks of CB columns are owned round-robin (owner = (j / CB) % G).
// Per Householder step: cluster-wide pivot reductions through distributed
// shared memory, the swap and the reflector by CTA 0, every CTA sweeps its own
// columns, CTA 0 runs the ordered member-mass chain. Global data written by
// one CTA is read by the others only across cluster barriers
// (barrier.cluster release/acquire).
constexpr int CB = NT;

// Member-mass downdates of one step (linalg.cpp:312-321), lead CTA. Members
// are contiguous ranges of original columns, and position j initially holds
// column j; only pivot swaps displace columns, so the positions (> s) where
// a column of another member sits form a short sorted list D. Each thread
// owns whole members and runs each member's ordered chain over its range
// (skipping D) merged with its own displaced columns — every member's chain
// sees the reference's position order, members run in parallel.
__device__ void member_step(const Scratch& S, int s, int nmem, const int64_t* off,
                            const int* D, int nd, double* mmsh) {
  for (int g = threadIdx.x; g < nmem; g += NT) {
    const int a = max(s + 1, int(off[g])), b = int(off[g + 1]);
    double val = mmsh[g];
    auto step = [&](int j) {
      const double v = val - S.sq[j];
      val = v < 0.0 ? 0.0 : v;
    };
    int p = 0;
    for (; p < nd && D[p] < a; ++p)
      if (S.grp[S.piv[D[p]]] == g) step(D[p]);
    for (int j = a; j < b; ++j) {
      if (p < nd && D[p] == j) {
        ++p;
        continue;
      }
      step(j);
    }
    for (; p < nd; ++p)
      if (D[p] >= b && S.grp[S.piv[D[p]]] == g) step(D[p]);
    mmsh[g] = val;
  }
}

struct ClSlots {
  double d;
  int piv, pos;
  int flag;
  int nd;
};

// Dynamic shared memory: [ v (m) | member masses (nmem) | column tile ].
__global__ void __launch_bounds__(NT, 2) qr_kernel(const QrJob* __restrict__ jobs, int tile_doubles,
                                                   int nmem_cap) {
  extern __shared__ double dsm[];
  __shared__ double redd[32];
  __shared__ int redi[32];
  __shared__ double sh_tau;
  __shared__ ClSlots slot;
  __shared__ __align__(8) uint64_t mbar[NT / 32][2];
  __shared__ unsigned mpar[NT / 32][2];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = int(cluster.num_blocks());
  const int cr = int(cluster.block_rank());
  const QrJob job = jobs[blockIdx.x / G];
  const int m = job.m, n = job.n, nmem = job.nmem;
  double* W = job.work;
  const int64_t ldw = job.ldw;
  const int tid = threadIdx.x;
  double* vsh = dsm;
  double* mmsh = dsm + m;
  double* T = dsm + ((m + nmem_cap + 1) & ~1);  // 16-byte aligned tile
  Scratch S = carve(job.scratch, m, n, nmem);
  const int kmax0 = m < n ? m : n;
  int kmax = kmax0;
  if (job.cap > 0 && job.cap < kmax) kmax = job.cap;
  const bool lead = cr == 0;
  if (tid < NT / 32) {
    mbar_init(&mbar[tid][0], 1);
    mbar_init(&mbar[tid][1], 1);
    mpar[tid][0] = mpar[tid][1] = 0;
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  // R = A (skipped when factoring in place): own columns.
  if (!(job.A.p == W && job.A.rs == 1 && job.A.cs == ldw)) {
    for (int b = cr; b * CB < n; b += G)
      for (int j = b * CB; j < min(n, (b + 1) * CB); ++j)
        for (int i = tid; i < m; i += NT) W[int64_t(j) * ldw + i] = job.A.at(i, j);
    __syncthreads();
  }
  // Column norms of own columns (pattern P2 over all rows), tile by tile.
  {
    const int pitch = m | 1;
    const int twmax = max(1, min(NT, tile_doubles / pitch));
    for (int b = cr; b * CB < n; b += G) {
      const int j1 = min(n, (b + 1) * CB);
      for (int jt = b * CB; jt < j1; jt += twmax) {
        const int tw = min(twmax, j1 - jt);
        load_tile(T, pitch, W, ldw, 0, m, jt, tw);
        __syncthreads();
        if (tid < tw) {
          const double* col = T + tid * pitch;
          const double s = red_p2([&](int i, double& a, double& b2) { a = b2 = col[i]; }, 0, m);
          S.cn2[jt + tid] = s;
          S.cn2o[jt + tid] = s;
          S.piv[jt + tid] = jt + tid;
        }
        __syncthreads();
      }
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
  int nd = 0;  // length of the displaced-position list D
  long long t_piv = 0, t_refl = 0, t_tile = 0, t_mem = 0, t0c;
  for (int k = 0; k < kmax; ++k) {
    t0c = clock64();
    // Pivot: cluster-wide max of the remaining norms, then the lowest
    // original index within the 4e-15 tie band (linalg.cpp:263-274).
    double mx = -1.0;
    for (int b = cr; b * CB < n; b += G) {
      const int j = max(k, b * CB) + tid;
      if (j < min(n, (b + 1) * CB)) mx = fmax(mx, S.cn2[j]);
    }
    mx = block_max(mx, redd);
    if (tid == 0) slot.d = mx;
    cluster.sync();
    double best = -1.0;
    for (int q = 0; q < G; ++q) best = fmax(best, cluster.map_shared_rank(&slot, q)->d);
    const int members_not_done = cluster.map_shared_rank(&slot, 0)->flag;
    if (best <= 0.0) break;
    const double tie = best * (1.0 - 4e-15);
    int cand = 0x7fffffff;
    for (int b = cr; b * CB < n; b += G) {
      const int j = max(k, b * CB) + tid;
      if (j < min(n, (b + 1) * CB) && S.cn2[j] >= tie) cand = min(cand, S.piv[j]);
    }
    cand = block_min_int(cand, redi);
    int cpos = 0x7fffffff;
    for (int b = cr; b * CB < n; b += G) {
      const int j = max(k, b * CB) + tid;
      if (j < min(n, (b + 1) * CB) && S.piv[j] == cand && S.cn2[j] >= tie) cpos = j;
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
    // apply_reflector to own columns k+1.. (linalg.cpp:137-149) + downdate.
    // Every warp streams its own column tiles through a private slice of the
    // shared tile (cp.async load -> per-lane column update -> store), with no
    // CTA barrier inside the step. (A TMA bulk-copy variant with double
    // buffering measured 1.9x slower here: the per-column segments are only
    // 2 KB and the buffer turnaround serialises.)
    {
      const int rows = m - k;
      const int pitch = rows | 1;
      const int warp = tid >> 5, lane = tid & 31;
      constexpr int NW = NT / 32;
      const int per_warp = tile_doubles / NW;
      const int cw = max(1, min(32, per_warp / pitch));
      double* Tw = T + warp * per_warp;
      for (int b = cr; b * CB < n; b += G) {
        const int j0 = max(k + 1, b * CB), j1 = min(n, (b + 1) * CB);
        for (int jt = j0 + warp * cw; jt < j1; jt += NW * cw) {
          const int tw = min(cw, j1 - jt);
          for (int c = 0; c < tw; ++c) {
            const double* src = W + int64_t(jt + c) * ldw + k;
            for (int r = lane; r < rows; r += 32) cp_async8(Tw + c * pitch + r, src + r);
          }
          cp_async_wait_all();
          __syncwarp();
          if (tau != 0.0) {
            // Sequential dot chain: one lane per column. The rank-1 update is
            // element-wise, so the whole warp applies it column by column.
            double sc = 0.0;
            if (lane < tw) sc = -(tau * red_h_smem(vsh + k, Tw + lane * pitch, 1, rows));
            for (int c = 0; c < tw; ++c) {
              const double s_c = __shfl_sync(0xffffffffu, sc, c);
              double* colc = Tw + c * pitch;
              for (int r = lane; r < rows; r += 32) colc[r] = fma(s_c, vsh[k + r], colc[r]);
            }
            __syncwarp();
          }
          if (lane < tw) {
            double* col = Tw + lane * pitch;
            // GCC computes rkj*rkj once (rounded) for the norm and member downdates.
            const int j = jt + lane;
            const double rkj = col[0];
            const double sq = rkj * rkj;
            double upd = S.cn2[j] - sq;
            if (upd < 1e-8 * S.cn2o[j])
              upd = red_p2([&](int r, double& a, double& b2) { a = b2 = col[r]; }, 1, rows - 1);
            S.cn2[j] = fmax(0.0, upd);
            S.sq[j] = sq;
          }
          __syncwarp();
          for (int c = 0; c < tw; ++c) {
            double* dst = W + int64_t(jt + c) * ldw + k;
            for (int r = lane; r < rows; r += 32) dst[r] = Tw[c * pitch + r];
          }
          __syncwarp();
        }
      }
    }
    cluster.sync();
    t_tile += clock64() - t0c; t0c = clock64();
    ++rank;
    if (lead && members) {
      // D: positions > k holding a column of another member (sorted). The
      // swap of step k moved the column from position k to position sel.
      int* D = S.swp;
      if (tid == 0) {
        const int sel = S.swp[kmax0 + k];
        int w = 0;
        for (int q = 0; q < nd; ++q)
          if (D[q] > k && D[q] != sel) D[w++] = D[q];
        if (sel > k && S.grp[S.piv[sel]] != S.grp[sel]) {
          int q = w;
          while (q > 0 && D[q - 1] > sel) {
            D[q] = D[q - 1];
            --q;
          }
          D[q] = sel;
          ++w;
        }
        slot.nd = w;
      }
      __syncthreads();
      nd = slot.nd;
      member_step(S, k, nmem, job.member_off, D, nd, mmsh);
      __syncthreads();
      if (tid == 0) {
        const int gk = S.grp[S.piv[k]];
        const double v = mmsh[gk] - S.pn2[k];
        mmsh[gk] = v < 0.0 ? 0.0 : v;
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

}  // namespace

size_t qr_scratch_doubles(int m, int n, int nmem) {
  const size_t kmax0 = size_t(m < n ? m : n);
  return 4 * size_t(n) + 2 * size_t(nmem) + 3 * kmax0 + size_t(m) * kmax0 + 8;
}

void launch_qr(const QrJob* jobs, int njobs, int max_m, int max_nmem, int cluster,
               cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  // Two CTAs per SM (~100 KB of shared memory each, most of it the tile) so
  // one CTA's load/compute/store phases overlap the other's.
  const size_t budget = 100 * 1024;
  const size_t fixed = sizeof(double) * size_t((max_m + max_nmem + 1) & ~1);
  size_t tile = budget > fixed + 8192 ? (budget - fixed) / sizeof(double) : 1024;
  // Every warp needs two buffers of at least one (even-padded) column.
  const size_t min_tile = size_t(NT / 32) * 2 * size_t((max_m + 2) & ~1);
  if (tile < min_tile) tile = min_tile;
  if (tile < 1536) tile = 1536;                             // member staging (2 x 512)
  const size_t smem = fixed + tile * sizeof(double);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(njobs * cluster));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(cluster);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, qr_kernel, jobs, int(tile), max_nmem);
}

int qr_cluster_size(int njobs, int min_n) {
  // Aim for ~2 CTAs per SM over 148 SMs; split a basis only when its panel is
  // wide enough to give every CTA whole column blocks.
  int g = 1;
  while (g < 8 && njobs * g * 2 <= 296 && min_n >= 4 * CB * g) g *= 2;
  return g;
}

}  // namespace h2g
