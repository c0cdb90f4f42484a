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
constexpr int NBUF = 3;  // max column tiles in flight per warp in the sweep

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

__device__ __forceinline__ double block_max(double v, double* red) {
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

__device__ __forceinline__ int block_min_int(int v, int* red) {
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
  const int ng = npair >> 2;  // groups of 4 pairs, the next group's loads in flight
  if (ng > 0) {
    double2 x[4], y[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      x[w] = c2[w];
      y[w] = v2[w];
    }
    for (int g = 0; g < ng; ++g) {
      double2 xn[4], yn[4];
      const int qn = g + 1 < ng ? 4 * (g + 1) : 4 * g;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        xn[w] = c2[qn + w];
        yn[w] = v2[qn + w];
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        s = s + x[w].x * y[w].x;
        s = s + x[w].y * y[w].y;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        x[w] = xn[w];
        y[w] = yn[w];
      }
    }
    q = 4 * ng;
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

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One-instruction column load: global -> shared bulk copy (TMA engine)
// completing on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Shared -> global bulk copy (TMA engine) in this thread's bulk async-group.
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// All but the newest N bulk groups of this thread have finished reading shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
// Every bulk group of this thread complete; its global writes ordered before
// this thread's later generic accesses (and the cluster barrier's release).
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\nfence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
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

// Member masses (linalg.cpp:240-256, :312-321). Member g is owned by CTA
// g % G of the cluster and, inside it, by one warp; members are contiguous
// ranges of original columns and position j initially holds column j, so
// only pivot swaps displace columns: the positions (> k) where a column of
// another member sits form a short sorted list D (positions Dp, their
// columns' members Dg, in shared memory, maintained identically by every
// CTA). A member's chain runs over its range, skipping D, merged with its
// own displaced positions: the reference's position order.
__device__ __forceinline__ double mass_sub(double val, double x) {
  const double v = val - x;
  return v < 0.0 ? 0.0 : v;
}

// Ordered chain of one warp over x[a, b), skipping the positions Dp[p..]
// (sorted; p advances past the skipped ones): val = val - x[j] clamped at 0
// (CLAMP) or val = val + x[j]. Every lane computes the same chain; the
// values arrive 256 at a time (8 per lane, the next 256 in flight) and are
// broadcast by shuffles, so the dependent chain runs at FP64 latency.
template <bool CLAMP>
__device__ __forceinline__ double warp_chain(const double* __restrict__ x, int a, int b,
                                             const int* Dp, int& p, int nd, double val) {
  const int lane = threadIdx.x & 31;
  auto fetch = [&](int j0) {
    const int j = j0 + lane;
    return j < b ? __ldcg(&x[j]) : 0.0;
  };
  // Four rounds of 32 in flight ahead of the chain.
  double c0 = fetch(a), c1 = fetch(a + 32), c2 = fetch(a + 64), c3 = fetch(a + 96);
  for (int base = a; base < b; base += 32) {
    // Skip mask of these 32 positions: past b, or in D.
    const int left = b - base;
    unsigned skip = left >= 32 ? 0u : ~0u << left;
    const int lim = min(base + 32, b);
    while (p < nd && Dp[p] < lim) {
      skip |= 1u << (Dp[p] - base);
      ++p;
    }
    const double cur = c0;
    c0 = c1;
    c1 = c2;
    c2 = c3;
    c3 = fetch(base + 128);
    // A skipped position subtracts (adds) +0, which leaves val unchanged
    // (val >= +0); masking the bits keeps the skip off the dependent chain.
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const double xv = __shfl_sync(0xffffffffu, cur, l);
      const long long keep = ((skip >> l) & 1u) ? 0ll : -1ll;
      const double xl = __longlong_as_double(__double_as_longlong(xv) & keep);
      val = CLAMP ? mass_sub(val, xl) : val + xl;
    }
  }
  return val;
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
                                                   int nmem_cap, int m_cap, int nbuf) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double redd[32];
  __shared__ int redi[32];
  __shared__ double sh_tau;
  __shared__ int sh_nd;
  __shared__ ClSlots slot;
  __shared__ __align__(8) uint64_t wbar[NBUF * (NT / 32)];
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
  if (tid < NBUF * (NT / 32)) mbar_init(&wbar[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  unsigned wpar = 0;  // bit b: phase parity of this warp's buffer-b barrier

  // R = A (skipped when factoring in place): own columns.
  if (!(job.A.p == W && job.A.rs == 1 && job.A.cs == ldw)) {
    for (int li = 0; li < nloc; ++li) {
      const int j = own.l2g(li);
      for (int i = tid; i < m; i += NT) W[int64_t(j) * ldw + i] = job.A.at(i, j);
    }
    __syncthreads();
  }
  // Column norms of own columns (pattern P2 over all rows), tile by tile;
  // their max is step 0's pivot value (later steps take it from the sweep).
  double lmax = -1.0;
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
        lmax = fmax(lmax, s);
      }
      __syncthreads();
    }
  }
  {
    const double mx = block_max(lmax, redd);
    if (tid == 0) slot.d = mx;
  }
  cluster.sync();
  const bool members = nmem >= 1;
  if (lead && members)
    for (int g = tid; g < nmem; g += NT)
      for (int64_t j = job.member_off[g]; j < job.member_off[g + 1]; ++j) S.grp[j] = g;
  // Own members: g = cr + G * (warp + NW * t).
  auto member_of_warp = [&](int t) { return cr + G * (warp + NW * t); };
  if (members) {
    for (int t = 0; member_of_warp(t) < nmem; ++t) {
      const int g = member_of_warp(t);
      int p = 0;
      const double mass = warp_chain<false>(S.cn2, int(job.member_off[g]),
                                            int(job.member_off[g + 1]), Dp, p, 0, 0.0);
      if (lane == 0) {
        mmsh[g] = mass;
        S.mt[g] = job.member_tol * job.member_tol * mass;
      }
    }
  }
  __syncthreads();
  {
    int not_done = 0;
    if (members)
      for (int g = cr + G * tid; g < nmem; g += G * NT) not_done |= (mmsh[g] > S.mt[g]);
    not_done = __syncthreads_or(not_done);
    if (tid == 0) slot.flag = not_done;
  }

  double r11 = -1.0;
  int rank = 0;
  int nd = 0;  // length of the displaced-position list D
  long long t_piv = 0, t_refl = 0, t_tile = 0, t_mem = 0, t0c;
  long long t_w = 0, t_c = 0, t_s = 0, n_t = 0, n_rc = 0, n_ch = 0;
  for (int k = 0; k < kmax; ++k) {
    t0c = clock64();
    // Pivot: cluster-wide max of the remaining norms (each CTA's max was
    // published by its previous sweep), then the lowest original index
    // within the 4e-15 tie band (linalg.cpp:263-274): one scan for the
    // minimum candidate and its position.
    const int lk = own.below(k);
    double best = -1.0;
    for (int q = 0; q < G; ++q) best = fmax(best, cluster.map_shared_rank(&slot, q)->d);
    if (best <= 0.0) break;
    const double tie = best * (1.0 - 4e-15);
    int cand = 0x7fffffff, cpos = 0x7fffffff;
    {
      int li = lk + tid;
      for (; li + 3 * NT < nloc; li += 4 * NT) {
        int jj[4];
        double cv[4];
        int pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          jj[u] = own.l2g(li + u * NT);
          cv[u] = __ldcg(&S.cn2[jj[u]]);
          pv[u] = __ldcg(&S.piv[jj[u]]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (cv[u] >= tie && pv[u] < cand) {
            cand = pv[u];
            cpos = jj[u];
          }
      }
      for (; li < nloc; li += NT) {
        const int j = own.l2g(li);
        const int pv = __ldcg(&S.piv[j]);
        if (__ldcg(&S.cn2[j]) >= tie && pv < cand) {
          cand = pv;
          cpos = j;
        }
      }
    }
    const int cmin = block_min_int(cand, redi);
    cpos = block_min_int(cand == cmin ? cpos : 0x7fffffff, redi);
    if (tid == 0) {
      slot.piv = cmin;
      slot.pos = cpos;
    }
    cluster.sync();
    int members_not_done = 0;
    for (int q = 0; q < G; ++q) members_not_done |= cluster.map_shared_rank(&slot, q)->flag;
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
    lmax = -1.0;
    {
      const int rows = m - k;
      const int k0 = k & ~1, off = k - k0;
      const int np = (m - k0 + 1) >> 1;  // pairs per segment
      const int P = (np & 1) ? 2 * np : 2 * np + 2;
      const int per_warp = (tile_doubles / NW) & ~1;
      // NBUF column tiles per warp: tile t's chain runs while tiles t+1 and
      // t+2 load and tile t-1's bulk stores drain.
      const int cw = max(1, min(32, per_warp / (nbuf * P)));
      double* Tw = T + warp * per_warp;
      // Store pairs start at k1 = (k + 1) rounded down to even: row k is
      // R's final row k (rkj), stored with its updated value.
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
      const int stride = NW * cw;
      const int a0 = l0 + warp * cw;
      const int ntile = a0 < nloc ? (nloc - a0 + stride - 1) / stride : 0;
      // Tile loads: one bulk copy per column (lane c issues column c) on the
      // buffer's mbarrier; lane 0 arms it with the tile's byte count first.
      // Lane c also issues column c's bulk store, so the slot a lane reloads
      // is only ever read by its own earlier store (wait_group.read).
      const unsigned colbytes = unsigned(16 * np);
      auto load_tile = [&](int t) {
        const int b = t % nbuf, abase = a0 + t * stride, cnt = min(cw, nloc - abase);
        if (lane == 0) mbar_expect_tx(&wbar[warp * NBUF + b], colbytes * unsigned(cnt));
        __syncwarp();
        if (lane < cnt) {
          fence_proxy_async();
          bulk_load(Tw + (b * cw + lane) * P, W + int64_t(own.l2g(abase + lane)) * ldw + k0, colbytes,
                    &wbar[warp * NBUF + b]);
        }
      };
      // Tiles loaded ahead: nbuf - 1 (the buffer reloaded at the end of
      // iteration t held tile t - 1), or 1 with a single buffer (tile t's own).
      const int ahead = nbuf == 1 ? 1 : nbuf - 1;
      for (int t = 0; t < ahead && t < ntile; ++t) load_tile(t);
      for (int t = 0; t < ntile; ++t) {
        const int b = t % nbuf, a = a0 + t * stride;
        const int tw = min(cw, nloc - a);
        double* Tb = Tw + b * cw * P;
        long long c0 = clock64();
        mbar_wait(&wbar[warp * NBUF + b], (wpar >> b) & 1u);
        wpar ^= 1u << b;
        long long c1 = clock64();
        double sc = 0.0;
        int jl = 0;
        bool need_rc = false;
        if (lane < tw) {
          jl = own.l2g(a + lane);
          const double cn2j = S.cn2[jl], cn2oj = S.cn2o[jl];  // in flight during the chain
          const double* col = Tb + lane * P;
          if (tau != 0.0) sc = -(tau * dot_h_pairs(col, vb, off, rows));
          // GCC computes rkj*rkj once (rounded) for the norm and member downdates.
          const double rkj = tau != 0.0 ? fma(sc, vsh[k], col[off]) : col[off];
          const double sq = rkj * rkj;
          const double upd = cn2j - sq;
          ++n_ch;
          S.sq[jl] = sq;
          // Cancellation: the norm is recomputed from the updated column
          // (linalg.cpp:300-311) after the update, overlapping the stores.
          need_rc = upd < 1e-8 * cn2oj;
          if (!need_rc) {
            const double nc = fmax(0.0, upd);
            S.cn2[jl] = nc;
            lmax = fmax(lmax, nc);
          }
        }
        __syncwarp();
        long long c2 = clock64();
        // Update in place in shared memory, warp-wide (two columns per pass),
        // then one bulk store per column straight from the slot.
        if (tau != 0.0) {
          for (int c = 0; c < tw; c += 2) {
            const bool two = c + 1 < tw;
            const double s_0 = __shfl_sync(0xffffffffu, sc, c);
            const double s_1 = __shfl_sync(0xffffffffu, sc, two ? c + 1 : c);
            double* col0 = Tb + c * P + (k1 - k0);
            double* col1 = col0 + P;
            if (nps <= 128) {
              double2 x0[4], x1[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int p = lane + 32 * u;
                x0[u] = p < nps ? *reinterpret_cast<const double2*>(col0 + 2 * p) : make_double2(0.0, 0.0);
                x1[u] = (two && p < nps) ? *reinterpret_cast<const double2*>(col1 + 2 * p)
                                         : make_double2(0.0, 0.0);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int p = lane + 32 * u;
                if (p < nps) {
                  *reinterpret_cast<double2*>(col0 + 2 * p) =
                      make_double2(fma(s_0, vr[u].x, x0[u].x), fma(s_0, vr[u].y, x0[u].y));
                  if (two)
                    *reinterpret_cast<double2*>(col1 + 2 * p) =
                        make_double2(fma(s_1, vr[u].x, x1[u].x), fma(s_1, vr[u].y, x1[u].y));
                }
              }
            } else {
              for (int p = lane; p < nps; p += 32) {
                const double2 v = *reinterpret_cast<const double2*>(vsh + k1 + 2 * p);
                const double2 x = *reinterpret_cast<const double2*>(col0 + 2 * p);
                *reinterpret_cast<double2*>(col0 + 2 * p) = make_double2(fma(s_0, v.x, x.x), fma(s_0, v.y, x.y));
                if (two) {
                  const double2 y = *reinterpret_cast<const double2*>(col1 + 2 * p);
                  *reinterpret_cast<double2*>(col1 + 2 * p) = make_double2(fma(s_1, v.x, y.x), fma(s_1, v.y, y.y));
                }
              }
            }
          }
          fence_proxy_async();
          __syncwarp();
          if (lane < tw) bulk_store(W + int64_t(jl) * ldw + k1, Tb + lane * P + (k1 - k0), unsigned(16 * nps));
          bulk_commit();
        }
        // Deferred norm recomputes: rows k+1.. of the updated column, read
        // from the slot while the bulk stores drain it (both only read).
        if (need_rc) {
          ++n_rc;
          const double* col = Tb + lane * P;
          const double nc = fmax(0.0, red_p2([&](int r, double& x, double& y) { x = y = col[off + r]; }, 1, rows - 1));
          S.cn2[jl] = nc;
          lmax = fmax(lmax, nc);
        }
        // Tile t-1's buffer is reloaded next: its stores must have read it.
        if (nbuf == 1)
          bulk_wait_read<0>();
        else
          bulk_wait_read<1>();
        __syncwarp();
        if (t + ahead < ntile) load_tile(t + ahead);
        long long c3 = clock64();
        t_w += c1 - c0; t_c += c2 - c1; t_s += c3 - c2; ++n_t;
      }
      // Every store complete (and visible) before the cluster barrier: the
      // next step's swap and reflector read these columns from other CTAs.
      bulk_wait_all();
    }
    {
      const double mx = block_max(lmax, redd);
      if (tid == 0) slot.d = mx;  // next step's pivot value
    }
    cluster.sync();
    t_tile += clock64() - t0c; t0c = clock64();
    ++rank;
    if (members) {
      // D: positions > k holding a column of another member (sorted). The
      // swap of step k moved the column from position k to position sel.
      if (tid == 0) {
        const int sel = __ldcg(&S.swp[kmax0 + k]);
        int w = 0;
        for (int q = 0; q < nd; ++q)
          if (Dp[q] > k && Dp[q] != sel) {
            Dp[w] = Dp[q];
            Dg[w] = Dg[q];
            ++w;
          }
        const int gs = __ldcg(&S.grp[__ldcg(&S.piv[sel])]);
        if (sel > k && gs != __ldcg(&S.grp[sel])) {
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
      for (int t = 0; member_of_warp(t) < nmem; ++t) {
        const int g = member_of_warp(t);
        const int a = max(k + 1, int(job.member_off[g])), b = int(job.member_off[g + 1]);
        double val = mmsh[g];
        int p = 0;
        for (; p < nd && Dp[p] < a; ++p)
          if (Dg[p] == g) val = mass_sub(val, __ldcg(&S.sq[Dp[p]]));
        val = warp_chain<true>(S.sq, a, b, Dp, p, nd, val);
        for (; p < nd; ++p)
          if (Dg[p] == g) val = mass_sub(val, __ldcg(&S.sq[Dp[p]]));
        __syncwarp();
        if (lane == 0) mmsh[g] = val;
      }
      __syncthreads();
      if (tid == 0) {
        // The processed column's leftover mass is gone entirely.
        const int gk = __ldcg(&S.grp[__ldcg(&S.piv[k])]);
        if (gk % G == cr) mmsh[gk] = mass_sub(mmsh[gk], __ldcg(&S.pn2[k]));
      }
      __syncthreads();
      int not_done = 0;
      for (int g = cr + G * tid; g < nmem; g += G * NT) not_done |= (mmsh[g] > S.mt[g]);
      not_done = __syncthreads_or(not_done);
      if (tid == 0) slot.flag = not_done;
    }
    t_mem += clock64() - t0c;
  }
  // No CTA may reuse its slots while others can still read them.
  cluster.sync();
  if (lead && tid == 0 && job.dbg) {
    job.dbg[0] = double(t_piv); job.dbg[1] = double(t_refl); job.dbg[2] = double(t_tile);
    job.dbg[3] = double(t_mem); job.dbg[4] = double(rank); job.dbg[5] = double(n);
    job.dbg[8] = double(t_w); job.dbg[9] = double(t_c); job.dbg[10] = double(t_s); job.dbg[11] = double(n_t);
    job.dbg[12] = double(n_rc); job.dbg[13] = double(n_ch);
  }
  long long tq = clock64();

  // form_q (linalg.cpp:181-185): Q = I, reflectors applied backward. Every
  // column of Q evolves independently, so the cluster's CTAs split the
  // columns and each lane carries one column in shared memory through all
  // reflectors (dot chain and update in the reference's order).
  {
    double* Q = job.Q;
    const int jc0 = (m * cr) / G, jc1 = (m * (cr + 1)) / G;
    const int pitch = m | 1;
    const int per_warp = tile_doubles / NW;
    const int cwq = max(1, min(32, per_warp / pitch));
    for (int jb = jc0; jb < jc1; jb += NW * cwq) {
      const int jw = jb + warp * cwq;
      const int tw = max(0, min(cwq, jc1 - jw));
      const bool act = lane < tw;
      const int j = jw + lane;
      double* q = T + warp * per_warp + lane * pitch;
      if (act)
        for (int i = 0; i < m; ++i) q[i] = (i == j) ? 1.0 : 0.0;
      for (int k = rank - 1; k >= 0; --k) {
        __syncthreads();
        for (int i = tid; i < m; i += NT) vsh[i] = __ldcg(&S.V[int64_t(k) * m + i]);
        if (tid == 0) sh_tau = __ldcg(&S.tau[k]);
        __syncthreads();
        const double tau = sh_tau;
        if (tau == 0.0 || !act) continue;
        const double dot = red_h([&](int i, double& x, double& y) { x = vsh[i]; y = q[i]; }, k, m - k, 0.0);
        const double sk = tau * dot;
        for (int i = k; i < m; ++i) q[i] = fma(-sk, vsh[i], q[i]);
      }
      __syncwarp();
      for (int i = 0; i < m; ++i)
        if (act) Q[int64_t(i) * m + j] = q[i];
      __syncthreads();
    }
  }
  if (lead && tid == 0) *job.rank_out = rank;
  if (lead && tid == 0 && job.dbg) job.dbg[6] = double(clock64() - tq);
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
  // Every warp needs at least one column slot per buffer (pitch <= max_m + 4).
  const size_t min_tile = size_t(NT / 32) * NBUF * size_t(max_m + 4);
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
  smem_attr((const void*)qr_kernel, 220 * 1024, "qr smem attribute");
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
  static const int nbuf = [] {
    const char* e = getenv("H2G_QR_NBUF");
    return e ? std::max(1, std::min(NBUF, atoi(e))) : 1;
  }();
  cudaLaunchKernelEx(&cfg, qr_kernel, jobs, int(tile), max_nmem, max_m, nbuf);
}

// Clusters of g CTAs that can be co-resident (occupancy API, GPC packing
// included), cached per (g, shared-memory size).
int qr_fit(int g, int max_m, int max_nmem) {
  qr_attr();
  const size_t smem = qr_smem_bytes(max_m, max_nmem, nullptr);
  static int cache_key[9] = {0};
  static int cache_val[9] = {0};
  if (g < 1 || g > 8) return 0;
  if (cache_key[g] == int(smem)) return cache_val[g];
  int fit = 0;
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = qr_config(g, g, smem, nullptr, at);
  if (cudaOccupancyMaxActiveClusters(&fit, qr_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    fit = 0;
  }
  cache_key[g] = int(smem);
  cache_val[g] = fit;
  return fit;
}

int qr_max_cluster(int n) {
  int g = 1;
  while (g < 8 && n >= 2 * CB * (g + 1)) ++g;
  return g;
}

int qr_cluster_size(int njobs, int min_n, int max_m, int max_nmem) {
  // A basis is a ~100-step sequential sweep, so the batch runs in waves of
  // co-resident clusters. Pick the cluster size g (CTAs per basis) that
  // minimises waves / g, using the occupancy API for how many clusters of
  // size g fit at once; every CTA must own at least two column blocks. Ties
  // go to the smaller cluster.
  int best = 1;
  double best_cost = 1e30;
  for (int g = 1; g <= qr_max_cluster(min_n); ++g) {
    const int fit = qr_fit(g, max_m, max_nmem);
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
