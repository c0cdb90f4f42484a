// Blocked column-pivoted Householder QR with the member-mass stopping rule
// ("blocked" QR mode; the default "exact" mode is k_qr.cu).
//
// The reference (linalg.cpp:216-332) updates the whole trailing panel after
// every reflector, so each step reads and writes it: the exact mode streams
// 16 bytes per element per step through HBM. Here, as in LAPACK's xLAQPS,
// reflectors are accumulated NB at a time: per step the trailing panel is
// only READ (one pass computes v^T a_j for every column, from which the
// column's F row, its r_kj and its norm downdate follow), and the panel is
// written once per block (rank-NB trailing update fused with the exact
// recomputation of every column norm). Traffic per element-step drops from
// 16 to ~8 + 24/NB bytes.
//
// Same decisions as the reference, different rounding: pivots are the
// largest (downdated) norm with the 4e-15 lowest-index tie band, the stop
// tests use the exact norm of the updated pivot column, member masses are
// the remaining norm^2 of each member's columns. Ranks and bases agree with
// the exact mode to rounding (tests/test_qr_blocked.py), not bit for bit.
#include <cooperative_groups.h>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace h2g {

void cuda_check(cudaError_t e, const char* what);  // batch.cu

namespace {

constexpr int NT = 256;  // 8 warps
constexpr int NW = NT / 32;
constexpr int NB = 32;   // reflectors per trailing update
constexpr int CB = 256;  // column ownership blocks (round-robin over the cluster)

struct Own {
  int G, cr;
  __device__ __forceinline__ int l2g(int li) const { return ((li / CB) * G + cr) * CB + li % CB; }
  __device__ __forceinline__ int below(int x) const {
    const int bx = x / CB;
    int c = bx > cr ? ((bx - cr + G - 1) / G) * CB : 0;
    if (bx % G == cr) c += x % CB;
    return c;
  }
};

struct Scr {
  double *cn2, *sq, *mm0, *mt, *tau, *V, *F, *acc;  // acc: 2 x nmem member sums (step parity)
  int *piv, *grp;
  double* wv;  // NB
  int* ctl;    // [0] stop flag, [1] rank
};

__host__ __device__ inline size_t scr_doubles(int m, int n, int nmem) {
  const size_t kmax0 = size_t(m < n ? m : n);
  return 2 * size_t(n) + 2 * size_t(n) + 2 * size_t(nmem) + 2 * size_t(nmem) + kmax0 + size_t(m) * kmax0 +
         size_t(n) * NB + NB + 8;
}

__device__ inline Scr carve_b(double* s, int m, int n, int nmem) {
  const int kmax0 = m < n ? m : n;
  Scr c;
  c.cn2 = s;
  c.sq = c.cn2 + n;
  c.piv = reinterpret_cast<int*>(c.sq + n);
  c.grp = c.piv + n;  // 2n ints = n doubles
  c.mm0 = c.sq + 2 * int64_t(n);
  c.mt = c.mm0 + nmem;
  c.acc = c.mt + nmem;
  c.tau = c.acc + 2 * int64_t(nmem);
  c.V = c.tau + kmax0;
  c.F = c.V + int64_t(m) * kmax0;
  c.wv = c.F + int64_t(n) * NB;
  c.ctl = reinterpret_cast<int*>(c.wv + NB);
  return c;
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int q = 0; q < NW; ++q) r += red[q];
  __syncthreads();
  return r;
}

__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = -1.0;
  for (int q = 0; q < NW; ++q) r = fmax(r, red[q]);
  __syncthreads();
  return r;
}

__device__ int block_min_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  int r = 0x7fffffff;
  for (int q = 0; q < NW; ++q) r = min(r, red[q]);
  __syncthreads();
  return r;
}

struct Slot {
  double d;
  int piv, pos;
};

// Dynamic shared memory: [ Vb (m_cap x NB, column t = reflector k0 + t) |
//   v (m_cap) | wv (NB) ].
__global__ void __launch_bounds__(NT, 2) qrb_kernel(const QrJob* __restrict__ jobs, int nmem_cap, int m_cap) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double redd[NW];
  __shared__ int redi[NW];
  __shared__ Slot slot;
  __shared__ double sh_tau;
  __shared__ double rowk[NW * 16];  // per warp: row k of the current column tile
  cg::cluster_group cluster = cg::this_cluster();
  const int G = int(cluster.num_blocks()), cr = int(cluster.block_rank());
  const Own own{G, cr};
  const QrJob job = jobs[blockIdx.x / G];
  const int m = job.m, n = job.n, nmem = job.nmem;
  double* W = job.work;
  const int64_t ldw = job.ldw;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Vb = dsm;
  double* vsh = Vb + int64_t(m_cap) * NB;
  double* wvs = vsh + m_cap;
  Scr S = carve_b(job.scratch, m, n, nmem);
  const int kmax0 = m < n ? m : n;
  int kmax = kmax0;
  if (job.cap > 0 && job.cap < kmax) kmax = job.cap;
  const bool lead = cr == 0;
  const int nloc = own.below(n);
  auto VB = [&](int r, int t) -> double& { return Vb[int64_t(t) * m_cap + r]; };

  // R = A when not factoring in place.
  if (!(job.A.p == W && job.A.rs == 1 && job.A.cs == ldw)) {
    for (int li = 0; li < nloc; ++li) {
      const int j = own.l2g(li);
      for (int i = tid; i < m; i += NT) W[int64_t(j) * ldw + i] = job.A.at(i, j);
    }
    __syncthreads();
  }
  int* ipos = reinterpret_cast<int*>(S.sq);  // original column -> position
  // Member masses (linalg.cpp:240-256, :312-321): the remaining norm^2 of each
  // member's columns at positions > kk, a warp per member summing in the
  // member's column order (deterministic; no atomics).
  auto member_masses = [&](int kk) {
    for (int g = cr + G * warp; g < nmem; g += G * NW) {
      double sm = 0.0;
      for (int64_t j = job.member_off[g] + lane; j < job.member_off[g + 1]; j += 32) {
        const int pos = __ldcg(&ipos[j]);
        if (pos > kk) sm += __ldcg(&S.cn2[pos]);
      }
      sm = warp_sum(sm);
      if (lane == 0) S.acc[g] = sm;
    }
  };
  // Initial column norms (exact, warp per column) and member masses.
  double lmax = -1.0;
  for (int li = warp; li < nloc; li += NW) {
    const int j = own.l2g(li);
    const double* col = W + int64_t(j) * ldw;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(col[r], col[r], s);
    s = warp_sum(s);
    if (lane == 0) {
      S.cn2[j] = s;
      S.piv[j] = j;
      ipos[j] = j;
    }
    lmax = fmax(lmax, s);
  }
  {
    const double mx = block_max(lmax, redd);
    if (tid == 0) slot.d = mx;
  }
  cluster.sync();
  member_masses(-1);
  cluster.sync();
  bool members_not_done = false;
  for (int g = 0; g < nmem; ++g) {
    const double mass = __ldcg(&S.acc[g]);
    if (lead && tid == 0) {
      S.mm0[g] = mass;
      S.mt[g] = job.member_tol * job.member_tol * mass;
    }
    members_not_done |= mass > job.member_tol * job.member_tol * mass;
  }

  double r11 = -1.0;
  int rank = 0;
  bool stop = false;
  long long t_piv = 0, t_lead = 0, t_pass = 0, t_mem = 0, t_upd = 0;  // H2G_QR_DEBUG cycle counters
  int k = 0;
  while (k < kmax && !stop) {
    const int k0 = k;
    int i = 0;
    for (; i < NB && k < kmax; ++i, ++k) {
      long long tc0 = clock64();
      // ---- pivot: cluster max, then the lowest original index in the tie band
      double best = -1.0;
      for (int q = 0; q < G; ++q) best = fmax(best, cluster.map_shared_rank(&slot, q)->d);
      if (best <= 0.0) {
        stop = true;
        break;
      }
      const double tie = best * (1.0 - 4e-15);
      int cand = 0x7fffffff, cpos = 0x7fffffff;
      for (int li = own.below(k) + tid; li < nloc; li += NT) {
        const int j = own.l2g(li);
        const int pv = __ldcg(&S.piv[j]);
        if (__ldcg(&S.cn2[j]) >= tie && pv < cand) {
          cand = pv;
          cpos = j;
        }
      }
      const int cmin = block_min_int(cand, redi);
      cpos = block_min_int(cand == cmin ? cpos : 0x7fffffff, redi);
      cluster.sync();  // every CTA finished reading the previous slots
      if (tid == 0) {
        slot.piv = cmin;
        slot.pos = cpos;
      }
      cluster.sync();
      int sel_orig = 0x7fffffff, sel = 0x7fffffff;
      for (int q = 0; q < G; ++q) {
        const Slot* o = cluster.map_shared_rank(&slot, q);
        if (o->piv < sel_orig) {
          sel_orig = o->piv;
          sel = o->pos;
        }
      }
      long long tc1 = clock64();
      t_piv += tc1 - tc0;
      // ---- lead: swap, bring the pivot column up to date, stop tests, reflector
      if (lead) {
        if (sel != k) {
          for (int r = tid; r < m; r += NT) {
            const double t = W[int64_t(k) * ldw + r];
            W[int64_t(k) * ldw + r] = W[int64_t(sel) * ldw + r];
            W[int64_t(sel) * ldw + r] = t;
          }
          if (tid < i) {
            const double t = S.F[int64_t(tid) * n + k];
            S.F[int64_t(tid) * n + k] = S.F[int64_t(tid) * n + sel];
            S.F[int64_t(tid) * n + sel] = t;
          }
          if (tid == 0) {
            double t = S.cn2[k];
            S.cn2[k] = S.cn2[sel];
            S.cn2[sel] = t;
            const int ti = S.piv[k];
            S.piv[k] = S.piv[sel];
            S.piv[sel] = ti;
            ipos[S.piv[k]] = k;
            ipos[ti] = sel;
          }
          __syncthreads();
        }
        double* wk = W + int64_t(k) * ldw;
        // a_k -= V_blk F_k^T over rows k0.. (block-start values -> current)
        for (int r = k0 + tid; r < m; r += NT) {
          double a = wk[r];
          for (int t = 0; t < i; ++t) a = fma(-VB(r, t), S.F[int64_t(t) * n + k], a);
          wk[r] = a;
        }
        __syncthreads();
        double s = 0.0;
        for (int r = k + tid; r < m; r += NT) s = fma(wk[r], wk[r], s);
        const double normsq = block_sum(s, redd);
        const double pivot_norm = sqrt(normsq);
        if (k == 0) r11 = pivot_norm;
        const bool diag_done = pivot_norm <= job.tol * r11;
        const bool floor_hit = pivot_norm <= 1e-15 * r11;
        const int halt = floor_hit || (diag_done && !members_not_done);
        if (tid == 0) S.ctl[0] = halt;
        if (!halt) {
          // make_reflector (linalg.cpp:152-178): v = a - alpha e_k, tau = 2 / v^T v.
          const double a0 = wk[k];
          const double alpha = (a0 >= 0.0) ? -pivot_norm : pivot_norm;
          double* vk = S.V + int64_t(k) * m;
          for (int r = tid; r < m; r += NT) vk[r] = r < k ? 0.0 : (r == k ? a0 - alpha : wk[r]);
          __syncthreads();
          double vs = 0.0;
          for (int r = k + tid; r < m; r += NT) vs = fma(vk[r], vk[r], vs);
          const double vn = block_sum(vs, redd);
          const double tau = (pivot_norm == 0.0 || vn == 0.0) ? 0.0 : 2.0 / vn;
          for (int r = k + 1 + tid; r < m; r += NT) wk[r] = 0.0;
          if (tid == 0) {
            wk[k] = alpha;
            S.tau[k] = tau;
          }
          // wv[t] = V_t^T v over rows k.. for the block's earlier reflectors.
          for (int t = warp; t < i; t += NW) {
            double d = 0.0;
            for (int r = k + lane; r < m; r += 32) d = fma(VB(r, t), vk[r], d);
            d = warp_sum(d);
            if (lane == 0) S.wv[t] = d;
          }
        }
      }
      cluster.sync();
      if (__ldcg(&S.ctl[0])) {
        stop = true;
        break;
      }
      long long tc2 = clock64();
      t_lead += tc2 - tc1;
      // ---- every CTA: the new reflector into its block copy
      const double* vk = S.V + int64_t(k) * m;
      for (int r = tid; r < m; r += NT) {
        const double v = __ldcg(&vk[r]);
        vsh[r] = v;
        VB(r, i) = v;
      }
      if (tid < i) wvs[tid] = __ldcg(&S.wv[tid]);
      if (tid == 0) sh_tau = __ldcg(&S.tau[k]);
      __syncthreads();
      const double tau = sh_tau;
      // ---- column pass: one read of every trailing column (block-start values).
      // A warp takes TC = 16 columns at a time: every lane accumulates partial
      // dot products of all 16 columns over its rows, row chunk by row chunk
      // (16 independent coalesced loads in flight per lane), a transpose-
      // reduction leaves column c's v^T a_j on lanes c and c + 16, and lane
      // c < 16 then finishes its own column.
      constexpr int TC = 16;
      lmax = -1.0;
      const int l1 = own.below(k + 1);
      // Tiles are TC-aligned in the local index, so a tile's positions are
      // consecutive (TC divides CB); columns below l1 are masked out.
      const int lt0 = l1 & ~(TC - 1);
      for (int li0 = lt0 + warp * TC; li0 < nloc; li0 += NW * TC) {
        const int cnt = min(TC, nloc - li0);
        const int c0 = li0 < l1 ? l1 - li0 : 0;  // first live column of the tile
        const double* base = W + int64_t(own.l2g(li0)) * ldw;
        double acc[TC];
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[c] = 0.0;
        // Rows in 16-byte pairs from the even row ke <= k (ldw is even, so
        // every pair is aligned): 16 columns x 16 bytes in flight per lane.
        const int ke = k & ~1;
        for (int r = ke + 2 * lane; r < m; r += 64) {
          const double v0 = r >= k ? vsh[r] : 0.0, v1 = r + 1 < m ? vsh[r + 1] : 0.0;
          double2 a[TC];
#pragma unroll
          for (int c = 0; c < TC; ++c)
            a[c] = (c >= c0 && c < cnt) ? __ldcg(reinterpret_cast<const double2*>(&base[int64_t(c) * ldw + r]))
                                        : make_double2(0.0, 0.0);
          if (r <= k && k <= r + 1) {  // row k of the tile's columns
#pragma unroll
            for (int c = 0; c < TC; ++c) rowk[warp * TC + c] = r == k ? a[c].x : a[c].y;
          }
#pragma unroll
          for (int c = 0; c < TC; ++c) acc[c] = fma(v1, a[c].y, fma(v0, a[c].x, acc[c]));
        }
        __syncwarp();
#pragma unroll
        for (int off = TC / 2; off > 0; off >>= 1) {
          const bool upper = (lane & off) != 0;
#pragma unroll
          for (int c = 0; c < off; ++c) {
            const double send = upper ? acc[c] : acc[c + off];
            const double keep = upper ? acc[c + off] : acc[c];
            acc[c] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 16);  // lanes c and c + 16 hold column c
        if (lane >= c0 && lane < cnt) {
          const int j = own.l2g(li0 + lane);
          const double d = acc[0];
          const double akj = rowk[warp * TC + lane];
          double* Fj = S.F + j;  // F is stored t-major: F(j, t) at F[t * n + j] (coalesced over j)
          double corr = 0.0, rc = 0.0;
          for (int t = 0; t < i; ++t) {
            const double ft = Fj[int64_t(t) * n];
            corr = fma(wvs[t], ft, corr);
            rc = fma(VB(k, t), ft, rc);
          }
          const double f = tau * (d - corr);
          Fj[int64_t(i) * n] = f;
          // r_kj = a_kj - sum_{t <= i} V(k, t) F(j, t)
          const double rkj = akj - rc - VB(k, i) * f;
          const double nc = fmax(0.0, S.cn2[j] - rkj * rkj);
          S.cn2[j] = nc;
          lmax = fmax(lmax, nc);
        }
        __syncwarp();  // rowk is rewritten by the next tile
      }
      {
        const double mx = block_max(lmax, redd);
        if (tid == 0) slot.d = mx;
      }
      long long tc3 = clock64();
      t_pass += tc3 - tc2;
      cluster.sync();  // every column's norm of this step is in place
      member_masses(k);
      cluster.sync();
      members_not_done = false;
      for (int g = 0; g < nmem; ++g) members_not_done |= __ldcg(&S.acc[g]) > __ldcg(&S.mt[g]);
      ++rank;
      t_mem += clock64() - tc3;
    }
    long long tb0 = clock64();
    // ---- block end: rank-nb trailing update + exact norms of the trailing columns
    const int nb = rank - k0;
    if (stop || k >= kmax || nb == 0) break;
    // W(k0:m, trailing) -= V_blk F_blk^T on the DMMA path: a warp takes 8
    // consecutive trailing columns (8-aligned local index, so contiguous
    // positions), keeps their F rows as B fragments in registers and walks
    // the rows in 16-row fragments (C loaded, two m16n8k16 steps with A = -V
    // from shared memory, stored back); the updated column norms over rows
    // >= k accumulate on the fly.
    lmax = -1.0;
    const int l1 = own.below(k);
    const int g = lane >> 2, tq = lane & 3;
    for (int lg = (l1 & ~7) + warp * 8; lg < nloc; lg += NW * 8) {
      const int c0 = lg < l1 ? l1 - lg : 0;
      const int cnt = min(8, nloc - lg);
      const int jb = own.l2g(lg);
      // B fragments: b_i = F(kk + tq + 4i, jb + g), zero past nb / dead columns.
      double bf[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int t = 16 * h + tq + 4 * q;
          bf[h][q] = (t < nb && g >= c0 && g < cnt) ? S.F[int64_t(t) * n + jb + g] : 0.0;
        }
      // This lane's C columns: jb + 2 tq + {0, 1}.
      const bool live0 = 2 * tq >= c0 && 2 * tq < cnt, live1 = 2 * tq + 1 >= c0 && 2 * tq + 1 < cnt;
      double* col0 = W + int64_t(jb + 2 * tq) * ldw;
      double* col1 = col0 + ldw;
      double s0 = 0.0, s1 = 0.0;
      for (int r0 = k0; r0 < m; r0 += 16) {
        double c[4];
        const int ra = r0 + g, rb = r0 + g + 8;
        c[0] = (live0 && ra < m) ? col0[ra] : 0.0;
        c[1] = (live1 && ra < m) ? col1[ra] : 0.0;
        c[2] = (live0 && rb < m) ? col0[rb] : 0.0;
        c[3] = (live1 && rb < m) ? col1[rb] : 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double af[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = r0 + g + 8 * (q % 2), t = 16 * h + tq + 4 * (q / 2);
            af[q] = (r < m && t < nb) ? -VB(r, t) : 0.0;  // stale columns may hold NaN patterns
          }
          asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
              "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
              : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
              : "d"(af[0]), "d"(af[1]), "d"(af[2]), "d"(af[3]), "d"(af[4]), "d"(af[5]), "d"(af[6]), "d"(af[7]),
                "d"(bf[h][0]), "d"(bf[h][1]), "d"(bf[h][2]), "d"(bf[h][3]));
        }
        if (ra < m) {
          if (live0) col0[ra] = c[0];
          if (live1) col1[ra] = c[1];
          if (ra >= k) {
            s0 = fma(c[0], c[0], s0);
            s1 = fma(c[1], c[1], s1);
          }
        }
        if (rb < m) {
          if (live0) col0[rb] = c[2];
          if (live1) col1[rb] = c[3];
          if (rb >= k) {
            s0 = fma(c[2], c[2], s0);
            s1 = fma(c[3], c[3], s1);
          }
        }
      }
      // Column norms: reduce over the 8 lanes with the same tq (g = lane >> 2).
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      if (g == 0) {
        if (live0) {
          S.cn2[jb + 2 * tq] = s0;
          lmax = fmax(lmax, s0);
        }
        if (live1) {
          S.cn2[jb + 2 * tq + 1] = s1;
          lmax = fmax(lmax, s1);
        }
      }
    }
    {
      const double mx = block_max(lmax, redd);
      if (tid == 0) slot.d = mx;
    }
    cluster.sync();
    t_upd += clock64() - tb0;
  }
  cluster.sync();

  if (lead && tid == 0 && job.dbg) {
    job.dbg[0] = double(t_piv);
    job.dbg[1] = double(t_lead);
    job.dbg[2] = double(t_pass);
    job.dbg[3] = double(t_mem);
    job.dbg[4] = double(rank);
    job.dbg[5] = double(n);
    job.dbg[8] = double(t_upd);
  }
  // form_q (linalg.cpp:181-185): Q = H_0 ... H_{rank-1} I; a warp per column
  // of Q, columns split over the cluster. Output row-major Q[i*m + j].
  {
    double* Q = job.Q;
    const int jc0 = (m * cr) / G, jc1 = (m * (cr + 1)) / G;
    for (int j = jc0 + warp; j < jc1; j += NW) {
      // q = e_j; for k = rank-1..0: q -= tau_k v_k (v_k^T q). Rows live in
      // registers, 32-strided over the lanes (m <= 32 * 12 rows).
      constexpr int RPL = 12;
      double q[RPL];
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int r = lane + 32 * u;
        q[u] = (r < m && r == j) ? 1.0 : 0.0;
      }
      for (int kk = rank - 1; kk >= 0; --kk) {
        const double tk = __ldcg(&S.tau[kk]);
        if (tk == 0.0) continue;
        const double* v = S.V + int64_t(kk) * m;
        double d = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int r = lane + 32 * u;
          if (r < m && r >= kk) d = fma(__ldcg(&v[r]), q[u], d);
        }
        d = warp_sum(d) * tk;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int r = lane + 32 * u;
          if (r < m && r >= kk) q[u] = fma(-d, __ldcg(&v[r]), q[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int r = lane + 32 * u;
        if (r < m) Q[int64_t(r) * m + j] = q[u];
      }
    }
  }
  if (lead && tid == 0) *job.rank_out = rank;
}

size_t qrb_smem_bytes(int max_m, int max_nmem) {
  (void)max_nmem;
  return sizeof(double) * (size_t(max_m) * NB + size_t(max_m) + NB + 8);
}

cudaLaunchConfig_t qrb_config(int njobs, int cluster, size_t smem, cudaStream_t st, cudaLaunchAttribute* at) {
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

}  // namespace

size_t qrb_scratch_doubles(int m, int n, int nmem) { return scr_doubles(m, n, nmem); }

int qrb_max_rows() { return 32 * 12; }

void launch_qrb(const QrJob* jobs, int njobs, int max_m, int max_nmem, int cluster, cudaStream_t st) {
  if (njobs <= 0) return;
  const size_t smem = qrb_smem_bytes(max_m, max_nmem);
  cuda_check(cudaFuncSetAttribute(qrb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
             "qrb smem attribute");
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = qrb_config(njobs, cluster, smem, st, at);
  cuda_check(cudaLaunchKernelEx(&cfg, qrb_kernel, jobs, max_nmem, max_m), "qrb launch");
}

// Cluster size for a batch whose typical basis has n columns: a cluster of g
// CTAs splits the panel's CB-column blocks, so its speed-up is at most the
// number of blocks; waves / min(g, blocks) is minimised (small batches of
// compressed panels take large clusters, large batches small ones).
int qrb_cluster_size(int njobs, int typ_n, int max_m, int max_nmem) {
  const size_t smem = qrb_smem_bytes(max_m, max_nmem);
  cudaFuncSetAttribute(qrb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int best = 1;
  double best_cost = 1e30;
  const int nblk = std::max(1, (typ_n + CB - 1) / CB);
  if (const char* e = getenv("H2G_QRB_CLUSTER")) {  // experiment override
    const int g = atoi(e);
    if (g >= 1 && g <= 8) return std::min(g, std::max(1, nblk));
  }
  for (int g = 1; g <= 8; ++g) {
    if (g > 1 && g > nblk) break;
    int fit = 0;
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = qrb_config(g, g, smem, nullptr, at);
    if (cudaOccupancyMaxActiveClusters(&fit, qrb_kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      fit = 0;
    }
    if (fit <= 0) continue;
    const int waves = (njobs + fit - 1) / fit;
    const double cost = double(waves) / std::min(g, nblk) * (1.0 + 0.02 * (g - 1));
    if (cost < best_cost) {
      best_cost = cost;
      best = g;
    }
  }
  return best;
}

}  // namespace h2g
