// Cluster tree (2-means bisection) and block classification on the GPU,
// bitwise equal to the reference build_cluster_tree / classify_blocks
// (geometry.cpp:130-277, hstructure.cpp:64-114).
//
// Per level all nodes are processed at once:
//   seed_kernel    farthest pair of 32 strided candidates (first strict max
//                  in (a, b) loop order), one warp per node;
//   lloyd_kernel   <=100 Lloyd iterations, one CTA per node: assignment in
//                  parallel, centroid sums as sequential chains over the
//                  members compacted per chunk in shared memory (one warp
//                  per cluster), then the signed margins;
//   merge passes   stable merge sort of the margins inside every node, each
//                  element placed by binary search in the sibling run
//                  (std::stable_sort semantics incl. -0.0 == +0.0);
//   split_kernel   n1 = #(margin < 0) clamped, child ranges;
//   gather_kernel  permutes points, charges and original indices.
// compute_geometry: sequential centre sums per (node, dim) and a parallel
// max for the radius (max is order independent).
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "tree.hpp"

namespace h2g {

namespace {

__device__ __forceinline__ double d2(double ax, double ay, double az, double bx, double by,
                                     double bz) {
  const double dx = ax - bx, dy = ay - by, dz = az - bz;
  return fma(dz, dz, fma(dx, dx, dy * dy));
}

struct TreeBufs {
  double* x;
  double* y;
  double* z;
};

__global__ void seed_kernel(TreeBufs P, const int64_t* be, int level, double* cent) {
  const int node = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (node >= (1 << level)) return;
  const int64_t hb = (int64_t(1) << level) - 1 + node;
  const int64_t b = be[2 * hb], e = be[2 * hb + 1], len = e - b;
  const int64_t ncand = len < 32 ? len : 32;
  // Pair (a, bb) linear index in loop order.
  double best = -1.0;
  int besti = 0x7fffffff;
  int t = 0;
  for (int a = 0; a < ncand; ++a)
    for (int bb = a + 1; bb < ncand; ++bb, ++t) {
      if ((t & 31) != lane) continue;
      const int64_t ia = b + (ncand == 1 ? 0 : a * (len - 1) / (ncand - 1));
      const int64_t ib = b + (ncand == 1 ? 0 : bb * (len - 1) / (ncand - 1));
      const double d = d2(P.x[ia], P.y[ia], P.z[ia], P.x[ib], P.y[ib], P.z[ib]);
      if (d > best) {
        best = d;
        besti = t;
      }
    }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const int oi = __shfl_down_sync(0xffffffffu, besti, o);
    if (ob > best || (ob == best && oi < besti)) {
      best = ob;
      besti = oi;
    }
  }
  if (lane == 0) {
    int64_t i1 = b, i2 = e - 1;
    if (best > -1.0) {
      int tt = 0;
      for (int a = 0; a < ncand; ++a)
        for (int bb = a + 1; bb < ncand; ++bb, ++tt)
          if (tt == besti) {
            i1 = b + (ncand == 1 ? 0 : a * (len - 1) / (ncand - 1));
            i2 = b + (ncand == 1 ? 0 : bb * (len - 1) / (ncand - 1));
          }
    }
    double* c = cent + 6 * node;
    c[0] = P.x[i1]; c[1] = P.y[i1]; c[2] = P.z[i1];
    c[3] = P.x[i2]; c[4] = P.y[i2]; c[5] = P.z[i2];
  }
}

constexpr int LT = 256;

// Lloyd iterations of one node (geometry.cpp:148-170). Per iteration the
// points stream through in chunks of LT (one point per thread, the next
// chunk prefetched into registers): each thread assigns its point, the
// chunk's members are compacted in point order into shared memory per
// cluster (ballot + warp-count scan), and lanes 0-2 of warp 0 (cluster 0)
// and warp 1 (cluster 1) extend their sequential coordinate sums over the
// compacted members. Each chain adds exactly the reference's members in the
// reference's order, so the sums are bitwise the reference's; the two
// clusters' chains run concurrently and never wait on global loads.
__global__ void __launch_bounds__(LT) lloyd_kernel(TreeBufs P, const int64_t* be, int level,
                                                   double* cent, unsigned char* assign,
                                                   double* margin) {
  __shared__ double c[6];
  __shared__ double sums[6];
  __shared__ int wc[LT / 32];
  __shared__ double mv[2][3][LT];
  const int node = blockIdx.x;
  const int64_t hb = (int64_t(1) << level) - 1 + node;
  const int64_t b = be[2 * hb], e = be[2 * hb + 1], len = e - b;
  const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const bool chain = wid < 2 && ln < 3;
  if (threadIdx.x < 6) c[threadIdx.x] = cent[6 * node + threadIdx.x];
  for (int64_t i = threadIdx.x; i < len; i += LT) assign[b + i] = 0;
  __syncthreads();
  for (int iter = 0; iter < 100; ++iter) {
    int changed = 0;
    double s = 0.0;
    int64_t n1 = 0;  // members of cluster 0 (uniform)
    double px = 0.0, py = 0.0, pz = 0.0;
    unsigned char pa = 0;
    if (threadIdx.x < len) {
      px = P.x[b + threadIdx.x]; py = P.y[b + threadIdx.x]; pz = P.z[b + threadIdx.x];
      pa = assign[b + threadIdx.x];
    }
    for (int64_t i0 = 0; i0 < len; i0 += LT) {
      const int64_t i = i0 + threadIdx.x;
      const bool live = i < len;
      const double cx = px, cy = py, cz = pz;
      const unsigned char old = pa;
      if (i + LT < len) {
        px = P.x[b + i + LT]; py = P.y[b + i + LT]; pz = P.z[b + i + LT];
        pa = assign[b + i + LT];
      }
      unsigned char a = 0;
      if (live) {
        a = d2(cx, cy, cz, c[3], c[4], c[5]) < d2(cx, cy, cz, c[0], c[1], c[2]);
        if (a != old) {
          assign[b + i] = a;
          changed = 1;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, live && a == 0);
      if (ln == 0) wc[wid] = __popc(bal);
      __syncthreads();  // also: the previous chunk's chains are done with mv
      int off = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < LT / 32; ++w) {
        const int cw = wc[w];
        off += w < wid ? cw : 0;
        tot += cw;
      }
      if (live) {
        const int r0 = off + __popc(bal & ((1u << ln) - 1u));
        const int cl = a == 0 ? 0 : 1, r = a == 0 ? r0 : threadIdx.x - r0;
        mv[cl][0][r] = cx;
        mv[cl][1][r] = cy;
        mv[cl][2][r] = cz;
      }
      __syncthreads();
      if (chain) {
        const int64_t rem = len - i0;
        const int m = wid == 0 ? tot : int(rem < LT ? rem : LT) - tot;
        const double* v = mv[wid][ln];
        int k = 0;
        for (; k + 8 <= m; k += 8) {
          double t[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) t[u] = v[k + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) s += t[u];
        }
        for (; k < m; ++k) s += v[k];
      }
      n1 += tot;
    }
    changed = __syncthreads_or(changed);
    if (chain) sums[3 * wid + ln] = s;
    __syncthreads();
    if (threadIdx.x < 6) {
      if (threadIdx.x < 3) {
        if (n1 > 0) c[threadIdx.x] = sums[threadIdx.x] / double(n1);
      } else {
        if (len - n1 > 0) c[threadIdx.x] = sums[threadIdx.x] / double(len - n1);
      }
    }
    __syncthreads();
    if (!changed && iter > 0) break;
  }
  for (int64_t i = threadIdx.x; i < len; i += LT) {
    const int64_t p = b + i;
    const double px = P.x[p], py = P.y[p], pz = P.z[p];
    margin[p] = d2(px, py, pz, c[0], c[1], c[2]) - d2(px, py, pz, c[3], c[4], c[5]);
  }
}

__global__ void node_of_kernel(const int64_t* be, int level, int* node_of) {
  const int node = blockIdx.x;
  const int64_t hb = (int64_t(1) << level) - 1 + node;
  for (int64_t i = be[2 * hb] + threadIdx.x; i < be[2 * hb + 1]; i += blockDim.x) node_of[i] = node;
}

__global__ void init_sort_kernel(const double* margin, double* key, int* idx, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) {
    key[i] = margin[i];
    idx[i] = int(i);
  }
}

// One bottom-up merge pass of width w inside every node.
__global__ void merge_pass_kernel(const int64_t* be, int level, const int* node_of,
                                  const double* kin, const int* iin, double* kout, int* iout,
                                  int64_t n, int64_t w) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t hb = (int64_t(1) << level) - 1 + node_of[i];
  const int64_t b = be[2 * hb], len = be[2 * hb + 1] - b;
  const int64_t local = i - b;
  const int64_t base = (local / (2 * w)) * (2 * w);
  const int64_t mid = min(base + w, len), end = min(base + 2 * w, len);
  const double key = kin[i];
  int64_t pos;
  if (local < mid) {
    // count right-run keys strictly less than key
    int64_t lo = mid, hi = end;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (kin[b + m] < key) lo = m + 1; else hi = m;
    }
    pos = base + (local - base) + (lo - mid);
  } else {
    // count left-run keys <= key, i.e. !(key < k)
    int64_t lo = base, hi = mid;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (!(key < kin[b + m])) lo = m + 1; else hi = m;
    }
    pos = base + (local - mid) + (lo - base);
  }
  kout[b + pos] = key;
  iout[b + pos] = iin[i];
}

// n1 = #(margin < 0) clamped to [min_side, len - min_side]; child ranges.
__global__ void split_kernel(int64_t* be, int level, const double* key, int64_t min_side) {
  __shared__ unsigned long long cnt;
  const int node = blockIdx.x;
  const int64_t hb = (int64_t(1) << level) - 1 + node;
  const int64_t b = be[2 * hb], e = be[2 * hb + 1], len = e - b;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  unsigned long long c = 0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) c += key[b + i] < 0.0;
  atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    long long n1 = cnt;
    if (n1 < min_side) n1 = min_side;
    if (n1 > len - min_side) n1 = len - min_side;
    const int64_t ch = (int64_t(1) << (level + 1)) - 1 + 2 * node;
    be[2 * ch] = b;
    be[2 * ch + 1] = b + n1;
    be[2 * ch + 2] = b + n1;
    be[2 * ch + 3] = e;
  }
}

__global__ void gather_kernel(TreeBufs Pin, const double* qin, const int64_t* oin, TreeBufs Pout,
                              double* qout, int64_t* oout, const int* idx, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int s = idx[i];
  Pout.x[i] = Pin.x[s];
  Pout.y[i] = Pin.y[s];
  Pout.z[i] = Pin.z[s];
  qout[i] = qin[s];
  oout[i] = oin[s];
}

// compute_geometry (geometry.cpp:207-218), one CTA per node of all levels.
__global__ void geometry_kernel(TreeBufs P, const int64_t* be, double* geo) {
  __shared__ double c[3];
  __shared__ double red[32];
  const int64_t k = blockIdx.x;
  const int64_t b = be[2 * k], e = be[2 * k + 1], len = e - b;
  if (threadIdx.x < 3) {
    const double* src = threadIdx.x == 0 ? P.x : (threadIdx.x == 1 ? P.y : P.z);
    double s = 0.0;
    for (int64_t i = b; i < e; ++i) s += src[i];
    c[threadIdx.x] = s / double(len);
  }
  __syncthreads();
  double r2 = 0.0;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x)
    r2 = fmax(r2, d2(P.x[i], P.y[i], P.z[i], c[0], c[1], c[2]));
  for (int o = 16; o > 0; o >>= 1) r2 = fmax(r2, __shfl_down_sync(0xffffffffu, r2, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
    geo[4 * k] = c[0];
    geo[4 * k + 1] = c[1];
    geo[4 * k + 2] = c[2];
    geo[4 * k + 3] = sqrt(r);
  }
}

__global__ void distinct_kernel(TreeBufs P, int64_t n, int* flag) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= 1 && i < n && d2(P.x[i], P.y[i], P.z[i], P.x[0], P.y[0], P.z[0]) > 0.0) *flag = 1;
}

__global__ void iota_kernel(int64_t* o, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) o[i] = i;
}

__global__ void aos_to_soa_kernel(const double* xyz, TreeBufs P, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) {
    P.x[i] = xyz[3 * i];
    P.y[i] = xyz[3 * i + 1];
    P.z[i] = xyz[3 * i + 2];
  }
}

// ---- classification -------------------------------------------------------
// Candidates of row i at level l are the children of its parent's near list
// (or {0, 1} at level 1), generated in ascending order, so near/far lists come
// out sorted exactly like the reference's std::sort.
__global__ void cand_count_kernel(int level, const int64_t* pnear_ptr, int64_t* cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= (int64_t(1) << level)) return;
  cnt[i] = level == 1 ? 2 : 2 * (pnear_ptr[(i >> 1) + 1] - pnear_ptr[i >> 1]);
}

__global__ void classify_kernel(int level, int weak, double eta, const double* geo,
                                const int64_t* pnear_ptr, const int64_t* pnear_idx,
                                const int64_t* cand_ptr, int64_t ncand_total, int64_t* cand_col,
                                unsigned char* cand_far) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= ncand_total) return;
  // Row by binary search over cand_ptr.
  int64_t lo = 0, hi = (int64_t(1) << level);
  while (hi - lo > 1) {
    const int64_t m = (lo + hi) >> 1;
    if (cand_ptr[m] <= t) lo = m; else hi = m;
  }
  const int64_t i = lo, r = t - cand_ptr[i];
  const int64_t J = level == 1 ? 0 : pnear_idx[pnear_ptr[i >> 1] + (r >> 1)];
  const int64_t j = 2 * J + (r & 1);
  cand_col[t] = j;
  bool far;
  if (weak) {
    far = i != j;
  } else {
    const double* a = geo + 4 * ((int64_t(1) << level) - 1 + i);
    const double* b = geo + 4 * ((int64_t(1) << level) - 1 + j);
    const double d = sqrt(d2(a[0], a[1], a[2], b[0], b[1], b[2]));
    far = d > eta * (a[3] + b[3]);
  }
  cand_far[t] = far;
}

// Per-row near/far counts (one thread per row, sequential over its candidates).
__global__ void row_counts_kernel(int level, const int64_t* cand_ptr, const unsigned char* cand_far,
                                  int64_t* ncnt, int64_t* fcnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= (int64_t(1) << level)) return;
  int64_t nn = 0, nf = 0;
  for (int64_t t = cand_ptr[i]; t < cand_ptr[i + 1]; ++t) (cand_far[t] ? nf : nn)++;
  ncnt[i] = nn;
  fcnt[i] = nf;
}

__global__ void compact_kernel(int level, const int64_t* cand_ptr, const unsigned char* cand_far,
                               const int64_t* cand_col, const int64_t* near_ptr,
                               const int64_t* far_ptr, int64_t* near_idx, int64_t* far_idx) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= (int64_t(1) << level)) return;
  int64_t a = near_ptr[i], f = far_ptr[i];
  for (int64_t t = cand_ptr[i]; t < cand_ptr[i + 1]; ++t) {
    if (cand_far[t]) far_idx[f++] = cand_col[t];
    else near_idx[a++] = cand_col[t];
  }
}

// Exclusive scan of cnt[0..m) into ptr[0..m] (single CTA, sequential chunks).
__global__ void scan_kernel(const int64_t* cnt, int64_t* ptr, int64_t m) {
  __shared__ int64_t part[1024];
  const int64_t per = (m + blockDim.x - 1) / blockDim.x;
  const int64_t s = threadIdx.x * per, e = min(m, s + per);
  int64_t acc = 0;
  for (int64_t i = s; i < e; ++i) acc += cnt[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < int(blockDim.x); ++t) {
      const int64_t v = part[t];
      part[t] = run;
      run += v;
    }
    ptr[m] = run;
  }
  __syncthreads();
  acc = part[threadIdx.x];
  for (int64_t i = s; i < e; ++i) {
    ptr[i] = acc;
    acc += cnt[i];
  }
}

inline unsigned blocks(int64_t n, int t) { return unsigned((n + t - 1) / t); }

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " +
                                                 cudaGetErrorString(e));
}

}  // namespace

int tree_levels(int64_t n, int64_t leaf) {
  int levels = 0;
  while ((int64_t(1) << levels) * leaf < n) ++levels;
  return levels;
}

void build_tree_device(DeviceTree& T, const double* d_xyz_aos, const double* d_q, int64_t n,
                       int64_t leaf, cudaStream_t st) {
  if (leaf < 2) throw std::invalid_argument("build_cluster_tree: leaf_size must be >= 2");
  if (n < 2 * leaf) throw std::invalid_argument("build_cluster_tree: need N >= 2 * leaf_size");
  T.n = n;
  T.levels = tree_levels(n, leaf);
  T.leaf = leaf;
  const int L = T.levels;
  const int64_t nn = (int64_t(1) << (L + 1)) - 1;
  T.alloc(n, nn);
  TreeBufs A{T.x, T.y, T.z}, B{T.x2, T.y2, T.z2};
  aos_to_soa_kernel<<<blocks(n, 256), 256, 0, st>>>(d_xyz_aos, A, n);
  check(cudaMemcpyAsync(T.q, d_q, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "q copy");
  iota_kernel<<<blocks(n, 256), 256, 0, st>>>(T.order, n);
  check(cudaMemsetAsync(T.flag, 0, sizeof(int), st), "memset");
  distinct_kernel<<<blocks(n, 256), 256, 0, st>>>(A, n, T.flag);
  int flag = 0;
  check(cudaMemcpyAsync(&flag, T.flag, sizeof(int), cudaMemcpyDeviceToHost, st), "flag");
  check(cudaStreamSynchronize(st), "distinct");
  if (!flag) throw std::runtime_error("build_cluster_tree: degenerate cloud, all points identical");
  const int64_t root[2] = {0, n};
  check(cudaMemcpyAsync(T.be, root, sizeof(root), cudaMemcpyHostToDevice, st), "root");
  for (int level = 0; level < L; ++level) {
    const int nodes = 1 << level;
    const int64_t min_side = int64_t(1) << (L - level - 1);
    seed_kernel<<<(nodes + 7) / 8, 256, 0, st>>>(A, T.be, level, T.cent);
    lloyd_kernel<<<nodes, LT, 0, st>>>(A, T.be, level, T.cent, T.assign, T.margin);
    node_of_kernel<<<nodes, 256, 0, st>>>(T.be, level, T.node_of);
    init_sort_kernel<<<blocks(n, 256), 256, 0, st>>>(T.margin, T.key0, T.idx0, n);
    // Every node keeps >= 2^(L-level) points (the min_side clamp), which bounds its length.
    const int64_t maxlen = n - int64_t(nodes - 1) * (int64_t(1) << (L - level));
    double* kin = T.key0; double* kout = T.key1;
    int* iin = T.idx0; int* iout = T.idx1;
    for (int64_t w = 1; w < maxlen; w *= 2) {
      merge_pass_kernel<<<blocks(n, 256), 256, 0, st>>>(T.be, level, T.node_of, kin, iin, kout,
                                                         iout, n, w);
      std::swap(kin, kout);
      std::swap(iin, iout);
    }
    split_kernel<<<nodes, 256, 0, st>>>(T.be, level, kin, min_side);
    gather_kernel<<<blocks(n, 256), 256, 0, st>>>(A, T.q, T.order, B, T.q2, T.order2, iin, n);
    std::swap(T.x, T.x2); std::swap(T.y, T.y2); std::swap(T.z, T.z2);
    std::swap(T.q, T.q2); std::swap(T.order, T.order2);
    A = TreeBufs{T.x, T.y, T.z};
    B = TreeBufs{T.x2, T.y2, T.z2};
  }
  geometry_kernel<<<unsigned(nn), 256, 0, st>>>(A, T.be, T.geo);
  check(cudaGetLastError(), "tree kernels");
}

void classify_device(DeviceTree& T, double eta, int weak, Structure& S, cudaStream_t st) {
  const int L = T.levels;
  S.levels = L;
  S.level.assign(L + 1, {});
  int64_t* d_pnear_ptr = nullptr;
  int64_t* d_pnear_idx = nullptr;
  std::vector<void*> to_free;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    check(cudaMallocAsync(&p, bytes < 8 ? 8 : bytes, st), "classify alloc");
    to_free.push_back(p);
    return p;
  };
  for (int l = 1; l <= L; ++l) {
    const int64_t m = int64_t(1) << l;
    auto* cnt = static_cast<int64_t*>(dalloc(8 * m));
    auto* cptr = static_cast<int64_t*>(dalloc(8 * (m + 1)));
    cand_count_kernel<<<blocks(m, 256), 256, 0, st>>>(l, d_pnear_ptr, cnt);
    scan_kernel<<<1, 1024, 0, st>>>(cnt, cptr, m);
    int64_t total = 0;
    check(cudaMemcpyAsync(&total, cptr + m, 8, cudaMemcpyDeviceToHost, st), "cand total");
    check(cudaStreamSynchronize(st), "cand total");
    auto* ccol = static_cast<int64_t*>(dalloc(8 * total));
    auto* cfar = static_cast<unsigned char*>(dalloc(total));
    classify_kernel<<<blocks(total, 256), 256, 0, st>>>(l, weak, eta, T.geo, d_pnear_ptr,
                                                        d_pnear_idx, cptr, total, ccol, cfar);
    auto* ncnt = static_cast<int64_t*>(dalloc(8 * m));
    auto* fcnt = static_cast<int64_t*>(dalloc(8 * m));
    row_counts_kernel<<<blocks(m, 256), 256, 0, st>>>(l, cptr, cfar, ncnt, fcnt);
    auto* nptr = static_cast<int64_t*>(dalloc(8 * (m + 1)));
    auto* fptr = static_cast<int64_t*>(dalloc(8 * (m + 1)));
    scan_kernel<<<1, 1024, 0, st>>>(ncnt, nptr, m);
    scan_kernel<<<1, 1024, 0, st>>>(fcnt, fptr, m);
    int64_t tn = 0, tf = 0;
    check(cudaMemcpyAsync(&tn, nptr + m, 8, cudaMemcpyDeviceToHost, st), "near total");
    check(cudaMemcpyAsync(&tf, fptr + m, 8, cudaMemcpyDeviceToHost, st), "far total");
    check(cudaStreamSynchronize(st), "totals");
    auto* nidx = static_cast<int64_t*>(dalloc(8 * tn));
    auto* fidx = static_cast<int64_t*>(dalloc(8 * tf));
    compact_kernel<<<blocks(m, 256), 256, 0, st>>>(l, cptr, cfar, ccol, nptr, fptr, nidx, fidx);
    auto& LP = S.level[l];
    LP.near_ptr.resize(m + 1);
    LP.far_ptr.resize(m + 1);
    LP.near_idx.resize(tn);
    LP.far_idx.resize(tf);
    check(cudaMemcpyAsync(LP.near_ptr.data(), nptr, 8 * (m + 1), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaMemcpyAsync(LP.far_ptr.data(), fptr, 8 * (m + 1), cudaMemcpyDeviceToHost, st), "d2h");
    if (tn) check(cudaMemcpyAsync(LP.near_idx.data(), nidx, 8 * tn, cudaMemcpyDeviceToHost, st), "d2h");
    if (tf) check(cudaMemcpyAsync(LP.far_idx.data(), fidx, 8 * tf, cudaMemcpyDeviceToHost, st), "d2h");
    d_pnear_ptr = nptr;
    d_pnear_idx = nidx;
  }
  check(cudaStreamSynchronize(st), "classify");
  for (void* p : to_free) cudaFreeAsync(p, st);
}

}  // namespace h2g

namespace h2g {

void DeviceTree::alloc(int64_t n_, int64_t nodes) {
  // A rebuild of the same size (every step of a factorization sequence) keeps
  // its buffers: 21 cudaFree + cudaMalloc pairs would each synchronise the device.
  if (!owned.empty() && alloc_n == n_ && alloc_nodes == nodes) return;
  for (void* p : owned) cudaFree(p);
  owned.clear();
  alloc_n = n_;
  alloc_nodes = nodes;
  auto get = [&](size_t bytes) {
    void* p = nullptr;
    check(cudaMalloc(&p, bytes < 8 ? 8 : bytes), "tree alloc");
    owned.push_back(p);
    return p;
  };
  x = static_cast<double*>(get(8 * n_));
  y = static_cast<double*>(get(8 * n_));
  z = static_cast<double*>(get(8 * n_));
  q = static_cast<double*>(get(8 * n_));
  order = static_cast<int64_t*>(get(8 * n_));
  x2 = static_cast<double*>(get(8 * n_));
  y2 = static_cast<double*>(get(8 * n_));
  z2 = static_cast<double*>(get(8 * n_));
  q2 = static_cast<double*>(get(8 * n_));
  order2 = static_cast<int64_t*>(get(8 * n_));
  be = static_cast<int64_t*>(get(16 * nodes));
  geo = static_cast<double*>(get(32 * nodes));
  cent = static_cast<double*>(get(48 * nodes));
  assign = static_cast<unsigned char*>(get(n_));
  margin = static_cast<double*>(get(8 * n_));
  key0 = static_cast<double*>(get(8 * n_));
  key1 = static_cast<double*>(get(8 * n_));
  idx0 = static_cast<int*>(get(4 * n_));
  idx1 = static_cast<int*>(get(4 * n_));
  node_of = static_cast<int*>(get(4 * n_));
  flag = static_cast<int*>(get(4));
}

void DeviceTree::release_scratch() {}

DeviceTree::~DeviceTree() {
  for (void* p : owned) cudaFree(p);
}

}  // namespace h2g
