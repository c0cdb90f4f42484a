// extern "C" boundary (include/h2g.h). Converts C++ exceptions into status
// codes + h2g_last_error(), copies host buffers in/out, and exposes the
// factor objects for inspection and parity tests.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/h2g.h"
#include "h2.hpp"

struct h2g_problem {
  h2g::Problem P;
};

struct h2g_comm {
  std::shared_ptr<h2g::Comm> c;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { h2g::cuda_check(cudaMalloc(&p, bytes ? bytes : 8), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  double* d() { return static_cast<double*>(p); }
};

// Host <-> device copies ordered on the problem's stream (a non-blocking
// stream is not ordered against the legacy default stream, and a pageable
// cudaMemcpy may return before its DMA lands), completed before returning.
void h2d(h2g::Problem& P, void* dst, const void* src, size_t bytes) {
  h2g::cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, P.c.stream), "h2d");
  h2g::cuda_check(cudaStreamSynchronize(P.c.stream), "h2d");
}
void d2h(h2g::Problem& P, void* dst, const void* src, size_t bytes) {
  h2g::cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, P.c.stream), "d2h");
  h2g::cuda_check(cudaStreamSynchronize(P.c.stream), "d2h");
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw std::runtime_error("h2g: no CUDA device (the B200 path has no CPU fallback)");
  }
}

}  // namespace

extern "C" {

const char* h2g_last_error(void) { return g_err.c_str(); }
int h2g_version(void) { return 1; }

int h2g_create(h2g_problem** out) {
  return guarded([&] {
    require_device();
    *out = new h2g_problem();
  });
}

void h2g_destroy(h2g_problem* p) { delete p; }

int h2g_set_kernel(h2g_problem* p, const h2g_kernel* k) {
  return guarded([&] {
    h2g::KernelParams kp;
    if (k->kind < 0 || k->kind > 2)
      throw std::invalid_argument("kernel: kind must be 0 (laplace), 1 (yukawa) or 2 (gaussian)");
    kp.kind = k->kind;
    kp.alpha_m = k->alpha_m;
    kp.scale = k->permittivity_scale;
    kp.reg = k->eta_reg;
    p->P.set_kernel(kp);
  });
}

int h2g_set_options(h2g_problem* p, const h2g_options* o) {
  return guarded([&] {
    if (o->tol <= 0) throw std::invalid_argument("config: tol must be positive");
    if (o->eta <= 0) throw std::invalid_argument("config: eta must be positive");
    auto& op = p->P.opt;
    op.tol = o->tol;
    op.cap = o->cap > 0 ? int(o->cap) : 0;
    op.rr_pivot_tol = o->rr_pivot_tol;
    op.absorb_coupling = o->absorb_coupling != 0;
    op.abort_residual_factor = o->abort_residual_factor;
    if (o->structure < 0 || o->structure > 2) throw std::invalid_argument("config: structure must be h2, hss or blr2");
    op.structure = o->structure;
    op.eta = o->eta;
    if (o->qr_mode < 0 || o->qr_mode > 2)
      throw std::invalid_argument("config: qr_mode must be 0 (exact), 1 (blocked) or 2 (compressed)");
    // Compressed mode drops up to eta >= 64 eps of each member's Gram trace
    // (batch.cu pchol), a relative member residual of sqrt(64 eps) ~ 1.2e-7;
    // below tol = 2.5e-7 the member rule (tol / 2) cannot be met, so those
    // tolerances run the blocked QR on the uncompressed panels instead.
    op.qr_mode = (o->qr_mode == 2 && o->tol < 2.5e-7) ? 1 : o->qr_mode;
    op.reference_compat = o->reference_compat != 0;
    if (o->qr_mem_budget > 0) {
      op.qr_mem_budget = size_t(o->qr_mem_budget);
      p->P.auto_budget_ = false;
    }
  });
}

int h2g_set_sampling(h2g_problem* p, int64_t sample_cols) {
  return guarded([&] {
    if (sample_cols < 0) throw std::invalid_argument("config: sample_cols must be >= 0");
    if (sample_cols > 0 && sample_cols < 64)
      throw std::invalid_argument("config: sample_cols must be 0 (off) or at least 64");
    p->P.opt.sample_cols = int(std::min<int64_t>(sample_cols, 1 << 30));
  });
}

void h2g_trim_memory(void) { h2g::trim_device_memory(); }

int h2g_build_dev(h2g_problem* p, int64_t n, const double* d_xyz, const double* d_q, int64_t leaf) {
  return guarded([&] { p->P.build(d_xyz, d_q, n, leaf); });
}

int h2g_build(h2g_problem* p, int64_t n, const double* xyz, const double* q, int64_t leaf) {
  return guarded([&] {
    DevBuf a(sizeof(double) * 3 * n), b(sizeof(double) * n);
    h2d(p->P, a.p, xyz, sizeof(double) * 3 * n);
    h2d(p->P, b.p, q, sizeof(double) * n);
    p->P.build(a.d(), b.d(), n, leaf);
  });
}

int h2g_factor(h2g_problem* p) {
  return guarded([&] { p->P.factor(); });
}

int h2g_solve_dev(h2g_problem* p, int64_t nrhs, const double* d_b, double* d_x) {
  return guarded([&] { p->P.solve(d_b, d_x, int(nrhs)); });
}

int h2g_solve(h2g_problem* p, int64_t nrhs, const double* b, double* x) {
  return guarded([&] {
    const size_t bytes = sizeof(double) * size_t(p->P.T.n) * nrhs;
    DevBuf db(bytes), dx(bytes);
    h2d(p->P, db.p, b, bytes);
    p->P.solve(db.d(), dx.d(), int(nrhs));
    d2h(p->P, x, dx.p, bytes);
  });
}

int h2g_matvec(h2g_problem* p, int64_t nrhs, const double* x, double* y) {
  return guarded([&] {
    const size_t bytes = sizeof(double) * size_t(p->P.T.n) * nrhs;
    DevBuf dx(bytes), dy(bytes);
    h2d(p->P, dx.p, x, bytes);
    p->P.matvec(dx.d(), dy.d(), int(nrhs));
    d2h(p->P, y, dy.p, bytes);
  });
}

int h2g_levels(h2g_problem* p) { return p->P.T.levels; }

int h2g_tree_perm(h2g_problem* p, int64_t* out) {
  return guarded([&] {
    d2h(p->P, out, p->P.T.order, sizeof(int64_t) * p->P.T.n);
  });
}

int h2g_nodes(h2g_problem* p, int64_t* be, double* geo) {
  return guarded([&] {
    const int64_t nn = (int64_t(1) << (p->P.T.levels + 1)) - 1;
    std::memcpy(be, p->P.be.data(), sizeof(int64_t) * 2 * nn);
    d2h(p->P, geo, p->P.T.geo, sizeof(double) * 4 * nn);
  });
}

int h2g_reordered_points(h2g_problem* p, double* xyz, double* q) {
  return guarded([&] {
    const int64_t n = p->P.T.n;
    std::vector<double> x(n), y(n), z(n);
    d2h(p->P, x.data(), p->P.T.x, 8 * n);
    d2h(p->P, y.data(), p->P.T.y, 8 * n);
    d2h(p->P, z.data(), p->P.T.z, 8 * n);
    d2h(p->P, q, p->P.T.q, 8 * n);
    for (int64_t i = 0; i < n; ++i) {
      xyz[3 * i] = x[i];
      xyz[3 * i + 1] = y[i];
      xyz[3 * i + 2] = z[i];
    }
  });
}

void check_level(h2g_problem* p, int level) {
  if (level < 0 || size_t(level) >= p->P.S.level.size())
    throw std::out_of_range("h2g_list: no level " + std::to_string(level));
}

int64_t h2g_list_count(h2g_problem* p, int level, int far) {
  int64_t out = -1;
  if (guarded([&] {
        check_level(p, level);
        const auto& L = p->P.S.level[size_t(level)];
        out = int64_t(far ? L.far_idx.size() : L.near_idx.size());
      }))
    return -1;
  return out;
}

int h2g_list(h2g_problem* p, int level, int far, int64_t* ptr, int64_t* idx) {
  return guarded([&] {
    check_level(p, level);
    const auto& L = p->P.S.level[size_t(level)];
    const auto& pv = far ? L.far_ptr : L.near_ptr;
    const auto& iv = far ? L.far_idx : L.near_idx;
    std::memcpy(ptr, pv.data(), sizeof(int64_t) * pv.size());
    if (!iv.empty()) std::memcpy(idx, iv.data(), sizeof(int64_t) * iv.size());
  });
}

int64_t h2g_near_entries(h2g_problem* p) {
  int64_t s = 0;
  for (auto& b : p->P.near) s += b.m.size();
  return s;
}

int h2g_near_dense(h2g_problem* p, double* out) {
  return guarded([&] {
    int64_t at = 0;
    for (auto& b : p->P.near) {
      d2h(p->P, out + at, b.m.p, sizeof(double) * b.m.size());
      at += b.m.size();
    }
  });
}

int h2g_num_factor_levels(h2g_problem* p) { return int(p->P.levels.size()); }

int h2g_factor_level(h2g_problem* p, int li, int64_t* ranks) {
  int level = -1;
  if (guarded([&] {
        if (li < 0 || size_t(li) >= p->P.levels.size())
          throw std::out_of_range("h2g_factor_level: no factorized level " + std::to_string(li));
        const auto& lf = p->P.levels[size_t(li)];
        for (size_t k = 0; k < lf.ranks.size(); ++k) ranks[k] = lf.ranks[k];
        level = lf.level;
      }))
    return -1;
  return level;
}

int64_t h2g_cutoff(h2g_problem* p, int64_t* dims) {
  for (size_t k = 0; k < p->P.cutoff_dims.size(); ++k) dims[k] = p->P.cutoff_dims[k];
  return int64_t(p->P.cutoff_dims.size()) | (int64_t(p->P.cutoff_level) << 32);
}

int64_t h2g_top_n(h2g_problem* p) { return p->P.top.n(); }

int h2g_top(h2g_problem* p, double* lu, int64_t* perm) {
  return guarded([&] {
    const int64_t n = p->P.top.n();
    d2h(p->P, lu, p->P.top.lu.m.p, sizeof(double) * n * n);
    d2h(p->P, perm, p->P.top.perm, sizeof(int64_t) * n);
  });
}

int64_t h2g_basis(h2g_problem* p, int level, int64_t k, int side, double* sq) {
  int64_t out = -1;
  if (guarded([&] {
        const auto& sets = side == 0 ? p->P.U : p->P.V;
        if (level < 0 || size_t(level) >= sets.size() || k < 0 || size_t(k) >= sets[size_t(level)].size())
          throw std::out_of_range("h2g_basis: no basis at level " + std::to_string(level) + " box " +
                                  std::to_string(k));
        const auto& B = sets[size_t(level)][size_t(k)];
        if (sq && B.dim > 0) d2h(p->P, sq, B.SQ.m.p, sizeof(double) * B.dim * B.dim);
        out = int64_t(B.dim) | (int64_t(B.rank) << 32);
      }))
    return -1;
  return out;
}

double h2g_max_fill_residual(h2g_problem* p) { return p->P.stats.max_fill_residual; }

int64_t h2g_kernel_evals(h2g_problem* p) { return int64_t(p->P.c.kernel_evals); }

int h2g_stats(h2g_problem* p, double* t5, double* f6, int64_t* launches) {
  const auto& s = p->P.stats;
  t5[0] = s.t_tree;
  t5[1] = s.t_classify;
  t5[2] = s.t_near;
  t5[3] = s.t_factor;
  t5[4] = s.t_solve;
  auto get = [&](const char* k) {
    auto it = p->P.c.phase_flops.find(k);
    return it == p->P.c.phase_flops.end() ? 0.0 : it->second;
  };
  f6[0] = get("fill_precompute");
  f6[1] = get("basis");
  f6[2] = get("skeleton");
  f6[3] = get("factorize");
  f6[4] = get("assemble");
  f6[5] = get("solve");
  *launches = p->P.c.launches;
  return 0;
}

int h2g_set_stream(h2g_problem* p, void* stream) {
  return guarded([&] {
    if (p->P.built) throw std::logic_error("h2g_set_stream: call before build");
    p->P.use_stream(static_cast<cudaStream_t>(stream));
  });
}

int h2g_nccl_unique_id(void* id128) {
  return guarded([&] { h2g::nccl_unique_id(id128); });
}

int h2g_comm_nccl(int nranks, int rank, const void* id128, h2g_comm** out) {
  return guarded([&] { *out = new h2g_comm{h2g::make_nccl_comm(nranks, rank, id128)}; });
}

int h2g_comm_host(int nranks, int rank, h2g_host_allgather_fn fn, void* user, h2g_comm** out) {
  return guarded([&] { *out = new h2g_comm{h2g::make_host_comm(nranks, rank, fn, user)}; });
}

void h2g_comm_destroy(h2g_comm* c) { delete c; }

int h2g_set_comm(h2g_problem* p, h2g_comm* c) {
  return guarded([&] {
    if (p->P.factored) throw std::logic_error("h2g_set_comm: call before factor");
    p->P.comm = (c && c->c->size > 1) ? c->c : nullptr;
  });
}

int h2g_partition_range(int64_t m, int nranks, int rank, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks || m < 0)
      throw std::invalid_argument("h2g_partition_range: bad arguments");
    struct Plain : h2g::Comm {
      void allgatherv(void*, const std::vector<int64_t>&, cudaStream_t) override {}
    } c;
    c.rank = rank;
    c.size = nranks;
    if (c.partitioned(m)) {
      *lo = c.lo(m);
      *hi = c.hi(m);
    } else {
      *lo = 0;
      *hi = m;
    }
  });
}

int h2g_stats_dev(h2g_problem* p, double* t3) {
  t3[0] = p->P.stats.t_build_dev;
  t3[1] = p->P.stats.t_factor_dev;
  t3[2] = p->P.stats.t_solve_dev;
  return 0;
}

int h2g_phase_seconds(h2g_problem* p, int idx, char* name, int name_len, double* sec) {
  int i = 0;
  for (auto& [k, v] : p->P.stats.phase_seconds) {
    if (i++ != idx) continue;
    std::snprintf(name, size_t(name_len), "%s", k.c_str());
    *sec = v;
    return 1;
  }
  return 0;
}

int h2g_set_profile(h2g_problem* p, int on) {
  p->P.c.prof = on != 0;
  return 0;
}

int h2g_reset_profile(h2g_problem* p) {
  p->P.c.pagg.clear();
  p->P.c.launches = 0;
  return 0;
}

int h2g_kernel_stats(h2g_problem* p, int idx, char* name, int name_len, double* ms,
                     int64_t* launches, double* flops, double* bytes) {
  int i = 0;
  for (auto& [k, v] : p->P.c.pagg) {
    if (i++ != idx) continue;
    std::snprintf(name, size_t(name_len), "%s", k.c_str());
    *ms = v.ms;
    *launches = v.launches;
    *flops = v.flops;
    *bytes = v.bytes;
    return 1;
  }
  return 0;
}

// ---- single primitives ---------------------------------------------------
int h2g_lu_factor(int64_t n, const double* a, double tol, double* lu, int64_t* perm) {
  return guarded([&] {
    require_device();
    h2g::Problem P;
    auto f = h2g::alloc_lu(P.c, int(n));
    h2g::cuda_check(cudaMemcpy(f.lu.m.p, a, sizeof(double) * n * n, cudaMemcpyHostToDevice), "h2d");
    h2g::LuBatch lb;
    lb.add(f, tol, "block");
    lb.run(P.c);
    P.c.sync();  // completes the batch and reports a singular pivot
    h2g::cuda_check(cudaMemcpy(lu, f.lu.m.p, sizeof(double) * n * n, cudaMemcpyDeviceToHost), "d2h");
    h2g::cuda_check(cudaMemcpy(perm, f.perm, sizeof(int64_t) * n, cudaMemcpyDeviceToHost), "d2h");
  });
}

int h2g_lu_solve(int64_t n, const double* lu, const int64_t* perm, int kind, int64_t rows,
                 int64_t cols, double* x) {
  return guarded([&] {
    require_device();
    h2g::Problem P;
    auto f = h2g::alloc_lu(P.c, int(n));
    auto X = h2g::alloc_mat(P.c, int(rows), int(cols));
    h2g::cuda_check(cudaMemcpy(f.lu.m.p, lu, sizeof(double) * n * n, cudaMemcpyHostToDevice), "h2d");
    h2g::cuda_check(cudaMemcpy(f.perm, perm, sizeof(int64_t) * n, cudaMemcpyHostToDevice), "h2d");
    h2g::cuda_check(cudaMemcpy(X.m.p, x, sizeof(double) * rows * cols, cudaMemcpyHostToDevice), "h2d");
    h2g::SolveBatch sb;
    sb.add(f, X.m, kind);
    sb.run(P.c);
    P.c.sync();
    h2g::cuda_check(cudaMemcpy(x, X.m.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost), "d2h");
  });
}

int h2g_gemm(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int transa,
             const double* b, int transb, int acc, double* c) {
  return guarded([&] {
    require_device();
    h2g::Problem P;
    const int ar = transa ? int(k) : int(m), ac = transa ? int(m) : int(k);
    const int br = transb ? int(n) : int(k), bc = transb ? int(k) : int(n);
    auto A = h2g::alloc_mat(P.c, ar, ac), B = h2g::alloc_mat(P.c, br, bc), C = h2g::alloc_mat(P.c, int(m), int(n));
    h2g::cuda_check(cudaMemcpy(A.m.p, a, sizeof(double) * ar * ac, cudaMemcpyHostToDevice), "h2d");
    h2g::cuda_check(cudaMemcpy(B.m.p, b, sizeof(double) * br * bc, cudaMemcpyHostToDevice), "h2d");
    h2g::cuda_check(cudaMemcpy(C.m.p, c, sizeof(double) * m * n, cudaMemcpyHostToDevice), "h2d");
    h2g::GemmBatch gb;
    gb.job(C.m, acc != 0);
    gb.seg(transa ? A.m.t() : A.m, transb ? B.m.t() : B.m, alpha);
    gb.run(P.c);
    P.c.sync();
    h2g::cuda_check(cudaMemcpy(c, C.m.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost), "d2h");
  });
}

int h2g_basis_from_members(int64_t dim, int64_t width, const double* concat, int64_t nmem,
                           const int64_t* offsets, double tol, int64_t cap, int64_t min_rank,
                           double* sq, int64_t* rank) {
  return h2g_basis_from_members_mode(dim, width, concat, nmem, offsets, tol, cap, min_rank, 0, sq, rank);
}

int h2g_basis_from_members_mode(int64_t dim, int64_t width, const double* concat, int64_t nmem,
                                const int64_t* offsets, double tol, int64_t cap, int64_t min_rank,
                                int32_t qr_mode, double* sq, int64_t* rank) {
  return guarded([&] {
    require_device();
    if (qr_mode < 0 || qr_mode > 2)
      throw std::invalid_argument("config: qr_mode must be 0 (exact), 1 (blocked) or 2 (compressed)");
    h2g::Problem P;
    P.c.qr_blocked = qr_mode >= 1;
    P.c.qr_compress = qr_mode == 2;
    auto Cm = h2g::alloc_mat(P.c, int(dim), int(width > 0 ? width : 1));
    if (width > 0)
      h2g::cuda_check(cudaMemcpy(Cm.m.p, concat, sizeof(double) * dim * width, cudaMemcpyHostToDevice), "h2d");
    Cm.m.cols = int(width);
    h2g::QrBatch qb;
    qb.add(Cm, int(dim), int(width), std::vector<int64_t>(offsets, offsets + nmem + 1), tol, int(cap));
    std::vector<h2g::DMat> Q;
    std::vector<int> rk;
    qb.run(P.c, Q, rk, size_t(1) << 30);
    const int r = int(std::min<int64_t>(dim, std::max<int64_t>(rk[0], min_rank)));
    std::vector<double> q(size_t(dim) * dim);
    h2g::cuda_check(cudaMemcpy(q.data(), Q[0].m.p, sizeof(double) * dim * dim, cudaMemcpyDeviceToHost), "d2h");
    // row-major Q -> square [Qr | Qs] column-major.
    for (int64_t j = 0; j < dim; ++j) {
      const int64_t src = j < dim - r ? r + j : j - (dim - r);
      for (int64_t i = 0; i < dim; ++i) sq[j * dim + i] = q[i * dim + src];
    }
    *rank = r;
  });
}


// ---- ULVFactors views (the façade's LevelFactors / DenseSystem / ClusterFactors) ----
namespace {
const h2g::LevelF& level_of(h2g_problem* p, int li) {
  if (!p->P.factored) throw std::logic_error("h2g: factor first");
  if (li < 0 || size_t(li) >= p->P.levels.size())
    throw std::out_of_range("h2g: no factorized level " + std::to_string(li));
  return p->P.levels[size_t(li)];
}
void copy_mat(h2g_problem* p, const h2g::Mat& m, int64_t* rows, int64_t* cols, double* out) {
  *rows = m.rows;
  *cols = m.cols;
  if (!out || m.rows == 0 || m.cols == 0) return;
  // strided device view -> column-major host copy
  if (m.rs == 1 && m.cs == m.rows) {
    d2h(p->P, out, m.p, sizeof(double) * size_t(m.rows) * m.cols);
    return;
  }
  if (m.rs == 1) {
    h2g::cuda_check(cudaMemcpy2DAsync(out, sizeof(double) * m.rows, m.p, sizeof(double) * m.cs,
                                      sizeof(double) * m.rows, m.cols, cudaMemcpyDeviceToHost, p->P.c.stream),
                    "d2h");
    h2g::cuda_check(cudaStreamSynchronize(p->P.c.stream), "d2h");
    return;
  }
  throw std::logic_error("h2g: unexpected row-strided factor view");
}
}  // namespace

int h2g_level_dims(h2g_problem* p, int li, int64_t* dims, int64_t* ranks, int32_t* use_z) {
  int64_t m = -1;
  if (guarded([&] {
        const auto& lf = level_of(p, li);
        m = int64_t(lf.dims.size());
        for (size_t k = 0; k < lf.dims.size(); ++k) {
          if (dims) dims[k] = lf.dims[k];
          if (ranks) ranks[k] = lf.ranks[k];
        }
        if (use_z) *use_z = lf.use_z ? 1 : 0;
      }))
    return -1;
  return int(m);
}

int h2g_level_block(h2g_problem* p, int li, int64_t i, int64_t j, int64_t* rows, int64_t* cols,
                    double* out) {
  return guarded([&] {
    const auto& lf = level_of(p, li);
    const auto& S = p->P.S;
    const int l = lf.level;
    if (i < 0 || i >= (int64_t(1) << l)) throw std::out_of_range("DenseSystem::block: no dense block");
    const int64_t* b = S.near(l, i);
    const int64_t n = S.nnear(l, i);
    const int64_t* it = std::lower_bound(b, b + n, j);
    if (it == b + n || *it != j) throw std::out_of_range("DenseSystem::block: no dense block");
    const size_t t = size_t(S.level[l].near_ptr[i] + (it - b));
    if (t >= lf.sys.blocks.size()) throw std::out_of_range("DenseSystem::block: no dense block");
    copy_mat(p, lf.sys.blocks[t].m, rows, cols, out);
  });
}

int h2g_level_lu(h2g_problem* p, int li, int which, int64_t k, int64_t* n, double* lu, int64_t* perm) {
  return guarded([&] {
    const auto& lf = level_of(p, li);
    if (k < 0 || size_t(k) >= lf.dims.size()) throw std::out_of_range("h2g_level_lu: no box " + std::to_string(k));
    const h2g::LuF* f = nullptr;
    if (which == 0) {
      if (lf.sys.diag_lu.empty()) throw std::out_of_range("h2g_level_lu: level has no cached diagonal LUs");
      f = &lf.sys.diag_lu[size_t(k)];
    } else {
      f = &lf.elim[size_t(k)].piv;
    }
    const int64_t nn = f->n();
    *n = nn;
    if (nn == 0 || !lu) return;
    d2h(p->P, lu, f->lu.m.p, sizeof(double) * size_t(nn) * nn);
    d2h(p->P, perm, f->perm, sizeof(int64_t) * size_t(nn));
  });
}

int h2g_level_elim(h2g_problem* p, int li, int64_t k, int which, int64_t* rows, int64_t* cols, double* out) {
  return guarded([&] {
    const auto& lf = level_of(p, li);
    if (k < 0 || size_t(k) >= lf.elim.size()) throw std::out_of_range("h2g_level_elim: no box " + std::to_string(k));
    const auto& e = lf.elim[size_t(k)];
    const h2g::DMat& m = which == 0 ? e.urs : e.lsr;
    if (!m.m.p) {
      *rows = which == 0 ? e.rdim : e.sdim;
      *cols = which == 0 ? e.sdim : e.rdim;
      if (out && *rows * *cols > 0) throw std::logic_error("h2g_level_elim: factor not stored");
      return;
    }
    copy_mat(p, m.m, rows, cols, out);
  });
}

// assemble_block (kernels.cpp:242-268) of a host cloud on the device:
// out (rows x cols, column-major) = kernel(x_{r0+i}, x_{c0+j}, q_{c0+j}).
int h2g_assemble_block(const h2g_kernel* k, int64_t n, const double* xyz, const double* q, int64_t r0,
                       int64_t r1, int64_t c0, int64_t c1, double* out) {
  return guarded([&] {
    require_device();
    if (r1 <= r0 || c1 <= c0) throw std::invalid_argument("assemble_block: empty range");
    if (r0 < 0 || c0 < 0 || r1 > n || c1 > n) throw std::out_of_range("assemble_block: range outside cloud");
    h2g::Problem P;
    h2g::KernelParams kp;
    kp.kind = k->kind;
    kp.alpha_m = k->alpha_m;
    kp.scale = k->permittivity_scale;
    kp.reg = k->eta_reg;
    P.c.kp = kp;
    std::vector<double> soa(size_t(4 * n));
    for (int64_t i = 0; i < n; ++i) {
      soa[size_t(i)] = xyz[3 * i];
      soa[size_t(n + i)] = xyz[3 * i + 1];
      soa[size_t(2 * n + i)] = xyz[3 * i + 2];
      soa[size_t(3 * n + i)] = q[i];
    }
    DevBuf pts(sizeof(double) * soa.size());
    h2d(P, pts.p, soa.data(), sizeof(double) * soa.size());
    const double* d = pts.d();
    P.c.cloud = h2g::Cloud{d, d + n, d + 2 * n, d + 3 * n, n};
    auto B = h2g::alloc_mat(P.c, int(r1 - r0), int(c1 - c0));
    h2g::EvalBatch eb;
    eb.add(B.m, r0, c0);
    eb.run(P.c);
    P.c.sync();  // reports a singular evaluation with the reference's message
    d2h(P, out, B.m.p, sizeof(double) * size_t(r1 - r0) * size_t(c1 - c0));
  });
}

// glibc exp restated (common.cuh exp_glibc_core) on the host, for the CPU
// tests that pin the restatement against libm without a device.
int h2g_exp_glibc_host(int64_t n, const double* x, double* y) {
  static const uint64_t tab[2 * 128] = {H2G_EXP_TABLE_INIT};
  for (int64_t i = 0; i < n; ++i) {
    bool special = false;
    const double v = h2g::exp_glibc_core(x[i], tab, &special);
    y[i] = special ? std::exp(x[i]) : v;
  }
  return 0;
}

}  // extern "C"
