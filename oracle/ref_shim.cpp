// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Tests,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load it through ctypes to (a) generate golden fixtures, (b) pin the C
// restatement in oracle/h2oracle.c, and (c) time the reference CPU path.
//
// Every entry point drives the reference's own public API (proj/include):
//   generate_uniform_cube / generate_line / generate_sphere_surface (geometry.hpp:18-24)
//   build_cluster_tree (geometry.hpp:58), classify_blocks (hstructure.hpp:55-56)
//   materialize_dense (hstructure.hpp:101-103), build_and_factorize (ulv.hpp:123)
//   solve (solve.hpp:10), matvec_dense_oracle / dense_solve_oracle (solve.hpp:14-19)
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "h2ulv/compression.hpp"
#include "h2ulv/flops.hpp"
#include "h2ulv/geometry.hpp"
#include "h2ulv/hstructure.hpp"
#include "h2ulv/kernels.hpp"
#include "h2ulv/solve.hpp"
#include "h2ulv/ulv.hpp"

using namespace h2ulv;

namespace {

thread_local std::string g_err;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct RefRun {
  PointCloud original;
  std::unique_ptr<ClusterTreeResult> tree;
  std::unique_ptr<HMatrix> H;
  KernelSpec kernel;
  ULVFactors f;
  bool factored = false;
  double t_tree = 0, t_classify = 0, t_near = 0, t_factor = 0, t_solve = 0;
  uint64_t flops_fills = 0, flops_basis = 0, flops_skel = 0, flops_fact = 0, kernel_evals = 0;
};

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

// Kernel/factor configuration mirrored by tests/_ref.py (ctypes Structure).
struct RefConfig {
  int64_t leaf_size;
  double tol;
  int64_t cap;  // <= 0: no cap
  int32_t kernel;  // 0 laplace, 1 yukawa
  int32_t structure;  // 0 h2, 1 hss, 2 blr2
  double alpha_m;
  double reg;
  double scale;
  double eta;
  int32_t threads;
  int32_t absorb_coupling;
};

const char* ref_last_error() { return g_err.c_str(); }

// Point generators (geometry.cpp:42-95). xyz is AoS n*3, q has n entries.
int ref_generate(int32_t geometry, int64_t n, uint64_t seed, int64_t spheres, double spacing,
                 double* xyz, double* q) {
  return guarded([&] {
    PointCloud c = geometry == 0   ? generate_uniform_cube(n, seed)
                   : geometry == 1 ? generate_line(n, seed)
                                   : generate_sphere_surface(n, spheres, spacing, seed);
    for (int64_t i = 0; i < n; ++i) {
      for (int d = 0; d < 3; ++d) xyz[3 * i + d] = c.points[i][d];
      q[i] = c.charges[i];
    }
  });
}

double ref_domain_diameter(int64_t n, const double* xyz) {
  PointCloud c;
  c.points.resize(n);
  for (int64_t i = 0; i < n; ++i) c.points[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return c.domain_diameter();
}

double ref_default_eta_reg(double diam, int64_t n) { return default_eta_reg(diam, n); }

void* ref_new(int64_t n, const double* xyz, const double* q) {
  auto* r = new RefRun;
  r->original.points.resize(n);
  r->original.charges.assign(q, q + n);
  for (int64_t i = 0; i < n; ++i)
    r->original.points[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return r;
}

void ref_free(void* h) { delete static_cast<RefRun*>(h); }

// Tree + classification + near-field (Pipeline::build, report.cpp:79-91).
int ref_build(void* h, const RefConfig* cfg) {
  auto* r = static_cast<RefRun*>(h);
  return guarded([&] {
    r->kernel = cfg->kernel == 0 ? KernelSpec::laplace(cfg->reg)
                                 : KernelSpec::yukawa(cfg->alpha_m, cfg->reg);
    r->kernel.permittivity_scale = cfg->scale;
    double t0 = now_s();
    r->tree = std::make_unique<ClusterTreeResult>(build_cluster_tree(r->original, cfg->leaf_size));
    double t1 = now_s();
    StructureVariant sv = cfg->structure == 0   ? StructureVariant::h2
                          : cfg->structure == 1 ? StructureVariant::hss
                                                : StructureVariant::blr2;
    AdmissibilityRule rule{cfg->structure == 0 ? AdmissibilityKind::strong : AdmissibilityKind::weak,
                           cfg->eta};
    BlockStructure bs = classify_blocks(r->tree->tree, rule, sv);
    double t2 = now_s();
    FlopCounter::instance().reset();
    r->H = std::make_unique<HMatrix>(
        materialize_dense(bs, r->tree->tree, r->tree->cloud, r->kernel, sv, cfg->threads));
    double t3 = now_s();
    r->t_tree = t1 - t0;
    r->t_classify = t2 - t1;
    r->t_near = t3 - t2;
  });
}

int ref_levels(void* h) { return static_cast<RefRun*>(h)->tree->tree.levels; }

// original_index (geometry.hpp:40): reordered position -> original position.
void ref_tree_perm(void* h, int64_t* out) {
  auto* r = static_cast<RefRun*>(h);
  const auto& oi = r->tree->tree.original_index;
  std::memcpy(out, oi.data(), oi.size() * sizeof(int64_t));
}

// Node table in heap order: begin, end (int64) and center xyz + radius (double).
void ref_nodes(void* h, int64_t* be, double* geo) {
  auto* r = static_cast<RefRun*>(h);
  const auto& nodes = r->tree->tree.nodes;
  for (size_t k = 0; k < nodes.size(); ++k) {
    be[2 * k] = nodes[k].begin;
    be[2 * k + 1] = nodes[k].end;
    for (int d = 0; d < 3; ++d) geo[4 * k + d] = nodes[k].center[d];
    geo[4 * k + 3] = nodes[k].radius;
  }
}

void ref_reordered_points(void* h, double* xyz, double* q) {
  auto* r = static_cast<RefRun*>(h);
  const auto& c = r->tree->cloud;
  for (int64_t i = 0; i < c.size(); ++i) {
    for (int d = 0; d < 3; ++d) xyz[3 * i + d] = c.points[i][d];
    q[i] = c.charges[i];
  }
}

// Per-level CSR sizes: returns total near (far) entries at level lvl.
int64_t ref_list_count(void* h, int lvl, int far) {
  auto* r = static_cast<RefRun*>(h);
  const auto& L = r->H->structure.level[lvl];
  const auto& rows = far ? L.far_cols : L.near_cols;
  int64_t s = 0;
  for (const auto& row : rows) s += static_cast<int64_t>(row.size());
  return s;
}

// CSR export: ptr has 2^lvl + 1 entries.
void ref_list(void* h, int lvl, int far, int64_t* ptr, int64_t* idx) {
  auto* r = static_cast<RefRun*>(h);
  const auto& L = r->H->structure.level[lvl];
  const auto& rows = far ? L.far_cols : L.near_cols;
  ptr[0] = 0;
  for (size_t i = 0; i < rows.size(); ++i) {
    std::memcpy(idx + ptr[i], rows[i].data(), rows[i].size() * sizeof(int64_t));
    ptr[i + 1] = ptr[i] + static_cast<int64_t>(rows[i].size());
  }
}

// Leaf dense arena: blocks in (row, near_cols order), each column-major.
int64_t ref_leaf_dense_entries(void* h) { return static_cast<RefRun*>(h)->H->stored_dense_entries(); }

void ref_leaf_dense(void* h, double* out) {
  auto* r = static_cast<RefRun*>(h);
  int64_t at = 0;
  for (const auto& row : r->H->leaf_dense)
    for (const auto& B : row) {
      std::memcpy(out + at, B.data(), B.size() * sizeof(double));
      at += B.size();
    }
}

// build_and_factorize (ulv.hpp:123) timed like Pipeline::factor (report.cpp:93-106).
int ref_factor(void* h, const RefConfig* cfg) {
  auto* r = static_cast<RefRun*>(h);
  return guarded([&] {
    FactorOptions opts;
    opts.variant = cfg->structure == 0   ? FactorVariant::h2nodep
                   : cfg->structure == 1 ? FactorVariant::hss
                                         : FactorVariant::blr2;
    opts.tol = cfg->tol;
    if (cfg->cap > 0) opts.cap = cfg->cap;
    opts.threads = cfg->threads;
    opts.absorb_coupling = cfg->absorb_coupling != 0;
    FlopCounter& fc = FlopCounter::instance();
    fc.reset();
    double t0 = now_s();
    r->f = build_and_factorize(*r->H, opts);
    r->t_factor = now_s() - t0;
    r->flops_fills = fc.phase_total(Phase::fills);
    r->flops_basis = fc.phase_total(Phase::basis);
    r->flops_skel = fc.phase_total(Phase::skeleton);
    r->flops_fact = fc.phase_total(Phase::factorize);
    r->kernel_evals = fc.kernel_evals();
    r->factored = true;
  });
}

// Timings [tree, classify, near, factor, solve] and counted flops
// [fills, basis, skeleton, factorize, kernel_evals, metric_flops].
void ref_stats(void* h, double* t5, uint64_t* f6) {
  auto* r = static_cast<RefRun*>(h);
  t5[0] = r->t_tree;
  t5[1] = r->t_classify;
  t5[2] = r->t_near;
  t5[3] = r->t_factor;
  t5[4] = r->t_solve;
  f6[0] = r->flops_fills;
  f6[1] = r->flops_basis;
  f6[2] = r->flops_skel;
  f6[3] = r->flops_fact;
  f6[4] = r->kernel_evals;
  f6[5] = r->f.metric_flops;
}

int ref_num_factor_levels(void* h) { return static_cast<int>(static_cast<RefRun*>(h)->f.levels.size()); }

// Per processed level: tree level and the ranks of its clusters.
int ref_factor_level(void* h, int li, int64_t* ranks) {
  auto* r = static_cast<RefRun*>(h);
  const LevelFactors& lf = r->f.levels[li];
  for (size_t k = 0; k < lf.ranks.size(); ++k) ranks[k] = lf.ranks[k];
  return lf.level;
}

int64_t ref_cutoff(void* h, int64_t* dims) {
  auto* r = static_cast<RefRun*>(h);
  for (size_t k = 0; k < r->f.cutoff_dims.size(); ++k) dims[k] = r->f.cutoff_dims[k];
  return static_cast<int64_t>(r->f.cutoff_dims.size()) | (int64_t(r->f.cutoff_level) << 32);
}

int64_t ref_top_n(void* h) { return static_cast<RefRun*>(h)->f.top.n(); }

void ref_top(void* h, double* lu, int64_t* perm) {
  auto* r = static_cast<RefRun*>(h);
  const auto& t = r->f.top;
  std::memcpy(lu, t.lu.data(), t.lu.size() * sizeof(double));
  std::memcpy(perm, t.perm.forward.data(), t.perm.forward.size() * sizeof(int64_t));
}

// Shared basis of cluster k at tree level lvl: side 0 = U, 1 = V.
// Returns dim | rank << 32 when out == nullptr; otherwise writes [Qr | Qs].
int64_t ref_basis(void* h, int lvl, int64_t k, int side, double* out) {
  auto* r = static_cast<RefRun*>(h);
  const SharedBasis& b = side == 0 ? r->f.bases.U[lvl][k] : r->f.bases.V[lvl][k];
  if (out) {
    Matrix sq = b.square();
    std::memcpy(out, sq.data(), sq.size() * sizeof(double));
  }
  return b.dim() | (b.rank() << 32);
}

double ref_max_fill_residual(void* h) {
  auto* r = static_cast<RefRun*>(h);
  double m = 0;
  for (double v : r->f.max_fill_residual_rel) m = std::max(m, v);
  return m;
}

// solve (solve.hpp:10): b and x in the original point order, nrhs columns.
int ref_solve(void* h, int64_t nrhs, const double* b, double* x) {
  auto* r = static_cast<RefRun*>(h);
  return guarded([&] {
    const int64_t n = r->original.size();
    Matrix B(n, nrhs);
    std::memcpy(B.data(), b, sizeof(double) * n * nrhs);
    double t0 = now_s();
    Matrix X = solve(r->f, B);
    r->t_solve = now_s() - t0;
    std::memcpy(x, X.data(), sizeof(double) * n * nrhs);
  });
}

// Dense oracle products (solve.cpp:234-247) on the ORIGINAL cloud.
int ref_dense_matvec(void* h, const double* x, double* y) {
  auto* r = static_cast<RefRun*>(h);
  return guarded([&] {
    const int64_t n = r->original.size();
    Matrix X(n, 1);
    std::memcpy(X.data(), x, sizeof(double) * n);
    Matrix Y = matvec_dense_oracle(r->original, r->kernel, X, 1 << 20);
    std::memcpy(y, Y.data(), sizeof(double) * n);
  });
}

int ref_dense_solve(void* h, const double* b, double* x) {
  auto* r = static_cast<RefRun*>(h);
  return guarded([&] {
    const int64_t n = r->original.size();
    Matrix B(n, 1);
    std::memcpy(B.data(), b, sizeof(double) * n);
    Matrix X = dense_solve_oracle(r->original, r->kernel, B, 1 << 20);
    std::memcpy(x, X.data(), sizeof(double) * n);
  });
}

// Single-block primitives for kernel-level parity tests (linalg.hpp).
int ref_lu_factor(int64_t n, const double* a, double tol, double* lu, int64_t* perm) {
  return guarded([&] {
    Matrix A(n, n);
    std::memcpy(A.data(), a, sizeof(double) * n * n);
    LuFactors f = lu_factor(A, tol, "block");
    std::memcpy(lu, f.lu.data(), sizeof(double) * n * n);
    std::memcpy(perm, f.perm.forward.data(), sizeof(int64_t) * n);
  });
}

// basis_from_members (compression.cpp:111-146): members given as one
// concatenated dim x width matrix plus member column offsets.
int ref_basis_from_members(int64_t dim, int64_t width, const double* concat, int64_t nmem,
                           const int64_t* offsets, double tol, int64_t cap, int64_t min_rank,
                           double* q_out, int64_t* rank_out) {
  return guarded([&] {
    std::vector<Matrix> members;
    for (int64_t g = 0; g < nmem; ++g) {
      Matrix M(dim, offsets[g + 1] - offsets[g]);
      std::memcpy(M.data(), concat + dim * offsets[g], sizeof(double) * M.size());
      members.push_back(std::move(M));
    }
    BasisBuildOptions o;
    o.tol = tol;
    if (cap > 0) o.cap = cap;
    SharedBasis b = basis_from_members(members, dim, o, min_rank);
    Matrix sq = b.square();
    std::memcpy(q_out, sq.data(), sizeof(double) * sq.size());
    *rank_out = b.rank();
  });
}

}  // extern "C"

extern "C" {

// gemm / matmul / gemm_acc (linalg.cpp:86-126).
int ref_gemm(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int transa,
             const double* b, int transb, int acc, double* c) {
  return guarded([&] {
    const int64_t ar = transa ? k : m, ac = transa ? m : k, br = transb ? n : k, bc = transb ? k : n;
    Matrix A(ar, ac), B(br, bc), C(m, n);
    std::memcpy(A.data(), a, sizeof(double) * ar * ac);
    std::memcpy(B.data(), b, sizeof(double) * br * bc);
    std::memcpy(C.data(), c, sizeof(double) * m * n);
    if (acc) {
      Matrix Ae = transa ? transpose(A) : A, Be = transb ? transpose(B) : B;
      gemm_acc(C, Ae, Be, alpha);
    } else {
      C = matmul(A, B, transa != 0, transb != 0, alpha);
    }
    std::memcpy(c, C.data(), sizeof(double) * m * n);
  });
}

// LuFactors solve family (linalg.cpp:404-559) from given packed factors.
int ref_lu_solve(int64_t n, const double* lu, const int64_t* perm, int kind, int64_t rows,
                 int64_t cols, double* x) {
  return guarded([&] {
    LuFactors f;
    f.lu = Matrix(n, n);
    std::memcpy(f.lu.data(), lu, sizeof(double) * n * n);
    f.perm.forward.assign(perm, perm + n);
    Matrix X(rows, cols);
    std::memcpy(X.data(), x, sizeof(double) * rows * cols);
    switch (kind) {
      case 0: f.solve_in_place(X); break;
      case 1: f.solve_lower_in_place(X); break;
      case 2: f.solve_upper_in_place(X); break;
      case 3: f.solve_transpose_in_place(X); break;
      case 4: f.solve_right_in_place(X); break;
      default: f.solve_upper_right_in_place(X); break;
    }
    std::memcpy(x, X.data(), sizeof(double) * rows * cols);
  });
}

}  // extern "C"
