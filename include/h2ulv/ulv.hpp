// Drop-in for proj/include/h2ulv/ulv.hpp (ulv.hpp:15-132): the factor types
// and the factorization entry points. prepare_factor_inputs + factorize =
// build_and_factorize = h2g_factor on the device problem the HMatrix holds
// (fills, fill-augmented bases, level-parallel ULV, top LU: sm_100a kernels).
// The returned ULVFactors is a host snapshot of the device factors in the
// reference's layout (bases, level systems, diagonal LUs, eliminations, top),
// plus the device problem itself, which solve() runs on.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "h2ulv/compression.hpp"
#include "h2ulv/hstructure.hpp"

namespace h2ulv {

enum class FactorVariant { blr2, hss, h2dep, h2nodep };

inline const char* variant_name(FactorVariant v) {
  switch (v) {
    case FactorVariant::blr2: return "blr2";
    case FactorVariant::hss: return "hss";
    case FactorVariant::h2dep: return "h2dep";
    default: return "h2nodep";
  }
}

struct FillEvent {
  int level = 0;
  int64_t row = 0;
  int64_t col = 0;
  double norm = 0.0;
  double residual = 0.0;
};

struct FactorOptions {
  FactorVariant variant = FactorVariant::h2nodep;
  double tol = 1e-8;
  std::optional<int64_t> cap;
  int threads = 1;
  double rr_pivot_tol = 1e-13;
  bool absorb_coupling = true;
  double abort_residual_factor = 100.0;
  std::function<void(const FillEvent&)> fill_observer;  // not invoked by the device path
  std::optional<uint64_t> task_order_seed;               // order-independent by construction
  bool keep_diag_skeletons = false;                      // not kept by the device path
  // B200 extensions (h2g_options): member-panel QR mode (0 exact, 1 blocked,
  // 2 compressed) and the reference's assembly bit for bit (1) or corrected (0).
  int b200_qr_mode = 0;
  bool b200_reference_compat = true;
  int64_t b200_sample_cols = 0;  // h2g_set_sampling: 0 = the reference's full far-field members
};

struct ClusterFactors {
  LuFactors pivot;
  Matrix urs;
  Matrix lsr;
  int64_t rdim = 0;
  int64_t sdim = 0;
};

// eliminate_block (ulv.cpp:25-48) through the device primitives (bit-exact
// lu_factor, the lower / upper-right solves and gemm_acc).
inline ClusterFactors eliminate_block(Matrix& S, int64_t rdim, double pivot_tol) {
  if (S.rows != S.cols) throw std::invalid_argument("eliminate_block: S not square");
  if (rdim < 0 || rdim > S.rows) throw std::invalid_argument("eliminate_block: bad split");
  ClusterFactors f;
  f.rdim = rdim;
  f.sdim = S.rows - rdim;
  if (rdim == 0) {
    f.urs = Matrix(0, f.sdim);
    f.lsr = Matrix(f.sdim, 0);
    return f;
  }
  f.pivot = lu_factor(S.block(0, 0, rdim, rdim), pivot_tol, "S^RR");
  f.urs = S.block(0, rdim, rdim, f.sdim);
  f.pivot.solve_lower_in_place(f.urs);
  f.lsr = S.block(rdim, 0, f.sdim, rdim);
  f.pivot.solve_upper_right_in_place(f.lsr);
  if (f.sdim > 0) {
    Matrix ss = S.block(rdim, rdim, f.sdim, f.sdim);
    gemm_acc(ss, f.lsr, f.urs, -1.0);
    S.set_block(rdim, rdim, ss);
  }
  return f;
}

struct LevelFactors {
  int level = 0;
  std::vector<int64_t> dims;
  std::vector<int64_t> ranks;
  std::vector<ClusterFactors> elim;
  DenseSystem sys;
  bool use_z = false;
  std::vector<Matrix> diag_pre;
};

struct ULVFactors {
  FactorVariant variant = FactorVariant::h2nodep;
  const HMatrix* H = nullptr;
  SharedBasisSet bases;
  std::vector<LevelFactors> levels;
  int cutoff_level = 0;
  std::vector<int64_t> cutoff_dims;
  LuFactors top;
  uint64_t metric_flops = 0;
  std::vector<double> max_fill_residual_rel;  // the device reports the maximum (one per level)

  int64_t n() const { return H ? H->cloud->size() : 0; }

  std::shared_ptr<b200::Device> b200;  // the device factors solve() runs on
};

struct FactorInputs {
  SharedBasisSet bases;
  FillInSet leaf_fills;
  DenseSystem leaf_sys;
  std::shared_ptr<b200::Device> b200;  // the prepared device problem
};

namespace b200 {
inline void apply_options(Device& d, const FactorOptions& o) {
  auto& op = d.setup.options;
  op.tol = o.tol;
  op.cap = o.cap.value_or(0);
  op.rr_pivot_tol = o.rr_pivot_tol;
  op.absorb_coupling = o.absorb_coupling ? 1 : 0;
  op.abort_residual_factor = o.abort_residual_factor;
  op.qr_mode = o.b200_qr_mode;
  op.reference_compat = o.b200_reference_compat ? 1 : 0;
  check(h2g_set_options(d.handle->p, &op));
  check(h2g_set_sampling(d.handle->p, o.b200_sample_cols));
}

inline LuFactors read_lu(h2g_problem* p, int li, int which, int64_t k) {
  int64_t n = 0;
  check(h2g_level_lu(p, li, which, k, &n, nullptr, nullptr));
  LuFactors f;
  f.lu = Matrix(n, n);
  f.perm.forward.resize(size_t(n));
  if (n > 0) check(h2g_level_lu(p, li, which, k, &n, f.lu.data(), f.perm.forward.data()));
  return f;
}

inline Matrix read_mat(const std::function<int(int64_t*, int64_t*, double*)>& get) {
  int64_t r = 0, c = 0;
  check(get(&r, &c, nullptr));
  Matrix M(r, c);
  if (r * c > 0) check(get(&r, &c, M.data()));
  return M;
}

inline SharedBasis read_basis(h2g_problem* p, int lvl, int64_t k, int side) {
  const int64_t v = h2g_basis(p, lvl, k, side, nullptr);
  if (v < 0) check(1);
  const int64_t dim = v & 0xFFFFFFFF, rank = v >> 32;
  Matrix sq(dim, dim);
  if (dim > 0) h2g_basis(p, lvl, k, side, sq.data());
  SharedBasis b;
  b.Qr = sq.block(0, 0, dim, dim - rank);
  b.Qs = sq.block(0, dim - rank, dim, rank);
  return b;
}

// Host snapshot of the device factors in the reference's layout.
inline ULVFactors snapshot(const HMatrix& H, const std::shared_ptr<Device>& dev, FactorVariant variant) {
  h2g_problem* p = dev->handle->p;
  ULVFactors f;
  f.variant = variant;
  f.H = &H;
  f.b200 = dev;
  f.bases.init(H.tree.levels);
  const int nl = h2g_num_factor_levels(p);
  for (int li = 0; li < nl; ++li) {
    int32_t use_z = 0;
    const int m = h2g_level_dims(p, li, nullptr, nullptr, &use_z);
    if (m < 0) check(1);
    LevelFactors lf;
    lf.dims.resize(size_t(m));
    lf.ranks.resize(size_t(m));
    h2g_level_dims(p, li, lf.dims.data(), lf.ranks.data(), &use_z);
    std::vector<int64_t> tmp(size_t(int64_t(1) << H.tree.levels));
    lf.level = h2g_factor_level(p, li, tmp.data());
    lf.use_z = use_z != 0;
    const int l = lf.level;
    for (int64_t k = 0; k < m; ++k) {
      f.bases.U[size_t(l)][size_t(k)] = read_basis(p, l, k, 0);
      f.bases.V[size_t(l)][size_t(k)] = read_basis(p, l, k, 1);
    }
    lf.sys.dims = lf.dims;
    lf.sys.near_cols = H.structure.level[size_t(l)].near_cols;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j : lf.sys.near_cols[size_t(i)])
        lf.sys.put(i, j, read_mat([&](int64_t* r, int64_t* c, double* o) { return h2g_level_block(p, li, i, j, r, c, o); }));
    if (lf.sys.has_offdiag() && H.variant != StructureVariant::blr2)
      for (int64_t k = 0; k < m; ++k) lf.sys.diag_lu.push_back(read_lu(p, li, 0, k));
    lf.elim.resize(size_t(m));
    for (int64_t k = 0; k < m; ++k) {
      auto& e = lf.elim[size_t(k)];
      e.rdim = lf.dims[size_t(k)] - lf.ranks[size_t(k)];
      e.sdim = lf.ranks[size_t(k)];
      if (e.rdim > 0) e.pivot = read_lu(p, li, 1, k);
      e.urs = read_mat([&](int64_t* r, int64_t* c, double* o) { return h2g_level_elim(p, li, k, 0, r, c, o); });
      e.lsr = read_mat([&](int64_t* r, int64_t* c, double* o) { return h2g_level_elim(p, li, k, 1, r, c, o); });
    }
    f.levels.push_back(std::move(lf));
  }
  std::vector<int64_t> dims(size_t(int64_t(1) << H.tree.levels));
  const int64_t cv = h2g_cutoff(p, dims.data());
  f.cutoff_level = int(cv >> 32);
  f.cutoff_dims.assign(dims.begin(), dims.begin() + (cv & 0xFFFFFFFF));
  const int64_t tn = h2g_top_n(p);
  f.top.lu = Matrix(tn, tn);
  f.top.perm.forward.resize(size_t(tn));
  if (tn > 0) check(h2g_top(p, f.top.lu.data(), f.top.perm.forward.data()));
  double t5[5], f6[6];
  int64_t launches = 0;
  h2g_stats(p, t5, f6, &launches);
  f.metric_flops = uint64_t(f6[0] + f6[3]);
  f.max_fill_residual_rel.assign(size_t(nl), h2g_max_fill_residual(p));
  return f;
}

inline FactorVariant variant_of(StructureVariant v) {
  return v == StructureVariant::h2 ? FactorVariant::h2nodep
                                   : v == StructureVariant::hss ? FactorVariant::hss : FactorVariant::blr2;
}
}  // namespace b200

namespace b200 {
inline bool same_options(const h2g_options& a, const h2g_options& b) {
  return a.tol == b.tol && a.cap == b.cap && a.rr_pivot_tol == b.rr_pivot_tol &&
         a.absorb_coupling == b.absorb_coupling && a.abort_residual_factor == b.abort_residual_factor &&
         a.structure == b.structure && a.eta == b.eta && a.qr_mode == b.qr_mode &&
         a.reference_compat == b.reference_compat;
}
// One device factorization per option set: the leaf fills, the fill-augmented
// leaf bases and the level-parallel elimination run as one h2g_factor call.
inline void factor_once(Device& d, const FactorOptions& o) {
  apply_options(d, o);
  if (d.factored && same_options(d.factored_with, d.setup.options)) return;
  check(h2g_factor(d.handle->p));
  d.factored = true;
  d.factored_with = d.setup.options;
}
}  // namespace b200

// prepare_factor_inputs (ulv.cpp:1108-1126): the leaf DenseSystem with its
// cached diagonal LUs and the fill-augmented leaf bases. On the device these
// are the first stage of h2g_factor, so preparing runs the factorization and
// returns its leaf stage (the fills stay on the device: leaf_fills is empty).
inline FactorInputs prepare_factor_inputs(const HMatrix& H, const FactorOptions& opts) {
  if (!H.b200) throw std::invalid_argument("prepare_factor_inputs: HMatrix not from materialize_dense");
  if (opts.variant == FactorVariant::h2dep)
    throw std::invalid_argument("prepare_factor_inputs: h2dep is not on the B200 path (sequential driver)");
  b200::factor_once(*H.b200, opts);
  h2g_problem* p = H.b200->handle->p;
  FactorInputs in;
  in.b200 = H.b200;
  const int L = H.tree.levels;
  const int64_t m = int64_t(1) << L;
  in.bases.init(L);
  for (int64_t k = 0; k < m; ++k) {
    in.bases.U[size_t(L)][size_t(k)] = b200::read_basis(p, L, k, 0);
    in.bases.V[size_t(L)][size_t(k)] = b200::read_basis(p, L, k, 1);
  }
  in.leaf_sys.near_cols = H.structure.level[size_t(L)].near_cols;
  for (int64_t k = 0; k < m; ++k) in.leaf_sys.dims.push_back(H.cluster_range(L, k).size());
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j : in.leaf_sys.near_cols[size_t(i)]) in.leaf_sys.put_view(i, j, &H.leaf_block(i, j));
  if (in.leaf_sys.has_offdiag() && H.variant != StructureVariant::blr2)
    for (int64_t k = 0; k < m; ++k) in.leaf_sys.diag_lu.push_back(b200::read_lu(p, 0, 0, k));
  return in;
}

// factorize (ulv.cpp:1128-1143): h2g_factor (once per option set), then the
// host snapshot of the factors.
inline ULVFactors factorize(const HMatrix& H, FactorInputs inputs, const FactorOptions& opts) {
  if (!inputs.b200) inputs.b200 = H.b200;
  if (!inputs.b200) throw std::invalid_argument("factorize: HMatrix not from materialize_dense");
  b200::factor_once(*inputs.b200, opts);
  return b200::snapshot(H, inputs.b200, opts.variant == FactorVariant::h2nodep ? b200::variant_of(H.variant) : opts.variant);
}

inline ULVFactors build_and_factorize(const HMatrix& H, const FactorOptions& opts) {
  if (!H.b200) throw std::invalid_argument("build_and_factorize: HMatrix not from materialize_dense");
  FactorInputs in;
  in.b200 = H.b200;
  return factorize(H, std::move(in), opts);
}

}  // namespace h2ulv
