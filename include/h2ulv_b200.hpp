// h2ulv_b200 — C++ host façade of the B200 hot path, mirroring the
// reference's proj/include/h2ulv API (RunConfig / Pipeline / PointCloud /
// ClusterTree / BlockStructure / solve) over the C ABI in h2g.h, so a C++
// caller of the reference switches by changing the namespace and linking
// libh2g.so. Header-only; C++17.
//
//   reference (proj/include/h2ulv)              here
//   PointCloud, generate_* (geometry.hpp:10-24)  same names, same SplitMix64 streams
//   build_cluster_tree (geometry.hpp:58)         build_cluster_tree (2-means on the GPU, bit-exact)
//   classify_blocks (hstructure.hpp:55-56)       classify_blocks (GPU lists, bit-exact)
//   RunConfig / Pipeline (report.hpp:13-99)      RunConfig / Pipeline (build, factor, solve_rhs)
//   solve (solve.hpp:10)                         solve(const Pipeline&, const Matrix&)
//   matvec_dense_oracle (solve.cpp:234-239)      matvec (matrix-free, no N guard)
//
// Errors keep the reference's exception types and messages: invalid_argument
// for configuration errors (RunConfig::validate, report.cpp:43-58),
// runtime_error for numerical ones ("singular block in LU of S^RR at step
// 3", "basis does not absorb fill-in at level 5 block (2,7)", ...).
#pragma once
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2g.h"

namespace h2ulv_b200 {

// ---- Matrix (matrix.hpp:9-53): column-major FP64, (i, j) at data[j*rows + i]
struct Matrix {
  int64_t rows = 0, cols = 0;
  std::vector<double> values;
  Matrix() = default;
  Matrix(int64_t r, int64_t c) : rows(r), cols(c), values(size_t(r * c), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return values[size_t(j * rows + i)]; }
  double operator()(int64_t i, int64_t j) const { return values[size_t(j * rows + i)]; }
  double* data() { return values.data(); }
  const double* data() const { return values.data(); }
};

// ---- SplitMix64 (prng.hpp:10-29)
class SplitMix64 {
 public:
  explicit SplitMix64(uint64_t seed) : state_(seed) {}
  uint64_t next_u64() {
    uint64_t z = (state_ += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_signed() { return 2.0 * next_double() - 1.0; }

 private:
  uint64_t state_;
};

// ---- geometry (geometry.hpp:10-24, geometry.cpp:42-95)
struct PointCloud {
  std::vector<std::array<double, 3>> points;
  std::vector<double> charges;
  int64_t size() const { return static_cast<int64_t>(points.size()); }
  double domain_diameter() const {  // geometry.cpp:28-40 (bounding-box diagonal)
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (const auto& p : points)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], p[d]);
        hi[d] = std::max(hi[d], p[d]);
      }
    const double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
    return std::sqrt(std::fma(d2, d2, d0 * d0 + d1 * d1));
  }
};

inline PointCloud generate_uniform_cube(int64_t n, uint64_t seed) {
  if (n < 2) throw std::invalid_argument("generate_uniform_cube: n must be >= 2");
  SplitMix64 rng(seed);
  PointCloud c;
  c.points.resize(size_t(n));
  c.charges.assign(size_t(n), 1.0);
  for (auto& p : c.points)
    for (int d = 0; d < 3; ++d) p[d] = rng.next_double();
  return c;
}

inline PointCloud generate_line(int64_t n, uint64_t seed) {
  if (n < 2) throw std::invalid_argument("generate_line: n must be >= 2");
  SplitMix64 rng(seed);
  PointCloud c;
  c.points.resize(size_t(n));
  c.charges.assign(size_t(n), 1.0);
  for (auto& p : c.points) p = {rng.next_double(), 0.0, 0.0};
  return c;
}

// ---- kernels / structure (kernels.hpp:11-39, geometry.hpp:60-67, hstructure.hpp:15)
enum class KernelKind { laplace, yukawa, gaussian };
enum class StructureVariant { blr2, hss, h2 };  // hstructure.hpp:15
enum class AdmissibilityKind { weak, strong };
struct AdmissibilityRule {
  AdmissibilityKind kind = AdmissibilityKind::strong;
  double eta = 1.0;
};
struct KernelSpec {
  KernelKind kind = KernelKind::laplace;
  double alpha_m = 1.0;
  double permittivity_scale = 4.0 * 3.14159265358979323846;
  double eta_reg = 1e-3;
};

namespace detail {
inline void check(int rc) {
  if (rc == 0) return;
  const std::string msg = h2g_last_error();
  if (msg.rfind("config:", 0) == 0 || msg.find("need N >=") != std::string::npos ||
      msg.find("must be") != std::string::npos)
    throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
struct Handle {
  h2g_problem* p = nullptr;
  Handle() { check(h2g_create(&p)); }
  ~Handle() { h2g_destroy(p); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
};
inline void soa(const PointCloud& c, std::vector<double>& xyz) {
  xyz.resize(size_t(3 * c.size()));
  for (int64_t i = 0; i < c.size(); ++i)
    for (int d = 0; d < 3; ++d) xyz[size_t(3 * i + d)] = c.points[size_t(i)][d];
}
inline std::shared_ptr<Handle> build(const PointCloud& cloud, int64_t leaf, const KernelSpec& k,
                                     double eta, StructureVariant v, double tol,
                                     std::optional<int64_t> cap, bool absorb, int qr_mode = 0) {
  auto h = std::make_shared<Handle>();
  h2g_kernel hk{k.kind == KernelKind::laplace ? 0 : k.kind == KernelKind::yukawa ? 1 : 2, k.alpha_m, k.permittivity_scale, k.eta_reg};
  h2g_options o{tol, cap.value_or(0), 1e-13, absorb ? 1 : 0, 100.0, v == StructureVariant::h2 ? 0 : v == StructureVariant::hss ? 1 : 2, eta, 0, qr_mode, 1};
  check(h2g_set_kernel(h->p, &hk));
  check(h2g_set_options(h->p, &o));
  std::vector<double> xyz;
  soa(cloud, xyz);
  check(h2g_build(h->p, cloud.size(), xyz.data(), cloud.charges.data(), leaf));
  return h;
}
}  // namespace detail

// ---- ClusterTree (geometry.hpp:29-55)
struct ClusterNode {
  int64_t begin = 0, end = 0;
  std::array<double, 3> center{};
  double radius = 0.0;
};
struct ClusterTree {
  int levels = 0;
  int64_t leaf_size_target = 0;
  std::vector<ClusterNode> nodes;       // heap layout, offset 2^l - 1 + i
  std::vector<int64_t> original_index;  // reordered position -> original position
  int64_t num_clusters(int level) const { return int64_t(1) << level; }
  int64_t num_leaves() const { return num_clusters(levels); }
  const ClusterNode& node(int level, int64_t i) const { return nodes[size_t((int64_t(1) << level) - 1 + i)]; }
};
struct ClusterTreeResult {
  ClusterTree tree;
  PointCloud cloud;  // reordered
};

namespace detail {
inline ClusterTreeResult read_tree(h2g_problem* p, int64_t n, int64_t leaf) {
  ClusterTreeResult r;
  r.tree.levels = h2g_levels(p);
  r.tree.leaf_size_target = leaf;
  const size_t nn = (size_t(2) << r.tree.levels) - 1;
  std::vector<int64_t> be(2 * nn);
  std::vector<double> cr(4 * nn);
  r.tree.original_index.resize(size_t(n));
  check(h2g_tree_perm(p, r.tree.original_index.data()));
  check(h2g_nodes(p, be.data(), cr.data()));
  r.tree.nodes.resize(nn);
  for (size_t k = 0; k < nn; ++k)
    r.tree.nodes[k] = {be[2 * k], be[2 * k + 1], {cr[4 * k], cr[4 * k + 1], cr[4 * k + 2]}, cr[4 * k + 3]};
  std::vector<double> xyz(size_t(3 * n));
  r.cloud.charges.resize(size_t(n));
  check(h2g_reordered_points(p, xyz.data(), r.cloud.charges.data()));
  r.cloud.points.resize(size_t(n));
  for (int64_t i = 0; i < n; ++i) r.cloud.points[size_t(i)] = {xyz[size_t(3 * i)], xyz[size_t(3 * i + 1)], xyz[size_t(3 * i + 2)]};
  return r;
}
}  // namespace detail

// build_cluster_tree (geometry.hpp:58): 2-means bisection, on the GPU.
inline ClusterTreeResult build_cluster_tree(const PointCloud& cloud, int64_t leaf_size) {
  auto h = detail::build(cloud, leaf_size, KernelSpec{}, 1.0, StructureVariant::h2, 1e-8, std::nullopt, true);
  return detail::read_tree(h->p, cloud.size(), leaf_size);
}

// ---- BlockStructure (hstructure.hpp:33-53)
struct LevelBlocks {
  std::vector<std::vector<int64_t>> near_cols, far_cols;  // sorted, near includes the diagonal
};
struct BlockStructure {
  int levels = 0;
  std::vector<LevelBlocks> level;  // index 0..levels
};

namespace detail {
inline BlockStructure read_lists(h2g_problem* p) {
  BlockStructure s;
  s.levels = h2g_levels(p);
  s.level.resize(size_t(s.levels + 1));
  for (int l = 1; l <= s.levels; ++l)
    for (int far = 0; far < 2; ++far) {
      const int64_t m = int64_t(1) << l;
      std::vector<int64_t> ptr(size_t(m + 1)), idx(size_t(std::max<int64_t>(1, h2g_list_count(p, l, far))));
      check(h2g_list(p, l, far, ptr.data(), idx.data()));
      auto& out = far ? s.level[size_t(l)].far_cols : s.level[size_t(l)].near_cols;
      out.resize(size_t(m));
      for (int64_t i = 0; i < m; ++i) out[size_t(i)].assign(idx.begin() + ptr[size_t(i)], idx.begin() + ptr[size_t(i + 1)]);
    }
  return s;
}
}  // namespace detail

// classify_blocks (hstructure.hpp:55-56) for the tree build_cluster_tree
// makes of `cloud` (the tree is deterministic, so it is rebuilt on the GPU).
inline BlockStructure classify_blocks(const PointCloud& cloud, int64_t leaf_size, const AdmissibilityRule& rule,
                                      StructureVariant v = StructureVariant::h2) {
  if (rule.kind == AdmissibilityKind::weak && v == StructureVariant::h2) v = StructureVariant::hss;
  auto h = detail::build(cloud, leaf_size, KernelSpec{}, rule.eta, v, 1e-8, std::nullopt, true);
  return detail::read_lists(h->p);
}

// ---- RunConfig / Pipeline (report.hpp:13-99)
struct RunConfig {
  int64_t n = 1024;
  int64_t leaf_size = 256;
  double tol = 1e-8;
  std::optional<int64_t> cap;
  KernelKind kernel = KernelKind::laplace;
  double alpha_m = 1.0;
  std::optional<double> reg;  // default: 1e-3 * domain diameter / N^(1/3)
  double scale = 4.0 * 3.14159265358979323846;
  std::string geometry = "cube";  // cube | line (others: pass points)
  double eta = 1.0;
  StructureVariant structure = StructureVariant::h2;
  uint64_t seed = 42;
  bool absorb_coupling = true;
  std::optional<PointCloud> points;  // import instead of generating
  // B200 extension: 0 = exact QR (bit-exact with the reference), 1 = blocked QR
  // (reflectors applied 32 at a time; parity within tolerance).
  int qr_mode = 0;

  void validate() const {  // report.cpp:43-58
    if (n < 2) throw std::invalid_argument("config: n must be >= 2");
    if (leaf_size < 2) throw std::invalid_argument("config: leaf size must be >= 2");
    if (n < 2 * leaf_size) throw std::invalid_argument("config: need n >= 2 * leaf size");
    if (!(tol > 0)) throw std::invalid_argument("config: tol must be positive");
    if (cap && *cap < 1) throw std::invalid_argument("config: rank cap must be >= 1");
    if (!(eta > 0)) throw std::invalid_argument("config: eta must be positive");
    if (!points && geometry != "cube" && geometry != "line")
      throw std::invalid_argument("config: unknown geometry " + geometry);
  }
};

inline PointCloud make_cloud(const RunConfig& cfg) {  // report.cpp:60-65
  if (cfg.points) return *cfg.points;
  return cfg.geometry == "line" ? generate_line(cfg.n, cfg.seed) : generate_uniform_cube(cfg.n, cfg.seed);
}

inline KernelSpec make_kernel(const RunConfig& cfg, const PointCloud& cloud) {  // report.cpp:67-77
  KernelSpec k;
  k.kind = cfg.kernel;
  k.alpha_m = cfg.kernel == KernelKind::laplace ? 0.0 : cfg.alpha_m;
  k.permittivity_scale = cfg.scale;
  k.eta_reg = cfg.reg ? *cfg.reg : 1e-3 * cloud.domain_diameter() / std::cbrt(double(cloud.size()));
  return k;
}

class Pipeline {
 public:
  explicit Pipeline(const RunConfig& cfg) : cfg_(cfg) { cfg_.validate(); }
  void build() {  // points, tree, classification, near field (report.cpp:79-91)
    if (built_) return;
    original_ = make_cloud(cfg_);
    kernel_ = make_kernel(cfg_, original_);
    h_ = detail::build(original_, cfg_.leaf_size, kernel_, cfg_.eta, cfg_.structure, cfg_.tol, cfg_.cap,
                       cfg_.absorb_coupling, cfg_.qr_mode);
    built_ = true;
  }
  void factor() {  // bases + fills + ULV factorization (report.cpp:93-106)
    build();
    if (!factored_) detail::check(h2g_factor(h_->p));
    factored_ = true;
  }
  // b: n x nrhs column-major in the original point order (solve.hpp:10).
  Matrix solve_rhs(const Matrix& b) const {
    if (!factored_) throw std::logic_error("Pipeline::solve_rhs: factor() first");
    Matrix x(b.rows, b.cols);
    detail::check(h2g_solve(h_->p, b.cols, b.data(), x.data()));
    return x;
  }
  // y = A x by direct summation on the GPU (matvec_dense_oracle without the N guard).
  Matrix matvec(const Matrix& x) const {
    if (!built_) throw std::logic_error("matvec: build() first");
    Matrix y(x.rows, x.cols);
    detail::check(h2g_matvec(h_->p, x.cols, x.data(), y.data()));
    return y;
  }
  ClusterTreeResult tree() const { return detail::read_tree(h_->p, original_.size(), cfg_.leaf_size); }
  BlockStructure structure() const { return detail::read_lists(h_->p); }
  // Per factorized level: (tree level, skeleton ranks) (ULVFactors::levels, ulv.hpp:60-68).
  std::vector<std::pair<int, std::vector<int64_t>>> ranks() const {
    std::vector<std::pair<int, std::vector<int64_t>>> out;
    const int nl = h2g_num_factor_levels(h_->p);
    for (int li = 0; li < nl; ++li) {
      std::vector<int64_t> r(size_t(int64_t(1) << h2g_levels(h_->p)));
      const int lvl = h2g_factor_level(h_->p, li, r.data());
      r.resize(size_t(int64_t(1) << lvl));
      out.push_back({lvl, r});
    }
    return out;
  }
  // Partition the factorization over a communicator's ranks (multi-GPU).
  void set_comm(h2g_comm* c) {
    build();
    detail::check(h2g_set_comm(h_->p, c));
  }
  const RunConfig& config() const { return cfg_; }
  const PointCloud& original_cloud() const { return original_; }
  const KernelSpec& kernel() const { return kernel_; }
  h2g_problem* handle() const { return h_ ? h_->p : nullptr; }

 private:
  RunConfig cfg_;
  PointCloud original_;
  KernelSpec kernel_;
  std::shared_ptr<detail::Handle> h_;
  bool built_ = false, factored_ = false;
};

inline Matrix solve(const Pipeline& pipe, const Matrix& b) { return pipe.solve_rhs(b); }

}  // namespace h2ulv_b200
