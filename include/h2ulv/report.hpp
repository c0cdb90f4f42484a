// Drop-in for proj/include/h2ulv/report.hpp (report.hpp:13-109): RunConfig,
// RunReport (h2ulv-report/1, same keys and layout as RunReport::to_json,
// report.cpp:182-237), Pipeline and run_pipeline. One device problem carries
// the whole pipeline; hmatrix() and factors() are host views of it, read back
// on first use.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "h2ulv/solve.hpp"
#include "h2ulv/ulv.hpp"

namespace h2ulv {

struct RunConfig {
  int64_t n = 1024;
  int64_t leaf_size = 256;
  double tol = 1e-8;
  std::optional<int64_t> cap;
  KernelKind kernel = KernelKind::laplace;
  double alpha_m = 1.0;
  std::optional<double> reg;
  double scale = 4.0 * 3.14159265358979323846;
  std::string geometry = "cube";  // cube | line | sphere
  int64_t spheres = 1;
  double spacing = 3.0;
  std::optional<AdmissibilityKind> admissibility;
  double eta = 1.0;
  StructureVariant structure = StructureVariant::h2;
  bool dep = false;
  int threads = 1;
  uint64_t seed = 42;
  bool oracle = true;
  int64_t oracle_guard = 16384;
  bool absorb_coupling = true;
  std::string points_file;
  // B200 extensions: member-panel QR mode and the assembly (FactorOptions).
  int b200_qr_mode = 0;
  bool b200_reference_compat = true;
  int64_t b200_sample_cols = 0;

  AdmissibilityKind effective_admissibility() const {
    if (admissibility) return *admissibility;
    return structure == StructureVariant::h2 ? AdmissibilityKind::strong : AdmissibilityKind::weak;
  }
  FactorVariant factor_variant() const {
    if (structure == StructureVariant::blr2) return FactorVariant::blr2;
    if (structure == StructureVariant::hss) return FactorVariant::hss;
    return dep ? FactorVariant::h2dep : FactorVariant::h2nodep;
  }
  void validate() const {  // report.cpp:43-58
    if (n < 2) throw std::invalid_argument("config: n must be >= 2");
    if (leaf_size < 2) throw std::invalid_argument("config: leaf size must be >= 2");
    if (n < 2 * leaf_size) throw std::invalid_argument("config: need n >= 2 * leaf size");
    if (tol <= 0) throw std::invalid_argument("config: tol must be positive");
    if (cap && *cap < 1) throw std::invalid_argument("config: rank cap must be >= 1");
    if (eta <= 0) throw std::invalid_argument("config: eta must be positive");
    if (threads < 1) throw std::invalid_argument("config: threads must be >= 1");
    if (geometry != "cube" && geometry != "line" && geometry != "sphere")
      throw std::invalid_argument("config: unknown geometry " + geometry);
    if (dep && structure != StructureVariant::h2)
      throw std::invalid_argument("config: the dep variant requires the h2 structure");
    if (structure != StructureVariant::h2 && effective_admissibility() == AdmissibilityKind::strong)
      throw std::invalid_argument("config: hss/blr2 require weak admissibility");
  }
};

struct LevelRankStats {
  int level = 0;
  int64_t dense_blocks = 0;
  int64_t lowrank_blocks = 0;
  int64_t max_rank = 0;
  double mean_rank = 0.0;
};

namespace b200 {
// Shortest round-trip double, integral values with ".0" (nlohmann::json's dump).
inline std::string jnum(double v) {
  if (std::isnan(v) || std::isinf(v)) return "null";
  char buf[40];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof(buf), "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}
inline std::string jstr(const std::string& s) { return "\"" + s + "\""; }
// Insertion-ordered object writer with nlohmann::ordered_json's 2-space
// layout (report.cpp:13 uses ordered_json).
struct JObj {
  std::vector<std::pair<std::string, std::string>> kv;  // values already serialised
  void put(const std::string& k, const std::string& v) { kv.emplace_back(k, v); }
  std::string dump(int indent) const {
    if (kv.empty()) return "{}";
    std::string pad(size_t(indent + 2), ' '), out = "{\n";
    size_t i = 0;
    for (const auto& [k, v] : kv) {
      out += pad + jstr(k) + ": " + v + (++i < kv.size() ? ",\n" : "\n");
    }
    return out + std::string(size_t(indent), ' ') + "}";
  }
};
inline const char* structure_name(StructureVariant v) {
  return v == StructureVariant::h2 ? "h2" : v == StructureVariant::hss ? "hss" : "blr2";
}
}  // namespace b200

struct RunReport {
  std::string schema = "h2ulv-report/1";
  RunConfig config;
  std::map<std::string, double> phase_seconds;
  std::map<std::string, uint64_t> phase_flops;
  uint64_t total_flops = 0;
  uint64_t factorization_flops = 0;
  uint64_t kernel_evals = 0;
  std::vector<LevelRankStats> levels;
  int64_t top_level_max_rank = 0;
  int64_t max_leaf_rank = 0;
  int64_t dense_blocks_leaf = 0;
  int64_t stored_entries = 0;
  int64_t memory_bytes = 0;
  double solve_rel_error = -1.0;
  double max_fill_residual_rel = 0.0;
  int64_t dependency_edges = 0;
  double total_seconds = 0.0;

  std::string to_json() const {
    using b200::jnum;
    using b200::jstr;
    b200::JObj cfg;
    cfg.put("n", std::to_string(config.n));
    cfg.put("leaf_size", std::to_string(config.leaf_size));
    cfg.put("tol", jnum(config.tol));
    if (config.cap) cfg.put("cap", std::to_string(*config.cap));
    cfg.put("kernel", jstr(config.kernel == KernelKind::laplace ? "laplace" : "yukawa"));
    if (config.kernel == KernelKind::yukawa) cfg.put("alpha_m", jnum(config.alpha_m));
    cfg.put("reg", jnum(config.reg ? *config.reg : -1.0));
    cfg.put("geometry", jstr(config.geometry));
    if (config.geometry == "sphere") {
      cfg.put("spheres", std::to_string(config.spheres));
      cfg.put("spacing", jnum(config.spacing));
    }
    cfg.put("admissibility", jstr(config.effective_admissibility() == AdmissibilityKind::weak ? "weak" : "strong"));
    cfg.put("eta", jnum(config.eta));
    cfg.put("structure", jstr(b200::structure_name(config.structure)));
    cfg.put("variant", jstr(config.dep ? "dep" : "nodep"));
    cfg.put("threads", std::to_string(config.threads));
    cfg.put("seed", std::to_string(config.seed));
    b200::JObj walls, flops, j;
    for (const auto& [k, v] : phase_seconds) walls.put(k, jnum(v));
    for (const auto& [k, v] : phase_flops) flops.put(k, std::to_string(v));
    std::string lv = "[]";
    if (!levels.empty()) {
      lv = "[\n";
      for (size_t i = 0; i < levels.size(); ++i) {
        b200::JObj l;
        l.put("level", std::to_string(levels[i].level));
        l.put("dense_blocks", std::to_string(levels[i].dense_blocks));
        l.put("lowrank_blocks", std::to_string(levels[i].lowrank_blocks));
        l.put("max_rank", std::to_string(levels[i].max_rank));
        l.put("mean_rank", jnum(levels[i].mean_rank));
        lv += "    " + l.dump(4) + (i + 1 < levels.size() ? ",\n" : "\n");
      }
      lv += "  ]";
    }
    j.put("schema", jstr(schema));
    j.put("config", cfg.dump(2));
    j.put("wall_seconds", walls.dump(2));
    j.put("flops", flops.dump(2));
    j.put("total_flops", std::to_string(total_flops));
    j.put("factorization_flops", std::to_string(factorization_flops));
    j.put("kernel_evals", std::to_string(kernel_evals));
    j.put("total_seconds", jnum(total_seconds));
    j.put("levels", lv);
    j.put("top_level_max_rank", std::to_string(top_level_max_rank));
    j.put("max_leaf_rank", std::to_string(max_leaf_rank));
    j.put("dense_blocks_leaf", std::to_string(dense_blocks_leaf));
    j.put("stored_entries", std::to_string(stored_entries));
    j.put("memory_bytes", std::to_string(memory_bytes));
    j.put("max_fill_residual_rel", jnum(max_fill_residual_rel));
    j.put("dependency_edges", std::to_string(dependency_edges));
    j.put("solve_rel_error", jnum(solve_rel_error));
    return j.dump(0);
  }
};

inline PointCloud make_cloud(const RunConfig& cfg) {  // report.cpp:60-65
  if (!cfg.points_file.empty()) return read_point_cloud(cfg.points_file);
  if (cfg.geometry == "cube") return generate_uniform_cube(cfg.n, cfg.seed);
  if (cfg.geometry == "line") return generate_line(cfg.n, cfg.seed);
  return generate_sphere_surface(cfg.n, cfg.spheres, cfg.spacing, cfg.seed);
}

inline KernelSpec make_kernel(const RunConfig& cfg, const PointCloud& cloud) {  // report.cpp:67-75
  const double reg = cfg.reg ? *cfg.reg : default_eta_reg(cloud.domain_diameter(), cloud.size());
  KernelSpec spec = cfg.kernel == KernelKind::laplace ? KernelSpec::laplace(reg) : KernelSpec::yukawa(cfg.alpha_m, reg);
  if (cfg.kernel == KernelKind::gaussian) {
    spec.kind = KernelKind::gaussian;
    spec.alpha_m = cfg.alpha_m;
  }
  spec.permittivity_scale = cfg.scale;
  return spec;
}

class Pipeline {
 public:
  explicit Pipeline(const RunConfig& cfg) : cfg_(cfg) { cfg_.validate(); }

  // points, tree, classification, near field (report.cpp:79-91): one device build
  void build() {
    if (built_) return;
    const auto t0 = std::chrono::steady_clock::now();
    original_ = make_cloud(cfg_);
    kernel_ = make_kernel(cfg_, original_);
    dev_ = std::make_shared<b200::Device>();
    dev_->original = original_;
    dev_->leaf = cfg_.leaf_size;
    dev_->setup.kernel = b200::kernel_of(kernel_);
    const AdmissibilityRule rule{cfg_.effective_admissibility(), cfg_.eta};
    dev_->setup.options.structure = b200::structure_code(b200::device_variant(rule, cfg_.structure));
    dev_->setup.options.eta = cfg_.eta;
    dev_->handle = b200::build(original_, cfg_.leaf_size, dev_->setup);
    tree_ = std::make_unique<ClusterTreeResult>(b200::read_tree(dev_->handle->p, original_, cfg_.leaf_size));
    H_ = std::make_unique<HMatrix>();
    H_->variant = cfg_.structure;
    H_->tree = tree_->tree;
    H_->cloud = &tree_->cloud;
    H_->kernel = kernel_;
    H_->structure = b200::read_lists(dev_->handle->p, cfg_.structure, rule);
    H_->b200 = dev_;
    built_ = true;
    build_seconds_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  // fills + bases + ULV factorization (report.cpp:93-106), on the device
  void factor() {
    build();
    if (factored_) return;
    const auto t0 = std::chrono::steady_clock::now();
    b200::factor_once(*dev_, factor_options());
    factored_ = true;
    factor_seconds_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  Matrix solve_rhs(const Matrix& b) const {
    if (!factored_) throw std::logic_error("Pipeline::solve_rhs: factor() first");
    Matrix x(b.rows, b.cols);
    if (b.cols > 0) b200::check(h2g_solve(dev_->handle->p, b.cols, b.data(), x.data()));
    return x;
  }
  RunReport report();

  const RunConfig& config() const { return cfg_; }
  const PointCloud& original_cloud() const { return original_; }
  const HMatrix& hmatrix() const {
    if (!built_) throw std::logic_error("Pipeline::hmatrix: build() first");
    if (H_->leaf_dense.empty()) b200::read_leaf_dense(*H_);
    return *H_;
  }
  const ULVFactors& factors() const {
    if (!factored_) throw std::logic_error("Pipeline::factors: factor() first");
    if (!factors_) factors_ = std::make_unique<ULVFactors>(b200::snapshot(hmatrix(), dev_, cfg_.factor_variant()));
    return *factors_;
  }
  const KernelSpec& kernel() const { return kernel_; }
  // B200 additions: the device problem, and y = A x by direct summation
  // (matvec_dense_oracle without the N guard).
  h2g_problem* handle() const { return dev_ ? dev_->handle->p : nullptr; }
  Matrix matvec(const Matrix& x) const {
    if (!built_) throw std::logic_error("Pipeline::matvec: build() first");
    Matrix y(x.rows, x.cols);
    b200::check(h2g_matvec(dev_->handle->p, x.cols, x.data(), y.data()));
    return y;
  }

 private:
  FactorOptions factor_options() const {
    FactorOptions o;
    o.variant = cfg_.factor_variant();
    o.tol = cfg_.tol;
    o.cap = cfg_.cap;
    o.threads = cfg_.threads;
    o.absorb_coupling = cfg_.absorb_coupling;
    o.b200_qr_mode = cfg_.b200_qr_mode;
    o.b200_reference_compat = cfg_.b200_reference_compat;
    o.b200_sample_cols = cfg_.b200_sample_cols;
    if (o.variant == FactorVariant::h2dep)
      throw std::invalid_argument("config: the dep variant is not on the B200 path (sequential driver)");
    return o;
  }
  RunConfig cfg_;
  PointCloud original_;
  std::unique_ptr<ClusterTreeResult> tree_;
  std::unique_ptr<HMatrix> H_;
  mutable std::unique_ptr<ULVFactors> factors_;
  KernelSpec kernel_;
  std::shared_ptr<b200::Device> dev_;
  bool built_ = false;
  bool factored_ = false;
  double build_seconds_ = 0.0;
  double factor_seconds_ = 0.0;
};

// Pipeline::report (report.cpp:113-180): the device's flop ledger (the
// reference's counting rules) and phase times; the oracle check is the
// reference's: x for b = A 1 against the dense LU solution, N <= guard.
inline RunReport Pipeline::report() {
  factor();
  RunReport rep;
  rep.config = cfg_;
  h2g_problem* p = dev_->handle->p;
  double t5[5], f6[6];
  int64_t launches = 0;
  h2g_stats(p, t5, f6, &launches);
  const char* fnames[6] = {"fill_precompute", "basis", "skeleton", "factorize", "assemble", "solve"};
  for (int k = 0; k < 6; ++k) rep.phase_flops[fnames[k]] = uint64_t(f6[k]);
  // the reference's full phase key set (flops.cpp phase_name), oracle/other included
  rep.phase_flops["oracle"] = 0;
  rep.phase_flops["other"] = 0;
  for (const auto& [k, v] : rep.phase_flops) rep.phase_seconds[k] = 0.0;
  for (int idx = 0;; ++idx) {
    char name[64];
    double sec = 0;
    if (!h2g_phase_seconds(p, idx, name, int(sizeof(name)), &sec)) break;
    // driver sub-phases ("skeleton_leaf_pieces") fold into their reference phase
    std::string key = "other";
    for (const auto& [k, v] : rep.phase_flops) {
      const std::string n(name);
      if (n == k || n.rfind(k + "_", 0) == 0) key = k;
    }
    rep.phase_seconds[key] += sec;
  }
  for (const auto& [k, v] : rep.phase_flops) rep.total_flops += v;
  rep.factorization_flops = rep.phase_flops["fill_precompute"] + rep.phase_flops["factorize"];
  rep.kernel_evals = uint64_t(h2g_kernel_evals(p));
  rep.total_seconds = build_seconds_ + factor_seconds_;
  const ULVFactors& f = factors();
  const HMatrix& H = hmatrix();
  for (int lvl = 1; lvl <= H.structure.levels; ++lvl) {
    LevelRankStats ls;
    ls.level = lvl;
    ls.dense_blocks = H.structure.dense_count(lvl);
    ls.lowrank_blocks = H.structure.far_count(lvl);
    if (lvl < int(f.bases.U.size())) {
      int64_t total = 0, count = 0;
      for (const auto& b : f.bases.U[size_t(lvl)]) {
        if (b.dim() == 0 && b.rank() == 0) continue;
        ls.max_rank = std::max(ls.max_rank, b.rank());
        total += b.rank();
        ++count;
      }
      ls.mean_rank = count ? double(total) / double(count) : 0.0;
    }
    rep.levels.push_back(ls);
  }
  if (!f.levels.empty()) {
    const int top_lvl = f.levels.back().level;
    for (const auto& ls : rep.levels)
      if (ls.level == top_lvl) rep.top_level_max_rank = ls.max_rank;
    for (const auto& ls : rep.levels)
      if (ls.level == H.structure.levels) rep.max_leaf_rank = ls.max_rank;
  }
  rep.dense_blocks_leaf = H.structure.dense_count(H.structure.levels);
  int64_t entries = H.stored_dense_entries();
  for (int lvl = 1; lvl <= f.bases.levels; ++lvl)
    for (const auto& b : f.bases.U[size_t(lvl)]) entries += 2 * (b.Qs.size() + b.Qr.size());
  for (const auto& lf : f.levels)
    for (const auto& e : lf.elim) entries += e.pivot.lu.size() + e.urs.size() + e.lsr.size();
  entries += f.top.lu.size();
  rep.stored_entries = entries;
  rep.memory_bytes = entries * 8;
  for (double r : f.max_fill_residual_rel) rep.max_fill_residual_rel = std::max(rep.max_fill_residual_rel, r);
  rep.dependency_edges = 0;  // level-parallel variants: no intra-level edges (ulv.cpp:1184-1193)
  if (cfg_.oracle && cfg_.n <= cfg_.oracle_guard) {
    Matrix ones(cfg_.n, 1);
    for (int64_t i = 0; i < cfg_.n; ++i) ones(i, 0) = 1.0;
    Matrix b = matvec_dense_oracle(original_, kernel_, ones, cfg_.oracle_guard);
    Matrix x_ref = dense_solve_oracle(original_, kernel_, b, cfg_.oracle_guard);
    rep.solve_rel_error = rel_error(solve_rhs(b), x_ref);
  }
  return rep;
}

inline RunReport run_pipeline(const RunConfig& cfg) {
  Pipeline pipe(cfg);
  return pipe.report();
}

}  // namespace h2ulv
