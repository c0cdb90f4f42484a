// Drop-in for proj/include/h2ulv/hstructure.hpp (hstructure.hpp:15-114).
// classify_blocks and materialize_dense run on the B200 (bit-exact lists and
// near-field blocks); HMatrix keeps the device problem they were built on, so
// prepare_factor_inputs / factorize continue on the GPU without re-uploading.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <utility>
#include <vector>

#include "h2ulv/geometry.hpp"
#include "h2ulv/kernels.hpp"
#include "h2ulv/linalg.hpp"
#include "h2ulv/matrix.hpp"

namespace h2ulv {

enum class StructureVariant { blr2, hss, h2 };

struct BlockId {
  int level = 0;
  int64_t row = 0;
  int64_t col = 0;
  bool operator<(const BlockId& o) const {
    if (level != o.level) return level < o.level;
    if (row != o.row) return row < o.row;
    return col < o.col;
  }
};

enum class BlockKind { dense, lowrank, subdivided, covered };

struct BlockStructure {
  StructureVariant variant = StructureVariant::h2;
  int levels = 0;
  struct LevelPattern {
    std::vector<std::vector<int64_t>> near_cols;  // sorted, diagonal included
    std::vector<std::vector<int64_t>> far_cols;   // sorted
  };
  std::vector<LevelPattern> level;  // indexed by tree level; [0] unused
  AdmissibilityRule b200_rule;      // B200: the rule the lists were classified with

  BlockKind kind(int lvl, int64_t i, int64_t j) const {
    if (lvl <= 0 || lvl > levels) throw std::invalid_argument("BlockStructure::kind: bad level");
    if (is_far(lvl, i, j)) return BlockKind::lowrank;
    if (is_near(lvl, i, j)) return lvl == levels ? BlockKind::dense : BlockKind::subdivided;
    return BlockKind::covered;
  }
  bool is_near(int lvl, int64_t i, int64_t j) const {
    const auto& r = level[size_t(lvl)].near_cols[size_t(i)];
    return std::binary_search(r.begin(), r.end(), j);
  }
  bool is_far(int lvl, int64_t i, int64_t j) const {
    const auto& r = level[size_t(lvl)].far_cols[size_t(i)];
    return std::binary_search(r.begin(), r.end(), j);
  }
  int covering_level(int64_t leaf_i, int64_t leaf_j) const {
    int64_t i = leaf_i, j = leaf_j;
    for (int lvl = levels; lvl >= 1; --lvl) {
      if (is_near(lvl, i, j) || is_far(lvl, i, j)) return lvl;
      i >>= 1;
      j >>= 1;
    }
    throw std::logic_error("covering_level: pair not covered by any level");
  }
  int64_t dense_count(int lvl) const {
    int64_t s = 0;
    for (const auto& row : level[size_t(lvl)].near_cols) s += int64_t(row.size());
    return s;
  }
  int64_t far_count(int lvl) const {
    int64_t s = 0;
    for (const auto& row : level[size_t(lvl)].far_cols) s += int64_t(row.size());
    return s;
  }
  int64_t max_dense_per_row(int lvl) const {
    int64_t s = 0;
    for (const auto& row : level[size_t(lvl)].near_cols) s = std::max(s, int64_t(row.size()));
    return s;
  }
};

namespace b200 {
inline int structure_code(StructureVariant v) { return v == StructureVariant::h2 ? 0 : v == StructureVariant::hss ? 1 : 2; }
// The device classifies h2 with the strong rule and hss / blr2 with the weak one.
inline StructureVariant device_variant(const AdmissibilityRule& rule, StructureVariant v) {
  if (v == StructureVariant::h2 && rule.kind == AdmissibilityKind::weak) return StructureVariant::hss;
  if (v != StructureVariant::h2 && rule.kind == AdmissibilityKind::strong)
    throw std::invalid_argument("classify_blocks: hss/blr2 use weak admissibility");
  return v;
}
inline BlockStructure read_lists(h2g_problem* p, StructureVariant v, const AdmissibilityRule& rule) {
  BlockStructure s;
  s.variant = v;
  s.b200_rule = rule;
  s.levels = h2g_levels(p);
  s.level.resize(size_t(s.levels + 1));
  for (int l = 1; l <= s.levels; ++l)
    for (int far = 0; far < 2; ++far) {
      const int64_t m = int64_t(1) << l;
      const int64_t cnt = h2g_list_count(p, l, far);
      if (cnt < 0) check(1);
      std::vector<int64_t> ptr(size_t(m + 1)), idx(size_t(std::max<int64_t>(1, cnt)));
      check(h2g_list(p, l, far, ptr.data(), idx.data()));
      auto& out = far ? s.level[size_t(l)].far_cols : s.level[size_t(l)].near_cols;
      out.resize(size_t(m));
      for (int64_t i = 0; i < m; ++i)
        out[size_t(i)].assign(idx.begin() + ptr[size_t(i)], idx.begin() + ptr[size_t(i + 1)]);
    }
  return s;
}
inline const PointCloud& original_of(const ClusterTree& tree, const char* who) {
  if (!tree.b200_original)
    throw std::invalid_argument(std::string(who) + ": the B200 path needs a tree made by build_cluster_tree");
  return *tree.b200_original;
}
}  // namespace b200

// classify_blocks (hstructure.cpp:64-114), on the device.
inline BlockStructure classify_blocks(const ClusterTree& tree, const AdmissibilityRule& rule,
                                      StructureVariant variant) {
  const PointCloud& cloud = b200::original_of(tree, "classify_blocks");
  b200::Setup s;
  s.options.structure = b200::structure_code(b200::device_variant(rule, variant));
  s.options.eta = rule.eta;
  auto h = b200::build(cloud, tree.leaf_size_target, s);
  return b200::read_lists(h->p, variant, rule);
}

struct SharedBasis {
  Matrix Qs;
  Matrix Qr;
  int64_t rank() const { return Qs.cols; }
  int64_t dim() const { return Qs.rows; }
  Matrix square() const { return hconcat(Qr, Qs); }  // [Qr | Qs]
};

struct SharedBasisSet {
  int levels = 0;
  std::vector<std::vector<SharedBasis>> U;
  std::vector<std::vector<SharedBasis>> V;
  void init(int levels_) {
    levels = levels_;
    U.assign(size_t(levels_ + 1), {});
    V.assign(size_t(levels_ + 1), {});
    for (int l = 0; l <= levels_; ++l) {
      U[size_t(l)].resize(size_t(int64_t(1) << l));
      V[size_t(l)].resize(size_t(int64_t(1) << l));
    }
  }
  int64_t rank(int lvl, int64_t i) const { return U[size_t(lvl)][size_t(i)].rank(); }
};

namespace b200 {
// The device problem an HMatrix / ULVFactors lives on, with its settings.
struct Device {
  std::shared_ptr<Handle> handle;
  Setup setup;
  PointCloud original;
  int64_t leaf = 0;
  bool factored = false;
  h2g_options factored_with{};
};
}  // namespace b200

struct HMatrix {
  StructureVariant variant = StructureVariant::h2;
  ClusterTree tree;
  const PointCloud* cloud = nullptr;  // reordered cloud (owned by the caller, or by b200_cloud)
  KernelSpec kernel;
  BlockStructure structure;
  std::vector<std::vector<Matrix>> leaf_dense;  // aligned with structure.level[levels].near_cols

  int leaf_level() const { return tree.levels; }
  IndexRange cluster_range(int lvl, int64_t i) const {
    const ClusterNode& nd = tree.node(lvl, i);
    return {nd.begin, nd.end};
  }
  const Matrix& leaf_block(int64_t i, int64_t j) const {
    const auto& cols = structure.level[size_t(tree.levels)].near_cols[size_t(i)];
    auto it = std::lower_bound(cols.begin(), cols.end(), j);
    if (it == cols.end() || *it != j) throw std::out_of_range("HMatrix::leaf_block: no dense block");
    return leaf_dense[size_t(i)][size_t(it - cols.begin())];
  }
  int64_t stored_dense_entries() const {
    int64_t s = 0;
    for (const auto& row : leaf_dense)
      for (const auto& B : row) s += B.size();
    return s;
  }

  std::shared_ptr<b200::Device> b200;  // B200: the device problem
};

namespace b200 {
inline void read_leaf_dense(HMatrix& H) {
  h2g_problem* p = H.b200->handle->p;
  std::vector<double> arena(size_t(h2g_near_entries(p)));
  check(h2g_near_dense(p, arena.data()));
  const int L = H.tree.levels;
  const auto& near = H.structure.level[size_t(L)].near_cols;
  H.leaf_dense.assign(near.size(), {});
  size_t at = 0;
  for (size_t i = 0; i < near.size(); ++i)
    for (int64_t j : near[i]) {
      const IndexRange r = H.cluster_range(L, int64_t(i)), c = H.cluster_range(L, j);
      Matrix B(r.size(), c.size());
      std::copy(arena.begin() + int64_t(at), arena.begin() + int64_t(at + size_t(B.size())), B.data());
      at += size_t(B.size());
      H.leaf_dense[i].push_back(std::move(B));
    }
}
}  // namespace b200

// materialize_dense (hstructure.cpp:142-164): the leaf near field evaluated on
// the device; the returned HMatrix holds the device problem.
inline HMatrix materialize_dense(const BlockStructure& structure, const ClusterTree& tree, const PointCloud& cloud,
                                 const KernelSpec& kernel, StructureVariant variant, int threads = 1) {
  (void)threads;  // one device stream; host threads are not used
  auto dev = std::make_shared<b200::Device>();
  dev->original = b200::original_of(tree, "materialize_dense");
  dev->leaf = tree.leaf_size_target;
  dev->setup.kernel = b200::kernel_of(kernel);
  dev->setup.options.structure = b200::structure_code(b200::device_variant(structure.b200_rule, variant));
  dev->setup.options.eta = structure.b200_rule.eta;
  dev->handle = b200::build(dev->original, dev->leaf, dev->setup);
  HMatrix H;
  H.variant = variant;
  H.tree = tree;
  H.cloud = &cloud;
  H.kernel = kernel;
  H.structure = structure;
  H.b200 = dev;
  b200::read_leaf_dense(H);
  return H;
}

}  // namespace h2ulv
