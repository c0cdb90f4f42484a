// Drop-in for proj/include/h2ulv/compression.hpp (the types the factor
// objects expose: DenseSystem, FillInSet). The compression itself (fills,
// fill-augmented bases, transfers) runs inside the device factorization.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <utility>
#include <vector>

#include "h2ulv/hstructure.hpp"
#include "h2ulv/kernels.hpp"
#include "h2ulv/linalg.hpp"

namespace h2ulv {

using PairKey = std::pair<int64_t, int64_t>;

// Per-level dense block system (compression.hpp:21-38). In the B200 façade
// every block is owned (copied back from the device).
struct DenseSystem {
  std::vector<int64_t> dims;
  std::vector<std::vector<int64_t>> near_cols;
  std::map<PairKey, int64_t> slots;
  std::vector<Matrix> owned;
  std::vector<const Matrix*> views;
  std::vector<LuFactors> diag_lu;

  int64_t m() const { return static_cast<int64_t>(dims.size()); }
  bool has(int64_t i, int64_t j) const { return slots.count({i, j}) != 0; }
  const Matrix& block(int64_t i, int64_t j) const {
    auto it = slots.find({i, j});
    if (it == slots.end()) throw std::out_of_range("DenseSystem::block: no dense block");
    const int64_t s = it->second;
    return s >= 0 ? owned[size_t(s)] : *views[size_t(-1 - s)];
  }
  void put(int64_t i, int64_t j, Matrix&& B) {
    slots[{i, j}] = static_cast<int64_t>(owned.size());
    owned.push_back(std::move(B));
  }
  void put_view(int64_t i, int64_t j, const Matrix* B) {
    slots[{i, j}] = -1 - static_cast<int64_t>(views.size());
    views.push_back(B);
  }
  bool has_offdiag() const {
    for (int64_t i = 0; i < m(); ++i)
      for (int64_t j : near_cols[size_t(i)])
        if (j != i) return true;
    return false;
  }
  int64_t total_dim() const {
    int64_t s = 0;
    for (int64_t d : dims) s += d;
    return s;
  }
};

struct FillInSet {
  std::map<PairKey, Matrix> fills;
  bool empty() const { return fills.empty(); }
  const Matrix* find(int64_t i, int64_t j) const {
    auto it = fills.find({i, j});
    return it == fills.end() ? nullptr : &it->second;
  }
};

// Composed point x rank bases per level (compression.hpp:97-102, :288-322).
struct BigBasisLayer {
  int level = 0;
  std::vector<Matrix> Ubig, Vbig;
};

inline BigBasisLayer make_leaf_layer(const SharedBasisSet& bases) {
  BigBasisLayer layer;
  layer.level = bases.levels;
  const auto& U = bases.U[size_t(bases.levels)];
  const auto& V = bases.V[size_t(bases.levels)];
  for (size_t i = 0; i < U.size(); ++i) {
    layer.Ubig.push_back(U[i].Qs);
    layer.Vbig.push_back(V[i].Qs);
  }
  return layer;
}

inline BigBasisLayer lift_layer(const BigBasisLayer& child, const SharedBasisSet& bases, int level) {
  if (child.level != level + 1) throw std::logic_error("lift_layer: layer level mismatch");
  BigBasisLayer layer;
  layer.level = level;
  const int64_t m = int64_t(1) << level;
  for (int64_t k = 0; k < m; ++k) {
    const Matrix& Tu = bases.U[size_t(level)][size_t(k)].Qs;
    const Matrix& Tv = bases.V[size_t(level)][size_t(k)].Qs;
    const Matrix& u0 = child.Ubig[size_t(2 * k)];
    const Matrix& u1 = child.Ubig[size_t(2 * k + 1)];
    const Matrix& v0 = child.Vbig[size_t(2 * k)];
    const Matrix& v1 = child.Vbig[size_t(2 * k + 1)];
    layer.Ubig.push_back(vconcat(matmul(u0, Tu.block(0, 0, u0.cols, Tu.cols)),
                                 matmul(u1, Tu.block(u0.cols, 0, u1.cols, Tu.cols))));
    layer.Vbig.push_back(vconcat(matmul(v0, Tv.block(0, 0, v0.cols, Tv.cols)),
                                 matmul(v1, Tv.block(v0.cols, 0, v1.cols, Tv.cols))));
  }
  return layer;
}

// Rows of K's two children projected on their Ubig, raw columns `cols`
// (compression.cpp:324-341), in 512-column panels.
inline Matrix project_rows_to_merged(const HMatrix& H, const BigBasisLayer& child_layer, int lvl, int64_t K,
                                     IndexRange cols) {
  const int64_t c0 = 2 * K, c1 = 2 * K + 1;
  const Matrix& u0 = child_layer.Ubig[size_t(c0)];
  const Matrix& u1 = child_layer.Ubig[size_t(c1)];
  const IndexRange r0 = H.cluster_range(lvl + 1, c0), r1 = H.cluster_range(lvl + 1, c1);
  Matrix out(u0.cols + u1.cols, cols.size());
  const int64_t panel = 512;
  for (int64_t at = cols.begin; at < cols.end; at += panel) {
    const IndexRange pc{at, std::min(cols.end, at + panel)};
    out.set_block(0, at - cols.begin, matmul(u0, assemble_block(H.kernel, *H.cloud, r0, pc), true, false));
    out.set_block(u0.cols, at - cols.begin, matmul(u1, assemble_block(H.kernel, *H.cloud, r1, pc), true, false));
  }
  return out;
}

inline Matrix project_pair_to_merged(const HMatrix& H, const BigBasisLayer& child_layer, int lvl, int64_t K,
                                     int64_t J) {
  const IndexRange jr = H.cluster_range(lvl, J);
  Matrix P = project_rows_to_merged(H, child_layer, lvl, K, jr);
  const Matrix& v0 = child_layer.Vbig[size_t(2 * J)];
  const Matrix& v1 = child_layer.Vbig[size_t(2 * J + 1)];
  return hconcat(matmul(P.block(0, 0, P.rows, v0.rows), v0), matmul(P.block(0, v0.rows, P.rows, v1.rows), v1));
}

}  // namespace h2ulv
