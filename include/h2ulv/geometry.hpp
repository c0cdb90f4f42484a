// Drop-in for proj/include/h2ulv/geometry.hpp (geometry.hpp:10-72).
// Generators: h2g_generate_points (the reference's SplitMix64 streams and
// Fibonacci spheres bit for bit). build_cluster_tree: the 2-means tree built
// on the B200 (bit-exact permutation, ranges, centres and radii).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2g.h"
#include "h2ulv/linalg.hpp"

namespace h2ulv {

struct PointCloud {
  std::vector<std::array<double, 3>> points;
  std::vector<double> charges;
  int64_t size() const { return static_cast<int64_t>(points.size()); }
  double domain_diameter() const {  // geometry.cpp:28-40, the reference's contraction
    const double big = std::numeric_limits<double>::max();
    double lo[3] = {big, big, big}, hi[3] = {-big, -big, -big};
    for (const auto& p : points)
      for (int d = 0; d < 3; ++d) {
        if (p[d] < lo[d]) lo[d] = p[d];
        if (p[d] > hi[d]) hi[d] = p[d];
      }
    const double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
    return std::sqrt(std::fma(d2, d2, d0 * d0 + d1 * d1));
  }
};

namespace b200 {
inline PointCloud generate(int32_t geometry, int64_t n, uint64_t seed, int64_t spheres, double spacing) {
  std::vector<double> xyz(size_t(3 * (n > 0 ? n : 0))), q(size_t(n > 0 ? n : 0));
  if (h2g_generate_points(geometry, n, seed, spheres, spacing, xyz.data(), q.data()) != 0)
    throw std::invalid_argument(h2g_points_last_error());
  PointCloud c;
  c.points.resize(size_t(n));
  c.charges = std::move(q);
  for (int64_t i = 0; i < n; ++i) c.points[size_t(i)] = {xyz[size_t(3 * i)], xyz[size_t(3 * i + 1)], xyz[size_t(3 * i + 2)]};
  return c;
}
inline void aos(const PointCloud& c, std::vector<double>& xyz) {
  xyz.resize(size_t(3 * c.size()));
  for (int64_t i = 0; i < c.size(); ++i)
    for (int d = 0; d < 3; ++d) xyz[size_t(3 * i + d)] = c.points[size_t(i)][size_t(d)];
}
}  // namespace b200

inline PointCloud generate_uniform_cube(int64_t n, uint64_t seed) {
  if (n < 2) throw std::invalid_argument("generate_uniform_cube: n must be >= 2");
  return b200::generate(H2G_GEOM_CUBE, n, seed, 1, 3.0);
}
inline PointCloud generate_line(int64_t n, uint64_t seed) {
  if (n < 2) throw std::invalid_argument("generate_line: n must be >= 2");
  return b200::generate(H2G_GEOM_LINE, n, seed, 1, 3.0);
}
inline PointCloud generate_sphere_surface(int64_t n, int64_t spheres, double spacing, uint64_t seed) {
  if (n < 2) throw std::invalid_argument("generate_sphere_surface: n must be >= 2");
  return b200::generate(H2G_GEOM_SPHERE, n, seed, spheres, spacing);
}
// BASELINE.json geometries the reference lacks (B200 extensions).
inline PointCloud generate_uniform_sphere(int64_t n, uint64_t seed) {
  return b200::generate(H2G_GEOM_UNIFORM_SPHERE, n, seed, 1, 3.0);
}
inline PointCloud generate_ellipsoids(int64_t n, int64_t count, uint64_t seed) {
  return b200::generate(H2G_GEOM_ELLIPSOIDS, n, seed, count, 3.0);
}

// "%.17g x y z q" per line (geometry.cpp:97-119); exact round trip.
inline void write_point_cloud(const PointCloud& cloud, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("write_point_cloud: cannot open " + path);
  char buf[160];
  for (int64_t i = 0; i < cloud.size(); ++i) {
    const auto& p = cloud.points[size_t(i)];
    std::snprintf(buf, sizeof(buf), "%.17g %.17g %.17g %.17g\n", p[0], p[1], p[2], cloud.charges[size_t(i)]);
    f << buf;
  }
}
inline PointCloud read_point_cloud(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("read_point_cloud: cannot open " + path);
  PointCloud cloud;
  double x, y, z, q;
  while (f >> x >> y >> z >> q) {
    cloud.points.push_back({x, y, z});
    cloud.charges.push_back(q);
  }
  if (cloud.size() < 2) throw std::runtime_error("read_point_cloud: fewer than 2 points");
  return cloud;
}

struct ClusterNode {
  int64_t begin = 0;
  int64_t end = 0;
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
  ClusterNode& node(int level, int64_t i) { return nodes[size_t((int64_t(1) << level) - 1 + i)]; }
  // B200: the original-order cloud the tree was built from (the device
  // rebuilds the same, deterministic, tree from it for classify_blocks /
  // materialize_dense).
  std::shared_ptr<const PointCloud> b200_original;
};

struct ClusterTreeResult {
  ClusterTree tree;
  PointCloud cloud;  // reordered
};

enum class AdmissibilityKind { weak, strong };
struct AdmissibilityRule {
  AdmissibilityKind kind = AdmissibilityKind::strong;
  double eta = 1.0;
};
enum class Admissibility { admissible, dense, subdivide };

// admissible (geometry.cpp:263-277).
inline Admissibility admissible(const ClusterTree& tree, int level, int64_t a, int64_t b,
                                const AdmissibilityRule& rule) {
  const bool leaf = level == tree.levels;
  if (rule.kind == AdmissibilityKind::weak) {
    if (a != b) return Admissibility::admissible;
    return leaf ? Admissibility::dense : Admissibility::subdivide;
  }
  const ClusterNode& na = tree.node(level, a);
  const ClusterNode& nb = tree.node(level, b);
  const double dx = na.center[0] - nb.center[0], dy = na.center[1] - nb.center[1],
               dz = na.center[2] - nb.center[2];
  const double dist = std::sqrt(std::fma(dz, dz, std::fma(dx, dx, dy * dy)));
  if (dist > rule.eta * (na.radius + nb.radius)) return Admissibility::admissible;
  return leaf ? Admissibility::dense : Admissibility::subdivide;
}

namespace b200 {
struct Handle {
  h2g_problem* p = nullptr;
  Handle() { check(h2g_create(&p)); }
  ~Handle() { h2g_destroy(p); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
};

// Device settings a handle is built with (KernelSpec / structure / options).
struct Setup {
  // A tree-only build (build_cluster_tree / classify_blocks) still evaluates
  // the near field on the device; a unit regularisation keeps r = 0 regular
  // there (those blocks are discarded).
  h2g_kernel kernel{0, 0.0, 4.0 * 3.14159265358979323846, 1.0};
  h2g_options options{1e-8, 0, 1e-13, 1, 100.0, 0, 1.0, 0, 0, 1};
};

inline std::shared_ptr<Handle> build(const PointCloud& cloud, int64_t leaf, const Setup& s) {
  auto h = std::make_shared<Handle>();
  check(h2g_set_kernel(h->p, &s.kernel));
  check(h2g_set_options(h->p, &s.options));
  std::vector<double> xyz;
  aos(cloud, xyz);
  check(h2g_build(h->p, cloud.size(), xyz.data(), cloud.charges.data(), leaf));
  return h;
}

inline ClusterTreeResult read_tree(h2g_problem* p, const PointCloud& original, int64_t leaf) {
  const int64_t n = original.size();
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
  for (int64_t i = 0; i < n; ++i)
    r.cloud.points[size_t(i)] = {xyz[size_t(3 * i)], xyz[size_t(3 * i + 1)], xyz[size_t(3 * i + 2)]};
  r.tree.b200_original = std::make_shared<const PointCloud>(original);
  return r;
}
}  // namespace b200

// build_cluster_tree (geometry.cpp:222-261): 2-means bisection on the B200.
inline ClusterTreeResult build_cluster_tree(const PointCloud& cloud, int64_t leaf_size) {
  auto h = b200::build(cloud, leaf_size, b200::Setup{});
  return b200::read_tree(h->p, cloud, leaf_size);
}

}  // namespace h2ulv
