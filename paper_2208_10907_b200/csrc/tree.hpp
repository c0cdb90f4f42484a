// Device-resident cluster tree and host-side block structure.
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace h2g {

// Reordered cloud (SoA) and heap-layout node table on the device
// (ClusterTree, geometry.hpp:29-55; node(l, i) = nodes[2^l - 1 + i]).
struct DeviceTree {
  int64_t n = 0, leaf = 0;
  int levels = 0;
  double *x = nullptr, *y = nullptr, *z = nullptr, *q = nullptr;
  int64_t* order = nullptr;  // reordered position -> original index
  int64_t* be = nullptr;     // 2 per node: begin, end
  double* geo = nullptr;     // 4 per node: centre xyz, radius
  // scratch
  double *x2 = nullptr, *y2 = nullptr, *z2 = nullptr, *q2 = nullptr;
  int64_t* order2 = nullptr;
  double* cent = nullptr;
  unsigned char* assign = nullptr;
  double *margin = nullptr, *key0 = nullptr, *key1 = nullptr;
  int *idx0 = nullptr, *idx1 = nullptr, *node_of = nullptr, *flag = nullptr;
  std::vector<void*> owned;
  int64_t alloc_n = -1, alloc_nodes = -1;  // sizes the buffers were allocated for

  void alloc(int64_t n_, int64_t nodes);
  void release_scratch();
  ~DeviceTree();
};

// Near/far lists per level as CSR (BlockStructure, hstructure.hpp:33-53).
struct Structure {
  int levels = 0;
  struct Level {
    std::vector<int64_t> near_ptr, near_idx, far_ptr, far_idx;
  };
  std::vector<Level> level;  // [0] unused
  int64_t nnear(int l, int64_t i) const { return level[l].near_ptr[i + 1] - level[l].near_ptr[i]; }
  const int64_t* near(int l, int64_t i) const { return level[l].near_idx.data() + level[l].near_ptr[i]; }
  int64_t nfar(int l, int64_t i) const { return level[l].far_ptr[i + 1] - level[l].far_ptr[i]; }
  const int64_t* far(int l, int64_t i) const { return level[l].far_idx.data() + level[l].far_ptr[i]; }
  bool is_near(int l, int64_t i, int64_t j) const;
  bool is_far(int l, int64_t i, int64_t j) const;
};

int tree_levels(int64_t n, int64_t leaf);
void build_tree_device(DeviceTree& T, const double* d_xyz_aos, const double* d_q, int64_t n,
                       int64_t leaf, cudaStream_t st);
void classify_device(DeviceTree& T, double eta, int weak, Structure& S, cudaStream_t st);

}  // namespace h2g
