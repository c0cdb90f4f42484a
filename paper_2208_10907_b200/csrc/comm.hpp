// Multi-GPU level partition: one process per GPU, Morton-contiguous box
// ranges per rank (the reference's offline plan, report.cpp:245-296: P ranks
// own contiguous leaf ranges, a box at level l >= log2 P belongs to rank
// box >> (l - log2 P), coarser levels are replicated), and the one
// collective the partitioned stages need: an in-place all-gather-v of a
// device buffer whose per-rank segments are contiguous (outputs laid out in
// box order, so each owner's boxes form one byte range).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

namespace h2g {

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // Rank r holds bytes [offs[r], offs[r+1]) of buf (device); afterwards every
  // rank holds all of [offs[0], offs[size]). Ordered on `st`.
  virtual void allgatherv(void* buf, const std::vector<int64_t>& offs, cudaStream_t st) = 0;
  // Boxes of an m-box level owned by this rank: [lo, hi). Levels with fewer
  // boxes than ranks are replicated (every rank computes every box).
  bool partitioned(int64_t m) const { return size > 1 && m >= size; }
  int64_t lo(int64_t m, int r) const { return m * r / size; }
  int64_t lo(int64_t m) const { return lo(m, rank); }
  int64_t hi(int64_t m) const { return lo(m, rank + 1); }
};

// NCCL communicator (libnccl.so.2 resolved at run time, so the library loads
// without NCCL; the all-gather-v is a group of in-place broadcasts, one per
// owner, over NVLink/NVSwitch).
void nccl_unique_id(void* out128);
std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* unique_id);

// Host-mediated exchange through a caller callback (e.g. a gloo process group
// in tests): the owned segment is staged to pinned host memory, the callback
// all-gathers the host buffer, the result is copied back.
typedef int (*HostAllgatherFn)(void* user, void* host_buf, const int64_t* byte_offs, int nranks);
std::shared_ptr<Comm> make_host_comm(int nranks, int rank, HostAllgatherFn fn, void* user);

}  // namespace h2g
