// Communicators for the multi-GPU level partition (comm.hpp).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "comm.hpp"

namespace h2g {

void cuda_check(cudaError_t e, const char* what);  // batch.cu

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // The soname torch (or the host application) already loaded wins.
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) throw std::runtime_error(std::string("h2g: NCCL unavailable: ") + dlerror());
    auto sym = [&](const char* n) {
      void* s = dlsym(a.h, n);
      if (!s) throw std::runtime_error(std::string("h2g: NCCL symbol missing: ") + n);
      return s;
    };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(sym("ncclBroadcast"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("h2g: ") + what + ": " + nccl().error_string(r));
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().comm_destroy(comm);
  }
  void allgatherv(void* buf, const std::vector<int64_t>& offs, cudaStream_t st) override {
    auto* b = static_cast<char*>(buf);
    nccl_check(nccl().group_start(), "ncclGroupStart");
    for (int r = 0; r < size; ++r) {
      const int64_t n = offs[r + 1] - offs[r];
      if (n > 0) nccl_check(nccl().broadcast(b + offs[r], b + offs[r], size_t(n), ncclChar, r, comm, st),
                            "ncclBroadcast");
    }
    nccl_check(nccl().group_end(), "ncclGroupEnd");
  }
};

struct HostComm : Comm {
  HostAllgatherFn fn = nullptr;
  void* user = nullptr;
  void allgatherv(void* buf, const std::vector<int64_t>& offs, cudaStream_t st) override {
    const int64_t total = offs[size] - offs[0];
    if (total <= 0) return;
    void* host = nullptr;
    cuda_check(cudaMallocHost(&host, size_t(total)), "pinned exchange buffer");
    auto* h = static_cast<char*>(host);
    auto* d = static_cast<char*>(buf);
    const int64_t mine = offs[rank + 1] - offs[rank];
    try {
      if (mine > 0)
        cuda_check(cudaMemcpyAsync(h + offs[rank] - offs[0], d + offs[rank], size_t(mine),
                                   cudaMemcpyDeviceToHost, st),
                   "exchange d2h");
      cuda_check(cudaStreamSynchronize(st), "exchange sync");
      std::vector<int64_t> rel(offs.size());
      for (size_t r = 0; r < offs.size(); ++r) rel[r] = offs[r] - offs[0];
      if (fn(user, h, rel.data(), size) != 0) throw std::runtime_error("h2g: host all-gather callback failed");
      cuda_check(cudaMemcpyAsync(d + offs[0], h, size_t(total), cudaMemcpyHostToDevice, st), "exchange h2d");
      cuda_check(cudaStreamSynchronize(st), "exchange sync");
    } catch (...) {
      cudaFreeHost(host);
      throw;
    }
    cudaFreeHost(host);
  }
};

void check_ranks(int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("h2g: bad rank / world size");
}

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == NCCL_UNIQUE_ID_BYTES, "unique id size");
  std::memcpy(out128, &id, sizeof(id));
}

std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* unique_id) {
  check_ranks(nranks, rank);
  auto c = std::make_unique<NcclComm>();
  c->rank = rank;
  c->size = nranks;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  nccl_check(nccl().comm_init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  return c;
}

std::shared_ptr<Comm> make_host_comm(int nranks, int rank, HostAllgatherFn fn, void* user) {
  check_ranks(nranks, rank);
  if (!fn) throw std::invalid_argument("h2g: null all-gather callback");
  auto c = std::make_unique<HostComm>();
  c->rank = rank;
  c->size = nranks;
  c->fn = fn;
  c->user = user;
  return c;
}

}  // namespace h2g
