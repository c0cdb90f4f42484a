// Device memory arena of the factorization.
//
// A factorization step allocates and frees ~5,000 blocks, a few of them tens
// of GB. Through the stream-ordered allocator (cudaMallocAsync) a multi-GB
// request made next to other live multi-GB blocks re-maps physical memory
// inside the driver's pool: 1-4 ms of host time per GB, every step, while the
// stream runs dry (47 ms for one 13.6 GB slab at the bench size), and how
// often that happens depends on the pool's history, so identical steps
// differed by +-10 %. The arena takes the driver out of the steady state:
// memory is obtained in a few large segments (cudaMalloc, the first one a
// fixed share of the free memory), blocks are carved from them best-fit with
// splitting and coalescing, and nothing is returned to the driver until
// trim() or an out-of-memory retry. Every step of a sequence replays the same
// request sequence against the same free lists, so placement is identical and
// no allocation makes a driver call.
//
// Ordering: a block is reusable in stream order on the stream that freed it
// (all of a problem's work runs on one stream). A free block remembers that
// stream; handing it to another stream first waits for the releasing stream
// (or nothing once stream_gone() has said the stream was synchronised and
// retired), and blocks released by different streams are not coalesced.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "batch.hpp"

namespace h2g {

namespace {

constexpr size_t kAlign = 512;

struct Arena {
  struct Blk {
    size_t size;
    bool free;
    int seg;
    cudaStream_t owner;  // free blocks: the stream that released it (nullptr: usable by anyone)
  };
  struct Seg {
    char* base;
    size_t size;
  };
  std::mutex mu;
  std::map<char*, Blk> blocks;                  // every block, address-ordered
  std::multimap<size_t, char*> free_by_size;    // free blocks
  std::vector<Seg> segs;
  size_t free_total = 0, reserved = 0;

  void erase_free(char* p, size_t size) {
    auto r = free_by_size.equal_range(size);
    for (auto it = r.first; it != r.second; ++it)
      if (it->second == p) {
        free_by_size.erase(it);
        return;
      }
  }

  bool grow(size_t bytes) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
    static const double frac = getenv("H2G_ARENA_FRACTION") ? atof(getenv("H2G_ARENA_FRACTION")) : 0.7;
    size_t want = segs.empty() ? size_t(double(fr) * frac) : std::max<size_t>(bytes, size_t(4) << 30);
    want = std::max(want, bytes);
    want = (want + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    void* p = nullptr;
    while (true) {
      if (cudaMalloc(&p, want) == cudaSuccess) break;
      cudaGetLastError();
      if (want == ((bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1))) return false;
      want = std::max<size_t>(bytes, want / 2);
      want = (want + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    }
    segs.push_back({static_cast<char*>(p), want});
    blocks[static_cast<char*>(p)] = Blk{want, true, int(segs.size()) - 1, nullptr};
    free_by_size.emplace(want, static_cast<char*>(p));
    free_total += want;
    reserved += want;
    return true;
  }

  // Segments that are one free block go back to the driver.
  void trim_locked() {
    for (size_t s = 0; s < segs.size(); ++s) {
      if (!segs[s].base) continue;
      auto it = blocks.find(segs[s].base);
      if (it == blocks.end() || !it->second.free || it->second.size != segs[s].size) continue;
      if (it->second.owner) {
        if (cudaStreamSynchronize(it->second.owner) != cudaSuccess) cudaGetLastError();
      }
      erase_free(it->first, it->second.size);
      free_total -= segs[s].size;
      reserved -= segs[s].size;
      blocks.erase(it);
      cudaFree(segs[s].base);
      segs[s].base = nullptr;
    }
  }

  void* alloc(size_t bytes, cudaStream_t st) {
    bytes = (bytes + kAlign - 1) & ~(kAlign - 1);
    std::lock_guard<std::mutex> lock(mu);
    for (int attempt = 0; attempt < 3; ++attempt) {
      // best fit among blocks this stream may take directly, else the best fit of any stream
      auto pick = free_by_size.end();
      for (auto it = free_by_size.lower_bound(bytes); it != free_by_size.end(); ++it) {
        const Blk& b = blocks[it->second];
        if (b.owner == nullptr || b.owner == st) {
          pick = it;
          break;
        }
        if (pick == free_by_size.end()) pick = it;
        if (it->first > 2 * bytes + (size_t(64) << 20)) break;  // do not scan far past the fit
      }
      if (pick != free_by_size.end()) {
        char* p = pick->second;
        Blk b = blocks[p];
        free_by_size.erase(pick);
        if (b.owner && b.owner != st) {
          if (cudaStreamSynchronize(b.owner) != cudaSuccess) cudaGetLastError();  // a retired stream is done
        }
        if (b.size - bytes >= kAlign) {
          blocks[p + bytes] = Blk{b.size - bytes, true, b.seg, b.owner};
          free_by_size.emplace(b.size - bytes, p + bytes);
          b.size = bytes;
        }
        b.free = false;
        b.owner = nullptr;
        blocks[p] = b;
        free_total -= b.size;
        return p;
      }
      if (attempt == 0) {
        if (grow(bytes)) continue;
        trim_locked();
        if (grow(bytes)) continue;
      }
      break;
    }
    return nullptr;
  }

  void release(void* q, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    char* p = static_cast<char*>(q);
    auto it = blocks.find(p);
    if (it == blocks.end() || it->second.free) return;  // not ours (or a double free): ignore
    it->second.free = true;
    it->second.owner = st;
    free_total += it->second.size;
    // coalesce with the next and the previous block of the same segment and stream
    auto nx = std::next(it);
    if (nx != blocks.end() && nx->second.free && nx->second.seg == it->second.seg &&
        nx->second.owner == st && it->first + it->second.size == nx->first) {
      erase_free(nx->first, nx->second.size);
      it->second.size += nx->second.size;
      blocks.erase(nx);
    }
    if (it != blocks.begin()) {
      auto pv = std::prev(it);
      if (pv->second.free && pv->second.seg == it->second.seg && pv->second.owner == st &&
          pv->first + pv->second.size == it->first) {
        erase_free(pv->first, pv->second.size);
        pv->second.size += it->second.size;
        blocks.erase(it);
        it = pv;
      }
    }
    free_by_size.emplace(it->second.size, it->first);
  }

  void stream_gone(cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    for (auto& [p, b] : blocks)
      if (b.free && b.owner == st) b.owner = nullptr;
    // merge what the stream tags kept apart
    for (auto it = blocks.begin(); it != blocks.end();) {
      auto nx = std::next(it);
      if (nx != blocks.end() && it->second.free && nx->second.free && it->second.owner == nullptr &&
          nx->second.owner == nullptr && it->second.seg == nx->second.seg &&
          it->first + it->second.size == nx->first) {
        erase_free(it->first, it->second.size);
        erase_free(nx->first, nx->second.size);
        it->second.size += nx->second.size;
        blocks.erase(nx);
        free_by_size.emplace(it->second.size, it->first);
      } else {
        it = nx;
      }
    }
  }
};

// One arena per device, never destroyed (no CUDA calls at process exit).
Arena& arena() {
  static std::mutex mu;
  static std::map<int, Arena*> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  Arena*& a = per_dev[dev];
  if (!a) a = new Arena;
  return *a;
}

}  // namespace

void* arena_alloc(size_t bytes, cudaStream_t st) { return arena().alloc(bytes, st); }
void arena_free(void* p, cudaStream_t st) { arena().release(p, st); }
void arena_stream_gone(cudaStream_t st) { arena().stream_gone(st); }
size_t arena_free_bytes() {
  Arena& a = arena();
  std::lock_guard<std::mutex> lock(a.mu);
  return a.free_total;
}
void trim_device_memory() {
  Arena& a = arena();
  std::lock_guard<std::mutex> lock(a.mu);
  a.trim_locked();
}

}  // namespace h2g
