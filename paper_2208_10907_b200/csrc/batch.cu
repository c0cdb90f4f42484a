// Host-side batch launchers (see batch.hpp).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <map>
#include <mutex>

#include "batch.hpp"

#include <cstring>

namespace h2g {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void smem_attr(const void* kernel, size_t bytes, const char* what) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), what);
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (bytes <= have) return;
  cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)), what);
  have = bytes;
}

size_t Ctx::free_bytes() const {
  size_t fr = 0, tot = 0;
  cuda_check(cudaMemGetInfo(&fr, &tot), "meminfo");
  return fr + arena_free_bytes();
}

// Device blocks come from the arena (arena.cu); H2G_NO_ARENA=1 goes back to
// the stream-ordered allocator.
Slab Ctx::alloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 8;
  bytes = (bytes + 255) & ~size_t(255);
  static const bool hp = getenv("H2G_HOST_PROF") != nullptr;
  const auto t0 = hp ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
  cudaStream_t s = stream;
  if (use_arena) {
    p = arena_alloc(bytes, s);
    if (!p)
      throw std::runtime_error("device memory exhausted allocating " + std::to_string(bytes) +
                               " bytes in phase " + phase + ": out of memory");
  } else {
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error("device memory exhausted allocating " + std::to_string(bytes) +
                               " bytes in phase " + phase + ": " + cudaGetErrorString(e));
    }
  }
  if (hp) {
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 2.0) fprintf(stderr, "HOSTALLOC %.1f ms for %.3f GB in phase %s\n", ms, bytes / 1e9, phase.c_str());
  }
  if (use_arena) return Slab(p, [s](void* q) { arena_free(q, s); });
  return Slab(p, [s](void* q) { cudaFreeAsync(q, s); });
}

void Ctx::check_err() {
  ErrWord h{};
  cuda_check(cudaMemcpy(&h, err, sizeof(h), cudaMemcpyDeviceToHost), "error word");
  if (h.code == 0) return;
  cuda_check(cudaMemset(err, 0, sizeof(ErrWord)), "error reset");
  if (h.code == 1)
    throw std::runtime_error("assemble_block: singular evaluation (r + eta_reg == 0)");
  if (h.code == 2) {
    std::string what = "block";
    auto it = lu_names.find(h.tag);
    if (it != lu_names.end() && h.job >= 0 && h.job < int(it->second.size())) what = it->second[h.job];
    lu_names.clear();
    throw std::runtime_error("singular block in LU of " + what + " at step " +
                             std::to_string(h.step));
  }
  throw std::runtime_error("device error code " + std::to_string(h.code));
}

cudaEvent_t Ctx::prof_begin() {
  if (!prof) return nullptr;
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "event");
  cuda_check(cudaEventRecord(e, stream), "event record");
  return e;
}

void Ctx::prof_end(const char* name, cudaEvent_t a, double flops, double bytes) {
  if (!prof || !a) return;
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "event");
  cuda_check(cudaEventRecord(e, stream), "event record");
  std::string nm = name;
  if (prof_detail && nm.find('@') == std::string::npos) nm += "@" + phase;  // every record carries its phase
  prec.push_back({nm, a, e, flops, bytes, phase});
}

void Ctx::prof_resolve() {
  for (auto& r : prec) {
    float ms = 0;
    cuda_check(cudaEventSynchronize(r.b), "event sync");
    cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "elapsed");
    auto& g = pagg[r.name];
    g.ms += ms;
    g.flops += r.flops;
    g.bytes += r.bytes;
    g.launches++;
    if (prof_gaps && last_end) {
      float gms = 0;
      cuda_check(cudaEventElapsedTime(&gms, last_end, r.a), "elapsed");
      auto& gg = pagg["gap@" + r.phase];
      gg.ms += gms;
      gg.launches++;
      if (gms > 2.0f)
        fprintf(stderr, "TIMELINE gap %.1f ms after %s before %s@%s\n", gms, last_name.c_str(),
                r.name.c_str(), r.phase.c_str());
    }
    cudaEventDestroy(r.a);
    if (last_end) cudaEventDestroy(last_end);
    last_end = r.b;
    last_name = r.name;
  }
  prec.clear();
}

char* Ctx::stage_reserve(size_t bytes) {
  if (!pin) {
    pin_cap = size_t(64) << 20;
    if (cudaMallocHost(&pin, pin_cap) != cudaSuccess) {
      cudaGetLastError();
      pin = nullptr;
      pin_cap = 0;
    }
  }
  const size_t need = (bytes + 255) & ~size_t(255);
  if (!pin || need > pin_cap) return nullptr;
  if (pin_head + need > pin_cap) {
    cuda_check(cudaStreamSynchronize(stream), "stage sync");
    pin_head = 0;
  }
  char* d = pin + pin_head;
  pin_head += need;
  return d;
}

const void* Ctx::stage(const void* src, size_t bytes) {
  if (!pin) {
    pin_cap = size_t(64) << 20;
    if (cudaMallocHost(&pin, pin_cap) != cudaSuccess) {
      cudaGetLastError();
      pin = nullptr;
      pin_cap = 0;
    }
  }
  const size_t need = (bytes + 255) & ~size_t(255);
  if (!pin || need > pin_cap) return src;  // pageable fallback
  if (pin_head + need > pin_cap) {
    cuda_check(cudaStreamSynchronize(stream), "stage sync");
    pin_head = 0;
  }
  char* d = pin + pin_head;
  pin_head += need;
  memcpy(d, src, bytes);
  return d;
}

Ctx::~Ctx() {
  // The owner may already have destroyed the stream; cudaFreeHost waits for
  // the device itself.
  if (pin) cudaFreeHost(pin);
}


int* Ctx::ticket() {
  constexpr int kTickets = 8192;
  if (!tickets || tickets_used >= kTickets) {
    if (!tickets) tickets = alloc(sizeof(int) * kTickets);
    cuda_check(cudaMemsetAsync(tickets.get(), 0, sizeof(int) * kTickets, stream), "ticket reset");
    tickets_used = 0;
  }
  return static_cast<int*>(tickets.get()) + tickets_used++;
}

void Ctx::sync() {
  pin_head = 0;
  cuda_check(cudaStreamSynchronize(stream), "stream sync");
  check_err();
  lu_names.clear();  // every LU batch launched so far has completed without error
}

std::vector<DMat> alloc_mats(Ctx& c, const std::vector<std::pair<int, int>>& shapes) {
  size_t total = 0;
  std::vector<size_t> off(shapes.size());
  for (size_t t = 0; t < shapes.size(); ++t) {
    off[t] = total;
    total += (size_t(shapes[t].first) * shapes[t].second + 3) & ~size_t(3);  // 32 B aligned
  }
  Slab s = c.alloc(total * sizeof(double));
  std::vector<DMat> out(shapes.size());
  for (size_t t = 0; t < shapes.size(); ++t) {
    double* p = static_cast<double*>(s.get()) + off[t];
    out[t].m = Mat{p, shapes[t].first, shapes[t].second, 1, shapes[t].first > 0 ? shapes[t].first : 1};
    out[t].owner = s;
  }
  return out;
}

DMat alloc_mat(Ctx& c, int rows, int cols) { return alloc_mats(c, {{rows, cols}})[0]; }

LuF alloc_lu(Ctx& c, int n) { return alloc_lus(c, {n})[0]; }

std::vector<LuF> alloc_lus(Ctx& c, const std::vector<int>& ns) {
  std::vector<std::pair<int, int>> shapes;
  size_t np = 0;
  for (int n : ns) {
    shapes.push_back({n, n});
    np += n;
  }
  auto mats = alloc_mats(c, shapes);
  Slab ps = c.alloc(sizeof(int64_t) * (np ? np : 1));
  std::vector<LuF> out(ns.size());
  size_t at = 0;
  for (size_t t = 0; t < ns.size(); ++t) {
    out[t].lu = mats[t];
    out[t].pslab = ps;
    out[t].perm = static_cast<int64_t*>(ps.get()) + at;
    at += ns[t];
  }
  return out;
}

namespace {

// Prefix sums of the jobs' 64 x 64 tile counts (njobs + 1 entries).
template <class J>
std::vector<int> tiles_of(const std::vector<J>& jobs, Mat J::*field) {
  std::vector<int> ptr(jobs.size() + 1, 0);
  for (size_t j = 0; j < jobs.size(); ++j) {
    const Mat& m = jobs[j].*field;
    const int64_t t = (m.rows <= 0 || m.cols <= 0) ? 0 : int64_t((m.rows + 63) / 64) * ((m.cols + 63) / 64);
    if (ptr[j] + t > int64_t(0x7fffffff)) throw std::runtime_error("batch: too many tiles in one launch");
    ptr[j + 1] = ptr[j] + int(t);
  }
  return ptr;
}

}  // namespace

// H2G_HOST_PROF: host seconds spent inside the batch launchers (descriptor
// building, uploads, launches), by kind; printed by host_prof_report().
namespace {
struct HostTimer {
  static std::map<std::string, std::pair<double, int64_t>>& acc() {
    static std::map<std::string, std::pair<double, int64_t>> a;
    return a;
  }
  static bool on() {
    static const bool v = getenv("H2G_HOST_PROF") != nullptr;
    return v;
  }
  const char* name;
  std::chrono::steady_clock::time_point t0;
  explicit HostTimer(const char* n) : name(n) {
    if (on()) t0 = std::chrono::steady_clock::now();
  }
  ~HostTimer() {
    if (!on()) return;
    auto& e = acc()[name];
    e.first += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    e.second++;
  }
};
}  // namespace

void host_prof_report() {
  if (!HostTimer::on()) return;
  for (auto& [k, v] : HostTimer::acc())
    fprintf(stderr, "HOSTBATCH %-10s %8.2f ms in %6ld calls (%.1f us each)\n", k.c_str(), v.first * 1e3, long(v.second),
            v.second ? v.first * 1e6 / v.second : 0.0);
  HostTimer::acc().clear();
}

void GemmBatch::run(Ctx& c, int tag) {
  if (jobs.empty()) return;
  HostTimer ht("gemm");
  std::vector<GemmTile> tiles;
  double fl = 0;
  int max_rows = 0;
  for (auto& j : jobs) max_rows = std::max(max_rows, j.C.rows);
  const int bm = gemm_tile_rows(max_rows);
  // Plain operands (no generated B, no symmetric tile skipping): the persistent
  // m8n8k4 kernel with 8-row tile granularity (k_gemm8.cu).
  static const bool p8_on = getenv("H2G_GEMM_P8") == nullptr || atoi(getenv("H2G_GEMM_P8")) != 0;
  bool p8 = p8_on && bm == 128;
  for (size_t s = 0; p8 && s < segs.size(); ++s) p8 = !segs[s].gen;
  for (size_t j = 0; j < jobs.size(); ++j) {
    const Mat& C = jobs[j].C;
    if (C.rows <= 0 || C.cols <= 0) continue;
    if (p8) {
      const int tm = gemm_p8_row_tiles(C.rows), tn = gemm_p8_col_tiles(C.cols);
      // Symmetric C: a tile is kept when its first column is below its last row.
      auto keep = [&](int a, int b) { return !lower[j] || b * gemm_p8_tile_cols() < gemm_p8_row_end(C.rows, a); };
      int kept = 0;
      for (int b = 0; b < tn; ++b)
        for (int a = 0; a < tm; ++a)
          if (keep(a, b)) {
            tiles.push_back({int(j), a, b});
            ++kept;
          }
      const double frac = double(kept) / (tm * tn);
      for (int s = 0; s < jobs[j].nseg; ++s)
        fl += frac * 2.0 * C.rows * double(segs[jobs[j].seg0 + s].A.cols) * C.cols;
      continue;
    }
    const int tm = (C.rows + bm - 1) / bm, tn = (C.cols + 63) / 64;
    // Symmetric C: tiles entirely above the diagonal are skipped (and not counted).
    auto above = [&](int a, int b) { return lower[j] && b * 64 >= (a + 1) * bm; };
    int kept = 0;
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b) kept += above(a, b) ? 0 : 1;
    const double frac = double(kept) / (tm * tn);
    for (int s = 0; s < jobs[j].nseg; ++s) {
      const GemmSeg& sg = segs[jobs[j].seg0 + s];
      fl += frac * 2.0 * C.rows * double(sg.A.cols) * C.cols;
      if (sg.gen) {
        fl += double(sg.A.cols) * C.cols * kernel_entry_flops(c.kp.kind);
        c.kernel_evals += double(sg.A.cols) * C.cols;
      }
    }
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b)
        if (!above(a, b)) tiles.push_back({int(j), a, b});
  }
  c.add_flops(fl);
  if (tiles.empty()) return;
  Slab k1, k4;
  const int2* dmask = masks.empty() ? nullptr : upload(c, masks, k4);  // (its address goes into the segments)
  for (size_t s = 0; s < segs.size(); ++s)
    if (segs[s].gen && seg_mask_off[s] >= 0) segs[s].g.mask = dmask + seg_mask_off[s];
  for (size_t j = 0; j < jobs.size(); ++j) jobs[j].lower = lower[j] ? 1 : 0;
  void *pj = nullptr, *ps = nullptr, *ptl = nullptr;
  upload_parts(c, k1, {{jobs.data(), sizeof(GemmJob) * jobs.size(), &pj},
                       {segs.data(), sizeof(GemmSeg) * segs.size(), &ps},
                       {tiles.data(), sizeof(GemmTile) * tiles.size(), &ptl}});
  const GemmJob* dj = static_cast<const GemmJob*>(pj);
  const GemmSeg* ds = static_cast<const GemmSeg*>(ps);
  const GemmTile* dt = static_cast<const GemmTile*>(ptl);
  double by = 0;
  for (auto& j : jobs) {
    by += 8.0 * j.C.rows * double(j.C.cols) * (j.acc ? 2 : 1);
    for (int s = 0; s < j.nseg; ++s) {
      const GemmSeg& sg = segs[j.seg0 + s];
      by += 8.0 * sg.A.rows * double(sg.A.cols) + (sg.gen ? 0.0 : 8.0 * sg.B.rows * double(sg.B.cols));
    }
  }
  static const bool shapes = getenv("H2G_GEMM_SHAPES") != nullptr;
  if (shapes) {  // launch shape census (profiling aid)
    double sr = 0, sc = 0, sk = 0, nseg = 0, ngen = 0;
    for (auto& j : jobs) {
      sr += j.C.rows;
      sc += j.C.cols;
      for (int q = 0; q < j.nseg; ++q) {
        sk += segs[j.seg0 + q].A.cols;
        ngen += segs[j.seg0 + q].gen;
      }
      nseg += j.nseg;
    }
    int rmin = 1 << 30, rmax = 0, cmin = 1 << 30, cmax = 0, kmin = 1 << 30, kmax = 0, acc = 0, acm = 0, bcm = 0;
    for (auto& j : jobs) {
      rmin = std::min(rmin, j.C.rows); rmax = std::max(rmax, j.C.rows);
      cmin = std::min(cmin, j.C.cols); cmax = std::max(cmax, j.C.cols);
      acc += j.acc ? 1 : 0;
      int kt = 0;
      for (int q = 0; q < j.nseg; ++q) {
        kt += segs[j.seg0 + q].A.cols;
        acm += segs[j.seg0 + q].A.rs == 1;
        bcm += segs[j.seg0 + q].B.rs == 1;
      }
      kmin = std::min(kmin, kt); kmax = std::max(kmax, kt);
    }
    fprintf(stderr, "GEMMRANGE rows %d-%d cols %d-%d Ktot %d-%d acc %d Acolmajor %d Bcolmajor %d of %.0f segs\n", rmin, rmax,
            cmin, cmax, kmin, kmax, acc, acm, bcm, nseg);
    const double nj = double(jobs.size());
    fprintf(stderr, "GEMMSHAPE %s@%s jobs %zu tiles %zu bm %d rows %.0f cols %.0f segs %.1f K/seg %.0f gen %.0f%% GF %.2f\n",
            name ? name : "gemm", c.phase.c_str(), jobs.size(), tiles.size(), bm, sr / nj, sc / nj, nseg / nj,
            sk / std::max(1.0, nseg), 100.0 * ngen / std::max(1.0, nseg), fl * 1e-9);
  }
  cudaEvent_t sh0 = nullptr, sh1 = nullptr;
  if (shapes) {  // per-launch time of the census (serialises the stream: profiling only)
    cudaEventCreate(&sh0);
    cudaEventCreate(&sh1);
    cudaEventRecord(sh0, c.stream);
  }
  auto ev = c.prof_begin();
  if (p8)
    launch_gemm_p8(dj, ds, dt, int(tiles.size()), c.ticket(), c.stream);
  else
    launch_gemm(dj, ds, dt, int(tiles.size()), bm, c.kp, c.cloud, c.err, tag, c.stream,
                name && std::string(name) == "gram" ? 1 : 0);
  if (shapes) {
    cudaEventRecord(sh1, c.stream);
    cudaEventSynchronize(sh1);
    float ms = 0;
    cudaEventElapsedTime(&ms, sh0, sh1);
    fprintf(stderr, "GEMMTIME %.3f ms %.2f TF/s\n", ms, ms > 0 ? fl / (ms * 1e-3) * 1e-12 : 0.0);
    cudaEventDestroy(sh0);
    cudaEventDestroy(sh1);
  }
  const std::string nm = name ? name : "gemm";
  c.prof_end(c.prof_detail ? (nm + "@" + c.phase).c_str() : nm.c_str(), ev, fl, by);
  c.launches++;
  cuda_check(cudaGetLastError(), "gemm launch");
}

void EvalBatch::run(Ctx& c, int tag) {
  if (jobs.empty()) return;
  HostTimer ht("eval");
  const std::vector<int> tp = tiles_of(jobs, &EvalJob::out);
  double evn_ = 0;
  for (auto& j : jobs) evn_ += double(j.out.rows) * j.out.cols;
  const double ev_flops_ = evn_ * kernel_entry_flops(c.kp.kind);
  c.kernel_evals += evn_;
  c.add_flops(ev_flops_);
  if (tp.back() == 0) return;
  Slab k1;
  void *pj = nullptr, *pt = nullptr;
  upload_parts(c, k1, {{jobs.data(), sizeof(EvalJob) * jobs.size(), &pj}, {tp.data(), sizeof(int) * tp.size(), &pt}});
  auto* dj = static_cast<const EvalJob*>(pj);
  auto* dtp = static_cast<const int*>(pt);
  auto ev = c.prof_begin();
  launch_eval(dj, dtp, int(jobs.size()), tp.back(), c.kp, c.cloud, c.err, tag, c.stream);
  c.prof_end(c.prof_detail ? ("eval@" + c.phase).c_str() : "eval", ev, ev_flops_, 8.0 * evn_);
  c.launches++;
  cuda_check(cudaGetLastError(), "eval launch");
}

void CopyBatch::run(Ctx& c) {
  if (jobs.empty()) return;
  HostTimer ht("copy");
  const std::vector<int> tp = tiles_of(jobs, &CopyJob::dst);
  if (tp.back() == 0) return;
  Slab k1;
  void *pj = nullptr, *pt = nullptr;
  upload_parts(c, k1, {{jobs.data(), sizeof(CopyJob) * jobs.size(), &pj}, {tp.data(), sizeof(int) * tp.size(), &pt}});
  auto* dj = static_cast<const CopyJob*>(pj);
  auto* dtp = static_cast<const int*>(pt);
  double by = 0;
  for (auto& j : jobs) by += 8.0 * j.dst.rows * double(j.dst.cols) * (1 + (j.src.p ? 1 : 0) + j.add);
  auto ev = c.prof_begin();
  launch_copy(dj, dtp, int(jobs.size()), tp.back(), c.stream);
  c.prof_end(c.prof_detail ? ("copy@" + c.phase).c_str() : "copy", ev, 0.0, by);
  c.launches++;
  cuda_check(cudaGetLastError(), "copy launch");
}

void AccBatch::run(Ctx& c) {
  if (jobs.empty()) return;
  HostTimer ht("accum");
  const std::vector<int> tp = tiles_of(jobs, &AccJob::dst);
  if (tp.back() == 0) return;
  Slab k1, k2, k4;
  auto* dj = upload(c, jobs, k1);
  auto* ds = upload(c, srcs, k4);
  auto* dtp = upload(c, tp, k2);
  double by = 0;
  for (auto& j : jobs) by += 8.0 * j.dst.rows * double(j.dst.cols) * (1 + j.nsrc + (j.zero_init ? 0 : 1));
  auto ev = c.prof_begin();
  launch_accum(dj, ds, dtp, int(jobs.size()), tp.back(), c.stream);
  c.prof_end("accum", ev, 0.0, by);
  c.launches++;
  cuda_check(cudaGetLastError(), "accum launch");
}

std::vector<double> NormBatch::run(Ctx& c) {
  std::vector<double> out(mats.size(), 0.0);
  if (mats.empty()) return out;
  Slab res = c.alloc(sizeof(double) * mats.size());
  std::vector<NormJob> jobs(mats.size());
  for (size_t t = 0; t < mats.size(); ++t) jobs[t] = {mats[t], static_cast<double*>(res.get()) + t};
  Slab k1;
  auto* dj = upload(c, jobs, k1);
  launch_norms(dj, int(jobs.size()), c.stream);
  c.launches++;
  cuda_check(cudaMemcpyAsync(out.data(), res.get(), sizeof(double) * mats.size(),
                             cudaMemcpyDeviceToHost, c.stream),
             "norms d2h");
  c.sync();
  return out;
}

static void run_blocked_lu(Ctx& c, const std::vector<LuJob>& js, const std::vector<std::string>& names) {
  double fl = 0, by = 0;
  int max_n = 1;
  for (auto& j : js) {
    const double n = j.A.rows;
    for (double k = 0; k < n; ++k) fl += (n - k - 1) + 2.0 * (n - k - 1) * (n - k - 1);
    by += 16.0 * n * n;
    max_n = std::max(max_n, j.A.rows);
  }
  c.add_flops(fl);
  c.lu_names[++c.lu_tag] = names;
  const int tag = c.lu_tag;
  const int nj = int(js.size());
  Slab am = c.alloc(sizeof(double) * js.size()), k1;
  double* amax = static_cast<double*>(am.get());
  const LuJob* dj = upload(c, js, k1);
  auto ev = c.prof_begin();
  launch_lu_amax(dj, nj, amax, c.stream);
  constexpr int NB = 32;
  for (int kb = 0; kb < max_n; kb += NB) {
    const int nb = std::min(NB, max_n - kb);
    launch_lu_panel(dj, nj, max_n, kb, nb, amax, c.err, tag, c.stream);
    launch_lu_rows(dj, nj, max_n, kb, nb, c.stream);
    GemmBatch gb;
    for (auto& j : js) {
      const int n = j.A.rows;
      if (kb >= n) continue;
      const int nbj = std::min(NB, n - kb), r = n - kb - nbj;
      if (r <= 0) continue;
      gb.job(j.A.sub(kb + nbj, kb + nbj, r, r), true);
      gb.seg(j.A.sub(kb + nbj, kb, r, nbj), j.A.sub(kb, kb + nbj, nbj, r), -1.0);
      c.add_flops(-2.0 * r * double(nbj) * r);  // counted once above (reference LU rule)
    }
    const bool pr = c.prof;
    c.prof = false;  // the trailing GEMMs are part of this "lu" record
    gb.run(c, tag);
    c.prof = pr;
    c.launches += 2;
  }
  c.prof_end("lu", ev, fl, by);
  cuda_check(cudaGetLastError(), "blocked lu");
}

void LuBatch::run(Ctx& c) {
  if (jobs.empty()) return;
  HostTimer ht("lu");
  // Large blocks (the top system) go through the blocked LU: one CTA would
  // walk a ~1000-column factorization alone (100 ms at the bench size).
  static const bool unblocked = getenv("H2G_LU_UNBLOCKED") != nullptr;
  if (!unblocked) {
    // Blocks of kLuBlocked rows or more (H2G_LU_BLOCKED_MIN) take the blocked
    // path together: panel kernels touch 32 columns per step instead of the
    // whole trailing block, which goes through the DMMA GEMM once per panel.
    // Default 384 = the top system only. Measured at the bench size with 128
    // (every leaf block blocked): LU kernels 27 -> 15 ms, but the ~300 extra
    // small launches cost more stream idle time than that (factor 1.21 -> 1.28 s).
    static const int kLuBlocked = getenv("H2G_LU_BLOCKED_MIN") ? atoi(getenv("H2G_LU_BLOCKED_MIN")) : 384;
    std::vector<LuJob> small, big;
    std::vector<std::string> snames, bnames;
    for (size_t t = 0; t < jobs.size(); ++t) {
      if (jobs[t].A.rows >= kLuBlocked) {
        big.push_back(jobs[t]);
        bnames.push_back(names[t]);
      } else {
        small.push_back(jobs[t]);
        snames.push_back(names[t]);
      }
    }
    if (!big.empty()) run_blocked_lu(c, big, bnames);
    if (small.size() != jobs.size()) {
      jobs.swap(small);
      names.swap(snames);
      if (jobs.empty()) return;
    }
  }
  double fl = 0;
  for (auto& j : jobs) {
    const double n = j.A.rows;
    for (double k = 0; k < n; ++k) fl += (n - k - 1) + 2.0 * (n - k - 1) * (n - k - 1);
  }
  c.add_flops(fl);
  Slab k1;
  auto* dj = upload(c, jobs, k1);
  c.lu_names[c.lu_tag + 1] = names;
  double by = 0;
  int max_n = 1;
  for (auto& j : jobs) {
    by += 16.0 * j.A.rows * double(j.A.cols);
    max_n = std::max(max_n, j.A.rows);
  }
  auto ev = c.prof_begin();
  launch_lu(dj, int(jobs.size()), max_n, c.err, ++c.lu_tag, c.stream);
  c.prof_end("lu", ev, fl, by);
  c.launches++;
  cuda_check(cudaGetLastError(), "lu launch");
  // A singular pivot surfaces at the next sync (check_err maps its tag to
  // this batch's names).
}

// Blocked left solve (forward/backward substitution with GEMM updates between
// 32-row diagonal blocks) for wide right-hand sides.
static void run_trsm_chunks(Ctx& c, const std::vector<SolveJob>& bj);
static void run_blocked_gemm(Ctx& c, const std::vector<SolveJob>& bj);

static void run_blocked(Ctx& c, const std::vector<SolveJob>& bj) {
  if (bj.empty()) return;
  // Default: GEMM (DMMA) updates between 32-row diagonal blocks. H2G_TRSM_FUSED=1
  // selects the single-launch shared-memory kernel (trsm_chunk_kernel): bitwise
  // identical, measured no faster on the bench (332 ms vs ~330 ms for the GEMM path),
  // kept for further work. It keeps a 32-column chunk of X in shared memory: m <= 800.
  static const bool gemm_updates = getenv("H2G_TRSM_FUSED") == nullptr;
  std::vector<SolveJob> big;
  if (!gemm_updates) {
    std::vector<SolveJob> small;
    for (auto& s : bj) (s.lu.rows <= 800 ? small : big).push_back(s);
    run_trsm_chunks(c, small);
    if (big.empty()) return;
  }
  const std::vector<SolveJob>& rest = gemm_updates ? bj : big;
  run_blocked_gemm(c, rest);
}

static void run_trsm_chunks(Ctx& c, const std::vector<SolveJob>& bj) {
  if (bj.empty()) return;
  {
    std::vector<int2> tiles;
    int max_m = 1;
    double fl = 0, by = 0;
    const int w = trsm_chunk_cols();
    for (size_t t = 0; t < bj.size(); ++t) {
      const SolveJob& s = bj[t];
      for (int g = 0; g * w < s.X.cols; ++g) tiles.push_back(make_int2(int(t), g));
      max_m = std::max(max_m, s.lu.rows);
      const double mm = s.lu.rows;
      fl += (s.kind == SOLVE_FULL ? 2.0 : 1.0) * mm * mm * s.X.cols;
      by += 8.0 * mm * mm + 16.0 * s.X.rows * double(s.X.cols);
    }
    c.add_flops(fl);
    Slab k1, k2;
    auto* dj = upload(c, bj, k1);
    auto* dt = upload(c, tiles, k2);
    auto ev = c.prof_begin();
    launch_trsm_chunk(dj, dt, int(tiles.size()), max_m, c.stream);
    c.prof_end(c.prof_detail ? ("trsm@" + c.phase).c_str() : "trsm", ev, fl, by);
    c.launches++;
    cuda_check(cudaGetLastError(), "trsm chunk");
  }
}

static void run_blocked_gemm(Ctx& c, const std::vector<SolveJob>& bj) {
  if (bj.empty()) return;
  constexpr int NB = 32;
  // X <- P X for the permuted kinds.
  {
    std::vector<std::pair<int, int>> shapes;
    std::vector<size_t> idx;
    for (size_t t = 0; t < bj.size(); ++t)
      if (bj[t].kind == SOLVE_FULL || bj[t].kind == SOLVE_LOWER) {
        shapes.push_back({bj[t].X.rows, bj[t].X.cols});
        idx.push_back(t);
      }
    if (!idx.empty()) {
      auto tmp = alloc_mats(c, shapes);
      CopyBatch cb;
      std::vector<GatherJob> gj;
      std::vector<int2> tiles;
      for (size_t u = 0; u < idx.size(); ++u) {
        const SolveJob& s = bj[idx[u]];
        cb.copy(tmp[u].m, s.X);
        gj.push_back({s.X, tmp[u].m, s.perm});
        const int64_t tot = int64_t(s.X.rows) * s.X.cols;
        for (int64_t e = 0; e < tot; e += 4096) tiles.push_back(make_int2(int(gj.size() - 1), int(e / 4096)));
      }
      cb.run(c);
      Slab k1, k2;
      auto* dg = upload(c, gj, k1);
      auto* dt = upload(c, tiles, k2);
      launch_gather_rows(dg, dt, int(tiles.size()), c.stream);
      c.launches++;
      cuda_check(cudaGetLastError(), "gather rows");
    }
  }
  int maxm = 0;
  for (auto& s : bj) maxm = std::max(maxm, s.lu.rows);
  const int nblk = (maxm + NB - 1) / NB;
  auto block_step = [&](const std::vector<SolveJob>& js, int b, bool lower) {
    if (js.empty()) return;
    std::vector<TrsmBlockJob> tj;
    std::vector<int2> tiles;
    GemmBatch gb;
    for (const SolveJob& s : js) {
      const int m = s.lu.rows;
      const int kb = b * NB;
      if (kb >= m) continue;
      const int nb = std::min(NB, m - kb);
      tj.push_back({s.lu, s.X, kb, nb, lower ? 1 : 0});
      for (int g = 0; g < (s.X.cols + 127) / 128; ++g) tiles.push_back(make_int2(int(tj.size() - 1), g));
    }
    Slab k1, k2;
    auto* dj = upload(c, tj, k1);
    auto* dt = upload(c, tiles, k2);
    launch_trsm_block(dj, dt, int(tiles.size()), c.stream);
    c.launches++;
    cuda_check(cudaGetLastError(), "trsm block");
    for (const SolveJob& s : js) {
      const int m = s.lu.rows;
      const int kb = b * NB;
      if (kb >= m) continue;
      const int nb = std::min(NB, m - kb);
      const Mat& L = s.lu;
      const Mat& X = s.X;
      if (lower) {
        if (kb + nb >= m) continue;
        // rows below: x[i] -= sum_k L(i,k) x[k], k ascending
        gb.job(X.sub(kb + nb, 0, m - kb - nb, X.cols), true);
        gb.seg(L.sub(kb + nb, kb, m - kb - nb, nb), X.sub(kb, 0, nb, X.cols), -1.0);
      } else {
        if (kb == 0) continue;
        // rows above: k descending -> reversed column / row views
        const Mat Arev{&L.at(0, kb + nb - 1), kb, nb, L.rs, -L.cs};
        const Mat Brev{&X.at(kb + nb - 1, 0), nb, X.cols, -X.rs, X.cs};
        gb.job(X.sub(0, 0, kb, X.cols), true);
        gb.seg(Arev, Brev, -1.0);
      }
    }
    gb.run(c);
  };
  // Forward sweep for FULL/LOWER, backward sweep for FULL/UPPER.
  std::vector<SolveJob> fwd, bwd;
  for (auto& s : bj) {
    if (s.kind != SOLVE_UPPER) fwd.push_back(s);
    if (s.kind != SOLVE_LOWER) bwd.push_back(s);
  }
  for (int b = 0; b < nblk; ++b) block_step(fwd, b, true);
  for (int b = nblk - 1; b >= 0; --b) block_step(bwd, b, false);
}

// Tolerance-parity mode (qr_mode = 2): wide A^-1 X / A^-T X applications as
// DMMA GEMMs with the explicit inverse. Each distinct factor's inverse is
// formed once (exact blocked solve of the identity); X is then overwritten
// with Inv X (or Inv^T X) through a temporary, in memory-bounded groups.
static void run_inverse(Ctx& c, const std::vector<SolveJob>& ij, size_t budget) {
  std::map<const double*, size_t> idx;
  std::vector<SolveJob> inv;  // identity right-hand sides, solved in place
  std::vector<int> ns;
  for (auto& s : ij)
    if (idx.emplace(s.lu.p, ns.size()).second) ns.push_back(s.lu.rows);
  std::vector<std::pair<int, int>> shapes;
  for (int n : ns) shapes.push_back({n, n});
  std::vector<DMat> invm = alloc_mats(c, shapes);
  {
    CopyBatch id;
    for (auto& im : invm) id.ident(im.m);
    id.run(c);
    std::vector<SolveJob> sj(ns.size());
    for (auto& s : ij) {
      const size_t k = idx[s.lu.p];
      sj[k] = SolveJob{s.lu, s.perm, invm[k].m, SOLVE_FULL};
    }
    run_blocked(c, sj);
  }
  size_t t0 = 0;
  while (t0 < ij.size()) {
    size_t t1 = t0, bytes = 0;
    std::vector<std::pair<int, int>> ts;
    while (t1 < ij.size()) {
      const size_t need = sizeof(double) * size_t(ij[t1].X.rows) * ij[t1].X.cols + 32;
      if (t1 > t0 && bytes + need > budget) break;
      bytes += need;
      ts.push_back({ij[t1].X.rows, ij[t1].X.cols});
      ++t1;
    }
    std::vector<DMat> tmp = alloc_mats(c, ts);
    GemmBatch gb;
    CopyBatch cb;
    for (size_t t = t0; t < t1; ++t) {
      const SolveJob& s = ij[t];
      const Mat A = invm[idx[s.lu.p]].m;
      gemm1(gb, tmp[t - t0].m, s.kind == SOLVE_TRANSPOSE ? A.t() : A, s.X);
      cb.copy(s.X, tmp[t - t0].m);
    }
    gb.run(c);
    cb.run(c);
    t0 = t1;
  }
}

void SolveBatch::run(Ctx& c) {
  HostTimer ht("solve");
  if (jobs.empty()) return;
  if (c.fast_solve) {
    std::vector<SolveJob> ij, rest;
    for (auto& s : jobs)
      ((s.kind == SOLVE_FULL || s.kind == SOLVE_TRANSPOSE) && s.X.cols >= 48 && s.lu.rows >= 64 ? ij : rest)
          .push_back(s);
    if (!ij.empty()) {
      run_inverse(c, ij, size_t(2) << 30);
      jobs = rest;
      if (jobs.empty()) return;
    }
  }
  {
    // Wide left solves go through the blocked path (GEMM updates).
    std::vector<SolveJob> blocked, rest;
    for (auto& s : jobs) {
      const bool left = s.kind == SOLVE_FULL || s.kind == SOLVE_LOWER || s.kind == SOLVE_UPPER;
      if (left && s.X.cols >= 48 && s.lu.rows >= 64) blocked.push_back(s);
      else rest.push_back(s);
    }
    if (!blocked.empty()) {
      run_blocked(c, blocked);  // flops counted by its GEMM + block launches
      jobs = rest;
      if (jobs.empty()) return;
    }
  }
  std::vector<SolveChunk> chunks;
  size_t smem = 1;
  double fl = 0;
  for (size_t j = 0; j < jobs.size(); ++j) {
    const SolveJob& s = jobs[j];
    const int m = s.lu.rows;
    const bool right = s.kind >= SOLVE_RIGHT;
    const int total = right ? s.X.rows : s.X.cols;
    const int w = solve_chunk_width(m);
    for (int c0 = 0; c0 < total; c0 += w) chunks.push_back({int(j), c0, std::min(w, total - c0)});
    smem = std::max(smem, size_t(m) * size_t(std::min(w, total)));
    const double full = (s.kind == SOLVE_FULL || s.kind == SOLVE_TRANSPOSE || s.kind == SOLVE_RIGHT) ? 2.0 : 1.0;
    fl += full * double(m) * m * total;
  }
  c.add_flops(fl);
  Slab k1, k2;
  auto* dj = upload(c, jobs, k1);
  auto* dc = upload(c, chunks, k2);
  double by = 0;
  for (auto& s : jobs) by += 8.0 * s.lu.rows * double(s.lu.rows) + 16.0 * s.X.rows * double(s.X.cols);
  auto ev = c.prof_begin();
  launch_solve(dj, dc, int(chunks.size()), smem, c.stream);
  static const char* kinds[] = {"full", "lower", "upper", "trans", "right", "upper_right"};
  c.prof_end(c.prof_detail ? ("solve@" + c.phase + ":" + kinds[jobs[0].kind]).c_str() : "solve", ev, fl, by);
  c.launches++;
  cuda_check(cudaGetLastError(), "solve launch");
}

// Compressed QR mode (qr_mode = 2): every member at least kPcholMinWidth wide
// is replaced by the columns of a pivoted Cholesky factor of its Gram matrix
// (k_pchol.cu), so the pivoted QR sees the same range and the same member
// masses (up to a dropped trace <= eta) on a panel whose width is the sum of
// the members' numerical ranks instead of O(N). G = M M^T runs as one batched
// GEMM (DMMA) reading each member once.
static constexpr int kPcholMinWidth = 48;

static void compress_members(Ctx& c, std::vector<QrBatch::Item>& items, size_t mem_budget) {
  struct Wide {
    size_t item;
    int mem, w, kmax;
  };
  std::vector<Wide> wide;
  for (size_t t = 0; t < items.size(); ++t) {
    const auto& it = items[t];
    if (it.m == 0 || it.n == 0) continue;
    for (size_t s = size_t(it.fixed); s + 1 < it.offs.size(); ++s) {
      const int w = int(it.offs[s + 1] - it.offs[s]);
      if (w >= kPcholMinWidth) wide.push_back({t, int(s), w, std::min(it.m, w)});
    }
  }
  auto view_of = [](const QrBatch::Item& it, size_t s) {
    return s < it.views.size() && it.views[s].p ? it.views[s] : Mat{};
  };
  std::vector<char> has_view(items.size(), 0);
  bool any_view = false;
  for (size_t t = 0; t < items.size(); ++t)
    for (auto& v : items[t].views)
      if (v.p) has_view[t] = 1, any_view = true;
  if (wide.empty() && !any_view) return;
  std::vector<std::vector<DMat>> comp(items.size());  // per item, per member (wide only)
  for (size_t t = 0; t < items.size(); ++t) comp[t].resize(items[t].offs.size() > 0 ? items[t].offs.size() - 1 : 0);
  size_t g0 = 0;
  while (g0 < wide.size()) {
    size_t g1 = g0, bytes = 0;
    while (g1 < wide.size()) {
      const int m = items[wide[g1].item].m;
      const size_t need = sizeof(double) * size_t(m) * (m + wide[g1].kmax) + 64;
      if (g1 > g0 && bytes + need > mem_budget / 2) break;
      bytes += need;
      ++g1;
    }
    std::vector<std::pair<int, int>> shapes;
    for (size_t g = g0; g < g1; ++g) {
      const int m = items[wide[g].item].m;
      shapes.push_back({m, m});
      shapes.push_back({m, wide[g].kmax});
    }
    std::vector<DMat> gr = alloc_mats(c, shapes);
    Slab kc = c.alloc(sizeof(int) * (g1 - g0));
    int* dcount = static_cast<int*>(kc.get());
    GemmBatch gb;
    gb.name = "gram";
    std::vector<PcholJob> pj;
    int max_m = 1, max_k = 1;
    for (size_t g = g0; g < g1; ++g) {
      const auto& it = items[wide[g].item];
      const Mat vw = view_of(it, size_t(wide[g].mem));
      const Mat A = vw.p ? vw : it.concat.m.sub(0, int(it.offs[wide[g].mem]), it.m, wide[g].w);
      const DMat& G = gr[2 * (g - g0)];
      const DMat& R = gr[2 * (g - g0) + 1];
      gemm1(gb, G.m, A, A.t());
      gb.lower.back() = 1;  // pchol reads the lower triangle only
      const double mt = it.tol * 0.5;  // member_tol (compression.hpp:67)
      const double eta = std::max(64.0 * 2.220446049250313e-16, 0.01 * mt * mt);
      pj.push_back({G.m.p, G.m.cs, R.m.p, R.m.cs, it.m, wide[g].kmax, eta, dcount + (g - g0)});
      max_m = std::max(max_m, it.m);
      max_k = std::max(max_k, wide[g].kmax);
    }
    gb.run(c);
    Slab kj;
    auto* dj = upload(c, pj, kj);
    auto ev = c.prof_begin();
    launch_pchol(dj, int(pj.size()), max_m, max_k, c.stream);
    c.prof_end("pchol", ev, 0.0, 0.0);  // flops/bytes filled in once the counts are back
    const size_t prof_at = c.prec.size();
    c.launches++;
    cuda_check(cudaGetLastError(), "pchol launch");
    std::vector<int> cnt(g1 - g0);
    cuda_check(cudaMemcpyAsync(cnt.data(), dcount, sizeof(int) * cnt.size(), cudaMemcpyDeviceToHost, c.stream),
               "pchol counts");
    c.sync();
    double fl = 0, by = 0;
    std::vector<std::pair<int, int>> cs;
    for (size_t g = g0; g < g1; ++g) {
      const int m = items[wide[g].item].m, k = cnt[g - g0];
      fl += double(m) * k * k;  // left-looking updates: m * k^2 / 2 FMAs
      // lower triangle of G read once, k columns of the factor written
      by += 8.0 * (0.5 * double(m) * (m + 1) + double(m) * std::max(k, 0));
      cs.push_back({m, std::max(k, 0)});
    }
    c.add_flops(fl);
    if (prof_at > 0 && prof_at == c.prec.size() && c.prec.back().name.rfind("pchol", 0) == 0) {
      c.prec.back().flops = fl;
      c.prec.back().bytes = by;
    }
    std::vector<DMat> cm = alloc_mats(c, cs);
    CopyBatch cb;
    for (size_t g = g0; g < g1; ++g) {
      const int k = cnt[g - g0];
      if (k > 0) cb.copy(cm[g - g0].m, gr[2 * (g - g0) + 1].m.sub(0, 0, items[wide[g].item].m, k));
      comp[wide[g].item][wide[g].mem] = cm[g - g0];
    }
    cb.run(c);
    g0 = g1;
  }
  // Re-pack every item that had a wide member: narrow members verbatim,
  // wide ones as their compressed columns; offsets follow.
  CopyBatch cb;
  std::vector<DMat> old;  // source concats stay alive until the copies are enqueued
  std::vector<size_t> touched;
  {
    std::vector<char> mark(items.size(), 0);
    for (const auto& w : wide) mark[w.item] = 1;
    for (size_t t = 0; t < items.size(); ++t)
      if (mark[t] || has_view[t]) touched.push_back(t);  // a view member must be packed into the panel
  }
  for (size_t t : touched) {
    auto& it = items[t];
    std::vector<int64_t> offs{0};
    for (size_t s = 0; s + 1 < it.offs.size(); ++s) {
      const int w = int(it.offs[s + 1] - it.offs[s]);
      const int nw = comp[t][s].owner ? comp[t][s].cols() : w;
      offs.push_back(offs.back() + nw);
    }
    const int n2 = int(offs.back());
    const int ld = std::max(2, (it.m + 1) & ~1);
    DMat nc = alloc_mat(c, ld, std::max(n2, 1));
    nc.m = Mat{nc.m.p, it.m, n2, 1, ld};
    for (size_t s = 0; s + 1 < it.offs.size(); ++s) {
      const int w2 = int(offs[s + 1] - offs[s]);
      if (w2 == 0) continue;
      const Mat dst = nc.m.sub(0, int(offs[s]), it.m, w2);
      if (comp[t][s].owner)
        cb.copy(dst, comp[t][s].m);
      else if (view_of(it, s).p)
        cb.copy(dst, view_of(it, s));
      else
        cb.copy(dst, it.concat.m.sub(0, int(it.offs[s]), it.m, w2));
    }
    old.push_back(std::move(it.concat));
    it.concat = nc;
    it.n = n2;
    it.offs = std::move(offs);
    it.views.clear();
    it.inplace = true;
  }
  cb.run(c);
  old.clear();  // stream-ordered frees behind the copies
}

void QrBatch::compress(Ctx& c, size_t mem_budget) {
  if (c.qr_compress && !compressed) compress_members(c, items, mem_budget);
  compressed = true;
}

static int median_n(const std::vector<QrJob>& js) {
  std::vector<int> ns;
  for (auto& j : js) ns.push_back(j.n);
  if (ns.empty()) return 1;
  std::nth_element(ns.begin(), ns.begin() + ns.size() / 2, ns.end());
  return ns[ns.size() / 2];
}

void QrBatch::run(Ctx& c, std::vector<DMat>& Q, std::vector<int>& rank, size_t mem_budget) {
  if (c.qr_compress && !compressed) compress_members(c, items, mem_budget);
  const size_t n_items = items.size();
  int max_rows = 0;
  for (auto& it : items) max_rows = std::max(max_rows, it.m);
  // Blocked mode when asked for and every basis fits its register-resident Q formation.
  const bool blocked = c.qr_blocked && max_rows <= qrb_max_rows();
  auto scratch_doubles = [&](int m, int n, int nmem) {
    return blocked ? qrb_scratch_doubles(m, n, nmem) : qr_scratch_doubles(m, n, nmem);
  };
  Q.assign(n_items, DMat{});
  rank.assign(n_items, 0);
  if (n_items == 0) return;
  std::vector<std::pair<int, int>> qs;
  for (auto& it : items) qs.push_back({it.m, it.m});
  std::vector<DMat> qm = alloc_mats(c, qs);
  for (size_t t = 0; t < n_items; ++t) {
    // Q is produced row-major: view element (i, j) at p[i*m + j].
    Q[t] = qm[t];
    Q[t].m = Mat{qm[t].m.p, items[t].m, items[t].m, items[t].m > 0 ? items[t].m : 1, 1};
  }
  Slab rk = c.alloc(sizeof(int) * n_items);
  cuda_check(cudaMemsetAsync(rk.get(), 0, sizeof(int) * n_items, c.stream), "rank memset");
  CopyBatch idents;
  struct QrRec { size_t rec, t0, t1; };
  std::vector<QrRec> qr_recs;
  size_t t0 = 0;
  while (t0 < n_items) {
    // Chunk so the working copies + scratch stay under the budget.
    size_t bytes = 0, t1 = t0;
    while (t1 < n_items) {  // (+32 B per item: 16-byte alignment padding)
      const auto& it = items[t1];
      const size_t need = sizeof(double) * ((it.inplace ? 0 : size_t((it.m + 1) & ~1) * it.n) +
                                            scratch_doubles(it.m, it.n, int(it.offs.size()) - 1)) +
                          sizeof(int64_t) * it.offs.size() + 1024 + 32;
      if (t1 > t0 && bytes + need > mem_budget) break;
      bytes += need;
      ++t1;
    }
    Slab work = c.alloc(bytes);
    std::vector<QrJob> jobs;
    std::vector<int64_t> offs_all;
    std::vector<size_t> offs_at;
    for (size_t t = t0; t < t1; ++t) {
      offs_at.push_back(offs_all.size());
      offs_all.insert(offs_all.end(), items[t].offs.begin(), items[t].offs.end());
    }
    Slab ko;
    int64_t* doffs = upload(c, offs_all, ko);
    char* at = static_cast<char*>(work.get());
    int max_m = 1, max_nmem = 1, min_n = 1 << 30;
    double fl = 0;
    for (size_t t = t0; t < t1; ++t) {
      const auto& it = items[t];
      if (it.n == 0 || it.m == 0) {
        if (it.m > 0) idents.ident(Q[t].m);
        continue;
      }
      QrJob j;
      j.A = it.concat.m;
      j.m = it.m;
      j.n = it.n;
      j.member_off = doffs + offs_at[t - t0];
      j.nmem = int(it.offs.size()) - 1;
      j.tol = it.tol;
      j.member_tol = it.tol * 0.5;  // BasisBuildOptions::member_tol_factor (compression.hpp:67)
      j.cap = it.cap;
      if (it.inplace) {  // column-major concat factored in place
        j.work = it.concat.m.p;
        j.ldw = it.concat.m.cs;
      } else {
        j.work = reinterpret_cast<double*>(at);
        j.ldw = (it.m + 1) & ~1;  // even: 16-byte aligned column segments
        at += sizeof(double) * size_t(j.ldw) * it.n;
        at = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(at) + 15) & ~uintptr_t(15));
      }
      j.scratch = reinterpret_cast<double*>(at);
      at += sizeof(double) * scratch_doubles(it.m, it.n, j.nmem);
      at = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(at) + 15) & ~uintptr_t(15));
      j.Q = Q[t].m.p;
      j.rank_out = static_cast<int*>(rk.get()) + t;
      jobs.push_back(j);
      max_m = std::max(max_m, it.m);
      max_nmem = std::max(max_nmem, j.nmem);
      min_n = std::min(min_n, it.n);
      fl += 2.0 * it.m * double(it.n);  // column norms
    }
    c.add_flops(fl);
    // Launch plan: one cluster size for the batch (qr_cluster_size), the
    // largest bases first so later waves hold the short ones. (Giving spare
    // CTAs of a single wave to the largest bases, as concurrent launches of
    // mixed cluster sizes, was measured slower: mixed clusters pack worse.)
    std::vector<int> G(jobs.size(), 1);
    {
      const char* ecl = getenv("H2G_QR_CLUSTER");
      auto work = [&](const QrJob& j) { return double(j.m) * j.n; };
      std::fill(G.begin(), G.end(),
                ecl ? std::max(1, std::min(8, atoi(ecl)))
                    : blocked ? qrb_cluster_size(int(jobs.size()), median_n(jobs), max_m, max_nmem)
                              : qr_cluster_size(int(jobs.size()), min_n, max_m, max_nmem));
      std::vector<size_t> ord(jobs.size());
      for (size_t q = 0; q < ord.size(); ++q) ord[q] = q;
      std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) {
        return G[x] != G[y] ? G[x] > G[y] : work(jobs[x]) > work(jobs[y]);
      });
      std::vector<QrJob> js(jobs.size());
      std::vector<int> gs(jobs.size());
      for (size_t q = 0; q < ord.size(); ++q) {
        js[q] = jobs[ord[q]];
        gs[q] = G[ord[q]];
      }
      jobs.swap(js);
      G.swap(gs);
    }
    Slab kdbg;
    double* ddbg = nullptr;
    if (getenv("H2G_QR_DEBUG")) {
      kdbg = c.alloc(sizeof(double) * 16 * jobs.size());
      ddbg = static_cast<double*>(kdbg.get());
      cudaMemsetAsync(ddbg, 0, sizeof(double) * 16 * jobs.size(), c.stream);
      for (size_t q = 0; q < jobs.size(); ++q) jobs[q].dbg = ddbg + 16 * q;
    }
    Slab kj;
    auto* dj = upload(c, jobs, kj);
    auto ev = c.prof_begin();
    cudaEvent_t dbg_a = nullptr, dbg_b = nullptr;
    if (ddbg) {
      cudaEventCreate(&dbg_a);
      cudaEventCreate(&dbg_b);
      cudaEventRecord(dbg_a, c.stream);
    }
    const int cl = G.empty() ? 1 : G[0];
    if (blocked)
      launch_qrb(dj, int(jobs.size()), max_m, max_nmem, cl, c.stream);
    else
      launch_qr(dj, int(jobs.size()), max_m, max_nmem, cl, c.stream);
    if (ddbg) {
      cudaEventRecord(dbg_b, c.stream);
      cudaEventSynchronize(dbg_b);
      float ms = 0;
      cudaEventElapsedTime(&ms, dbg_a, dbg_b);
      cudaEventDestroy(dbg_a);
      cudaEventDestroy(dbg_b);
      int gh[10] = {0};
      for (int g : G) ++gh[g];
      fprintf(stderr, "QRDBG launch %.1f ms, clusters by size:", ms);
      for (int g = 1; g <= 8; ++g)
        if (gh[g]) fprintf(stderr, " %dx%d", gh[g], g);
      fprintf(stderr, "\n");
      std::vector<double> h(16 * jobs.size());
      cudaMemcpyAsync(h.data(), ddbg, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.stream);
      cudaStreamSynchronize(c.stream);
      double a[14] = {0};
      for (size_t q = 0; q < jobs.size(); ++q)
        for (int u = 0; u < 14; ++u) a[u] += h[16 * q + u];
      if (blocked)
        fprintf(stderr, "QRDBG blocked jobs=%zu avg cycles: pivot %.3g lead %.3g pass %.3g masses %.3g update %.3g rank %.1f n %.0f\n",
                jobs.size(), a[0] / jobs.size(), a[1] / jobs.size(), a[2] / jobs.size(), a[3] / jobs.size(),
                a[8] / jobs.size(), a[4] / jobs.size(), a[5] / jobs.size());
      fprintf(stderr, "QRDBG jobs=%zu avg: piv %.3g refl %.3g tile %.3g mem %.3g rank %.1f n %.0f formq %.3g (cycles)\n",
              jobs.size(), a[0] / jobs.size(), a[1] / jobs.size(), a[2] / jobs.size(), a[3] / jobs.size(),
              a[4] / jobs.size(), a[5] / jobs.size(), a[6] / jobs.size());
      {
        double mx = 0, sum = 0, wmx = 0, wsum = 0;
        size_t qm = 0;
        for (size_t q = 0; q < jobs.size(); ++q) {
          const double tot = h[16 * q] + h[16 * q + 1] + h[16 * q + 2] + h[16 * q + 3] + h[16 * q + 6];
          sum += tot;
          if (tot > mx) { mx = tot; qm = q; }
          const double w = double(jobs[q].m) * jobs[q].n;
          wsum += w;
          wmx = std::max(wmx, w);
        }
        fprintf(stderr, "QRDBG   G=%d job cycles max %.3g mean %.3g (max job m=%d n=%d rank %.0f); m*n max/mean %.2f\n",
                cl, mx, sum / jobs.size(), jobs[qm].m, jobs[qm].n, h[16 * qm + 4], wmx / (wsum / jobs.size()));
      }
      fprintf(stderr, "QRDBG   warp0 per tile: wait %.0f chain %.0f store %.0f tiles %.0f; lane0 norm recomputes %.4f of chains\n",
              a[8] / a[11], a[9] / a[11], a[10] / a[11], a[11] / jobs.size(), a[12] / (a[13] > 0 ? a[13] : 1));
    }
    c.prof_end("qr", ev, 0.0, 0.0);
    qr_recs.push_back({c.prof ? c.prec.size() - 1 : size_t(-1), t0, t1});
    c.launches++;
    cuda_check(cudaGetLastError(), "qr launch");
    t0 = t1;
  }
  idents.run(c);
  cuda_check(cudaMemcpyAsync(rank.data(), rk.get(), sizeof(int) * n_items, cudaMemcpyDeviceToHost,
                             c.stream),
             "rank d2h");
  c.sync();
  // Reference flop rules for the executed steps (linalg.cpp:148, :176); the
  // algorithmic bytes: exact mode reads and writes the trailing panel every
  // step, blocked mode reads it every step and rewrites it once per block;
  // Q formation reads/writes its active rows.
  double fl = 0;
  std::vector<double> fl_item(n_items, 0.0), by_item(n_items, 0.0);
  for (size_t t = 0; t < n_items; ++t) {
    const double m = items[t].m, n = items[t].n;
    for (int k = 0; k < rank[t]; ++k) {
      const double f = 4.0 * (m - k) + 4.0 * (m - k) * (n - k - 1) + 4.0 * (m - k) * m;
      fl += f;
      fl_item[t] += f;
      if (!blocked) {
        by_item[t] += 16.0 * (m - k) * (n - k) + 16.0 * (m - k) * m;
      } else {
        // one read of the trailing panel per step; one read+write per block of
        // 32 reflectors (k = 32 b: the update of the previous block's rows).
        by_item[t] += 8.0 * (m - k) * (n - k) + 8.0 * (m - k) * m;  // + Q formation reads V
        if (k > 0 && k % 32 == 0) by_item[t] += 16.0 * (m - k + 32) * (n - k);
      }
    }
    by_item[t] += 8.0 * m * n;  // initial column norms
  }
  c.add_flops(fl);
  if (c.prof)
    for (auto& r : qr_recs) {
      if (r.rec == size_t(-1) || r.rec >= c.prec.size()) continue;
      for (size_t t = r.t0; t < r.t1; ++t) {
        c.prec[r.rec].flops += fl_item[t];
        c.prec[r.rec].bytes += by_item[t];
      }
    }
}

}  // namespace h2g
