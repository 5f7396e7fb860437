// fs_host.cu -- evaluate_field from host memory to host memory, pipelined.
//
// The reference's evaluate_field (estimators.py:260-323) takes host arrays and
// returns host arrays.  On the device the cost of that contract is the PCIe
// traffic (24 B in, up to 41 B out per query), so the query set is split into
// slabs and three streams overlap slab k's evaluation with slab k+1's
// host->device copy and slab k-1's device->host copies.  The RNG streams of the
// stochastic estimator are keyed on global query indices (query_offset + slab
// start, _core.py:219, 258), so the result is identical to one whole launch.
#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/fastsum_b200.h"
#include "fs_eval.h"
#include "fs_internal.h"

struct fsb_tree {
  fsb::FsTree* t;
};

namespace fsb {

int query_order(const double* q, int64_t n, int32_t* perm, cudaStream_t s);

namespace {

// Streams and events of the host pipeline, created once per (thread, device)
// and reused: creating them per call costs more than a small evaluation.
struct Streams {
  cudaStream_t h2d = nullptr, d2h = nullptr, c2 = nullptr;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  int init() {
    if (h2d) return 0;
    FS_CK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    FS_CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    FS_CK(cudaStreamCreateWithFlags(&c2, cudaStreamNonBlocking));
    return 0;
  }
  int event(cudaEvent_t* out) {
    if (used == ev.size()) {
      cudaEvent_t e;
      FS_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    *out = ev[used++];
    return 0;
  }
  // page-locked staging of pageable query arrays (grown, kept)
  double* qstage = nullptr;
  size_t qstage_bytes = 0;
  int query_staging(size_t bytes) {
    if (bytes <= qstage_bytes) return 0;
    if (qstage) FS_CK(cudaFreeHost(qstage));
    qstage = nullptr;
    qstage_bytes = 0;
    FS_CK(cudaHostAlloc(reinterpret_cast<void**>(&qstage), bytes, cudaHostAllocDefault));
    qstage_bytes = bytes;
    return 0;
  }
};

Streams& streams_for_device() {
  static thread_local Streams per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Streams& st = per_dev[dev & 63];
  st.used = 0;
  return st;
}

#ifndef FSB_STAGE_PAGEABLE
#define FSB_STAGE_PAGEABLE 1  // pageable queries: staged by the worker threads
#endif

// Host-side work of the pipeline (raw = values copies, constant columns) on a
// few persistent worker threads, so it overlaps the PCIe transfers of later
// slabs: host memory moves ~40 GB/s with four threads, one thread ~16 GB/s.
class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { run(); });
  }
  int size() const { return (int)th_.size(); }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(f));
    }
    cv_.notify_one();
  }

 private:
  void run() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return !q_.empty(); });
        f = std::move(q_.front());
        q_.pop_front();
      }
      f();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
};

HostPool& host_pool() {  // never destroyed: workers outlive static destruction
  static HostPool* p = new HostPool(
      (int)std::max(1u, std::min(4u, std::thread::hardware_concurrency() / 4)));
  return *p;
}

// one call's outstanding host jobs
struct Latch {
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  void add(int k) {
    std::lock_guard<std::mutex> lk(mu);
    count += k;
  }
  void done() {
    std::lock_guard<std::mutex> lk(mu);
    if (--count == 0) cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return count == 0; });
  }
};
// waits for the latches on every exit path (jobs capture the caller's frame)
struct LatchGuard {
  Latch* l;
  size_t count;
  ~LatchGuard() {
    for (size_t i = 0; i < count; ++i) l[i].wait();
  }
};

// true when p is ordinary pageable host memory (not page-locked / registered)
bool pageable(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // (older drivers: unregistered pointers are an error)
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

// fn(b, e) over [0, n) in one part per worker (one part below 64 K elements)
template <class F>
void parallel_parts(Latch& latch, int64_t n, F fn) {
  if (n <= 0) return;
  HostPool& pool = host_pool();
  const int parts = n < (1 << 16) ? 1 : pool.size();
  latch.add(parts);
  for (int i = 0; i < parts; ++i) {
    const int64_t b = n * i / parts, e = n * (i + 1) / parts;
    pool.submit([&latch, fn, b, e] {
      fn(b, e);
      latch.done();
    });
  }
}

}  // namespace

static int evaluate_host(FsTree* t, const fsb_eval_args* a, const double* q_host, int64_t n,
                         double* values, double* raw_h, uint8_t* flagged, int64_t* visited,
                         int64_t* path_steps, int64_t* path_count, int chunks, cudaStream_t s) {
  const bool f32 = a->precision == 1;
  const size_t rsz = f32 ? sizeof(float) : sizeof(double);
  // device buffers (stream-ordered pool allocations on the compute stream)
  // the 8-byte result columns are rows of one block with pitch 8 n (values,
  // visited, path_steps, raw), so a slab's columns leave in one 2-D copy when
  // the host columns are equally spaced too (evaluate_field's pinned block)
  Scratch qd, raw, cols, flg, cnt, perm;
  FS_TRY(qd.alloc(sizeof(double) * 3 * (size_t)n, s));
  FS_TRY(raw.alloc(rsz * (size_t)n, s));
  FS_TRY(cols.alloc(sizeof(double) * 4 * (size_t)n, s));
  FS_TRY(flg.alloc((size_t)n, s));
  FS_TRY(cnt.alloc(sizeof(int64_t) * (size_t)n, s));
  double* const val_d = cols.as<double>();
  int64_t* const vis_d = reinterpret_cast<int64_t*>(val_d + n);
  int64_t* const stp_d = reinterpret_cast<int64_t*>(val_d + 2 * n);
  double* const raw64_d = val_d + 3 * n;
  const bool shared = a->method == FSB_METHOD_STOCHASTIC && a->rng_group_log2 > 0;
  if (a->method == FSB_METHOD_BARNES_HUT && a->query_order)
    FS_TRY(perm.alloc(sizeof(int32_t) * (size_t)n, s));

  Streams& st = streams_for_device();
  FS_TRY(st.init());
  cudaEvent_t ready;
  FS_TRY(st.event(&ready));
  FS_CK(cudaEventRecord(ready, s));  // allocations visible to the other streams
  FS_CK(cudaStreamWaitEvent(st.h2d, ready, 0));
  FS_CK(cudaStreamWaitEvent(st.c2, ready, 0));

  // FSB_TRACE=1: per-slab timeline (ms from the first H2D) on stderr
  const bool trace = std::getenv("FSB_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t on) -> int {
    if (!trace) return 0;
    cudaEvent_t e;
    FS_CK(cudaEventCreate(&e));
    FS_CK(cudaEventRecord(e, on));
    tev.push_back(e);
    return 0;
  };
  // slab boundaries: the first and last slabs are half-size, since the first
  // H2D and the last D2H copies cannot overlap any evaluation
  chunks = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, n));
  // warp-voting BH: the groups come from the whole set's Morton order (one slab)
  if (a->method == FSB_METHOD_BARNES_HUT && a->bh_warp_vote) chunks = 1;
  std::vector<int64_t> cut(chunks + 1, 0);
  for (int k = 1; k < chunks; ++k) {
    cut[k] = (int64_t)((double)n * (k - 0.5) / (chunks - 1.0));
    // warp-shared streams: slabs start on shuffle windows (order is window-local)
    if (shared) cut[k] = std::min(n, (cut[k] + kShuffleWindow / 2) / kShuffleWindow * kShuffleWindow);
  }
  cut[chunks] = n;
  const bool counters = a->method == FSB_METHOD_STOCHASTIC;
  // Constant columns need no PCIe transfer: they are written on the host while
  // the pipeline runs -- path_count (n_samples x internal subdomains for the
  // stochastic method, _core.py:215-267, else 0), path_steps (0 unless
  // stochastic), flagged (false unless smooth_exp, kernels.py:110-122) and, for
  // brute force, visited (the source count); and raw, which equals values
  // bit for bit unless smooth_exp, is copied from values on the host as each
  // slab arrives: 41 -> 24 bytes per query cross PCIe for the stochastic method.
  // (Narrowing visited / path_steps to int32 for the copy and widening them on
  // the host measured slower: 0.96 vs 0.94 ms on C4.)
  const bool smooth = a->smooth != 0;
  const bool raw_dev = raw_h && smooth;  // raw crosses PCIe (smooth_exp only)
  int64_t count_value = 0;
  if (counters && t) {
    int ni = 0;
    FS_TRY(internal_level1(t, s, &ni));
    count_value = (int64_t)a->n_samples * ni;
  }
  // the device->host 8-byte columns of a slab: values, visited (not brute
  // force: host-filled) and path_steps (stochastic only); `rows` > 1 when the
  // caller's columns are equally spaced (pitch hpitch), so one 2-D copy moves them
  const bool vis_dev = visited && a->method != FSB_METHOD_BRUTE_FORCE;
  const bool stp_dev = path_steps && counters;
  int rows = 0;
  ptrdiff_t hpitch = 0;
  if (vis_dev) {
    hpitch = reinterpret_cast<const char*>(visited) - reinterpret_cast<const char*>(values);
    if (hpitch >= (ptrdiff_t)(sizeof(double) * n)) {  // rows do not overlap
      rows = 2;
      if (stp_dev)
        rows = reinterpret_cast<const char*>(path_steps) ==
                       reinterpret_cast<const char*>(values) + 2 * hpitch
                   ? 3
                   : 0;
    }
  }
  // host work on the worker threads: a pageable query array copied slab by
  // slab into page-locked staging (first: the copies wait on it; the driver's
  // own staging of pageable copies is single-threaded and synchronous), the
  // constant columns, raw as slabs land
  std::unique_ptr<Latch[]> latches(new Latch[chunks + 1]);
  LatchGuard latch_guard{latches.get(), (size_t)chunks + 1};
  Latch& latch = latches[chunks];
  const double* q_src = q_host;
  if (FSB_STAGE_PAGEABLE && pageable(q_host)) {
    FS_TRY(st.query_staging(sizeof(double) * 3 * (size_t)n));
    double* const qs_h = st.qstage;
    q_src = qs_h;
    for (int k = 0; k < chunks; ++k) {
      const int64_t lo = cut[k];
      parallel_parts(latches[k], cut[k + 1] - lo, [=](int64_t b, int64_t e) {
        std::memcpy(qs_h + 3 * (lo + b), q_host + 3 * (lo + b), sizeof(double) * 3 * (size_t)(e - b));
      });
    }
  }
  if (path_count)
    parallel_parts(latch, n, [=](int64_t b, int64_t e) {
      std::fill(path_count + b, path_count + e, count_value);
    });
  if (path_steps && !counters)
    parallel_parts(latch, n, [=](int64_t b, int64_t e) {
      std::fill(path_steps + b, path_steps + e, (int64_t)0);
    });
  if (flagged && !smooth)
    parallel_parts(latch, n, [=](int64_t b, int64_t e) {
      std::memset(flagged + b, 0, (size_t)(e - b));
    });
  if (visited && a->method == FSB_METHOD_BRUTE_FORCE) {
    const int64_t mv = a->m;
    parallel_parts(latch, n, [=](int64_t b, int64_t e) { std::fill(visited + b, visited + e, mv); });
  }
  std::vector<cudaEvent_t> slab_done(chunks, nullptr);
  // Slabs alternate between two compute streams so that one slab's last
  // blocks overlap the next slab's first ones (no launch tail per slab).
  for (int k = 0; k < chunks; ++k) {
    const int64_t lo = cut[k], m = cut[k + 1] - cut[k];
    if (m <= 0) continue;
    const cudaStream_t cs = (k & 1) ? st.c2 : s;
    cudaEvent_t in_done, out_ready;
    FS_TRY(st.event(&in_done));
    FS_TRY(st.event(&out_ready));
    double* qs = qd.as<double>() + 3 * lo;
    FS_TRY(mark(st.h2d));
    latches[k].wait();  // (staged queries: this slab's copy is done)
    FS_CK(cudaMemcpyAsync(qs, q_src + 3 * lo, sizeof(double) * 3 * (size_t)m,
                          cudaMemcpyHostToDevice, st.h2d));
    FS_TRY(mark(st.h2d));
    FS_CK(cudaEventRecord(in_done, st.h2d));
    FS_CK(cudaStreamWaitEvent(cs, in_done, 0));
    FS_TRY(mark(cs));

    void* r = static_cast<char*>(raw.p) + rsz * (size_t)lo;
    int64_t* v = vis_d + lo;
    int64_t* ps = stp_d + lo;
    int64_t* pc = cnt.as<int64_t>() + lo;
    switch (a->method) {
      case FSB_METHOD_BRUTE_FORCE:
        FS_TRY(brute_force(a->kid, a->alpha, a->dfloor, !f32, a->src_pts, a->src_ms, a->m, a->c,
                           qs, m, r, cs));  // (visited = m for every query: filled on the host)
        break;
      case FSB_METHOD_BARNES_HUT: {
        int32_t* pp = nullptr;
        if (a->query_order && m > 1) {
          pp = perm.as<int32_t>() + lo;
          FS_TRY(query_order(qs, m, pp, cs));
        }
        FS_TRY(barnes_hut(t, a->kid, a->alpha, a->dfloor, !f32, qs, m, pp, a->beta, r, v, cs,
                          a->bh_warp_vote != 0));
        break;
      }
      case FSB_METHOD_TELESCOPING:
        FS_TRY(telescoping(t, a->kid, a->alpha, a->dfloor, !f32, qs, m, r, v, cs));
        break;
      default:
        // shared streams: the slab's window-local shuffle, keyed on global positions
        FS_TRY(stochastic(t, a->kid, a->alpha, a->dfloor, !f32, qs, m, nullptr,
                          (int)a->n_samples, a->rr_mode, a->seed, a->query_offset + lo, r, v, ps,
                          pc, cs, shared ? a->rng_group_log2 : 0,
                          (a->path_variant ? kFlagAlg2 : 0) | (shared ? kFlagShuffled : 0)));
    }
    double* vd = val_d + lo;
    double* r64 = raw_dev ? raw64_d + lo : nullptr;
    uint8_t* fd = flg.as<uint8_t>() + lo;
    FS_TRY(post_transform(r, f32 ? 1 : 0, m, a->smooth, a->alpha, vd, r64, fd, cs));
    FS_TRY(mark(cs));
    FS_CK(cudaEventRecord(out_ready, cs));
    FS_CK(cudaStreamWaitEvent(st.d2h, out_ready, 0));
    FS_TRY(mark(st.d2h));
    auto d2h = [&](void* dst, const void* src, size_t bytes) -> int {
      if (dst) FS_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st.d2h));
      return 0;
    };
    if (rows > 1) {  // values, visited[, path_steps]: one 2-D copy
      FS_CK(cudaMemcpy2DAsync(values + lo, (size_t)hpitch, vd, sizeof(double) * (size_t)n,
                              sizeof(double) * (size_t)m, (size_t)rows, cudaMemcpyDeviceToHost,
                              st.d2h));
    } else {
      FS_TRY(d2h(values + lo, vd, sizeof(double) * (size_t)m));
      if (vis_dev) FS_TRY(d2h(visited + lo, v, sizeof(int64_t) * (size_t)m));
      if (stp_dev) FS_TRY(d2h(path_steps + lo, ps, sizeof(int64_t) * (size_t)m));
    }
    if (raw_dev) FS_TRY(d2h(raw_h + lo, r64, sizeof(double) * (size_t)m));
    if (smooth) FS_TRY(d2h(flagged ? flagged + lo : nullptr, fd, (size_t)m));
    FS_TRY(mark(st.d2h));
    FS_TRY(st.event(&slab_done[k]));
    FS_CK(cudaEventRecord(slab_done[k], st.d2h));
  }
  // raw = values (identity post-transform): copied on the worker threads as
  // each slab lands
  if (raw_h && !raw_dev) {
    for (int k = 0; k < chunks; ++k) {
      if (!slab_done[k]) continue;
      FS_CK(cudaEventSynchronize(slab_done[k]));
      const int64_t lo = cut[k];
      parallel_parts(latch, cut[k + 1] - lo, [=](int64_t b, int64_t e) {
        std::memcpy(raw_h + lo + b, values + lo + b, sizeof(double) * (size_t)(e - b));
      });
    }
  }
  latch.wait();
  // device buffers are freed on `s` after the last D2H copy
  cudaEvent_t done;
  FS_TRY(st.event(&done));
  FS_CK(cudaEventRecord(done, st.d2h));
  FS_CK(cudaStreamWaitEvent(s, done, 0));  // (d2h waited on every slab, c2's included)
  FS_CK(cudaStreamSynchronize(st.d2h));
  FS_CK(cudaStreamSynchronize(s));
  if (trace) {
    for (size_t k = 0; k + 6 <= tev.size(); k += 6) {
      float t[6];
      for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[k + i]);
      fprintf(stderr, "slab %zu: h2d %.3f-%.3f  compute %.3f-%.3f  d2h %.3f-%.3f\n", k / 6, t[0],
              t[1], t[2], t[3], t[4], t[5]);
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  FS_CK(cudaGetLastError());
  return 0;
}

}  // namespace fsb

extern "C" int fsb_evaluate_field_host(fsb_tree* tree, const fsb_eval_args* a,
                                       const double* queries, int64_t n, double* values,
                                       double* raw, uint8_t* flagged, int64_t* visited,
                                       int64_t* path_steps, int64_t* path_count, int chunks,
                                       void* stream) {
  FSB_RANGE("fsb_evaluate_field_host");
  using fsb::set_error;
  if (!a || !values || (n > 0 && !queries)) {
    set_error("null argument");
    return 1;
  }
  if (a->kid < 0 || a->kid > 2 || (a->precision != 0 && a->precision != 1) || n < 0) {
    set_error("bad kernel id / precision / query count");
    return 1;
  }
  if (a->method < FSB_METHOD_BRUTE_FORCE || a->method > FSB_METHOD_STOCHASTIC) {
    set_error("unknown method %d", a->method);
    return 1;
  }
  if (a->method == FSB_METHOD_BRUTE_FORCE) {
    if (!a->src_pts || !a->src_ms || a->m < 1 || (a->kid == 1 ? a->c != 3 : a->c < 1)) {
      set_error("brute force needs device sources (m >= 1, channels matching the kernel)");
      return 1;
    }
  } else if (!tree || !tree->t) {
    set_error("null tree");
    return 1;
  }
  if (a->method == FSB_METHOD_BARNES_HUT && !(a->beta > 0)) {
    set_error("beta must be positive");
    return 1;
  }
  if (a->method == FSB_METHOD_STOCHASTIC &&
      (a->n_samples < 1 || a->n_samples > (1LL << 30) || a->rr_mode < 0 || a->rr_mode > 2 ||
       a->rng_group_log2 < 0 || a->rng_group_log2 > 20 || a->path_variant < 0 ||
       a->path_variant > 1)) {
    set_error("bad samples_per_subdomain / rr mode");
    return 1;
  }
  if (n == 0) return 0;
  return fsb::evaluate_host(tree ? tree->t : nullptr, a, queries, n, values, raw, flagged,
                            visited, path_steps, path_count, chunks,
                            reinterpret_cast<cudaStream_t>(stream));
}
