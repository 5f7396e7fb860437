// fs_bh_split.cu -- load-balanced Barnes-Hut for precision="f32".
//
// The warp-coherent BH of fs_eval.cu (one query per lane, the warp walks the
// union of its lanes' preorder sequences) is bound by a few 32-query chunks
// next to the surface: their union walk is ~10^4 nodes long and one warp
// serialises it (measured on C4, beta = 6: the longest chunk takes 13 M cycles
// of a 14 M-cycle kernel; capping chunks at 3000 iterations would finish the
// rest in 2 ms).  Here a warp that has spent more than `split_after` iterations
// on its unit stops descending into large subtrees itself: when lanes open a
// node whose subtree holds >= `min_split` nodes, it emits a work item (chunk,
// [first child, end of subtree), mask of the opening lanes) and skips the
// subtree.  Items are walked by other warps in follow-up launches (and may be
// split again); each unit's per-lane partial sums land in their own slots, and
// k_bh_fold adds a chunk's items in (chunk, subtree start) = preorder order,
// so results are deterministic and independent of scheduling.  The node set
// each query sums is exactly the warp-coherent kernel's (visited counts equal);
// only the association of the FP64 accumulation differs.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fs_common.cuh"
#include "fs_eval.h"
#include "fs_internal.h"

namespace fsb {

struct BhItem {
  int32_t chunk, first, end;
  uint32_t mask;
};

struct BhSplitCtx {
  const float4* __restrict__ rec;  // preorder {cx, cy, cz, diam} {m0, m1, m2, skip}
  const float4* __restrict__ pa;   // permuted points {x, y, z, m0}
  const float4* __restrict__ pb;   // {m1, m2, 0, 0}
  const double* __restrict__ q;
  const int32_t* __restrict__ qperm;
  int64_t n;
  uint32_t nn;
  float beta;
  int split_after, min_split;
  BhItem* items;                   // item queue
  unsigned int* n_items;           // emitted items
  unsigned int* overflow;          // set when the queue was full (caller falls back)
  int cap;
  unsigned int* chunk_items;       // items per chunk
  double* acc_top;                 // per query: the chunk walk's partial sum
  int32_t* seen_top;
  double* acc_item;                // per (item, lane)
  int32_t* seen_item;
};

template <int KID>
__device__ __forceinline__ double bh_node_value(const BhSplitCtx& C, const float4& g,
                                                const float4& mm, float qx, float qy, float qz,
                                                const KParams& kp) {
  if (g.w < 0) {  // multi-point leaf: exact per-point sum (_core.py:59-64)
    double acc = 0.0;
    for (int j = __float_as_int(mm.x); j < __float_as_int(mm.y); ++j) {
      const float4 u = C.pa[j];
      float m1 = 0.f, m2 = 0.f;
      if (KID == KID_WINDING) {
        const float4 v = C.pb[j];
        m1 = v.x;
        m2 = v.y;
      }
      acc += (double)contrib_fast<KID>(u.w, m1, m2, u.x, u.y, u.z, qx, qy, qz, kp);
    }
    return acc;
  }
  return (double)contrib_fast<KID>(mm.x, mm.y, mm.z, g.x, g.y, g.z, qx, qy, qz, kp);
}

// units [u0, u1): top-level chunks (items == false) or queued items (items == true)
template <int KID, bool ITEMS, bool VOTE>
__global__ void __launch_bounds__(128) k_bh_units(BhSplitCtx C, KParams kp, unsigned int u0,
                                                  unsigned int u1, unsigned int* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned int u = 0;
    if (lane == 0) u = atomicAdd(work, 1u);
    u = __shfl_sync(0xffffffffu, u, 0) + u0;
    if (u >= u1) break;
    int32_t chunk;
    uint32_t start, end, mask;
    if (ITEMS) {
      const BhItem it = C.items[u];
      chunk = it.chunk;
      start = (uint32_t)it.first;
      end = (uint32_t)it.end;
      mask = it.mask;
    } else {
      chunk = (int32_t)u;
      start = 0;
      end = C.nn;
      mask = 0xffffffffu;
    }
    const int64_t t = (int64_t)chunk * 32 + lane;
    const bool live = t < C.n && ((mask >> lane) & 1u);
    float qx = 0.f, qy = 0.f, qz = 0.f;
    if (t < C.n) {
      const int64_t qi = C.qperm ? (int64_t)C.qperm[t] : t;
      qx = (float)C.q[3 * qi];
      qy = (float)C.q[3 * qi + 1];
      qz = (float)C.q[3 * qi + 2];
    }
    uint32_t i = live ? start : end;
    double acc = 0.0;
    int seen = 0;
    int iters = 0;
    while (true) {
      const uint32_t cur = warp_min_u32(i);
      if (cur >= end) break;
      ++iters;
      const bool mine = i == cur;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f), mm = g;
      bool opens = false, accept = false;
      uint32_t skip = 0;
      if (mine) {
        g = C.rec[2 * (int64_t)cur];
        mm = C.rec[2 * (int64_t)cur + 1];
        ++seen;
        skip = (uint32_t)__float_as_int(mm.w);
        const bool leaf = skip == cur + 1;
        const float dx = qx - g.x, dy = qy - g.y, dz = qz - g.z;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const float thr = C.beta * fmaxf(g.w, 1e-12f);
        accept = leaf || d2 >= thr * thr;
      }
      // warp voting: open unless every live lane accepts
      if (VOTE) accept = __all_sync(0xffffffffu, !mine || accept);
      if (mine) {
        if (accept) {
          acc += bh_node_value<KID>(C, g, mm, qx, qy, qz, kp);
          i = skip;
        } else {
          opens = true;
          i = cur + 1;
        }
      }
      // a long walk hands large opened subtrees to other warps
      if (iters > C.split_after) {
        const unsigned om = __ballot_sync(0xffffffffu, opens);
        if (om) {
          const int src = __ffs(om) - 1;
          const uint32_t sk = __shfl_sync(0xffffffffu, skip, src);
          if ((int)(sk - cur) >= C.min_split) {
            int ok = 0;
            if (lane == 0) {
              const unsigned int pos = atomicAdd(C.n_items, 1u);
              if ((int)pos < C.cap) {
                C.items[pos] = BhItem{chunk, (int32_t)(cur + 1), (int32_t)sk, om};
                atomicAdd(&C.chunk_items[chunk], 1u);
                ok = 1;
              } else {
                atomicOr(C.overflow, 1u);
              }
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            if (ok && opens) i = sk;  // the item walks [cur + 1, sk) for these lanes
          }
        }
      }
    }
    if (ITEMS) {
      C.acc_item[(int64_t)u * 32 + lane] = acc;
      C.seen_item[(int64_t)u * 32 + lane] = seen;
    } else if (t < C.n) {
      C.acc_top[t] = acc;
      C.seen_top[t] = seen;
    }
  }
}

__global__ void k_bh_item_keys(const BhItem* __restrict__ items, int m,
                               uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  key[k] = ((uint64_t)(uint32_t)items[k].chunk << 32) | (uint32_t)items[k].first;
  idx[k] = k;
}

__global__ void k_bh_fold(const BhSplitCtx C, const int32_t* __restrict__ order,
                          const unsigned int* __restrict__ off, float* __restrict__ out,
                          int64_t* __restrict__ visited) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= C.n) return;
  const int64_t chunk = t >> 5;
  const int lane = (int)(t & 31);
  double acc = C.acc_top[t];
  int64_t seen = C.seen_top[t];
  for (unsigned int k = off[chunk]; k < off[chunk + 1]; ++k) {  // preorder of subtree starts
    const int64_t it = order[k];
    acc += C.acc_item[it * 32 + lane];
    seen += C.seen_item[it * 32 + lane];
  }
  const int64_t qi = C.qperm ? (int64_t)C.qperm[t] : t;
  out[qi] = (float)acc;
  if (visited) visited[qi] = seen;
}

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <int KID, bool VOTE>
static int bh_split_launch(FsTree* t, const double* q, int64_t n, const int32_t* qperm,
                           double beta, KParams kp, float* out, int64_t* visited, int sms,
                           int cap, cudaStream_t s, bool* done, unsigned int* emitted) {
  *done = false;
  const int64_t nchunks = (n + 31) / 32;
  BhSplitCtx C;
  C.rec = reinterpret_cast<const float4*>(t->bh32);
  C.pa = t->pts32a;
  C.pb = t->pts32b;
  C.q = q;
  C.qperm = qperm;
  C.n = n;
  C.nn = (uint32_t)t->n;
  C.beta = (float)beta;
  C.split_after = env_int("FSB_BH_SPLIT_AFTER", 192);
  C.min_split = env_int("FSB_BH_MIN_SPLIT", 32);
  C.cap = cap;
  Scratch items, ctrs, cnt, atop, stop, aitem, sitem, work;
  FS_TRY(items.alloc(sizeof(BhItem) * (size_t)C.cap, s));
  FS_TRY(ctrs.alloc(2 * sizeof(unsigned int), s));
  FS_TRY(cnt.alloc(sizeof(unsigned int) * (size_t)(nchunks + 1), s));
  FS_TRY(atop.alloc(sizeof(double) * (size_t)n, s));
  FS_TRY(stop.alloc(sizeof(int32_t) * (size_t)n, s));
  FS_TRY(aitem.alloc(sizeof(double) * 32 * (size_t)C.cap, s));
  FS_TRY(sitem.alloc(sizeof(int32_t) * 32 * (size_t)C.cap, s));
  FS_TRY(work.alloc(sizeof(unsigned int), s));
  FS_CK(cudaMemsetAsync(ctrs.p, 0, 2 * sizeof(unsigned int), s));
  FS_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned int) * (size_t)(nchunks + 1), s));
  C.items = items.as<BhItem>();
  C.n_items = ctrs.as<unsigned int>();
  C.overflow = ctrs.as<unsigned int>() + 1;
  C.chunk_items = cnt.as<unsigned int>();
  C.acc_top = atop.as<double>();
  C.seen_top = stop.as<int32_t>();
  C.acc_item = aitem.as<double>();
  C.seen_item = sitem.as<int32_t>();

  int per_sm = 1;
  FS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bh_units<KID, false, VOTE>, 128,
                                                      0));
  const int64_t max_grid = (int64_t)sms * std::max(per_sm, 1);
  auto run = [&](auto kern, unsigned int u0, unsigned int u1) -> int {
    FS_CK(cudaMemsetAsync(work.p, 0, sizeof(unsigned int), s));
    const int64_t grid = std::min<int64_t>(((int64_t)(u1 - u0) + 3) / 4, max_grid);
    kern<<<(unsigned)std::max<int64_t>(grid, 1), 128, 0, s>>>(C, kp, u0, u1,
                                                              work.as<unsigned int>());
    FS_CK(cudaGetLastError());
    return 0;
  };
  FS_TRY(run(k_bh_units<KID, false, VOTE>, 0u, (unsigned int)nchunks));
  // follow-up launches walk the emitted items (which may emit more)
  unsigned int done_items = 0, h[2] = {0, 0};
  while (true) {
    FS_CK(cudaMemcpyAsync(h, ctrs.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    FS_CK(cudaStreamSynchronize(s));
    if (h[1]) {  // queue overflow: the caller retries with a larger queue
      *emitted = h[0];
      return 0;
    }
    const unsigned int total = std::min<unsigned int>(h[0], (unsigned int)C.cap);
    if (total == done_items) break;
    FS_TRY(run(k_bh_units<KID, true, VOTE>, done_items, total));
    done_items = total;
  }
  // order each chunk's items by subtree start (preorder) and fold
  const int m = (int)done_items;
  Scratch k0, k1, i0, order, off, tmp;
  FS_TRY(k0.alloc(8 * (size_t)std::max(m, 1), s));
  FS_TRY(k1.alloc(8 * (size_t)std::max(m, 1), s));
  FS_TRY(i0.alloc(4 * (size_t)std::max(m, 1), s));
  FS_TRY(order.alloc(4 * (size_t)std::max(m, 1), s));
  FS_TRY(off.alloc(sizeof(unsigned int) * (size_t)(nchunks + 1), s));
  if (m > 0) {
    k_bh_item_keys<<<grid_for(m, 256), 256, 0, s>>>(C.items, m, k0.as<uint64_t>(),
                                                    i0.as<int32_t>());
    size_t tb = 0;
    FS_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                          i0.as<int32_t>(), order.as<int32_t>(), m, 0, 64, s));
    FS_TRY(tmp.alloc(tb, s));
    FS_CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                          i0.as<int32_t>(), order.as<int32_t>(), m, 0, 64, s));
  }
  {
    size_t tb = 0;
    FS_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<unsigned int>(),
                                        off.as<unsigned int>(), (int)(nchunks + 1), s));
    Scratch tmp2;
    FS_TRY(tmp2.alloc(tb, s));
    FS_CK(cub::DeviceScan::ExclusiveSum(tmp2.p, tb, cnt.as<unsigned int>(),
                                        off.as<unsigned int>(), (int)(nchunks + 1), s));
    k_bh_fold<<<grid_for(n, 256), 256, 0, s>>>(C, order.as<int32_t>(), off.as<unsigned int>(),
                                               out, visited);
    FS_CK(cudaGetLastError());
  }
  *emitted = done_items;
  *done = true;
  return 0;
}

int barnes_hut_split(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                     const int32_t* qperm, double beta, float* out, int64_t* visited,
                     cudaStream_t s, bool* done, bool vote) {
  KParams kp;
  kp.alpha = alpha;
  kp.dfloor = dfloor;
  kp.alpha_log2e_neg = (float)(-alpha * 1.4426950408889634);
  kp.dfloor_f = (float)dfloor;
  kp.inv_dfloor_f = (float)(1.0 / dfloor);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (t->n >= (1ll << 31)) {
    *done = false;
    return 0;
  }
  // item queue sized from the last call's count on this tree (a size hint only,
  // so concurrent calls on other streams stay safe); an overflow retries bigger
  const int64_t nchunks = (n + 31) / 32;
  int64_t cap = std::max<int64_t>(std::max<int64_t>(4096, 32 * nchunks),
                                  (int64_t)t->bh_items_hint.load() * 5 / 4);
  if (const char* e = std::getenv("FSB_BH_ITEM_CAP")) cap = std::atoll(e);
  for (int attempt = 0; attempt < 4; ++attempt) {
    unsigned int emitted = 0;
    int rc = 0;
    auto go = [&](auto launch) {
      return launch(t, q, n, qperm, beta, kp, out, visited, sms, (int)cap, s, done, &emitted);
    };
    switch (kid * 2 + (vote ? 1 : 0)) {
      case 0: rc = go(bh_split_launch<0, false>); break;
      case 1: rc = go(bh_split_launch<0, true>); break;
      case 2: rc = go(bh_split_launch<1, false>); break;
      case 3: rc = go(bh_split_launch<1, true>); break;
      case 4: rc = go(bh_split_launch<2, false>); break;
      default: rc = go(bh_split_launch<2, true>); break;
    }
    if (rc) return rc;
    if (std::getenv("FSB_BH_DEBUG"))
      fprintf(stderr, "bh split: cap %lld, emitted %u, %s\n", (long long)cap, emitted,
              *done ? "ok" : "overflow");
    if (*done) {
      t->bh_items_hint.store((int)std::min<int64_t>(emitted, 1 << 30));
      return 0;
    }
    cap = std::min<int64_t>(std::max<int64_t>(cap * 4, (int64_t)emitted * 2), (int64_t)1 << 25);
  }
  return 0;  // not done: the caller falls back to the warp-coherent kernel
}

}  // namespace fsb
