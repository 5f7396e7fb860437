// fs_pack.cu -- packed node records for the evaluators, and device trees
// assembled from reference-layout arrays (Octree.core_arrays(), octree.py:110-115).
#include <algorithm>
#include <vector>

#include "fs_common.cuh"
#include "fs_internal.h"

namespace fsb {

template <class T>
static int dalloc(T** p, int64_t count, cudaStream_t s) {  // stream-ordered pool (fs_build.cu)
  retain_pool_memory();
  FS_CK(cudaMallocAsync((void**)p, sizeof(T) * (size_t)std::max<int64_t>(count, 1), s));
  return 0;
}

void free_tree(FsTree* t) {
  if (!t) return;
  void* ptrs[] = {t->bbox_min, t->bbox_max, t->diameter, t->agg_mass, t->agg_weight, t->com,
                  t->child_start, t->child_count, t->child_index, t->begin, t->end, t->depth,
                  t->perm, t->points, t->masses, t->weights, t->lo2pre, t->pre2lo, t->skip,
                  t->fc_lo, t->bh32, t->bh64, t->lo_geo32, t->lo_mass32, t->lo_geo64,
                  t->lo_mass64, t->lo_topo, t->pts32a, t->pts32b, t->pts64a, t->pts64b,
                  t->lo_cm32, t->lo_m12_32, t->lo_begin, t->pt_path, t->lo_cmp, t->lo_cm64,
                  t->lo_m12_64};
  // the handle's owner may still have work queued on any stream: wait for the
  // device once, then return every array to the pool
  cudaDeviceSynchronize();
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, 0);
  delete t;
}

// ------------------------------------------------------------ from arrays
__global__ void k_parent(const int64_t* __restrict__ cs, const int64_t* __restrict__ cc,
                         const int64_t* __restrict__ ci, int64_t n, int32_t* __restrict__ parent) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0) parent[0] = 0;
  int64_t s = cs[i], k = cc[i];
  for (int64_t t = 0; t < k; ++t) parent[ci[s + t]] = (int32_t)i;
}

__global__ void k_jump(const int32_t* __restrict__ anc, const int32_t* __restrict__ dist, int64_t n,
                       int32_t* __restrict__ anc2, int32_t* __restrict__ dist2) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t a = anc[i];
  dist2[i] = dist[i] + dist[a];
  anc2[i] = anc[a];
}

__global__ void k_init_dist(int64_t n, int32_t* __restrict__ dist) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dist[i] = i == 0 ? 0 : 1;
}

__global__ void k_begin32(const int64_t* __restrict__ b, int64_t n, int32_t* __restrict__ nb,
                          int32_t* __restrict__ first_at) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  nb[i] = (int32_t)b[i];
  if (i == 0 || b[i - 1] != b[i]) first_at[b[i]] = (int32_t)i;
}

__global__ void k_fc_skip(const int64_t* __restrict__ cs, const int64_t* __restrict__ cc,
                          const int64_t* __restrict__ ci, const int64_t* __restrict__ end,
                          const int32_t* __restrict__ pre2lo, const int32_t* __restrict__ first_at,
                          int64_t n, int64_t m, int32_t* __restrict__ fc, int32_t* __restrict__ skip) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  fc[i] = cc[i] > 0 ? pre2lo[ci[cs[i]]] : 0;
  int64_t e = end[i];
  skip[i] = e < m ? first_at[e] : (int32_t)n;
}

int tree_from_arrays(FsTree** out, const double* diameter, const double* agg_mass,
                     const double* com, const int64_t* child_start, const int64_t* child_count,
                     const int64_t* child_index, const int64_t* begin, const int64_t* end,
                     const double* points, const double* masses, int64_t n, int64_t m, int c,
                     cudaStream_t s) {
  *out = nullptr;
  if (n < 1 || m < 1 || c < 1 || n >= (int64_t(1) << 31) - 2) {
    set_error("tree_from_arrays: bad sizes");
    return 1;
  }
  FsTree* t = new FsTree();
  t->n = n;
  t->m = m;
  t->c = c;
  int rc = 0;
  auto cp = [&](auto** dst, const auto* src, int64_t count) -> int {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(*dst)>>;
    FS_TRY(dalloc(dst, count, s));
    if (count > 0)
      FS_CK(cudaMemcpyAsync(*dst, src, sizeof(T) * count, cudaMemcpyDeviceToDevice, s));
    return 0;
  };
  if ((rc = cp(&t->diameter, diameter, n)) || (rc = cp(&t->agg_mass, agg_mass, n * c)) ||
      (rc = cp(&t->com, com, 3 * n)) || (rc = cp(&t->child_start, child_start, n)) ||
      (rc = cp(&t->child_count, child_count, n)) ||
      (rc = cp(&t->child_index, child_index, n - 1)) || (rc = cp(&t->begin, begin, n)) ||
      (rc = cp(&t->end, end, n)) || (rc = cp(&t->points, points, 3 * m)) ||
      (rc = cp(&t->masses, masses, m * c)) || (rc = dalloc(&t->lo2pre, n, s)) ||
      (rc = dalloc(&t->pre2lo, n, s)) || (rc = dalloc(&t->skip, n, s)) || (rc = dalloc(&t->fc_lo, n, s))) {
    free_tree(t);
    return rc;
  }
  const int B = 256;
  Scratch anc, dist, anc2, dist2, nb, first_at;
  if ((rc = anc.alloc(4 * n, s)) || (rc = dist.alloc(4 * n, s)) || (rc = anc2.alloc(4 * n, s)) ||
      (rc = dist2.alloc(4 * n, s)) || (rc = nb.alloc(4 * n, s)) || (rc = first_at.alloc(4 * m, s))) {
    free_tree(t);
    return rc;
  }
  k_parent<<<grid_for(n, B), B, 0, s>>>(t->child_start, t->child_count, t->child_index, n,
                                        anc.as<int32_t>());
  k_init_dist<<<grid_for(n, B), B, 0, s>>>(n, dist.as<int32_t>());
  int32_t *a = anc.as<int32_t>(), *d = dist.as<int32_t>(), *a2 = anc2.as<int32_t>(),
          *d2 = dist2.as<int32_t>();
  for (int round = 0; round < 12; ++round) {  // depths < 4096
    k_jump<<<grid_for(n, B), B, 0, s>>>(a, d, n, a2, d2);
    std::swap(a, a2);
    std::swap(d, d2);
  }
  k_begin32<<<grid_for(n, B), B, 0, s>>>(t->begin, n, nb.as<int32_t>(), first_at.as<int32_t>());
  int64_t* lstart = nullptr;
  if ((rc = level_order(t, nb.as<int32_t>(), d, 4095, &lstart, s))) {
    free_tree(t);
    return rc;
  }
  cudaFreeAsync(lstart, s);
  k_fc_skip<<<grid_for(n, B), B, 0, s>>>(t->child_start, t->child_count, t->child_index, t->end,
                                         t->pre2lo, first_at.as<int32_t>(), n, m, t->fc_lo,
                                         t->skip);
  int64_t rk = 0;
  FS_CK(cudaMemcpyAsync(&rk, t->child_count, 8, cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  FS_CK(cudaGetLastError());
  t->root_kids = (int)rk;
  *out = t;
  return 0;
}

// ------------------------------------------------------------ BH records
template <class T>
__device__ __forceinline__ T int_bits(int64_t v);
template <>
__device__ __forceinline__ float int_bits<float>(int64_t v) { return __int_as_float((int)v); }
template <>
__device__ __forceinline__ double int_bits<double>(int64_t v) { return __longlong_as_double(v); }

template <class T, class V4>
__global__ void k_pack_bh(const double* __restrict__ com, const double* __restrict__ diam,
                          const double* __restrict__ am, const int64_t* __restrict__ cc,
                          const int64_t* __restrict__ b, const int64_t* __restrict__ e,
                          const int32_t* __restrict__ skip, int64_t n, int c, V4* __restrict__ g,
                          V4* __restrict__ mrec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool multi = cc[i] == 0 && e[i] - b[i] > 1;
  V4 gg, mm;
  gg.x = (T)com[3 * i];
  gg.y = (T)com[3 * i + 1];
  gg.z = (T)com[3 * i + 2];
  gg.w = multi ? (T)-1 : (T)diam[i];
  mm.x = (T)am[(int64_t)c * i];
  mm.y = c >= 3 ? (T)am[(int64_t)c * i + 1] : (T)0;
  mm.z = c >= 3 ? (T)am[(int64_t)c * i + 2] : (T)0;
  mm.w = int_bits<T>(skip[i]);
  if (multi) {
    mm.x = int_bits<T>(b[i]);
    mm.y = int_bits<T>(e[i]);
  }
  g[2 * i] = gg;  // interleaved: record i = {g, m}
  g[2 * i + 1] = mm;
  (void)mrec;
}

int ensure_bh(FsTree* t, bool f64, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  const int B = 256;
  if (f64 && !t->bh64) {
    BhRec64* rec = nullptr;
    FS_TRY(dalloc(&rec, t->n, s));
    k_pack_bh<double, double4><<<grid_for(t->n, B), B, 0, s>>>(
        t->com, t->diameter, t->agg_mass, t->child_count, t->begin, t->end, t->skip, t->n, t->c,
        reinterpret_cast<double4*>(rec), nullptr);
    FS_CK(cudaStreamSynchronize(s));
    t->bh64 = rec;
  } else if (!f64 && !t->bh32) {
    BhRec32* rec = nullptr;
    FS_TRY(dalloc(&rec, t->n, s));
    k_pack_bh<float, float4><<<grid_for(t->n, B), B, 0, s>>>(
        t->com, t->diameter, t->agg_mass, t->child_count, t->begin, t->end, t->skip, t->n, t->c,
        reinterpret_cast<float4*>(rec), nullptr);
    FS_CK(cudaStreamSynchronize(s));
    t->bh32 = rec;
  }
  FS_CK(cudaGetLastError());
  return 0;
}

// ------------------------------------------------------- level-order records
template <class T, class V4>
__global__ void k_pack_lo(const int32_t* __restrict__ lo2pre, const double* __restrict__ com,
                          const double* __restrict__ diam, const double* __restrict__ am,
                          const int64_t* __restrict__ cc, const int64_t* __restrict__ b,
                          const int64_t* __restrict__ e, const int32_t* __restrict__ fc, int64_t n,
                          int c, V4* __restrict__ geo, V4* __restrict__ mass,
                          int4* __restrict__ topo) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t i = lo2pre[r];
  V4 g, mm;
  g.x = (T)com[3 * i];
  g.y = (T)com[3 * i + 1];
  g.z = (T)com[3 * i + 2];
  g.w = (T)diam[i];
  mm.x = (T)am[(int64_t)c * i];
  mm.y = c >= 3 ? (T)am[(int64_t)c * i + 1] : (T)0;
  mm.z = c >= 3 ? (T)am[(int64_t)c * i + 2] : (T)0;
  mm.w = (T)0;
  geo[r] = g;
  mass[r] = mm;
  if (topo) topo[r] = make_int4(fc[i], (int)cc[i], (int)b[i], (int)e[i]);
}

template <class T, class V4>
__global__ void k_pack_pts(const double* __restrict__ pts, const double* __restrict__ ms, int64_t m,
                           int c, V4* __restrict__ a, V4* __restrict__ bq) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  V4 u, v;
  u.x = (T)pts[3 * j];
  u.y = (T)pts[3 * j + 1];
  u.z = (T)pts[3 * j + 2];
  u.w = (T)ms[(int64_t)c * j];
  v.x = c >= 3 ? (T)ms[(int64_t)c * j + 1] : (T)0;
  v.y = c >= 3 ? (T)ms[(int64_t)c * j + 2] : (T)0;
  v.z = (T)0;
  v.w = (T)0;
  a[j] = u;
  bq[j] = v;
}

int ensure_lo(FsTree* t, bool f64, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  const int B = 256;
  if ((f64 && t->lo_geo64) || (!f64 && t->lo_geo32)) return 0;
  // the topology is shared by both precisions: packed by the first call only
  int4* topo = nullptr;
  if (!t->lo_topo) FS_TRY(dalloc(&topo, t->n, s));
  if (f64) {
    double4 *geo = nullptr, *mass = nullptr, *pa = nullptr, *pb = nullptr;
    FS_TRY(dalloc(&geo, t->n, s));
    FS_TRY(dalloc(&mass, t->n, s));
    FS_TRY(dalloc(&pa, t->m, s));
    FS_TRY(dalloc(&pb, t->m, s));
    k_pack_lo<double, double4><<<grid_for(t->n, B), B, 0, s>>>(
        t->lo2pre, t->com, t->diameter, t->agg_mass, t->child_count, t->begin, t->end, t->fc_lo,
        t->n, t->c, geo, mass, topo);
    k_pack_pts<double, double4><<<grid_for(t->m, B), B, 0, s>>>(t->points, t->masses, t->m, t->c,
                                                                pa, pb);
    FS_CK(cudaStreamSynchronize(s));
    t->lo_geo64 = geo;
    t->lo_mass64 = mass;
    t->pts64a = pa;
    t->pts64b = pb;
  } else {
    float4 *geo = nullptr, *mass = nullptr, *pa = nullptr, *pb = nullptr;
    FS_TRY(dalloc(&geo, t->n, s));
    FS_TRY(dalloc(&mass, t->n, s));
    FS_TRY(dalloc(&pa, t->m, s));
    FS_TRY(dalloc(&pb, t->m, s));
    k_pack_lo<float, float4><<<grid_for(t->n, B), B, 0, s>>>(
        t->lo2pre, t->com, t->diameter, t->agg_mass, t->child_count, t->begin, t->end, t->fc_lo,
        t->n, t->c, geo, mass, topo);
    k_pack_pts<float, float4><<<grid_for(t->m, B), B, 0, s>>>(t->points, t->masses, t->m, t->c,
                                                              pa, pb);
    FS_CK(cudaStreamSynchronize(s));
    t->lo_geo32 = geo;
    t->lo_mass32 = mass;
    t->pts32a = pa;
    t->pts32b = pb;
  }
  if (topo) t->lo_topo = topo;
  FS_CK(cudaGetLastError());
  return 0;
}

// ------------------------------------------------------------ fast records
__global__ void k_pack_fast(const int32_t* __restrict__ lo2pre, const double* __restrict__ com,
                            const double* __restrict__ am, const int64_t* __restrict__ b, int64_t n,
                            int c, float4* __restrict__ cm, float2* __restrict__ m12,
                            int32_t* __restrict__ lb) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t i = lo2pre[r];
  cm[r] = make_float4((float)com[3 * i], (float)com[3 * i + 1], (float)com[3 * i + 2],
                      (float)am[(int64_t)c * i]);
  if (m12) m12[r] = make_float2((float)am[(int64_t)c * i + 1], (float)am[(int64_t)c * i + 2]);
  lb[r] = (int32_t)b[i];
}

// per level: is the cell diameter uniform, and does the level hold a multi-point leaf?
__global__ void k_level_check(int64_t r0, int64_t r1, int level, const int32_t* __restrict__ lo2pre,
                              const double* __restrict__ diam, const int64_t* __restrict__ cc,
                              const int64_t* __restrict__ b, const int64_t* __restrict__ e,
                              int* __restrict__ flags) {
  int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= r1) return;
  int64_t i = lo2pre[r];
  if (diam[i] != diam[lo2pre[r0]]) flags[0] = 1;
  if (cc[i] == 0 && e[i] - b[i] > 1) atomicMin(&flags[1], level);
}

// rank of point j's ancestor among its siblings, per level, packed LSB-first
__global__ void k_point_path(const int4* __restrict__ topo, int64_t m, int bits, int levels,
                             uint64_t* __restrict__ path) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  uint64_t p = 0;
  int node = 0;
  for (int l = 1; l <= levels; ++l) {
    const int4 tp = topo[node];  // {first child, count, begin, end}
    if (tp.y == 0) break;
    int lo = 0, hi = tp.y;  // last child whose begin <= j
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (topo[tp.x + mid].z <= j)
        lo = mid;
      else
        hi = mid;
    }
    p |= (uint64_t)lo << (bits * (l - 1));
    node = tp.x + lo;
  }
  path[j] = p;
}

__global__ void k_max_children(const int4* __restrict__ topo, int64_t n, int* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int v = r < n ? topo[r].y : 0;
  v = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(out, v);
}

int ensure_path(FsTree* t, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  if (t->pt_path) return 0;
  FS_TRY(ensure_lo(t, false, s));
  Scratch mx;
  FS_TRY(mx.alloc(sizeof(int), s));
  FS_CK(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
  k_max_children<<<grid_for(t->n, 256), 256, 0, s>>>(t->lo_topo, t->n, mx.as<int>());
  int kids = 0;
  FS_CK(cudaMemcpyAsync(&kids, mx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  int bits = 1;
  while ((1ll << bits) < kids) ++bits;
  uint64_t* path = nullptr;
  FS_TRY(dalloc(&path, t->m, s));
  const int levels = bits <= 16 ? 64 / bits : 0;
  k_point_path<<<grid_for(t->m, 256), 256, 0, s>>>(t->lo_topo, t->m, bits, levels, path);
  FS_CK(cudaStreamSynchronize(s));
  t->path_bits = bits;
  t->path_levels = levels;
  t->max_children = kids;
  t->pt_path = path;
  FS_CK(cudaGetLastError());
  return 0;
}

__global__ void k_pack_pairs(const float4* __restrict__ cm, int64_t n, float4* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (2 * i >= n) return;
  const float4 u = cm[2 * i];
  const float4 v = 2 * i + 1 < n ? cm[2 * i + 1] : make_float4(u.x, u.y, u.z, 0.f);
  out[2 * i] = make_float4(u.x, v.x, u.y, v.y);
  out[2 * i + 1] = make_float4(u.z, v.z, -u.w, -v.w);
}

int ensure_pairs(FsTree* t, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  if (t->lo_cmp) return 0;
  FS_TRY(ensure_fast(t, s));
  const int64_t np = (t->n + 1) / 2;
  float4* pairs = nullptr;
  FS_TRY(dalloc(&pairs, 2 * np, s));
  k_pack_pairs<<<grid_for(np, 256), 256, 0, s>>>(t->lo_cm32, t->n, pairs);
  FS_CK(cudaStreamSynchronize(s));
  t->lo_cmp = pairs;
  FS_CK(cudaGetLastError());
  return 0;
}

__global__ void k_level_diam(const int64_t* __restrict__ start, int nl,
                             const int32_t* __restrict__ lo2pre, const double* __restrict__ diam,
                             double* __restrict__ out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < nl) out[l] = diam[lo2pre[start[l]]];
}

int ensure_fast(FsTree* t, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  if (t->fast_ready) return 0;
  const int B = 256;
  // (an earlier call that failed half-way may have left buffers behind)
  if (!t->lo_cm32) FS_TRY(dalloc(&t->lo_cm32, t->n, s));
  if (!t->lo_begin) FS_TRY(dalloc(&t->lo_begin, t->n, s));
  if (t->c >= 3 && !t->lo_m12_32) FS_TRY(dalloc(&t->lo_m12_32, t->n, s));
  k_pack_fast<<<grid_for(t->n, B), B, 0, s>>>(t->lo2pre, t->com, t->agg_mass, t->begin, t->n, t->c,
                                              t->lo_cm32, t->c >= 3 ? t->lo_m12_32 : nullptr,
                                              t->lo_begin);
  Scratch fl;
  FS_TRY(fl.alloc(2 * sizeof(int), s));
  int init[2] = {0, 1 << 30};
  FS_CK(cudaMemcpyAsync(fl.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  for (int l = 0; l < t->num_levels; ++l) {
    int64_t r0 = t->level_off[l], r1 = t->level_off[l + 1];
    if (r1 > r0)
      k_level_check<<<grid_for(r1 - r0, B), B, 0, s>>>(r0, r1, l, t->lo2pre, t->diameter,
                                                       t->child_count, t->begin, t->end,
                                                       fl.as<int>());
  }
  int res[2];
  FS_CK(cudaMemcpyAsync(res, fl.p, sizeof(res), cudaMemcpyDeviceToHost, s));
  // one diameter per level (the level's first node), gathered on the device
  const int nl = std::min(t->num_levels, FsTree::kMaxLevels);
  std::vector<int64_t> starts(t->level_off.begin(), t->level_off.begin() + nl);
  std::vector<double> ldiam(std::max(nl, 1));
  Scratch dstart, ddiam;
  FS_TRY(dstart.alloc(sizeof(int64_t) * std::max(nl, 1), s));
  FS_TRY(ddiam.alloc(sizeof(double) * std::max(nl, 1), s));
  if (nl > 0) {
    FS_CK(cudaMemcpyAsync(dstart.p, starts.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice,
                          s));
    k_level_diam<<<grid_for(nl, 64), 64, 0, s>>>(dstart.as<int64_t>(), nl, t->lo2pre,
                                                 t->diameter, ddiam.as<double>());
    FS_CK(cudaMemcpyAsync(ldiam.data(), ddiam.p, sizeof(double) * nl, cudaMemcpyDeviceToHost, s));
  }
  FS_CK(cudaStreamSynchronize(s));
  for (int l = 0; l < nl; ++l) {
    t->level_diam[l] = (float)ldiam[l];
    t->level_diam64[l] = ldiam[l];
  }
  t->uniform_diam = res[0] == 0 && t->num_levels <= FsTree::kMaxLevels;
  t->first_multi_level = res[1];
  t->fast_ready = true;
  FS_CK(cudaGetLastError());
  return 0;
}

// ------------------------------------------------ FP64 queue-kernel records
__global__ void k_pack_cm64(const int32_t* __restrict__ lo2pre, const double* __restrict__ com,
                            const double* __restrict__ am, int64_t n, int c,
                            double4* __restrict__ cm, double2* __restrict__ m12) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t i = lo2pre[r];
  cm[r] = make_double4(com[3 * i], com[3 * i + 1], com[3 * i + 2], am[(int64_t)c * i]);
  if (m12) m12[r] = make_double2(am[(int64_t)c * i + 1], am[(int64_t)c * i + 2]);
}

// operand ranges of the FP64 division fast path (contrib_parity_fast): bit 0 set
// when a node coordinate exceeds 2^100 in magnitude (or is not finite), bit 1
// when a node's first mass channel is outside [2^-800, 2^800] (or zero / NaN)
__global__ void k_div_range(const double4* __restrict__ cm, int64_t n, unsigned int* flags) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned int f = 0;
  if (r < n) {
    const double4 c = cm[r];
    if (!(fabs(c.x) <= 0x1p100 && fabs(c.y) <= 0x1p100 && fabs(c.z) <= 0x1p100)) f |= 1u;
    if (!(fabs(c.w) >= 0x1p-800 && fabs(c.w) <= 0x1p800)) f |= 2u;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

int internal_level1(FsTree* t, cudaStream_t s, int* out) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  if (t->internal_kids < 0) {
    int cnt = 0;
    if (t->root_kids > 0) {
      if (!t->lo_topo) FS_TRY(ensure_lo(t, false, s));  // level-order topology
      std::vector<int4> tp((size_t)t->root_kids);
      FS_CK(cudaMemcpyAsync(tp.data(), t->lo_topo + 1, sizeof(int4) * tp.size(),
                            cudaMemcpyDeviceToHost, s));
      FS_CK(cudaStreamSynchronize(s));
      for (const int4& v : tp) cnt += v.y > 0;
    }
    t->internal_kids = cnt;
  }
  *out = t->internal_kids;
  return 0;
}

int ensure_cm64(FsTree* t, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(t->mu);
  if (t->lo_cm64) return 0;
  double4* cm = nullptr;
  double2* m12 = nullptr;
  FS_TRY(dalloc(&cm, t->n, s));
  if (t->c >= 3) FS_TRY(dalloc(&m12, t->n, s));
  k_pack_cm64<<<grid_for(t->n, 256), 256, 0, s>>>(t->lo2pre, t->com, t->agg_mass, t->n, t->c, cm,
                                                  m12);
  Scratch fl;
  FS_TRY(fl.alloc(sizeof(unsigned int), s));
  FS_CK(cudaMemsetAsync(fl.p, 0, sizeof(unsigned int), s));
  k_div_range<<<grid_for(t->n, 256), 256, 0, s>>>(cm, t->n, fl.as<unsigned int>());
  unsigned int flags = 3;
  FS_CK(cudaMemcpyAsync(&flags, fl.p, sizeof(flags), cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  t->coords_in_range = (flags & 1u) == 0;
  t->masses_in_range = (flags & 2u) == 0;
  t->lo_m12_64 = m12;
  t->lo_cm64 = cm;
  FS_CK(cudaGetLastError());
  return 0;
}

}  // namespace fsb
