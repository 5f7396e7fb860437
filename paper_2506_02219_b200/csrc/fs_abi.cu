// fs_abi.cu -- extern "C" boundary (include/fastsum_b200.h) over the device code.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/fastsum_b200.h"
#include "fs_common.cuh"
#include "fs_eval.h"
#include "fs_internal.h"

struct fsb_tree {
  fsb::FsTree* t;
};

namespace fsb {
static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void retain_pool_memory() {
  static thread_local int done_mask = 0;  // one bit per device (first 32 devices)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32 || (done_mask >> dev) & 1) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_mask |= 1 << dev;
}

// ---------------------------------------------------------- query ordering
__global__ void k_qbbox(const double* __restrict__ q, int64_t n, float* __restrict__ part) {
  __shared__ float sm[6][256];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      float v = (float)q[3 * i + k];
      lo[k] = fminf(lo[k], v);
      hi[k] = fmaxf(hi[k], v);
    }
  for (int k = 0; k < 3; ++k) {
    sm[k][threadIdx.x] = lo[k];
    sm[3 + k][threadIdx.x] = hi[k];
  }
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 3; ++k) {
        sm[k][threadIdx.x] = fminf(sm[k][threadIdx.x], sm[k][threadIdx.x + st]);
        sm[3 + k][threadIdx.x] = fmaxf(sm[3 + k][threadIdx.x], sm[3 + k][threadIdx.x + st]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sm[threadIdx.x][0];
}

__global__ void k_qbbox_final(float* __restrict__ part, int nb) {
  if (threadIdx.x >= 6) return;
  int k = threadIdx.x;
  float v = part[k];
  for (int b = 1; b < nb; ++b) v = k < 3 ? fminf(v, part[b * 6 + k]) : fmaxf(v, part[b * 6 + k]);
  part[k] = v;
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

__global__ void k_qmorton(const double* __restrict__ q, int64_t n, const float* __restrict__ bb,
                          uint32_t* __restrict__ code, int32_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c[3];
  for (int k = 0; k < 3; ++k) {
    float ext = bb[3 + k] - bb[k];
    float u = ext > 0.f ? ((float)q[3 * i + k] - bb[k]) / ext : 0.f;
    c[k] = (uint32_t)fminf(fmaxf(u * 1024.f, 0.f), 1023.f);
  }
  code[i] = (spread10(c[0]) << 2) | (spread10(c[1]) << 1) | spread10(c[2]);
  idx[i] = (int32_t)i;
}

int query_order(const double* q, int64_t n, int32_t* perm, cudaStream_t s) {
  if (n <= 0) return 0;
  Scratch bb, code, code2, idx;
  const int nb = (int)std::min<int64_t>(296, (n + 255) / 256);
  FS_TRY(bb.alloc(6 * sizeof(float) * nb, s));
  FS_TRY(code.alloc(4 * n, s));
  FS_TRY(code2.alloc(4 * n, s));
  FS_TRY(idx.alloc(4 * n, s));
  k_qbbox<<<nb, 256, 0, s>>>(q, n, bb.as<float>());
  k_qbbox_final<<<1, 32, 0, s>>>(bb.as<float>(), nb);
  k_qmorton<<<grid_for(n, 256), 256, 0, s>>>(q, n, bb.as<float>(), code.as<uint32_t>(),
                                             idx.as<int32_t>());
  size_t tb = 0;
  FS_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, code.as<uint32_t>(), code2.as<uint32_t>(),
                                        idx.as<int32_t>(), perm, (int)n, 0, 30, s));
  Scratch tmp;
  FS_TRY(tmp.alloc(tb, s));
  FS_CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, code.as<uint32_t>(), code2.as<uint32_t>(),
                                        idx.as<int32_t>(), perm, (int)n, 0, 30, s));
  return 0;
}
// seeded pseudo-random evaluation order (the paper shuffles the query grid so that
// RNG-sharing groups are spatially scattered)
// Seeded evaluation order of the warp-shared mode: positions are cut into
// windows of kShuffleWindow = 2^16, and window w (positions [wW, min((w+1)W, n)))
// is permuted by a 4-round balanced Feistel network (32-bit lowbias32 rounds)
// keyed on (seed, query_offset + wW) over the smallest 2^(2h) >= its size
// (exactly 2^16 for full windows), cycle-walked back into range for the last
// partial window (a bijection).  One pass, no sort.
// Windows keep the order slab-local, so the host pipeline can copy, evaluate
// and return window-aligned slabs independently (same result as one launch).
// blocks of 256 positions never straddle a window (kShuffleWindow % 256 == 0):
// thread 0 derives the window's round keys once per block
__global__ void __launch_bounds__(256) k_shuffle(int64_t n, uint64_t h, int64_t qoff,
                                                 int32_t* __restrict__ perm) {
  __shared__ uint32_t s_ks[4];
  const int64_t b0 = blockIdx.x * (int64_t)blockDim.x;
  const int64_t base = b0 & ~(int64_t)(kShuffleWindow - 1);
  if (threadIdx.x == 0) {
    const uint64_t hw = key_fold(h, (uint64_t)(qoff + base));
    const uint64_t hw1 = key_fold(hw, 1);
    s_ks[0] = (uint32_t)hw;
    s_ks[1] = (uint32_t)(hw >> 32);
    s_ks[2] = (uint32_t)hw1;
    s_ks[3] = (uint32_t)(hw1 >> 32);
  }
  __syncthreads();
  const int64_t i = b0 + threadIdx.x;
  if (i >= n) return;
  const uint32_t size = (uint32_t)min((int64_t)kShuffleWindow, n - base);
  int hb = 1;  // full windows: 2^(2 hb) == size, no cycle walking
  while ((1u << (2 * hb)) < size) ++hb;
  const uint32_t ks[4] = {s_ks[0], s_ks[1], s_ks[2], s_ks[3]};
  uint32_t y = feistel4((uint32_t)(i - base), hb, ks);
  while (y >= size) y = feistel4(y, hb, ks);
  perm[i] = (int32_t)(base + (int64_t)y);
}

static_assert(kShuffleWindow == kShuffleWindowC, "one shuffle window size");
static_assert(FSB_FLAG_ALG2 == kFlagAlg2 && FSB_FLAG_SHUFFLED == kFlagShuffled, "flag values");

int shuffle_order(int64_t n, uint64_t seed, int64_t qoff, int32_t* perm, cudaStream_t s) {
  if (n <= 0) return 0;
  const uint64_t h = shuffle_key(seed);
  k_shuffle<<<grid_for(n, 256), 256, 0, s>>>(n, h, qoff, perm);
  FS_CK(cudaGetLastError());
  return 0;
}
}  // namespace fsb

using fsb::set_error;

#define ABI_TREE(tree)                              \
  if (!(tree) || !(tree)->t) {                      \
    set_error("null tree handle");                  \
    return 1;                                       \
  }

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int check_common(int kid, int precision, int64_t n) {
  if (kid < 0 || kid > 2) {
    set_error("unknown kernel id %d", kid);
    return 1;
  }
  if (precision != 0 && precision != 1) {
    set_error("precision must be 0 (f64) or 1 (f32)");
    return 1;
  }
  if (n < 0) {
    set_error("negative query count");
    return 1;
  }
  return 0;
}

extern "C" {

int fsb_abi_version(void) { return 2; }

const char* fsb_last_error(void) { return fsb::g_last_error.c_str(); }

int fsb_brute_force_batch(int kid, double alpha, double dfloor, int precision, const double* pts,
                          const double* ms, int64_t m, int c, const double* queries, int64_t n,
                          void* out, void* stream) {
  FSB_RANGE("fsb_brute_force_batch");
  if (int rc = check_common(kid, precision, n)) return rc;
  if (m < 1 || (kid == 1 ? c != 3 : c < 1)) {
    set_error("bad source count / channel count (m=%lld c=%d)", (long long)m, c);
    return 1;
  }
  return fsb::brute_force(kid, alpha, dfloor, precision == 0, pts, ms, m, c, queries, n, out,
                          S(stream));
}

int fsb_brute_force_f32acc64(int kid, double alpha, double dfloor, const double* pts,
                             const double* ms, int64_t m, int c, const double* queries, int64_t n,
                             double* out, void* stream) {
  FSB_RANGE("fsb_brute_force_f32acc64");
  if (int rc = check_common(kid, 1, n)) return rc;
  if (n == 0) return 0;
  return fsb::brute_force_f32_acc64(kid, alpha, dfloor, pts, ms, m, c, queries, n, out, S(stream));
}

int fsb_build_tree(const double* positions, const double* masses, const double* weights,
                   int64_t m, int c, int branching_per_dim, int max_depth, fsb_tree** out,
                   void* stream) {
  FSB_RANGE("fsb_build_tree");
  if (!out) {
    set_error("null output handle");
    return 1;
  }
  *out = nullptr;
  fsb::FsTree* t = nullptr;
  int rc = fsb::build_tree(&t, positions, masses, weights, m, c, branching_per_dim, max_depth,
                           S(stream));
  if (rc) return rc;
  *out = new fsb_tree{t};
  return 0;
}

int fsb_tree_from_core_arrays(const double* diameter, const double* aggregate_mass,
                              const double* center_of_mass, const int64_t* child_start,
                              const int64_t* child_count, const int64_t* child_index,
                              const int64_t* begin, const int64_t* end, const double* points,
                              const double* masses, int64_t num_nodes, int64_t num_points,
                              int channels, fsb_tree** out, void* stream) {
  FSB_RANGE("fsb_tree_from_core_arrays");
  if (!out) {
    set_error("null output handle");
    return 1;
  }
  *out = nullptr;
  fsb::FsTree* t = nullptr;
  int rc = fsb::tree_from_arrays(&t, diameter, aggregate_mass, center_of_mass, child_start,
                                 child_count, child_index, begin, end, points, masses, num_nodes,
                                 num_points, channels, S(stream));
  if (rc) return rc;
  *out = new fsb_tree{t};
  return 0;
}

int fsb_tree_info(const fsb_tree* tree, int64_t* info) {
  ABI_TREE(tree);
  const fsb::FsTree* t = tree->t;
  info[0] = t->n;
  info[1] = t->m;
  info[2] = t->c;
  info[3] = t->d;
  info[4] = t->max_depth;
  info[5] = t->num_levels;
  info[6] = t->root_kids;
  info[7] = t->owns_export ? 1 : 0;
  return 0;
}

int fsb_tree_export(const fsb_tree* tree, void* const* dst, void* stream) {
  FSB_RANGE("fsb_tree_export");
  ABI_TREE(tree);
  const fsb::FsTree* t = tree->t;
  if (!t->owns_export) {
    set_error("tree was assembled from core arrays; nothing to export");
    return 1;
  }
  int64_t n = t->n, m = t->m, c = t->c;
  const void* src[16] = {t->bbox_min, t->bbox_max, t->diameter, t->agg_mass, t->agg_weight,
                         t->com, t->child_start, t->child_count, t->child_index, t->begin,
                         t->end, t->depth, t->perm, t->points, t->masses, t->weights};
  size_t bytes[16] = {24 * (size_t)n, 24 * (size_t)n, 8 * (size_t)n, 8 * (size_t)(n * c),
                      8 * (size_t)n, 24 * (size_t)n, 8 * (size_t)n, 8 * (size_t)n,
                      8 * (size_t)(n - 1), 8 * (size_t)n, 8 * (size_t)n, 8 * (size_t)n,
                      8 * (size_t)m, 24 * (size_t)m, 8 * (size_t)(m * c), 8 * (size_t)m};
  for (int k = 0; k < 16; ++k) {
    if (!dst[k] || bytes[k] == 0) continue;
    FS_CK(cudaMemcpyAsync(dst[k], src[k], bytes[k], cudaMemcpyDefault, S(stream)));
  }
  FS_CK(cudaStreamSynchronize(S(stream)));
  return 0;
}

int fsb_tree_free(fsb_tree* tree) {
  if (!tree) return 0;
  fsb::free_tree(tree->t);
  delete tree;
  return 0;
}

int fsb_barnes_hut_batch(fsb_tree* tree, int kid, double alpha, double dfloor, int precision,
                         const double* queries, int64_t n, const int32_t* qperm, double beta,
                         void* out, int64_t* visited, void* stream) {
  FSB_RANGE("fsb_barnes_hut_batch");
  ABI_TREE(tree);
  if (int rc = check_common(kid, precision, n)) return rc;
  if (!(beta > 0)) {
    set_error("beta must be positive");
    return 1;
  }
  return fsb::barnes_hut(tree->t, kid, alpha, dfloor, precision == 0, queries, n, qperm, beta,
                         out, visited, S(stream));
}

int fsb_barnes_hut_vote_batch(fsb_tree* tree, int kid, double alpha, double dfloor,
                              int precision, const double* queries, int64_t n,
                              const int32_t* order, double beta, void* out, int64_t* visited,
                              void* stream) {
  FSB_RANGE("fsb_barnes_hut_vote_batch");
  ABI_TREE(tree);
  if (int rc = check_common(kid, precision, n)) return rc;
  if (!(beta > 0)) {
    set_error("beta must be positive");
    return 1;
  }
  return fsb::barnes_hut(tree->t, kid, alpha, dfloor, precision == 0, queries, n, order, beta,
                         out, visited, S(stream), true);
}

int fsb_stochastic_batch(fsb_tree* tree, int kid, double alpha, double dfloor, int precision,
                         const double* queries, int64_t n, const int32_t* qperm,
                         int64_t n_samples, int rr_mode, uint64_t seed, int64_t query_offset,
                         void* out, int64_t* visited, int64_t* path_steps, int64_t* path_count,
                         void* stream) {
  FSB_RANGE("fsb_stochastic_batch");
  ABI_TREE(tree);
  if (int rc = check_common(kid, precision, n)) return rc;
  if (n_samples < 1 || n_samples > (1LL << 30)) {
    set_error("samples_per_subdomain must be >= 1");
    return 1;
  }
  if (rr_mode < 0 || rr_mode > 2) {
    set_error("unknown rr mode %d", rr_mode);
    return 1;
  }
  return fsb::stochastic(tree->t, kid, alpha, dfloor, precision == 0, queries, n, qperm,
                         (int)n_samples, rr_mode, seed, query_offset, out, visited, path_steps,
                         path_count, S(stream));
}

int fsb_stochastic_batch_ex(fsb_tree* tree, int kid, double alpha, double dfloor, int precision,
                            const double* queries, int64_t n, const int32_t* order,
                            int64_t n_samples, int rr_mode, uint64_t seed, int64_t query_offset,
                            int group_log2, int flags, void* out, int64_t* visited,
                            int64_t* path_steps, int64_t* path_count, void* stream) {
  FSB_RANGE("fsb_stochastic_batch_ex");
  ABI_TREE(tree);
  if (int rc = check_common(kid, precision, n)) return rc;
  if (n_samples < 1 || n_samples > (1LL << 30) || rr_mode < 0 || rr_mode > 2 || group_log2 < 0 ||
      group_log2 > 20 || flags < 0 || flags > 3) {
    set_error("bad samples_per_subdomain / rr mode / group size / flags");
    return 1;
  }
  if ((flags & FSB_FLAG_SHUFFLED) && order) {
    set_error("FSB_FLAG_SHUFFLED computes the order itself: pass order = NULL");
    return 1;
  }
  return fsb::stochastic(tree->t, kid, alpha, dfloor, precision == 0, queries, n, order,
                         (int)n_samples, rr_mode, seed, query_offset, out, visited, path_steps,
                         path_count, S(stream), group_log2, flags);
}

int fsb_stochastic_moments_batch(fsb_tree* tree, int kid, double alpha, double dfloor,
                                 const double* queries, int64_t n, int64_t n_reps, int rr_mode,
                                 uint64_t seed, double* mean_out, double* var_out, void* stream) {
  FSB_RANGE("fsb_stochastic_moments_batch");
  ABI_TREE(tree);
  if (int rc = check_common(kid, 0, n)) return rc;
  if (n_reps < 1 || rr_mode < 0 || rr_mode > 2) {
    set_error("bad n_reps / rr_mode");
    return 1;
  }
  return fsb::stochastic_moments(tree->t, kid, alpha, dfloor, queries, n, n_reps, rr_mode, seed,
                                 mean_out, var_out, S(stream));
}

int fsb_telescoping_batch(fsb_tree* tree, int kid, double alpha, double dfloor, int precision,
                          const double* queries, int64_t n, void* out, int64_t* visited,
                          void* stream) {
  FSB_RANGE("fsb_telescoping_batch");
  ABI_TREE(tree);
  if (int rc = check_common(kid, precision, n)) return rc;
  return fsb::telescoping(tree->t, kid, alpha, dfloor, precision == 0, queries, n, out, visited,
                          S(stream));
}

int fsb_query_order(const double* queries, int64_t n, int32_t* perm_out, void* stream) {
  FSB_RANGE("fsb_query_order");
  if (n < 0) {
    set_error("negative query count");
    return 1;
  }
  return fsb::query_order(queries, n, perm_out, S(stream));
}

int fsb_shuffle_order(int64_t n, uint64_t seed, int64_t query_offset, int32_t* perm_out,
                      void* stream) {
  FSB_RANGE("fsb_shuffle_order");
  if (n < 0 || (n > 0 && !perm_out)) {
    set_error("bad shuffle arguments");
    return 1;
  }
  return fsb::shuffle_order(n, seed, query_offset, perm_out, S(stream));
}

int fsb_post_transform(const void* raw, int raw_is_f32, int64_t n, int smooth, double alpha,
                       double* values, double* raw64, uint8_t* flagged, void* stream) {
  FSB_RANGE("fsb_post_transform");
  if (n < 0) {
    set_error("negative count");
    return 1;
  }
  return fsb::post_transform(raw, raw_is_f32, n, smooth, alpha, values, raw64, flagged, S(stream));
}

}  // extern "C"
