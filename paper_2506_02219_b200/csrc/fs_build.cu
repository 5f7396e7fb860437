// fs_build.cu -- data-parallel GPU construction of the reference's uniform-cell tree.
//
// Reproduces build_tree (octree.py:118-239) bit for bit without recursion:
//   1. root cube from a bbox reduction (octree.py:133-136)
//   2. per-point digit keys from the reference's FP64 recurrence
//      floor((p - cell_min)/csize), clipped, cell_min += digit*csize
//      (octree.py:178-193), packed ceil(log2 d^3) bits per level, MSB first
//   3. stable multi-word LSD radix sort (== the chain of per-level stable
//      argsorts, octree.py:183-184, starting from arange)
//   4. L[b] = common digit prefix of sorted keys b, b+1 (capped at the depth cap)
//   5. position b opens one node per level in [L[b-1]+1, min(max(L[b-1],L[b])+1, D)];
//      numbering nodes by (begin, depth) is the reference's DFS preorder
//   6. node end = first b' > b whose key shares < depth digits (exponential search)
//   7. level order (sorted by depth, begin) makes every child list contiguous
//   8. bottom-up FP64 aggregates, one launch per level, children in order
//      with explicit _rn intrinsics (octree.py:196-205); depth-capped leaves use
//      numpy's pairwise summation order (octree.py:170-176)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "fs_common.cuh"
#include "fs_internal.h"

namespace fsb {

constexpr double kSqrt3 = 1.7320508075688772;  // math.sqrt(3.0), octree.py:225
constexpr int kMaxChannels = 8;

// ---------------------------------------------------------------- bbox
__global__ void k_bbox(const double* __restrict__ pos, int64_t m, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double v = pos[3 * i + k];
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
  }
  __shared__ double sm[6][256];
  for (int k = 0; k < 3; ++k) {
    sm[k][threadIdx.x] = lo[k];
    sm[3 + k][threadIdx.x] = hi[k];
  }
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 3; ++k) {
        sm[k][threadIdx.x] = fmin(sm[k][threadIdx.x], sm[k][threadIdx.x + st]);
        sm[3 + k][threadIdx.x] = fmax(sm[3 + k][threadIdx.x], sm[3 + k][threadIdx.x + st]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sm[threadIdx.x][0];
}

// the per-block extents reduced by one 256-thread block (min / max are exact
// and order-free, so any reduction order gives the same bits)
__global__ void k_bbox_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  double r[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      r[k] = fmin(r[k], part[b * 6 + k]);
      r[3 + k] = fmax(r[3 + k], part[b * 6 + 3 + k]);
    }
  __shared__ double sm[6][256];
  for (int k = 0; k < 6; ++k) sm[k][threadIdx.x] = r[k];
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 3; ++k) {
        sm[k][threadIdx.x] = fmin(sm[k][threadIdx.x], sm[k][threadIdx.x + st]);
        sm[3 + k][threadIdx.x] = fmax(sm[3 + k][threadIdx.x], sm[3 + k][threadIdx.x + st]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) out[threadIdx.x] = sm[threadIdx.x][0];
}

// numpy float64 -> int64 cast on x86 (cvttsd2si): NaN / out of range -> INT64_MIN
__device__ __forceinline__ int64_t cast_i64(double f) {
  if (!(f >= -9.2233720368547758e18 && f < 9.2233720368547758e18)) return INT64_MIN;
  return (int64_t)f;
}

struct Geo {
  double rmin[3];
  int d, D, bpl, dpw, W;
};

// one digit of the recurrence (octree.py:179-182, 193)
__device__ __forceinline__ int digit_step(const double p[3], double cmin[3], double cs, int d) {
  int64_t r[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // (the branch-free division fast path measured slower here: 5.27 vs 4.95 ms)
    int64_t v = cast_i64(floor(__ddiv_rn(__dsub_rn(p[k], cmin[k]), cs)));
    v = v < 0 ? 0 : v;
    v = v > d - 1 ? d - 1 : v;
    r[k] = v;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) cmin[k] = __dadd_rn(cmin[k], __dmul_rn((double)r[k], cs));
  return (int)((r[0] * d + r[1]) * d + r[2]);
}

// the digit key words of point i over levels [0, levels) (word w at keys[w m + i])
__device__ __forceinline__ void point_key(const double* __restrict__ pos, int64_t m, int64_t i,
                                          const double* __restrict__ csz, const Geo& g,
                                          int levels, uint64_t* __restrict__ keys) {
  double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  double cmin[3] = {g.rmin[0], g.rmin[1], g.rmin[2]};
  uint64_t word = 0;
  int w = 0, t = 0;
  for (int l = 0; l < levels; ++l) {
    uint64_t dig = (uint64_t)digit_step(p, cmin, csz[l], g.d);
    word |= dig << (64 - (t + 1) * g.bpl);
    if (++t == g.dpw) {
      keys[w * m + i] = word;
      ++w;
      word = 0;
      t = 0;
    }
  }
  if (t > 0) keys[w * m + i] = word;
}

// every point's key over the first `levels` levels (the first word, or all D)
__global__ void k_keys(const double* __restrict__ pos, int64_t m, const double* __restrict__ csz,
                       Geo g, int levels, uint64_t* __restrict__ keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) point_key(pos, m, i, csz, g, levels, keys);
}

// the full key (all D levels) of the points whose first word ties with a
// neighbour's in the first-word order: the only keys whose deeper words the
// tie refinement, the LCPs and the node ends ever compare
__global__ void k_keys_tied(const double* __restrict__ pos, int64_t m,
                            const double* __restrict__ csz, Geo g,
                            const uint64_t* __restrict__ w0s, const int32_t* __restrict__ perm,
                            uint64_t* __restrict__ keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = w0s[i];
  const bool tied = (i > 0 && w0s[i - 1] == k) || (i + 1 < m && w0s[i + 1] == k);
  if (tied) point_key(pos, m, perm[i], csz, g, g.D, keys);
}

__global__ void k_gather_key(const uint64_t* __restrict__ kw, const int32_t* __restrict__ perm,
                             int64_t m, uint64_t* __restrict__ out) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < m) out[b] = kw[perm[b]];
}
// the same for the sorted positions whose first word ties with a neighbour's
// (the others are never read: 0)
__global__ void k_gather_key_tied(const uint64_t* __restrict__ kw, const int32_t* __restrict__ perm,
                                  const uint64_t* __restrict__ w0s, int64_t m,
                                  uint64_t* __restrict__ out) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= m) return;
  const uint64_t k = w0s[b];
  const bool tied = (b > 0 && w0s[b - 1] == k) || (b + 1 < m && w0s[b + 1] == k);
  out[b] = tied ? kw[perm[b]] : 0ull;
}

// Runs of equal first key words after the stable sort by word 0: each run's
// permutation is insertion-sorted (stable) by the remaining words, which gives
// the full multi-word stable order.  A run longer than kMaxTieRun (duplicate-
// heavy inputs) sets *overflow and the caller runs the full LSD sort instead.
constexpr int kMaxTieRun = 64;
#ifndef FSB_GEOM_FROM_KEYS
#define FSB_GEOM_FROM_KEYS 1  // node cell mins from the sorted keys' digits (no divisions)
#endif
#ifndef FSB_LEVEL_SORT_FULL
#define FSB_LEVEL_SORT_FULL 0  // 1: the level-order sort over (depth, begin) bits
#endif
#ifndef FSB_BUILD_FULL_SORT
#define FSB_BUILD_FULL_SORT 0  // 1: always the full multi-word LSD sort
#endif
__global__ void k_refine_ties(const uint64_t* __restrict__ w0s, const uint64_t* __restrict__ keys,
                              int W, int64_t m, int32_t* __restrict__ perm,
                              int* __restrict__ overflow) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i + 1 >= m) return;
  const uint64_t k = w0s[i];
  if (w0s[i + 1] != k || (i > 0 && w0s[i - 1] == k)) return;  // not the start of a run
  int64_t j = i + 2;
  while (j < m && w0s[j] == k) {
    if (j - i >= kMaxTieRun) {
      atomicExch(overflow, 1);
      return;
    }
    ++j;
  }
  auto less = [&](int32_t a, int32_t b) {  // words 1 .. W-1 (ties: keep the stable order)
    for (int w = 1; w < W; ++w) {
      const uint64_t x = keys[(int64_t)w * m + a], y = keys[(int64_t)w * m + b];
      if (x != y) return x < y;
    }
    return false;
  };
  for (int64_t a = i + 1; a < j; ++a) {
    const int32_t v = perm[a];
    int64_t b = a;
    while (b > i && less(v, perm[b - 1])) {
      perm[b] = perm[b - 1];
      --b;
    }
    perm[b] = v;
  }
}

__global__ void k_iota(int32_t* __restrict__ a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

__device__ __forceinline__ int lcp_keys(const uint64_t* __restrict__ sk, int64_t m, const Geo& g,
                                        int64_t a, int64_t b) {
  for (int w = 0; w < g.W; ++w) {
    uint64_t x = sk[w * m + a] ^ sk[w * m + b];
    if (x) {
      int l = w * g.dpw + __clzll((long long)x) / g.bpl;
      return l < g.D ? l : g.D;
    }
  }
  return g.D;
}

__global__ void k_lcp(const uint64_t* __restrict__ sk, int64_t m, Geo g, int32_t* __restrict__ L) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < m - 1) L[b] = lcp_keys(sk, m, g, b, b + 1);
}

__device__ __forceinline__ void level_span(const int32_t* __restrict__ L, int64_t m, int D,
                                           int64_t b, int& s, int& e) {
  int lp = b == 0 ? -1 : L[b - 1];
  int ln = b == m - 1 ? -1 : L[b];
  s = lp + 1;
  e = min(max(lp, ln) + 1, D);
}

__global__ void k_count(const int32_t* __restrict__ L, int64_t m, int D, int32_t* __restrict__ cnt) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= m) return;
  int s, e;
  level_span(L, m, D, b, s, e);
  cnt[b] = e >= s ? e - s + 1 : 0;
}

__global__ void k_emit(const int32_t* __restrict__ L, const int32_t* __restrict__ off, int64_t m,
                       int D, int32_t* __restrict__ nb, int32_t* __restrict__ nd) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= m) return;
  int s, e;
  level_span(L, m, D, b, s, e);
  for (int l = s; l <= e; ++l) {
    int32_t id = off[b] + (l - s);
    nb[id] = (int32_t)b;
    nd[id] = l;
  }
}

__global__ void k_level_starts(const uint64_t* __restrict__ lkey_sorted, int64_t n,
                               int64_t* __restrict__ lstart) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int dep = (int)(lkey_sorted[r] >> 32);
  if (r == 0 || (int)(lkey_sorted[r - 1] >> 32) != dep) lstart[dep] = r;
}

__global__ void k_invert(const int32_t* __restrict__ lo2pre, int64_t n, int32_t* __restrict__ pre2lo) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) pre2lo[lo2pre[r]] = (int32_t)r;
}

// node end: first b' > b whose key shares fewer than `depth` digits with key b
__global__ void k_end(const uint64_t* __restrict__ sk, int64_t m, Geo g,
                      const int32_t* __restrict__ nb, const int32_t* __restrict__ nd, int64_t n,
                      int64_t* __restrict__ end_out) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= n) return;
  int64_t b = nb[id];
  int l = nd[id];
  int64_t e;
  if (l == 0) {
    e = m;
  } else {
    int64_t lo = b, step = 1;
    while (b + step < m && lcp_keys(sk, m, g, b, b + step) >= l) {
      lo = b + step;
      step <<= 1;
    }
    int64_t hi = min(b + step, m);
    while (hi - lo > 1) {
      int64_t mid = lo + (hi - lo) / 2;
      if (lcp_keys(sk, m, g, b, mid) >= l)
        lo = mid;
      else
        hi = mid;
    }
    e = hi;
  }
  end_out[id] = e;
}

// children of internal nodes are contiguous in level order
__global__ void k_children(const int32_t* __restrict__ nb, const int32_t* __restrict__ nd,
                           const int64_t* __restrict__ nend, const int32_t* __restrict__ lo2pre,
                           const int32_t* __restrict__ pre2lo, const int64_t* __restrict__ lstart,
                           int num_levels, int64_t n, int D, int64_t* __restrict__ cc_out,
                           int32_t* __restrict__ fc_out) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= n) return;
  int64_t b = nb[id], e = nend[id];
  int l = nd[id];
  if (e - b < 2 || l >= D) {
    cc_out[id] = 0;
    fc_out[id] = 0;
    return;
  }
  int64_t r1 = pre2lo[id + 1];
  int64_t le = (l + 2 <= num_levels - 1) ? lstart[l + 2] : n;
  // first r in [r1, le) with begin >= e; child count <= d^3
  int64_t lo = r1, step = 1;
  while (lo + step < le && nb[lo2pre[lo + step]] < e) {
    lo += step;
    step <<= 1;
  }
  int64_t hi = min(lo + step, le);
  while (hi - lo > 1) {
    int64_t mid = lo + (hi - lo) / 2;
    if (nb[lo2pre[mid]] < e)
      lo = mid;
    else
      hi = mid;
  }
  cc_out[id] = hi - r1;
  fc_out[id] = (int32_t)r1;
}

__global__ void k_child_index(const int64_t* __restrict__ cc, const int64_t* __restrict__ cs,
                              const int32_t* __restrict__ fc, const int32_t* __restrict__ lo2pre,
                              int64_t n, int64_t* __restrict__ child_index) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= n) return;
  int64_t k = cc[id], s = cs[id];
  int32_t f = fc[id];
  for (int64_t t = 0; t < k; ++t) child_index[s + t] = lo2pre[f + t];
}

__global__ void k_permute(const double* __restrict__ pos, const double* __restrict__ ms,
                          const double* __restrict__ w, const int32_t* __restrict__ perm, int64_t m,
                          int c, double* __restrict__ pts, double* __restrict__ msp,
                          double* __restrict__ wp, int64_t* __restrict__ perm64) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= m) return;
  int64_t j = perm[b];
  for (int k = 0; k < 3; ++k) pts[3 * b + k] = pos[3 * j + k];
  for (int k = 0; k < c; ++k) msp[(int64_t)c * b + k] = ms[(int64_t)c * j + k];
  wp[b] = w[j];
  perm64[b] = j;
}

__global__ void k_node_geom(const int32_t* __restrict__ nb, const int32_t* __restrict__ nd,
                            const int64_t* __restrict__ nend, const double* __restrict__ pts,
                            const uint64_t* __restrict__ sk,
                            const double* __restrict__ csz, const double* __restrict__ sides,
                            Geo g, int64_t n, const int32_t* __restrict__ off, int64_t m,
                            double* __restrict__ bmin, double* __restrict__ bmax,
                            double* __restrict__ diam, int64_t* __restrict__ begin64,
                            int64_t* __restrict__ end64, int64_t* __restrict__ depth64,
                            int32_t* __restrict__ skip) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= n) return;
  int64_t b = nb[id], e = nend[id];
  int l = nd[id];
  double cmin[3] = {g.rmin[0], g.rmin[1], g.rmin[2]};
#if FSB_GEOM_FROM_KEYS
  // the cell-min recurrence (octree.py:193) from the node's first point's key
  // digits, which k_keys computed with the same recurrence: the same additions,
  // without re-deriving each digit by division.  (A node deeper than the first
  // key word has >= 2 points sharing that word, so its first point's deeper
  // words were computed: k_keys_tied.)
  (void)pts;
  const uint64_t mask = (1ull << g.bpl) - 1ull;
  for (int k = 0; k < l; ++k) {
    const int w = k / g.dpw, tt = k - w * g.dpw;
    const int dig = (int)((sk[(int64_t)w * m + b] >> (64 - (tt + 1) * g.bpl)) & mask);
    const int r[3] = {dig / (g.d * g.d), (dig / g.d) % g.d, dig % g.d};
    const double cs = csz[k];
#pragma unroll
    for (int kk = 0; kk < 3; ++kk) cmin[kk] = __dadd_rn(cmin[kk], __dmul_rn((double)r[kk], cs));
  }
#else
  (void)sk;
  double p[3] = {pts[3 * b], pts[3 * b + 1], pts[3 * b + 2]};
  for (int k = 0; k < l; ++k) digit_step(p, cmin, csz[k], g.d);
#endif
  double side = sides[l];
  for (int k = 0; k < 3; ++k) {
    bmin[3 * id + k] = cmin[k];
    bmax[3 * id + k] = __dadd_rn(cmin[k], side);
  }
  diam[id] = __dmul_rn(side, kSqrt3);
  begin64[id] = b;
  end64[id] = e;
  depth64[id] = l;
  skip[id] = e < m ? off[e] : (int32_t)n;  // next preorder node outside the subtree
}

// numpy's pairwise add-reduction (1-D / (n,1) float64 sums), see oracle
__device__ __noinline__ double np_pairwise(const double* a, int64_t n, int64_t stride) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int k = 0; k < 8; ++k) r[k] = a[k * stride];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[(i + k) * stride]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2, stride), np_pairwise(a + n2 * stride, n - n2, stride));
}

// bottom-up aggregates for one level (octree.py:161-176, 196-205)
__global__ void k_aggregate(int64_t r0, int64_t r1, const int32_t* __restrict__ lo2pre,
                            const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                            const int64_t* __restrict__ cc, const int32_t* __restrict__ fc,
                            const double* __restrict__ pts, const double* __restrict__ msp,
                            const double* __restrict__ wp, int c, double* __restrict__ am,
                            double* __restrict__ aw, double* __restrict__ com,
                            double* __restrict__ lam, double* __restrict__ law,
                            double* __restrict__ lcom) {
  // (am, aw, com: preorder, the tree's arrays; lam, law, lcom: the same values in
  // level order, where a node's children are contiguous, so the children's
  // aggregates are read sequentially rather than gathered through lo2pre)
  int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= r1) return;
  int64_t id = lo2pre[r];
  int64_t b = begin[id], e = end[id], k_n = cc[id];
  if (e - b == 1) {  // verbatim copy, octree.py:161-168
    for (int k = 0; k < c; ++k)
      am[(int64_t)c * id + k] = lam[(int64_t)c * r + k] = msp[(int64_t)c * b + k];
    aw[id] = law[r] = wp[b];
    for (int k = 0; k < 3; ++k) com[3 * id + k] = lcom[3 * r + k] = pts[3 * b + k];
    return;
  }
  if (k_n == 0) {  // depth-capped / zero-side multi-point leaf, octree.py:169-176
    int64_t n = e - b;
    double wsum = __dadd_rn(0.0, np_pairwise(wp + b, n, 1));
    for (int k = 0; k < c; ++k) {
      double acc;
      if (c == 1) {
        acc = __dadd_rn(0.0, np_pairwise(msp + b, n, 1));
      } else {
        acc = 0.0;
        for (int64_t i = b; i < e; ++i) acc = __dadd_rn(acc, msp[(int64_t)c * i + k]);
      }
      am[(int64_t)c * id + k] = lam[(int64_t)c * r + k] = acc;
    }
    aw[id] = law[r] = wsum;
    for (int k = 0; k < 3; ++k) {
      double acc = 0.0;
      for (int64_t i = b; i < e; ++i) acc = __dadd_rn(acc, __dmul_rn(wp[i], pts[3 * i + k]));
      com[3 * id + k] = lcom[3 * r + k] = __ddiv_rn(acc, wsum);
    }
    return;
  }
  double w = 0.0, wc[3] = {0.0, 0.0, 0.0}, ms[kMaxChannels];
  for (int k = 0; k < c; ++k) ms[k] = 0.0;
  const int64_t f = fc[id];  // first child, level order
  for (int64_t t = 0; t < k_n; ++t) {
    const int64_t k2 = f + t;
    double wk = law[k2];
    w = __dadd_rn(w, wk);
    for (int k = 0; k < c; ++k) ms[k] = __dadd_rn(ms[k], lam[(int64_t)c * k2 + k]);
    for (int k = 0; k < 3; ++k) wc[k] = __dadd_rn(wc[k], __dmul_rn(wk, lcom[3 * k2 + k]));
  }
  for (int k = 0; k < c; ++k) am[(int64_t)c * id + k] = lam[(int64_t)c * r + k] = ms[k];
  aw[id] = law[r] = w;
  for (int k = 0; k < 3; ++k) com[3 * id + k] = lcom[3 * r + k] = __ddiv_rn(wc[k], w);
}

// ------------------------------------------------------------ host helpers
template <class T>
// tree arrays come from the stream-ordered pool (retained across builds, see
// retain_pool_memory): a C4 tree is ~1 GB in ~40 arrays, and cudaMalloc would
// map (and cudaFree synchronise) every one of them on every build
static int dalloc(T** p, int64_t count, cudaStream_t s) {
  size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
  retain_pool_memory();
  FS_CK(cudaMallocAsync((void**)p, bytes, s));
  return 0;
}

static int scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  FS_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, s));
  Scratch t;
  FS_TRY(t.alloc(tb, s));
  FS_CK(cub::DeviceScan::ExclusiveSum(t.p, tb, in, out, (int)n, s));
  return 0;
}
static int scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  FS_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, s));
  Scratch t;
  FS_TRY(t.alloc(tb, s));
  FS_CK(cub::DeviceScan::ExclusiveSum(t.p, tb, in, out, (int)n, s));
  return 0;
}
static int sort_pairs_u64(const uint64_t* kin, uint64_t* kout, const int32_t* vin, int32_t* vout,
                          int64_t n, int bb, int eb, cudaStream_t s) {
  size_t tb = 0;
  FS_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, (int)n, bb, eb, s));
  Scratch t;
  FS_TRY(t.alloc(tb, s));
  FS_CK(cub::DeviceRadixSort::SortPairs(t.p, tb, kin, kout, vin, vout, (int)n, bb, eb, s));
  return 0;
}

static int bits_for(int64_t v) {  // bits to represent values 0..v
  int b = 0;
  while ((int64_t(1) << b) <= v) ++b;
  return std::max(b, 1);
}

__global__ void k_make_lkey(const int32_t* __restrict__ nb, const int32_t* __restrict__ nd,
                            int64_t n, uint64_t* __restrict__ lk) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) lk[i] = ((uint64_t)(uint32_t)nd[i] << 32) | (uint32_t)nb[i];
}

// Level order = nodes sorted by (depth, begin): every child list is a contiguous
// run and every level a contiguous segment.  Fills lo2pre / pre2lo / level_off and
// returns a device copy of level_off in *lstart_dev (caller frees).
int level_order(FsTree* t, const int32_t* nb, const int32_t* nd, int max_dep,
                int64_t** lstart_dev, cudaStream_t s) {
  int64_t n = t->n;
  const int B = 256;
  Scratch lkey, lkey_s, ids;
  FS_TRY(lkey.alloc(sizeof(uint64_t) * n, s));
  FS_TRY(lkey_s.alloc(sizeof(uint64_t) * n, s));
  FS_TRY(ids.alloc(sizeof(int32_t) * n, s));
  k_iota<<<grid_for(n, B), B, 0, s>>>(ids.as<int32_t>(), n);
  k_make_lkey<<<grid_for(n, B), B, 0, s>>>(nb, nd, n, lkey.as<uint64_t>());
  // Preorder ids of one depth already increase with begin (the nodes are emitted
  // point by point), so a stable sort on the depth bits alone gives the
  // (depth, begin) order: one radix pass instead of one per 8 key bits.
  FS_TRY(sort_pairs_u64(lkey.as<uint64_t>(), lkey_s.as<uint64_t>(), ids.as<int32_t>(), t->lo2pre,
                        n, FSB_LEVEL_SORT_FULL ? 0 : 32, 32 + bits_for(max_dep), s));
  uint64_t lastkey = 0;
  FS_CK(cudaMemcpyAsync(&lastkey, lkey_s.as<uint64_t>() + (n - 1), 8, cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  int nl = (int)(lastkey >> 32) + 1;
  retain_pool_memory();
  FS_CK(cudaMallocAsync((void**)lstart_dev, sizeof(int64_t) * (nl + 1), s));
  k_level_starts<<<grid_for(n, B), B, 0, s>>>(lkey_s.as<uint64_t>(), n, *lstart_dev);
  k_invert<<<grid_for(n, B), B, 0, s>>>(t->lo2pre, n, t->pre2lo);
  t->level_off.assign(nl + 1, n);
  FS_CK(cudaMemcpyAsync(t->level_off.data(), *lstart_dev, sizeof(int64_t) * nl,
                        cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  t->level_off[nl] = n;
  t->num_levels = nl;
  FS_CK(cudaMemcpyAsync(*lstart_dev + nl, &t->level_off[nl], sizeof(int64_t),
                        cudaMemcpyHostToDevice, s));
  FS_CK(cudaStreamSynchronize(s));
  return 0;
}

static int alloc_export(FsTree* t, cudaStream_t s) {
  int64_t n = t->n, m = t->m;
  int c = t->c;
  FS_TRY(dalloc(&t->bbox_min, 3 * n, s));
  FS_TRY(dalloc(&t->bbox_max, 3 * n, s));
  FS_TRY(dalloc(&t->diameter, n, s));
  FS_TRY(dalloc(&t->agg_mass, (int64_t)c * n, s));
  FS_TRY(dalloc(&t->agg_weight, n, s));
  FS_TRY(dalloc(&t->com, 3 * n, s));
  FS_TRY(dalloc(&t->child_start, n, s));
  FS_TRY(dalloc(&t->child_count, n, s));
  FS_TRY(dalloc(&t->child_index, n - 1, s));
  FS_TRY(dalloc(&t->begin, n, s));
  FS_TRY(dalloc(&t->end, n, s));
  FS_TRY(dalloc(&t->depth, n, s));
  FS_TRY(dalloc(&t->perm, m, s));
  FS_TRY(dalloc(&t->points, 3 * m, s));
  FS_TRY(dalloc(&t->masses, (int64_t)c * m, s));
  FS_TRY(dalloc(&t->weights, m, s));
  FS_TRY(dalloc(&t->lo2pre, n, s));
  FS_TRY(dalloc(&t->pre2lo, n, s));
  FS_TRY(dalloc(&t->skip, n, s));
  FS_TRY(dalloc(&t->fc_lo, n, s));
  t->owns_export = true;
  return 0;
}

int build_tree(FsTree** out, const double* pos, const double* masses, const double* weights,
               int64_t m, int c, int d, int max_depth, cudaStream_t s) {
  *out = nullptr;
  if (m < 1 || d < 2 || max_depth < 1 || c < 1 || c > kMaxChannels) {
    set_error("build_tree: bad arguments (m=%lld c=%d d=%d max_depth=%d)", (long long)m, c, d,
              max_depth);
    return 1;
  }
  if (m >= (int64_t(1) << 31) - 2) {
    set_error("build_tree: more than 2^31 points is not supported");
    return 1;
  }
  const int B = 256;
  // -------- 1. root cube (octree.py:133-136)
  double bb[6];
  {
    int nb = (int)std::min<int64_t>(1024, (m + B - 1) / B);
    Scratch part, res;
    FS_TRY(part.alloc(sizeof(double) * 6 * nb, s));
    FS_TRY(res.alloc(sizeof(double) * 6, s));
    k_bbox<<<nb, B, 0, s>>>(pos, m, part.as<double>());
    k_bbox_final<<<1, 256, 0, s>>>(part.as<double>(), nb, res.as<double>());
    FS_CK(cudaMemcpyAsync(bb, res.p, sizeof(bb), cudaMemcpyDeviceToHost, s));
    FS_CK(cudaStreamSynchronize(s));
  }
  double side = bb[3] - bb[0];
  for (int k = 1; k < 3; ++k) side = std::max(side, bb[3 + k] - bb[k]);
  Geo g;
  for (int k = 0; k < 3; ++k) g.rmin[k] = (bb[k] + bb[3 + k]) / 2.0 - side / 2.0;
  // a node at depth k is subdivided iff k < max_depth and side_k != 0 (octree.py:169)
  std::vector<double> sides{side};
  int D = 0;
  while (D < max_depth && sides[D] != 0.0) {
    sides.push_back(sides[D] / (double)d);
    ++D;
  }
  g.d = d;
  g.D = D;
  g.bpl = bits_for((int64_t)d * d * d - 1);
  if (g.bpl > 32) {
    set_error("build_tree: branching_per_dim too large");
    return 1;
  }
  g.dpw = 64 / g.bpl;
  g.W = std::max(1, (D + g.dpw - 1) / g.dpw);

  FsTree* t = new FsTree();
  t->m = m;
  t->c = c;
  t->d = d;
  t->max_depth = max_depth;
  t->d_eff = D;

  Scratch dsides, dcsz;
  FS_TRY(dsides.alloc(sizeof(double) * sides.size(), s));
  FS_TRY(dcsz.alloc(sizeof(double) * std::max<size_t>(1, sides.size() - 1), s));
  FS_CK(cudaMemcpyAsync(dsides.p, sides.data(), sizeof(double) * sides.size(),
                        cudaMemcpyHostToDevice, s));
  if (sides.size() > 1)
    FS_CK(cudaMemcpyAsync(dcsz.p, sides.data() + 1, sizeof(double) * (sides.size() - 1),
                          cudaMemcpyHostToDevice, s));

  // -------- 2-3. keys + stable LSD multi-word sort
  Scratch keys, perm_a, perm_b, kw, kw_s, skeys;
  const int W = g.W;
  FS_TRY(keys.alloc(sizeof(uint64_t) * W * m, s));
  FS_TRY(perm_a.alloc(sizeof(int32_t) * m, s));
  FS_TRY(perm_b.alloc(sizeof(int32_t) * m, s));
  FS_TRY(kw.alloc(sizeof(uint64_t) * m, s));
  FS_TRY(kw_s.alloc(sizeof(uint64_t) * m, s));
  FS_TRY(skeys.alloc(sizeof(uint64_t) * W * m, s));
  int32_t* perm = perm_a.as<int32_t>();
  int32_t* perm2 = perm_b.as<int32_t>();
  k_iota<<<grid_for(m, B), B, 0, s>>>(perm, m);
  if (D > 0) {
    FS_CK(cudaMemsetAsync(keys.p, 0, sizeof(uint64_t) * W * m, s));
    // stable sort by the first word (the top levels), then the short runs of equal
    // first words refined by the remaining words; the full stable LSD sort over
    // every word (one radix pass group per word) only when some run is long.
    // Only the tied points need their deeper words (k_keys_tied).
    bool full = W > 1 && FSB_BUILD_FULL_SORT;
    const int lv0 = full ? D : std::min(g.dpw, D);
    k_keys<<<grid_for(m, 128), 128, 0, s>>>(pos, m, dcsz.as<double>(), g, lv0,
                                            keys.as<uint64_t>());
    if (!full) {
      const int used0 = std::min(g.dpw, D) * g.bpl;
      FS_TRY(sort_pairs_u64(keys.as<uint64_t>(), kw_s.as<uint64_t>(), perm, perm2, m, 64 - used0,
                            64, s));
      std::swap(perm, perm2);
      if (W > 1 && m > 1) {
        Scratch ovf;
        FS_TRY(ovf.alloc(sizeof(int), s));
        FS_CK(cudaMemsetAsync(ovf.p, 0, sizeof(int), s));
        k_keys_tied<<<grid_for(m, 128), 128, 0, s>>>(pos, m, dcsz.as<double>(), g,
                                                     kw_s.as<uint64_t>(), perm,
                                                     keys.as<uint64_t>());
        k_refine_ties<<<grid_for(m, B), B, 0, s>>>(kw_s.as<uint64_t>(), keys.as<uint64_t>(), W, m,
                                                   perm, ovf.as<int>());
        int over = 0;
        FS_CK(cudaMemcpyAsync(&over, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        FS_CK(cudaStreamSynchronize(s));
        if (over) {  // every point's full key, then the multi-word LSD sort
          full = true;
          k_iota<<<grid_for(m, B), B, 0, s>>>(perm, m);
          k_keys<<<grid_for(m, 128), 128, 0, s>>>(pos, m, dcsz.as<double>(), g, D,
                                                  keys.as<uint64_t>());
        }
      }
    }
    if (full) {
      for (int w = W - 1; w >= 0; --w) {
        int digits = std::min(g.dpw, D - w * g.dpw);
        int used = digits * g.bpl;
        k_gather_key<<<grid_for(m, B), B, 0, s>>>(keys.as<uint64_t>() + (int64_t)w * m, perm, m,
                                                  kw.as<uint64_t>());
        FS_TRY(sort_pairs_u64(kw.as<uint64_t>(), kw_s.as<uint64_t>(), perm, perm2, m, 64 - used,
                              64, s));
        std::swap(perm, perm2);
      }
    }
    if (full) {
      for (int w = 0; w < W; ++w)
        k_gather_key<<<grid_for(m, B), B, 0, s>>>(keys.as<uint64_t>() + (int64_t)w * m, perm, m,
                                                  skeys.as<uint64_t>() + (int64_t)w * m);
    } else {
      // the sorted first words are kw_s (the refinement only permutes within runs
      // of equal first words); the deeper words are gathered for tied points only,
      // the only ones whose deeper words are ever compared
      FS_CK(cudaMemcpyAsync(skeys.p, kw_s.p, sizeof(uint64_t) * m, cudaMemcpyDeviceToDevice, s));
      for (int w = 1; w < W; ++w)
        k_gather_key_tied<<<grid_for(m, B), B, 0, s>>>(keys.as<uint64_t>() + (int64_t)w * m, perm,
                                                       kw_s.as<uint64_t>(), m,
                                                       skeys.as<uint64_t>() + (int64_t)w * m);
    }
  } else {
    FS_CK(cudaMemsetAsync(skeys.p, 0, sizeof(uint64_t) * W * m, s));
  }

  // -------- 4-5. LCP, node counts, preorder ids
  Scratch Ls, cnt, off;
  FS_TRY(Ls.alloc(sizeof(int32_t) * m, s));
  FS_TRY(cnt.alloc(sizeof(int32_t) * m, s));
  FS_TRY(off.alloc(sizeof(int32_t) * (m + 1), s));
  if (m > 1) k_lcp<<<grid_for(m - 1, B), B, 0, s>>>(skeys.as<uint64_t>(), m, g, Ls.as<int32_t>());
  k_count<<<grid_for(m, B), B, 0, s>>>(Ls.as<int32_t>(), m, D, cnt.as<int32_t>());
  FS_TRY(scan_i32(cnt.as<int32_t>(), off.as<int32_t>(), m, s));
  int32_t last_off = 0, last_cnt = 0;
  FS_CK(cudaMemcpyAsync(&last_off, off.as<int32_t>() + (m - 1), 4, cudaMemcpyDeviceToHost, s));
  FS_CK(cudaMemcpyAsync(&last_cnt, cnt.as<int32_t>() + (m - 1), 4, cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  int64_t n = (int64_t)last_off + last_cnt;
  t->n = n;
  {
    int rc = alloc_export(t, s);
    if (rc) {
      free_tree(t);
      return rc;
    }
  }

  Scratch nbuf, dbuf;
  FS_TRY(nbuf.alloc(sizeof(int32_t) * n, s));
  FS_TRY(dbuf.alloc(sizeof(int32_t) * n, s));
  int32_t* nb = nbuf.as<int32_t>();
  int32_t* nd = dbuf.as<int32_t>();
  k_emit<<<grid_for(m, B), B, 0, s>>>(Ls.as<int32_t>(), off.as<int32_t>(), m, D, nb, nd);
  int64_t* lstart = nullptr;
  {
    int rc = level_order(t, nb, nd, D, &lstart, s);
    if (rc) {
      free_tree(t);
      return rc;
    }
  }
  // -------- 6. ends, children, CSR
  k_end<<<grid_for(n, 128), 128, 0, s>>>(skeys.as<uint64_t>(), m, g, nb, nd, n, t->end);
  k_children<<<grid_for(n, B), B, 0, s>>>(nb, nd, t->end, t->lo2pre, t->pre2lo, lstart,
                                          t->num_levels, n, D, t->child_count, t->fc_lo);
  FS_TRY(scan_i64(t->child_count, t->child_start, n, s));
  k_child_index<<<grid_for(n, B), B, 0, s>>>(t->child_count, t->child_start, t->fc_lo, t->lo2pre,
                                             n, t->child_index);
  // -------- permuted point arrays
  k_permute<<<grid_for(m, B), B, 0, s>>>(pos, masses, weights, perm, m, c, t->points, t->masses,
                                         t->weights, t->perm);
  // -------- geometry, skip links
  k_node_geom<<<grid_for(n, 128), 128, 0, s>>>(nb, nd, t->end, t->points, skeys.as<uint64_t>(),
                                               dcsz.as<double>(),
                                               dsides.as<double>(), g, n, off.as<int32_t>(), m,
                                               t->bbox_min, t->bbox_max, t->diameter, t->begin,
                                               t->end, t->depth, t->skip);
  // -------- 8. aggregates, deepest level first (level-order copies as scratch)
  Scratch lam, law, lcom;
  FS_TRY(lam.alloc(sizeof(double) * (size_t)c * n, s));
  FS_TRY(law.alloc(sizeof(double) * (size_t)n, s));
  FS_TRY(lcom.alloc(sizeof(double) * 3 * (size_t)n, s));
  for (int l = t->num_levels - 1; l >= 0; --l) {
    int64_t r0 = t->level_off[l], r1 = t->level_off[l + 1];
    if (r1 <= r0) continue;
    k_aggregate<<<grid_for(r1 - r0, 128), 128, 0, s>>>(
        r0, r1, t->lo2pre, t->begin, t->end, t->child_count, t->fc_lo, t->points, t->masses,
        t->weights, c, t->agg_mass, t->agg_weight, t->com, lam.as<double>(), law.as<double>(),
        lcom.as<double>());
  }
  FS_CK(cudaGetLastError());
  int64_t rk = 0;
  FS_CK(cudaMemcpyAsync(&rk, t->child_count, 8, cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  FS_CK(cudaFreeAsync(lstart, s));
  t->root_kids = (int)rk;
  *out = t;
  return 0;
}

}  // namespace fsb
