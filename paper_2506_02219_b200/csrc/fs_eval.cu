// fs_eval.cu -- the evaluators: brute force, Barnes-Hut, stochastic, moments, telescoping.
//
// F64 = parity flavour (bitwise with the reference's numba cores for coulomb and
// winding); F32 = FP32 inputs/terms with FP64 accumulation (the reference's
// precision="f32" contract, estimators.py:270-298), MUFU fast math for terms.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <type_traits>

#include "fs_common.cuh"
#include "fs_eval.h"
#include "fs_internal.h"

namespace fsb {

template <bool F64>
struct Prec;
template <>
struct Prec<true> {
  using T = double;
  using V4 = double4;
  using Out = double;
};
template <>
struct Prec<false> {
  using T = float;
  using V4 = float4;
  using Out = float;
};

__device__ __forceinline__ void load_query(const double* __restrict__ q, int64_t qi, double& x,
                                           double& y, double& z) {
  x = q[3 * qi];
  y = q[3 * qi + 1];
  z = q[3 * qi + 2];
}

#ifndef FSB_F64_TERM_FAST
#define FSB_F64_TERM_FAST 1  // FP64 terms through the branch-free fast paths (same bits)
#endif
// FP64 term through the branch-free IEEE fast paths (bit-identical whenever
// they apply, else the intrinsic sequence)
template <int KID>
__device__ __forceinline__ double term_parity(double m0, double m1, double m2, double px,
                                              double py, double pz, double qx, double qy,
                                              double qz, const KParams& kp) {
  if constexpr (KID == KID_SMOOTH) {
    return contrib_parity<KID>(m0, m1, m2, px, py, pz, qx, qy, qz, kp);
  } else {
    bool ok;
    const double v = contrib_parity_fast<KID, true>(m0, m1, m2, px, py, pz, qx, qy, qz, kp, ok);
    return ok ? v : contrib_parity<KID>(m0, m1, m2, px, py, pz, qx, qy, qz, kp);
  }
}

// term of one aggregate / point (contribution_rows)
template <int KID, bool F64>
__device__ __forceinline__ double term(const typename Prec<F64>::V4& g,
                                       const typename Prec<F64>::V4& mm, double qx, double qy,
                                       double qz, const KParams& kp) {
  if constexpr (F64) {
#if FSB_F64_TERM_FAST
    return term_parity<KID>(mm.x, mm.y, mm.z, g.x, g.y, g.z, qx, qy, qz, kp);
#else
    return contrib_parity<KID>(mm.x, mm.y, mm.z, g.x, g.y, g.z, qx, qy, qz, kp);
#endif
  } else {
    return (double)contrib_fast<KID>(mm.x, mm.y, mm.z, g.x, g.y, g.z, (float)qx, (float)qy,
                                     (float)qz, kp);
  }
}

template <bool F64>
__device__ __forceinline__ double dadd(double a, double b) {
  return F64 ? __dadd_rn(a, b) : a + b;
}

// exact per-point sum of a multi-point leaf (_node_term, _core.py:59-64)
template <int KID, bool F64>
__device__ double leaf_points_sum(const typename Prec<F64>::V4* __restrict__ pa,
                                  const typename Prec<F64>::V4* __restrict__ pb, int64_t b,
                                  int64_t e, double qx, double qy, double qz, const KParams& kp) {
  using V4 = typename Prec<F64>::V4;
  double acc = 0.0;
  for (int64_t j = b; j < e; ++j) {
    V4 u = pa[j];
    V4 mm;
    mm.x = u.w;
    if (KID == KID_WINDING) {
      V4 v = pb[j];
      mm.y = v.x;
      mm.z = v.y;
    } else {
      mm.y = 0;
      mm.z = 0;
    }
    acc = dadd<F64>(acc, term<KID, F64>(u, mm, qx, qy, qz, kp));
  }
  return acc;
}

template <bool F64>
__device__ __forceinline__ double ffr(const typename Prec<F64>::V4& g, double qx, double qy,
                                      double qz) {
  if constexpr (F64)
    return ffr_parity(g.x, g.y, g.z, g.w, qx, qy, qz);
  else
    return ffr_f32(g.x, g.y, g.z, g.w, (float)qx, (float)qy, (float)qz);
}

// _ffr(q, node) >= beta exactly as _core.py:44-52 decides it, without the square
// root and division for all but a vanishing band: RN(RN(sqrt(d2)) / dm) >= beta
// is monotone in d2, so d2 >= (beta dm)^2 (1 + 2^-46) proves "far" and
// d2 <= (beta dm)^2 (1 - 2^-46) proves "near" (the bound's own rounding is
// <= 2^-51 relative); inside the band, or when (beta dm)^2 is not a normal
// double, the reference's sequence decides.
__device__ __forceinline__ bool far_parity(double cx, double cy, double cz, double diam,
                                           double qx, double qy, double qz, double beta) {
  const double dx = __dsub_rn(qx, cx), dy = __dsub_rn(qy, cy), dz = __dsub_rn(qz, cz);
  const double d2 =
      __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double dm = diam < kDiamFloor ? kDiamFloor : diam;
  const double p = __dmul_rn(beta, dm), p2 = __dmul_rn(p, p);
  if (p2 >= 0x1p-1000 && p2 <= 0x1p1000) {
    if (d2 >= __dmul_rn(p2, 1.0 + 0x1p-46)) return true;
    if (d2 <= __dmul_rn(p2, 1.0 - 0x1p-46)) return false;
  }
  return __ddiv_rn(__dsqrt_rn(d2), dm) >= beta;
}

// ====================================================================== BH
// barnes_hut_batch (_core.py:101-129).  The reference pops an explicit stack
// with children pushed in reverse, i.e. it walks the accepted frontier in DFS
// preorder.  Here each query walks preorder with skip links (open: i+1,
// accept: skip[i]); a warp processes the union of its lanes' node sequences in
// increasing preorder index, so every record load is one broadcast transaction
// while each lane still sees exactly its own sequence (results unchanged).
#ifndef FSB_BH_MINB
#define FSB_BH_MINB 1
#endif
#ifdef FSB_BH_CHUNK_PROF
__device__ long long* g_bh_chunk_cycles;
#endif
#ifndef FSB_BH_FAR_FAST
#define FSB_BH_FAR_FAST 1  // FP64 acceptance test without sqrt / division (exact)
#endif
template <int KID, bool F64, bool VOTE>
__global__ void __launch_bounds__(128, FSB_BH_MINB) k_bh(const typename Prec<F64>::V4* __restrict__ rec,
                                            const typename Prec<F64>::V4* __restrict__ pa,
                                            const typename Prec<F64>::V4* __restrict__ pb,
                                            uint32_t nn, const double* __restrict__ q, int64_t n,
                                            const int32_t* __restrict__ qperm, double beta,
                                            KParams kp, typename Prec<F64>::Out* __restrict__ out,
                                            int64_t* __restrict__ visited,
                                            unsigned int* __restrict__ work) {
  using V4 = typename Prec<F64>::V4;
  const int lane = threadIdx.x & 31;
  const float beta_f = (float)beta;
  // persistent warps take 32-query chunks (in the caller's coherent order) from a
  // global counter: per-chunk cost varies by orders of magnitude near the surface
  while (true) {
    unsigned int chunk = 0;
    if (lane == 0) chunk = atomicAdd(work, 1u);
    chunk = __shfl_sync(0xffffffffu, chunk, 0);
    const int64_t t = (int64_t)chunk * 32 + lane;
    if ((int64_t)chunk * 32 >= n) break;
#ifdef FSB_BH_CHUNK_PROF
    const long long c_t0 = clock64();
#endif
    const bool live = t < n;
    const int64_t qi = live ? (qperm ? (int64_t)qperm[t] : t) : 0;
    double qx = 0, qy = 0, qz = 0;
    if (live) load_query(q, qi, qx, qy, qz);
    uint32_t i = live ? 0u : nn;
    double acc = 0.0;
    int64_t seen = 0;
#ifdef FSB_BH_CHUNK_PROF
    long long iters = 0;
#endif
    if constexpr (F64) {  // pipelined: the load overlaps the FP64 term
    // software-pipelined union walk: the next union node is known once this
    // node's accept / open decisions are made, so its records are fetched before
    // this node's term is evaluated (the load overlaps the FP64 term chain);
    // every lane still adds its accepted terms in its own preorder
    uint32_t cur = warp_min_u32(i);
    V4 g_n, mm_n;
    if (cur < nn) {
      g_n = rec[2 * (int64_t)cur];
      mm_n = rec[2 * (int64_t)cur + 1];
    }
    while (cur < nn) {
#ifdef FSB_BH_CHUNK_PROF
      ++iters;
#endif
      const bool mine = i == cur;
      const V4 g = g_n, mm = mm_n;
      uint32_t skip = 0;
      bool accept = false;
      if (mine) {
        ++seen;
        if constexpr (F64)
          skip = (uint32_t)__double_as_longlong(mm.w);
        else
          skip = (uint32_t)__float_as_int(mm.w);
        const bool leaf = skip == cur + 1;
        bool far;
        if constexpr (F64) {
#if FSB_BH_FAR_FAST
          far = far_parity(g.x, g.y, g.z, g.w, qx, qy, qz, beta);  // exact _ffr >= beta
#else
          far = ffr<F64>(g, qx, qy, qz) >= beta;  // exact _ffr (_core.py:44-52)
#endif
        } else {
          float dx = (float)qx - g.x, dy = (float)qy - g.y, dz = (float)qz - g.z;
          float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
          float thr = beta_f * fmaxf(g.w, 1e-12f);
          far = d2 >= thr * thr;
        }
        accept = leaf || far;
      }
      if (VOTE) accept = __all_sync(0xffffffffu, !mine || accept);
      const uint32_t i_next = mine ? (accept ? skip : cur + 1) : i;
      const uint32_t cur_next = warp_min_u32(i_next);
      if (cur_next < nn) {  // the next node's records, in flight during this term
        g_n = rec[2 * (int64_t)cur_next];
        mm_n = rec[2 * (int64_t)cur_next + 1];
      }
      if (mine && accept) {
        double v;
        if (g.w < 0) {  // multi-point leaf: exact per-point sum
          int64_t b, e;
          if constexpr (F64) {
            b = __double_as_longlong(mm.x);
            e = __double_as_longlong(mm.y);
          } else {
            b = __float_as_int(mm.x);
            e = __float_as_int(mm.y);
          }
          v = leaf_points_sum<KID, F64>(pa, pb, b, e, qx, qy, qz, kp);
        } else {
          v = term<KID, F64>(g, mm, qx, qy, qz, kp);
        }
        acc = dadd<F64>(acc, v);
      }
      i = i_next;
      cur = cur_next;
    }
    } else {  // FP32: the plain union walk (the pipelined one measured slower: the term is cheap)
    while (true) {
      uint32_t cur = warp_min_u32(i);
      if (cur >= nn) break;
#ifdef FSB_BH_CHUNK_PROF
      ++iters;
#endif
      const bool mine = i == cur;
      V4 g, mm;
      uint32_t skip = 0;
      bool accept = false;
      if (mine) {
        g = rec[2 * (int64_t)cur];
        mm = rec[2 * (int64_t)cur + 1];
        ++seen;
        if constexpr (F64)
          skip = (uint32_t)__double_as_longlong(mm.w);
        else
          skip = (uint32_t)__float_as_int(mm.w);
        bool leaf = skip == cur + 1;
        bool far;
        if constexpr (F64) {
#if FSB_BH_FAR_FAST
          far = far_parity(g.x, g.y, g.z, g.w, qx, qy, qz, beta);  // exact _ffr >= beta
#else
          far = ffr<F64>(g, qx, qy, qz) >= beta;  // exact _ffr (_core.py:44-52)
#endif
        } else {
          // FP32 mode: ||q - c||^2 >= (beta * max(diam, 1e-12))^2, no sqrt / division
          float dx = (float)qx - g.x, dy = (float)qy - g.y, dz = (float)qz - g.z;
          float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
          float thr = beta_f * fmaxf(g.w, 1e-12f);
          far = d2 >= thr * thr;
        }
        accept = leaf || far;
      }
      // warp voting: a node is accepted only when every live
      // lane accepts it, else the whole warp opens it (all live lanes walk one
      // sequence: more accurate per query, no divergence)
      if (VOTE) accept = __all_sync(0xffffffffu, !mine || accept);
      if (mine) {
        if (accept) {
          double v;
          if (g.w < 0) {  // multi-point leaf: exact per-point sum
            int64_t b, e;
            if constexpr (F64) {
              b = __double_as_longlong(mm.x);
              e = __double_as_longlong(mm.y);
            } else {
              b = __float_as_int(mm.x);
              e = __float_as_int(mm.y);
            }
            v = leaf_points_sum<KID, F64>(pa, pb, b, e, qx, qy, qz, kp);
          } else {
            v = term<KID, F64>(g, mm, qx, qy, qz, kp);
          }
          acc = dadd<F64>(acc, v);
          i = skip;
        } else {
          i = cur + 1;
        }
      }
    }
    }
    if (live) {
      out[qi] = (typename Prec<F64>::Out)acc;
      if (visited) visited[qi] = seen;
    }
#ifdef FSB_BH_CHUNK_PROF
    {  // cycles, union iterations, longest lane sequence (seen)
      const long long mx = __reduce_max_sync(0xffffffffu, (unsigned)(live ? seen : 0));
      if (lane == 0 && g_bh_chunk_cycles) {
        g_bh_chunk_cycles[3 * chunk] = clock64() - c_t0;
        g_bh_chunk_cycles[3 * chunk + 1] = iters;
        g_bh_chunk_cycles[3 * chunk + 2] = mx;
      }
    }
#endif
  }
}

// ============================================================== level order
template <int KID, bool F64>
struct LoTree {
  using V4 = typename Prec<F64>::V4;
  const V4* __restrict__ geo;
  const V4* __restrict__ mass;
  const int4* __restrict__ topo;
  const V4* __restrict__ pa;
  const V4* __restrict__ pb;
  // per point: sibling rank per level (ensure_path; null: binary search over begins)
  const uint64_t* __restrict__ path;
  int path_bits, path_levels;

  __device__ __forceinline__ double agg_term(int r, double qx, double qy, double qz,
                                             const KParams& kp) const {
    return term<KID, F64>(geo[r], mass[r], qx, qy, qz, kp);
  }
  // _node_term, _core.py:55-66
  __device__ __forceinline__ double node_term(int r, double qx, double qy, double qz,
                                              const KParams& kp) const {
    int4 tp = topo[r];
    if (tp.y == 0 && tp.w - tp.z > 1)
      return leaf_points_sum<KID, F64>(pa, pb, tp.z, tp.w, qx, qy, qz, kp);
    return agg_term(r, qx, qy, qz, kp);
  }
  // _children_term_sum, _core.py:69-77
  __device__ __forceinline__ double children_sum(const int4& tp, double qx, double qy, double qz,
                                                 const KParams& kp) const {
    double acc = 0.0;
    for (int t = 0; t < tp.y; ++t) acc = dadd<F64>(acc, node_term(tp.x + t, qx, qy, qz, kp));
    return acc;
  }
  // the child whose point range holds j (children are contiguous and ordered)
  __device__ __forceinline__ int child_of(const int4& tp, int64_t j) const {
    int lo = 0, hi = tp.y;  // invariant: begin(child lo) <= j
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (topo[tp.x + mid].z <= j)
        lo = mid;
      else
        hi = mid;
    }
    return tp.x + lo;
  }
  // child of the level-`lvl` node `tp` holding point j: from the point's path of
  // sibling ranks when available (one load per walk instead of a search per level)
  __device__ __forceinline__ int pick_child(const int4& tp, int64_t j, uint64_t pj,
                                            int lvl) const {
    if (path && lvl < path_levels)
      return tp.x + (int)((pj >> (path_bits * lvl)) & ((1ull << path_bits) - 1ull));
    return child_of(tp, j);
  }
};

// _sample_residual, _core.py:159-212 (one path from subdomain a)
template <int KID, bool F64, int VARIANT = 0>
__device__ __forceinline__ double sample_residual(const LoTree<KID, F64>& T, int a,
                                                  const int4& tpa, double delta_a,
                                                  uint64_t key_i, uint64_t key_r, int rr_mode,
                                                  double qx, double qy, double qz,
                                                  const KParams& kp, int64_t& steps,
                                                  int64_t& seen) {
  int64_t count_a = (int64_t)tpa.w - tpa.z;
  double u0 = uniform_draw(key_i, 0);
  int64_t j = tpa.z + (int64_t)__dmul_rn(u0, (double)count_a);
  if (j >= tpa.w) j = tpa.w - 1;
  int node = a;
  int4 tp = tpa;
  double prr = 1.0, resid = 0.0;
  uint64_t rctr = 0;
  const uint64_t pj = T.path ? T.path[j] : 0;
  int lvl = 1;  // subdomains are the root's children
  if constexpr (VARIANT == 1) {
    // the paper's Alg. 2 (pathSampleEstimator, PAPER.md supplemental): the
    // roulette at T_{I,k} gates the swap at T_{I,k} (the reference commits the
    // swap first); counters: +1 per roulette test, +children per swap
    while (tp.y > 0) {
      int child = T.pick_child(tp, j, pj, lvl);
      double rp = ffr<F64>(T.geo[node], qx, qy, qz);
      double rc = ffr<F64>(T.geo[child], qx, qy, qz);
      double p = rr_probability(rp, rc, rr_mode);
      double u = uniform_draw(key_r, rctr);
      ++rctr;
      ++seen;
      if (u >= p) break;
      double delta;
      if (node == a)
        delta = delta_a;
      else
        delta = F64 ? __dsub_rn(T.children_sum(tp, qx, qy, qz, kp), T.agg_term(node, qx, qy, qz, kp))
                    : T.children_sum(tp, qx, qy, qz, kp) - T.agg_term(node, qx, qy, qz, kp);
      seen += tp.y;
      prr = __dmul_rn(prr, p);
      double pagg = __ddiv_rn((double)(tp.w - tp.z), (double)count_a);
      resid = __dadd_rn(resid, __ddiv_rn(delta, __dmul_rn(pagg, prr)));
      node = child;
      tp = T.topo[node];
      ++steps;
      ++lvl;
    }
    return resid;
  } else {  // the reference walk (_core.py:177-211)
    while (tp.y > 0) {
      int child = T.pick_child(tp, j, pj, lvl);
      double delta;
      if (node == a)
        delta = delta_a;
      else
        delta = F64 ? __dsub_rn(T.children_sum(tp, qx, qy, qz, kp), T.agg_term(node, qx, qy, qz, kp))
                    : T.children_sum(tp, qx, qy, qz, kp) - T.agg_term(node, qx, qy, qz, kp);
      seen += tp.y;
      double pagg = __ddiv_rn((double)(tp.w - tp.z), (double)count_a);
      resid = __dadd_rn(resid, __ddiv_rn(delta, __dmul_rn(pagg, prr)));
      double rp = ffr<F64>(T.geo[node], qx, qy, qz);
      double rc = ffr<F64>(T.geo[child], qx, qy, qz);
      double p = rr_probability(rp, rc, rr_mode);
      double u = uniform_draw(key_r, rctr);
      ++rctr;
      ++seen;
      if (u >= p) break;
      prr = __dmul_rn(prr, p);
      node = child;
      tp = T.topo[node];
      ++steps;
      ++lvl;
    }
    return resid;
  }
}

// stochastic_batch, _core.py:215-267
#ifndef FSB_GEN_MINB
#define FSB_GEN_MINB 12  // 17.9 / 11.8 / 10.7 / 10.6 ms at 1 / 8 / 12 / 16 (C4, FP64)
#endif
template <int KID, bool F64, int VARIANT>
__global__ void __launch_bounds__(128, FSB_GEN_MINB) k_stochastic(LoTree<KID, F64> T, int root_kids,
                                                    const double* __restrict__ q, int64_t n,
                                                    const int32_t* __restrict__ qperm, int S,
                                                    int rr_mode, uint64_t seed, int64_t qoff,
                                                    int share, KParams kp,
                                                    typename Prec<F64>::Out* __restrict__ out,
                                                    int64_t* __restrict__ visited,
                                                    int64_t* __restrict__ path_steps,
                                                    int64_t* __restrict__ path_count) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  int64_t qi = qperm ? (int64_t)qperm[t] : t;
  double qx, qy, qz;
  load_query(q, qi, qx, qy, qz);
  int64_t seen = 0, steps = 0, paths = 0;
  double acc = 0.0;
  if (root_kids == 0) {
    acc = T.node_term(0, qx, qy, qz, kp);
    seen = 1;
  } else {
    uint64_t hq = key_fold(mix64(seed + kGamma),
                           share ? (uint64_t)((t + qoff) >> share) : (uint64_t)(qi + qoff));
    for (int a_ord = 0; a_ord < root_kids; ++a_ord) {
      int a = 1 + a_ord;  // level order: the root's children follow the root
      ++seen;
      int4 tpa = T.topo[a];
      if (tpa.y == 0) {
        acc = dadd<F64>(acc, T.node_term(a, qx, qy, qz, kp));
        continue;
      }
      double cv = T.agg_term(a, qx, qy, qz, kp);
      double ks = T.children_sum(tpa, qx, qy, qz, kp);
      double delta_a = F64 ? __dsub_rn(ks, cv) : ks - cv;
      uint64_t ha = key_fold(hq, (uint64_t)a_ord);
      double fa = 0.0;
      for (int s = 0; s < S; ++s) {
        uint64_t hs = key_fold(ha, (uint64_t)s);
        uint64_t key_i = key_fold(hs, 0), key_r = key_fold(hs, 1);
        double resid = sample_residual<KID, F64, VARIANT>(T, a, tpa, delta_a, key_i, key_r,
                                                          rr_mode, qx, qy, qz, kp, steps, seen);
        fa = __dadd_rn(fa, resid);
        ++paths;
      }
      acc = __dadd_rn(acc, __dadd_rn(cv, __ddiv_rn(fa, (double)S)));
    }
  }
  out[qi] = (typename Prec<F64>::Out)acc;
  if (visited) visited[qi] = seen;
  if (path_steps) path_steps[qi] = steps;
  if (path_count) path_count[qi] = paths;
}

// stochastic_moments_batch, _core.py:270-336 (per-subdomain swaps cached in `work`)
template <int KID, bool F64>
__global__ void __launch_bounds__(128) k_moments(LoTree<KID, F64> T, int root_kids,
                                                 const double* __restrict__ q, int64_t n,
                                                 int64_t n_reps, int rr_mode, uint64_t seed,
                                                 KParams kp, double* __restrict__ work,
                                                 double* __restrict__ mean_out,
                                                 double* __restrict__ var_out) {
  int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (qi >= n) return;
  double qx, qy, qz;
  load_query(q, qi, qx, qy, qz);
  if (root_kids == 0) {
    mean_out[qi] = T.node_term(0, qx, qy, qz, kp);
    var_out[qi] = 0.0;
    return;
  }
  double* delta = work + qi * (int64_t)root_kids;
  double base = 0.0;
  for (int a_ord = 0; a_ord < root_kids; ++a_ord)
    if (T.topo[1 + a_ord].y == 0) base = dadd<F64>(base, T.node_term(1 + a_ord, qx, qy, qz, kp));
  for (int a_ord = 0; a_ord < root_kids; ++a_ord) {
    int a = 1 + a_ord;
    int4 tpa = T.topo[a];
    if (tpa.y == 0) continue;
    double cv = T.agg_term(a, qx, qy, qz, kp);
    base = dadd<F64>(base, cv);
    double ks = T.children_sum(tpa, qx, qy, qz, kp);
    delta[a_ord] = F64 ? __dsub_rn(ks, cv) : ks - cv;
  }
  uint64_t hq = key_fold(mix64(seed + kGamma), (uint64_t)qi);
  double acc = 0.0, acc2 = 0.0;
  int64_t st = 0, se = 0;
  for (int64_t r = 0; r < n_reps; ++r) {
    double tsum = 0.0;
    for (int a_ord = 0; a_ord < root_kids; ++a_ord) {
      int a = 1 + a_ord;
      int4 tpa = T.topo[a];
      if (tpa.y == 0) continue;
      uint64_t hs = key_fold(key_fold(hq, (uint64_t)a_ord), (uint64_t)r);
      tsum = __dadd_rn(tsum, sample_residual<KID, F64>(T, a, tpa, delta[a_ord], key_fold(hs, 0),
                                                       key_fold(hs, 1), rr_mode, qx, qy, qz, kp,
                                                       st, se));
    }
    acc = __dadd_rn(acc, tsum);
    acc2 = __dadd_rn(acc2, __dmul_rn(tsum, tsum));
  }
  double mr = __ddiv_rn(acc, (double)n_reps);
  mean_out[qi] = __dadd_rn(base, mr);
  double v = __dsub_rn(__ddiv_rn(acc2, (double)n_reps), __dmul_rn(mr, mr));
  var_out[qi] = v > 0.0 ? v : 0.0;
}

// Few queries: G lanes per query.  Lane 0 of the group stages the query's
// deltas; the group's lanes then evaluate consecutive repetitions' estimates in
// parallel (each one exactly as above) and every lane adds them to (acc, acc2)
// in repetition order through width-G shuffles: the same bits.
template <int KID, bool F64, int G>
__global__ void __launch_bounds__(128) k_moments_g(LoTree<KID, F64> T, int root_kids,
                                                   const double* __restrict__ q, int64_t n,
                                                   int64_t n_reps, int rr_mode, uint64_t seed,
                                                   KParams kp, double* __restrict__ work,
                                                   double* __restrict__ mean_out,
                                                   double* __restrict__ var_out) {
  const int sub = threadIdx.x & (G - 1);
  const int64_t qi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = qi < n;
  double qx = 0, qy = 0, qz = 0;
  if (live) load_query(q, qi, qx, qy, qz);
  double* delta = work + (live ? qi : 0) * (int64_t)root_kids;
  double base = 0.0;
  if (live && sub == 0 && root_kids > 0) {
    for (int a_ord = 0; a_ord < root_kids; ++a_ord)
      if (T.topo[1 + a_ord].y == 0) base = dadd<F64>(base, T.node_term(1 + a_ord, qx, qy, qz, kp));
    for (int a_ord = 0; a_ord < root_kids; ++a_ord) {
      const int a = 1 + a_ord;
      const int4 tpa = T.topo[a];
      if (tpa.y == 0) continue;
      const double cv = T.agg_term(a, qx, qy, qz, kp);
      base = dadd<F64>(base, cv);
      const double ks = T.children_sum(tpa, qx, qy, qz, kp);
      delta[a_ord] = F64 ? __dsub_rn(ks, cv) : ks - cv;
    }
  }
  __syncwarp();  // the group's deltas are staged
  const uint64_t hq = key_fold(mix64(seed + kGamma), (uint64_t)qi);
  double acc = 0.0, acc2 = 0.0;
  int64_t st = 0, se = 0;
  const int64_t reps = root_kids > 0 ? n_reps : 0;
  for (int64_t r0 = 0; r0 < reps; r0 += G) {  // (uniform across the block)
    const int64_t r = r0 + sub;
    double tsum = 0.0;
    if (live && r < reps) {
      for (int a_ord = 0; a_ord < root_kids; ++a_ord) {
        const int a = 1 + a_ord;
        const int4 tpa = T.topo[a];
        if (tpa.y == 0) continue;
        const uint64_t hs = key_fold(key_fold(hq, (uint64_t)a_ord), (uint64_t)r);
        tsum = __dadd_rn(tsum, sample_residual<KID, F64>(T, a, tpa, delta[a_ord], key_fold(hs, 0),
                                                         key_fold(hs, 1), rr_mode, qx, qy, qz, kp,
                                                         st, se));
      }
    }
    const int take = reps - r0 < G ? (int)(reps - r0) : G;
    for (int t = 0; t < take; ++t) {
      const double ts = __shfl_sync(0xffffffffu, tsum, t, G);
      acc = __dadd_rn(acc, ts);
      acc2 = __dadd_rn(acc2, __dmul_rn(ts, ts));
    }
  }
  if (!live || sub != 0) return;
  if (root_kids == 0) {
    mean_out[qi] = T.node_term(0, qx, qy, qz, kp);
    var_out[qi] = 0.0;
    return;
  }
  const double mr = __ddiv_rn(acc, (double)n_reps);
  mean_out[qi] = __dadd_rn(base, mr);
  const double v = __dsub_rn(__ddiv_rn(acc2, (double)n_reps), __dmul_rn(mr, mr));
  var_out[qi] = v > 0.0 ? v : 0.0;
}

// telescoping_batch, _core.py:132-156 (preorder sweep over every internal node)
template <int KID, bool F64>
__global__ void __launch_bounds__(128) k_telescoping(LoTree<KID, F64> T,
                                                     const int32_t* __restrict__ pre2lo,
                                                     int64_t nn, const double* __restrict__ q,
                                                     int64_t n, KParams kp,
                                                     typename Prec<F64>::Out* __restrict__ out,
                                                     int64_t* __restrict__ visited) {
  int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (qi >= n) return;
  double qx, qy, qz;
  load_query(q, qi, qx, qy, qz);
  double acc = T.node_term(0, qx, qy, qz, kp);
  int64_t seen = 1;
  for (int64_t a = 0; a < nn; ++a) {
    int r = pre2lo[a];
    int4 tp = T.topo[r];
    if (tp.y > 0) {
      double kids = T.children_sum(tp, qx, qy, qz, kp);
      double parent = T.agg_term(r, qx, qy, qz, kp);
      acc = F64 ? __dadd_rn(acc, __dsub_rn(kids, parent)) : acc + (kids - parent);
      seen += 1 + tp.y;
    }
  }
  out[qi] = (typename Prec<F64>::Out)acc;
  if (visited) visited[qi] = seen;
}

// Few queries: G lanes per query.  The group's lanes evaluate consecutive
// preorder nodes' deltas (children sum - node term, each in its one lane, in
// the reference's order) in parallel; every lane then adds the internal nodes'
// deltas to the accumulator in preorder (width-G shuffles): the same additions
// in the same order as the one-thread-per-query kernel, so the same bits.
template <int KID, bool F64, int G>
__global__ void __launch_bounds__(128) k_telescoping_g(LoTree<KID, F64> T,
                                                       const int32_t* __restrict__ pre2lo,
                                                       int64_t nn, const double* __restrict__ q,
                                                       int64_t n, KParams kp,
                                                       typename Prec<F64>::Out* __restrict__ out,
                                                       int64_t* __restrict__ visited) {
  const int sub = threadIdx.x & (G - 1);
  const int64_t qi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = qi < n;
  double qx = 0, qy = 0, qz = 0;
  if (live) load_query(q, qi, qx, qy, qz);
  double acc = live ? T.node_term(0, qx, qy, qz, kp) : 0.0;
  int64_t seen = 0;  // this lane's share of the visited count
  for (int64_t a0 = 0; a0 < nn; a0 += G) {  // (uniform across the block)
    const int64_t a = a0 + sub;
    double delta = 0.0;
    bool internal = false;
    if (live && a < nn) {
      const int r = pre2lo[a];
      const int4 tp = T.topo[r];
      if (tp.y > 0) {
        const double kids = T.children_sum(tp, qx, qy, qz, kp);
        const double parent = T.agg_term(r, qx, qy, qz, kp);
        delta = F64 ? __dsub_rn(kids, parent) : (kids - parent);
        internal = true;
        seen += 1 + tp.y;
      }
    }
    const unsigned im = __ballot_sync(0xffffffffu, internal);
    const int take = nn - a0 < G ? (int)(nn - a0) : G;
    const unsigned gm = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (threadIdx.x & 31 & ~(G - 1));
    const unsigned mine = im & gm;  // this group's internal nodes
    for (int t = 0; t < take; ++t) {
      const double dt = __shfl_sync(0xffffffffu, delta, t, G);
      if (mine >> ((threadIdx.x & 31 & ~(G - 1)) + t) & 1u)
        acc = F64 ? __dadd_rn(acc, dt) : acc + dt;
    }
  }
  // visited: 1 (root) + the group's counts
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) seen += __shfl_xor_sync(0xffffffffu, seen, o, G);
  if (live && sub == 0) {
    out[qi] = (typename Prec<F64>::Out)acc;
    if (visited) visited[qi] = 1 + seen;
  }
}

// ============================================================== brute force
// brute_force_batch (_core.py:80-98).  Parity flavour: one query per thread,
// sources streamed through shared memory in the reference's order with the
// same Kahan recurrence.
constexpr int kBruteTile64 = 512;
// lanes per query for the few-query kernels: 1 when the queries alone give
// 148 SMs x 16 warps, else 8, or 32 below ~9.5 K queries (two instantiations)
static inline int lane_groups(int64_t n) {
  const int64_t want = (int64_t)148 * 16 * 32;
  return n >= want ? 1 : (n * 8 >= want ? 8 : 32);
}
#ifndef FSB_MOMENTS_GROUPS
#define FSB_MOMENTS_GROUPS 1  // few queries: repetitions on several lanes per query (same bits)
#endif
#ifndef FSB_TELESCOPING_GROUPS
#define FSB_TELESCOPING_GROUPS 1  // few queries: several lanes per query (same bits)
#endif
#ifndef FSB_BRUTE64_GROUPS
#define FSB_BRUTE64_GROUPS 1  // few queries: several lanes per query (same bits)
#endif
template <int KID>
__global__ void __launch_bounds__(256) k_brute64(const double* __restrict__ pts,
                                                 const double* __restrict__ ms, int64_t m, int c,
                                                 const double* __restrict__ q, int64_t n,
                                                 KParams kp, double* __restrict__ out) {
  __shared__ double4 sa[kBruteTile64];
  __shared__ double2 sb[KID == KID_WINDING ? kBruteTile64 : 1];
  int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool live = qi < n;
  double qx = 0, qy = 0, qz = 0;
  if (live) load_query(q, qi, qx, qy, qz);
  double acc = 0.0, comp = 0.0;
  for (int64_t base = 0; base < m; base += kBruteTile64) {
    int cnt = (int)(m - base < kBruteTile64 ? m - base : kBruteTile64);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      int64_t j = base + k;
      sa[k] = make_double4(pts[3 * j], pts[3 * j + 1], pts[3 * j + 2], ms[(int64_t)c * j]);
      if (KID == KID_WINDING) sb[k] = make_double2(ms[(int64_t)c * j + 1], ms[(int64_t)c * j + 2]);
    }
    __syncthreads();
    if (live) {
      for (int k = 0; k < cnt; ++k) {
        double4 s = sa[k];
        double m1 = 0, m2 = 0;
        if (KID == KID_WINDING) {
          m1 = sb[k].x;
          m2 = sb[k].y;
        }
        double v = contrib_parity<KID>(s.w, m1, m2, s.x, s.y, s.z, qx, qy, qz, kp);
        double y = __dsub_rn(v, comp);
        double tt = __dadd_rn(acc, y);
        comp = __dsub_rn(__dsub_rn(tt, acc), y);
        acc = tt;
      }
    }
  }
  if (live) out[qi] = acc;
}

// Few queries: G lanes per query (G a power of two, chosen so the launch has
// enough warps).  The group's lanes evaluate consecutive sources' terms in
// parallel; then every lane of the group applies the reference's Kahan
// recurrence to the G terms in source order (width-G shuffles), so each lane
// holds the same (acc, comp) as the one-thread-per-query kernel, bit for bit.
template <int KID, int G>
__global__ void __launch_bounds__(256) k_brute64g(const double* __restrict__ pts,
                                                  const double* __restrict__ ms, int64_t m, int c,
                                                  const double* __restrict__ q, int64_t n,
                                                  KParams kp, double* __restrict__ out) {
  __shared__ double4 sa[kBruteTile64];
  __shared__ double2 sb[KID == KID_WINDING ? kBruteTile64 : 1];
  const int sub = threadIdx.x & (G - 1);
  const int64_t qi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = qi < n;
  double qx = 0, qy = 0, qz = 0;
  if (live) load_query(q, qi, qx, qy, qz);
  double acc = 0.0, comp = 0.0;
  for (int64_t base = 0; base < m; base += kBruteTile64) {
    const int cnt = (int)(m - base < kBruteTile64 ? m - base : kBruteTile64);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      const int64_t j = base + k;
      sa[k] = make_double4(pts[3 * j], pts[3 * j + 1], pts[3 * j + 2], ms[(int64_t)c * j]);
      if (KID == KID_WINDING) sb[k] = make_double2(ms[(int64_t)c * j + 1], ms[(int64_t)c * j + 2]);
    }
    __syncthreads();
    for (int k0 = 0; k0 < cnt; k0 += G) {  // (uniform across the block)
      const int k = k0 + sub;
      double v = 0.0;
      if (live && k < cnt) {
        const double4 sv = sa[k];
        const double m1 = KID == KID_WINDING ? sb[k].x : 0.0;
        const double m2 = KID == KID_WINDING ? sb[k].y : 0.0;
        v = term_parity<KID>(sv.w, m1, m2, sv.x, sv.y, sv.z, qx, qy, qz, kp);
      }
      const int take = min(G, cnt - k0);
      for (int t = 0; t < take; ++t) {
        const double vt = __shfl_sync(0xffffffffu, v, t, G);
        const double y = __dsub_rn(vt, comp);
        const double tt = __dadd_rn(acc, y);
        comp = __dsub_rn(__dsub_rn(tt, acc), y);
        acc = tt;
      }
    }
  }
  if (live && sub == 0) out[qi] = acc;
}

// Fast flavour: FP32 terms, each thread owns QPT queries (register tiling over
// one broadcast LDS.128 per source), FP32 partials folded into FP64 every
// kFold = 32 sources (bounds FP32 cancellation error in signed-mass sums); sources split across blockIdx.y when the query count alone
// cannot fill 148 SMs (deterministic: partials reduced in chunk order).
constexpr int kBruteTile32 = 1024;
constexpr int kFold = 32;
template <int KID, int QPT>
__global__ void __launch_bounds__(256) k_brute32(const float4* __restrict__ sa_g,
                                                 const float4* __restrict__ sb_g, int64_t m,
                                                 int64_t chunk, const double* __restrict__ q,
                                                 int64_t n, KParams kp,
                                                 double* __restrict__ partial) {
  __shared__ float4 sa[kBruteTile32];
  __shared__ float2 sb[KID == KID_WINDING ? kBruteTile32 : 1];
  int64_t q0 = blockIdx.x * (int64_t)blockDim.x * QPT + threadIdx.x;
  float qx[QPT], qy[QPT], qz[QPT];
  double accd[QPT];
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    int64_t qi = q0 + (int64_t)k * blockDim.x;
    qx[k] = qy[k] = qz[k] = 0.f;
    if (qi < n) {
      qx[k] = (float)q[3 * qi];
      qy[k] = (float)q[3 * qi + 1];
      qz[k] = (float)q[3 * qi + 2];
    }
    accd[k] = 0.0;
  }
  int64_t s0 = blockIdx.y * chunk, s1 = min(m, s0 + chunk);
  for (int64_t base = s0; base < s1; base += kBruteTile32) {
    int cnt = (int)(s1 - base < kBruteTile32 ? s1 - base : kBruteTile32);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      sa[k] = sa_g[base + k];
      if (KID == KID_WINDING) {
        float4 v = sb_g[base + k];
        sb[k] = make_float2(v.x, v.y);
      }
    }
    __syncthreads();
    for (int f0 = 0; f0 < cnt; f0 += kFold) {
      int f1 = min(cnt, f0 + kFold);
      float accf[QPT];
#pragma unroll
      for (int k = 0; k < QPT; ++k) accf[k] = 0.f;
#pragma unroll 4
      for (int j = f0; j < f1; ++j) {
        float4 s = sa[j];
        float m1 = 0.f, m2 = 0.f;
        if (KID == KID_WINDING) {
          float2 v = sb[j];
          m1 = v.x;
          m2 = v.y;
        }
#pragma unroll
        for (int k = 0; k < QPT; ++k)
          accf[k] += contrib_fast<KID>(s.w, m1, m2, s.x, s.y, s.z, qx[k], qy[k], qz[k], kp);
      }
#pragma unroll
      for (int k = 0; k < QPT; ++k) accd[k] += (double)accf[k];
    }
  }
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    int64_t qi = q0 + (int64_t)k * blockDim.x;
    if (qi < n) partial[blockIdx.y * n + qi] = accd[k];
  }
}

// Coulomb on the packed FP32 pipe (FADD2/FFMA2, sm_100): query pairs share one
// instruction, so an interaction issues 3.5 FP32 instructions + MUFU.RSQ
// instead of 8 + MUFU and the kernel becomes MUFU-bound.  Sources are staged
// pre-broadcast ({x,x,y,y}, {z,z,-m,-m}) so the pairs land in register pairs
// straight from LDS.128.  The distance floor is applied as r2 + floor^2 inside
// the first FFMA2: identical to max(r, floor) at r = 0 and for every pair
// farther apart than 4e-9 (below that the FP32 cast of the coordinates has
// already lost the distance).
template <int QPT>
__global__ void __launch_bounds__(256) k_brute32_coulomb2(const float4* __restrict__ sa_g,
                                                          int64_t m, int64_t chunk,
                                                          const double* __restrict__ q, int64_t n,
                                                          KParams kp,
                                                          double* __restrict__ partial) {
  static_assert(QPT % 2 == 0, "query pairs");
  constexpr int P = QPT / 2;
  __shared__ float4 sa[2 * kBruteTile32];
  int64_t q0 = blockIdx.x * (int64_t)blockDim.x * QPT + threadIdx.x;
  float2 qx[P], qy[P], qz[P];
  double accd[QPT];
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    int64_t qi = q0 + (int64_t)k * blockDim.x;
    float x = 0.f, y = 0.f, z = 0.f;
    if (qi < n) {
      x = (float)q[3 * qi];
      y = (float)q[3 * qi + 1];
      z = (float)q[3 * qi + 2];
    }
    if (k & 1) {
      qx[k / 2].y = -x, qy[k / 2].y = -y, qz[k / 2].y = -z;
    } else {
      qx[k / 2].x = -x, qy[k / 2].x = -y, qz[k / 2].x = -z;
    }
    accd[k] = 0.0;
  }
  const float f2 = kp.dfloor_f * kp.dfloor_f;
  const float2 floor2 = make_float2(f2, f2);
  int64_t s0 = blockIdx.y * chunk, s1 = min(m, s0 + chunk);
  for (int64_t base = s0; base < s1; base += kBruteTile32) {
    int cnt = (int)(s1 - base < kBruteTile32 ? s1 - base : kBruteTile32);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      float4 v = sa_g[base + k];
      sa[2 * k] = make_float4(v.x, v.x, v.y, v.y);
      sa[2 * k + 1] = make_float4(v.z, v.z, -v.w, -v.w);
    }
    __syncthreads();
    for (int f0 = 0; f0 < cnt; f0 += kFold) {
      int f1 = min(cnt, f0 + kFold);
      float2 acc[P];
#pragma unroll
      for (int k = 0; k < P; ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int j = f0; j < f1; ++j) {
        const float4 a = sa[2 * j], b = sa[2 * j + 1];
        const float2 sx = make_float2(a.x, a.y), sy = make_float2(a.z, a.w),
                     sz = make_float2(b.x, b.y), nm = make_float2(b.z, b.w);
#pragma unroll
        for (int k = 0; k < P; ++k) {
          float2 dx = __fadd2_rn(sx, qx[k]), dy = __fadd2_rn(sy, qy[k]), dz = __fadd2_rn(sz, qz[k]);
          float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __ffma2_rn(dz, dz, floor2)));
          float2 ri = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
          acc[k] = __ffma2_rn(nm, ri, acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < P; ++k) {
        accd[2 * k] += (double)acc[k].x;
        accd[2 * k + 1] += (double)acc[k].y;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    int64_t qi = q0 + (int64_t)k * blockDim.x;
    if (qi < n) partial[blockIdx.y * n + qi] = accd[k];
  }
}

__global__ void k_reduce_chunks(const double* __restrict__ partial, int chunks, int64_t n,
                                double* __restrict__ out64, float* __restrict__ out32) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int y = 0; y < chunks; ++y) acc += partial[y * n + i];
  if (out64) out64[i] = acc;
  if (out32) out32[i] = (float)acc;
}

__global__ void k_pack_src32(const double* __restrict__ pts, const double* __restrict__ ms,
                             int64_t m, int c, float4* __restrict__ a, float4* __restrict__ b) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  a[j] = make_float4((float)pts[3 * j], (float)pts[3 * j + 1], (float)pts[3 * j + 2],
                     (float)ms[(int64_t)c * j]);
  if (b) b[j] = make_float4(c >= 3 ? (float)ms[(int64_t)c * j + 1] : 0.f,
                            c >= 3 ? (float)ms[(int64_t)c * j + 2] : 0.f, 0.f, 0.f);
}

// post_transform (kernels.py:110-122) over the raw sums, plus the FP64 raw copy
// FieldResult exposes (estimators.py:313-323)
__global__ void k_post_transform(const void* __restrict__ raw, int raw_f32, int64_t n, int smooth,
                                 double alpha, double* __restrict__ values,
                                 double* __restrict__ raw64, uint8_t* __restrict__ flagged) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = raw_f32 ? (double)static_cast<const float*>(raw)[i] : static_cast<const double*>(raw)[i];
  if (raw64) raw64[i] = r;
  double v = r;
  uint8_t f = 0;
  if (smooth) {
    if (r <= 0.0) {
      v = INFINITY;
      f = 1;
    } else {
      v = __ddiv_rn(-log(r), alpha);
    }
  }
  values[i] = v;
  flagged[i] = f;
}

int post_transform(const void* raw, int raw_f32, int64_t n, int smooth, double alpha,
                   double* values, double* raw64, uint8_t* flagged, cudaStream_t s) {
  if (n <= 0) return 0;
  k_post_transform<<<grid_for(n, 256), 256, 0, s>>>(raw, raw_f32, n, smooth, alpha, values, raw64,
                                                    flagged);
  FS_CK(cudaGetLastError());
  return 0;
}

// ================================================================ dispatch
static KParams make_kp(double alpha, double dfloor) {
  KParams kp;
  kp.alpha = alpha;
  kp.dfloor = dfloor;
  kp.alpha_log2e_neg = (float)(-alpha * 1.4426950408889634);
  kp.dfloor_f = (float)dfloor;
  kp.inv_dfloor_f = (float)(1.0 / dfloor);
  return kp;
}

// calls f(integral_constant<KID>, bool_constant<F64>) for the runtime pair
template <class F>
static int with_kid(int kid, bool f64, F&& f) {
  using std::bool_constant;
  using std::integral_constant;
  switch (kid * 2 + (f64 ? 1 : 0)) {
    case 0: f(integral_constant<int, 0>{}, bool_constant<false>{}); break;
    case 1: f(integral_constant<int, 0>{}, bool_constant<true>{}); break;
    case 2: f(integral_constant<int, 1>{}, bool_constant<false>{}); break;
    case 3: f(integral_constant<int, 1>{}, bool_constant<true>{}); break;
    case 4: f(integral_constant<int, 2>{}, bool_constant<false>{}); break;
    case 5: f(integral_constant<int, 2>{}, bool_constant<true>{}); break;
    default: set_error("unknown kernel id %d", kid); return 1;
  }
  FS_CK(cudaGetLastError());
  return 0;
}

static int sm_count() {
  static int cnt = 0;
  if (!cnt) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cnt, cudaDevAttrMultiProcessorCount, dev);
    if (cnt <= 0) cnt = 148;
  }
  return cnt;
}

#ifndef FSB_BRUTE_QPT
#define FSB_BRUTE_QPT 8  // scalar flavour: 2.87e12 interactions/s at 8 vs 2.66e12 at 4
#endif
#ifndef FSB_BRUTE_QPT2
#define FSB_BRUTE_QPT2 16  // packed Coulomb: 0.79 of the MUFU.RSQ bound (0.72 at 4, 8, 32)
#endif
#ifndef FSB_BRUTE_PACKED
#define FSB_BRUTE_PACKED 1
#endif
template <int KID>
static int brute32_launch(const float4* sa, const float4* sb, int64_t m, const double* q, int64_t n,
                          const KParams& kp, double* out64, float* out32, cudaStream_t s) {
  constexpr bool packed = KID == KID_COULOMB && FSB_BRUTE_PACKED;
  constexpr int QPT = packed ? FSB_BRUTE_QPT2 : FSB_BRUTE_QPT, B = 256;
  int64_t per_block = (int64_t)B * QPT;
  int64_t gx = (n + per_block - 1) / per_block;
  int64_t want = 4LL * sm_count();  // ~4 resident blocks per SM
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(want / std::max<int64_t>(gx, 1),
                                                          (m + kBruteTile32 - 1) / kBruteTile32));
  chunks = std::min<int64_t>(chunks, 65535);
  int64_t chunk = (m + chunks - 1) / chunks;
  chunk = ((chunk + kBruteTile32 - 1) / kBruteTile32) * kBruteTile32;
  chunks = (m + chunk - 1) / chunk;
  Scratch part;
  FS_TRY(part.alloc(sizeof(double) * chunks * n, s));
  dim3 grid((unsigned)gx, (unsigned)chunks);
  if (packed)
    k_brute32_coulomb2<QPT><<<grid, B, 0, s>>>(sa, m, chunk, q, n, kp, part.as<double>());
  else
    k_brute32<KID, QPT><<<grid, B, 0, s>>>(sa, sb, m, chunk, q, n, kp, part.as<double>());
  k_reduce_chunks<<<grid_for(n, 256), 256, 0, s>>>(part.as<double>(), (int)chunks, n, out64, out32);
  FS_CK(cudaGetLastError());
  return 0;
}

int brute_force(int kid, double alpha, double dfloor, bool f64, const double* pts,
                const double* ms, int64_t m, int c, const double* q, int64_t n, void* out,
                cudaStream_t s) {
  if (n <= 0) return 0;
  KParams kp = make_kp(alpha, dfloor);
  if (f64) {
    // lanes per query (lane_groups): several when the queries alone cannot fill the GPU
    const int G = FSB_BRUTE64_GROUPS ? lane_groups(n) : 1;
    return with_kid(kid, true, [&](auto K, auto) {
      constexpr int KD = decltype(K)::value;
      const int64_t threads = n * G;
      if (G == 1)
        k_brute64<KD><<<grid_for(n, 256), 256, 0, s>>>(pts, ms, m, c, q, n, kp, (double*)out);
      else if (G == 8)
        k_brute64g<KD, 8><<<grid_for(threads, 256), 256, 0, s>>>(pts, ms, m, c, q, n, kp, (double*)out);
      else
        k_brute64g<KD, 32><<<grid_for(threads, 256), 256, 0, s>>>(pts, ms, m, c, q, n, kp, (double*)out);
    });
  }
  Scratch sa, sb;
  FS_TRY(sa.alloc(sizeof(float4) * m, s));
  FS_TRY(sb.alloc(sizeof(float4) * (kid == KID_WINDING ? m : 1), s));
  k_pack_src32<<<grid_for(m, 256), 256, 0, s>>>(pts, ms, m, c, sa.as<float4>(),
                                                kid == KID_WINDING ? sb.as<float4>() : nullptr);
  switch (kid) {
    case 0: return brute32_launch<0>(sa.as<float4>(), sb.as<float4>(), m, q, n, kp, nullptr, (float*)out, s);
    case 1: return brute32_launch<1>(sa.as<float4>(), sb.as<float4>(), m, q, n, kp, nullptr, (float*)out, s);
    case 2: return brute32_launch<2>(sa.as<float4>(), sb.as<float4>(), m, q, n, kp, nullptr, (float*)out, s);
  }
  set_error("unknown kernel id %d", kid);
  return 1;
}

int brute_force_f32_acc64(int kid, double alpha, double dfloor, const double* pts,
                          const double* ms, int64_t m, int c, const double* q, int64_t n,
                          double* out, cudaStream_t s) {
  KParams kp = make_kp(alpha, dfloor);
  Scratch sa, sb;
  FS_TRY(sa.alloc(sizeof(float4) * m, s));
  FS_TRY(sb.alloc(sizeof(float4) * (kid == KID_WINDING ? m : 1), s));
  k_pack_src32<<<grid_for(m, 256), 256, 0, s>>>(pts, ms, m, c, sa.as<float4>(),
                                                kid == KID_WINDING ? sb.as<float4>() : nullptr);
  switch (kid) {
    case 0: return brute32_launch<0>(sa.as<float4>(), sb.as<float4>(), m, q, n, kp, out, nullptr, s);
    case 1: return brute32_launch<1>(sa.as<float4>(), sb.as<float4>(), m, q, n, kp, out, nullptr, s);
    case 2: return brute32_launch<2>(sa.as<float4>(), sb.as<float4>(), m, q, n, kp, out, nullptr, s);
  }
  set_error("unknown kernel id %d", kid);
  return 1;
}

template <int KID, bool F64>
static LoTree<KID, F64> lo_view(const FsTree* t) {
  LoTree<KID, F64> T;
  if constexpr (F64) {
    T.geo = t->lo_geo64;
    T.mass = t->lo_mass64;
    T.pa = t->pts64a;
    T.pb = t->pts64b;
  } else {
    T.geo = t->lo_geo32;
    T.mass = t->lo_mass32;
    T.pa = t->pts32a;
    T.pb = t->pts32b;
  }
  T.topo = t->lo_topo;
  T.path = t->pt_path;
  T.path_bits = t->path_bits;
  T.path_levels = t->path_levels;
  return T;
}

int barnes_hut(FsTree* t, int kid, double alpha, double dfloor, bool f64, const double* q,
               int64_t n, const int32_t* qperm, double beta, void* out, int64_t* visited,
               cudaStream_t s, bool vote) {
  if (n <= 0) return 0;
  FS_TRY(ensure_bh(t, f64, s));
  FS_TRY(ensure_lo(t, f64, s));  // packed points for multi-point leaves
  KParams kp = make_kp(alpha, dfloor);
  const char* split_env = std::getenv("FSB_BH_SPLIT");
  if (!f64 && !(split_env && split_env[0] == '0')) {  // load-balanced FP32 BH
    bool done = false;
    FS_TRY(barnes_hut_split(t, kid, alpha, dfloor, q, n, qperm, beta, (float*)out, visited, s,
                            &done, vote));
    if (done) return 0;
  }
  Scratch work;  // chunk counter of the persistent warps
  FS_TRY(work.alloc(sizeof(unsigned int), s));
  FS_CK(cudaMemsetAsync(work.p, 0, sizeof(unsigned int), s));
  return with_kid(kid, f64, [&](auto K, auto P) {
    constexpr int KID = decltype(K)::value;
    constexpr bool F64 = decltype(P)::value;
    using V4 = typename Prec<F64>::V4;
    const V4 *rec, *pa, *pb;
    if constexpr (F64) {
      rec = reinterpret_cast<const V4*>(t->bh64);
      pa = t->pts64a;
      pb = t->pts64b;
    } else {
      rec = reinterpret_cast<const V4*>(t->bh32);
      pa = t->pts32a;
      pb = t->pts32b;
    }
    auto launch = [&](auto kern) {
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
      const int64_t grid =
          std::min<int64_t>((n + 127) / 128, (int64_t)sm_count() * std::max(per_sm, 1));
      kern<<<(unsigned)grid, 128, 0, s>>>(rec, pa, pb, (uint32_t)t->n, q, n, qperm, beta, kp,
                                          (typename Prec<F64>::Out*)out, visited,
                                          work.as<unsigned int>());
    };
#ifdef FSB_BH_CHUNK_PROF
    const int64_t nch = (n + 31) / 32;
    long long* prof = nullptr;
    cudaMalloc(&prof, 3 * sizeof(long long) * nch);
    cudaMemset(prof, 0, 3 * sizeof(long long) * nch);
    cudaMemcpyToSymbol(g_bh_chunk_cycles, &prof, sizeof(prof));
#endif
    if (vote)
      launch(k_bh<KID, F64, true>);
    else
      launch(k_bh<KID, F64, false>);
#ifdef FSB_BH_CHUNK_PROF
    std::vector<long long> h(3 * nch);
    cudaMemcpy(h.data(), prof, 3 * sizeof(long long) * nch, cudaMemcpyDeviceToHost);
    std::vector<int64_t> idx(nch);
    for (int64_t k = 0; k < nch; ++k) idx[k] = k;
    std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return h[3 * a] > h[3 * b]; });
    long long sum = 0;
    for (int64_t k = 0; k < nch; ++k) sum += h[3 * k];
    fprintf(stderr, "bh chunks %lld: sum %.3e cycles; top chunks (cycles / union iters / max lane seen):",
            (long long)nch, (double)sum);
    for (int k = 0; k < 8 && k < nch; ++k)
      fprintf(stderr, " [%lld: %lld/%lld/%lld]", (long long)idx[k], h[3 * idx[k]], h[3 * idx[k] + 1],
              h[3 * idx[k] + 2]);
    const int64_t med = idx[nch / 2];
    fprintf(stderr, " median chunk %lld/%lld/%lld\n", h[3 * med], h[3 * med + 1], h[3 * med + 2]);
    cudaFree(prof);
    long long* z = nullptr;
    cudaMemcpyToSymbol(g_bh_chunk_cycles, &z, sizeof(z));
#endif
  });
}

int stochastic(FsTree* t, int kid, double alpha, double dfloor, bool f64, const double* q,
               int64_t n, const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed,
               int64_t query_offset, void* out, int64_t* visited, int64_t* path_steps,
               int64_t* path_count, cudaStream_t s, int share, int flags) {
  if (n <= 0) return 0;
  const int variant = flags & kFlagAlg2;
  bool shuffled = (flags & kFlagShuffled) != 0;  // order = shuffle_order(n, seed, qoff)
  // the fast FP32 kernels implement the reference variant; Alg. 2 runs the
  // generic per-query kernel in either precision
  if (!f64 && variant == 0 && !std::getenv("FSB_DISABLE_FAST")) {
    bool used = false;
    FS_TRY(stochastic_fast(t, kid, alpha, dfloor, q, n, qperm, n_samples, rr_mode, seed,
                           query_offset, share, (float*)out, visited, path_steps, path_count, s,
                           &used, shuffled));
    if (used) return 0;
    if (std::getenv("FSB_REQUIRE_FAST")) {  // tests: a silent fallback is an error
      set_error("the fast FP32 stochastic kernel declined this tree / launch");
      return 2;
    }
  }
  Scratch order;  // the generic kernel reads the shuffled order from memory
  if (shuffled) {
    FS_TRY(order.alloc(sizeof(int32_t) * (size_t)n, s));
    FS_TRY(shuffle_order(n, seed, query_offset, order.as<int32_t>(), s));
    qperm = order.as<int32_t>();
    shuffled = false;
  }
  // FP64 reference variant: the queue kernel (fs_sto64.cu), same bits
  if (f64 && variant == 0) {
    bool used = false;
    FS_TRY(stochastic64(t, kid, alpha, dfloor, q, n, qperm, n_samples, rr_mode, seed,
                        query_offset, share, (double*)out, visited, path_steps, path_count, s,
                        &used));
    if (used) return 0;
  }
  if (shuffled) {
    FS_TRY(order.alloc(sizeof(int32_t) * (size_t)n, s));
    FS_TRY(shuffle_order(n, seed, query_offset, order.as<int32_t>(), s));
    qperm = order.as<int32_t>();
  }
  FS_TRY(ensure_lo(t, f64, s));
  FS_TRY(ensure_path(t, s));
  KParams kp = make_kp(alpha, dfloor);
  return with_kid(kid, f64, [&](auto K, auto P) {
    constexpr int KID = decltype(K)::value;
    constexpr bool F64 = decltype(P)::value;
    auto go = [&](auto kern) {
      kern<<<grid_for(n, 128), 128, 0, s>>>(lo_view<KID, F64>(t), t->root_kids, q, n, qperm,
                                           n_samples, rr_mode, seed, query_offset, share, kp,
                                           (typename Prec<F64>::Out*)out, visited, path_steps,
                                           path_count);
    };
    if (variant)
      go(k_stochastic<KID, F64, 1>);
    else
      go(k_stochastic<KID, F64, 0>);
  });
}

int stochastic_moments(FsTree* t, int kid, double alpha, double dfloor, const double* q,
                       int64_t n, int64_t n_reps, int rr_mode, uint64_t seed, double* mean_out,
                       double* var_out, cudaStream_t s) {
  if (n <= 0) return 0;
  FS_TRY(ensure_lo(t, true, s));
  FS_TRY(ensure_path(t, s));
  KParams kp = make_kp(alpha, dfloor);
  Scratch work;
  FS_TRY(work.alloc(sizeof(double) * n * std::max(1, t->root_kids), s));
  // lanes per query (repetitions in parallel) when the queries alone cannot fill
  // 148 SMs x 16 warps
  int G = FSB_MOMENTS_GROUPS ? lane_groups(n) : 1;
  if (n_reps < 2 * G) G = 1;
  return with_kid(kid, true, [&](auto K, auto) {
    constexpr int KID = decltype(K)::value;
    const auto V = lo_view<KID, true>(t);
    double* w = work.as<double>();
    const int64_t th = n * G;
    if (G == 1)
      k_moments<KID, true><<<grid_for(n, 128), 128, 0, s>>>(V, t->root_kids, q, n, n_reps, rr_mode, seed, kp, w, mean_out, var_out);
    else if (G == 8)
      k_moments_g<KID, true, 8><<<grid_for(th, 128), 128, 0, s>>>(V, t->root_kids, q, n, n_reps, rr_mode, seed, kp, w, mean_out, var_out);
    else
      k_moments_g<KID, true, 32><<<grid_for(th, 128), 128, 0, s>>>(V, t->root_kids, q, n, n_reps, rr_mode, seed, kp, w, mean_out, var_out);
  });
}

int telescoping(FsTree* t, int kid, double alpha, double dfloor, bool f64, const double* q,
                int64_t n, void* out, int64_t* visited, cudaStream_t s) {
  if (n <= 0) return 0;
  FS_TRY(ensure_lo(t, f64, s));
  KParams kp = make_kp(alpha, dfloor);
  // lanes per query (lane_groups): several when the queries alone cannot fill the GPU
  const int G = FSB_TELESCOPING_GROUPS ? lane_groups(n) : 1;
  return with_kid(kid, f64, [&](auto K, auto P) {
    constexpr int KID = decltype(K)::value;
    constexpr bool F64 = decltype(P)::value;
    using O = typename Prec<F64>::Out;
    const auto V = lo_view<KID, F64>(t);
    const int64_t th = n * G;
    if (G == 1)
      k_telescoping<KID, F64><<<grid_for(n, 128), 128, 0, s>>>(V, t->pre2lo, t->n, q, n, kp, (O*)out, visited);
    else if (G == 8)
      k_telescoping_g<KID, F64, 8><<<grid_for(th, 128), 128, 0, s>>>(V, t->pre2lo, t->n, q, n, kp, (O*)out, visited);
    else
      k_telescoping_g<KID, F64, 32><<<grid_for(th, 128), 128, 0, s>>>(V, t->pre2lo, t->n, q, n, kp, (O*)out, visited);
  });
}

}  // namespace fsb

namespace fsb {
// self-test of far_parity against the reference's acceptance test
// (_ffr(q, node) >= beta, _core.py:44-52 / 117) on operands that put the query
// within a few ulps to 1e-9 of the acceptance sphere, plus general positions and
// degenerate diameters / betas
__global__ void k_bh_far_selftest(int64_t n, uint64_t seed, unsigned long long* counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t h = mix64(seed + (uint64_t)i * kGamma);
  auto u01 = [&]() {
    h = mix64(h + kGamma);
    return (double)(h >> 11) * 0x1p-53;
  };
  const double cx = 2.0 * u01() - 1.0, cy = 2.0 * u01() - 1.0, cz = 2.0 * u01() - 1.0;
  const int kind = (int)(i & 7);
  double diam = kind == 6 ? 1e-13 * u01() : ldexp(0.5 + u01(), -(int)(h & 15));
  double beta = kind == 7 ? ldexp(1.0 + u01(), (int)(h >> 60) * 80 - 600) : 0.25 + 16.0 * u01();
  // a direction, then a distance on the sphere of radius beta * max(diam, 1e-12)
  // perturbed by a few ulps (kinds 0-2), up to 1e-9 relative (3-4), or anywhere (5+)
  double ux = 2.0 * u01() - 1.0, uy = 2.0 * u01() - 1.0, uz = 2.0 * u01() - 1.0;
  const double un = sqrt(ux * ux + uy * uy + uz * uz) + 1e-300;
  ux /= un;
  uy /= un;
  uz /= un;
  const double dm = diam < kDiamFloor ? kDiamFloor : diam;
  double t = beta * dm;
  if (kind <= 2)
    t *= 1.0 + (double)((int)(h & 63) - 32) * 0x1p-52;
  else if (kind <= 4)
    t *= 1.0 + (2.0 * u01() - 1.0) * 1e-9;
  else
    t *= 4.0 * u01();
  const double qx = cx + t * ux, qy = cy + t * uy, qz = cz + t * uz;
  const bool fast = far_parity(cx, cy, cz, diam, qx, qy, qz, beta);
  const bool exact = ffr_parity(cx, cy, cz, diam, qx, qy, qz) >= beta;
  atomicAdd(&counts[0], 1ull);
  if (fast != exact) atomicAdd(&counts[1], 1ull);
}
}  // namespace fsb

// counts2 (host) = {cases, mismatches} of the exact-acceptance shortcut
extern "C" int fsb_selftest_bh_far(int64_t n, uint64_t seed, unsigned long long* counts2) {
  using namespace fsb;
  FSB_RANGE("fsb_selftest_bh_far");
  if (n < 1 || !counts2) {
    set_error("fsb_selftest_bh_far: bad arguments");
    return 1;
  }
  Scratch c;
  FS_TRY(c.alloc(2 * sizeof(unsigned long long), nullptr));
  FS_CK(cudaMemset(c.p, 0, 2 * sizeof(unsigned long long)));
  k_bh_far_selftest<<<grid_for(n, 256), 256>>>(n, seed, c.as<unsigned long long>());
  FS_CK(cudaGetLastError());
  FS_CK(cudaMemcpy(counts2, c.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return 0;
}
