// fs_sto64.cu -- the FP64 stochastic estimator (precision="f64", the API default),
// bitwise equal to the reference's stochastic_batch (_core.py:159-267).
//
// The thread-per-query parity kernel (k_stochastic, fs_eval.cu) runs each
// query's paths in place: lanes of a warp walk different nodes for different
// lengths, every node term reads 80 bytes of scattered records, and the
// query-independent level-1/2 terms are re-read from L1/L2 by every thread.
// This kernel keeps every FP64 operation of the reference in the reference's
// order and reorganises the work around it:
//
//  * Level 1 (the subdomains) and level 2 (their children) are staged once per
//    persistent block in shared memory ({com, m0} + topology, 48 B per node),
//    so the dense part of every query -- cv(a) and the hoisted swap
//    delta_a = sum(children) - cv(a), _core.py:244-250 -- and the first step
//    of every sample (index draw, child, two far-field ratios, roulette,
//    _core.py:164-211 at node == a) read broadcast shared memory.
//  * A sample whose roulette lets it descend below level 2 is queued (48-byte
//    walk start: owner, slot, node, point, the exact FP64 state resid / prr /
//    ratio and the roulette key) and the block's lanes drain the queue
//    together, each carrying a walk to completion one level per iteration
//    (_core.py:177-211 from the second level on): no lane idles while another
//    lane of its warp walks.
//  * Every sample's residual lands in its (query, a, s) slot; after the drain
//    the owner folds acc += cv + fa / S in the reference's order
//    (_core.py:237-263), so each value is bitwise the reference's whichever
//    lane ran the walk.
// Deeper records are read as {com, m0} (32 B) plus the topology only at levels
// that can hold multi-point leaves; cell diameters are per level (uniform
// splits, octree.py:225; checked by ensure_fast).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "fs_common.cuh"
#include "fs_eval.h"
#include "fs_internal.h"

namespace fsb {

#ifndef FSB_S64_BLOCK
#define FSB_S64_BLOCK 128
#endif
#ifndef FSB_S64_MINB
#define FSB_S64_MINB 5  // C4: 3.47 ms (groups of 2, 96 registers) vs 3.71 (groups of 4, 4 blocks)
#endif
#ifndef FSB_S64_FASTDIV
#define FSB_S64_FASTDIV 1  // branch-free division / square root (bitwise the intrinsics')
#endif
#ifndef FSB_S64_GROUP
#define FSB_S64_GROUP 2  // node terms evaluated together per thread (4, 2 or 1)
#endif
#ifndef FSB_S64_QCAP
#define FSB_S64_QCAP 4608  // walk starts per drain round and block
#endif
constexpr int kB64 = FSB_S64_BLOCK;
constexpr int kMaxLevels64 = 64;

struct View64 {
  const double4* __restrict__ cm;    // {cx, cy, cz, m0} per level-order node
  const double2* __restrict__ m12;   // {m1, m2} (winding)
  const int4* __restrict__ topo;     // {first child, count, begin, end}
  const double4* __restrict__ pa;    // permuted points {x, y, z, m0}
  const double4* __restrict__ pb;    // {m1, m2, 0, 0}
  const uint64_t* __restrict__ path; // per point: sibling rank per level
  int path_bits, path_levels;
  int n1, base2, n2, first_multi;
  int qcap;
  bool div_safe;  // masses / coordinates / floor in range: no division range test
  double diam[kMaxLevels64];  // cell diameter per level (exact)
};

template <int KID>
__device__ __forceinline__ double term64(const double4& c, const double2& w, double qx, double qy,
                                         double qz, const KParams& kp) {
  return contrib_parity<KID>(c.w, w.x, w.y, c.x, c.y, c.z, qx, qy, qz, kp);
}

// sum over the contiguous records [c, ce) of their terms, added left to right
// from ks (_children_term_sum, _core.py:69-77, no multi-point leaves): groups
// of four evaluated through the branch-free division / square root (bitwise
// the intrinsics'; the rare out-of-range operand is recomputed with them), so
// four terms are in flight per thread
template <int KID, bool CHK, class Rec>
__device__ __forceinline__ double terms_sum64(double ks, int c, int ce, Rec rec, double qx,
                                              double qy, double qz, const KParams& kp) {
  auto slow = [&](int i) {
    double4 cm;
    double2 w;
    rec(i, cm, w);
    return contrib_parity<KID>(cm.w, w.x, w.y, cm.x, cm.y, cm.z, qx, qy, qz, kp);
  };
  if constexpr (KID != KID_SMOOTH && FSB_S64_FASTDIV) {
    auto fast = [&](int i, bool& ok) {
      double4 cm;
      double2 w;
      rec(i, cm, w);
      return contrib_parity_fast<KID, CHK>(cm.w, w.x, w.y, cm.x, cm.y, cm.z, qx, qy, qz, kp, ok);
    };
#if FSB_S64_GROUP == 4
    for (; c + 4 <= ce; c += 4) {
      bool o0, o1, o2, o3;
      double v0 = fast(c, o0), v1 = fast(c + 1, o1), v2 = fast(c + 2, o2), v3 = fast(c + 3, o3);
      if (!(o0 && o1 && o2 && o3)) {
        if (!o0) v0 = slow(c);
        if (!o1) v1 = slow(c + 1);
        if (!o2) v2 = slow(c + 2);
        if (!o3) v3 = slow(c + 3);
      }
      ks = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(ks, v0), v1), v2), v3);
    }
#elif FSB_S64_GROUP == 2
    for (; c + 2 <= ce; c += 2) {
      bool o0, o1;
      double v0 = fast(c, o0), v1 = fast(c + 1, o1);
      if (!(o0 && o1)) {
        if (!o0) v0 = slow(c);
        if (!o1) v1 = slow(c + 1);
      }
      ks = __dadd_rn(__dadd_rn(ks, v0), v1);
    }
#endif
    for (; c < ce; ++c) {
      bool o;
      double v = fast(c, o);
      if (!o) v = slow(c);
      ks = __dadd_rn(ks, v);
    }
  } else {
    for (; c < ce; ++c) ks = __dadd_rn(ks, slow(c));
  }
  return ks;
}

// exact per-point sum of a multi-point leaf (_core.py:59-64)
template <int KID>
__device__ double leaf_sum64(const View64& V, int b, int e, double qx, double qy, double qz,
                             const KParams& kp) {
  double acc = 0.0;
  for (int j = b; j < e; ++j) {
    const double4 u = V.pa[j];
    double2 w = make_double2(0.0, 0.0);
    if (KID == KID_WINDING) {
      const double4 v = V.pb[j];
      w = make_double2(v.x, v.y);
    }
    acc = __dadd_rn(acc, term64<KID>(u, w, qx, qy, qz, kp));
  }
  return acc;
}

// _ffr (_core.py:44-52) with the level's cell diameter
__device__ __forceinline__ double ffr64(const double4& c, double diam, double qx, double qy,
                                        double qz) {
  return ffr_parity(c.x, c.y, c.z, diam, qx, qy, qz);
}

extern __shared__ double4 sh64_d4[];
#ifdef FSB_S64_PROF
__device__ unsigned long long g_s64_prof[4];
#endif

template <int KID, int RR>
__global__ void __launch_bounds__(kB64, FSB_S64_MINB)
    k_sto64(const __grid_constant__ View64 V, const double* __restrict__ q, int64_t n,
            const int32_t* __restrict__ qperm, int S, uint64_t seed, int64_t qoff, int share,
            KParams kp, unsigned char* __restrict__ queues, double* __restrict__ slots_g,
            unsigned int* __restrict__ tile_ctr, double* __restrict__ out,
            int64_t* __restrict__ visited, int64_t* __restrict__ path_steps,
            int64_t* __restrict__ path_count) {
  // shared: {com, m0} of levels 1-2 (n12 = n1 + n2 nodes, level-order index - 1),
  // their topology, {m1, m2} (winding), per-query coordinates and counters
  const int n1 = V.n1, n2 = V.n2, n12 = n1 + n2;
  double4* s_cm = sh64_d4;                                   // [n12]
  double4* s_q = s_cm + n12;                                 // [kB64] {x, y, z, -}
  int4* s_tp = reinterpret_cast<int4*>(s_q + kB64);          // [n12]
  double2* s_w = reinterpret_cast<double2*>(s_tp + n12);     // [n12] (winding)
  int* s_int = reinterpret_cast<int*>(s_w + (KID == KID_WINDING ? n12 : 0));
  int* s_seen = s_int;                                       // [kB64]
  int* s_steps = s_seen + kB64;                              // [kB64]
  int* s_ctl = s_steps + kB64;                               // [4]: queue length, drain head, tile
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < n12; i += kB64) {
    s_cm[i] = V.cm[1 + i];  // level order: 1..n1 level 1, then level 2 (base2 == 1 + n1)
    s_tp[i] = V.topo[1 + i];
    if (KID == KID_WINDING) s_w[i] = V.m12[1 + i];
  }
  if (tid < 4) s_ctl[tid] = 0;
  s_seen[tid] = 0;
  s_steps[tid] = 0;
  __syncthreads();

  int4* const qrec = reinterpret_cast<int4*>(queues + (size_t)blockIdx.x * V.qcap * 48);
  const int nsl = n1 * S + n1;  // slots: resid per (a, s), then cv / leaf term per a
  double* const slots = slots_g + (size_t)blockIdx.x * nsl * kB64;
  const uint64_t hseed = mix64(seed + kGamma);
  const double d1 = V.diam[1], d2 = V.diam[2];
  const double2 w0 = make_double2(0.0, 0.0);
  const bool multi12 = V.first_multi <= 2;
  const int nflat = n1 * S;
  // per drain round at most rmax (a, s) pairs per thread: the queue never overflows
  const int rmax = max(1, V.qcap / kB64);
  const int64_t ntiles = (n + kB64 - 1) / kB64;

  while (true) {
    if (tid == 0) s_ctl[2] = (int)atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_ctl[2];
    if (tile >= ntiles) break;
    const int64_t t = tile * kB64 + tid;
    const bool live = t < n;
    const int64_t qi = live ? (qperm ? (int64_t)qperm[t] : t) : 0;
    double qx = 0.0, qy = 0.0, qz = 0.0;
    if (live) {
      qx = q[3 * qi];
      qy = q[3 * qi + 1];
      qz = q[3 * qi + 2];
    }
    s_q[tid] = make_double4(qx, qy, qz, 0.0);
    // the division range test can be dropped when every query of the tile is
    // bounded (|q| <= 2^100) on a div_safe tree (contrib_parity_fast)
    const bool tile_safe =
        __syncthreads_and(V.div_safe &&
                          (!live || (fabs(qx) <= 0x1p100 && fabs(qy) <= 0x1p100 &&
                                     fabs(qz) <= 0x1p100)));
    const uint64_t hq =
        key_fold(hseed, share ? (uint64_t)((t + qoff) >> share) : (uint64_t)(qi + qoff));
    int seen = 0, steps = 0;

    // per-subdomain state carried across drain rounds
    int4 tpa = make_int4(0, 0, 0, 0);
    double delta_a = 0.0, rp_a = 0.0;
    uint64_t ha = 0;
    int a_cur = -1;
    for (int f0 = 0; f0 < nflat; f0 += rmax) {
#ifdef FSB_S64_PROF
      const long long t_p1 = clock64();
#endif
      const int f1 = min(f0 + rmax, nflat);
      if (live) {
        for (int f = f0; f < f1; ++f) {
          const int a_ord = S == 1 ? f : f / S, sm = f - a_ord * S;
          if (a_ord != a_cur) {  // a new subdomain: dense part (_core.py:237-250)
            a_cur = a_ord;
            ++seen;
            tpa = s_tp[a_ord];
            if (tpa.y == 0) {  // leaf subdomain: exact term, never sampled
              const double v = (tpa.w - tpa.z > 1)
                                   ? leaf_sum64<KID>(V, tpa.z, tpa.w, qx, qy, qz, kp)
                                   : term64<KID>(s_cm[a_ord], KID == KID_WINDING ? s_w[a_ord] : w0,
                                                 qx, qy, qz, kp);
              slots[(size_t)(nflat + a_ord) * kB64 + tid] = v;
              continue;
            }
            const double cv =
                term64<KID>(s_cm[a_ord], KID == KID_WINDING ? s_w[a_ord] : w0, qx, qy, qz, kp);
            slots[(size_t)(nflat + a_ord) * kB64 + tid] = cv;
            double ks = 0.0;  // _children_term_sum over the level-2 children
            const int c0 = tpa.x - 1, ce = c0 + tpa.y;
            if (!multi12) {
              auto rec = [&](int i, double4& cm, double2& w) {
                cm = s_cm[i];
                w = KID == KID_WINDING ? s_w[i] : w0;
              };
              ks = tile_safe ? terms_sum64<KID, false>(ks, c0, ce, rec, qx, qy, qz, kp)
                             : terms_sum64<KID, true>(ks, c0, ce, rec, qx, qy, qz, kp);
            } else {
              for (int c = c0; c < ce; ++c) {
                double v;
                const int4 tc = s_tp[c];
                if (tc.y == 0 && tc.w - tc.z > 1)
                  v = leaf_sum64<KID>(V, tc.z, tc.w, qx, qy, qz, kp);
                else
                  v = term64<KID>(s_cm[c], KID == KID_WINDING ? s_w[c] : w0, qx, qy, qz, kp);
                ks = __dadd_rn(ks, v);
              }
            }
            delta_a = __dsub_rn(ks, cv);
            rp_a = ffr64(s_cm[a_ord], d1, qx, qy, qz);
            ha = key_fold(hq, (uint64_t)a_ord);
          }
          if (tpa.y == 0) continue;  // (the samples of a leaf subdomain)
          // one sample, first step at node == a (_core.py:164-211)
          const uint64_t hs = key_fold(ha, (uint64_t)sm);
          const uint64_t ki = key_fold(hs, 0), kr = key_fold(hs, 1);
          const int64_t count_a = (int64_t)tpa.w - tpa.z;
          const double u0 = uniform_draw(ki, 0);
          int64_t j = tpa.z + (int64_t)__dmul_rn(u0, (double)count_a);
          if (j >= tpa.w) j = tpa.w - 1;
          // the child holding j: children are ordered by begin (binary search)
          int lo = tpa.x - 1, hi = tpa.x - 1 + tpa.y;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_tp[mid].z <= j)
              lo = mid;
            else
              hi = mid;
          }
          seen += tpa.y;
          // _core.py:196-200 at node == a: p_agg = count_a / count_a = 1 and p_rr = 1,
          // so delta / (p_agg * p_rr) = delta exactly
          const double resid = __dadd_rn(0.0, delta_a);
          const double rc = ffr64(s_cm[lo], d2, qx, qy, qz);
          const double p = rr_probability(rp_a, rc, RR);
          const double u = uniform_draw(kr, 0);
          ++seen;
          if (u >= p) {
            slots[(size_t)f * kB64 + tid] = resid;
          } else {  // descends: queue the walk from the level-2 node
            ++steps;
            const int pos = atomicAdd(&s_ctl[0], 1);
            int4* r = qrec + 3 * (size_t)pos;
            r[0] = make_int4(tid | (f << 8), 1 + lo, (int)j, 0);
            r[1] = make_int4(__double2loint(resid), __double2hiint(resid),
                             __double2loint(__dmul_rn(1.0, p)), __double2hiint(__dmul_rn(1.0, p)));
            r[2] = make_int4(__double2loint(rc), __double2hiint(rc), (int)(uint32_t)kr,
                             (int)(uint32_t)(kr >> 32));
          }
        }
      }
      __syncthreads();
#ifdef FSB_S64_PROF
      if (tid == 0) atomicAdd(&g_s64_prof[0], (unsigned long long)(clock64() - t_p1));
      const long long t_drain = clock64();
#endif
      // ---- drain: lanes without a walk claim the next start (warp-aggregated)
      // and carry it to completion one level per iteration
      {
        const int cnt = s_ctl[0];
        bool act = false;
        int owner = 0, slot = 0, node = 0, lvl = 2, wseen = 0, wsteps = 0;
        int jj = 0, count_a = 1;  // (point indices and counts fit 32 bits)
        uint64_t path = 0, kr = 0;
        double resid = 0.0, prr = 1.0, rp = 0.0;
        int4 tp = make_int4(0, 0, 0, 0);
        while (true) {
          const unsigned need = __ballot_sync(0xffffffffu, !act);
          if (need) {
            int head = 0;
            if (lane == __ffs(need) - 1) head = atomicAdd(&s_ctl[1], __popc(need));
            head = __shfl_sync(0xffffffffu, head, __ffs(need) - 1);
            const int idx = head + __popc(need & ((1u << lane) - 1u));
            if (!act && idx < cnt) {
              const int4* r = qrec + 3 * (size_t)idx;
              const int4 r0 = r[0], r1 = r[1], r2 = r[2];
              owner = r0.x & 0xff;
              slot = r0.x >> 8;
              node = r0.y;
              jj = r0.z;
              resid = __hiloint2double(r1.y, r1.x);
              prr = __hiloint2double(r1.w, r1.z);
              rp = __hiloint2double(r2.y, r2.x);
              kr = ((uint64_t)(uint32_t)r2.w << 32) | (uint32_t)r2.z;
              const int4 ta = s_tp[slot / S];
              count_a = ta.w - ta.z;
              tp = s_tp[node - 1];  // level 2: staged
              path = V.path ? V.path[jj] : 0;
              lvl = 2;
              wseen = 0;
              wsteps = 0;
              act = true;
            }
          }
          if (!__any_sync(0xffffffffu, act)) break;
          if (!act) continue;
          bool cont = false;
          if (tp.y > 0) {  // _core.py:177-211 at a node below the subdomain
            // the owner's query, re-read from shared memory (fewer live registers)
            const double4 qq = s_q[owner];
            const double wx = qq.x, wy = qq.y, wz = qq.z;
            int child;
            if (V.path && lvl < V.path_levels) {
              child = tp.x + (int)((path >> (V.path_bits * lvl)) & ((1ull << V.path_bits) - 1ull));
            } else {
              int lo = 0, hi = tp.y;
              while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (V.topo[tp.x + mid].z <= jj)
                  lo = mid;
                else
                  hi = mid;
              }
              child = tp.x + lo;
            }
            const bool cmulti = lvl + 1 >= V.first_multi;
            double ks = 0.0;
            if (!cmulti) {
              auto rec = [&](int i, double4& cm, double2& w) {
                cm = V.cm[i];
                w = KID == KID_WINDING ? V.m12[i] : w0;
              };
              ks = tile_safe ? terms_sum64<KID, false>(ks, tp.x, tp.x + tp.y, rec, wx, wy, wz, kp)
                             : terms_sum64<KID, true>(ks, tp.x, tp.x + tp.y, rec, wx, wy, wz, kp);
            } else {
              for (int c = tp.x; c < tp.x + tp.y; ++c) {
                double v;
                const int4 tc = V.topo[c];
                if (tc.y == 0 && tc.w - tc.z > 1)
                  v = leaf_sum64<KID>(V, tc.z, tc.w, wx, wy, wz, kp);
                else
                  v = term64<KID>(V.cm[c], KID == KID_WINDING ? V.m12[c] : w0, wx, wy, wz, kp);
                ks = __dadd_rn(ks, v);
              }
            }
            const double4 cn = lvl == 2 ? s_cm[node - 1] : V.cm[node];
            const double2 wn = KID == KID_WINDING ? (lvl == 2 ? s_w[node - 1] : V.m12[node]) : w0;
            const double delta = __dsub_rn(ks, term64<KID>(cn, wn, wx, wy, wz, kp));
            wseen += tp.y;
            const double pagg = __ddiv_rn((double)(tp.w - tp.z), (double)count_a);
            resid = __dadd_rn(resid, __ddiv_rn(delta, __dmul_rn(pagg, prr)));
            const double rc = ffr64(V.cm[child], V.diam[min(lvl + 1, kMaxLevels64 - 1)], wx, wy, wz);
            const double p = rr_probability(rp, rc, RR);
            const double u = uniform_draw(kr, (uint64_t)(lvl - 1));  // rctr = levels so far
            ++wseen;
            if (u < p) {
              prr = __dmul_rn(prr, p);
              rp = rc;
              node = child;
              tp = V.topo[child];
              ++wsteps;
              ++lvl;
              cont = true;
            }
          }
          if (!cont) {
            slots[(size_t)slot * kB64 + owner] = resid;
            atomicAdd(&s_seen[owner], wseen);
            if (wsteps) atomicAdd(&s_steps[owner], wsteps);
            act = false;
          }
        }
      }
      __syncthreads();
#ifdef FSB_S64_PROF
      if (tid == 0) atomicAdd(&g_s64_prof[1], (unsigned long long)(clock64() - t_drain));
#endif
      if (tid == 0) {
        s_ctl[0] = 0;
        s_ctl[1] = 0;
      }
      __syncthreads();
    }
#ifdef FSB_S64_PROF
    const long long t_fold = clock64();
#endif
    // ---- fold in the reference's order: acc += term (leaf a) or cv + fa / S
    if (live) {
      double acc = 0.0;
      int n_int = 0;
      if (S == 1) {  // (the common case) eight subdomains' slots loaded at once
        for (int a0 = 0; a0 < n1; a0 += 8) {
          double v[8], r[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v[k] = a0 + k < n1 ? slots[(size_t)(nflat + a0 + k) * kB64 + tid] : 0.0;
            r[k] = a0 + k < n1 ? slots[(size_t)(a0 + k) * kB64 + tid] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (a0 + k >= n1) break;
            if (s_tp[a0 + k].y == 0) {
              acc = __dadd_rn(acc, v[k]);
            } else {
              ++n_int;
              acc = __dadd_rn(acc, __dadd_rn(v[k], __dadd_rn(0.0, r[k])));  // fa / S, S = 1
            }
          }
        }
      } else {
        for (int a_ord = 0; a_ord < n1; ++a_ord) {
          const double v = slots[(size_t)(nflat + a_ord) * kB64 + tid];
          if (s_tp[a_ord].y == 0) {
            acc = __dadd_rn(acc, v);
            continue;
          }
          ++n_int;
          double fa = 0.0;
          for (int sm = 0; sm < S; ++sm)
            fa = __dadd_rn(fa, slots[(size_t)(a_ord * S + sm) * kB64 + tid]);
          acc = __dadd_rn(acc, __dadd_rn(v, __ddiv_rn(fa, (double)S)));
        }
      }
      out[qi] = acc;
      if (visited) visited[qi] = (int64_t)seen + s_seen[tid];
      if (path_steps) path_steps[qi] = (int64_t)steps + s_steps[tid];
      if (path_count) path_count[qi] = (int64_t)n_int * S;
    }
    s_seen[tid] = 0;
    s_steps[tid] = 0;
    __syncthreads();
#ifdef FSB_S64_PROF
    if (tid == 0) { atomicAdd(&g_s64_prof[2], (unsigned long long)(clock64() - t_fold)); }
#endif
  }
}

// returns with *used = false when the tree does not suit this kernel (the
// caller runs the thread-per-query parity kernel)
int stochastic64(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                 const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed, int64_t qoff,
                 int share, double* out, int64_t* visited, int64_t* path_steps,
                 int64_t* path_count, cudaStream_t s, bool* used) {
  *used = false;
  const bool trace = std::getenv("FSB_TRACE_DISPATCH") != nullptr;
  auto decline = [&](const char* why) {
    if (trace) fprintf(stderr, "stochastic64: declined (%s)\n", why);
    return 0;
  };
  if (std::getenv("FSB_STO64_OFF")) return decline("FSB_STO64_OFF");
  if (t->root_kids <= 0 || t->num_levels > kMaxLevels64 || t->num_levels < 3)
    return decline("tree shape");
  FS_TRY(ensure_fast(t, s));  // per-level diameters, multi-point leaf levels
  if (!t->uniform_diam) return decline("non-uniform cell diameters");
  FS_TRY(ensure_lo(t, true, s));  // FP64 points (multi-point leaves), topology
  FS_TRY(ensure_path(t, s));
  FS_TRY(ensure_cm64(t, s));
  View64 V;
  V.cm = t->lo_cm64;
  V.m12 = t->lo_m12_64;
  V.topo = t->lo_topo;
  V.pa = t->pts64a;
  V.pb = t->pts64b;
  V.path = t->pt_path;
  V.path_bits = t->path_bits;
  V.path_levels = t->path_levels;
  V.n1 = t->root_kids;
  V.base2 = (int)t->level_off[2];
  V.n2 = (int)(t->level_off[3] - t->level_off[2]);
  V.first_multi = t->first_multi_level;
  // the division's range test is provably true when |coordinates| <= 2^100 (so
  // r <= 2^102), dfloor in [2^-100, 2^100] and, for Coulomb (-m0 / r), |m0| in
  // [2^-800, 2^800]: every quotient is a normal number and every operand finite
  // (winding divides the constant 1 / (4 pi) by r^3)
  V.div_safe = t->coords_in_range && (kid != KID_COULOMB || t->masses_in_range) &&
               dfloor >= 0x1p-100 && dfloor <= 0x1p100 &&
               !std::getenv("FSB_S64_DIVCHECK");
  for (int l = 0; l < kMaxLevels64; ++l) V.diam[l] = l < t->num_levels ? t->level_diam64[l] : 1.0;
  if (V.base2 != 1 + V.n1) return decline("level layout");
  const int64_t nflat = (int64_t)V.n1 * n_samples;
  if (nflat + V.n1 >= (1 << 22) || t->n >= (1ll << 30)) return decline("sizes");
  V.qcap = (int)std::min<int64_t>(FSB_S64_QCAP, std::max<int64_t>(kB64, nflat * kB64));
  V.qcap = std::max(V.qcap / kB64, 1) * kB64;
  const bool wind = kid == KID_WINDING;
  const size_t n12 = (size_t)V.n1 + V.n2;
  const size_t smem = 32 * (n12 + kB64) + 16 * n12 + (wind ? 16 * n12 : 0) + 4 * (2 * kB64 + 4);
  if (smem > 200 * 1024) return decline("shared memory");
  KParams kp;
  kp.alpha = alpha;
  kp.dfloor = dfloor;
  kp.alpha_log2e_neg = (float)(-alpha * 1.4426950408889634);
  kp.dfloor_f = (float)dfloor;
  kp.inv_dfloor_f = (float)(1.0 / dfloor);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto launch = [&](auto kern) -> int {
    FS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kB64, smem));
    const int64_t tiles = (n + kB64 - 1) / kB64;
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)sms * std::max(per_sm, 1));
    Scratch queues, slots, ctr;
    FS_TRY(queues.alloc((size_t)grid * V.qcap * 48, s));
    FS_TRY(slots.alloc(sizeof(double) * (size_t)grid * (nflat + V.n1) * kB64, s));
    FS_TRY(ctr.alloc(sizeof(unsigned int), s));
    FS_CK(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned int), s));
#ifdef FSB_S64_PROF
    unsigned long long z[4] = {0, 0, 0, 0};
    FS_CK(cudaMemcpyToSymbolAsync(g_s64_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
#endif
    kern<<<(unsigned)grid, kB64, smem, s>>>(V, q, n, qperm, n_samples, seed, qoff, share, kp,
                                            queues.as<unsigned char>(), slots.as<double>(),
                                            ctr.as<unsigned int>(), out, visited, path_steps,
                                            path_count);
    FS_CK(cudaGetLastError());
#ifdef FSB_S64_PROF
    FS_CK(cudaMemcpyFromSymbolAsync(z, g_s64_prof, sizeof(z), 0, cudaMemcpyDeviceToHost, s));
    FS_CK(cudaStreamSynchronize(s));
    const double tot = (double)(z[0] + z[1] + z[2]);
    fprintf(stderr, "k_sto64 block cycles: sampling+dense %.1f%%, drain %.1f%%, fold %.1f%%\n",
            100.0 * z[0] / tot, 100.0 * z[1] / tot, 100.0 * z[2] / tot);
#endif
    return 0;
  };
  int rc = 0;
  switch (kid * 3 + rr_mode) {
    case 0: rc = launch(k_sto64<0, 0>); break;
    case 1: rc = launch(k_sto64<0, 1>); break;
    case 2: rc = launch(k_sto64<0, 2>); break;
    case 3: rc = launch(k_sto64<1, 0>); break;
    case 4: rc = launch(k_sto64<1, 1>); break;
    case 5: rc = launch(k_sto64<1, 2>); break;
    case 6: rc = launch(k_sto64<2, 0>); break;
    case 7: rc = launch(k_sto64<2, 1>); break;
    case 8: rc = launch(k_sto64<2, 2>); break;
    default: set_error("unknown kernel id / rr mode"); return 1;
  }
  if (rc == 0) *used = true;
  return rc;
}

// self-test of the branch-free FP64 division / square root against the
// intrinsics on pseudo-random operands over the whole exponent range
__global__ void k_fp64_selftest(int64_t n, uint64_t seed, unsigned long long* counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t h1 = mix64(seed + (uint64_t)i * kGamma), h2 = mix64(h1 ^ kMix1);
  // mostly the normal range the kernels see, plus raw bit patterns (subnormals,
  // infinities, NaNs, zeros)
  const double a = (i & 7) == 0 ? __longlong_as_double((long long)h1)
                                : ldexp(1.0 + (double)(h1 >> 11) * 0x1p-53,
                                        (int)(h1 & 0x3f) - 32) * ((h1 >> 6) & 1 ? -1.0 : 1.0);
  const double b = (i & 7) == 1 ? __longlong_as_double((long long)h2)
                                : ldexp(1.0 + (double)(h2 >> 11) * 0x1p-53, (int)(h2 & 0x3f) - 32);
  bool ok1, ok2;
  const double q = ddiv_fast(a, b, ok1);
  const double r = dsqrt_fast(fabs(a), ok2);
  const double q0 = __ddiv_rn(a, b), r0 = __dsqrt_rn(fabs(a));
  if (ok1) atomicAdd(&counts[0], 1ull);
  if (ok1 && __double_as_longlong(q) != __double_as_longlong(q0)) atomicAdd(&counts[1], 1ull);
  if (ok2) atomicAdd(&counts[2], 1ull);
  if (ok2 && __double_as_longlong(r) != __double_as_longlong(r0)) atomicAdd(&counts[3], 1ull);
}

}  // namespace fsb

// counts4 (host) = {division fast-path operands, mismatches, sqrt fast-path
// operands, mismatches} over n pseudo-random operand pairs
extern "C" int fsb_selftest_fp64(int64_t n, uint64_t seed, unsigned long long* counts4) {
  using namespace fsb;
  if (n < 1 || !counts4) {
    set_error("fsb_selftest_fp64: bad arguments");
    return 1;
  }
  Scratch c;
  FS_TRY(c.alloc(4 * sizeof(unsigned long long), nullptr));
  FS_CK(cudaMemset(c.p, 0, 4 * sizeof(unsigned long long)));
  k_fp64_selftest<<<grid_for(n, 256), 256>>>(n, seed, c.as<unsigned long long>());
  FS_CK(cudaGetLastError());
  FS_CK(cudaMemcpy(counts4, c.p, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return 0;
}
