// fs_sto_fast.cu -- the FP32 stochastic estimator kernel (precision="f32").
//
// Same estimator as stochastic_batch (_core.py:159-267, the reference variant:
// the swap at each reached node is committed before the roulette that gates
// descent), same splitmix64 streams and index draws, reorganised for B200:
//
//  * Dense part.  Per subdomain a (root child) the reference adds cv(a) and
//    every sample of a commits the level-1 swap delta_a = sum(children) - cv(a)
//    with weight 1/(p_agg * p_rr) = 1 (_core.py:196-200, hoisted at 246-250),
//    so cv(a) cancels and the query-independent dense part is the sum of all
//    N2 level-2 records (children of internal level-1 nodes, contiguous in
//    level order) plus exact terms of leaf subdomains.  A persistent block
//    stages the level-1/2 records in shared memory once ({com, m0} = 16 B per
//    node, + {m1, m2} for winding) and every thread streams them with
//    broadcast LDS: an FP32 + MUFU.RSQ loop, "brute force over staged nodes".
//  * Sampling.  Per (a, s): the splitmix64 index draw, the level-1 step from
//    shared memory (a bucket table on the index draw's top bits plus a short
//    scan over the children's begins; far-field ratios from per-level cell
//    diameters: cells are uniform splits, octree.py:225), the roulette.
//  * Deeper steps (~1/3 of samples descend below level 2) would leave most
//    lanes idle if walked in place.  Descending samples are queued (16 B walk
//    starts per block in global memory, L2-resident), counting-sorted by
//    level-2 node, and served after the sampling loop by lanes that refill
//    independently from the queue and carry each walk to completion (the
//    child holding the sampled point comes from its per-point path of
//    sibling ranks).  A finished walk stores its residual in its owner's
//    creation-ordered slot and owners fold their slots in that ((a, s))
//    order, so a query's value never depends on which lane served its walks.
//  * FP32 terms and residuals, FP64 accumulation across chunks/subdomains.
//
// k_sto_warp (further down) is the same estimator with the paper's warp-shared
// RNG streams: 32 queries of a seeded shuffled order share
// the draws, so sampling is done once per warp and every walk is warp-uniform
// (no queue / sort / result slots; a walk level's child pairs are loaded by the
// warp's lanes at once into shared memory and summed from there).  The Coulomb
// (and winding) dense parts of both kernels run on the packed FP32 pipe
// (FADD2/FFMA2, dense_coulomb_pairs / dense_winding_pairs).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fs_common.cuh"
#include "fs_eval.h"
#include "fs_internal.h"

namespace fsb {

constexpr int kFastMaxLevels = 64;

struct FastView {
  const int4* __restrict__ topo;   // {first child (level order), child count, begin, end}
  const float4* __restrict__ cm;   // {cx, cy, cz, m0}
  const float2* __restrict__ m12;  // {m1, m2} (winding)
  const int32_t* __restrict__ lb;  // begin
  const float4* __restrict__ pa;   // permuted points {x, y, z, m0}
  const float4* __restrict__ pb;   // {m1, m2, 0, 0}
  const uint64_t* __restrict__ path;  // per point: sibling rank per level (ensure_path)
  const float4* __restrict__ cmp;  // Coulomb node pairs, packed (ensure_pairs; warp kernel)
  int path_bits, path_levels;
  int n1, base2, n2, first_multi;
  int per_chunk;                   // (a, s) samples per thread between drains
  int qcap;                        // queued walk starts per block
  int stage_kids;                  // (warp kernel) every node has <= 64 children: stage them
  float inv_diam[kFastMaxLevels];  // 1 / max(diam_level, 1e-12)
};



// two consecutive 16-byte records with one 256-bit read-only load (p 32-byte aligned)
__device__ __forceinline__ void ld_pair(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}

template <int KID>
__device__ __forceinline__ float fterm(float4 c, float2 w, float qx, float qy, float qz,
                                       const KParams& kp) {
  return contrib_fast<KID>(c.w, w.x, w.y, c.x, c.y, c.z, qx, qy, qz, kp);
}

template <int KID>
__device__ float leaf_exact(const FastView& V, int b, int e, float qx, float qy, float qz,
                            const KParams& kp) {
  float acc = 0.f;
  for (int j = b; j < e; ++j) {
    float4 u = V.pa[j];
    float2 w = make_float2(0.f, 0.f);
    if (KID == KID_WINDING) {
      float4 v = V.pb[j];
      w = make_float2(v.x, v.y);
    }
    acc += fterm<KID>(u, w, qx, qy, qz, kp);
  }
  return acc;
}

__device__ __forceinline__ float fdist(float4 c, float qx, float qy, float qz) {
  float dx = qx - c.x, dy = qy - c.y, dz = qz - c.z;
  float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  return d2 * rsqrt_ftz(fmaxf(d2, 1e-30f));
}

// roulette uniform from the top 24 bits of the same splitmix draw
__device__ __forceinline__ float draw24(uint64_t key, uint64_t ctr) {
  uint64_t x = mix64(key + (ctr + 1ull) * kGamma);
  return (float)(uint32_t)(x >> 40) * (1.0f / 16777216.0f);
}

#ifndef FSB_TILE
#define FSB_TILE 256
#endif
constexpr int kBlock = FSB_TILE;  // threads (= queries) per tile
constexpr int kOwnerBits = kBlock <= 256 ? 8 : (kBlock <= 512 ? 9 : 10);
#ifndef FSB_STO_MINB
#define FSB_STO_MINB (1024 / FSB_TILE)  // resident blocks per SM the register budget is sized for
#endif
#ifndef FSB_QCAP_MAX
#define FSB_QCAP_MAX 9216  // max queued walk starts per block (one drain per tile on C4)
#endif

// Walk starts, per block, SoA: int4 {owner | s << 8, a_ord, k (level-2 index), j}
// and uint2 {kr.lo, kr.hi} (roulette stream key).  Everything else a walk needs
// at level 2 (p_rr, ratio, control-variate term) is recomputed from the staged
// level-1/2 records in shared memory.
#ifndef FSB_KR_RECOMPUTE
#define FSB_KR_RECOMPUTE 1  // rederive the roulette key in the drain (16-byte walk starts)
#endif
constexpr size_t kWalkBytes = FSB_KR_RECOMPUTE ? 16 : 24;

extern __shared__ float4 sh_f4[];
extern __shared__ int4 sh_i4[];
extern __shared__ float2 sh_f2[];
extern __shared__ int sh_i[];
extern __shared__ uint2 sh_u2[];
extern __shared__ int2 sh_i2[];
extern __shared__ unsigned short sh_u16[];

// last index k in [lo, lo + cnt) whose begin (low 31 bits of sh_i[ob + k]) is <= j
__device__ __forceinline__ int child_search(int ob, int lo, int cnt, int j) {
  const int last = lo + cnt - 1;
  for (int step = cnt > 1 ? 1 << (31 - __clz(cnt - 1)) : 0; step > 0; step >>= 1) {
    const int t = min(lo + step, last);  // branch-free: probe a clamped index
    lo = (sh_i[ob + t] & 0x7fffffff) <= j ? t : lo;
  }
  return lo;
}

template <int RR>
__device__ __forceinline__ float rr_fast_t(float rp, float rc) {
  if (RR == 1) return 0.5f;
  if (RR == 2) return 1.0f;
  return fminf(fmaxf(rp, 1.0f) * rcp_ftz(fmaxf(rc, 1e-12f)), 1.0f);
}

// roulette: u < p with u the 24-bit draw; p == 1 needs no draw (u < 1 always)
template <int RR>
__device__ __forceinline__ bool survive(float p, uint64_t kr, uint64_t ctr) {
  if (RR == 2) return true;
  return p >= 1.0f || draw24(kr, ctr) < p;
}

#ifndef FSB_LUT_BITS
#define FSB_LUT_BITS 5
#endif
// index-draw buckets per subdomain (top FSB_LUT_BITS bits of the draw)
constexpr int kLutBits = FSB_LUT_BITS, kLut = 1 << kLutBits;

#ifndef FSB_WARP_DENSE2
#define FSB_WARP_DENSE2 1  // Coulomb dense part on the packed FP32 pipe
#endif
#ifndef FSB_DENSE_CHUNK
#define FSB_DENSE_CHUNK 16  // record pairs per FP32 partial of the dense part (0.513 / 0.499 / 0.494 ms at 4 / 8 / 16)
#endif
constexpr int kDenseChunk = FSB_DENSE_CHUNK;

// Coulomb dense part over level-2 records staged in shared memory as pairs
// {x0,x1,y0,y1}, {z0,z1,-m0,-m1} at sh_f4[o_p2 ...]: packed FP32 (FADD2/FFMA2),
// two records per instruction, the distance floor as r2 + floor^2 (see
// k_brute32_coulomb2), FP32 partials over 2 * kDenseChunk records in fully
// unrolled chunks folded into FP64.
__device__ __forceinline__ double dense_coulomb_pairs(int o_p2, int np2, float qx, float qy,
                                                      float qz, float dfloor) {
  const float2 nx = make_float2(-qx, -qx), ny = make_float2(-qy, -qy), nz = make_float2(-qz, -qz);
  const float f2 = dfloor * dfloor;
  const float2 fl2 = make_float2(f2, f2);
  auto pair_term = [&](int i, float2 a) {
    const float4 A = sh_f4[o_p2 + 2 * i], B = sh_f4[o_p2 + 2 * i + 1];
    const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx);
    const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny);
    const float2 dz = __fadd2_rn(make_float2(B.x, B.y), nz);
    const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __ffma2_rn(dz, dz, fl2)));
    const float2 ri = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
    return __ffma2_rn(make_float2(B.z, B.w), ri, a);
  };
  double acc = 0.0;
  int k = 0;
  for (; k + kDenseChunk <= np2; k += kDenseChunk) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll
    for (int u = 0; u < kDenseChunk; u += 2) {
      a0 = pair_term(k + u, a0);
      a1 = pair_term(k + u + 1, a1);
    }
    acc += (double)((a0.x + a0.y) + (a1.x + a1.y));
  }
  if (k < np2) {
    float2 a0 = make_float2(0.f, 0.f);
    for (; k < np2; ++k) a0 = pair_term(k, a0);
    acc += (double)(a0.x + a0.y);
  }
  return acc;
}

// stages level-2 records [base2, base2 + n2) as Coulomb pairs (odd tail: a massless copy)
__device__ __forceinline__ void stage_coulomb_pairs(const float4* __restrict__ cm, int base2,
                                                    int n2, int o_p2, int tid, int nthreads) {
  for (int i = tid; i < (n2 + 1) / 2; i += nthreads) {
    const float4 u = cm[base2 + 2 * i];
    const float4 v = 2 * i + 1 < n2 ? cm[base2 + 2 * i + 1] : make_float4(u.x, u.y, u.z, 0.f);
    sh_f4[o_p2 + 2 * i] = make_float4(u.x, v.x, u.y, v.y);
    sh_f4[o_p2 + 2 * i + 1] = make_float4(u.z, v.z, -u.w, -v.w);
  }
}

// Winding (dipole) dense part over level-2 records staged as pairs {x0,x1,y0,y1},
// {z0,z1,m0_0,m0_1}, {m1_0,m1_1,m2_0,m2_1}: (m . (p - q)) r^-3 / (4 pi) on the
// packed FP32 pipe, the floor as r2 + floor^2 (as the Coulomb form)
__device__ __forceinline__ double dense_winding_pairs(int o_p2, int np2, float qx, float qy,
                                                      float qz, float dfloor) {
  const float2 nx = make_float2(-qx, -qx), ny = make_float2(-qy, -qy), nz = make_float2(-qz, -qz);
  const float f2 = dfloor * dfloor;
  const float2 fl2 = make_float2(f2, f2);
  auto pair_term = [&](int i, float2 a) {
    const float4 A = sh_f4[o_p2 + 3 * i], B = sh_f4[o_p2 + 3 * i + 1], M = sh_f4[o_p2 + 3 * i + 2];
    const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx);
    const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny);
    const float2 dz = __fadd2_rn(make_float2(B.x, B.y), nz);
    const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __ffma2_rn(dz, dz, fl2)));
    const float2 ri = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
    const float2 ri3 = __fmul2_rn(__fmul2_rn(ri, ri), ri);
    const float2 dot = __ffma2_rn(make_float2(B.z, B.w), dx,
                                  __ffma2_rn(make_float2(M.x, M.y), dy,
                                             __fmul2_rn(make_float2(M.z, M.w), dz)));
    return __ffma2_rn(dot, ri3, a);
  };
  double acc = 0.0;
  int k = 0;
  for (; k + kDenseChunk <= np2; k += kDenseChunk) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll
    for (int u = 0; u < kDenseChunk; u += 2) {
      a0 = pair_term(k + u, a0);
      a1 = pair_term(k + u + 1, a1);
    }
    acc += (double)((a0.x + a0.y) + (a1.x + a1.y));
  }
  if (k < np2) {
    float2 a0 = make_float2(0.f, 0.f);
    for (; k < np2; ++k) a0 = pair_term(k, a0);
    acc += (double)(a0.x + a0.y);
  }
  return acc * kInv4Pi;
}

__device__ __forceinline__ void stage_winding_pairs(const float4* __restrict__ cm,
                                                    const float2* __restrict__ m12, int base2,
                                                    int n2, int o_p2, int tid, int nthreads) {
  for (int i = tid; i < (n2 + 1) / 2; i += nthreads) {
    const bool two = 2 * i + 1 < n2;
    const float4 u = cm[base2 + 2 * i];
    const float4 v = two ? cm[base2 + 2 * i + 1] : make_float4(u.x, u.y, u.z, 0.f);
    const float2 wu = m12[base2 + 2 * i];
    const float2 wv = two ? m12[base2 + 2 * i + 1] : make_float2(0.f, 0.f);
    sh_f4[o_p2 + 3 * i] = make_float4(u.x, v.x, u.y, v.y);
    sh_f4[o_p2 + 3 * i + 1] = make_float4(u.z, v.z, u.w, v.w);
    sh_f4[o_p2 + 3 * i + 2] = make_float4(wu.x, wv.x, wu.y, wv.y);
  }
}

// dense part dispatch for the packed kernels (Coulomb: 2, winding: 3 float4 per pair)
template <int KID>
__device__ __forceinline__ void stage_pairs(const FastView& V, int n2, int o_p2, int tid,
                                            int nthreads) {
  if (KID == KID_WINDING)
    stage_winding_pairs(V.cm, V.m12, V.base2, n2, o_p2, tid, nthreads);
  else
    stage_coulomb_pairs(V.cm, V.base2, n2, o_p2, tid, nthreads);
}
template <int KID>
__device__ __forceinline__ double dense_pairs(int o_p2, int np2, float qx, float qy, float qz,
                                              float dfloor) {
  return KID == KID_WINDING ? dense_winding_pairs(o_p2, np2, qx, qy, qz, dfloor)
                            : dense_coulomb_pairs(o_p2, np2, qx, qy, qz, dfloor);
}
template <int KID>
constexpr int pair_vecs() {
  return KID == KID_WINDING ? 3 : 2;
}

// sum of the Coulomb terms of the contiguous children [first, first + count)
// from the pair-interleaved records (ensure_pairs): one 32-byte load and packed
// FP32 arithmetic per two children, the floor as r2 + floor^2
__device__ __forceinline__ float children_coulomb_pairs(const float4* __restrict__ cmp,
                                                        const float4* __restrict__ cm, int first,
                                                        int count, float qx, float qy, float qz,
                                                        const KParams& kp) {
  const float2 nx = make_float2(-qx, -qx), ny = make_float2(-qy, -qy), nz = make_float2(-qz, -qz);
  const float f2 = kp.dfloor_f * kp.dfloor_f;
  const float2 fl2 = make_float2(f2, f2);
  auto pair_acc = [&](int r, float2 acc2) {
    float4 A, B;
    ld_pair(cmp + r, A, B);  // r even: records r, r + 1
    const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx);
    const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny);
    const float2 dz = __fadd2_rn(make_float2(B.x, B.y), nz);
    const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __ffma2_rn(dz, dz, fl2)));
    const float2 ri = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
    return __ffma2_rn(make_float2(B.z, B.w), ri, acc2);
  };
  const float2 z2 = make_float2(0.f, 0.f);
  const int e = first + count;
  int r = first;
  float ks = 0.f;
  if (r & 1) {
    ks += contrib_fast<KID_COULOMB>(cm[r].w, 0.f, 0.f, cm[r].x, cm[r].y, cm[r].z, qx, qy, qz, kp);
    ++r;
  }
  float2 a2 = z2, b2 = z2;
  for (; r + 3 < e; r += 4) {
    a2 = pair_acc(r, a2);
    b2 = pair_acc(r + 2, b2);
  }
  if (r + 1 < e) {
    a2 = pair_acc(r, a2);
    r += 2;
  }
  if (r < e) ks += contrib_fast<KID_COULOMB>(cm[r].w, 0.f, 0.f, cm[r].x, cm[r].y, cm[r].z, qx, qy, qz, kp);
  return ks + ((a2.x + a2.y) + (b2.x + b2.y));
}

template <int KID, int RR, bool PACK>
__global__ void __launch_bounds__(kBlock, FSB_STO_MINB)
    k_sto_fast(const __grid_constant__ FastView V, const double* __restrict__ q, int64_t n,
               const int32_t* __restrict__ qperm, int S, uint64_t seed, int64_t qoff, int share,
               KParams kp, float* __restrict__ res_g, unsigned char* __restrict__ queues,
               unsigned int* __restrict__ tile_ctr, float* __restrict__ out, int64_t* __restrict__ visited,
               int64_t* __restrict__ path_steps, int64_t* __restrict__ path_count) {
  // Dynamic shared memory, addressed by element index off the extern arrays
  // (all alias the same window), so every access is LDS [index + imm] with no
  // generic-pointer reconstruction.  Layout:
  //   16 B: s_q[kBlock] query coords, s_cm1[n1] {com, m0}, s_tp1[n1] topology,
  //         s_cm2[n2] {com, m0}
  //    8 B: s_w1[n1], s_w2[n2] {m1, m2} (winding), s_hq[kBlock] per-query RNG prefix
  //    4 B: s_b2[n2] begins (bit 31: multi-point leaf), s_seen, s_steps, s_count[4]
  //    2 B: s_lut[n1][kLut + 1] first candidate child per index-draw bucket
  const int n1 = V.n1, n2 = V.n2;
  const int o_cm1 = kBlock, o_tp1 = o_cm1 + n1, o_cm2 = o_tp1 + n1;
  const int o_w1 = 2 * (o_cm2 + n2), o_w2 = o_w1 + (KID == KID_WINDING ? n1 : 0);
  const int o_hq = o_w2 + (KID == KID_WINDING ? n2 : 0);
  const int o_b2 = 2 * (o_hq + kBlock);
  const int o_seen = o_b2 + n2, o_steps = o_seen + kBlock, o_count = o_steps + kBlock;
  const int o_t2 = (o_count + 5) / 2;  // (8-byte units, aligned) level-2 {first child | count << 25, points}
  const int o_hist = 2 * (o_t2 + n2);  // walk starts per level-2 node, then their offsets
  const int o_lut = 2 * (o_hist + n2 + (n2 & 1));
  // Coulomb: level-2 records also as packed pairs (16-B units, after the table)
  constexpr bool kPack = PACK && KID != KID_SMOOTH;
  const int o_p2 = (2 * (o_lut + n1 * (kLut + 1)) + 15) / 16;
#define s_q(i) sh_f4[(i)]
#define s_cm1(i) sh_f4[o_cm1 + (i)]
#define s_tp1(i) sh_i4[o_tp1 + (i)]
#define s_cm2(i) sh_f4[o_cm2 + (i)]
#define s_w1(i) sh_f2[o_w1 + (i)]
#define s_w2(i) sh_f2[o_w2 + (i)]
#define s_hq(i) sh_u2[o_hq + (i)]
#define s_b2(i) sh_i[o_b2 + (i)]
#define s_seen(i) sh_i[o_seen + (i)]
#define s_steps(i) sh_i[o_steps + (i)]
#define s_count(i) sh_i[o_count + (i)]
#define s_lut(i) sh_u16[o_lut + (i)]
#define s_hist(i) sh_i[o_hist + (i)]
#define s_t2(i) sh_i2[o_t2 + (i)]

  // two walk-start buffers: creation order (qa, qk) and sorted by level-2 node (sa, sk)
  int4* const qa = reinterpret_cast<int4*>(queues + (size_t)blockIdx.x * 2 * V.qcap * kWalkBytes);
  uint2* const qk = reinterpret_cast<uint2*>(qa + V.qcap);  // (unused with FSB_KR_RECOMPUTE)
  int4* const sa = FSB_KR_RECOMPUTE ? qa + V.qcap : reinterpret_cast<int4*>(qk + V.qcap);
  uint2* const sk = reinterpret_cast<uint2*>(sa + V.qcap);
  const int tid = threadIdx.x;
  const int nslot = n1 * S;
  // result slots of this block, slot-major: res[seq * kBlock + owner], seq = the
  // walk's creation index among its owner's walks this tile ((a, s) order)
  float* const my_res = res_g + (int64_t)blockIdx.x * kBlock * nslot;

  // ---- stage level 1 (root's children, level order 1..n1) and level 2
  for (int i = tid; i < n1; i += kBlock) {
    s_cm1(i) = V.cm[1 + i];
    s_tp1(i) = V.topo[1 + i];
    if (KID == KID_WINDING) s_w1(i) = V.m12[1 + i];
  }
  const bool l2_multi = V.first_multi <= 2;
  for (int i = tid; i < n2; i += kBlock) {
    s_cm2(i) = V.cm[V.base2 + i];
    if (KID == KID_WINDING) s_w2(i) = V.m12[V.base2 + i];
    int b = V.lb[V.base2 + i];
    const int4 tp = V.topo[V.base2 + i];
    if (l2_multi && tp.y == 0 && tp.w - tp.z > 1) b |= 0x80000000;
    s_b2(i) = b;
    s_t2(i) = make_int2(tp.y > 0 ? (tp.x | (tp.y << 25)) : 0, tp.w - tp.z);
  }
  if (kPack && !l2_multi) stage_pairs<KID>(V, n2, o_p2, tid, kBlock);
  if (tid < 4) s_count(tid) = 0;  // [0] queue length, [1] drain head
  s_seen(tid) = 0;
  s_steps(tid) = 0;
  for (int i = tid; i < n2; i += kBlock) s_hist(i) = 0;
  __syncthreads();
  // bucket table: j in bucket b (j - begin in [floor(b c / L), floor((b+1) c / L)],
  // c = count) lies in a child in [lut[b], lut[b+1]] (children are ordered by begin)
  for (int i = tid; i < n1 * (kLut + 1); i += kBlock) {
    const int a = i / (kLut + 1), b = i - a * (kLut + 1);
    const int4 tpa = s_tp1(a);
    int c = 0;
    if (tpa.y > 0) {
      int jb = tpa.z + (int)(((int64_t)b * (tpa.w - tpa.z)) >> kLutBits);
      if (jb > tpa.w - 1) jb = tpa.w - 1;
      const int k0 = tpa.x - V.base2;
      c = child_search(o_b2, k0, tpa.y, jb) - k0;
    }
    s_lut(i) = (unsigned short)c;
  }
  // query-independent counters: every sample of an internal subdomain a visits
  // a's children and the picked child (_core.py:195, 205); paths = samples
  int seen_base = n1, n_int = 0;
  for (int a = 0; a < n1; ++a) {
    const int4 tpa = s_tp1(a);
    if (tpa.y > 0) {
      seen_base += S * (tpa.y + 1);
      ++n_int;
    }
  }
  __syncthreads();

  const uint64_t hseed = mix64(seed + kGamma);
  const float id1 = V.inv_diam[1], id2 = V.inv_diam[2];
  const float2 w0 = make_float2(0.f, 0.f);

  // tiles are handed out dynamically (a block's tile count would otherwise
  // differ by one across blocks: up to 1/3 idle time on short launches)
  const int64_t ntiles = (n + kBlock - 1) / kBlock;
  while (true) {
    if (tid == 0) s_count(2) = (int)atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_count(2);
    if (tile >= ntiles) break;
    const int64_t base = tile * kBlock;
    float qx, qy, qz;
    bool live;
    {
      const int64_t t = base + tid;
      live = t < n;
      const int64_t qi = live ? (qperm ? (int64_t)qperm[t] : t) : 0;
      qx = live ? (float)q[3 * qi] : 0.f;
      qy = live ? (float)q[3 * qi + 1] : 0.f;
      qz = live ? (float)q[3 * qi + 2] : 0.f;
      s_q(tid) = make_float4(qx, qy, qz, 0.f);
      // stream key: the query's global index (reference), or with warp sharing
      // the index of its group of 2^share consecutive positions (paper recipe)
      const uint64_t hq = key_fold(
          hseed, share ? (uint64_t)((t + qoff) >> share) : (uint64_t)(qi + qoff));
      s_hq(tid) = make_uint2((uint32_t)hq, (uint32_t)(hq >> 32));
    }

    // ---- dense part (see the header): every level-2 record, FP32 partial
    // sums over 16 records folded into the FP64 accumulator
    double acc = 0.0;
    if (kPack && !l2_multi) {
      acc = dense_pairs<KID>(o_p2, (n2 + 1) / 2, qx, qy, qz, kp.dfloor_f);
    } else if (!l2_multi) {
      int k = 0;
      for (; k + 16 <= n2; k += 16) {
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
        for (int u = 0; u < 16; u += 4) {
          p0 += fterm<KID>(s_cm2(k + u), KID == KID_WINDING ? s_w2(k + u) : w0, qx, qy, qz, kp);
          p1 += fterm<KID>(s_cm2(k + u + 1), KID == KID_WINDING ? s_w2(k + u + 1) : w0, qx, qy,
                           qz, kp);
          p2 += fterm<KID>(s_cm2(k + u + 2), KID == KID_WINDING ? s_w2(k + u + 2) : w0, qx, qy,
                           qz, kp);
          p3 += fterm<KID>(s_cm2(k + u + 3), KID == KID_WINDING ? s_w2(k + u + 3) : w0, qx, qy,
                           qz, kp);
        }
        acc += (double)((p0 + p1) + (p2 + p3));
      }
      float p0 = 0.f;
      for (; k < n2; ++k)
        p0 += fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
      acc += (double)p0;
    } else {
      for (int k = 0; k < n2; ++k) {
        float v;
        if (s_b2(k) < 0) {
          const int4 tp = V.topo[V.base2 + k];
          v = leaf_exact<KID>(V, tp.z, tp.w, qx, qy, qz, kp);
        } else {
          v = fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
        }
        acc += (double)v;
      }
    }
    int steps = 0;

    // ---- sampling, in chunks of per_chunk (a, s) pairs (block-uniform), each
    // followed by a drain of the walks it queued (one chunk per tile unless
    // n1 * S is large)
    // one sample (a, s): index draw, level-1 step from shared memory, roulette
    auto sample = [&](int a_ord, int sm, const int4& tpa, int k0, int lut0, float rp_a,
                      uint64_t ha) {
      const uint64_t hs = key_fold(ha, (uint64_t)sm);
      const uint64_t ki = key_fold(hs, 0), kr = key_fold(hs, 1);
      // index draw, exactly as _core.py:166-169 (uniform_draw(ki, 0))
      const uint64_t x = mix64(ki + kGamma);
      const double u0 = __ull2double_rn(x >> 11) * (1.0 / 9007199254740992.0);
      int j = tpa.z + (int)__dmul_rn(u0, (double)(tpa.w - tpa.z));
      if (j >= tpa.w) j = tpa.w - 1;
      // level-1 step from shared memory (the swap at `a` is in the dense
      // part): bucket table, then a short forward scan over child begins
      const int bkt = (int)(x >> (64 - kLutBits));
      int c = s_lut(lut0 + bkt);
      const int ce = s_lut(lut0 + bkt + 1);
      while (c < ce && (s_b2(k0 + c + 1) & 0x7fffffff) <= j) ++c;
      const int lo = k0 + c;
      const float rc = fdist(s_cm2(lo), qx, qy, qz) * id2;
      const float p = rr_fast_t<RR>(rp_a, rc);
      // (lanes past the end of the query set sample too; results dropped)
      if (survive<RR>(p, kr, 0)) {  // descends: queue the walk start
        const int pos = atomicAdd(&s_count(0), 1);
        atomicAdd(&s_hist(lo), 1);
#if FSB_KR_RECOMPUTE
        qa[pos] = make_int4(tid | (steps << kOwnerBits), a_ord | (sm << 8), lo, j);
#else
        qa[pos] = make_int4(tid | (steps << kOwnerBits), a_ord, lo, j);
        qk[pos] = make_uint2((uint32_t)kr, (uint32_t)(kr >> 32));
#endif
        ++steps;
      }
    };
    auto leaf_term = [&](int a_ord, const int4& tpa) {
      return (double)((tpa.w - tpa.z > 1)
                          ? leaf_exact<KID>(V, tpa.z, tpa.w, qx, qy, qz, kp)
                          : fterm<KID>(s_cm1(a_ord), KID == KID_WINDING ? s_w1(a_ord) : w0, qx,
                                       qy, qz, kp));
    };
    const uint2 hqv = s_hq(tid);
    const uint64_t hq = ((uint64_t)hqv.y << 32) | hqv.x;

    for (int f0 = 0; f0 < nslot; f0 += V.per_chunk) {
      const int f1 = min(f0 + V.per_chunk, nslot);
      if (S == 1 && f1 - f0 == n1) {  // the common case: one sample per subdomain
        for (int a_ord = 0; a_ord < n1; ++a_ord) {  // block-uniform
          const int4 tpa = s_tp1(a_ord);
          if (tpa.y == 0) {  // leaf subdomain: exact term, never sampled
            acc += leaf_term(a_ord, tpa);
            continue;
          }
          const float rp_a = fdist(s_cm1(a_ord), qx, qy, qz) * id1;
          sample(a_ord, 0, tpa, tpa.x - V.base2, a_ord * (kLut + 1), rp_a,
                 key_fold(hq, (uint64_t)a_ord));
        }
      } else {
        int a_ord = f0 / S, s = f0 - a_ord * S;
        for (int f = f0; f < f1; ++a_ord, s = 0) {  // block-uniform
          const int4 tpa = s_tp1(a_ord);
          if (tpa.y == 0) {  // leaf subdomain: exact term, never sampled
            if (s == 0) acc += leaf_term(a_ord, tpa);
            const int take = min(S - s, f1 - f);
            f += take;
            continue;
          }
          const int k0 = tpa.x - V.base2, lut0 = a_ord * (kLut + 1);
          const float rp_a = fdist(s_cm1(a_ord), qx, qy, qz) * id1;
          const uint64_t ha = key_fold(hq, (uint64_t)a_ord);
          for (; s < S && f < f1; ++s, ++f) sample(a_ord, s, tpa, k0, lut0, rp_a, ha);
        }
      }
      __syncthreads();

      // ---- counting sort of the walk starts by level-2 node into (sa, sk):
      // lanes of a warp then sum the same node's children with the same load
      // instructions (one request per distinct node rather than per lane), and
      // the walk-start reads themselves are coalesced
      {
        const int cnt = s_count(0);
        const int per = (n2 + kBlock - 1) / kBlock, b0 = min(tid * per, n2),
                  b1 = min(b0 + per, n2);
        int seg = 0;
        for (int b = b0; b < b1; ++b) seg += s_hist(b);
        const int lane = tid & 31, wid = tid >> 5;
        int incl = seg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        __shared__ int s_wtot[kBlock / 32];  // per-warp totals of the scan
        if (lane == 31) s_wtot[wid] = incl;
        __syncthreads();
        int run = incl - seg;
        for (int w = 0; w < wid; ++w) run += s_wtot[w];
        for (int b = b0; b < b1; ++b) {
          const int c = s_hist(b);
          s_hist(b) = run;
          run += c;
        }
        __syncthreads();
        for (int i = tid; i < cnt; i += kBlock) {
          const int4 wa = qa[i];
          const int pos = atomicAdd(&s_hist(wa.z), 1);
          sa[pos] = wa;
          if (!FSB_KR_RECOMPUTE) sk[pos] = qk[i];
        }
        __syncthreads();
        for (int b = tid; b < n2; b += kBlock) s_hist(b) = 0;
      }
      // ---- drain: every lane holding no walk takes the next start (warp-
      // aggregated claim on a shared head counter) and carries it to completion
      // one level per iteration, so lanes refill independently and no block
      // barrier separates the levels.
      {
        const int cnt = s_count(0);
        const int lane = tid & 31;
        bool act = false;
        int owner = 0, slot = 0, lvl = 2, jj = 0, count_a = 1;
        int4 tp = make_int4(0, 0, 0, 0);  // {first child, count, begin, end} of the walk's node
        uint64_t path = 0;
        float prr = 1.f, rp = 0.f, cvn = 0.f, resid = 0.f;
        float4 qq = make_float4(0.f, 0.f, 0.f, 0.f);
        uint64_t kr = 0;
        while (true) {
          const unsigned need = __ballot_sync(0xffffffffu, !act);
          if (need) {
            int head = 0;
            if (lane == 0) head = atomicAdd(&s_count(1), __popc(need));
            head = __shfl_sync(0xffffffffu, head, 0);
            const int idx = head + __popc(need & ((1u << lane) - 1u));
            if (!act && idx < cnt) {
              const int4 wa = sa[idx];  // consecutive lanes, consecutive records
              owner = wa.x & ((1 << kOwnerBits) - 1);
              const int wa_ord = FSB_KR_RECOMPUTE ? (wa.y & 0xff) : wa.y, k = wa.z;
              slot = wa.x >> kOwnerBits;  // creation index among the owner's walks
              jj = wa.w;
              path = V.path[jj];
#if FSB_KR_RECOMPUTE
              {  // the roulette stream key of (owner query, a, s), as in the sampling
                const uint2 hv = s_hq(owner);
                const uint64_t hq_o = ((uint64_t)hv.y << 32) | hv.x;
                kr = key_fold(key_fold(key_fold(hq_o, (uint64_t)wa_ord), (uint64_t)(wa.y >> 8)), 1);
              }
#else
              const uint2 wk = sk[idx];
              kr = ((uint64_t)wk.y << 32) | wk.x;
#endif
              qq = s_q(owner);
              const int4 tpa = s_tp1(wa_ord);
              count_a = tpa.w - tpa.z;
              const float4 c2 = s_cm2(k);
              rp = fdist(c2, qq.x, qq.y, qq.z) * id2;
              prr = rr_fast_t<RR>(fdist(s_cm1(wa_ord), qq.x, qq.y, qq.z) * id1, rp);
              cvn = fterm<KID>(c2, KID == KID_WINDING ? s_w2(k) : w0, qq.x, qq.y, qq.z, kp);
              // level-2 topology from shared memory (begin only feeds end - begin)
              const int2 t2 = s_t2(k);
              tp = make_int4(t2.x & 0x1ffffff, (int)((unsigned)t2.x >> 25), 0, t2.y);
              lvl = 2;
              resid = 0.f;
              act = true;
            }
          }
          if (!__any_sync(0xffffffffu, act)) break;
          if (!act) continue;
          // one level: sum the node's contiguous children, pick the child
          // holding the sampled point, commit the swap, roulette
          bool cont = false;
          if (tp.y > 0) {
            const bool cmulti = lvl + 1 >= V.first_multi;
            float ks0 = 0.f, ks1 = 0.f;
            int le = 0;  // children whose begin <= j: the last of them holds j
            int c = 0;
            if (!cmulti && lvl < V.path_levels) {
              // the sampled point's path gives the child's rank: only the
              // aggregates are read (one 16-byte load per child)
              le = 1 + (int)((path >> (V.path_bits * lvl)) & ((1u << V.path_bits) - 1u));
              // 32-byte loads of child pairs (one request per two children).  (The
              // pair-interleaved copy k_sto_warp uses measured slower here: these
              // lanes walk different nodes, and the picked child is reread from cm.)
              if (tp.x & 1) {
                ks0 += fterm<KID>(V.cm[tp.x], KID == KID_WINDING ? V.m12[tp.x] : w0, qq.x, qq.y,
                                  qq.z, kp);
                c = 1;
              }
              for (; c + 3 < tp.y; c += 4) {
                const int r = tp.x + c;
                float4 c0, c1, c2, c3;
                ld_pair(V.cm + r, c0, c1);
                ld_pair(V.cm + r + 2, c2, c3);
                ks0 += fterm<KID>(c0, KID == KID_WINDING ? V.m12[r] : w0, qq.x, qq.y, qq.z, kp);
                ks1 += fterm<KID>(c1, KID == KID_WINDING ? V.m12[r + 1] : w0, qq.x, qq.y, qq.z,
                                  kp);
                ks0 += fterm<KID>(c2, KID == KID_WINDING ? V.m12[r + 2] : w0, qq.x, qq.y, qq.z,
                                  kp);
                ks1 += fterm<KID>(c3, KID == KID_WINDING ? V.m12[r + 3] : w0, qq.x, qq.y, qq.z,
                                  kp);
              }
              for (; c < tp.y; ++c)
                ks0 += fterm<KID>(V.cm[tp.x + c], KID == KID_WINDING ? V.m12[tp.x + c] : w0, qq.x,
                                  qq.y, qq.z, kp);
            } else if (!cmulti) {
              for (; c + 1 < tp.y; c += 2) {
                const int r = tp.x + c;
                const float4 c0 = V.cm[r], c1 = V.cm[r + 1];
                const int b0 = V.lb[r], b1 = V.lb[r + 1];
                const float2 u0 = KID == KID_WINDING ? V.m12[r] : w0;
                const float2 u1 = KID == KID_WINDING ? V.m12[r + 1] : w0;
                ks0 += fterm<KID>(c0, u0, qq.x, qq.y, qq.z, kp);
                ks1 += fterm<KID>(c1, u1, qq.x, qq.y, qq.z, kp);
                le += (b0 <= jj) + (b1 <= jj);
              }
            }
            for (; c < tp.y; ++c) {
              const int r = tp.x + c;
              const float4 cr = V.cm[r];
              const float2 wr = KID == KID_WINDING ? V.m12[r] : w0;
              float v;
              if (cmulti) {
                int4 tc = V.topo[r];
                v = (tc.y == 0 && tc.w - tc.z > 1)
                        ? leaf_exact<KID>(V, tc.z, tc.w, qq.x, qq.y, qq.z, kp)
                        : fterm<KID>(cr, wr, qq.x, qq.y, qq.z, kp);
              } else {
                v = fterm<KID>(cr, wr, qq.x, qq.y, qq.z, kp);
              }
              ks0 += v;
              le += V.lb[r] <= jj;
            }
            const float ks = ks0 + ks1;
            const int cidx = tp.x + le - 1;
            const float4 cch = V.cm[cidx];  // L1 hit: just streamed
            atomicAdd(&s_seen(owner), tp.y + 1);
            // swap / (p_agg * p_rr), p_agg = points(node) / points(a)
            resid += (ks - cvn) * ((float)count_a * rcp_ftz((float)(tp.w - tp.z) * prr));
            const float rc =
                fdist(cch, qq.x, qq.y, qq.z) * V.inv_diam[min(lvl + 1, kFastMaxLevels - 1)];
            const float p = rr_fast_t<RR>(rp, rc);
            if (survive<RR>(p, kr, (uint64_t)(lvl - 1))) {  // counter = levels descended
              cont = true;
              atomicAdd(&s_steps(owner), 1);
              const float2 wc = KID == KID_WINDING ? V.m12[cidx] : w0;
              cvn = fterm<KID>(cch, wc, qq.x, qq.y, qq.z, kp);
              prr *= p;
              rp = rc;
              tp = V.topo[cidx];
              ++lvl;
            }
          }
          if (!cont) {
            my_res[slot * kBlock + owner] = resid;
            act = false;
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        s_count(0) = 0;
        s_count(1) = 0;
      }
      __syncthreads();
    }

    // owners fold their walks' residuals in creation ((a, s)) order: the value
    // is query-intrinsic whatever lane served which walk
    double acc_deep = 0.0;
    for (int k2 = 0; k2 < steps; ++k2) acc_deep += (double)my_res[k2 * kBlock + tid];
    const int seen = seen_base + s_seen(tid);
    steps += s_steps(tid);
    s_seen(tid) = 0;
    s_steps(tid) = 0;
    const double total = acc + acc_deep / (double)S;
    if (live) {
      const int64_t t = base + tid;
      const int64_t qi = qperm ? (int64_t)qperm[t] : t;
      out[qi] = (float)total;
      if (visited) visited[qi] = seen;
      if (path_steps) path_steps[qi] = steps;
      if (path_count) path_count[qi] = (int64_t)S * n_int;
    }
    __syncthreads();
  }
#undef s_q
#undef s_cm1
#undef s_tp1
#undef s_cm2
#undef s_w1
#undef s_w2
#undef s_hq
#undef s_b2
#undef s_seen
#undef s_steps
#undef s_count
#undef s_lut
#undef s_hist
#undef s_t2
}

// ================================================ warp-shared streams (paper)
// The paper's GPU recipe: the 32 queries of a warp, taken
// in a seeded shuffled order, share the index and roulette streams (key = the
// group index (t + qoff) >> 5).  Same estimator per query as k_sto_fast with
// share = 5, but the shared draws turn the walk into warp-uniform work:
//  * sampling: lane L computes the (a, s) pair f0 + L (6 mixes once per warp
//    instead of once per lane), and the per-level roulette uniforms of a walk
//    in parallel (lane L holds the draw with counter L);
//  * walks: every lane descends the same path (same sampled point), so child
//    records are warp-broadcast loads and the control flow is uniform; each
//    lane keeps its own roulette state (p depends on the query) and stops
//    committing once its roulette fails; the walk ends when no lane is alive.
//    No queue, no sort, no result slots: residuals accumulate in (a, s) order.
#ifndef FSB_WARP_BLOCK
#define FSB_WARP_BLOCK 512  // with 2 blocks/SM: 0.476 vs 0.482 ms at 256 x 4 (same bits)
#endif
constexpr int kWarpBlock = FSB_WARP_BLOCK;
#ifdef FSB_WARP_STATS
__device__ unsigned long long g_warp_stats[8];
#define WSTAT(i, v) \
  if (lane == 0) atomicAdd(&g_warp_stats[i], (unsigned long long)(v))
#else
#define WSTAT(i, v)
#endif
#ifndef FSB_WARP_MINB
#define FSB_WARP_MINB (1024 / FSB_WARP_BLOCK)  // 1024 threads/SM: 64 registers
#endif

#ifndef FSB_WARP_STAGE_KIDS
#define FSB_WARP_STAGE_KIDS 1  // stage a walk level's child pairs in shared memory
#endif
constexpr int kKidPairs = 33;  // staged pairs per warp: up to 64 children (d <= 4)

// The children [first, first + count) of a walk-level node as the global pair
// records covering them (pairs p0 .. p0 + np - 1 of ensure_pairs' table), loaded
// by the warp's lanes at once (one 32-byte load per lane) into the warp's
// shared buffer -- one L2 round trip per level instead of one per two pair
// loads -- with the masses of the halves outside the range zeroed.  Returns np.
__device__ __forceinline__ int stage_kid_pairs(float4* __restrict__ buf,
                                               const float4* __restrict__ cmp, int first,
                                               int count, int lane) {
  const int p0 = first >> 1, np = ((first + count - 1) >> 1) - p0 + 1;
  __syncwarp();  // the previous level's readers are done
  for (int k = lane; k < np; k += 32) {
    float4 A, B;
    ld_pair(cmp + 2 * (p0 + k), A, B);
    if (k == 0 && (first & 1)) B.z = 0.f;                     // record first - 1
    if (k == np - 1 && ((first + count) & 1)) B.w = 0.f;      // record first + count
    buf[2 * k] = A;
    buf[2 * k + 1] = B;
  }
  __syncwarp();
  return np;
}
// Coulomb sum over the staged pairs (broadcast LDS), packed FP32, the floor as
// r2 + floor^2 (children_coulomb_pairs' arithmetic per pair)
__device__ __forceinline__ float staged_kid_sum(const float4* __restrict__ buf, int np, float qx,
                                                float qy, float qz, float dfloor) {
  const float2 nx = make_float2(-qx, -qx), ny = make_float2(-qy, -qy), nz = make_float2(-qz, -qz);
  const float f2 = dfloor * dfloor;
  const float2 fl2 = make_float2(f2, f2);
  auto pair_acc = [&](int k, float2 acc2) {
    const float4 A = buf[2 * k], B = buf[2 * k + 1];
    const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx);
    const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny);
    const float2 dz = __fadd2_rn(make_float2(B.x, B.y), nz);
    const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __ffma2_rn(dz, dz, fl2)));
    const float2 ri = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
    return __ffma2_rn(make_float2(B.z, B.w), ri, acc2);
  };
  float2 a2 = make_float2(0.f, 0.f), b2 = a2;
  int k = 0;
  for (; k + 1 < np; k += 2) {
    a2 = pair_acc(k, a2);
    b2 = pair_acc(k + 1, b2);
  }
  if (k < np) a2 = pair_acc(k, a2);
  return (a2.x + a2.y) + (b2.x + b2.y);
}
// {cx, cy, cz, m0} of the staged record at offset i from pair p0's first record
__device__ __forceinline__ float4 staged_kid(const float4* __restrict__ buf, int i) {
  const float4 A = buf[2 * (i >> 1)], B = buf[2 * (i >> 1) + 1];
  return (i & 1) ? make_float4(A.y, A.w, B.y, -B.w) : make_float4(A.x, A.z, B.x, -B.z);
}

template <int KID, int RR, bool PACK>
__global__ void __launch_bounds__(kWarpBlock, FSB_WARP_MINB)
    k_sto_warp(const __grid_constant__ FastView V, const double* __restrict__ q, int64_t n,
               const int32_t* __restrict__ qperm, int S, uint64_t seed, int64_t qoff, KParams kp,
               unsigned int* __restrict__ chunk_ctr, float* __restrict__ out,
               int64_t* __restrict__ visited, int64_t* __restrict__ path_steps,
               int64_t* __restrict__ path_count, int shuffled) {
  // shared layout: 16 B s_cm1[n1] {com, m0}, s_tp1[n1] topology, s_cm2[n2];
  // 8 B s_w1[n1], s_w2[n2] (winding), s_t2[n2] {first child | count << 25, points};
  // 4 B s_b2[n2] begins; 2 B s_lut[n1][kLut + 1]
  const int n1 = V.n1, n2 = V.n2;
  // Coulomb: level-2 records also as packed pairs {x0,x1,y0,y1}, {z0,z1,-m0,-m1}
  constexpr bool kPack = KID == KID_COULOMB && FSB_WARP_DENSE2;  // packed walk levels
  constexpr bool kStageKids = kPack && FSB_WARP_STAGE_KIDS;
  constexpr bool pack = PACK && KID != KID_SMOOTH;                // packed dense part
  const int np2 = pack ? (n2 + 1) / 2 : 0;
  // (16-B units) the warps' child-pair buffers first, then the level-1/2 tables
  constexpr int kKidBuf = kStageKids ? (kWarpBlock / 32) * 2 * kKidPairs : 0;
  const int o_cm1 = kKidBuf, o_tp1 = o_cm1 + n1, o_cm2 = o_tp1 + n1, o_p2 = o_cm2 + n2;
  const int o_w1 = 2 * (o_p2 + pair_vecs<KID>() * np2),
            o_w2 = o_w1 + (KID == KID_WINDING ? n1 : 0);
  const int o_t2 = o_w2 + (KID == KID_WINDING ? n2 : 0);
  const int o_b2 = 2 * (o_t2 + n2);
  const int o_lut = 2 * (o_b2 + n2);
#define s_cm1(i) sh_f4[o_cm1 + (i)]
#define s_tp1(i) sh_i4[o_tp1 + (i)]
#define s_cm2(i) sh_f4[o_cm2 + (i)]
#define s_w1(i) sh_f2[o_w1 + (i)]
#define s_w2(i) sh_f2[o_w2 + (i)]
#define s_t2(i) sh_i2[o_t2 + (i)]
#define s_b2(i) sh_i[o_b2 + (i)]
#define s_lut(i) sh_u16[o_lut + (i)]
  const int o_int = o_lut + n1 * (kLut + 1), o_leaf = o_int + n1;  // 2 B subdomain lists
#define s_int(i) sh_u16[o_int + (i)]
#define s_leaf(i) sh_u16[o_leaf + (i)]
  // per-warp sample table (16-B units, after the 2-B lists): 32 x {a_ord, lo, j, u0},
  // 32 x {kr.lo, kr.hi, u1, u2}, 32 x {path.lo, path.hi, -, -}
  const int o_smp = (o_leaf + n1 + 7) / 8;
  const int tid = threadIdx.x, lane = tid & 31;
  int4* const s_smp = reinterpret_cast<int4*>(sh_i4 + o_smp) + (tid >> 5) * 96;
  // per-warp staging of a walk level's child pairs (Coulomb): 2 float4 per pair
  float4* const s_kid = sh_f4 + (tid >> 5) * 2 * kKidPairs;
  for (int i = tid; i < n1; i += kWarpBlock) {
    s_cm1(i) = V.cm[1 + i];
    s_tp1(i) = V.topo[1 + i];
    if (KID == KID_WINDING) s_w1(i) = V.m12[1 + i];
  }
  const bool l2_multi = V.first_multi <= 2;
  for (int i = tid; i < n2; i += kWarpBlock) {
    s_cm2(i) = V.cm[V.base2 + i];
    if (KID == KID_WINDING) s_w2(i) = V.m12[V.base2 + i];
    int b = V.lb[V.base2 + i];
    const int4 tp = V.topo[V.base2 + i];
    if (l2_multi && tp.y == 0 && tp.w - tp.z > 1) b |= 0x80000000;
    s_b2(i) = b;
    s_t2(i) = make_int2(tp.y > 0 ? (tp.x | (tp.y << 25)) : 0, tp.w - tp.z);
  }
  if (pack) stage_pairs<KID>(V, n2, o_p2, tid, kWarpBlock);
  __syncthreads();
  for (int i = tid; i < n1 * (kLut + 1); i += kWarpBlock) {
    const int a = i / (kLut + 1), b = i - a * (kLut + 1);
    const int4 tpa = s_tp1(a);
    int c = 0;
    if (tpa.y > 0) {
      int jb = tpa.z + (int)(((int64_t)b * (tpa.w - tpa.z)) >> kLutBits);
      if (jb > tpa.w - 1) jb = tpa.w - 1;
      const int k0 = tpa.x - V.base2;
      c = child_search(o_b2, k0, tpa.y, jb) - k0;
    }
    s_lut(i) = (unsigned short)c;
  }
  // internal subdomains (sampled) and leaf subdomains (exact), in order
  int seen_base = n1, n_int = 0, n_leaf = 0;
  for (int a = 0; a < n1; ++a) {
    const int4 tpa = s_tp1(a);
    if (tpa.y > 0) {
      seen_base += S * (tpa.y + 1);
      if (tid == 0) s_int(n_int) = (unsigned short)a;
      ++n_int;
    } else {
      if (tid == 0) s_leaf(n_leaf) = (unsigned short)a;
      ++n_leaf;
    }
  }
  __syncthreads();

  const uint64_t hseed = mix64(seed + kGamma);
  const uint64_t shuf_h = shuffle_key(seed);
  const float id1 = V.inv_diam[1], id2 = V.inv_diam[2];
  const float2 w0 = make_float2(0.f, 0.f);
  const int nslot = n_int * S;
  const float inv_s = __frcp_rn((float)S);
  const int64_t nchunks = (n + 31) / 32;
  // 32-query chunks from a global counter; the next chunk is claimed one chunk
  // ahead so the atomic's latency hides behind the current chunk
  unsigned int next = 0;
  if (lane == 0) next = atomicAdd(chunk_ctr, 1u);
  next = __shfl_sync(0xffffffffu, next, 0);
  while (true) {
    const unsigned int ch = next;
    if ((int64_t)ch >= nchunks) break;
    unsigned int claim = 0;
    if (lane == 0) claim = atomicAdd(chunk_ctr, 1u);
    const int64_t t = (int64_t)ch * 32 + lane;
    const bool live = t < n;
    // shuffled order computed in place (fsb_shuffle_order's permutation): the
    // 32 positions of a chunk share one window
    uint32_t wks[4] = {0, 0, 0, 0};
    if (shuffled) shuffle_window_keys(shuf_h, qoff, t & ~(kShuffleWindowC - 1), wks);
    auto query_of = [&](int64_t tt) -> int64_t {
      return shuffled ? shuffled_position(tt, n, wks) : (qperm ? (int64_t)qperm[tt] : tt);
    };
    float qx = 0.f, qy = 0.f, qz = 0.f;
    if (live) {  // (the index is recomputed for the stores: fewer live registers)
      const int64_t qi = query_of(t);
      qx = (float)q[3 * qi];
      qy = (float)q[3 * qi + 1];
      qz = (float)q[3 * qi + 2];
    }
    const uint64_t hq = key_fold(hseed, (uint64_t)(((int64_t)ch * 32 + qoff) >> 5));

    // ---- dense part: every level-2 record (as k_sto_fast) + leaf subdomains
    double acc = 0.0;
    if (pack && !l2_multi) {
      acc = dense_pairs<KID>(o_p2, np2, qx, qy, qz, kp.dfloor_f);
    } else if (!l2_multi) {
      int k = 0;
      for (; k + 16 <= n2; k += 16) {
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
        for (int u = 0; u < 16; u += 4) {
          p0 += fterm<KID>(s_cm2(k + u), KID == KID_WINDING ? s_w2(k + u) : w0, qx, qy, qz, kp);
          p1 += fterm<KID>(s_cm2(k + u + 1), KID == KID_WINDING ? s_w2(k + u + 1) : w0, qx, qy,
                           qz, kp);
          p2 += fterm<KID>(s_cm2(k + u + 2), KID == KID_WINDING ? s_w2(k + u + 2) : w0, qx, qy,
                           qz, kp);
          p3 += fterm<KID>(s_cm2(k + u + 3), KID == KID_WINDING ? s_w2(k + u + 3) : w0, qx, qy,
                           qz, kp);
        }
        acc += (double)((p0 + p1) + (p2 + p3));
      }
      float p0 = 0.f;
      for (; k < n2; ++k)
        p0 += fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
      acc += (double)p0;
    } else {
      for (int k = 0; k < n2; ++k) {
        float v;
        if (s_b2(k) < 0) {
          const int4 tp = V.topo[V.base2 + k];
          v = leaf_exact<KID>(V, tp.z, tp.w, qx, qy, qz, kp);
        } else {
          v = fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
        }
        acc += (double)v;
      }
    }
    for (int l = 0; l < n_leaf; ++l) {  // leaf subdomains: exact, never sampled
      const int a_ord = s_leaf(l);
      const int4 tpa = s_tp1(a_ord);
      acc += (double)((tpa.w - tpa.z > 1)
                            ? leaf_exact<KID>(V, tpa.z, tpa.w, qx, qy, qz, kp)
                            : fterm<KID>(s_cm1(a_ord), KID == KID_WINDING ? s_w1(a_ord) : w0, qx,
                                         qy, qz, kp));
    }

    int seen = seen_base, steps = 0;
    float acc_deep = 0.f;  // FP32 sum of the walks' residuals (<= n1 * S terms)
    for (int f0 = 0; f0 < nslot; f0 += 32) {
      // lane L draws sample f0 + L for the whole warp: index draw exactly as
      // _core.py:166-169, level-1 step from shared memory
      // the warp's sample table (broadcast reads below): a_ord < 0 = no sample
      {
        int my_a = -1, my_lo = 0, my_j = 0;
        uint64_t my_kr = 0;
        float my_u0 = 0.f, my_u1 = 0.f, my_u2 = 0.f;  // roulette draws, counters 0..2
        uint64_t my_path = 0;  // the sampled point's sibling ranks (loaded early)
        const int f = f0 + lane;
        if (f < nslot) {
          const int ai = f / S, sm = f - ai * S;
          const int a_ord = s_int(ai);
          const int4 tpa = s_tp1(a_ord);
          {
            const uint64_t hs = key_fold(key_fold(hq, (uint64_t)a_ord), (uint64_t)sm);
            const uint64_t ki = key_fold(hs, 0);
            my_kr = key_fold(hs, 1);
            const uint64_t x = mix64(ki + kGamma);
            const double u0 = __ull2double_rn(x >> 11) * (1.0 / 9007199254740992.0);
            int j = tpa.z + (int)__dmul_rn(u0, (double)(tpa.w - tpa.z));
            if (j >= tpa.w) j = tpa.w - 1;
            const int k0 = tpa.x - V.base2, lut0 = a_ord * (kLut + 1);
            const int bkt = (int)(x >> (64 - kLutBits));
            int c = s_lut(lut0 + bkt);
            const int ce = s_lut(lut0 + bkt + 1);
            while (c < ce && (s_b2(k0 + c + 1) & 0x7fffffff) <= j) ++c;
            my_a = a_ord;
            my_lo = k0 + c;
            my_j = j;
            my_path = V.path[j];
            if (RR != 2) {
              my_u0 = draw24(my_kr, 0);
              my_u1 = draw24(my_kr, 1);
              my_u2 = draw24(my_kr, 2);
            }
          }
        }
        __syncwarp();  // the previous round's readers are done
        s_smp[lane] = make_int4(my_a, my_lo, my_j, __float_as_int(my_u0));
        s_smp[32 + lane] = make_int4((int)(uint32_t)my_kr, (int)(uint32_t)(my_kr >> 32),
                                     __float_as_int(my_u1), __float_as_int(my_u2));
        s_smp[64 + lane] = make_int4((int)(uint32_t)my_path, (int)(uint32_t)(my_path >> 32), 0, 0);
        __syncwarp();
      }
      const int cnt = min(32, nslot - f0);
      for (int i = 0; i < cnt; ++i) {
        const int4 sa = s_smp[i];
        const int a_ord = sa.x;
        if (a_ord < 0) continue;  // warp-uniform
        const int lo = sa.y, jj = sa.z;
        const float ua = __int_as_float(sa.w);
        const int4 tpa = s_tp1(a_ord);
        const float fcount_a = (float)(tpa.w - tpa.z);
        const float4 c2 = s_cm2(lo);
        float rp = fdist(c2, qx, qy, qz) * id2;
        float prr = rr_fast_t<RR>(fdist(s_cm1(a_ord), qx, qy, qz) * id1, rp);
        bool alive = live && (RR == 2 || prr >= 1.f || ua < prr);
        WSTAT(6, 1);
        if (!__any_sync(0xffffffffu, alive)) continue;
        WSTAT(0, 1);
        if (alive) ++steps;
        float cvn = fterm<KID>(c2, KID == KID_WINDING ? s_w2(lo) : w0, qx, qy, qz, kp);
        const int2 t2 = s_t2(lo);
        int4 tp = make_int4(t2.x & 0x1ffffff, (int)((unsigned)t2.x >> 25), 0, t2.y);
        const int2 sp = *reinterpret_cast<const int2*>(&s_smp[64 + i]);
        const uint64_t path = ((uint64_t)(uint32_t)sp.y << 32) | (uint32_t)sp.x;
        int lvl = 2;
        float resid = 0.f;
        while (tp.y > 0) {  // warp-uniform: every lane walks the same node
          const bool cmulti = lvl + 1 >= V.first_multi;
          float ks0 = 0.f, ks1 = 0.f;
          int le = 0, c = 0;
          const bool use_path = !cmulti && lvl < V.path_levels;
#ifdef FSB_WARP_STATS
          const unsigned am = __ballot_sync(0xffffffffu, alive);
#endif
          WSTAT(1, 1);
          WSTAT(2, __popc(am));
          WSTAT(5, tp.y);
          WSTAT(7, __popc(am) * tp.y);
          // with the path, the picked child is known up front: its record and
          // topology load while the children are summed
          int4 tpn = make_int4(0, 0, 0, 0);
          if (use_path) {  // the next node's topology loads while the children are summed
            le = 1 + (int)((path >> (V.path_bits * lvl)) & ((1u << V.path_bits) - 1u));
            tpn = V.topo[tp.x + le - 1];
          }
          float4 cch;
          if (kStageKids && V.stage_kids && use_path) {
            const int np = stage_kid_pairs(s_kid, V.cmp, tp.x, tp.y, lane);
            ks0 = staged_kid_sum(s_kid, np, qx, qy, qz, kp.dfloor_f);
            cch = staged_kid(s_kid, (tp.x & 1) + le - 1);  // the picked child, staged
          } else if (kPack && use_path) {
            ks0 = children_coulomb_pairs(V.cmp, V.cm, tp.x, tp.y, qx, qy, qz, kp);
          } else if (use_path) {
            if (tp.x & 1) {
              ks0 += fterm<KID>(V.cm[tp.x], KID == KID_WINDING ? V.m12[tp.x] : w0, qx, qy, qz, kp);
              c = 1;
            }
            for (; c + 3 < tp.y; c += 4) {
              const int r = tp.x + c;
              float4 c0, c1, c2_, c3;
              ld_pair(V.cm + r, c0, c1);
              ld_pair(V.cm + r + 2, c2_, c3);
              ks0 += fterm<KID>(c0, KID == KID_WINDING ? V.m12[r] : w0, qx, qy, qz, kp);
              ks1 += fterm<KID>(c1, KID == KID_WINDING ? V.m12[r + 1] : w0, qx, qy, qz, kp);
              ks0 += fterm<KID>(c2_, KID == KID_WINDING ? V.m12[r + 2] : w0, qx, qy, qz, kp);
              ks1 += fterm<KID>(c3, KID == KID_WINDING ? V.m12[r + 3] : w0, qx, qy, qz, kp);
            }
            for (; c < tp.y; ++c)
              ks0 += fterm<KID>(V.cm[tp.x + c], KID == KID_WINDING ? V.m12[tp.x + c] : w0, qx, qy,
                                qz, kp);
          } else {
            for (; c < tp.y; ++c) {
              const int r = tp.x + c;
              const float4 cr = V.cm[r];
              const float2 wr = KID == KID_WINDING ? V.m12[r] : w0;
              float v;
              if (cmulti) {
                const int4 tc = V.topo[r];
                v = (tc.y == 0 && tc.w - tc.z > 1)
                        ? leaf_exact<KID>(V, tc.z, tc.w, qx, qy, qz, kp)
                        : fterm<KID>(cr, wr, qx, qy, qz, kp);
              } else {
                v = fterm<KID>(cr, wr, qx, qy, qz, kp);
              }
              ks0 += v;
              le += V.lb[r] <= jj;
            }
          }
          const int cidx = tp.x + le - 1;
          if (!(kStageKids && V.stage_kids && use_path)) cch = V.cm[cidx];  // one of the children just summed
          if (!use_path) tpn = V.topo[cidx];
          if (alive) {  // swap / (p_agg * p_rr), p_agg = points(node) / points(a)
            seen += tp.y + 1;
            resid += ((ks0 + ks1) - cvn) * (fcount_a * rcp_ftz((float)(tp.w - tp.z) * prr));
          }
          const float rc = fdist(cch, qx, qy, qz) * V.inv_diam[min(lvl + 1, kFastMaxLevels - 1)];
          const float p = rr_fast_t<RR>(rp, rc);
          const int ctr = lvl - 1;  // levels descended so far (uniform)
          float u = 0.f;  // roulette draws from the sample table (counters 1, 2) or the stream
          if (RR != 2) {
            const int4 sb = s_smp[32 + i];
            u = ctr == 1   ? __int_as_float(sb.z)
                : ctr == 2 ? __int_as_float(sb.w)
                           : draw24(((uint64_t)(uint32_t)sb.y << 32) | (uint32_t)sb.x,
                                    (uint64_t)ctr);
          }
          alive = alive && (RR == 2 || p >= 1.f || u < p);
          if (!__any_sync(0xffffffffu, alive)) break;
          if (alive) {
            ++steps;
            cvn = fterm<KID>(cch, KID == KID_WINDING ? V.m12[cidx] : w0, qx, qy, qz, kp);
            prr *= p;
            rp = rc;
          }
          tp = tpn;
          ++lvl;
        }
        acc_deep += resid;
      }
    }
    next = __shfl_sync(0xffffffffu, claim, 0);
    if (live) {
      const int64_t qi = query_of(t);
      out[qi] = (float)(acc + (double)(acc_deep * inv_s));
      if (visited) visited[qi] = seen;
      if (path_steps) path_steps[qi] = steps;
      if (path_count) path_count[qi] = (int64_t)S * n_int;
    }
  }
#undef s_cm1
#undef s_tp1
#undef s_cm2
#undef s_w1
#undef s_w2
#undef s_t2
#undef s_b2
#undef s_lut
#undef s_int
#undef s_leaf
}

// returns 1 if the fast path does not apply (caller falls back), 0 on launch
int stochastic_fast(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                    const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed,
                    int64_t qoff, int share, float* out, int64_t* visited, int64_t* path_steps,
                    int64_t* path_count, cudaStream_t s, bool* used, bool shuffled) {
  *used = false;
  // an in-kernel shuffled order is only computed by the warp-uniform kernel
  if (shuffled && !(share == 5 && (qoff & 31) == 0 && !std::getenv("FSB_STO_WARP_OFF"))) return 0;
  if (t->root_kids <= 0 || t->num_levels > kFastMaxLevels) return 0;
  FS_TRY(ensure_fast(t, s));
  FS_TRY(ensure_lo(t, false, s));  // packed points for multi-point leaves
  if (!t->uniform_diam) return 0;
  FastView V;
  V.topo = t->lo_topo;
  V.cm = t->lo_cm32;
  V.m12 = t->lo_m12_32;
  V.lb = t->lo_begin;
  V.pa = t->pts32a;
  V.pb = t->pts32b;
  FS_TRY(ensure_path(t, s));
  // the packed level-2 topology {first child | count << 25} needs < 128 children
  // per node (branching <= 5) and < 2^25 nodes
  if (t->max_children >= 128 || t->n >= (1ll << 25)) return 0;
  V.path = t->pt_path;
  V.cmp = nullptr;
  V.stage_kids = t->max_children <= 2 * (kKidPairs - 1);
  V.path_bits = t->path_bits;
  V.path_levels = t->path_levels;
  V.n1 = t->root_kids;
  V.base2 = t->num_levels > 2 ? (int)t->level_off[2] : (int)t->n;
  V.n2 = t->num_levels > 2 ? (int)(t->level_off[3] - t->level_off[2]) : 0;
  V.first_multi = t->first_multi_level;
  for (int l = 0; l < kFastMaxLevels; ++l) {
    float d = l < t->num_levels ? t->level_diam[l] : 1.f;
    V.inv_diam[l] = 1.0f / std::max(d, 1e-12f);
  }
  bool wind = kid == KID_WINDING;
  if ((int64_t)V.n1 * n_samples > (1 << 20)) return 0;
  // a chunk of per_chunk (a, s) pairs queues at most per_chunk * kBlock walks
  const int64_t nslot = (int64_t)V.n1 * n_samples;
  V.per_chunk = (int)std::max<int64_t>(1, std::min<int64_t>(nslot, FSB_QCAP_MAX / kBlock));
  V.qcap = V.per_chunk * kBlock;
  const size_t n1 = (size_t)V.n1, n2 = (size_t)V.n2;
  // shared memory: the packed pair table is an option, used when it fits
  constexpr size_t kSmemMax = 220 * 1024;
  const bool can_pack = kid != KID_SMOOTH && FSB_WARP_DENSE2;
  const size_t pvec = kid == KID_WINDING ? 3 : 2;  // float4 per staged record pair
  const size_t pairs_bytes = 16 * pvec * ((n2 + 1) / 2);
  size_t smem = 16 * ((size_t)kBlock + 2 * n1 + n2) + 8 * ((wind ? n1 + n2 : 0) + kBlock) +
                4 * (2 * n2 + 2 * (size_t)kBlock + 6) + 8 * n2 + 2 * n1 * (kLut + 1);
  smem = (smem + 31) & ~(size_t)15;  // (+ alignment slack for the pair table)
  // resident blocks per SM a shared-memory size allows (228 KB per SM, 1 KB reserved
  // per block), capped by the register budget: the pair table is used only when it
  // does not cost occupancy
  auto fit = [](size_t bytes, int cap) {
    return std::min<int>(cap, (int)((228 * 1024) / (bytes + 1024)));
  };
  // (winding pairs measured slower in the per-query kernel: C2 torus 0.43 -> 0.46 ms)
  const bool pack_fast = can_pack && kid == KID_COULOMB && smem + pairs_bytes <= kSmemMax &&
                         fit(smem + pairs_bytes, FSB_STO_MINB) >= fit(smem, FSB_STO_MINB);
  if (pack_fast) smem += pairs_bytes;
  if (n2 >= 65535 || (int64_t)nslot * kBlock >= (1ll << 31) || t->n >= (1ll << 25)) return 0;
  // warp-uniform kernel's layout (sample tables after the level-1/2 records)
  auto warp_smem = [&](bool pk) {
    return ((16 * (2 * n1 + n2 + (pk ? pvec * ((n2 + 1) / 2) : 0)) +
             8 * ((wind ? n1 + n2 : 0) + n2) + 4 * n2 + 2 * n1 * (kLut + 3) + 128) &
            ~(size_t)127) +
           (size_t)(kWarpBlock / 32) * 96 * 16 +
           (kid == KID_COULOMB && FSB_WARP_DENSE2 && FSB_WARP_STAGE_KIDS
                ? (size_t)(kWarpBlock / 32) * 32 * kKidPairs
                : 0);
  };
  const bool pack_warp = can_pack && warp_smem(true) <= kSmemMax &&
                         fit(warp_smem(true), FSB_WARP_MINB) >= fit(warp_smem(false), FSB_WARP_MINB);
  const size_t wsmem = warp_smem(pack_warp);
  const bool warp_path = share == 5 && (qoff & 31) == 0 && !std::getenv("FSB_STO_WARP_OFF");
  if (warp_path ? wsmem > kSmemMax : smem > kSmemMax) return 0;
  KParams kp;
  kp.alpha = alpha;
  kp.dfloor = dfloor;
  kp.alpha_log2e_neg = (float)(-alpha * 1.4426950408889634);
  kp.dfloor_f = (float)dfloor;
  kp.inv_dfloor_f = (float)(1.0 / dfloor);
  const int B = kBlock;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto launch = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      FS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
#ifdef FSB_CARVE
    FS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, FSB_CARVE));
#endif
    FS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, B, smem));
    int64_t tiles = (n + B - 1) / B;
    int64_t grid = std::min<int64_t>(tiles, (int64_t)sms * std::max(per_sm, 1));
    Scratch res, queues, ctr;
    FS_TRY(res.alloc(sizeof(float) * (size_t)grid * B * nslot, s));
    FS_TRY(queues.alloc((size_t)grid * 2 * V.qcap * kWalkBytes, s));
    FS_TRY(ctr.alloc(sizeof(unsigned int), s));
    FS_CK(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned int), s));
    kern<<<(unsigned)grid, B, smem, s>>>(V, q, n, qperm, n_samples, seed, qoff, share, kp,
                                         res.as<float>(), queues.as<unsigned char>(),
                                         ctr.as<unsigned int>(), out, visited, path_steps,
                                         path_count);
    FS_CK(cudaGetLastError());
    return 0;
  };
  int rc = 0;
  if (rr_mode < 0 || rr_mode > 2) {
    set_error("unknown rr mode %d", rr_mode);
    return 1;
  }
  if (warp_path) {
    if (kid == KID_COULOMB && FSB_WARP_DENSE2) {  // pair-interleaved records for the walks
      FS_TRY(ensure_pairs(t, s));
      V.cmp = t->lo_cmp;
    }
    // warp-shared streams on warp-aligned groups: the warp-uniform kernel
    auto launch_w = [&](auto kern) -> int {
      if (wsmem > 48 * 1024)
        FS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
      FS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpBlock, wsmem));
      const int64_t blocks = (n + kWarpBlock - 1) / kWarpBlock;
      const int64_t grid = std::min<int64_t>(blocks, (int64_t)sms * std::max(per_sm, 1));
      Scratch ctr;
      FS_TRY(ctr.alloc(sizeof(unsigned int), s));
      FS_CK(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned int), s));
#ifdef FSB_WARP_STATS
      unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      FS_CK(cudaMemcpyToSymbolAsync(g_warp_stats, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
#endif
      kern<<<(unsigned)grid, kWarpBlock, wsmem, s>>>(V, q, n, qperm, n_samples, seed, qoff, kp,
                                                     ctr.as<unsigned int>(), out, visited,
                                                     path_steps, path_count, shuffled ? 1 : 0);
      FS_CK(cudaGetLastError());
#ifdef FSB_WARP_STATS
      FS_CK(cudaMemcpyFromSymbolAsync(z, g_warp_stats, sizeof(z), 0, cudaMemcpyDeviceToHost, s));
      FS_CK(cudaStreamSynchronize(s));
      const double nw = (double)((n + 31) / 32);
      fprintf(stderr,
              "warp stats per 32-query chunk: pairs %.1f, walks %.1f, levels %.1f, "
              "live lanes/level %.2f, children/level %.1f, useful child evals %.0f of %.0f\n",
              z[6] / nw, z[0] / nw, z[1] / nw, (double)z[2] / std::max(1ull, z[1]),
              (double)z[5] / std::max(1ull, z[1]), z[7] / nw, 32.0 * z[5] / nw);
#endif
      return 0;
    };
    switch (kid * 3 + rr_mode) {
      case 0: rc = pack_warp ? launch_w(k_sto_warp<0, 0, true>) : launch_w(k_sto_warp<0, 0, false>); break;
      case 1: rc = pack_warp ? launch_w(k_sto_warp<0, 1, true>) : launch_w(k_sto_warp<0, 1, false>); break;
      case 2: rc = pack_warp ? launch_w(k_sto_warp<0, 2, true>) : launch_w(k_sto_warp<0, 2, false>); break;
      case 3: rc = pack_warp ? launch_w(k_sto_warp<1, 0, true>) : launch_w(k_sto_warp<1, 0, false>); break;
      case 4: rc = pack_warp ? launch_w(k_sto_warp<1, 1, true>) : launch_w(k_sto_warp<1, 1, false>); break;
      case 5: rc = pack_warp ? launch_w(k_sto_warp<1, 2, true>) : launch_w(k_sto_warp<1, 2, false>); break;
      case 6: rc = launch_w(k_sto_warp<2, 0, false>); break;
      case 7: rc = launch_w(k_sto_warp<2, 1, false>); break;
      case 8: rc = launch_w(k_sto_warp<2, 2, false>); break;
      default: set_error("unknown kernel id"); return 1;
    }
    if (rc == 0) *used = true;
    return rc;
  }
  switch (kid * 3 + rr_mode) {
    case 0: rc = pack_fast ? launch(k_sto_fast<0, 0, true>) : launch(k_sto_fast<0, 0, false>); break;
    case 1: rc = pack_fast ? launch(k_sto_fast<0, 1, true>) : launch(k_sto_fast<0, 1, false>); break;
    case 2: rc = pack_fast ? launch(k_sto_fast<0, 2, true>) : launch(k_sto_fast<0, 2, false>); break;
    case 3: rc = launch(k_sto_fast<1, 0, false>); break;
    case 4: rc = launch(k_sto_fast<1, 1, false>); break;
    case 5: rc = launch(k_sto_fast<1, 2, false>); break;
    case 6: rc = launch(k_sto_fast<2, 0, false>); break;
    case 7: rc = launch(k_sto_fast<2, 1, false>); break;
    case 8: rc = launch(k_sto_fast<2, 2, false>); break;
    default: set_error("unknown kernel id"); return 1;
  }
  if (rc == 0) *used = true;
  return rc;
}

}  // namespace fsb
