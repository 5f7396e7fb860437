// fs_sto_fast.cu -- the FP32 stochastic estimator kernel (precision="f32").
//
// Same estimator as stochastic_batch (_core.py:159-267, the reference variant:
// the swap at each reached node is committed before the roulette that gates
// descent), same splitmix64 streams and index draws, reorganised for B200:
//
//  * The control-variate part is dense and query-independent in its node set:
//    every query evaluates the N1 level-1 aggregates and the N2 level-2
//    children of internal level-1 nodes.  A persistent block stages those
//    records in shared memory once ({com, m0} = 16 B per node, + {m1, m2} for
//    winding) and every thread streams them with broadcast LDS: an
//    FP32 + MUFU.RSQ loop, the N x (N1+N2) "brute force over staged nodes".
//  * The first path step (from the subdomain to a level-2 child) is resolved
//    from shared memory: binary search of the sampled point index over the
//    children's begins, far-field ratios from per-level cell diameters (cells
//    are uniform splits, so one diameter per level, octree.py:225).
//  * Deeper steps (only ~1/3 of samples descend below level 1, and fewer
//    further) would leave most lanes idle if walked in place.  Instead each
//    descending sample is pushed onto a block-wide shared-memory queue and the
//    block serves the queue in rounds: every thread takes one walk and
//    advances it by exactly one level (sum the node's contiguous children,
//    pick the child holding the sampled point, roulette), pushing it back if it
//    continues.  Finished walks store their residual in the owner's creation-
//    ordered slot, and owners fold their slots in that order, so a query's
//    result does not depend on which thread served its walks or when.
//  * FP32 terms and residuals, FP64 accumulation across subdomains.
#include <algorithm>

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
  int n1, base2, n2, first_multi;
  float inv_diam[kFastMaxLevels];  // 1 / max(diam_level, 1e-12)
};

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

__device__ __forceinline__ float rr_fast(float rp, float rc, int mode) {
  if (mode == 1) return 0.5f;
  if (mode == 2) return 1.0f;
  return fminf(fmaxf(rp, 1.0f) * rcp_ftz(fmaxf(rc, 1e-12f)), 1.0f);
}

// roulette uniform from the top 24 bits of the same splitmix draw
__device__ __forceinline__ float draw24(uint64_t key, uint64_t ctr) {
  uint64_t x = mix64(key + (ctr + 1ull) * kGamma);
  return (float)(uint32_t)(x >> 40) * (1.0f / 16777216.0f);
}

constexpr int kBlock = 256;  // threads (= queries) per tile
#ifndef FSB_STO_MINB
#define FSB_STO_MINB 4  // resident blocks per SM the register budget is sized for
#endif

// Walks below level 1, held per block in global memory (structure of arrays,
// L2-resident); two queues ping-pong between service rounds.  Field offsets
// (per queue of capacity cap): kr u64 | meta | seq | node | j | prr | rp | cvn | resid.
enum QField { QF_META = 0, QF_SEQ, QF_NODE, QF_J, QF_PRR, QF_RP, QF_CVN, QF_RESID };
constexpr int kQueueBytesPerTask = 40;

template <int KID>
__global__ void __launch_bounds__(kBlock, FSB_STO_MINB) k_sto_fast(FastView V, const double* __restrict__ q,
                                                        int64_t n,
                                                        const int32_t* __restrict__ qperm, int S,
                                                        int rr_mode, uint64_t seed, int64_t qoff,
                                                        KParams kp, float* __restrict__ res_g,
                                                        int res_stride,
                                                        unsigned char* __restrict__ queues,
                                                        int qcap, float* __restrict__ out,
                                                        int64_t* __restrict__ visited,
                                                        int64_t* __restrict__ path_steps,
                                                        int64_t* __restrict__ path_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n1 = V.n1, n2 = V.n2;
  float4* s_q = reinterpret_cast<float4*>(smem);
  int* s_seen = reinterpret_cast<int*>(s_q + kBlock);  // nodes read below level 1, per query
  int* s_steps = s_seen + kBlock;                        // descents below level 1, per query
  int* s_count = s_steps + kBlock;                       // [0]: queue A, [1]: queue B
  float4* s_cm1 = reinterpret_cast<float4*>(s_count + 4);
  int4* s_tp1 = reinterpret_cast<int4*>(s_cm1 + n1);
  float4* s_cm2 = reinterpret_cast<float4*>(s_tp1 + n1);
  float2* s_w1 = reinterpret_cast<float2*>(s_cm2 + n2);
  float2* s_w2 = s_w1 + (KID == KID_WINDING ? n1 : 0);
  int* s_b2 = reinterpret_cast<int*>(s_w2 + (KID == KID_WINDING ? n2 : 0));

  unsigned char* const qbase = queues + (size_t)blockIdx.x * 2 * qcap * kQueueBytesPerTask;
  // queue `w` (0/1), field f
  auto QI = [&](int w, int f) -> int* {
    return reinterpret_cast<int*>(qbase + (size_t)w * qcap * kQueueBytesPerTask +
                                  (size_t)qcap * (8 + 4 * f));
  };
  auto QF = [&](int w, int f) -> float* { return reinterpret_cast<float*>(QI(w, f)); };
  auto QK = [&](int w) -> uint2* {
    return reinterpret_cast<uint2*>(qbase + (size_t)w * qcap * kQueueBytesPerTask);
  };

  // ---- stage level 1 (root's children, level order 1..n1) and level 2
  for (int i = threadIdx.x; i < n1; i += blockDim.x) {
    s_cm1[i] = V.cm[1 + i];
    s_tp1[i] = V.topo[1 + i];
    if (KID == KID_WINDING) s_w1[i] = V.m12[1 + i];
  }
  const bool l2_multi = V.first_multi <= 2;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    s_cm2[i] = V.cm[V.base2 + i];
    if (KID == KID_WINDING) s_w2[i] = V.m12[V.base2 + i];
    int b = V.lb[V.base2 + i];
    if (l2_multi) {
      int4 tp = V.topo[V.base2 + i];
      if (tp.y == 0 && tp.w - tp.z > 1) b |= 0x80000000;
    }
    s_b2[i] = b;
  }
  if (threadIdx.x == 0) {
    s_count[0] = 0;
    s_count[1] = 0;
  }
  s_seen[threadIdx.x] = 0;
  s_steps[threadIdx.x] = 0;
  __syncthreads();

  const int tid = threadIdx.x;
  const uint64_t hseed = mix64(seed + kGamma);
  const float id1 = V.inv_diam[1], id2 = V.inv_diam[2];
  const float2 w0 = make_float2(0.f, 0.f);
  float* my_res = res_g + ((int64_t)blockIdx.x * kBlock) * res_stride;

  // Serve all queued walks: each service round advances every queued walk by
  // one level (sum the node's contiguous children, pick the child holding the
  // sampled point, roulette); survivors go to the other queue, finished walks
  // store their residual in the owner's creation-ordered slot.
  auto drain = [&]() {
    int src = 0;  // walks are always produced into queue 0 by the level-1 step
    int cnt = s_count[0];
    while (cnt > 0) {
      const int dst = src ^ 1;
      for (int i = tid; i < cnt; i += kBlock) {
        const int meta = QI(src, QF_META)[i];
        const int owner = meta & 0xff, lvl = (meta >> 8) & 0xff, a_ord = meta >> 16;
        const int node = QI(src, QF_NODE)[i], jj = QI(src, QF_J)[i];
        const float prr = QF(src, QF_PRR)[i], rp = QF(src, QF_RP)[i], cvn = QF(src, QF_CVN)[i];
        float resid = QF(src, QF_RESID)[i];
        const float4 qq = s_q[owner];
        const int4 tp = V.topo[node];
        bool cont = false;
        if (tp.y > 0) {
          const bool cmulti = lvl + 1 >= V.first_multi;
          float ks = 0.f, tch = 0.f;
          float4 cch = make_float4(0.f, 0.f, 0.f, 0.f);
          int cidx = tp.x;
#pragma unroll 4
          for (int c = 0; c < tp.y; ++c) {
            const int r = tp.x + c;
            const float4 cr = V.cm[r];
            const float2 wr = KID == KID_WINDING ? V.m12[r] : w0;
            const int b = V.lb[r];
            float v;
            if (cmulti) {
              int4 tc = V.topo[r];
              v = (tc.y == 0 && tc.w - tc.z > 1)
                      ? leaf_exact<KID>(V, tc.z, tc.w, qq.x, qq.y, qq.z, kp)
                      : fterm<KID>(cr, wr, qq.x, qq.y, qq.z, kp);
            } else {
              v = fterm<KID>(cr, wr, qq.x, qq.y, qq.z, kp);
            }
            ks += v;
            if (b <= jj) {  // children are ordered by begin: the last such holds j
              tch = v;
              cch = cr;
              cidx = r;
            }
          }
          atomicAdd(&s_seen[owner], tp.y + 1);
          const int4 tpa = s_tp1[a_ord];
          const float pagg = (float)(tp.w - tp.z) / (float)(tpa.w - tpa.z);
          resid += (ks - cvn) * rcp_ftz(pagg * prr);
          const float rc =
              fdist(cch, qq.x, qq.y, qq.z) * V.inv_diam[min(lvl + 1, kFastMaxLevels - 1)];
          const float p = rr_fast(rp, rc, rr_mode);
          const uint2 k2 = QK(src)[i];
          const uint64_t kr = ((uint64_t)k2.y << 32) | k2.x;
          if (draw24(kr, (uint64_t)(lvl - 1)) < p) {  // roulette counter = levels descended
            cont = true;
            atomicAdd(&s_steps[owner], 1);
            const int pos = atomicAdd(&s_count[dst], 1);
            QI(dst, QF_META)[pos] = owner | ((lvl + 1) << 8) | (a_ord << 16);
            QI(dst, QF_SEQ)[pos] = QI(src, QF_SEQ)[i];
            QI(dst, QF_NODE)[pos] = cidx;
            QI(dst, QF_J)[pos] = jj;
            QF(dst, QF_PRR)[pos] = prr * p;
            QF(dst, QF_RP)[pos] = rc;
            QF(dst, QF_CVN)[pos] = tch;
            QF(dst, QF_RESID)[pos] = resid;
            QK(dst)[pos] = k2;
          }
        }
        if (!cont) my_res[(int64_t)owner * res_stride + QI(src, QF_SEQ)[i]] = resid;
      }
      __syncthreads();
      cnt = s_count[dst];
      __syncthreads();
      if (tid == 0) s_count[src] = 0;
      src = dst;
      __syncthreads();
    }
    if (src == 1) {  // survivors ended in queue 1 (now empty): keep queue 0 as the producer
      __syncthreads();
    }
  };

  for (int64_t base = (int64_t)blockIdx.x * kBlock; base < n; base += (int64_t)gridDim.x * kBlock) {
    const int64_t t = base + tid;
    const bool live = t < n;
    const int64_t qi = live ? (qperm ? (int64_t)qperm[t] : t) : 0;
    float qx = 0.f, qy = 0.f, qz = 0.f;
    if (live) {
      qx = (float)q[3 * qi];
      qy = (float)q[3 * qi + 1];
      qz = (float)q[3 * qi + 2];
    }
    s_q[tid] = make_float4(qx, qy, qz, 0.f);
    const uint64_t hq = key_fold(hseed, (uint64_t)(qi + qoff));
    double acc = 0.0;  // control variates + level-1 residuals, (a, s) order
    int seen = 0, steps = 0, paths = 0;
    int nseq = 0;      // walks that went below level 1
    int qbound = 0;    // upper bound of queue 0's length (block-uniform)

    for (int a_ord = 0; a_ord < n1; ++a_ord) {  // block-uniform
      ++seen;
      const int4 tpa = s_tp1[a_ord];
      const float4 ca = s_cm1[a_ord];
      const float2 wa = KID == KID_WINDING ? s_w1[a_ord] : w0;
      if (tpa.y == 0) {  // leaf subdomain: exact term, never sampled
        float v = (tpa.w - tpa.z > 1) ? leaf_exact<KID>(V, tpa.z, tpa.w, qx, qy, qz, kp)
                                      : fterm<KID>(ca, wa, qx, qy, qz, kp);
        acc += (double)v;
        continue;
      }
      // ---- dense control variate: cv(a) and the hoisted swap over a's children
      const float cv = fterm<KID>(ca, wa, qx, qy, qz, kp);
      const int k0 = tpa.x - V.base2, cc = tpa.y;
      float ks0 = 0.f, ks1 = 0.f;
      int k = 0;
      for (; k + 1 < cc; k += 2) {
        const int i0 = k0 + k, i1 = i0 + 1;
        float v0, v1;
        if (l2_multi && s_b2[i0] < 0) {
          int4 tp = V.topo[V.base2 + i0];
          v0 = leaf_exact<KID>(V, tp.z, tp.w, qx, qy, qz, kp);
        } else {
          v0 = fterm<KID>(s_cm2[i0], KID == KID_WINDING ? s_w2[i0] : w0, qx, qy, qz, kp);
        }
        if (l2_multi && s_b2[i1] < 0) {
          int4 tp = V.topo[V.base2 + i1];
          v1 = leaf_exact<KID>(V, tp.z, tp.w, qx, qy, qz, kp);
        } else {
          v1 = fterm<KID>(s_cm2[i1], KID == KID_WINDING ? s_w2[i1] : w0, qx, qy, qz, kp);
        }
        ks0 += v0;
        ks1 += v1;
      }
      if (k < cc) {
        const int i0 = k0 + k;
        if (l2_multi && s_b2[i0] < 0) {
          int4 tp = V.topo[V.base2 + i0];
          ks0 += leaf_exact<KID>(V, tp.z, tp.w, qx, qy, qz, kp);
        } else {
          ks0 += fterm<KID>(s_cm2[i0], KID == KID_WINDING ? s_w2[i0] : w0, qx, qy, qz, kp);
        }
      }
      const float delta_a = (ks0 + ks1) - cv;
      const int count_a = tpa.w - tpa.z;
      const float rp_a = fdist(ca, qx, qy, qz) * id1;
      const uint64_t ha = key_fold(hq, (uint64_t)a_ord);
      for (int s = 0; s < S; ++s) {  // block-uniform
        ++paths;
        const uint64_t hs = key_fold(ha, (uint64_t)s);
        const uint64_t ki = key_fold(hs, 0), kr = key_fold(hs, 1);
        // index draw, exactly as _core.py:166-169
        const double u0 = uniform_draw(ki, 0);
        int j = tpa.z + (int)__dmul_rn(u0, (double)count_a);
        if (j >= tpa.w) j = tpa.w - 1;
        // level-1 step from shared memory: the swap at `a` is the hoisted delta_a
        int lo = k0, hi = k0 + cc;
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if ((s_b2[mid] & 0x7fffffff) <= j)
            lo = mid;
          else
            hi = mid;
        }
        seen += cc + 1;
        const float4 c2 = s_cm2[lo];
        const float rc = fdist(c2, qx, qy, qz) * id2;
        const float p = rr_fast(rp_a, rc, rr_mode);
        if (live && draw24(kr, 0) < p) {  // descends: queue the deeper steps
          ++steps;
          const int pos = atomicAdd(&s_count[0], 1);
          QI(0, QF_META)[pos] = tid | (2 << 8) | (a_ord << 16);
          QI(0, QF_SEQ)[pos] = nseq++;
          QI(0, QF_NODE)[pos] = V.base2 + lo;
          QI(0, QF_J)[pos] = j;
          QF(0, QF_PRR)[pos] = p;
          QF(0, QF_RP)[pos] = rc;
          QF(0, QF_CVN)[pos] = fterm<KID>(c2, KID == KID_WINDING ? s_w2[lo] : w0, qx, qy, qz, kp);
          QF(0, QF_RESID)[pos] = 0.f;
          QK(0)[pos] = make_uint2((uint32_t)kr, (uint32_t)(kr >> 32));
        }
        // an iteration queues at most kBlock walks: track a block-uniform upper
        // bound of the queue length and look at the real length only near capacity
        qbound += kBlock;
        if (qbound + kBlock > qcap) {
          __syncthreads();
          qbound = s_count[0];
          __syncthreads();
          if (qbound + kBlock > qcap) {
            drain();
            qbound = 0;
          }
        }
      }
      // every sample's level-1 residual is delta_a: cv + (S * delta_a) / S
      acc += (double)cv + (double)delta_a;
    }
    __syncthreads();
    drain();
    // owners fold their deeper residuals in creation order (query-intrinsic)
    double acc_deep = 0.0;
    for (int k2 = 0; k2 < nseq; ++k2) acc_deep += (double)my_res[(int64_t)tid * res_stride + k2];
    seen += s_seen[tid];
    steps += s_steps[tid];
    s_seen[tid] = 0;
    s_steps[tid] = 0;
    const double total = acc + acc_deep / (double)S;
    if (live) {
      out[qi] = (float)total;
      if (visited) visited[qi] = seen;
      if (path_steps) path_steps[qi] = steps;
      if (path_count) path_count[qi] = paths;
    }
    __syncthreads();
  }
}

// returns 1 if the fast path does not apply (caller falls back), 0 on launch
int stochastic_fast(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                    const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed,
                    int64_t qoff, float* out, int64_t* visited, int64_t* path_steps,
                    int64_t* path_count, cudaStream_t s, bool* used) {
  *used = false;
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
  size_t smem = kBlock * (sizeof(float4) + 2 * sizeof(int)) + 16 +
                (size_t)V.n1 * (sizeof(float4) + sizeof(int4)) + (size_t)V.n2 * sizeof(float4) +
                (wind ? (size_t)(V.n1 + V.n2) * sizeof(float2) : 0) + (size_t)V.n2 * sizeof(int);
  if (smem > 200 * 1024) return 0;
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
    FS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, B, smem));
    int64_t tiles = (n + B - 1) / B;
    int64_t grid = std::min<int64_t>(tiles, (int64_t)sms * std::max(per_sm, 1));
    const int stride = V.n1 * n_samples;  // result slots per query (walks below level 1)
    // per-block walk queues: room for one tile's worth of level-2 walks, capped
    const int qcap = (int)std::min<int64_t>((int64_t)B * stride + B, 4096) + 2 * B;
    Scratch res, queues;
    FS_TRY(res.alloc(sizeof(float) * (size_t)grid * B * stride, s));
    FS_TRY(queues.alloc((size_t)grid * 2 * qcap * kQueueBytesPerTask, s));
    kern<<<(unsigned)grid, B, smem, s>>>(V, q, n, qperm, n_samples, rr_mode, seed, qoff, kp,
                                         res.as<float>(), stride, queues.as<unsigned char>(), qcap,
                                         out, visited, path_steps, path_count);
    FS_CK(cudaGetLastError());
    return 0;
  };
  int rc = 0;
  switch (kid) {
    case 0: rc = launch(k_sto_fast<0>); break;
    case 1: rc = launch(k_sto_fast<1>); break;
    case 2: rc = launch(k_sto_fast<2>); break;
    default: set_error("unknown kernel id"); return 1;
  }
  if (rc == 0) *used = true;
  return rc;
}

}  // namespace fsb
