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

// Walks below level 1, held per block in global memory (array of 48-byte
// records, L2-resident); two queues ping-pong between service rounds.
// Record: int4 {meta = owner | lvl << 8 | a_ord << 16, seq, node, j},
//         float4 {prr, rp, cvn, resid}, uint4 {kr.lo, kr.hi, -, -}.
constexpr int kQcap = 4096 + 2 * kBlock;
constexpr size_t kQueueBytes = (size_t)kQcap * 48;  // one queue

struct Walk {
  int4 a;
  float4 f;
  uint4 k;
};

extern __shared__ int sh_i[];
// last index k in [lo, lo + cnt) whose begin (low 31 bits of sh_i[ob + k]) is <= j
__device__ __forceinline__ int child_search(int ob, int lo, int cnt, int j) {
  const int last = lo + cnt - 1;
  for (int step = cnt > 1 ? 1 << (31 - __clz(cnt - 1)) : 0; step > 0; step >>= 1) {
    const int t = min(lo + step, last);  // branch-free: probe a clamped index
    lo = (sh_i[ob + t] & 0x7fffffff) <= j ? t : lo;
  }
  return lo;
}

template <int KID>
__global__ void __launch_bounds__(kBlock, FSB_STO_MINB)
    k_sto_fast(FastView V, const double* __restrict__ q, int64_t n,
               const int32_t* __restrict__ qperm, int S, int rr_mode, uint64_t seed, int64_t qoff,
               KParams kp, float* __restrict__ res_g, int res_stride,
               unsigned char* __restrict__ queues, float* __restrict__ out,
               int64_t* __restrict__ visited, int64_t* __restrict__ path_steps,
               int64_t* __restrict__ path_count) {
  // Dynamic shared memory, addressed by element index off the extern arrays
  // (all alias the same window), so every access is LDS [index + imm] with no
  // generic-pointer reconstruction.  Layout in 16-byte units:
  //   [0, kBlock)          s_q    float4  query coordinates of this tile
  //   [o_cm1, +n1)         s_cm1  float4  level-1 {com, m0}
  //   [o_tp1, +n1)         s_tp1  int4    level-1 topology
  //   [o_cm2, +n2)         s_cm2  float4  level-2 {com, m0}
  //   then float2 s_w1[n1], s_w2[n2] (winding) and int s_b2[n2], s_seen, s_steps, s_count
  extern __shared__ float4 sh_f4[];
  extern __shared__ int4 sh_i4[];
  extern __shared__ float2 sh_f2[];
  extern __shared__ int sh_i[];
  const int n1 = V.n1, n2 = V.n2;
  const int o_cm1 = kBlock, o_tp1 = o_cm1 + n1, o_cm2 = o_tp1 + n1;
  const int o_w1 = 2 * (o_cm2 + n2), o_w2 = o_w1 + (KID == KID_WINDING ? n1 : 0);
  const int o_b2 = 2 * (o_w2 + (KID == KID_WINDING ? n2 : 0));
  const int o_seen = o_b2 + n2, o_steps = o_seen + kBlock, o_count = o_steps + kBlock;
#define s_q(i) sh_f4[(i)]
#define s_cm1(i) sh_f4[o_cm1 + (i)]
#define s_tp1(i) sh_i4[o_tp1 + (i)]
#define s_cm2(i) sh_f4[o_cm2 + (i)]
#define s_w1(i) sh_f2[o_w1 + (i)]
#define s_w2(i) sh_f2[o_w2 + (i)]
#define s_b2(i) sh_i[o_b2 + (i)]
#define s_seen(i) sh_i[o_seen + (i)]
#define s_steps(i) sh_i[o_steps + (i)]
#define s_count(i) sh_i[o_count + (i)]

  unsigned char* const qbase = queues + (size_t)blockIdx.x * 2 * kQueueBytes;

  // ---- stage level 1 (root's children, level order 1..n1) and level 2
  for (int i = threadIdx.x; i < n1; i += blockDim.x) {
    s_cm1(i) = V.cm[1 + i];
    s_tp1(i) = V.topo[1 + i];
    if (KID == KID_WINDING) s_w1(i) = V.m12[1 + i];
  }
  const bool l2_multi = V.first_multi <= 2;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    s_cm2(i) = V.cm[V.base2 + i];
    if (KID == KID_WINDING) s_w2(i) = V.m12[V.base2 + i];
    int b = V.lb[V.base2 + i];
    if (l2_multi) {
      int4 tp = V.topo[V.base2 + i];
      if (tp.y == 0 && tp.w - tp.z > 1) b |= 0x80000000;
    }
    s_b2(i) = b;
  }
  if (threadIdx.x == 0) {
    s_count(0) = 0;
    s_count(1) = 0;
  }
  s_seen(threadIdx.x) = 0;
  s_steps(threadIdx.x) = 0;
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
    int src = 0;  // the level-1 step always produces into queue 0
    int cnt = s_count(0);
    while (cnt > 0) {
      Walk* in = reinterpret_cast<Walk*>(qbase + (size_t)src * kQueueBytes);
      Walk* outq = reinterpret_cast<Walk*>(qbase + (size_t)(src ^ 1) * kQueueBytes);
      for (int i = tid; i < cnt; i += kBlock) {
        const int4 wa = in[i].a;
        const int meta = wa.x;
        const int owner = meta & 0xff, lvl = (meta >> 8) & 0xff, a_ord = meta >> 16;
        const int seq = wa.y, node = wa.z, jj = wa.w;
        const float4 wf = in[i].f;
        float resid = wf.w;
        const float4 qq = s_q(owner);
        const int4 tp = V.topo[node];
        bool cont = false;
        if (tp.y > 0) {
          const float prr = wf.x, rp = wf.y, cvn = wf.z;
          const bool cmulti = lvl + 1 >= V.first_multi;
          float ks0 = 0.f, ks1 = 0.f;
          int le = 0;  // children whose begin <= j: the last of them holds j
          int c = 0;
          if (!cmulti) {
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
          const int4 tpa = s_tp1(a_ord);
          const float pagg = (float)(tp.w - tp.z) / (float)(tpa.w - tpa.z);
          resid += (ks - cvn) * rcp_ftz(pagg * prr);
          const float rc =
              fdist(cch, qq.x, qq.y, qq.z) * V.inv_diam[min(lvl + 1, kFastMaxLevels - 1)];
          const float p = rr_fast(rp, rc, rr_mode);
          const uint4 k2 = in[i].k;
          const uint64_t kr = ((uint64_t)k2.y << 32) | k2.x;
          if (draw24(kr, (uint64_t)(lvl - 1)) < p) {  // roulette counter = levels descended
            cont = true;
            atomicAdd(&s_steps(owner), 1);
            const float2 wc = KID == KID_WINDING ? V.m12[cidx] : w0;
            const int pos = atomicAdd(&s_count(src ^ 1), 1);
            outq[pos].a = make_int4(owner | ((lvl + 1) << 8) | (a_ord << 16), seq, cidx, jj);
            outq[pos].f = make_float4(prr * p, rc, fterm<KID>(cch, wc, qq.x, qq.y, qq.z, kp), resid);
            outq[pos].k = k2;
          }
        }
        if (!cont) my_res[(int64_t)owner * res_stride + seq] = resid;
      }
      __syncthreads();
      cnt = s_count(src ^ 1);
      __syncthreads();
      if (tid == 0) s_count(src) = 0;
      src ^= 1;
      __syncthreads();
    }
  };

  Walk* const q0 = reinterpret_cast<Walk*>(qbase);
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
    s_q(tid) = make_float4(qx, qy, qz, 0.f);
    const uint64_t hq = key_fold(hseed, (uint64_t)(qi + qoff));
    double acc = 0.0;  // control variates + level-1 residuals, (a, s) order
    int seen = 0, steps = 0, paths = 0;
    int nseq = 0;      // walks that went below level 1
    int qbound = 0;    // upper bound of queue 0's length (block-uniform)

    for (int a_ord = 0; a_ord < n1; ++a_ord) {  // block-uniform
      ++seen;
      const int4 tpa = s_tp1(a_ord);
      const float4 ca = s_cm1(a_ord);
      const float2 wa = KID == KID_WINDING ? s_w1(a_ord) : w0;
      if (tpa.y == 0) {  // leaf subdomain: exact term, never sampled
        float v = (tpa.w - tpa.z > 1) ? leaf_exact<KID>(V, tpa.z, tpa.w, qx, qy, qz, kp)
                                      : fterm<KID>(ca, wa, qx, qy, qz, kp);
        acc += (double)v;
        continue;
      }
      // ---- dense control variate: cv(a) and the hoisted swap over a's children
      const float cv = fterm<KID>(ca, wa, qx, qy, qz, kp);
      const int k0 = tpa.x - V.base2, cc = tpa.y, kend = k0 + cc;
      float ks0 = 0.f, ks1 = 0.f, ks2 = 0.f, ks3 = 0.f;
      if (!l2_multi) {
        int k = k0;
        for (; k + 3 < kend; k += 4) {
          ks0 += fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
          ks1 += fterm<KID>(s_cm2(k + 1), KID == KID_WINDING ? s_w2(k + 1) : w0, qx, qy, qz, kp);
          ks2 += fterm<KID>(s_cm2(k + 2), KID == KID_WINDING ? s_w2(k + 2) : w0, qx, qy, qz, kp);
          ks3 += fterm<KID>(s_cm2(k + 3), KID == KID_WINDING ? s_w2(k + 3) : w0, qx, qy, qz, kp);
        }
        for (; k < kend; ++k)
          ks0 += fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
      } else {
        for (int k = k0; k < kend; ++k) {
          if (s_b2(k) < 0) {
            int4 tp = V.topo[V.base2 + k];
            ks0 += leaf_exact<KID>(V, tp.z, tp.w, qx, qy, qz, kp);
          } else {
            ks0 += fterm<KID>(s_cm2(k), KID == KID_WINDING ? s_w2(k) : w0, qx, qy, qz, kp);
          }
        }
      }
      const float delta_a = ((ks0 + ks1) + (ks2 + ks3)) - cv;
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
        const int lo = child_search(o_b2, k0, cc, j);
        seen += cc + 1;
        const float4 c2 = s_cm2(lo);
        const float rc = fdist(c2, qx, qy, qz) * id2;
        const float p = rr_fast(rp_a, rc, rr_mode);
        if (live && draw24(kr, 0) < p) {  // descends: queue the deeper steps
          ++steps;
          const int pos = atomicAdd(&s_count(0), 1);
          q0[pos].a = make_int4(tid | (2 << 8) | (a_ord << 16), nseq++, V.base2 + lo, j);
          q0[pos].f = make_float4(
              p, rc, fterm<KID>(c2, KID == KID_WINDING ? s_w2(lo) : w0, qx, qy, qz, kp), 0.f);
          q0[pos].k = make_uint4((uint32_t)kr, (uint32_t)(kr >> 32), 0u, 0u);
        }
        // an iteration queues at most kBlock walks: track a block-uniform upper
        // bound of the queue length and look at the real length only near capacity
        qbound += kBlock;
        if (qbound + kBlock > kQcap) {
          __syncthreads();
          qbound = s_count(0);
          __syncthreads();
          if (qbound + kBlock > kQcap) {
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
    seen += s_seen(tid);
    steps += s_steps(tid);
    s_seen(tid) = 0;
    s_steps(tid) = 0;
    const double total = acc + acc_deep / (double)S;
    if (live) {
      out[qi] = (float)total;
      if (visited) visited[qi] = seen;
      if (path_steps) path_steps[qi] = steps;
      if (path_count) path_count[qi] = paths;
    }
    __syncthreads();
  }
#undef s_q
#undef s_cm1
#undef s_tp1
#undef s_cm2
#undef s_w1
#undef s_w2
#undef s_b2
#undef s_seen
#undef s_steps
#undef s_count
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
  const size_t n1 = (size_t)V.n1, n2 = (size_t)V.n2;
  size_t smem = 16 * ((size_t)kBlock + 2 * n1 + n2) + (wind ? 8 * (n1 + n2) : 0) +
                4 * (n2 + 2 * (size_t)kBlock + 4);
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
    Scratch res, queues;
    FS_TRY(res.alloc(sizeof(float) * (size_t)grid * B * stride, s));
    FS_TRY(queues.alloc((size_t)grid * 2 * kQueueBytes, s));
    kern<<<(unsigned)grid, B, smem, s>>>(V, q, n, qperm, n_samples, rr_mode, seed, qoff, kp,
                                         res.as<float>(), stride, queues.as<unsigned char>(), out,
                                         visited, path_steps, path_count);
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
