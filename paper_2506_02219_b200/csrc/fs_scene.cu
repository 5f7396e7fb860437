// fs_scene.cu -- input generation on the device, byte-identical to the host
// generators (reference scene_io.py:112-148 sample_mesh_surface and
// scene_io.py:188-212 make_queries).
//
// The reference draws from numpy's default_rng(seed): PCG64 (128-bit LCG,
// state advanced before each XSL-RR output) and random() = (x >> 11) * 2^-53.
// Every GPU thread jumps the generator ahead to its own draw (LCG jump-ahead,
// O(log k) 128-bit multiplies), so draw i of the stream is computed
// independently of the others:
//   * sample_mesh_surface: choice(p) consumes draws [0, m) (inverse CDF with
//     numpy's searchsorted(side='right') on the host-computed cumsum), then u
//     [m, 2m) and v [2m, 3m); barycentric interpolation in numpy's evaluation
//     order with round-to-nearest intrinsics (no FMA contraction);
//   * make_queries: slice planes (o + sv * v) + su * u from the host axes,
//     grid3d as gathers of the host linspace axes, random clouds
//     low + (high - low) * random() per coordinate (numpy's uniform).
#include <cstdint>

#include "../../include/fastsum_b200.h"
#include "fs_internal.h"

namespace fsb {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | lo;
}
constexpr uint64_t kPcgMulHi = 0x2360ED051FC65DA4ull, kPcgMulLo = 0x4385DF649FCCF645ull;

// state after k LCG steps from s (Brown, "Random number generation with arbitrary
// strides"; the same recurrence as pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, uint64_t k) {
  u128 cur_mult = mk128(kPcgMulHi, kPcgMulLo), cur_plus = inc;
  u128 acc_mult = 1, acc_plus = 0;
  while (k) {
    if (k & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    k >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// the k-th double of the stream (k = 0 is the first draw): step, then XSL-RR
__device__ __forceinline__ double pcg_double(u128 s0, u128 inc, uint64_t k) {
  const u128 s = pcg_advance(s0, inc, k + 1);
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  const uint64_t x = hi ^ lo;
  const uint64_t r = (x >> rot) | (x << ((64u - rot) & 63u));
  return __ull2double_rn(r >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_sample_mesh(const double* __restrict__ cdf, int64_t nf,
                              const double* __restrict__ tri,  // (nf, 3 vertices, 3)
                              const double* __restrict__ normals, int64_t m, uint64_t s_hi,
                              uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, double w_each,
                              double mass, double* __restrict__ pos, double* __restrict__ ms,
                              double* __restrict__ w) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const u128 s0 = mk128(s_hi, s_lo), inc = mk128(i_hi, i_lo);
  // choice(len(areas), p=areas/total): cdf.searchsorted(random(), side='right')
  const double r = pcg_double(s0, inc, (uint64_t)i);
  int64_t lo = 0, hi = nf;  // first index with cdf > r
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= r)
      lo = mid + 1;
    else
      hi = mid;
  }
  const int64_t f = lo < nf ? lo : nf - 1;
  double u = pcg_double(s0, inc, (uint64_t)(m + i));
  double v = pcg_double(s0, inc, (uint64_t)(2 * m + i));
  if (__dadd_rn(u, v) > 1.0) {
    u = __dsub_rn(1.0, u);
    v = __dsub_rn(1.0, v);
  }
  const double a = __dsub_rn(__dsub_rn(1.0, u), v);  // 1 - u - v
  const double* t = tri + 9 * f;
  for (int d = 0; d < 3; ++d)
    pos[3 * i + d] = __dadd_rn(__dadd_rn(__dmul_rn(t[d], a), __dmul_rn(t[3 + d], u)),
                               __dmul_rn(t[6 + d], v));
  if (normals) {
    for (int d = 0; d < 3; ++d) ms[3 * i + d] = __dmul_rn(normals[3 * f + d], w_each);
  } else {
    ms[i] = mass;
  }
  w[i] = w_each;
}

__global__ void k_queries(int kind, int64_t n, const double* __restrict__ ax0,
                          const double* __restrict__ ax1, const double* __restrict__ ax2, int64_t r1,
                          int64_t r2, const double* __restrict__ geo, uint64_t s_hi,
                          uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                          double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (kind == 0) {  // grid3d, z fastest (meshgrid 'ij' of the three axes)
    const int64_t iz = i % r2, iy = (i / r2) % r1, ix = i / (r1 * r2);
    out[3 * i] = ax0[ix];
    out[3 * i + 1] = ax1[iy];
    out[3 * i + 2] = ax2[iz];
  } else if (kind == 1) {  // slice plane, v-major: (o + sv * v) + su * u
    const int64_t iu = i % r1, iv = i / r1;
    const double su = ax0[iu], sv = ax1[iv];
    for (int d = 0; d < 3; ++d)
      out[3 * i + d] = __dadd_rn(__dadd_rn(geo[d], __dmul_rn(sv, geo[6 + d])),
                                 __dmul_rn(su, geo[3 + d]));
  } else {  // random: uniform(lo, hi, (n, 3)) = lo + (hi - lo) * random(), row-major
    const u128 s0 = mk128(s_hi, s_lo), inc = mk128(i_hi, i_lo);
    for (int d = 0; d < 3; ++d) {
      const double r = pcg_double(s0, inc, (uint64_t)(3 * i + d));
      out[3 * i + d] = __dadd_rn(geo[d], __dmul_rn(__dsub_rn(geo[3 + d], geo[d]), r));
    }
  }
}

}  // namespace fsb

extern "C" int fsb_sample_mesh_surface(const double* cdf, int64_t num_faces, const double* tri,
                                       const double* normals, int64_t m, const uint64_t* state4,
                                       double w_each, double mass, double* positions,
                                       double* masses, double* weights, void* stream) {
  if (!cdf || !tri || !state4 || !positions || !masses || !weights || num_faces < 1 || m < 1) {
    fsb::set_error("bad mesh sampling arguments");
    return 1;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fsb::k_sample_mesh<<<fsb::grid_for(m, 256), 256, 0, s>>>(
      cdf, num_faces, tri, normals, m, state4[0], state4[1], state4[2], state4[3], w_each, mass,
      positions, masses, weights);
  FS_CK(cudaGetLastError());
  return 0;
}

extern "C" int fsb_make_queries(int kind, int64_t n, const double* ax0, const double* ax1,
                                const double* ax2, int64_t r1, int64_t r2, const double* geo,
                                const uint64_t* state4, double* out, void* stream) {
  if (kind < 0 || kind > 2 || n < 0 || !out || (kind == 2 ? !state4 || !geo : !ax0 || !ax1) ||
      (kind == 0 && !ax2) || (kind == 1 && !geo)) {
    fsb::set_error("bad query-generation arguments");
    return 1;
  }
  if (n == 0) return 0;
  static const uint64_t zero[4] = {0, 0, 0, 0};
  const uint64_t* st = state4 ? state4 : zero;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fsb::k_queries<<<fsb::grid_for(n, 256), 256, 0, s>>>(kind, n, ax0, ax1, ax2, r1, r2, geo, st[0],
                                                      st[1], st[2], st[3], out);
  FS_CK(cudaGetLastError());
  return 0;
}
