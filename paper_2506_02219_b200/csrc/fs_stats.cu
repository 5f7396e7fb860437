// fs_stats.cu -- the measurement path on the device: absolute-error statistics
// of an estimate against an oracle field (reference bench.py:66-95).
//
// error_stats (mean / lower median / max of |est - ref| over unflagged entries)
// and rmse over 10^6-10^7 queries, without copying the fields to the host:
//   1. k_err_keys: |d| per entry as an order-preserving uint64 key (IEEE bits of
//      a non-negative double), flagged entries -> UINT64_MAX; per-block FP64
//      partial sums of |d| and d^2, block max, kept count (fixed order);
//   2. k_err_final: one block folds the partials in block order (deterministic);
//   3. CUB radix sort of the keys; the lower median is key[(count - 1) / 2]
//      (numpy's sort + index, bench.py:62-63).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/fastsum_b200.h"
#include "fs_internal.h"

namespace fsb {

constexpr int kStatBlock = 256;

__global__ void __launch_bounds__(kStatBlock)
    k_err_keys(const double* __restrict__ est, const double* __restrict__ ref,
               const uint8_t* __restrict__ fa, const uint8_t* __restrict__ fb, int64_t n,
               uint64_t* __restrict__ keys, double* __restrict__ part) {
  __shared__ double s_sum[kStatBlock], s_sq[kStatBlock], s_max[kStatBlock];
  __shared__ long long s_cnt[kStatBlock];
  double sum = 0.0, sq = 0.0, mx = -INFINITY;
  long long cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)kStatBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kStatBlock) {
    const bool keep = !((fa && fa[i]) || (fb && fb[i]));
    uint64_t key = ~0ull;
    if (keep) {
      const double d = __dsub_rn(est[i], ref[i]);
      const double a = fabs(d);
      sum = __dadd_rn(sum, a);
      sq = __dadd_rn(sq, __dmul_rn(d, d));
      mx = fmax(mx, a);
      ++cnt;
      // NaN differences keep their bits (they sort after every number)
      key = (uint64_t)__double_as_longlong(a);
    }
    keys[i] = key;
  }
  s_sum[threadIdx.x] = sum;
  s_sq[threadIdx.x] = sq;
  s_max[threadIdx.x] = mx;
  s_cnt[threadIdx.x] = cnt;
  __syncthreads();
  for (int st = kStatBlock / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      s_sum[threadIdx.x] = __dadd_rn(s_sum[threadIdx.x], s_sum[threadIdx.x + st]);
      s_sq[threadIdx.x] = __dadd_rn(s_sq[threadIdx.x], s_sq[threadIdx.x + st]);
      s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + st]);
      s_cnt[threadIdx.x] += s_cnt[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[4 * blockIdx.x + 0] = s_sum[0];
    part[4 * blockIdx.x + 1] = s_sq[0];
    part[4 * blockIdx.x + 2] = s_max[0];
    part[4 * blockIdx.x + 3] = (double)s_cnt[0];
  }
}

__global__ void k_err_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double sum = 0.0, sq = 0.0, mx = -INFINITY, cnt = 0.0;
  for (int b = 0; b < nb; ++b) {  // block order: deterministic
    sum = __dadd_rn(sum, part[4 * b]);
    sq = __dadd_rn(sq, part[4 * b + 1]);
    mx = fmax(mx, part[4 * b + 2]);
    cnt += part[4 * b + 3];
  }
  out[0] = sum;
  out[1] = sq;
  out[2] = mx;
  out[3] = cnt;
}

static int error_stats(const double* est, const double* ref, const uint8_t* fa,
                       const uint8_t* fb, int64_t n, double* out, int64_t* count,
                       cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nb = (int)std::min<int64_t>((n + kStatBlock - 1) / kStatBlock, 4LL * sms);
  Scratch keys, keys2, part, fin;
  FS_TRY(keys.alloc(8 * (size_t)n, s));
  FS_TRY(keys2.alloc(8 * (size_t)n, s));
  FS_TRY(part.alloc(32 * (size_t)nb, s));
  FS_TRY(fin.alloc(4 * sizeof(double) + sizeof(uint64_t), s));
  k_err_keys<<<nb, kStatBlock, 0, s>>>(est, ref, fa, fb, n, keys.as<uint64_t>(),
                                       part.as<double>());
  k_err_final<<<1, 32, 0, s>>>(part.as<double>(), nb, fin.as<double>());
  double h[4];
  FS_CK(cudaMemcpyAsync(h, fin.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  FS_CK(cudaStreamSynchronize(s));
  const int64_t cnt = (int64_t)h[3];
  *count = cnt;
  if (cnt == 0) {
    out[0] = out[1] = out[2] = out[3] = NAN;
    return 0;
  }
  size_t tb = 0;
  FS_CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                       (int)n, 0, 64, s));
  Scratch tmp;
  FS_TRY(tmp.alloc(tb, s));
  FS_CK(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                       (int)n, 0, 64, s));
  uint64_t med = 0;
  FS_CK(cudaMemcpyAsync(&med, keys2.as<uint64_t>() + (cnt - 1) / 2, 8, cudaMemcpyDeviceToHost,
                        s));
  FS_CK(cudaStreamSynchronize(s));
  out[0] = h[0] / (double)cnt;                 // mean |d|
  double medv;
  std::memcpy(&medv, &med, sizeof(medv));
  out[1] = medv;                               // lower median |d|
  out[2] = h[2];                               // max |d|
  out[3] = std::sqrt(h[1] / (double)cnt);      // rmse
  return 0;
}

}  // namespace fsb

extern "C" int fsb_error_stats(const double* estimates, const double* reference,
                               const uint8_t* flags_a, const uint8_t* flags_b, int64_t n,
                               double* out4, int64_t* count, void* stream) {
  if (!out4 || !count || n < 0 || (n > 0 && (!estimates || !reference))) {
    fsb::set_error("null argument / negative count");
    return 1;
  }
  if (n == 0) {
    fsb::set_error("empty inputs");
    return 1;
  }
  if (n >= (1LL << 31)) {
    fsb::set_error("at most 2^31 - 1 entries");
    return 1;
  }
  return fsb::error_stats(estimates, reference, flags_a, flags_b, n, out4, count,
                          reinterpret_cast<cudaStream_t>(stream));
}
