// Microbenchmark: per-lane gathers of K consecutive 16-byte records at random
// record indices (the stochastic walk's child loads), 16 B vs 32 B loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(const float4* __restrict__ a, uint32_t nrec, int K,
                                         int iters, float* out) {
  float acc = 0.f;
  uint32_t st = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    st = hash(st + it);
    uint32_t r = (st % (nrec - 64)) & ~1u;
    if (MODE == 0) {  // 16-byte loads, unrolled by 4
      for (int c = 0; c < K; c += 4) {
        float4 x0 = a[r + c], x1 = a[r + c + 1], x2 = a[r + c + 2], x3 = a[r + c + 3];
        acc += x0.x + x1.y + x2.z + x3.w;
      }
    } else {  // 32-byte loads (2 records each)
      for (int c = 0; c < K; c += 4) {
        float v[16];
        const float* p = reinterpret_cast<const float*>(a + r + c);
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                       "=f"(v[6]), "=f"(v[7]) : "l"(p));
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
                       "=f"(v[14]), "=f"(v[15]) : "l"(p + 8));
        acc += v[0] + v[5] + v[10] + v[15];
      }
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4);
  for (size_t bytes : {(size_t)128 << 10, (size_t)2 << 20, (size_t)32 << 20, (size_t)512 << 20}) {
    uint32_t nrec = bytes / 16;
    float4* a; cudaMalloc(&a, bytes); cudaMemset(a, 0, bytes);
    for (int mode = 0; mode < 2; ++mode)
      for (int K : {4, 16}) {
        int iters = 64 * 16 / K;
        int blocks = sms * 4;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (mode == 0) k<0><<<blocks, 256>>>(a, nrec, K, iters, out);
          else k<1><<<blocks, 256>>>(a, nrec, K, iters, out);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double recs = (double)blocks * 256 * iters * K;
        double cyc = ms * 1e-3 * clk * 1e3 * sms;
        printf("array %6zu KB  %s  K=%2d: %.3f ms  %.2f records/cycle/SM  %.0f GB/s\n",
               bytes >> 10, mode ? "32B" : "16B", K, ms, recs / cyc, recs * 16 / (ms * 1e-3) / 1e9);
      }
    cudaFree(a);
  }
  return 0;
}
