// L2 read bandwidth on one B200: every CTA streams float4 loads over a buffer
// that fits in L2 (after a warm-up pass), many times; reports bytes / time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/micro/l2bw.cu && /tmp/l2bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const float4* __restrict__ a, size_t n, int reps, float* sink) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(a + i);  // L2 (bypass L1)
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 123.456f) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (size_t mb : {16, 32, 64, 96}) {
    size_t bytes = mb << 20, n = bytes / 16;
    float4* a;
    float* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, bytes);
    const int reps = 20;
    k_read<<<sms * 8, 256>>>(a, n, 1, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_read<<<sms * 8, 256>>>(a, n, reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("L2-resident read, %zu MB x %d: %.0f GB/s\n", mb, reps,
           (double)bytes * reps / (ms * 1e-3) / 1e9);
    cudaFree(a);
    cudaFree(sink);
  }
  return 0;
}
