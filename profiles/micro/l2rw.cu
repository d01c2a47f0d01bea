// SM <-> L2 bandwidth with an L2-resident working set (the C2 exchange lives in L2):
// read-only, write-only and read+write (copy) over a buffer of MB megabytes,
// 148 x 4 CTAs x 256 threads, 16-byte accesses, repeated REPS times per launch.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ p, size_t n, int reps, float* sink) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 1.2345f) *sink = acc.y + acc.z + acc.w;
}
__global__ void wr(float4* __restrict__ p, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      __stcg(p + i, make_float4(r, 0, 0, 0));
}
__global__ void cp(const float4* __restrict__ a, float4* __restrict__ b, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      __stcg(b + i, __ldcg(a + i));
}
int main() {
  float4 *a, *b;
  float* sink;
  cudaMalloc(&a, 256 << 20);
  cudaMalloc(&b, 256 << 20);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 0, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mb : {8, 16, 24, 32, 48, 64, 2048 / 8}) {
    const size_t n = (size_t)mb * (1 << 20) / 16;
    const int reps = mb <= 64 ? 40 : 4;
    for (int kind = 0; kind < 3; ++kind) {
      float best = 1e9;
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        if (kind == 0) rd<<<148 * 4, 256>>>(a, n, reps, sink);
        if (kind == 1) wr<<<148 * 4, 256>>>(b, n, reps);
        if (kind == 2) cp<<<148 * 4, 256>>>(a, b, n, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      const double bytes = (double)n * 16 * reps * (kind == 2 ? 2 : 1);
      printf("%4d MB %s: %8.1f GB/s\n", mb, kind == 0 ? "read " : kind == 1 ? "write" : "copy ", bytes / best / 1e6);
    }
  }
  return 0;
}
