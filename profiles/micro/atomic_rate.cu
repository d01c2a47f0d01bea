// Single-address atomicAdd throughput (the L2-ring kernels' ticket counter):
// G CTAs, one thread each, T tickets per CTA in a dependent loop (each ticket
// is used before the next is taken, like the producer does).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tickets(int* ctr, int per, int* sink) {
  int acc = 0;
  for (int i = 0; i < per; ++i) acc += atomicAdd(ctr, 1);
  if (acc == 0x7fffffff) *sink = acc;
}
__global__ void tickets_spread(int* ctr, int per, int* sink) {  // 32 counters, one per CTA group
  int acc = 0;
  int* c = ctr + 32 * (blockIdx.x & 31);
  for (int i = 0; i < per; ++i) acc += atomicAdd(c, 1);
  if (acc == 0x7fffffff) *sink = acc;
}
int main() {
  int *ctr, *sink;
  cudaMalloc(&ctr, 4096);
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148, 296, 444, 888}) {
    for (int spread = 0; spread < 2; ++spread) {
      const int per = 2000;
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(ctr, 0, 4096);
        cudaEventRecord(a);
        if (spread) tickets_spread<<<grid, 1>>>(ctr, per, sink);
        else tickets<<<grid, 1>>>(ctr, per, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("grid %d spread %d: %.3f ms, %.2f ns per ticket, %.2f us per ticket per CTA\n", grid, spread, ms,
                        ms * 1e6 / ((double)grid * per), ms * 1e3 / per);
      }
    }
  }
  return 0;
}
