// HBM efficiency of the C2 tile pattern with no arithmetic: persistent CTAs
// copy 4096 x 2^16 complex64 (2 GiB in, 2 GiB out) in 32 KB items through an
// S-stage TMA ring, either as the C2 P1 tile (256 rows x 128 B at a 2 KB
// stride, 128B-swizzled) or as 32 KB contiguous bulk copies.  Answers: is the
// 128-byte-column tile itself costing HBM efficiency?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1203_4938_b200/csrc \
//        profiles/micro/pattern.cu -o profiles/micro/pattern && ./profiles/micro/pattern
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "tma.cuh"

namespace dpp {
int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vprintf(fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace dpp

using namespace dpp;

constexpr int TILE_BYTES = 32768;

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// MODE 0: P1 tile (x = 16 g, y = 256 t); MODE 1: contiguous 32 KB
template <int MODE>
__global__ void copy_items(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                           const float2* in, float2* out, int items, int S, int* ticket, int dyn) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[8];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  int tick[8];
  auto next = [&](int k) { return dyn ? atomicAdd(ticket, 1) : (int)blockIdx.x + k * (int)gridDim.x; };
  auto issue = [&](int s, int it) {
    void* buf = smem + s * TILE_BYTES;
    mbar_arrive_expect_tx(&full[s], TILE_BYTES);
    if (MODE == 0) tma_load_2d(buf, &tin, 16 * (it & 15), 256 * (it >> 4), &full[s]);
    else bulk_g2s(buf, in + (size_t)it * 4096, TILE_BYTES, &full[s]);
  };
  int k = 0;
  for (int s = 0; s < S; ++s) {
    tick[s] = next(k++);
    if (tick[s] < items) issue(s, tick[s]);
  }
  for (int i = 0;; ++i) {
    const int s = i % S;
    if (tick[s] >= items) break;
    mbar_wait(&full[s], (i / S) & 1);
    void* buf = smem + s * TILE_BYTES;
    fence_proxy_async_smem();
    if (MODE == 0) tma_store_2d(&tout, 16 * (tick[s] & 15), 256 * (tick[s] >> 4), buf);
    else bulk_s2g(out + (size_t)tick[s] * 4096, buf, TILE_BYTES);
    commit();
    if (i > 0) {  // refill the previous stage once its store has read it
      const int ps = (i - 1) % S;
      wait_read1();
      tick[ps] = next(k++);
      if (tick[ps] < items) issue(ps, tick[ps]);
      else tick[ps] = items;
    }
  }
  wait_all();
}

int main() {
  const int B = 4096, N = 65536;
  const size_t bytes = (size_t)B * N * 8;
  float2 *in, *out;
  int* ticket;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&ticket, 4);
  cudaMemset(in, 0, bytes);
  CUtensorMap tin, tout;
  make_tmap_c64(&tin, in, (uint64_t)B * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B);
  make_tmap_c64(&tout, out, (uint64_t)B * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int items = B * 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int per_sm, S; };
  const Cfg cfgs[] = {{1, 6}, {1, 4}, {2, 3}, {3, 2}, {2, 2}};
  for (int mode = 0; mode < 2; ++mode)
    for (int dyn = 0; dyn < 2; ++dyn)
      for (const Cfg& c : cfgs) {
        const int smem = c.S * TILE_BYTES;
        auto kern = mode == 0 ? copy_items<0> : copy_items<1>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = c.per_sm * sms;
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
          cudaMemsetAsync(ticket, 0, 4);
          cudaEventRecord(e0);
          kern<<<grid, 32, smem>>>(tin, tout, in, out, items, c.S, ticket, dyn);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep > 0 && ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("%-10s %-6s ctas/SM %d stages %d : %.3f ms  %.0f GB/s %s\n", mode == 0 ? "P1-tile" : "contig",
               dyn ? "ticket" : "static", c.per_sm, c.S, best, 2.0 * bytes / (best * 1e6),
               err == cudaSuccess ? "" : cudaGetErrorString(err));
        fflush(stdout);
      }
  return 0;
}
