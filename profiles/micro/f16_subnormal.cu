// Does tcgen05.mma kind::f16 keep binary16 subnormal inputs?  A (128 x 16) =
// a constant, B (256 x 16) = 1: every fp32 result is 16 * a.  Prints the
// result for a = 2^-20 (subnormal in binary16) and a = 2^-10 (normal).
// nvcc -gencode arch=compute_100a,code=sm_100a f16_subnormal.cu -o f16_subnormal
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t off16(int row, int k) {  // K-major, no swizzle, 8 x 16 B core matrices
  return (uint32_t)((row >> 3) * 256 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void k(float a, float* out) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[256 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int e = tid; e < 128 * 16; e += 128) *reinterpret_cast<__half*>(sa + off16(e / 16, e % 16)) = __float2half_rn(a);
  for (int e = tid; e < 256 * 16; e += 128) *reinterpret_cast<__half*>(sb + off16(e / 16, e % 16)) = __float2half_rn(1.f);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
        "l"(sdesc(smem_u32(sa), 128, 256)), "l"(sdesc(smem_u32(sb), 128, 256)), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r0;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(tbase + ((uint32_t)((tid >> 5) * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[tid] = __uint_as_float(r0);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * sizeof(float));
  for (float a : {0x1p-20f, 0x1p-10f, 0x1p-24f}) {
    k<<<1, 128>>>(a, d);
    float h[128];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("a = %g: D[0] = %g (16 a = %g), D[127] = %g, err %s\n", a, h[0], 16 * a, h[127],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
