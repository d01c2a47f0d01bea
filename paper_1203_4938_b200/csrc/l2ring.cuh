// Device helpers shared by the L2-ring FFT kernels (fft_l2.cu: 1-D 2^16,
// fft2d_l2.cu: 2-D column pass): cache-hinted global accesses, the
// release/acquire counters of the item schedule, mbarrier/TMA wrappers, the
// 128B-swizzled tile address and the constant-twiddle radix-16 butterfly.
#pragma once

#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace dpp {

// Test hook (the one environment switch of the FFT kernels): DPP_RING_STRESS=1
// plans every L2-ring kernel with a 4-slot ring and lag 2, so ring slots are
// reused many times per launch and both cross-CTA waits (P2 on P1, P1 on slot
// release) fire — tests/test_fft_gpu.py runs the shipped kernels that way.
inline bool ring_stress() {
  static const int on = [] {
    const char* e = std::getenv("DPP_RING_STRESS");
    return e && std::atoi(e) != 0 ? 1 : 0;
  }();
  return on != 0;
}

namespace ring {

__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.cs.v2.f32 {%0, %1}, [%2];"
               : "=f"(v.x), "=f"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_l2(const float2* p) {
  float2 v;
  asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_stream(float2* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_l2(float2* p, float2 v) {
  asm volatile("st.global.cg.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_count(const int* p, int target) {
  if (ld_acquire(p) >= target) return;
  int ns = 32;
  while (ld_acquire(p) < target) {
    __nanosleep(ns);
    ns = ns < 512 ? ns * 2 : 512;
  }
}

// ticket group -> (pass, transform)
__device__ __forceinline__ void decode(int grp, int batch, int lag, int& pass, int& t) {
  if (grp < lag) {
    pass = 1;
    t = grp;
    return;
  }
  const int m = grp - lag;
  const int mid = 2 * (batch - lag);
  if (m < mid) {
    pass = (m & 1) ? 2 : 1;
    t = (m & 1) ? (m >> 1) : lag + (m >> 1);
  } else {
    pass = 2;
    t = batch - lag + (m - mid);
  }
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
// v * (c + i s) for a compile-time rotation: FMUL2 with a broadcast scalar, then
// FFMA2 on the swapped/negated pair (operand modifiers, no register pairs)
__device__ __forceinline__ float2 cmulc(float2 v, float c, float s) {
  return __ffma2_rn(make_float2(-v.y, v.x), make_float2(s, s), __fmul2_rn(v, make_float2(c, c)));
}
__device__ __forceinline__ void dft4c(float2& x0, float2& x1, float2& x2, float2& x3) {
  float2 s02 = cadd(x0, x2), d02 = csub(x0, x2);
  float2 s13 = cadd(x1, x3), d13 = csub(x1, x3);
  d13 = make_float2(d13.y, -d13.x);  // * -i
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, d13);
  x3 = csub(d02, d13);
}
// natural-order 16-point DFT (4 x 4), constant twiddles through cmulc
__device__ __forceinline__ void dft16c(float2 (&v)[16]) {
  dft4c(v[0], v[4], v[8], v[12]);
  dft4c(v[1], v[5], v[9], v[13]);
  dft4c(v[2], v[6], v[10], v[14]);
  dft4c(v[3], v[7], v[11], v[15]);
  const float c1 = 0.92387953251128676f, s1 = 0.38268343236508977f, h = 0.70710678118654752f;
  v[5] = cmulc(v[5], c1, -s1);    // W16^1
  v[9] = cmulc(v[9], h, -h);      // W16^2
  v[13] = cmulc(v[13], s1, -c1);  // W16^3
  v[6] = cmulc(v[6], h, -h);      // W16^2
  v[10] = make_float2(v[10].y, -v[10].x);  // W16^4 = -i
  v[14] = cmulc(v[14], -h, -h);   // W16^6
  v[7] = cmulc(v[7], s1, -c1);    // W16^3
  v[11] = cmulc(v[11], -h, -h);   // W16^6
  v[15] = cmulc(v[15], -c1, s1);  // W16^9
  float2 r[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 a0 = v[4 * k1 + 0], a1 = v[4 * k1 + 1], a2 = v[4 * k1 + 2], a3 = v[4 * k1 + 3];
    dft4c(a0, a1, a2, a3);
    r[k1 + 0] = a0;
    r[k1 + 4] = a1;
    r[k1 + 8] = a2;
    r[k1 + 12] = a3;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = r[i];
}

__device__ __forceinline__ int swz(int r, int c) { return r * 16 + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1); }

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_try_u32(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }


__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const void* tmap, int x, int y, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const void* tmap, int x, int y, const void* src, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(tmap),
               "r"(x), "r"(y), "r"(smem_u32(src)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_l2_hint(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

// two adjacent complex values (one 16-byte chunk, 16-byte aligned)
__device__ __forceinline__ void st_l2_hint2(float2* p, float2 a, float2 b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a.x), "f"(a.y), "f"(b.x),
               "f"(b.y), "l"(pol)
               : "memory");
}

// one 32-byte sector: four complex values (32-byte aligned; STG.256 on sm_100)
__device__ __forceinline__ void st_l2_hint4(float2* p, float2 a, float2 b, float2 c, float2 d, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "f"(a.x),
               "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y), "f"(d.x), "f"(d.y), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(x), "r"(y)
               : "memory");
}

}  // namespace ring
}  // namespace dpp
