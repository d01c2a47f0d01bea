// Shared helpers for the sm_100a library: error convention, complex math,
// in-register DFTs.  Error convention follows include/dpp_b200.h: every entry
// point returns DPP_OK or a code and records a message retrievable with
// dpp_last_error() (thread-local), mapped on the host onto the reference's
// PlanError / EngineRuntimeError (/root/reference/pkg/src/dpp/errors.py:62-81).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>

#include "../../include/dpp_b200.h"

namespace dpp {

void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

// A failed API call also leaves its code as the runtime's "last error"; it is
// consumed here so a later launch check does not report it again (e.g. a
// stream-ordering call refused inside a CUDA-graph capture attempt).
#define DPP_CUDA_CHECK(expr)                                                         \
  do {                                                                               \
    cudaError_t err__ = (expr);                                                      \
    if (err__ != cudaSuccess) {                                                      \
      (void)cudaGetLastError();                                                      \
      return ::dpp::fail(DPP_ECUDA, "%s failed: %s (%s:%d)", #expr,                  \
                         cudaGetErrorString(err__), __FILE__, __LINE__);             \
    }                                                                                \
  } while (0)

#define DPP_LAUNCH_CHECK(what)                                                       \
  do {                                                                               \
    cudaError_t err__ = cudaGetLastError();                                          \
    if (err__ != cudaSuccess)                                                        \
      return ::dpp::fail(DPP_ECUDA, "launch of %s failed: %s", what,                 \
                         cudaGetErrorString(err__));                                 \
  } while (0)

// ---------------------------------------------------------------------------
// complex helpers (float2 = re, im).  FFT arithmetic is tolerance-checked, so
// contraction to FFMA is allowed here; the bit-exact codec uses __f*_rn.

// sm_100 packed binary32 pairs (SASS FADD2 / FMUL2 / FFMA2): one instruction
// per complex add/sub, two per complex multiply (operand broadcast .F32 and
// negation are free modifiers).  Halves the FP issue slots of the butterflies.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a * w = a.x * (w.x, w.y) + a.y * (-w.y, w.x).  The rotated pair is the FIRST
// FFMA2 operand: only there does ptxas encode it as a swap + lane-negate
// modifier (-R.F32x2.LO_HI.NP); as the second operand it materialises the pair
// with a MOV + FADD per multiply.  Products commute, so the bits are the same.
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
  return __ffma2_rn(make_float2(-w.y, w.x), make_float2(a.y, a.y),
                    __fmul2_rn(w, make_float2(a.x, a.x)));
}
// same with the rotated twiddle (-w.y, w.x) precomputed (tables store both halves)
__device__ __forceinline__ float2 cmul_pre(float2 a, float2 w, float2 wrot) {
  return __ffma2_rn(wrot, make_float2(a.y, a.y), __fmul2_rn(w, make_float2(a.x, a.x)));
}
// multiply by -i
__device__ __forceinline__ float2 cmul_mi(float2 a) { return make_float2(a.y, -a.x); }

// W_8^1 = (1 - i)/sqrt2, W_8^3 = (-1 - i)/sqrt2
__device__ __forceinline__ float2 cmul_w8_1(float2 a) {
  const float h = 0.70710678118654752f;
  return cmul(a, make_float2(h, -h));
}
__device__ __forceinline__ float2 cmul_w8_3(float2 a) {
  const float h = 0.70710678118654752f;
  return cmul(a, make_float2(-h, -h));
}

// ---------------------------------------------------------------------------
// Natural-order in-register DFTs of size 2, 4, 8, 16 (forward, unnormalised).

__device__ __forceinline__ void dft2(float2& a, float2& b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

// in: x0..x3 natural, out: natural
// (folding the -i rotation into FFMA2s with 0/+-1 lane constants was measured:
// +67 FP and +38 MOV instructions per thread in the 2^16 kernel — kept simple)
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
  float2 s02 = cadd(x0, x2), d02 = csub(x0, x2);
  float2 s13 = cadd(x1, x3), d13 = cmul_mi(csub(x1, x3));
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, d13);
  x3 = csub(d02, d13);
}

__device__ __forceinline__ void dft8(float2 (&v)[8]) {
  // even/odd split: E = DFT4(v0,v2,v4,v6), O = DFT4(v1,v3,v5,v7)
  dft4(v[0], v[2], v[4], v[6]);
  dft4(v[1], v[3], v[5], v[7]);
  float2 o1 = cmul_w8_1(v[3]);
  float2 o2 = cmul_mi(v[5]);
  float2 o3 = cmul_w8_3(v[7]);
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1];
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

__device__ __forceinline__ void dft16(float2 (&v)[16]) {
  // n = 4*n1 + n0 ; k = k1 + 4*k2
  // step 1: A[n0][k1] = DFT4_{n1}(v[4 n1 + n0]) stored back in v[4 k1 + n0]
  dft4(v[0], v[4], v[8], v[12]);
  dft4(v[1], v[5], v[9], v[13]);
  dft4(v[2], v[6], v[10], v[14]);
  dft4(v[3], v[7], v[11], v[15]);
  // step 2: twiddle W16^{n0 k1}; element (n0, k1) lives at v[4 k1 + n0]
  const float c1 = 0.92387953251128676f, s1 = 0.38268343236508977f, h = 0.70710678118654752f;
  v[5] = cmul(v[5], make_float2(c1, -s1));     // n0=1,k1=1 : W^1
  v[9] = cmul_w8_1(v[9]);                       // n0=1,k1=2 : W^2
  v[13] = cmul(v[13], make_float2(s1, -c1));   // n0=1,k1=3 : W^3
  v[6] = cmul_w8_1(v[6]);                       // n0=2,k1=1 : W^2
  v[10] = cmul_mi(v[10]);                       // n0=2,k1=2 : W^4
  v[14] = cmul_w8_3(v[14]);                     // n0=2,k1=3 : W^6
  v[7] = cmul(v[7], make_float2(s1, -c1));     // n0=3,k1=1 : W^3
  v[11] = cmul_w8_3(v[11]);                     // n0=3,k1=2 : W^6
  v[15] = cmul(v[15], make_float2(-c1, s1));   // n0=3,k1=3 : W^9
  (void)h;
  // step 3: X[k1 + 4 k2] = DFT4_{n0}(A[n0][k1]) ; inputs v[4k1 + n0], outputs to
  // natural position k1 + 4 k2 — compute per k1 then scatter through temps.
  float2 r[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 a0 = v[4 * k1 + 0], a1 = v[4 * k1 + 1], a2 = v[4 * k1 + 2], a3 = v[4 * k1 + 3];
    dft4(a0, a1, a2, a3);
    r[k1 + 0] = a0; r[k1 + 4] = a1; r[k1 + 8] = a2; r[k1 + 12] = a3;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = r[i];
}

template <int R>
__device__ __forceinline__ void dft_r(float2 (&v)[R]);
template <> __device__ __forceinline__ void dft_r<1>(float2 (&)[1]) {}
template <> __device__ __forceinline__ void dft_r<2>(float2 (&v)[2]) { dft2(v[0], v[1]); }
template <> __device__ __forceinline__ void dft_r<4>(float2 (&v)[4]) { dft4(v[0], v[1], v[2], v[3]); }
template <> __device__ __forceinline__ void dft_r<8>(float2 (&v)[8]) { dft8(v); }
template <> __device__ __forceinline__ void dft_r<16>(float2 (&v)[16]) { dft16(v); }

// C5 adapter node body (apps/chain.py): m = sqrt(re^2 + im^2) in binary32,
// v = floor(alpha * log(1 + m)), u8 clamp; sqrt/log on the SFU (a
// transcendental node, compared with the reference as a mismatch count).
// Shared by the standalone node and the fused 2-D column pass.
__device__ __forceinline__ unsigned char spectrum_u8_one(float re, float im, float alpha) {
  const float m = sqrtf(__fadd_rn(__fmul_rn(re, re), __fmul_rn(im, im)));
  const float v = floorf(__fmul_rn(alpha, __logf(__fadd_rn(1.0f, m))));
  return (unsigned char)fminf(fmaxf(v, 0.f), 255.f);
}

__host__ __device__ constexpr int ilog2(long long n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// ---------------------------------------------------------------------------
// Thread-block cluster / DSMEM primitives (explicit shared::cluster state space:
// cluster-scope release/acquire instead of the generic-pointer GPU-scope fence).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory offset in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float2 ld_cluster(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync() {
  cluster_arrive();
  cluster_wait();
}
// arrive without a memory fence: callers only use it to say "my reads of
// this buffer are done" after consuming the loaded values
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copies (TMA engine, SASS UBLKCP / SYNCS)

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// global -> own shared memory, completion counted on `bar` (bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void st_async_f4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
      "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
      : "memory");
}
// 2-D tiled TMA load (tensor map in param/const space) into own shared memory
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global 3-D TMA store (bulk group); caller fences the async proxy first
__device__ __forceinline__ void tma_store_3d(const void* tmap, int x, int y, int z, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tmap),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// wait only until the bulk stores have READ their shared-memory source (the CTA
// may then exit or reuse it); global visibility is guaranteed at kernel end
__device__ __forceinline__ void bulk_commit_and_wait_all() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}
// asynchronous store into (possibly remote) shared memory; the destination
// CTA's mbarrier at `rbar` (same cluster address space) receives 8 tx bytes
__device__ __forceinline__ void st_async_f2(uint32_t raddr, float2 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
                   raddr),
               "f"(v.x), "f"(v.y), "r"(rbar)
               : "memory");
}

}  // namespace dpp
