// Pointwise adapter nodes of the C5 chain:
//   gray u8 -> complex64 (g, 0) -> 2-D FFT -> u8 log-magnitude -> compression
// Both adapters are written as kernel-language pointwise nodes in
// apps/chain.py (so the reference engine can run them too); these kernels are
// their native implementations.  to_complex is exact; spectrum_u8 uses the
// SFU log (<= 2 ulp), so against the reference interpreter's numpy log it
// is reported as a mismatch count, not bit-exact.
#include <cstdint>

#include "common.cuh"

namespace dpp {

// Both adapters are pure streams (1 B <-> 8 B per sample).  Grid-stride loops
// over a fixed grid of 16 CTAs per SM (a 4096^2 x 64 batch is 10^9 samples: one
// thread per sample made these CTA-launch bound at ~1 TB/s), lane-contiguous
// 16-byte complex-pair accesses, 4 independent pairs in flight per thread.

// y[i] = (float2)((float)(x[i]), 0.0f); pairs: uchar2 -> float4
__global__ void __launch_bounds__(256) u8_to_complex_kernel(const uchar2* __restrict__ x, float4* __restrict__ y,
                                                            int64_t n2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    uchar2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = x[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(y + i + u * stride, make_float4((float)v[u].x, 0.f, (float)v[u].y, 0.f));
  }
  for (; i < n2; i += stride) {
    const uchar2 v = x[i];
    __stcs(y + i, make_float4((float)v.x, 0.f, (float)v.y, 0.f));
  }
}

__device__ __forceinline__ unsigned char spectrum_one(float re, float im, float alpha) {
  return spectrum_u8_one(re, im, alpha);  // common.cuh
}

__global__ void __launch_bounds__(256) spectrum_u8_kernel(const float4* __restrict__ z, uchar2* __restrict__ y,
                                                          int64_t n2, float alpha) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldcs(z + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      y[i + u * stride] = make_uchar2(spectrum_one(a[u].x, a[u].y, alpha), spectrum_one(a[u].z, a[u].w, alpha));
  }
  for (; i < n2; i += stride) {
    const float4 a = __ldcs(z + i);
    y[i] = make_uchar2(spectrum_one(a.x, a.y, alpha), spectrum_one(a.z, a.w, alpha));
  }
}

static unsigned stream_grid(int64_t work) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t blocks = (work + 255) / 256;
  const int64_t cap = (int64_t)sms * 16;
  return (unsigned)(blocks < cap ? blocks : cap);
}

}  // namespace dpp

extern "C" {

int dpp_u8_to_complex(const uint8_t* x, float* y, int64_t n, void* stream) {
  if (n < 0 || n % 4) return dpp::fail(DPP_EINVAL, "u8_to_complex needs a multiple of 4 samples");
  if (n == 0) return DPP_OK;
  const int64_t n2 = n / 2;
  dpp::u8_to_complex_kernel<<<dpp::stream_grid(n2), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uchar2*>(x), reinterpret_cast<float4*>(y), n2);
  DPP_LAUNCH_CHECK("u8_to_complex_kernel");
  return DPP_OK;
}

int dpp_spectrum_u8(const float* z, uint8_t* y, int64_t n, float alpha, void* stream) {
  if (n < 0 || n % 2) return dpp::fail(DPP_EINVAL, "spectrum_u8 needs an even sample count");
  if (n == 0) return DPP_OK;
  const int64_t n2 = n / 2;
  dpp::spectrum_u8_kernel<<<dpp::stream_grid(n2), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(z), reinterpret_cast<uchar2*>(y), n2, alpha);
  DPP_LAUNCH_CHECK("spectrum_u8_kernel");
  return DPP_OK;
}

}  // extern "C"
