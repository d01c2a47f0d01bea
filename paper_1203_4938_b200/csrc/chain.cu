// Pointwise adapter nodes of the C5 chain:
//   gray u8 -> complex64 (g, 0) -> 2-D FFT -> u8 log-magnitude -> compression
// Both adapters are written as kernel-language pointwise nodes in
// apps/chain.py (so the reference engine can run them too); these kernels are
// their native implementations.  to_complex is exact; spectrum_u8 uses the
// device logf (<= 1 ulp), so against the reference interpreter's numpy log it
// is reported as a mismatch count, not bit-exact.
#include <cstdint>

#include "common.cuh"

namespace dpp {

// y[i] = (float2)((float)(x[i]), 0.0f)
__global__ void u8_to_complex_kernel(const uchar4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const uchar4 v = x[i];
  y[2 * i] = make_float4((float)v.x, 0.f, (float)v.y, 0.f);
  y[2 * i + 1] = make_float4((float)v.z, 0.f, (float)v.w, 0.f);
}

// m = sqrt(z.x*z.x + z.y*z.y); v = floor(alpha * log(1 + m)); y = (uchar)clamp(v, 0, 255)
__global__ void spectrum_u8_kernel(const float4* __restrict__ z, uchar2* __restrict__ y, int64_t n2, float alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const float4 a = z[i];
  const float m0 = __fsqrt_rn(__fadd_rn(__fmul_rn(a.x, a.x), __fmul_rn(a.y, a.y)));
  const float m1 = __fsqrt_rn(__fadd_rn(__fmul_rn(a.z, a.z), __fmul_rn(a.w, a.w)));
  const float v0 = floorf(__fmul_rn(alpha, logf(__fadd_rn(1.0f, m0))));
  const float v1 = floorf(__fmul_rn(alpha, logf(__fadd_rn(1.0f, m1))));
  y[i] = make_uchar2((unsigned char)fminf(fmaxf(v0, 0.f), 255.f), (unsigned char)fminf(fmaxf(v1, 0.f), 255.f));
}

}  // namespace dpp

extern "C" {

int dpp_u8_to_complex(const uint8_t* x, float* y, int64_t n, void* stream) {
  if (n < 0 || n % 4) return dpp::fail(DPP_EINVAL, "u8_to_complex needs a multiple of 4 samples");
  if (n == 0) return DPP_OK;
  const int64_t n4 = n / 4;
  dpp::u8_to_complex_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uchar4*>(x), reinterpret_cast<float4*>(y), n4);
  DPP_LAUNCH_CHECK("u8_to_complex_kernel");
  return DPP_OK;
}

int dpp_spectrum_u8(const float* z, uint8_t* y, int64_t n, float alpha, void* stream) {
  if (n < 0 || n % 2) return dpp::fail(DPP_EINVAL, "spectrum_u8 needs an even sample count");
  if (n == 0) return DPP_OK;
  const int64_t n2 = n / 2;
  dpp::spectrum_u8_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(z), reinterpret_cast<uchar2*>(y), n2, alpha);
  DPP_LAUNCH_CHECK("spectrum_u8_kernel");
  return DPP_OK;
}

}  // extern "C"
