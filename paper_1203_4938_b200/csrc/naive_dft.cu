// naive_dft on the device (apps/fft.py:32-42): X_k = sum_n x_n exp(-2 pi i k n / N),
// binary64 accumulation, rounded once to complex64 — the reference's quadratic
// oracle, offered by the product API (`apps.fft.naive_dft`) as an
// independent check of the fast transforms at sizes the host cannot reach.
// Phases are reduced exactly in integer arithmetic ((k*n) mod N) and evaluated
// with sincospi in binary64.
#include <cstdint>

#include "common.cuh"

namespace dpp {

__global__ void naive_dft_kernel(const float2* __restrict__ x, float2* __restrict__ y, int64_t n, int64_t batch) {
  extern __shared__ double2 tile[];  // x staged in binary64 chunks
  const int64_t b = blockIdx.y;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float2* xs = x + b * n;
  double re = 0.0, im = 0.0;
  const int64_t chunk = blockDim.x;
  for (int64_t base = 0; base < n; base += chunk) {
    __syncthreads();
    if (base + threadIdx.x < n) {
      const float2 v = xs[base + threadIdx.x];
      tile[threadIdx.x] = make_double2((double)v.x, (double)v.y);
    }
    __syncthreads();
    if (k < n) {
      const int64_t lim = n - base < chunk ? n - base : chunk;
      for (int64_t t = 0; t < lim; ++t) {
        const int64_t ph = (k * (base + t)) % n;
        double s, c;
        sincospi(-2.0 * (double)ph / (double)n, &s, &c);
        const double2 v = tile[t];
        re += v.x * c - v.y * s;
        im += v.x * s + v.y * c;
      }
    }
  }
  if (k < n) y[b * n + k] = make_float2((float)re, (float)im);
}

}  // namespace dpp

extern "C" int dpp_naive_dft(const float* x, float* y, int64_t n, int64_t batch, void* stream) {
  if (n < 1 || batch < 0) return dpp::fail(DPP_EINVAL, "signal must have at least one sample");
  if (batch == 0) return DPP_OK;
  const int threads = 256;
  dim3 grid((unsigned)((n + threads - 1) / threads), (unsigned)batch);
  dpp::naive_dft_kernel<<<grid, threads, threads * sizeof(double2), (cudaStream_t)stream>>>(
      reinterpret_cast<const float2*>(x), reinterpret_cast<float2*>(y), n, batch);
  DPP_LAUNCH_CHECK("naive_dft_kernel");
  return DPP_OK;
}
