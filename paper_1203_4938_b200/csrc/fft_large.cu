// 1-D transforms above 2^17 points (the reference's fft() takes any power of
// two, apps/fft.py:126-174): n = A * Bc with column length Bc in {4096, 16384}
// (the column ring's lengths) and row length A = n / Bc <= 65536.
//
// Index split n = Bc i + j (i < A, j < Bc), k = k1 + A k2:
//   X[k1 + A k2] = sum_j W_Bc^{j k2} W_n^{j k1} sum_i x[Bc i + j] W_A^{i k1}
// 1. transpose: the A x Bc view of x -> Bc x A (T[j][i] = x[Bc i + j]);
// 2. row pass: A-point FFTs of the Bc rows of T (any 1-D kernel <= 2^17);
// 3. column ring (fft2d_l2.cu, TW): W_n^{j k1} applied to the loaded tile,
//    Bc-point FFTs down the A columns; row k2 of the result is
//    X[A k2 .. A k2 + A) — natural order, no second transpose.
// Three HBM passes (48 B per point) against the 16 B compulsory; the two
// FFT passes are the tuned kernels, the transpose is a 32 x 32 tile copy.
//
// Two passes (32 B per point) when A is 4096 .. 32768 and Bc is 1024, 2048,
// 4096, 16384 or 32768 (n = 2^22 .. 2^30): steps 1 + 2 become ONE column ring over the A x Bc view of x
// (A-point FFTs down its Bc columns) whose ring slot is laid out per column,
// so each P2 block writes 16 consecutive k1 of one row of T by a TMA box
// (fft2d_l2.cu, XP) — the transpose rides on the exchange that the column
// FFT does anyway.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"

namespace dpp {
namespace {

// batch of rows x cols complex64 matrices -> cols x rows; 32 x 32 tiles,
// 32 x 8 threads, padded shared tile (no bank conflicts on the column read)
__global__ void __launch_bounds__(256) transpose_c64(const float2* __restrict__ in, float2* __restrict__ out,
                                                     int64_t rows, int64_t cols) {
  __shared__ float2 t[32][33];
  const int64_t mat = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const float2* src = in + mat * rows * cols;
  float2* dst = out + mat * rows * cols;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int k = 0; k < 32; k += 8) t[ty + k][tx] = __ldcs(src + (r0 + ty + k) * cols + c0 + tx);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) __stcs(dst + (c0 + ty + k) * rows + r0 + tx, t[tx][ty + k]);
}

// data[r][c] *= W_n^{r (c0 + c)} for a rows x cols row-major block: the
// four-step twiddle of the row-sharded 1-D transform (distributed.py), whose
// column slab of rank q starts at global column c0.  Angles in binary64 from
// the exact integer phase (r (c0 + c)) mod n, rounded once.
__global__ void __launch_bounds__(256) twiddle_slab(float2* __restrict__ data, int64_t rows, int64_t cols, int64_t c0,
                                                    int64_t n) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const int64_t m = (int64_t)(((unsigned __int128)r * (uint64_t)(c0 + c)) % (uint64_t)n);
    double sn, cs;
    sincospi(-2.0 * (double)m / (double)n, &sn, &cs);
    const float2 v = data[e];
    data[e] = cmul(v, make_float2((float)cs, (float)sn));
  }
}

}  // namespace

int fft_twiddle_slab(float2* data, int64_t rows, int64_t cols, int64_t c0, int64_t n, cudaStream_t s) {
  if (rows < 0 || cols < 0 || c0 < 0 || n < 1) return fail(DPP_EINVAL, "bad twiddle block");
  if (rows * cols == 0) return DPP_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (rows * cols + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 8LL * sms ? blocks : 8LL * sms);
  twiddle_slab<<<grid, 256, 0, s>>>(data, rows, cols, c0, n);
  DPP_LAUNCH_CHECK("twiddle_slab");
  return DPP_OK;
}

int fft_large_init(FftPlan* p) {
  const int64_t n = p->n0;
  // two passes need the second factor Bc in {1024, 2048, 4096, 16384, 32768}
  // (the twiddled ring) and the first A in 4096 .. 32768 (the transposed-output ring)
  auto xp_ok = [](int64_t a) { return a >= 4096 && a <= 32768; };
  int64_t bc = n <= (1LL << 24) ? 4096 : 16384;
  // 2^26 .. 2^28: the 8192-row twiddled ring (8192 x 8192, 16384 x 8192,
  // 32768 x 8192) measured 2-3 % faster than the 16384-row one (session 5)
  if (n >= (1LL << 26) && n <= (1LL << 28)) bc = 8192;
  // another column length that gives two passes (2^22: 4096 x 1024, 2^23:
  // 4096 x 2048, 2^30: 32768 x 32768)
  if (!xp_ok(n / bc))
    for (const int64_t c : {20480 - bc, (int64_t)2048, (int64_t)1024, (int64_t)32768})
      if (xp_ok(n / c)) {
        bc = c;
        break;
      }
  const int64_t a = n / bc;
  if (a < 32 || a > 65536)
    return fail(DPP_ENOTSUP, "1-D transform size %lld is outside 2^18..2^30", (long long)n);
  p->kind = FftPlan::LARGE;
  p->n1a = a;
  p->n2a = bc;
  // in-place calls go through a scratch of big_chunk transforms (<= 256 MB, or one transform)
  const int64_t per = (1LL << 25) / n > 1 ? (1LL << 25) / n : 1;
  p->big_chunk = p->batch < per ? (p->batch > 0 ? p->batch : 1) : per;
  const bool two_pass = xp_ok(a);
  if (two_pass) {
    p->xcols = new FftPlan();
    p->xcols->rank = 2;
    p->xcols->n0 = a;
    p->xcols->n1 = bc;
    p->xcols->batch = p->batch > 0 ? p->batch : 1;
    p->xcols->device = p->device;
    if (int rc = fft2d_colring_init(p->xcols))
      return rc == DPP_ENOTSUP ? fail(rc, "no column ring for %lld x %lld", (long long)a, (long long)bc) : rc;
  }
  if (!two_pass) {
    p->rows = new FftPlan();
    p->rows->rank = 1;
    p->rows->n0 = a;
    p->rows->n1 = 1;
    p->rows->batch = (p->batch > 0 ? p->batch : 1) * bc;
    p->rows->device = p->device;
    if (int rc = fft1d_plan_init(p->rows)) return rc;
  }
  p->cols = new FftPlan();
  p->cols->rank = 2;
  p->cols->n0 = bc;
  p->cols->n1 = a;
  p->cols->batch = p->batch > 0 ? p->batch : 1;
  p->cols->device = p->device;
  if (int rc = fft2d_colring_init(p->cols)) return rc == DPP_ENOTSUP ? fail(rc, "no column ring for %lld x %lld",
                                                                          (long long)bc, (long long)a) : rc;
  const int64_t nhi = n / 16384 + 1;
  std::vector<float2> tw((size_t)(16384 + nhi));
  for (int64_t m = 0; m < 16384; ++m) {
    const double ang = -2.0 * M_PI * (double)m / (double)n;
    tw[(size_t)m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  for (int64_t h = 0; h < nhi; ++h) {
    const double ang = -2.0 * M_PI * (double)((16384 * h) % n) / (double)n;
    tw[(size_t)(16384 + h)] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  DPP_CUDA_CHECK(cudaMalloc(&p->big_tw, tw.size() * sizeof(float2)));
  DPP_CUDA_CHECK(cudaMemcpy(p->big_tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
  if (two_pass)
    snprintf(p->desc, sizeof(p->desc),
             "%lld x %lld four-step in two passes: %lld-point column ring with transposed output, twiddled "
             "%lld-point column ring",
             (long long)a, (long long)bc, (long long)a, (long long)bc);
  else
    snprintf(p->desc, sizeof(p->desc),
             "%lld x %lld four-step: transpose, %lld-point rows (%.120s), twiddled %lld-point column ring",
             (long long)a, (long long)bc, (long long)a, p->rows->desc, (long long)bc);
  return DPP_OK;
}

int fft_large_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  const int64_t n = p->n0, a = p->n1a, bc = p->n2a;
  const bool inplace = in == out;
  if (inplace && !p->big_scratch) {
    // first in-place call: the scratch is created once and kept by the plan
    FftPlan* mp = const_cast<FftPlan*>(p);
    DPP_CUDA_CHECK(cudaMalloc(&mp->big_scratch, (size_t)p->big_chunk * n * sizeof(float2)));
  }
  const int64_t chunk = inplace ? p->big_chunk : batch;
  const float2* twlo = p->big_tw;
  const float2* twhi = p->big_tw + 16384;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t nb = batch - b0 < chunk ? batch - b0 : chunk;
    const float2* src = in + b0 * n;
    float2* dst = out + b0 * n;
    float2* t = inplace ? p->big_scratch : dst;
    if (p->xcols) {
      if (int rc = fft2d_colring_execute(p->xcols, const_cast<float2*>(src), nb, s, nullptr, 0.f, t, nullptr, nullptr,
                                         true))
        return rc;
      if (int rc = fft2d_colring_execute(p->cols, t, nb, s, nullptr, 0.f, dst, twlo, twhi)) return rc;
      continue;
    }
    transpose_c64<<<dim3((unsigned)(bc / 32), (unsigned)(a / 32), (unsigned)nb), dim3(32, 8), 0, s>>>(src, t, a, bc);
    DPP_LAUNCH_CHECK("transpose_c64");
    if (int rc = fft1d_execute(p->rows, t, t, nb * bc, s)) return rc;
    if (int rc = fft2d_colring_execute(p->cols, t, nb, s, nullptr, 0.f, dst, twlo, twhi)) return rc;
  }
  return DPP_OK;
}

}  // namespace dpp
