/* A plain C consumer of libdpp_b200.so: no Python, no torch — the drop-in
 * boundary as a reference-side binding sees it (include/dpp_b200.h).  Known
 * answers from the reference's own tests (test_fft.py:18-36): impulse -> all
 * ones, constant -> DC only, [1,2,3,4] -> [10, -2+2i, -2, -2-2i] (N=4), plus
 * the plan-time error convention (EINVAL + dpp_last_error). */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dpp_b200.h"

static int fails = 0;
#define CHECK(c, ...)                 \
  do {                                \
    if (!(c)) {                       \
      fprintf(stderr, __VA_ARGS__);   \
      fputc('\n', stderr);            \
      ++fails;                        \
    }                                 \
  } while (0)

static void run(int64_t n, int64_t batch) {
  const size_t bytes = (size_t)(n * batch) * 2 * sizeof(float);
  float* h = (float*)calloc(1, bytes);
  float* g = (float*)calloc(1, bytes);
  /* transform 0: impulse; transform 1: constant 1; others: impulse at 1 */
  h[0] = 1.f;
  for (int64_t i = 0; i < n; ++i) h[2 * (n + i)] = 1.f;
  for (int64_t b = 2; b < batch; ++b) h[2 * (b * n + 1)] = 1.f;
  float *din = NULL, *dout = NULL;
  CHECK(cudaMalloc((void**)&din, bytes) == cudaSuccess, "cudaMalloc");
  CHECK(cudaMalloc((void**)&dout, bytes) == cudaSuccess, "cudaMalloc");
  cudaMemcpy(din, h, bytes, cudaMemcpyHostToDevice);
  dpp_fft_plan* plan = NULL;
  size_t ws = 0;
  int rc = dpp_fft_plan_create(&plan, 1, n, 1, batch, &ws);
  CHECK(rc == DPP_OK, "plan n=%lld: %s", (long long)n, dpp_last_error());
  rc = dpp_fft_c2c_forward(plan, din, dout, NULL, NULL);
  CHECK(rc == DPP_OK, "execute n=%lld: %s", (long long)n, dpp_last_error());
  CHECK(cudaDeviceSynchronize() == cudaSuccess, "sync");
  cudaMemcpy(g, dout, bytes, cudaMemcpyDeviceToHost);
  double e0 = 0, e1 = 0, e2 = 0;
  for (int64_t k = 0; k < n; ++k) {
    e0 = fmax(e0, fabs(g[2 * k] - 1.0) + fabs(g[2 * k + 1]));
    const double want = k == 0 ? (double)n : 0.0;
    e1 = fmax(e1, fabs(g[2 * (n + k)] - want) + fabs(g[2 * (n + k) + 1]));
    if (batch > 2) { /* impulse at 1: X[k] = exp(-2 pi i k / n) */
      const double a = -2.0 * 3.14159265358979323846 * (double)k / (double)n;
      e2 = fmax(e2, fabs(g[2 * (2 * n + k)] - cos(a)) + fabs(g[2 * (2 * n + k) + 1] - sin(a)));
    }
  }
  CHECK(e0 < 1e-5, "n=%lld impulse: max err %g", (long long)n, e0);
  CHECK(e1 < 1e-6 * n, "n=%lld constant: max err %g", (long long)n, e1);
  CHECK(e2 < 1e-5, "n=%lld shifted impulse: max err %g", (long long)n, e2);
  dpp_fft_plan_destroy(plan);
  cudaFree(din);
  cudaFree(dout);
  free(h);
  free(g);
}

int main(void) {
  CHECK(dpp_abi_version() == DPP_ABI_VERSION, "ABI version %d", dpp_abi_version());
  /* test_fft.py:18-36: [1,2,3,4] -> [10, -2+2i, -2, -2-2i] */
  {
    float h[8] = {1, 0, 2, 0, 3, 0, 4, 0}, g[8];
    const float want[8] = {10, 0, -2, 2, -2, 0, -2, -2};
    float *d = NULL;
    cudaMalloc((void**)&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    dpp_fft_plan* p = NULL;
    CHECK(dpp_fft_plan_create(&p, 1, 4, 1, 1, NULL) == DPP_OK, "plan 4: %s", dpp_last_error());
    CHECK(dpp_fft_c2c_forward(p, d, d, NULL, NULL) == DPP_OK, "execute 4 in place: %s", dpp_last_error());
    cudaMemcpy(g, d, sizeof(g), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) CHECK(fabsf(g[i] - want[i]) < 1e-5f, "N=4 element %d: %g vs %g", i, g[i], want[i]);
    dpp_fft_plan_destroy(p);
    cudaFree(d);
  }
  run(1024, 4);
  run(4096, 3);
  run(65536, 5);
  run(1 << 18, 3);
  /* plan-time errors: EINVAL and a message (fft.py:133-139) */
  dpp_fft_plan* bad = NULL;
  CHECK(dpp_fft_plan_create(&bad, 1, 12, 1, 1, NULL) == DPP_EINVAL && bad == NULL, "n=12 accepted");
  CHECK(strstr(dpp_last_error(), "power of two") != NULL, "error text: %s", dpp_last_error());
  if (fails) {
    fprintf(stderr, "%d failure(s)\n", fails);
    return 1;
  }
  printf("abi smoke ok\n");
  return 0;
}
