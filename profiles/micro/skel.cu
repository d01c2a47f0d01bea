// Data-movement skeleton of the C2 kernel (4096 x 2^16 complex64): what the
// HBM side alone reaches for a given cluster size, with and without the DSMEM
// exchange, launched per FFT or as persistent clusters with a prefetched tile.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1203_4938_b200/csrc \
//        profiles/micro/skel.cu -o profiles/micro/skel -lcuda && ./profiles/micro/skel
//
// Every CTA moves one 256 x 16 tile (32 KB) of one transform: TMA load ->
// registers -> (optional st.async scatter inside the cluster) -> 16 B-segment
// streaming stores, exactly the per-CTA traffic of fft_cluster_rows<256,256,16>.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "tma.cuh"

#include <cstdarg>

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

constexpr int N1 = 256, N2 = 256, N = N1 * N2, W = 16, T1 = 16, THREADS = 256;
constexpr int TILE = N1 * W;  // elements

// EX: 0 = no exchange, 1 = st.async scatter to the cluster peers (+ cluster barrier)
template <int EX>
__global__ void __launch_bounds__(THREADS, 4) skel(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out,
                                                   int C) {
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  float2* buf = smem;
  const int p = (int)(blockIdx.x % 16);
  const int64_t t = blockIdx.x / 16;
  const int tid = threadIdx.x;
  const int q0 = EX ? (int)cluster_ctarank() : 0;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[0], TILE * 8);
    mbar_arrive_expect_tx(&bars[1], TILE * 8);
    tma_load_2d(buf, &tin, p * W, (int)(t * N1), &bars[0]);
  }
  __syncthreads();
  const int col = tid % W, j = tid / W;
  float2 v[16];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = buf[(j + T1 * i) * W + col];
  if (EX) {
    cluster_arrive_relaxed();
    cluster_wait();
    const uint32_t base = smem_u32(buf), rbar = smem_u32(&bars[1]);
    // element i goes to peer (q0 + i) % C at the slot it came from: every
    // slot of every receiver is written exactly once
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t off = (uint32_t)(((j + T1 * i) * W + col) * 8);
      const uint32_t peer = (uint32_t)((q0 + i) % C);
      st_async_f2(mapa_u32(base + off, peer), v[i], mapa_u32(rbar, peer));
    }
    mbar_wait(&bars[1], 0);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = buf[(j + T1 * i) * W + col];
  }
  float2* dst = out + t * N + p * W + col;
#pragma unroll
  for (int i = 0; i < 16; ++i) __stcs(dst + (int64_t)(j + T1 * i) * N1, v[i]);
}

// persistent: each CTA walks transforms t = first, first + stride, ... with the
// next tile's TMA load issued before the current one is consumed (2 buffers)
__global__ void __launch_bounds__(THREADS, 3) skel_pers(const __grid_constant__ CUtensorMap tin,
                                                        float2* __restrict__ out, int64_t batch, int nctas) {
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  const int tid = threadIdx.x;
  const int64_t units = batch * 16;
  int64_t u = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if (u < units) {
      mbar_arrive_expect_tx(&bars[0], TILE * 8);
      tma_load_2d(smem, &tin, (int)(u % 16) * W, (int)(u / 16 * N1), &bars[0]);
    }
  }
  __syncthreads();
  const int col = tid % W, j = tid / W;
  uint32_t phase[2] = {0, 0};
  for (int k = 0; u < units; u += nctas, ++k) {
    const int s = k & 1;
    const int64_t un = u + nctas;
    if (tid == 0 && un < units) {
      mbar_arrive_expect_tx(&bars[s ^ 1], TILE * 8);
      tma_load_2d(smem + (s ^ 1) * TILE, &tin, (int)(un % 16) * W, (int)(un / 16 * N1), &bars[s ^ 1]);
    }
    mbar_wait(&bars[s], phase[s]);
    phase[s] ^= 1;
    float2 v[16];
    const float2* buf = smem + s * TILE;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = buf[(j + T1 * i) * W + col];
    __syncthreads();  // buffer s free before it is refilled two units later
    float2* dst = out + (u / 16) * N + (u % 16) * W + col;
#pragma unroll
    for (int i = 0; i < 16; ++i) __stcs(dst + (int64_t)(j + T1 * i) * N1, v[i]);
  }
}

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main() {
  const int64_t batch = 4096;
  const size_t bytes = (size_t)batch * N * 8;
  float2 *in, *out;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 0, bytes));
  CUtensorMap tmap;
  if (make_tmap_c64(&tmap, in, (uint64_t)batch * N1, N2, N1, W)) return 1;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) -> float {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    std::vector<float> ms;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float m;
      cudaEventElapsedTime(&m, e0, e1);
      ms.push_back(m);
    }
    std::sort(ms.begin(), ms.end());
    return ms[ms.size() / 2];
  };
  const double gb = 2.0 * bytes / 1e9;
  CK(cudaFuncSetAttribute(skel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * 8));
  CK(cudaFuncSetAttribute(skel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * 8));
  CK(cudaFuncSetAttribute(skel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(skel<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(skel_pers, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TILE * 8));
  for (int C : {1, 2, 4, 8, 16}) {
    for (int smem_kb : {32, 37, 48, 68}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(batch * 16));
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = smem_kb * 1024;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      CK(cudaFuncSetAttribute(skel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024));
      CK(cudaOccupancyMaxActiveClusters(&n, skel<1>, &cfg));
      printf("{\"cluster\": %d, \"smem_kb\": %d, \"max_active_clusters\": %d, \"ctas\": %d, \"per_sm\": %.2f}\n", C,
             smem_kb, n, n * C, (double)n * C / sms);
    }
  }
  CK(cudaFuncSetAttribute(skel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * 8));
  for (int ex = 0; ex < 2; ++ex) {
    for (int C : {1, 2, 4, 8, 16}) {
      if (ex && C == 1) continue;
      auto launch = [&]() {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(batch * 16));
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = TILE * 8;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (ex)
          cudaLaunchKernelEx(&cfg, skel<1>, tmap, out, C);
        else
          cudaLaunchKernelEx(&cfg, skel<0>, tmap, out, C);
      };
      const float ms = timeit(launch);
      CK(cudaGetLastError());
      printf("{\"variant\": \"percta\", \"exchange\": %d, \"cluster\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", ex, C,
             ms, gb / ms * 1e3);
    }
  }
  for (int per : {2, 3}) {
    const int nctas = sms * per;
    const float ms = timeit([&]() {
      skel_pers<<<nctas, THREADS, 2 * TILE * 8>>>(tmap, out, batch, nctas);
    });
    CK(cudaGetLastError());
    printf("{\"variant\": \"persistent\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", per, ms,
           gb / ms * 1e3);
  }
  // plain device copy for reference
  const float ms = timeit([&]() { cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice); });
  printf("{\"variant\": \"memcpy\", \"ms\": %.4f, \"GBps\": %.1f}\n", ms, gb / ms * 1e3);
  return 0;
}
