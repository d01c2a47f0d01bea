// FFT node, n = 16384 (the C3 row pass, 1-D batches): one transform per CTA
// at a time, held in REGISTERS — 512 compute threads x 32 values — so the
// 128 KB shared-memory stage is free for the next transform's load as soon as
// it has been read, and no exchange leaves the SM (no L2 ring, no tickets).
//
// n = 512 a + t, k = c + 32 d; t = 16 u + v, d = p + 32 q:
//   X[c + 32 p + 1024 q] = sum_v W16^{v q} W512^{v p}
//                            sum_u W32^{u p} W16384^{t c} sum_a W32^{a c} x[512 a + t]
//   1. thread t loads x[512 a + t] (a < 32) from the stage, 32-point FFT over
//      a, twiddle W16384^{t c};
//   2. exchange 1 (through the stage, one round): thread 16 c + v gets the
//      32 values u of its (c, v), 32-point FFT over u, twiddle W512^{v p};
//      the stage then takes the next transform's load;
//   3. exchange 2 (two rounds over p): thread 32 p' + c gets the 16 values v
//      of (c, p') and (c, p' + 16), two 16-point FFTs over v;
//   4. X[c + 32 p + 1024 q] straight from registers: a warp store is 32
//      consecutive c = 256 contiguous bytes.
// Thread 0 issues the next transform's 128 KB bulk load as soon as exchange 1
// has been read out of the stage.  Per point: 8 B read + 8 B written in HBM,
// 48 B through shared memory.
#include <cmath>

#include "common.cuh"
#include "fft_plan.cuh"
#include "l2ring.cuh"

namespace dpp {
namespace rr16k {

using namespace ring;

constexpr int N = 16384;
constexpr int CT = 512;               // threads; thread 0 also issues the loads
constexpr int THREADS = CT;
constexpr size_t STAGE = (size_t)N * sizeof(float2);      // 128 KB
constexpr size_t XBUF = (size_t)(N / 2) * sizeof(float2);  // 64 KB
constexpr size_t SMEM = STAGE + XBUF;

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

// 32-point DFT in place: the caller loads the even inputs x[2i] into v[i]
// and the odd ones x[2i+1] into v[16 + i]; out: X[k] in v[k] (natural order)
__device__ __forceinline__ void dft32_eo(float2 (&v)[32]) {
  float2(&e)[16] = *reinterpret_cast<float2(*)[16]>(&v[0]);
  float2(&o)[16] = *reinterpret_cast<float2(*)[16]>(&v[16]);
  dft16c(e);
  dft16c(o);
  // W32^k = (cos, sin)(-2 pi k / 32)
  constexpr float wc[16] = {1.f, 0.98078528f, 0.923879533f, 0.831469612f, 0.707106781f, 0.555570233f, 0.382683432f, 0.195090322f, 0.f, -0.195090322f, -0.382683432f, -0.555570233f, -0.707106781f, -0.831469612f, -0.923879533f, -0.98078528f};
  constexpr float ws[16] = {-0.f, -0.195090322f, -0.382683432f, -0.555570233f, -0.707106781f, -0.831469612f, -0.923879533f, -0.98078528f, -1.f, -0.98078528f, -0.923879533f, -0.831469612f, -0.707106781f, -0.555570233f, -0.382683432f, -0.195090322f};
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const float2 t = k > 0 ? cmulc(o[k], wc[k], ws[k]) : o[k];
    const float2 ek = e[k];
    v[k] = cadd(ek, t);
    v[k + 16] = csub(ek, t);
  }
}

__global__ void __launch_bounds__(THREADS, 1)
fft16384_rr(const float2* __restrict__ in, float2* __restrict__ out, int batch, const float2* __restrict__ w16k) {
  extern __shared__ __align__(1024) float2 smem[];
  float2* stage = smem;
  float2* xb = smem + N;
  __shared__ __align__(8) uint64_t full;
  const int tid = threadIdx.x;
  const int ntr = blockIdx.x < batch ? (batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // the stage's loads are issued by thread 0: the first here, each next one as
  // soon as every thread has read the stage (no producer warp: all 128
  // registers per thread go to the 32 values in flight)
  auto load = [&](int i) {
    mbar_arrive_expect_tx(&full, (uint32_t)STAGE);
    bulk_g2s(stage, in + (blockIdx.x + (int64_t)gridDim.x * i) * N, (uint32_t)STAGE, &full);
  };
  if (tid == 0) {
    mbar_init(&full, 1);
    fence_mbar_init();
    if (ntr > 0) load(0);
  }
  __syncthreads();

  // -------------------------------------------------------------- compute
  const int t = tid;                      // step 1: column t of the [a][t] view
  const int c2 = tid >> 4, v2 = tid & 15;  // step 2: (c, v)
  const int c3 = tid & 31, p3 = tid >> 5;  // step 3: (c, p' ) with p in {p', p' + 16}
  const float2 wt = __ldg(w16k + t);              // W16384^t
  const float2 wv = __ldg(w16k + 32 * v2);        // W512^v = W16384^{32 v}
  float2 v[32];
  for (int i = 0; i < ntr; ++i) {
    const int64_t tr = blockIdx.x + (int64_t)gridDim.x * i;
    mbar_wait(&full, i & 1);
#pragma unroll
    for (int a = 0; a < 32; ++a) v[(a & 1) * 16 + (a >> 1)] = stage[a * 512 + t];  // even | odd
    // 1. 32-point FFT over a, twiddle W16384^{t c}
    dft32_eo(v);
    {
      float2 w = wt;
#pragma unroll
      for (int c = 1; c < 32; ++c) {
        v[c] = cmul(v[c], w);
        w = cmul(w, wt);
      }
    }
    // 2. exchange 1 through the stage itself, in one round (32 values live per
    //    thread): thread t stores its 32 c at stage[c][t]; thread (c, v) reads
    //    the 32 u (t = 16 u + v); then the stage takes the next transform
    bar_compute();  // every thread has read its inputs
#pragma unroll
    for (int c = 0; c < 32; ++c) stage[c * 512 + t] = v[c];
    bar_compute();
    float2 y[32];
#pragma unroll
    for (int u = 0; u < 32; ++u)  // even | odd split for dft32_eo
      y[(u & 1) * 16 + (u >> 1)] = stage[c2 * 512 + 16 * u + v2];
    bar_compute();
    if (tid == 0 && i + 1 < ntr) load(i + 1);
    dft32_eo(y);  // y[p]
    {
      float2 w = wv;
#pragma unroll
      for (int p = 1; p < 32; ++p) {
        y[p] = cmul(y[p], w);
        w = cmul(w, wv);
      }
    }
    // 3. exchange 2: round r moves p in [16 r, 16 r + 16): every thread (c, v)
    //    stores its 16 p of the round at xb[p - 16 r][v][c ^ v] (conflict-free
    //    both ways); thread (c, p') reads the 16 v of (c, p' + 16 r)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int pp = 0; pp < 16; ++pp) xb[pp * 512 + v2 * 32 + (c2 ^ v2)] = y[16 * r + pp];
      bar_compute();
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) v[16 * r + vv] = xb[p3 * 512 + vv * 32 + (c3 ^ vv)];
      bar_compute();
    }
    // 4. two 16-point FFTs over v; X[c + 32 p + 1024 q]
    float2* dst = out + tr * N + c3;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float2 z[16];
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) z[vv] = v[16 * r + vv];
      dft16c(z);
      const int p = p3 + 16 * r;
#pragma unroll
      for (int q = 0; q < 16; ++q) st_stream(dst + 32 * p + 1024 * q, z[q]);
    }
  }
}

}  // namespace rr16k

static int g_rr_grid = 0;

int fft16384_rr_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  if (batch <= 0) return DPP_OK;
  if (!g_rr_grid) {
    DPP_CUDA_CHECK(cudaFuncSetAttribute(rr16k::fft16384_rr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)rr16k::SMEM));
    int dev = 0, sms = 0;
    DPP_CUDA_CHECK(cudaGetDevice(&dev));
    DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    g_rr_grid = sms;
  }
  // in place is safe: a transform is read into shared memory before any of
  // its outputs is written, and nothing else reads its range
  const float2* w16k = reinterpret_cast<const float2*>(p->l2_tw + 256);
  const unsigned grid = (unsigned)(batch < g_rr_grid ? batch : g_rr_grid);
  rr16k::fft16384_rr<<<grid, rr16k::THREADS, rr16k::SMEM, s>>>(in, out, (int)batch, w16k);
  DPP_LAUNCH_CHECK("fft16384_rr");
  return DPP_OK;
}

}  // namespace dpp
