// FFT node, n = 4096 (C5's row pass, 1-D batches): warp-specialised,
// persistent, one transform per 32 KB stage, no exchange outside the CTA.
//
// n = 16 a + b (a < 256, b < 16), k = k1 + 256 k2:
//   P1: the transform is the [a][b] tile (256 rows x 128 B) — one 2-D TMA
//       box, 128B-swizzled — and the 256-point FFTs over a for the 16 columns
//       b are the L2-ring kernels' warp-local P1 (warp w owns columns 2w,
//       2w+1; fft_l2.cu), then twiddle W_4096^{b k1}.
//   P2: one CTA-wide exchange (named barrier over the 8 compute warps) to
//       [k1][b] rows, position b ^ rotl4(k1 & 15) (conflict-free for both the
//       write and the read), then one 16-point FFT over b per thread
//       (k1 = thread), X[k1 + 256 k2] stored straight from registers: each
//       warp store is 256 contiguous bytes.
// A producer warp keeps the next transform's TMA load in flight (2 stages,
// 2 CTAs per SM: 72 -> 96 registers removed the spills, 0.78 -> 0.71 ms); no scratch, no cross-CTA dependencies: per point 8 B read +
// 8 B written in HBM, 48 B through shared memory.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "l2ring.cuh"
#include "tma.cuh"

namespace dpp {
namespace ws4k {

using namespace ring;

constexpr int N = 4096;
constexpr int CW = 8;
constexpr int THREADS = (CW + 1) * 32;
constexpr int TILE = 4096;
#ifndef DPP_WS4K_S
#define DPP_WS4K_S 2
#endif
#ifndef DPP_WS4K_MINB
#define DPP_WS4K_MINB 2
#endif
constexpr int S = DPP_WS4K_S;

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ int rotl4(int x) { return ((x << 1) | (x >> 3)) & 15; }

// U8: real u8 input (the C5 chain's to_complex node fused in): each stage also
// carries the transform's 4 KB of pixels, widened to (x, 0) in stage A.
//
// PAIR (U8 only): two real images per transform.  Transform t is row r of the
// image pair (2p, 2p+1), z = a + i b; after the FFT the two half spectra are
// separated, A[k] = (Z[k] + conj Z[-k]) / 2, B[k] = (Z[k] - conj Z[-k]) / 2i,
// k = 0 .. N/2 - 1, and stored as one row [A | B] of the pair array with the
// real Nyquist terms packed into the imaginary parts of k = 0:
// A'[0] = (A[0], A[N/2]), B'[0] = (B[0], B[N/2]).  `rows` = rows per image.
template <bool U8, bool PAIR = false>
__global__ void __launch_bounds__(THREADS, DPP_WS4K_MINB)
fft4096_ws(const __grid_constant__ CUtensorMap tin, const uint8_t* __restrict__ inu8, float2* __restrict__ out,
           int batch, const float2* __restrict__ twn, const float4* __restrict__ tw256, int rows = 0) {
  static_assert(U8 || !PAIR, "the pair transform takes u8 images");
  constexpr int PIX = PAIR ? 2 * N : N;  // u8 bytes per stage
  extern __shared__ __align__(1024) float2 smem[];
  const uint8_t* pix = reinterpret_cast<const uint8_t*>(smem + S * TILE);  // U8: S x PIX bytes
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int G = gridDim.x;

  if (warp == CW) {
    if (lane != 0) return;
    const uint64_t stream_pol = policy_evict_first();
    int i = 0;
    for (int t = blockIdx.x; t < batch; t += G, ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&done[s], ((i - S) / S) & 1);
      if constexpr (PAIR) {
        const int pr = t / rows, r = t - pr * rows;
        const uint8_t* a = inu8 + ((size_t)2 * pr * rows + r) * N;
        mbar_arrive_expect_tx(&full[s], 2 * N);
        bulk_g2s(const_cast<uint8_t*>(pix) + s * PIX, a, N, &full[s]);
        bulk_g2s(const_cast<uint8_t*>(pix) + s * PIX + N, a + (size_t)rows * N, N, &full[s]);
      } else if constexpr (U8) {
        mbar_arrive_expect_tx(&full[s], N);
        bulk_g2s(const_cast<uint8_t*>(pix) + s * N, inu8 + (size_t)t * N, N, &full[s]);
      } else {
        mbar_arrive_expect_tx(&full[s], TILE * sizeof(float2));
        tma_load_2d_hint(smem + s * TILE, &tin, 0, t * 256, &full[s], stream_pol);
      }
    }
    return;
  }

  const int col = 2 * warp + (lane & 1);
  const int idx = lane >> 1;
  const int q = idx & 7, p = lane & 1;
  const uint32_t x9 = 16u * (uint32_t)((9 * q) ^ warp);
  const uint32_t offA = 128u * idx + 16u * (uint32_t)(warp ^ q) + 8u * p;
  const uint32_t offW = 2048u * idx + 8u * p + x9;
  const uint32_t offR = 1024u * (idx >> 3) + 8u * p + x9;
  const uint32_t sbase = smem_u32(smem);
  const float4 t1 = __ldg(tw256 + idx);
  const float2 w1 = make_float2(t1.x, t1.y);  // W256^idx
  float2 v[16];
  int i = 0;
  for (int t = blockIdx.x; t < batch; t += G, ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const uint32_t b = sbase + (uint32_t)s * (TILE * 8);
    // P1: 256-point FFTs over a, warp-local (see fft_l2.cu)
    if constexpr (PAIR) {
      const uint8_t* px = pix + s * PIX + idx * 16 + col;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = make_float2((float)px[256 * j], (float)px[N + 256 * j]);
    } else if constexpr (U8) {
      const uint8_t* px = pix + s * N + idx * 16 + col;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = make_float2((float)px[256 * j], 0.f);  // row a = 16 j + idx
    } else {
      const uint32_t bA = b + offA;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = lds64(bA + 2048 * j);
    }
    dft16c(v);
    float2 wk = w1;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      v[k] = cmul(v[k], wk);
      wk = cmul(wk, w1);
    }
    __syncwarp();
    const uint32_t bW = b + offW, bR = b + offR;
#pragma unroll
    for (int k = 0; k < 16; ++k) sts64((bW ^ (144u * (k & 7))) + 1024 * (k >> 3), v[k]);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = lds64((bR ^ (144u * (k & 7))) + 2048 * k);
    dft16c(v);  // v[c1] = Y[b = col][k1 = idx + 16 c1]
    {
      float2 w = __ldg(twn + col * idx);           // W_4096^{b idx}
      const float2 wstep = __ldg(twn + 16 * col);  // W_4096^{16 b}
      v[0] = cmul(v[0], w);
#pragma unroll
      for (int c1 = 1; c1 < 16; ++c1) {
        w = cmul(w, wstep);
        v[c1] = cmul(v[c1], w);
      }
    }
    bar_compute();  // every warp is done reading the tile layout
    // [k1][b]: k1 row of 16, column b ^ rotl4(k1 & 15)
#pragma unroll
    for (int c1 = 0; c1 < 16; ++c1) {
      const int k1 = idx + 16 * c1;
      sts64(b + 8u * (16 * k1 + (col ^ rotl4(idx))), v[c1]);
    }
    bar_compute();
    const int k1 = tid;  // 0..255
#pragma unroll
    for (int bb = 0; bb < 16; ++bb) v[bb] = lds64(b + 8u * (16 * k1 + (bb ^ rotl4(k1 & 15))));
    if constexpr (PAIR) {
      dft16c(v);  // v[k2] = Z[k1 + 256 k2]
      // Z[-k] for k = k1 + 256 k2, k2 < 8: thread (256 - k1) & 255, element
      // 15 - k2 (k1 > 0) or (16 - k2) & 15 (k1 = 0) — always >= 8 except the
      // DC, so the upper halves go through the thread's own [k1] row
#pragma unroll
      for (int k2 = 8; k2 < 16; ++k2) sts64(b + 8u * (16 * k1 + (k2 ^ rotl4(k1 & 15))), v[k2]);
      bar_compute();
      const int pk = (256 - k1) & 255;
      float2* dst = out + (size_t)t * N + k1;
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        const int e = k1 ? 15 - k2 : (16 - k2) & 15;
        const float2 z = v[k2];
        const float2 zm = (k1 | k2) ? lds64(b + 8u * (16 * pk + (e ^ rotl4(pk & 15)))) : z;
        float2 ra = make_float2(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y));
        float2 rb = make_float2(0.5f * (z.y + zm.y), 0.5f * (zm.x - z.x));
        if (k2 == 0 && k1 == 0) {  // DC and Nyquist are real: pack them
          ra = make_float2(z.x, v[8].x);
          rb = make_float2(z.y, v[8].y);
        }
        st_stream(dst + 256 * k2, ra);
        st_stream(dst + N / 2 + 256 * k2, rb);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&done[s]);
    } else {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&done[s]);  // stage free for the next load
      dft16c(v);  // v[k2]
      float2* dst = out + (size_t)t * N + k1;
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) st_stream(dst + 256 * k2, v[k2]);
    }
  }
}

}  // namespace ws4k

static int g_ws4k_ctas = 0, g_ws4k_pair_ctas = 0;

static size_t ws4k_smem(bool u8, bool pair = false) {
  return (size_t)ws4k::S * (ws4k::TILE * sizeof(float2) + (pair ? 2 * ws4k::N : u8 ? ws4k::N : 0));
}

int fft4096_ws_init(FftPlan* p) {
  using namespace ws4k;
  const size_t smem = ws4k_smem(false);
  DPP_CUDA_CHECK(cudaFuncSetAttribute(fft4096_ws<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DPP_CUDA_CHECK(cudaFuncSetAttribute(fft4096_ws<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ws4k_smem(true)));
  DPP_CUDA_CHECK(cudaFuncSetAttribute(fft4096_ws<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ws4k_smem(true, true)));
  if (!g_ws4k_ctas) {
    int per_sm = 0, dev = 0, sms = 0;
    DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft4096_ws<true>, THREADS,
                                                                 ws4k_smem(true)));
    DPP_CUDA_CHECK(cudaGetDevice(&dev));
    DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1) return fail(DPP_ECUDA, "fft4096_ws does not fit on an SM");
    g_ws4k_ctas = per_sm * sms;
    DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft4096_ws<true, true>, THREADS,
                                                                 ws4k_smem(true, true)));
    if (per_sm < 1) return fail(DPP_ECUDA, "fft4096_ws<pair> does not fit on an SM");
    g_ws4k_pair_ctas = per_sm * sms;
  }
  std::vector<float2> twn(N);
  for (int m = 0; m < N; ++m) {
    const double ang = -2.0 * M_PI * (double)m / (double)N;
    twn[(size_t)m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  std::vector<float4> t256(256);
  for (int m = 0; m < 256; ++m) {
    const double ang = -2.0 * M_PI * (double)m / 256.0;
    const float c = (float)std::cos(ang), s = (float)std::sin(ang);
    t256[(size_t)m] = make_float4(c, s, -s, c);
  }
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_tw, 256 * sizeof(float4) + (size_t)N * sizeof(float2)));
  DPP_CUDA_CHECK(cudaMemcpy(p->l2_tw, t256.data(), 256 * sizeof(float4), cudaMemcpyHostToDevice));
  DPP_CUDA_CHECK(cudaMemcpy(reinterpret_cast<float2*>(p->l2_tw + 256), twn.data(), (size_t)N * sizeof(float2),
                            cudaMemcpyHostToDevice));
  return DPP_OK;
}

int fft4096_ws_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  using namespace ws4k;
  if (batch <= 0) return DPP_OK;
  if (batch > 0x7fffffff / 256) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  CUtensorMap tin;
  if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 256, 16, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  const unsigned grid = (unsigned)(batch < g_ws4k_ctas ? batch : g_ws4k_ctas);
  fft4096_ws<false><<<grid, THREADS, ws4k_smem(false), s>>>(
      tin, nullptr, out, (int)batch, reinterpret_cast<const float2*>(p->l2_tw + 256), p->l2_tw);
  DPP_LAUNCH_CHECK("fft4096_ws");
  return DPP_OK;
}

// the same transform of real u8 rows (x -> (x, 0) fused into the load)
int fft4096_ws_execute_u8(const FftPlan* p, const uint8_t* in, float2* out, int64_t batch, cudaStream_t s) {
  using namespace ws4k;
  if (batch <= 0) return DPP_OK;
  if (batch > 0x7fffffff / 256) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  CUtensorMap unused;
  std::memset(&unused, 0, sizeof(unused));
  const unsigned grid = (unsigned)(batch < g_ws4k_ctas ? batch : g_ws4k_ctas);
  fft4096_ws<true><<<grid, THREADS, ws4k_smem(true), s>>>(
      unused, in, out, (int)batch, reinterpret_cast<const float2*>(p->l2_tw + 256), p->l2_tw);
  DPP_LAUNCH_CHECK("fft4096_ws<u8>");
  return DPP_OK;
}

// pairs of real u8 images of `rows` rows: pair array of npairs x rows rows of
// [A | B] half spectra (see PAIR above)
int fft4096_ws_execute_u8_pair(const FftPlan* p, const uint8_t* in, float2* out, int64_t npairs, int rows,
                               cudaStream_t s) {
  using namespace ws4k;
  const int64_t batch = npairs * rows;
  if (batch <= 0) return DPP_OK;
  if (batch > 0x7fffffff / 256) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  CUtensorMap unused;
  std::memset(&unused, 0, sizeof(unused));
  const unsigned grid = (unsigned)(batch < g_ws4k_pair_ctas ? batch : g_ws4k_pair_ctas);
  fft4096_ws<true, true><<<grid, THREADS, ws4k_smem(true, true), s>>>(
      unused, in, out, (int)batch, reinterpret_cast<const float2*>(p->l2_tw + 256), p->l2_tw, rows);
  DPP_LAUNCH_CHECK("fft4096_ws<pair>");
  return DPP_OK;
}

}  // namespace dpp
