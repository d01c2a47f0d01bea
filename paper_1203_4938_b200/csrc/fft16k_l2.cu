// 1-D FFT node, n = 256 B for B = 32, 64, 128 (n = 8192, 16384 — also the row
// pass of 16384 x C 2-D transforms — and 32768): two-pass four-step through
// the L2 exchange ring, n = B a + b (a < 256, b < B), k = k1 + 256 k2.
// (Written out below for B = 64; in general a unit is TPU = 256 / B
// transforms and a P2 sequence spans L = B / 16 lanes.)
//
//   P1(u, g): transform 4u + g/4, columns b in [16 (g%4), +16) of its
//             [a][b] view (256 rows x 128 B, one 2-D TMA box): 256-point
//             FFTs over a (the 1-D 2^16 kernel's P1), twiddle W_n^{b k1},
//             written to ring slot u as S[k1 / 16][4 b + g/4][k1 % 16].
//   P2(u, kg): the 32 KB block S[kg] (4 transforms x 64 b x 16 k1): 64-point
//             FFTs over b, four lanes per (transform, k1) sequence (the 2-D
//             column kernel's B = 64 P1 pattern), output tile
//             [k2][transform][k1 % 16] = rows 4 k2 + g/4, which is exactly
//             this warp's own rows, by one 3-D TMA store (16 x 4 x 64).
// A unit is 4 consecutive transforms, so both passes have 16 items of 32 KB
// per unit and the schedule/ring are the 2^16 kernel's (fft_l2.cu).
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "l2ring.cuh"
#include "tma.cuh"

namespace dpp {
namespace ring16k {

using namespace ring;

constexpr int CW = 8;
constexpr int THREADS = (CW + 1) * 32;
constexpr int TILE = 4096;
constexpr int S = 2;
constexpr int ITEMS = 16;

struct Args {
  float2* scratch;
  int* ctrl;
  const float2* twn;    // W_n^m, m < n
  const float4* tw256;  // W256^m as (w, i*w)
  int units, lag, ring;
};

// exchange slot of (b0, m0) in a sequence's B rows: beta = g(m0) ^ b0 with
// g(m0) = L m0 | ((m0 / Q) & (L/2 - 1)), Q = 16 / L: writes (fixed m0) and reads
// (fixed b0) both give a half-warp distinct row parities x its columns
template <int L>
__device__ __forceinline__ int gbeta(int m0) {
  constexpr int Q = 16 / L;
  return L * m0 | ((m0 / Q) & (L / 2 - 1));
}

template <int L>
__device__ __forceinline__ void dftL(float2* v) {
  if constexpr (L == 2) {
    dft2(v[0], v[1]);
  } else if constexpr (L == 4) {
    dft4c(v[0], v[1], v[2], v[3]);
  } else {
    float2 t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = v[q];
    dft8(t);
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = t[q];
  }
}

template <int B>
__global__ void __launch_bounds__(THREADS, 3)
fft16k_l2w(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, const Args a) {
  constexpr int N = 256 * B, TPU = 256 / B, L = B / 16, Q = 16 / L, LOGL = L == 2 ? 1 : (L == 4 ? 2 : 3);
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  __shared__ int s_tick[S];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int total = 2 * ITEMS * a.units;
  int* cnt1 = a.ctrl + 32;
  int* cnt2 = cnt1 + a.units;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    const uint64_t stream_pol = policy_evict_first();
    int head = 0, i = 0;
    auto publish = [&](int k) {
      const int s = k % S;
      int pass, u;
      decode(s_tick[s] >> 4, a.units, a.lag, pass, u);
      if (pass == 1) {
        red_release_add(cnt1 + u, 1);
      } else {
        if (u + a.ring < a.units) red_release_add(cnt2 + u, 1);
        tma_store_3d(&tout, 16 * (s_tick[s] & 15), TPU * u, 0, smem + s * TILE);
        bulk_commit();
      }
    };
    for (;; ++i) {
      const int s = i % S;
      while (head <= i - S) {
        mbar_wait(&done[head % S], (head / S) & 1);
        publish(head);
        ++head;
      }
      const int tick = atomicAdd(a.ctrl, 1);
      if (tick >= total) {
        s_tick[s] = -1;
        mbar_arrive1(&full[s]);
        break;
      }
      int pass, u;
      decode(tick >> 4, a.units, a.lag, pass, u);
      const int g = tick & 15;
      const int* dep = pass == 2 ? cnt1 + u : (u >= a.ring ? cnt2 + (u - a.ring) : nullptr);
      if (dep) {
        while (ld_acquire(dep) < ITEMS) {
          if (head < i && mbar_try(&done[head % S], (head / S) & 1)) {
            publish(head);
            ++head;
          } else {
            __nanosleep(32);
          }
        }
      }
      bulk_wait_read0();
      s_tick[s] = tick;
      float2* buf = smem + s * TILE;
      mbar_arrive_expect_tx(&full[s], TILE * sizeof(float2));
      if (pass == 1) {
        tma_load_2d(buf, &tin, 16 * (g & (L - 1)), (TPU * u + (g >> LOGL)) * 256, &full[s]);
      } else {
        fence_proxy_async_global();
        bulk_g2s(buf, a.scratch + (size_t)(u & (a.ring - 1)) * (TPU * N) + 4096 * g, TILE * sizeof(float2), &full[s]);
      }
    }
    while (head < i) {
      mbar_wait(&done[head % S], (head / S) & 1);
      publish(head);
      ++head;
    }
    bulk_wait0();
    return;
  }

  // -------------------------------------------------------------- compute
  const uint32_t sbase = smem_u32(smem);
  float2 v[16];
  for (int i = 0;; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const int tick = s_tick[s];
    if (tick < 0) break;
    int pass, u;
    decode(tick >> 4, a.units, a.lag, pass, u);
    const int g = tick & 15;
    const uint32_t b = sbase + (uint32_t)s * (TILE * 8);
    float2* slot = a.scratch + (size_t)(u & (a.ring - 1)) * (TPU * N);
    if (pass == 1) {
      // P1 mapping (as fft_l2.cu): column col = 2w + (lane & 1), row part idx = lane >> 1
      const int col = 2 * warp + (lane & 1);
      const int idx = lane >> 1;
      const int q = idx & 7, p = lane & 1;
      const uint32_t x9 = 16u * (uint32_t)((9 * q) ^ warp);
      const uint32_t offA = 128u * idx + 16u * (uint32_t)(warp ^ q) + 8u * p;
      const uint32_t offW = 2048u * idx + 8u * p + x9;
      const uint32_t offR = 1024u * (idx >> 3) + 8u * p + x9;
      const float4 t1 = __ldg(a.tw256 + idx);
      const float2 w1 = make_float2(t1.x, t1.y);  // W256^idx
      const uint32_t bA = b + offA;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = lds64(bA + 2048 * j);
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
      dft16c(v);  // v[c1] = Y[b][k1 = idx + 16 c1], b = 16 (g % L) + col
      const int bb = 16 * (g & (L - 1)) + col;
      float2 w = __ldg(a.twn + bb * idx);
      const float2 step = __ldg(a.twn + 16 * bb);
      v[0] = cmul(v[0], w);
#pragma unroll
      for (int c1 = 1; c1 < 16; ++c1) {
        w = cmul(w, step);
        v[c1] = cmul(v[c1], w);
      }
      float2* dst = slot + swz(TPU * bb + (g >> LOGL), idx);
      const uint64_t keep_pol = policy_evict_last();
#pragma unroll
      for (int c1 = 0; c1 < 16; ++c1) st_l2_hint(dst + 4096 * c1, v[c1], keep_pol);
    } else {
      // P2 mapping: a sequence (transform trl, k1 % 16 = kcol) spans L lanes
      // (b0 = lane / (32 / L)); 32 / L sequences per warp, 8 warps cover
      // TPU transforms x 16 k1 values.  Rows of the block: TPU b + trl.
      constexpr int SPW = 32 / L;
      const int trl = warp / (L / 2 > 0 ? (L / 2) : 1);
      const int kcol = SPW * (warp % (L / 2 > 0 ? (L / 2) : 1)) + (lane & (SPW - 1));
      const int b0 = lane / SPW;
      const float2 wB = __ldg(a.twn + 256 * b0);  // W_B^b0
      discard_l2(slot + 4096 * g + 16 * (tid & 255));
#pragma unroll
      for (int b1 = 0; b1 < 16; ++b1) v[b1] = lds64(b + 8u * swz(16 * b1 + TPU * b0 + trl, kcol));
      dft16c(v);  // v[m0]
      float2 w = wB;
#pragma unroll
      for (int m0 = 1; m0 < 16; ++m0) {
        v[m0] = cmul(v[m0], w);
        w = cmul(w, wB);
      }
      __syncwarp();
#pragma unroll
      for (int m0 = 0; m0 < 16; ++m0) sts64(b + 8u * swz(TPU * (gbeta<L>(m0) ^ b0) + trl, kcol), v[m0]);
      __syncwarp();
      const int j = b0;  // now owns m0 = Q j + ii
#pragma unroll
      for (int ii = 0; ii < Q; ++ii)
#pragma unroll
        for (int c = 0; c < L; ++c) v[L * ii + c] = lds64(b + 8u * swz(TPU * (gbeta<L>(Q * j + ii) ^ c) + trl, kcol));
#pragma unroll
      for (int ii = 0; ii < Q; ++ii) dftL<L>(v + L * ii);  // v[L ii + m1]
      __syncwarp();
      // X[k1 + 256 k2], k2 = Q j + ii + 16 m1, staged at row TPU k2 + trl, column kcol
#pragma unroll
      for (int ii = 0; ii < Q; ++ii)
#pragma unroll
        for (int m1 = 0; m1 < L; ++m1)
          sts64(b + 8u * swz(TPU * (Q * j + ii + 16 * m1) + trl, kcol), v[L * ii + m1]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive1(&done[s]);
  }
}

}  // namespace ring16k

template <int B>
static int ringb_prepare(int* ctas) {
  using namespace ring16k;
  const size_t smem = (size_t)S * TILE * sizeof(float2);
  DPP_CUDA_CHECK(cudaFuncSetAttribute(fft16k_l2w<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0, dev = 0, sms = 0;
  DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft16k_l2w<B>, THREADS, smem));
  DPP_CUDA_CHECK(cudaGetDevice(&dev));
  DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(DPP_ECUDA, "fft16k_l2w does not fit on an SM");
  *ctas = per_sm * sms;
  return DPP_OK;
}

static int g_ringb_ctas[3] = {0, 0, 0};

// n = 8192, 16384, 32768 (B = n / 256 = 32, 64, 128)
int fft16k_l2_init(FftPlan* p) {
  using namespace ring16k;
  const int64_t N = p->n0;
  const int B = (int)(N / 256), TPU = 256 / B;
  const int slot = B == 32 ? 0 : (B == 64 ? 1 : 2);
  if (!g_ringb_ctas[slot]) {
    int rc = B == 32 ? ringb_prepare<32>(&g_ringb_ctas[slot])
                     : (B == 64 ? ringb_prepare<64>(&g_ringb_ctas[slot]) : ringb_prepare<128>(&g_ringb_ctas[slot]));
    if (rc) return rc;
  }
  p->l2_lag = ring_stress() ? 2 : 48;
  p->l2_ring = ring_stress() ? 4 : 128;
  if (p->l2_ring <= p->l2_lag) p->l2_ring = p->l2_lag + 1;
  int r = 1;
  while (r < p->l2_ring) r <<= 1;
  p->l2_ring = r;
  std::vector<float2> twn((size_t)N);
  for (int64_t m = 0; m < N; ++m) {
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
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_scratch, (size_t)p->l2_ring * TPU * N * sizeof(float2)));
  const int64_t units = (p->batch + TPU - 1) / TPU;
  p->l2_ctrl_bytes = (32 + 2 * (size_t)(units > 0 ? units : 1)) * sizeof(int);
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_ctrl, p->l2_ctrl_bytes));
  DPP_CUDA_CHECK(cudaEventCreateWithFlags(&p->l2_done, cudaEventDisableTiming));
  return DPP_OK;
}

template <int B>
static int ringb_launch(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s, int ctas) {
  using namespace ring16k;
  constexpr int N = 256 * B, TPU = 256 / B;
  const int64_t units = batch / TPU;
  if (units == 0) return DPP_OK;
  if (units > 0x7fffffff / (2 * ITEMS)) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  CUtensorMap tin, tout;
  if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 256, B, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  {
    // output view (k1: 256 contiguous, transform: stride n, k2: stride 256), box 16 x TPU x B
    const uint64_t dims[3] = {256, (uint64_t)batch, (uint64_t)B};
    const uint64_t strides[2] = {(uint64_t)N * 8, 256 * 8};
    const uint32_t box[3] = {16, (uint32_t)TPU, (uint32_t)B};
    if (int rc = make_tmap_c64_3d(&tout, out, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  }
  Args a;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw;
  a.twn = reinterpret_cast<const float2*>(p->l2_tw + 256);
  a.units = (int)units;
  a.lag = (int)(units < p->l2_lag ? units : p->l2_lag);
  a.ring = p->l2_ring;
  DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
  DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)units) * sizeof(int), s));
  const int64_t items = 2 * ITEMS * units;
  const unsigned grid = (unsigned)(items < ctas ? items : ctas);
  fft16k_l2w<B><<<grid, THREADS, (size_t)S * TILE * sizeof(float2), s>>>(tin, tout, a);
  DPP_LAUNCH_CHECK("fft16k_l2w");
  DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
  return DPP_OK;
}

// batch: whole units of 256 / B transforms (the caller runs any remainder elsewhere)
int fft16k_l2_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  switch (p->n0) {
    case 8192: return ringb_launch<32>(p, in, out, batch, s, g_ringb_ctas[0]);
    case 16384: return ringb_launch<64>(p, in, out, batch, s, g_ringb_ctas[1]);
    case 32768: return ringb_launch<128>(p, in, out, batch, s, g_ringb_ctas[2]);
  }
  return fail(DPP_EINVAL, "no L2-ring kernel for n = %lld", (long long)p->n0);
}

}  // namespace dpp
