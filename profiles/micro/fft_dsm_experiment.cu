// FFT node, n = 2^16 (the C2 headline), exchange through distributed shared
// memory: one 8-CTA cluster owns a transform at a time.
//
// n = 256 a + b, k = c + 256 d, exactly the four-step of csrc/fft_l2.cu (same
// butterflies, same twiddle tables, so the outputs are bit-identical):
//   P1(t, g)  columns b in [16g, 16g+16) of transform t (one 32 KB TMA tile),
//             256-point FFTs over a, twiddle W_N^{bc}; value (b, c) goes
//             straight from registers to the CTA that owns P2 block c >> 4
//             (st.async into its receive buffer, 8 tx bytes on its mbarrier).
//   P2(t, g)  the received 32 KB block c in [16g, 16g+16): 256-point FFTs over
//             b, output rows d by one TMA store.
// CTA r of a cluster runs P1 and P2 for g = 2r, 2r+1 of every transform the
// cluster owns (t = cluster, cluster + clusters, ...).  The exchange never
// touches L2: per point HBM read once, written once (16 B), nothing else
// leaves the SM pair.
//
// Roles per CTA (one CTA per SM): a LOADER warp (P1 tiles into a 3-stage TMA
// ring), a STORER warp (TMA-stores finished P2 blocks, then re-arms the
// receive buffer and tells every CTA of the cluster it is free), and G groups
// of 8 compute warps taking the item sequence P1(i,0) P1(i,1) P2(i-1,0)
// P2(i-1,1) (i = local transform) round robin.  Two receive buffers: the P1
// scatter of transform i+1 overlaps the P2 of transform i.  Every wait is on
// an earlier item of the sequence (of this CTA or of a cluster peer), so the
// schedule cannot deadlock.
#include <cmath>

#include "common.cuh"
#include "fft_plan.cuh"
#include "l2ring.cuh"
#include "tma.cuh"

namespace dpp {
namespace dsm {

using namespace ring;

constexpr int CS = 8;           // CTAs per cluster
constexpr int TPC = 16 / CS;    // P1 (and P2) tiles per CTA per transform
constexpr int NS = 3;           // P1 load stages
constexpr int NB = 2;           // receive buffers
constexpr int TILE = 4096;      // complex64 per 32 KB tile
constexpr size_t SMEM = (size_t)(NS + NB * TPC) * TILE * sizeof(float2);

struct Args {
  const float4* tw256;    // [k][idx] = W256^{k idx} as (w, i w)
  const float2* tw4096;   // W4096^e, e < 256
  const float2* tw65536;  // W65536^e, e < 256
  int batch;
};

__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void arrive_expect_tx_u32(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void init_u32(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

template <int G>
__global__ void __launch_bounds__((8 * G + 2) * 32, 1)
fft65536_dsm(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, const Args a) {
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ __align__(8) uint64_t full[NS], sfree[NS], rfull[NB][TPC], rfree[NB], p2done[NB][TPC];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t r = cluster_ctarank();
  const int q = blockIdx.x / CS, Q = gridDim.x / CS;
  const int nt = q < a.batch ? (a.batch - 1 - q) / Q + 1 : 0;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t rbase = sbase + NS * TILE * 8;  // receive buffers [NB][TPC]
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      init_u32(smem_u32(&full[s]), 1);
      init_u32(smem_u32(&sfree[s]), 8);
    }
    for (int b = 0; b < NB; ++b) {
      init_u32(smem_u32(&rfree[b]), CS);
      for (int j = 0; j < TPC; ++j) {
        init_u32(smem_u32(&rfull[b][j]), 1);
        init_u32(smem_u32(&p2done[b][j]), 8);
      }
    }
    fence_mbar_init();
  }
  cluster_sync();  // every peer's barriers exist before the first remote arrive

  if (warp == 8 * G) {
    // ------------------------------------------------------------ loader
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int p = 0; p < 2 * nt; ++p) {
        const int s = p % NS;
        if (p >= NS) mbar_wait_u32(smem_u32(&sfree[s]), ((p / NS) - 1) & 1);
        const int i = p >> 1, j = p & 1;
        const int t = q + i * Q, g = TPC * (int)r + j;
        mbar_arrive_expect_tx(&full[s], TILE * 8);
        tma_load_2d_hint(smem + s * TILE, &tin, 16 * g, t * 256, &full[s], pol);
      }
    }
  } else if (warp == 8 * G + 1) {
    // ------------------------------------------------------------ storer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      auto release = [&](int b) {  // receive buffer b may take the next transform
        for (int j = 0; j < TPC; ++j) arrive_expect_tx_u32(smem_u32(&rfull[b][j]), TILE * 8);
        const uint32_t bar = smem_u32(&rfree[b]);
        for (int d = 0; d < CS; ++d) mbar_arrive_remote(mapa_u32(bar, (uint32_t)d));
      };
      for (int b = 0; b < NB; ++b)
        if (b < nt) release(b);
      for (int i = 0; i < nt; ++i) {
        const int b = i & 1, t = q + i * Q;
        for (int j = 0; j < TPC; ++j) {
          mbar_wait_u32(smem_u32(&p2done[b][j]), (i >> 1) & 1);
          tma_store_2d_hint(&tout, 16 * (TPC * (int)r + j), t * 256, smem + (NS + b * TPC + j) * TILE, pol);
        }
        bulk_commit();
        bulk_wait_read0();
        if (i + NB < nt) release(b);
      }
      bulk_wait0();
    }
  } else {
    // ------------------------------------------------------------ compute
    const int grp = warp >> 3, w = warp & 7;
    const int col = 2 * w + (lane & 1);
    const int idx = lane >> 1;
    const int qq = idx & 7, pp = lane & 1;
    const uint32_t x9 = 16u * (uint32_t)((9 * qq) ^ w);
    const uint32_t offA = 128u * idx + 16u * (uint32_t)(w ^ qq) + 8u * pp;
    const uint32_t offW = 2048u * idx + 8u * pp + x9;
    const uint32_t offR = 1024u * (idx >> 3) + 8u * pp + x9;
    const float4 t1 = __ldg(a.tw256 + 16 + idx);
    const float2 w1 = make_float2(t1.x, t1.y);  // W256^idx
    float2 v[16];
    for (int k = grp; k < 4 * (nt + 1); k += G) {
      const int i = k >> 2, s4 = k & 3;
      if (s4 < 2) {
        if (i >= nt) continue;
        // ------------------------------------------------------------ P1
        const int j = s4, p = 2 * i + j, s = p % NS;
        mbar_wait(&full[s], (p / NS) & 1);
        const uint32_t b = sbase + (uint32_t)s * (TILE * 8);
        const uint32_t bA = b + offA;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = lds64(bA + 2048 * e);
        dft16c(v);
        float2 wk = w1;
#pragma unroll
        for (int e = 1; e < 16; ++e) {
          v[e] = cmul(v[e], wk);
          wk = cmul(wk, w1);
        }
        __syncwarp();
        const uint32_t bW = b + offW, bR = b + offR;
#pragma unroll
        for (int e = 0; e < 16; ++e) sts64((bW ^ (144u * (e & 7))) + 1024 * (e >> 3), v[e]);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = lds64((bR ^ (144u * (e & 7))) + 2048 * e);
        __syncwarp();
        if (lane == 0) mbar_arrive1(&sfree[s]);  // the stage is in registers
        dft16c(v);
        {
          // W_N^{b c}, b = 16 g + col, c = idx + 16 c1 (tables in L1: the 72-register
          // budget of 26 warps has no room to keep them per tile)
          const int g = TPC * (int)r + j;
          float2 tw = cmul(__ldg(a.tw4096 + g * idx), __ldg(a.tw65536 + col * idx));
          const float2 st = __ldg(a.tw4096 + 16 * g + col);
          v[0] = cmul(v[0], tw);
#pragma unroll
          for (int c1 = 1; c1 < 16; ++c1) {
            tw = cmul(tw, st);
            v[c1] = cmul(v[c1], tw);
          }
        }
        // value (b, c = idx + 16 c1) -> CTA c1 / TPC, block c1 % TPC, row b, column idx
        const int bsel = i & 1;
        mbar_wait_cluster(smem_u32(&rfree[bsel]), (i >> 1) & 1);
        const int bb = 16 * (TPC * (int)r + j) + col;
        const uint32_t la = rbase + (uint32_t)(bsel * TPC * TILE * 8) + 8u * (uint32_t)swz(bb, idx);
        const uint32_t lbar = smem_u32(&rfull[bsel][0]);
#pragma unroll
        for (int d = 0; d < CS; ++d) {
          // a peer's window is contiguous: one mapa per peer, offsets added
          const uint32_t ra = mapa_u32(la, (uint32_t)d), rb = mapa_u32(lbar, (uint32_t)d);
#pragma unroll
          for (int jj = 0; jj < TPC; ++jj) st_async_f2(ra + jj * TILE * 8, v[TPC * d + jj], rb + 8 * jj);
        }
      } else {
        if (i == 0) continue;
        // ------------------------------------------------------------ P2
        const int ii = i - 1, j = s4 - 2, bsel = ii & 1;
        mbar_wait_cluster(smem_u32(&rfull[bsel][j]), (ii >> 1) & 1);
        const uint32_t b = rbase + (uint32_t)((bsel * TPC + j) * TILE * 8);
        const uint32_t bA = b + offA;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = lds64(bA + 2048 * e);
        dft16c(v);
        float2 wk = w1;
#pragma unroll
        for (int e = 1; e < 16; ++e) {
          v[e] = cmul(v[e], wk);
          wk = cmul(wk, w1);
        }
        __syncwarp();
        const uint32_t bW = b + offW, bR = b + offR;
#pragma unroll
        for (int e = 0; e < 16; ++e) sts64((bW ^ (144u * (e & 7))) + 1024 * (e >> 3), v[e]);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = lds64((bR ^ (144u * (e & 7))) + 2048 * e);
        dft16c(v);
        __syncwarp();
#pragma unroll
        for (int d1 = 0; d1 < 16; ++d1) sts64(bA + 2048 * d1, v[d1]);  // output row d = idx + 16 d1
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive1(&p2done[bsel][j]);
      }
    }
  }
  __syncwarp();
  // no CTA leaves while a peer may still write its buffers or arrive on its barriers
  cluster_sync();
}

}  // namespace dsm

static int g_dsm_grid = 0, g_dsm_groups = 3;

template <int G>
static int dsm_prepare(int* grid) {
  auto k = dsm::fft65536_dsm<G>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm::SMEM));
  DPP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = dsm::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(dsm::CS * 64);
  cfg.blockDim = dim3((8 * G + 2) * 32);
  cfg.dynamicSmemBytes = dsm::SMEM;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  DPP_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&clusters, k, &cfg));
  if (clusters < 1) return fail(DPP_ECUDA, "no 8-CTA cluster of the 2^16 DSMEM kernel fits");
  *grid = clusters * dsm::CS;
  return DPP_OK;
}

// A/B hook for the C2 kernel choice (fft_l2.cu calls this when DPP_FFT_DSM is set)
int fft65536_dsm_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  if (batch <= 0) return DPP_OK;
  if (!g_dsm_grid) {
    const char* e = getenv("DPP_FFT_DSM");
    g_dsm_groups = e && e[0] == '2' ? 2 : 3;
    if (int rc = g_dsm_groups == 2 ? dsm_prepare<2>(&g_dsm_grid) : dsm_prepare<3>(&g_dsm_grid)) return rc;
  }
  CUtensorMap tin, tout;
  if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  if (int rc = make_tmap_c64(&tout, out, (uint64_t)batch * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  dsm::Args a;
  a.tw256 = p->l2_tw;
  a.tw4096 = reinterpret_cast<const float2*>(p->l2_tw + 256);
  a.tw65536 = reinterpret_cast<const float2*>(p->l2_tw + 256 + 128);
  a.batch = (int)batch;
  const int clusters = (int)((batch < g_dsm_grid / dsm::CS) ? batch : g_dsm_grid / dsm::CS);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = dsm::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(clusters * dsm::CS));
  cfg.blockDim = dim3((8 * g_dsm_groups + 2) * 32);
  cfg.dynamicSmemBytes = dsm::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g_dsm_groups == 2)
    DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, dsm::fft65536_dsm<2>, tin, tout, a));
  else
    DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, dsm::fft65536_dsm<3>, tin, tout, a));
  return DPP_OK;
}

}  // namespace dpp
