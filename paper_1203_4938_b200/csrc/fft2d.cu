// 2-D FFT: row pass (the 1-D kernels of fft.cu) + one column pass.
//
// The reference has no 2-D transform; its 2-D result is defined (SURVEY §8d,
// C3) as the composition fft(rows) then fft(columns) of apps/fft.py:150-174.
//
// Column pass (fft_columns_tma<L1, L2, C, W>): a cluster of C CTAs owns a tile
// of W adjacent columns over all L = L1*L2 rows, rows r = L2*a + b.
//   - CTA p loads rows {L2*a + b : b in its slice of B1 = L2/C} with ONE 3-D
//     TMA box (W x B1 x L1) into [a][b][col] order;
//   - pass A: L1-point FFTs over a for its B1*W (b, col) sequences,
//     exchanges in conflict-free [element][sequence] rows;
//   - W_L^{b c} by per-thread recurrence, st.async scatter of every element
//     to the owner of c (B2 = L1/C values of c per CTA), each store signalling
//     the owner's receive mbarrier; XOR-swizzled receive rows;
//   - pass B: L2-point FFTs over b, results staged in [d][c][col] order and
//     written with ONE 3-D TMA store (rows c + L1*d).
// One HBM read + one HBM write per element, in place.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "fft_block.cuh"
#include "tma.cuh"

namespace dpp {

template <int L1, int L2, int C, int W>
struct ColCfg {
  static constexpr int R = L1 < 16 ? L1 : 16;
  static_assert(L1 % R == 0 && L2 % R == 0, "radix must divide both factors");
  static constexpr int L = L1 * L2;
  static constexpr int B1 = L2 / C, B2 = L1 / C;  // b per CTA (pass A), c per CTA (pass B)
  static constexpr int F1 = B1 * W, F2 = B2 * W;  // sequences per CTA
  static constexpr int T1 = L1 / R, T2 = L2 / R;
  static constexpr int THREADS = F1 * T1;
  static_assert(THREADS == F2 * T2, "pass thread counts must agree");
  static constexpr int G = 32 / W > 1 ? 32 / W : 1;  // receive swizzle period
  static constexpr int NC = L1 > L2 ? L1 : L2;
  static constexpr int S = L / NC;
  static constexpr int LOGS = ilog2(S);
  static constexpr int TILE = L1 * F1;
  static_assert(TILE == L2 * F2, "tile sizes must agree");
  static constexpr size_t SMEM = (size_t)(2 * NC + TILE) * sizeof(float2);
};

struct MapRow2 {
  int w, col;
  __device__ __forceinline__ int operator()(int e) const { return e * w + col; }
};

template <int L1, int L2, int C, int W>
__global__ void __launch_bounds__(ColCfg<L1, L2, C, W>::THREADS, 1024 / ColCfg<L1, L2, C, W>::THREADS)
fft_columns_tma(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                int64_t tiles_per_image, const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ColCfg<L1, L2, C, W>;
  constexpr int R = Cfg::R, B1 = Cfg::B1, B2 = Cfg::B2, F1 = Cfg::F1, F2 = Cfg::F2, T1 = Cfg::T1, T2 = Cfg::T2;
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  float4* coarse = reinterpret_cast<float4*>(smem);  // (w, i*w)
  float2* buf = smem + 2 * Cfg::NC;

  const int p = (int)cluster_ctarank();
  const int64_t tile = blockIdx.x / C;
  const int64_t img = tile / tiles_per_image;
  const int c0 = (int)((tile - img * tiles_per_image) * W);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[0], (uint32_t)(Cfg::TILE * sizeof(float2)));
    mbar_arrive_expect_tx(&bars[1], (uint32_t)(Cfg::TILE * sizeof(float2)));
    tma_load_3d(buf, &tin, c0, p * B1, (int)(img * L1), &bars[0]);
  }
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) {
    const float2 w = coarse_g[e];
    coarse[e] = make_float4(w.x, w.y, -w.y, w.x);
  }
  __syncthreads();

  // pass A: sequence f = (bl, col), FFT over a
  const int f = tid % F1, j = tid / F1;
  const int bl = f / W, col = f - bl * W;
  const int b = p * B1 + bl;
  // four-step twiddle bases fetched before the tile wait (latency hidden)
  const float2 tw0a = __ldg(coarse_g + ((b * j) >> Cfg::LOGS)), tw0b = __ldg(fine_g + ((b * j) & (Cfg::S - 1)));
  const float2 tw1a = __ldg(coarse_g + ((b * T1) >> Cfg::LOGS)), tw1b = __ldg(fine_g + ((b * T1) & (Cfg::S - 1)));
  float2 v[R];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = buf[(j + T1 * i) * F1 + f];
  __syncthreads();
  block_fft<L1, R>(v, j, buf, MapRow2{F1, f}, coarse, Cfg::NC / L1);
  cluster_arrive_relaxed();  // this CTA no longer reads buf
  {
    float2 w = cmul(tw0a, tw0b);
    const float2 sw = cmul(tw1a, tw1b);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v[i] = cmul(v[i], w);
      w = cmul(w, sw);
    }
  }
  cluster_wait();
  {
    const uint32_t base = smem_u32(buf);
    const uint32_t rbar = smem_u32(&bars[1]);
    const int swz = (b % Cfg::G) * W;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = j + T1 * i;
      const int q = c / B2, cl = c - q * B2;
      const uint32_t off = (uint32_t)((b * F2 + ((cl * W + col) ^ swz)) * sizeof(float2));
      st_async_f2(mapa_u32(base + off, q), v[i], mapa_u32(rbar, q));
    }
  }
  mbar_wait(&bars[1], 0);

  // pass B: sequence f2 = (cl, col), FFT over b
  const int f2 = tid % F2, j2 = tid / F2;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int bb = j2 + T2 * i;
    v[i] = buf[bb * F2 + (f2 ^ ((bb % Cfg::G) * W))];
  }
  __syncthreads();
  block_fft<L2, R>(v, j2, buf, MapRow2{F2, f2}, coarse, Cfg::NC / L2);  // ends with a CTA barrier
#pragma unroll
  for (int i = 0; i < R; ++i) buf[(j2 + T2 * i) * F2 + f2] = v[i];  // [d][cl][col] = TMA box order
  fence_proxy_async_smem();
  __syncthreads();
  if (tid == 0) {
    tma_store_3d(&tout, c0, p * B2, (int)(img * L2), buf);
    bulk_commit_and_wait_all();
  }
}

template <int L1, int L2, int C, int W>
static int prepare_columns() {
  auto kern = fft_columns_tma<L1, L2, C, W>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ColCfg<L1, L2, C, W>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int L1, int L2, int C, int W>
static int launch_columns(float2* data, int64_t ncols, int64_t batch, const float2* coarse, const float2* fine,
                          cudaStream_t s) {
  using Cfg = ColCfg<L1, L2, C, W>;
  CUtensorMap tin, tout;
  {
    const uint64_t dims[3] = {(uint64_t)ncols, (uint64_t)L2, (uint64_t)(batch * L1)};
    const uint64_t strides[2] = {(uint64_t)ncols * 8, (uint64_t)ncols * 8 * L2};
    const uint32_t box[3] = {(uint32_t)W, (uint32_t)Cfg::B1, (uint32_t)L1};
    if (int rc = make_tmap_c64_3d(&tin, data, dims, strides, box)) return rc;
  }
  {
    const uint64_t dims[3] = {(uint64_t)ncols, (uint64_t)L1, (uint64_t)(batch * L2)};
    const uint64_t strides[2] = {(uint64_t)ncols * 8, (uint64_t)ncols * 8 * L1};
    const uint32_t box[3] = {(uint32_t)W, (uint32_t)Cfg::B2, (uint32_t)L2};
    if (int rc = make_tmap_c64_3d(&tout, data, dims, strides, box)) return rc;
  }
  const int64_t tiles = ncols / W;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * tiles * C), 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_columns_tma<L1, L2, C, W>, tin, tout, tiles, coarse, fine));
  return DPP_OK;
}

// Column schedules (L, L1, L2, C, W): 4096-8192 points per CTA, 256-512 threads.
#define DPP_COLUMN_TABLE(X)   \
  X(256, 16, 16, 1, 16)       \
  X(512, 16, 32, 2, 16)       \
  X(1024, 32, 32, 4, 16)      \
  X(2048, 32, 64, 8, 16)      \
  X(4096, 64, 64, 16, 16)     \
  X(8192, 64, 128, 16, 8)     \
  X(16384, 128, 128, 16, 8)

std::vector<float2> twiddle_table(int64_t n, int64_t count);
int upload_table(const std::vector<float2>& h, float2** d);

// the shape rules of fft2d_plan_init / fft2d_colring_init, without the device
bool fft2d_shape_supported(int64_t n0, int64_t n1) {
  if (n0 < 2 || (n0 & (n0 - 1)) || n1 < 2 || (n1 & (n1 - 1)) || n1 > (1LL << 30)) return false;
  int width = 0;
  switch (n0) {
#define WIDTH(L, A, B, C, W) \
  case L: width = W; break;
    DPP_COLUMN_TABLE(WIDTH)
#undef WIDTH
    case 32768: width = 16; break;
  }
  return width && n1 % width == 0;
}

int fft2d_plan_init(FftPlan* p) {
  const int64_t n0 = p->n0, n1 = p->n1;
  if (n0 < 2 || (n0 & (n0 - 1)) || n1 < 2 || (n1 & (n1 - 1)))
    return fail(DPP_EINVAL, "2-D sizes must be powers of two, got %lld x %lld", (long long)n0, (long long)n1);
  int width = 0, rc = DPP_ENOTSUP;
  int64_t l1 = 0;
  int cl = 1;
  const bool ring_only = n0 == 32768;  // no cluster column kernel: the column ring only
  switch (n0) {
#define PREP(L, A, B, C, W) \
  case L: width = W; l1 = A; cl = C; rc = prepare_columns<A, B, C, W>(); break;
    DPP_COLUMN_TABLE(PREP)
#undef PREP
  }
  if (ring_only) {
    width = 16;
    l1 = 128;
    rc = DPP_OK;
  }
  if (rc == DPP_ENOTSUP)
    return fail(DPP_ENOTSUP, "2-D column length %lld not supported (256..32768)", (long long)n0);
  if (rc) return rc;
  if (n1 % width)
    return fail(DPP_ENOTSUP, "2-D row length %lld must be a multiple of the %d-column tile", (long long)n1, width);
  p->col_width = width;
  p->col_split = l1;
  p->col_cluster = cl;
  const int64_t l2 = n0 / l1;
  const int64_t nc = l1 > l2 ? l1 : l2;
  if (upload_table(twiddle_table(nc, nc), &p->ctw_a)) return DPP_ECUDA;
  if (upload_table(twiddle_table(n0, n0 / nc), &p->ctw_b)) return DPP_ECUDA;
  p->rows = new FftPlan();
  p->rows->rank = 1;
  p->rows->n0 = n1;
  p->rows->batch = p->batch * n0;
  p->rows->device = p->device;
  rc = fft1d_plan_init(p->rows);
  if (rc) return rc;
  rc = fft2d_colring_init(p);
  if (rc != DPP_OK && rc != DPP_ENOTSUP) return rc;
  if (ring_only && !p->col_ring)
    return fail(DPP_ENOTSUP, "2-D column length 32768 needs the column ring (row length a multiple of 16)");
  char rows[200];
  snprintf(rows, sizeof(rows), "%s", p->rows->desc);
  if (p->col_ring)
    snprintf(p->desc, sizeof(p->desc), "rows: %s | columns: L2-ring four-step 256x%lld (ring %d, lag %d)", rows,
             (long long)(n0 / 256), p->l2_ring, p->l2_lag);
  else
    snprintf(p->desc, sizeof(p->desc), "rows: %s | columns: TMA cluster<%lldx%lld, C=%d, W=%d>", rows,
             (long long)l1, (long long)l2, cl, width);
  return DPP_OK;
}

int fft2d_columns_execute(const FftPlan* p, float2* data, int64_t batch, cudaStream_t s) {
  if (batch == 0) return DPP_OK;
  if (p->col_ring) return fft2d_colring_execute(p, data, batch, s);
  switch (p->n0) {
#define RUN(L, A, B, C, W) \
  case L: return launch_columns<A, B, C, W>(data, p->n1, batch, p->ctw_a, p->ctw_b, s);
    DPP_COLUMN_TABLE(RUN)
#undef RUN
  }
  return fail(DPP_EINVAL, "no column kernel for %lld", (long long)p->n0);
}

int fft2d_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  if (batch == 0) return DPP_OK;
  int rc = fft1d_execute(p->rows, in, out, batch * p->n0, s);
  if (rc) return rc;
  return fft2d_columns_execute(p, out, batch, s);
}

}  // namespace dpp
