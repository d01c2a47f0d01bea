// 2-D FFT: row pass (1-D kernels of fft.cu) + one column pass.
//
// The reference has no 2-D transform; its 2-D result is defined (SURVEY §8d,
// C3) as the composition fft(rows) then fft(columns) of apps/fft.py:150-174.
//
// Column pass kernel (fft_columns_kernel<L1, L2, C, W>): a thread-block
// cluster of C CTAs owns a tile of W adjacent columns over all L = L1*L2
// rows.  Rows r = L2*a + b: pass A runs L1-point FFTs over a for the CTA's
// slice of b (every load is a W-wide contiguous row segment), multiplies by
// W_L^{b c}, scatters through DSMEM, pass B runs L2-point FFTs over b and
// stores rows c + L1*d.  One HBM read and one HBM write per element, in place.
#include <cooperative_groups.h>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "fft_block.cuh"

namespace cg = cooperative_groups;

namespace dpp {

template <int L1, int L2, int C, int W>
struct ColCfg {
  static constexpr int R = L1 < 16 ? L1 : 16;
  static_assert(L2 % R == 0, "L2 must be a multiple of the radix");
  static constexpr int L = L1 * L2;
  static constexpr int B1 = L2 / C, B2 = L1 / C;  // b-slice in pass A, c-slice in pass B
  static constexpr int T1 = L1 / R, T2 = L2 / R;
  static constexpr int THREADS = B1 * W * T1;
  static_assert(THREADS == B2 * W * T2, "pass thread counts must agree");
  static constexpr int NC = L1 > L2 ? L1 : L2;
  static constexpr int S = L / NC;
  static constexpr int LOGS = ilog2(S);
  static constexpr int BUF1 = B1 * W * (L1 + 1), BUF2 = B2 * W * (L2 + 1);
  static constexpr int BUF = BUF1 > BUF2 ? BUF1 : BUF2;
  static constexpr size_t SMEM = (size_t)(NC + S + BUF) * sizeof(float2);
};

template <int L1, int L2, int C, int W>
__global__ void __launch_bounds__(ColCfg<L1, L2, C, W>::THREADS)
fft_columns_kernel(float2* __restrict__ data, int64_t ncols, int64_t image_elems,
                   const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ColCfg<L1, L2, C, W>;
  constexpr int R = Cfg::R, B1 = Cfg::B1, B2 = Cfg::B2, T1 = Cfg::T1, T2 = Cfg::T2;
  extern __shared__ float2 smem[];
  float2* coarse = smem;
  float2* fine = smem + Cfg::NC;
  float2* buf = fine + Cfg::S;

  cg::cluster_group cluster = cg::this_cluster();
  const int p = (int)cluster.block_rank();
  const int64_t tile = blockIdx.x / C;               // over images x column tiles
  const int64_t tiles_per_image = ncols / W;
  const int64_t img = tile / tiles_per_image;
  const int64_t c0 = (tile - img * tiles_per_image) * W;
  float2* base = data + img * image_elems + c0;
  const int tid = threadIdx.x;

  // pass A: thread = ((j * B1) + bl) * W + col
  const int col = tid % W;
  const int bl = (tid / W) % B1;
  const int j = tid / (W * B1);
  const int b = p * B1 + bl;
  float2 v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = __ldcs(base + (int64_t)(L2 * (j + T1 * i) + b) * ncols + col);
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) coarse[e] = coarse_g[e];
  for (int e = tid; e < Cfg::S; e += Cfg::THREADS) fine[e] = fine_g[e];
  __syncthreads();
  block_fft<L1, R>(v, j, buf + (bl * W + col) * (L1 + 1), MapIdentity{}, coarse, Cfg::NC / L1);
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int e = b * (j + T1 * i);
    v[i] = cmul(v[i], cmul(coarse[e >> Cfg::LOGS], fine[e & (Cfg::S - 1)]));
  }
  cluster.sync();
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int c = j + T1 * i;
    const int q = c / B2, cl = c - q * B2;
    float2* dst = cluster.map_shared_rank(buf, q);
    dst[(cl * W + col) * (L2 + 1) + b] = v[i];
  }
  cluster.sync();

  // pass B: thread = ((j2 * B2) + cl) * W + col
  const int cl = (tid / W) % B2;
  const int j2 = tid / (W * B2);
  float2* seq = buf + (cl * W + col) * (L2 + 1);
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = seq[j2 + T2 * i];
  __syncthreads();
  block_fft<L2, R>(v, j2, seq, MapIdentity{}, coarse, Cfg::NC / L2);
  const int c = p * B2 + cl;
#pragma unroll
  for (int i = 0; i < R; ++i) __stcs(base + (int64_t)(c + L1 * (j2 + T2 * i)) * ncols + col, v[i]);
}

template <int L1, int L2, int C, int W>
static int prepare_columns() {
  auto kern = fft_columns_kernel<L1, L2, C, W>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ColCfg<L1, L2, C, W>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int L1, int L2, int C, int W>
static int launch_columns(float2* data, int64_t ncols, int64_t image_elems, int64_t batch,
                          const float2* coarse, const float2* fine, cudaStream_t s) {
  using Cfg = ColCfg<L1, L2, C, W>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * (ncols / W) * C), 1, 1);
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
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_columns_kernel<L1, L2, C, W>, data, ncols, image_elems,
                                    coarse, fine));
  return DPP_OK;
}

// Column schedules: (L1, L2, C, W) with L*W/C = 8192 points per CTA.
#define DPP_COLUMN_TABLE(X)   \
  X(256, 16, 16, 1, 32)       \
  X(512, 16, 32, 1, 16)       \
  X(1024, 32, 32, 2, 16)      \
  X(2048, 32, 64, 4, 16)      \
  X(4096, 64, 64, 8, 16)      \
  X(8192, 64, 128, 8, 8)      \
  X(16384, 128, 128, 16, 8)

std::vector<float2> twiddle_table(int64_t n, int64_t count);
int upload_table(const std::vector<float2>& h, float2** d);

int fft2d_plan_init(FftPlan* p) {
  const int64_t n0 = p->n0, n1 = p->n1;
  if (n0 < 2 || (n0 & (n0 - 1)) || n1 < 2 || (n1 & (n1 - 1)))
    return fail(DPP_EINVAL, "2-D sizes must be powers of two, got %lld x %lld", (long long)n0, (long long)n1);
  int width = 0, rc = DPP_ENOTSUP;
  int64_t l1 = 0;
  int cl = 1;
  switch (n0) {
#define PREP(L, A, B, C, W) \
  case L: width = W; l1 = A; cl = C; rc = prepare_columns<A, B, C, W>(); break;
    DPP_COLUMN_TABLE(PREP)
#undef PREP
  }
  if (rc == DPP_ENOTSUP)
    return fail(DPP_ENOTSUP, "2-D column length %lld not supported (256..16384)", (long long)n0);
  if (rc) return rc;
  if (n1 % width)
    return fail(DPP_ENOTSUP, "2-D row length %lld must be a multiple of the %d-column tile",
                (long long)n1, width);
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
  snprintf(p->desc, sizeof(p->desc), "rows: %s | columns: cluster<%lldx%lld, C=%d, W=%d>",
           p->rows->desc, (long long)l1, (long long)l2, cl, width);
  return DPP_OK;
}

int fft2d_columns_execute(const FftPlan* p, float2* data, int64_t batch, cudaStream_t s) {
  if (batch == 0) return DPP_OK;
  switch (p->n0) {
#define RUN(L, A, B, C, W) \
  case L: return launch_columns<A, B, C, W>(data, p->n1, p->n0 * p->n1, batch, p->ctw_a, p->ctw_b, s);
    DPP_COLUMN_TABLE(RUN)
#undef RUN
  }
  return fail(DPP_EINVAL, "no column kernel for %lld", (long long)p->n0);
}

int fft2d_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  if (batch == 0) return DPP_OK;
  int rc = fft1d_execute(p->rows, in, out, batch * p->n0, s);
  if (rc) return rc;
  switch (p->n0) {
#define RUN(L, A, B, C, W) \
  case L: return launch_columns<A, B, C, W>(out, p->n1, p->n0 * p->n1, batch, p->ctw_a, p->ctw_b, s);
    DPP_COLUMN_TABLE(RUN)
#undef RUN
  }
  return fail(DPP_EINVAL, "no column kernel for %lld", (long long)p->n0);
}

}  // namespace dpp
