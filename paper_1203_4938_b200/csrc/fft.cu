// FFT node for sm_100a: batched forward complex FFTs (1-D and 2-D).
//
// Replaces the reference's radix-2 FFT (/root/reference/pkg/src/dpp/apps/fft.py:150-174:
// host bit-reversal, platform leaf DFTs of size 2^k, host binary64 butterflies)
// with Stockham autosort radix-16 transforms that never leave the GPU.
//
// Kernels
//   fft_small_kernel<M>      n <= 4096: F transforms per CTA, one HBM read and
//                            one HBM write; passes exchange through SMEM.
//   fft_cluster_kernel<N1,N2,C>  n = N1*N2 (8192 .. 131072): four-step inside a
//                            thread-block cluster.  Pass 1 (N1-point column
//                            FFTs + twiddle) and pass 2 (N2-point row FFTs)
//                            exchange through distributed shared memory, so
//                            the transform still costs exactly one HBM read +
//                            one HBM write (the 16*n compulsory bytes).
//   fft_columns_kernel       2-D column pass (strided FFTs over rows), see fft2d.cu.
//   leaf_dft_kernel          the reference's dft2/4/8 node, bit-exact.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "fft_block.cuh"
#include "tma.cuh"

namespace dpp {

// ---------------------------------------------------------------------------
// n <= 4096

template <int M>
struct SmallCfg {
  static constexpr int R = M < 16 ? M : 16;
  static constexpr int T = M / R;
  static constexpr int F = T >= 256 ? 1 : 256 / T;  // transforms per CTA
  static constexpr int THREADS = F * T;
  static constexpr int STRIDE = M + M / 16 + 1;      // per-transform SMEM region
  static constexpr bool EXCHANGE = M > R;
  static constexpr size_t SMEM = EXCHANGE ? (size_t)(M + F * STRIDE) * sizeof(float2) : 0;
};

template <int M>
__global__ void __launch_bounds__(SmallCfg<M>::THREADS, 1024 / SmallCfg<M>::THREADS)
fft_small_kernel(const float2* __restrict__ in, float2* __restrict__ out, int64_t batch,
                 const float2* __restrict__ twg) {
  using Cfg = SmallCfg<M>;
  constexpr int R = Cfg::R, T = Cfg::T, F = Cfg::F;
  extern __shared__ float2 smem[];
  const int f = threadIdx.x / T;
  const int j = threadIdx.x - f * T;
  const int64_t g = (int64_t)blockIdx.x * F + f;
  const bool active = g < batch;
  float2 v[R];
  const float2* src = in + g * M;
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = active ? __ldcs(src + j + T * i) : make_float2(0.f, 0.f);
  if constexpr (Cfg::EXCHANGE) {
    float2* tw = smem;
    float2* buf = smem + M;
    for (int e = threadIdx.x; e < M; e += Cfg::THREADS) tw[e] = twg[e];
    __syncthreads();
    block_fft<M, R>(v, j, buf + f * Cfg::STRIDE, MapPad16{}, tw, 1);
  } else {
    dft_r<R>(v);
  }
  if (active) {
    float2* dst = out + g * M;
#pragma unroll
    for (int i = 0; i < R; ++i) __stcs(dst + j + T * i, v[i]);
  }
}

// ---------------------------------------------------------------------------
// n = N1 * N2 in one thread-block cluster of C CTAs.
//   n = N2*a + b  (a < N1, b < N2);  k = c + N1*d  (c < N1, d < N2)
//   Z[b][c]  = sum_a x[N2 a + b] W_N1^{ac}            pass 1, CTA p owns b in [p*W1, (p+1)*W1)
//   Z'[b][c] = Z[b][c] * W_N^{bc}
//   X[c+N1 d]= sum_b Z'[b][c] W_N2^{bd}                pass 2, CTA q owns c in [q*W2, (q+1)*W2)
// Global loads of pass 1 and stores of pass 2 are W-wide contiguous runs
// (W >= 32 complex = 256 B per warp instruction).  The Z' exchange is one
// all-to-all over DSMEM between two cluster barriers.

template <int N1, int N2, int C>
struct ClusterCfg {
  static constexpr int R = 16;
  static constexpr int N = N1 * N2;
  static constexpr int W1 = N2 / C, W2 = N1 / C;
  static constexpr int T1 = N1 / R, T2 = N2 / R;
  static constexpr int THREADS = W1 * T1;
  static_assert(THREADS == W2 * T2, "pass thread counts must agree");
  static constexpr int NC = N1 > N2 ? N1 : N2;  // coarse table W_NC
  static constexpr int S = N / NC;              // fine table W_N^lo, lo < S
  static constexpr int LOGS = ilog2(S);
  static constexpr int BUF1 = W1 * (N1 + 1), BUF2 = W2 * (N2 + 1);
  static constexpr int XPULL = N1 * (W1 + 1);   // pull layout: [c][b_local]
  static constexpr int BUF = BUF1 > BUF2 ? (BUF1 > XPULL ? BUF1 : XPULL) : (BUF2 > XPULL ? BUF2 : XPULL);
  static constexpr size_t SMEM = (size_t)(NC + S + BUF) * sizeof(float2);
};

// ---------------------------------------------------------------------------
// Reference leaf node dft{2,4,8} (fft.py:86-117), bit-exact.

struct LeafTerm {
  int8_t lane;   // operand component index in the float{2^(k+1)} vector
  int8_t neg;    // 1: subtract (or negate when first)
  int8_t unit;   // 1: coefficient is exactly 1 (operand used bare)
  int8_t pad;
  float coef;    // |coefficient| rounded to binary32 (the printed literal)
};
struct LeafProgram {
  int width;              // floats per work-item
  int nterms[16];         // terms per output component
  LeafTerm terms[16][16];
};

__global__ void leaf_dft_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t items,
                                const LeafProgram prog) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= items) return;
  const int w = prog.width;
  float in[16];
  for (int l = 0; l < w; ++l) in[l] = x[it * w + l];
  for (int o = 0; o < w; ++o) {
    float acc = 0.f;
    for (int tix = 0; tix < prog.nterms[o]; ++tix) {
      const LeafTerm tm = prog.terms[o][tix];
      const float opnd = in[tm.lane];
      const float term = tm.unit ? opnd : __fmul_rn(tm.coef, opnd);
      if (tix == 0) acc = tm.neg ? -term : term;
      else acc = tm.neg ? __fsub_rn(acc, term) : __fadd_rn(acc, term);
    }
    y[it * w + o] = acc;
  }
}

static LeafProgram make_leaf_program(int k) {
  // Coefficient generation as fft.py:56-83: cos/sin(-2*pi*t/size) in binary64,
  // exact 0/+-1 snapped, other magnitudes printed as the shortest binary32
  // literal (which parses back to (float)|c|).
  LeafProgram prog;
  std::memset(&prog, 0, sizeof(prog));
  const int size = 1 << k;
  prog.width = 2 * size;
  auto bitrev = [k](int n) {
    int r = 0;
    for (int b = 0; b < k; ++b) r = (r << 1) | ((n >> b) & 1);
    return r;
  };
  auto coeff = [size](int t, double& c, double& s) {
    const double ang = -2.0 * M_PI * (double)(t % size) / (double)size;
    c = std::cos(ang);
    s = std::sin(ang);
    const double exact[3] = {-1.0, 0.0, 1.0};
    for (double e : exact) {
      if (std::fabs(c - e) < 1e-12) c = e;
      if (std::fabs(s - e) < 1e-12) s = e;
    }
  };
  auto push = [&prog](int out, double cf, int lane) {
    if (cf == 0.0) return;
    LeafTerm tm;
    tm.lane = (int8_t)lane;
    tm.neg = cf < 0 ? 1 : 0;
    tm.unit = std::fabs(cf) == 1.0 ? 1 : 0;
    tm.pad = 0;
    tm.coef = (float)std::fabs(cf);
    prog.terms[out][prog.nterms[out]++] = tm;
  };
  for (int jj = 0; jj < size; ++jj) {
    for (int n = 0; n < size; ++n) {
      double c, s;
      coeff(jj * n, c, s);
      const int at = bitrev(n);
      push(2 * jj, c, 2 * at);          // re: + c*re_n
      push(2 * jj, -s, 2 * at + 1);     //      - s*im_n
      push(2 * jj + 1, s, 2 * at);      // im: + s*re_n
      push(2 * jj + 1, c, 2 * at + 1);  //      + c*im_n
    }
  }
  return prog;
}

// ---------------------------------------------------------------------------
// plan construction / dispatch

std::vector<float2> twiddle_table(int64_t n, int64_t count) {
  // W_n^e, e < count, computed in binary64 and rounded once
  std::vector<float2> t((size_t)count);
  for (int64_t e = 0; e < count; ++e) {
    const double a = -2.0 * M_PI * (double)e / (double)n;
    t[(size_t)e] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  return t;
}

int upload_table(const std::vector<float2>& h, float2** d) {
  DPP_CUDA_CHECK(cudaMalloc(d, h.size() * sizeof(float2)));
  DPP_CUDA_CHECK(cudaMemcpy(*d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice));
  return DPP_OK;
}

template <int M>
static int prepare_small() {
  DPP_CUDA_CHECK(cudaFuncSetAttribute(fft_small_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)SmallCfg<M>::SMEM));
  return DPP_OK;
}

template <int M>
static int launch_small(const float2* in, float2* out, int64_t batch, const float2* tw, cudaStream_t s) {
  using Cfg = SmallCfg<M>;
  const int64_t blocks = (batch + Cfg::F - 1) / Cfg::F;
  fft_small_kernel<M><<<(unsigned)blocks, Cfg::THREADS, Cfg::SMEM, s>>>(in, out, batch, tw);
  DPP_LAUNCH_CHECK("fft_small_kernel");
  return DPP_OK;
}

// The cluster kernel (the sizes the L2-ring kernels do not cover: 2048 and the
// 2^13..2^15 batch remainders): one column per thread, exchanges in
// [element][W] rows (a warp's 32 columns = one 256 B row), an XOR-swizzled
// receive buffer, one TMA tile load and recurrence twiddles.
struct MapRow {
  int w, col;
  __device__ __forceinline__ int operator()(int e) const { return e * w + col; }
};

template <int N1, int N2, int C>
struct RowsCfg {
  using Base = ClusterCfg<N1, N2, C>;
  static constexpr int TILE = N1 * N2 / C;
  static constexpr int BUF = TILE;
  // coarse twiddles as float4 (w, i*w): 2 float2 slots per entry
  static constexpr size_t SMEM = (size_t)(2 * Base::NC + BUF) * sizeof(float2);
};

template <int THREADS>
struct RowsMinBlocks {
  static constexpr int value = THREADS == 256 ? 4 : 1024 / THREADS;
};

template <int N1, int N2, int C>
__global__ void __launch_bounds__(ClusterCfg<N1, N2, C>::THREADS, RowsMinBlocks<ClusterCfg<N1, N2, C>::THREADS>::value)
fft_cluster_rows(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out,
                 const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ClusterCfg<N1, N2, C>;
  constexpr int R = Cfg::R, N = Cfg::N, W1 = Cfg::W1, W2 = Cfg::W2, T1 = Cfg::T1, T2 = Cfg::T2;
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  float4* coarse = reinterpret_cast<float4*>(smem);
  float2* buf = smem + 2 * Cfg::NC;
  float2* recv = buf;

  const int p = (int)cluster_ctarank();
  const int64_t t = blockIdx.x / C;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[0], (uint32_t)(N1 * W1 * sizeof(float2)));
    mbar_arrive_expect_tx(&bars[1], (uint32_t)(N2 * W2 * sizeof(float2)));
    tma_load_2d(buf, &tin, p * W1, (int)(t * N1), &bars[0]);
  }
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) {
    const float2 w = coarse_g[e];
    coarse[e] = make_float4(w.x, w.y, -w.y, w.x);
  }
  __syncthreads();

  const int col = tid % W1, j = tid / W1;
  const int b = p * W1 + col;
  // per-thread four-step bases from the global tables (L1-cached, no bank
  // conflicts), fetched before the tile wait so their latency hides behind it
  const float2 tw0a = __ldg(coarse_g + ((b * j) >> Cfg::LOGS)), tw0b = __ldg(fine_g + ((b * j) & (Cfg::S - 1)));
  const float2 tw1a = __ldg(coarse_g + ((b * T1) >> Cfg::LOGS)), tw1b = __ldg(fine_g + ((b * T1) & (Cfg::S - 1)));
  float2 v[R];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = buf[(j + T1 * i) * W1 + col];
  __syncthreads();
  block_fft<N1, R>(v, j, buf, MapRow{W1, col}, coarse, Cfg::NC / N1);
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
    const uint32_t base = smem_u32(recv);
    const uint32_t rbar = smem_u32(&bars[1]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = j + T1 * i;
      const int q = c / W2, cl = c - q * W2;
      const uint32_t off = (uint32_t)((cl * N2 + (b ^ (cl & 15))) * sizeof(float2));
      st_async_f2(mapa_u32(base + off, q), v[i], mapa_u32(rbar, q));
    }
  }
  mbar_wait(&bars[1], 0);
  const int cl = tid % W2, j2 = tid / W2;
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = recv[cl * N2 + ((j2 + T2 * i) ^ (cl & 15))];
  __syncthreads();
  block_fft<N2, R>(v, j2, buf, MapRow{W2, cl}, coarse, Cfg::NC / N2);
  float2* dst = out + t * N + p * W2 + cl;
#pragma unroll
  for (int i = 0; i < R; ++i) __stcs(dst + (int64_t)(j2 + T2 * i) * N1, v[i]);
}

template <int N1, int N2, int C>
static int prepare_rows() {
  auto kern = fft_cluster_rows<N1, N2, C>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)RowsCfg<N1, N2, C>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int N1, int N2, int C>
static int launch_rows(const float2* in, float2* out, int64_t batch, const float2* coarse, const float2* fine,
                       cudaStream_t s) {
  using Cfg = ClusterCfg<N1, N2, C>;
  CUtensorMap tmap;
  int rc = make_tmap_c64(&tmap, in, (uint64_t)batch * N1, N2, N1, Cfg::W1);
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * C), 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = RowsCfg<N1, N2, C>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_cluster_rows<N1, N2, C>, tmap, out, coarse, fine));
  return DPP_OK;
}

template <int N1, int N2, int C>
static int prepare_cluster(FftPlan*) {
  return prepare_rows<N1, N2, C>();
}

template <int N1, int N2, int C>
static int launch_cluster(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  return launch_rows<N1, N2, C>(in, out, batch, p->tw_a, p->tw_b, s);
}

// One schedule per size (the variants measured against them are in
// profiles/r1_*.md and profiles/r2_*.md):
//   2..1024                small<M>: radix-16 Stockham, one CTA
//   2048                   cluster rows (1 CTA), 32 x 64
//   4096                   fft4096_ws (fft4k.cu): warp-specialised single-CTA
//   8192, 16384, 32768     fft16k_l2w (fft16k_l2.cu): L2 ring; batch remainders
//                          (< 65536 / n transforms) on the cluster kernel
//   65536                  fft65536_l2w (fft_l2.cu): L2 ring, the C2 kernel
//   2^17 .. 2^20           fft_ring512_l2w (fft128k_l2.cu): L2 ring
//   2^21 .. 2^30           fft_large.cu: transpose + rows + twiddled column ring
int fft1d_plan_init(FftPlan* p) {
  const int64_t n = p->n0;
  const int lg = ilog2(n);
  if (n < 2 || (n & (n - 1)) != 0)
    return fail(DPP_EINVAL, "transform size must be a power of two, got %lld", (long long)n);
  if (lg <= 10) {
    p->kind = FftPlan::SMALL;
    int rc = DPP_OK;
    switch (n) {
#define SMALL_PREP(M) case M: rc = prepare_small<M>(); break;
      SMALL_PREP(2) SMALL_PREP(4) SMALL_PREP(8) SMALL_PREP(16) SMALL_PREP(32) SMALL_PREP(64)
      SMALL_PREP(128) SMALL_PREP(256) SMALL_PREP(512) SMALL_PREP(1024) SMALL_PREP(2048) SMALL_PREP(4096)
#undef SMALL_PREP
    }
    if (rc) return rc;
    if (upload_table(twiddle_table(n, n), &p->tw_a)) return DPP_ECUDA;
    snprintf(p->desc, sizeof(p->desc), "small<%lld> radix-16 stockham, 1 CTA", (long long)n);
    return DPP_OK;
  }
  if (n == 65536) {
    p->kind = FftPlan::L2X;
    if (int rc = fft65536_l2x_init(p)) return rc;
    snprintf(p->desc, sizeof(p->desc),
             "two-pass 256x256 four-step, L2-resident exchange (ring %d, lag %d), 32 KB SMEM transpose per item",
             p->l2_ring, p->l2_lag);
    return DPP_OK;
  }
  if (lg >= 17 && lg <= 20) {
    p->kind = FftPlan::CLUSTER;
    if (int rc = fft128k_l2_init(p)) return rc;
    p->ring128k = 1;
    snprintf(p->desc, sizeof(p->desc),
             "two-pass %lldx%lld four-step, L2-resident exchange (ring %d, lag %d), warp-wide 512-point FFTs",
             (long long)(n <= 262144 ? 256 : (n <= 524288 ? 512 : 1024)),
             (long long)(n <= 262144 ? n / 256 : (n <= 524288 ? n / 512 : 1024)), p->l2_ring, p->l2_lag);
    return DPP_OK;
  }
  if (lg > 20) return fft_large_init(p);
  // 2048 .. 32768: n = N1 * N2 (N1 <= N2), C CTAs of <= 8192 points
  p->kind = FftPlan::CLUSTER;
  p->n1a = 1LL << (lg / 2);
  p->n2a = n / p->n1a;
  p->cluster = (int)(n / 8192 > 1 ? n / 8192 : 1);
  int rc = DPP_OK;
  switch (n) {
    case 2048: rc = prepare_cluster<32, 64, 1>(p); break;
    case 4096: rc = prepare_cluster<64, 64, 1>(p); break;
    case 8192: rc = prepare_cluster<64, 128, 1>(p); break;
    case 16384: rc = prepare_cluster<128, 128, 2>(p); break;
    case 32768: rc = prepare_cluster<128, 256, 4>(p); break;
  }
  if (rc) return rc;
  const int64_t nc = p->n1a > p->n2a ? p->n1a : p->n2a;
  if (upload_table(twiddle_table(nc, nc), &p->tw_a)) return DPP_ECUDA;
  if (upload_table(twiddle_table(n, n / nc), &p->tw_b)) return DPP_ECUDA;
  if (n == 4096) {
    if (int rc2 = fft4096_ws_init(p)) return rc2;
    p->ws4k = 1;
    snprintf(p->desc, sizeof(p->desc),
             "256x16 in one CTA, warp-specialised TMA pipeline (2 stages, P1 warp-local, P2 in-thread)");
    return DPP_OK;
  }
  if (n >= 8192) {
    if (int rc2 = fft16k_l2_init(p)) return rc2;
    p->ring16k = 1;
    snprintf(p->desc, sizeof(p->desc),
             "two-pass 256x%lld four-step, L2-resident exchange (ring %d, lag %d), units of %lld transforms",
             (long long)(n / 256), p->l2_ring, p->l2_lag, (long long)(65536 / n));
    return DPP_OK;
  }
  snprintf(p->desc, sizeof(p->desc), "cluster<%lldx%lld, C=%d> four-step over DSMEM, row layouts",
           (long long)p->n1a, (long long)p->n2a, p->cluster);
  return DPP_OK;
}

int fft1d_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  if (batch == 0) return DPP_OK;
  if (p->kind == FftPlan::SMALL) {
    switch (p->n0) {
#define SMALL_CASE(M) case M: return launch_small<M>(in, out, batch, p->tw_a, s);
      SMALL_CASE(2) SMALL_CASE(4) SMALL_CASE(8) SMALL_CASE(16) SMALL_CASE(32) SMALL_CASE(64)
      SMALL_CASE(128) SMALL_CASE(256) SMALL_CASE(512) SMALL_CASE(1024) SMALL_CASE(2048) SMALL_CASE(4096)
#undef SMALL_CASE
    }
  } else if (p->kind == FftPlan::L2X) {
    return fft65536_l2x_execute(p, in, out, batch, s);
  } else if (p->kind == FftPlan::LARGE) {
    return fft_large_execute(p, in, out, batch, s);
  } else if (p->kind == FftPlan::CLUSTER) {
    if (p->ws4k) return fft4096_ws_execute(p, in, out, batch, s);
    if (p->ring128k) return fft128k_l2_execute(p, in, out, batch, s);
    if (p->ring16k) {
      const int64_t tpu = 65536 / p->n0;  // transforms per ring unit
      const int64_t main = batch - batch % tpu;
      if (int rc = fft16k_l2_execute(p, in, out, main, s)) return rc;
      if (main == batch) return DPP_OK;
      const int64_t n = p->n0, rest = batch - main;
      if (n == 8192) return launch_cluster<64, 128, 1>(p, in + main * n, out + main * n, rest, s);
      if (n == 16384) return launch_cluster<128, 128, 2>(p, in + main * n, out + main * n, rest, s);
      return launch_cluster<128, 256, 4>(p, in + main * n, out + main * n, rest, s);
    }
    if (p->n0 == 2048) return launch_cluster<32, 64, 1>(p, in, out, batch, s);
  }
  return fail(DPP_EINVAL, "no kernel for 1-D size %lld", (long long)p->n0);
}

int leaf_execute(int k, const float* x, float* y, int64_t items, cudaStream_t s) {
  static LeafProgram progs[4];
  static bool built[4] = {false, false, false, false};
  if (k < 1 || k > 3) return fail(DPP_EINVAL, "leaf order must be 1..3, got %d", k);
  if (!built[k]) {
    progs[k] = make_leaf_program(k);
    built[k] = true;
  }
  if (items == 0) return DPP_OK;
  const int threads = 128;
  const int64_t blocks = (items + threads - 1) / threads;
  leaf_dft_kernel<<<(unsigned)blocks, threads, 0, s>>>(x, y, items, progs[k]);
  DPP_LAUNCH_CHECK("leaf_dft_kernel");
  return DPP_OK;
}

}  // namespace dpp
