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
#include <cooperative_groups.h>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "fft_block.cuh"

namespace cg = cooperative_groups;

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
__global__ void __launch_bounds__(SmallCfg<M>::THREADS)
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
  static constexpr int BUF = BUF1 > BUF2 ? BUF1 : BUF2;
  static constexpr size_t SMEM = (size_t)(NC + S + BUF) * sizeof(float2);
};

template <int N1, int N2, int C>
__global__ void __launch_bounds__(ClusterCfg<N1, N2, C>::THREADS)
fft_cluster_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                   const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ClusterCfg<N1, N2, C>;
  constexpr int R = Cfg::R, N = Cfg::N, W1 = Cfg::W1, W2 = Cfg::W2, T1 = Cfg::T1, T2 = Cfg::T2;
  extern __shared__ float2 smem[];
  float2* coarse = smem;
  float2* fine = smem + Cfg::NC;
  float2* buf = fine + Cfg::S;

  cg::cluster_group cluster = cg::this_cluster();
  const int p = (int)cluster.block_rank();
  const int64_t t = blockIdx.x / C;
  const int tid = threadIdx.x;

  // pass 1: column FFTs over a for b in this CTA's slice
  const int j = tid / W1, col = tid - (tid / W1) * W1;
  const int b = p * W1 + col;
  float2 v[R];
  const float2* src = in + t * N + b;
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = __ldcs(src + (int64_t)(j + T1 * i) * N2);
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) coarse[e] = coarse_g[e];
  for (int e = tid; e < Cfg::S; e += Cfg::THREADS) fine[e] = fine_g[e];
  __syncthreads();
  block_fft<N1, R>(v, j, buf + col * (N1 + 1), MapIdentity{}, coarse, Cfg::NC / N1);
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int e = b * (j + T1 * i);  // b*c < N: exact in int32
    v[i] = cmul(v[i], cmul(coarse[e >> Cfg::LOGS], fine[e & (Cfg::S - 1)]));
  }

  cluster.sync();  // every CTA has finished reading its own buffer
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int c = j + T1 * i;
    const int q = c / W2, cl = c - (c / W2) * W2;
    float2* dst = cluster.map_shared_rank(buf, q);
    dst[cl * (N2 + 1) + b] = v[i];
  }
  cluster.sync();  // all Z' slices delivered

  // pass 2: row FFTs over b for c in this CTA's slice
  const int j2 = tid / W2, cl = tid - (tid / W2) * W2;
  float2* row = buf + cl * (N2 + 1);
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = row[j2 + T2 * i];
  __syncthreads();
  block_fft<N2, R>(v, j2, row, MapIdentity{}, coarse, Cfg::NC / N2);
  const int c = p * W2 + cl;
  float2* dst = out + t * N + c;
#pragma unroll
  for (int i = 0; i < R; ++i) __stcs(dst + (int64_t)(j2 + T2 * i) * N1, v[i]);
}

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

template <int N1, int N2, int C>
static int prepare_cluster() {
  auto kern = fft_cluster_kernel<N1, N2, C>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ClusterCfg<N1, N2, C>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int N1, int N2, int C>
static int launch_cluster(const float2* in, float2* out, int64_t batch, const float2* coarse,
                          const float2* fine, cudaStream_t s) {
  using Cfg = ClusterCfg<N1, N2, C>;
  auto kern = fft_cluster_kernel<N1, N2, C>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * C), 1, 1);
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
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, in, out, coarse, fine));
  return DPP_OK;
}

int fft1d_plan_init(FftPlan* p) {
  const int64_t n = p->n0;
  const int lg = ilog2(n);
  if (n < 2 || (n & (n - 1)) != 0)
    return fail(DPP_EINVAL, "transform size must be a power of two, got %lld", (long long)n);
  if (lg <= 12) {
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
  if (lg <= 17) {
    // split n = N1 * N2 with N1 <= N2, cluster C so that each CTA holds <= 8192 points
    p->kind = FftPlan::CLUSTER;
    p->n1a = 1LL << (lg / 2);
    p->n2a = n / p->n1a;
    p->cluster = (int)(n / 8192 > 1 ? n / 8192 : 1);
    int rc = DPP_OK;
    switch (n) {
      case 8192: rc = prepare_cluster<64, 128, 1>(); break;
      case 16384: rc = prepare_cluster<128, 128, 2>(); break;
      case 32768: rc = prepare_cluster<128, 256, 4>(); break;
      case 65536: rc = prepare_cluster<256, 256, 8>(); break;
      case 131072: rc = prepare_cluster<256, 512, 16>(); break;
    }
    if (rc) return rc;
    const int64_t nc = p->n1a > p->n2a ? p->n1a : p->n2a;
    if (upload_table(twiddle_table(nc, nc), &p->tw_a)) return DPP_ECUDA;
    if (upload_table(twiddle_table(n, n / nc), &p->tw_b)) return DPP_ECUDA;
    snprintf(p->desc, sizeof(p->desc), "cluster<%lldx%lld, C=%d> four-step over DSMEM",
             (long long)p->n1a, (long long)p->n2a, p->cluster);
    return DPP_OK;
  }
  return fail(DPP_ENOTSUP, "1-D transform size 2^%d is above the 2^17 single-pass limit", lg);
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
  } else if (p->kind == FftPlan::CLUSTER) {
    switch (p->n0) {
      case 8192: return launch_cluster<64, 128, 1>(in, out, batch, p->tw_a, p->tw_b, s);
      case 16384: return launch_cluster<128, 128, 2>(in, out, batch, p->tw_a, p->tw_b, s);
      case 32768: return launch_cluster<128, 256, 4>(in, out, batch, p->tw_a, p->tw_b, s);
      case 65536: return launch_cluster<256, 256, 8>(in, out, batch, p->tw_a, p->tw_b, s);
      case 131072: return launch_cluster<256, 512, 16>(in, out, batch, p->tw_a, p->tw_b, s);
    }
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
