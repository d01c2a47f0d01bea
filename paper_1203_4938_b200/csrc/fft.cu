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

// MODE 0: push — each CTA stores its Z' slices into the owners' buffers
//         (st.shared::cluster) between two cluster barriers.
// MODE 1: pull — each CTA publishes Z' in its own buffer and loads what it
//         owns from the others (ld.shared::cluster).  Measured 3x slower.
// MODE 2: async — the input tile arrives by bulk copies (TMA engine,
//         cp.async.bulk, one 256 B row per thread) on an mbarrier; Z' goes
//         out with st.async, each element signalling the owner's receive
//         mbarrier, so the only cluster-wide barrier is a split, fence-free
//         "my buffer is free" arrive/wait that overlaps the twiddle pass.
template <int N1, int N2, int C, int MODE>
__global__ void __launch_bounds__(ClusterCfg<N1, N2, C>::THREADS, 1024 / ClusterCfg<N1, N2, C>::THREADS)
fft_cluster_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                   const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ClusterCfg<N1, N2, C>;
  constexpr int R = Cfg::R, N = Cfg::N, W1 = Cfg::W1, W2 = Cfg::W2, T1 = Cfg::T1, T2 = Cfg::T2;
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];  // [0] input tile landed, [1] Z' slice received
  float2* coarse = smem;
  float2* fine = smem + Cfg::NC;
  float2* buf = fine + Cfg::S;

  const int p = (int)cluster_ctarank();
  const int64_t t = blockIdx.x / C;
  const int tid = threadIdx.x;
  const int j = tid / W1, col = tid - (tid / W1) * W1;
  const int b = p * W1 + col;
  float2 v[R];

  if constexpr (MODE == 2) {
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&bars[0], (uint32_t)(N1 * W1 * sizeof(float2)));
      mbar_arrive_expect_tx(&bars[1], (uint32_t)(N2 * W2 * sizeof(float2)));
    }
    __syncthreads();
    if (tid < N1)  // row a of the tile: W1 contiguous complex values
      bulk_g2s(buf + tid * W1, in + t * N + (int64_t)tid * N2 + p * W1, W1 * sizeof(float2), &bars[0]);
    for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) coarse[e] = coarse_g[e];
    for (int e = tid; e < Cfg::S; e += Cfg::THREADS) fine[e] = fine_g[e];
    mbar_wait(&bars[0], 0);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[(j + T1 * i) * W1 + col];
  } else {
    const float2* src = in + t * N + b;
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = __ldcs(src + (int64_t)(j + T1 * i) * N2);
    for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) coarse[e] = coarse_g[e];
    for (int e = tid; e < Cfg::S; e += Cfg::THREADS) fine[e] = fine_g[e];
  }
  __syncthreads();

  // pass 1: column FFTs over a for b in this CTA's slice
  block_fft<N1, R>(v, j, buf + col * (N1 + 1), MapIdentity{}, coarse, Cfg::NC / N1);
  if constexpr (MODE == 2) cluster_arrive_relaxed();  // this CTA no longer reads buf
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int e = b * (j + T1 * i);  // b*c < N: exact in int32
    v[i] = cmul(v[i], cmul(coarse[e >> Cfg::LOGS], fine[e & (Cfg::S - 1)]));
  }

  const int j2 = tid / W2, cl = tid - (tid / W2) * W2;
  float2* row = buf + cl * (N2 + 1);
  if constexpr (MODE == 2) {
    cluster_wait();  // every destination buffer is free and its mbarrier initialised
    const uint32_t base = smem_u32(buf);
    const uint32_t rbar = smem_u32(&bars[1]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = j + T1 * i;
      const int q = c / W2, cq = c - (c / W2) * W2;
      st_async_f2(mapa_u32(base + (uint32_t)((cq * (N2 + 1) + b) * sizeof(float2)), q), v[i],
                  mapa_u32(rbar, q));
    }
    mbar_wait(&bars[1], 0);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = row[j2 + T2 * i];
    __syncthreads();
  } else if constexpr (MODE == 0) {
    cluster_sync();  // every CTA has finished reading its own buffer
    const uint32_t base = smem_u32(buf);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = j + T1 * i;
      const int q = c / W2, cq = c - (c / W2) * W2;
      st_cluster(mapa_u32(base + (uint32_t)((cq * (N2 + 1) + b) * sizeof(float2)), q), v[i]);
    }
    cluster_sync();  // all Z' slices delivered
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = row[j2 + T2 * i];
    __syncthreads();
  } else {
    __syncthreads();  // pass-1 exchange reads of buf are done
#pragma unroll
    for (int i = 0; i < R; ++i) buf[(j + T1 * i) * (W1 + 1) + col] = v[i];
    cluster_sync();  // every Z' slice is published
    const int c = p * W2 + cl;
    const uint32_t base = smem_u32(buf) + (uint32_t)(c * (W1 + 1) * sizeof(float2));
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int bb = j2 + T2 * i;
      const int q = bb / W1, bl = bb - (bb / W1) * W1;
      v[i] = ld_cluster(mapa_u32(base + (uint32_t)(bl * sizeof(float2)), q));
    }
    cluster_arrive();  // done reading the other CTAs' buffers
    cluster_wait();    // ... and they are done reading ours before it is reused
  }

  // pass 2: row FFTs over b for c in this CTA's slice
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

// ---------------------------------------------------------------------------
// MODE 3 (default): persistent clusters.  Each cluster loops over transforms
// t = cluster, cluster + nclusters, ...  Per transform and CTA:
//   one TMA tile load (64 KB box) on mbarrier bars[0] — issued for t+1 as
//   soon as pass 2 has drained the buffer, so it overlaps the stores and the
//   next iteration's wait; pass 1; split fence-free cluster barrier ("my
//   buffer is free"); four-step twiddles by a per-thread recurrence (no
//   table lookups); st.async scatter signalling the owners' bars[1]; pass 2;
//   streaming stores.  Twiddle tables are loaded once per CTA.
template <int N1, int N2, int C>
__global__ void __launch_bounds__(ClusterCfg<N1, N2, C>::THREADS, 1024 / ClusterCfg<N1, N2, C>::THREADS)
fft_cluster_persistent(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, int64_t batch,
                       const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ClusterCfg<N1, N2, C>;
  constexpr int R = Cfg::R, N = Cfg::N, W1 = Cfg::W1, W2 = Cfg::W2, T1 = Cfg::T1, T2 = Cfg::T2;
  constexpr uint32_t TILE_BYTES = N1 * W1 * sizeof(float2);
  constexpr uint32_t RECV_BYTES = N2 * W2 * sizeof(float2);
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  float2* coarse = smem;
  float2* fine = smem + Cfg::NC;
  float2* buf = fine + Cfg::S;

  const int p = (int)cluster_ctarank();
  const int64_t cluster = blockIdx.x / C;
  const int64_t nclusters = gridDim.x / C;
  const int tid = threadIdx.x;
  const int j = tid / W1, col = tid - (tid / W1) * W1;
  const int b = p * W1 + col;
  const int j2 = tid / W2, cl = tid - (tid / W2) * W2;
  float2* row = buf + cl * (N2 + 1);

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if (cluster < batch) {
      mbar_arrive_expect_tx(&bars[0], TILE_BYTES);
      tma_load_2d(buf, &tin, p * W1, (int)(cluster * N1), &bars[0]);
    }
  }
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) coarse[e] = coarse_g[e];
  for (int e = tid; e < Cfg::S; e += Cfg::THREADS) fine[e] = fine_g[e];
  __syncthreads();
  const uint32_t base = smem_u32(buf);
  const uint32_t rbar = smem_u32(&bars[1]);

  uint32_t phase = 0;
  for (int64_t t = cluster; t < batch; t += nclusters, phase ^= 1) {
    float2 v[R];
    mbar_wait(&bars[0], phase);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[(j + T1 * i) * W1 + col];
    if (tid == 0) mbar_arrive_expect_tx(&bars[1], RECV_BYTES);
    __syncthreads();
    block_fft<N1, R>(v, j, buf + col * (N1 + 1), MapIdentity{}, coarse, Cfg::NC / N1);
    cluster_arrive_relaxed();  // this CTA no longer reads buf
    {
      // four-step twiddles W_N^{b*(j + T1*i)} = w0 * step^i (a short recurrence
      // instead of 2 bank-conflicting table reads per element)
      const int e0 = b * j, es = b * T1;
      float2 w = cmul(coarse[e0 >> Cfg::LOGS], fine[e0 & (Cfg::S - 1)]);
      const float2 step = cmul(coarse[es >> Cfg::LOGS], fine[es & (Cfg::S - 1)]);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        v[i] = cmul(v[i], w);
        w = cmul(w, step);
      }
    }
    cluster_wait();  // every destination buffer is free (and its mbarrier armed)
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = j + T1 * i;
      const int q = c / W2, cq = c - (c / W2) * W2;
      st_async_f2(mapa_u32(base + (uint32_t)((cq * (N2 + 1) + b) * sizeof(float2)), q), v[i],
                  mapa_u32(rbar, q));
    }
    mbar_wait(&bars[1], phase);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = row[j2 + T2 * i];
    __syncthreads();
    block_fft<N2, R>(v, j2, row, MapIdentity{}, coarse, Cfg::NC / N2);  // ends with a CTA barrier
    if (tid == 0 && t + nclusters < batch) {
      mbar_arrive_expect_tx(&bars[0], TILE_BYTES);
      tma_load_2d(buf, &tin, p * W1, (int)((t + nclusters) * N1), &bars[0]);
    }
    float2* dst = out + t * N + p * W2 + cl;
#pragma unroll
    for (int i = 0; i < R; ++i) __stcs(dst + (int64_t)(j2 + T2 * i) * N1, v[i]);
  }
}

template <int N1, int N2, int C>
static int prepare_persistent(int* max_clusters) {
  using Cfg = ClusterCfg<N1, N2, C>;
  auto kern = fft_cluster_persistent<N1, N2, C>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 1024, 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DPP_CUDA_CHECK(cudaOccupancyMaxActiveClusters(max_clusters, kern, &cfg));
  if (*max_clusters < 1) return fail(DPP_ENOTSUP, "cluster of %d CTAs cannot be scheduled", C);
  return DPP_OK;
}

template <int N1, int N2, int C>
static int launch_persistent(const float2* in, float2* out, int64_t batch, const float2* coarse,
                             const float2* fine, int max_clusters, cudaStream_t s) {
  using Cfg = ClusterCfg<N1, N2, C>;
  CUtensorMap tmap;
  int rc = make_tmap_c64(&tmap, in, (uint64_t)batch * N1, N2, N1, Cfg::W1);
  if (rc) return rc;
  const int64_t clusters = batch < max_clusters ? batch : max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * C), 1, 1);
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
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_cluster_persistent<N1, N2, C>, tmap, out, batch, coarse, fine));
  return DPP_OK;
}

// ---------------------------------------------------------------------------
// MODE 4 (default): column pairs.  Same four-step/DSMEM schedule as MODE 2,
// but every thread carries two adjacent columns (256 threads per CTA), so
//   - the input tile arrives by ONE 2-D TMA load (box W1 x N1) per CTA;
//   - all shared-memory traffic is 16-byte LDS.128/STS.128 over contiguous
//     256-byte rows (block_fft_pair): no bank conflicts, half the MIO ops;
//   - the Z' scatter is one 16-byte st.async per element pair, into an
//     XOR-swizzled receive layout so the pass-2 reads are conflict-free too;
//   - outputs leave as 16-byte streaming stores (256 B per half-warp).
template <int N1, int N2, int C>
struct PairCfg {
  static constexpr int R = 16;
  static constexpr int N = N1 * N2;
  static constexpr int W1 = N2 / C, W2 = N1 / C;
  static constexpr int P1 = W1 / 2, P2 = W2 / 2;
  static constexpr int T1 = N1 / R, T2 = N2 / R;
  static constexpr int THREADS = P1 * T1;
  static_assert(THREADS == P2 * T2, "pass thread counts must agree");
  static constexpr int NC = N1 > N2 ? N1 : N2;
  static constexpr int S = N / NC;
  static constexpr int LOGS = ilog2(S);
  static constexpr int BUF = N / C;
  static constexpr size_t SMEM = (size_t)(NC + S + BUF) * sizeof(float2);
};

// receive-layout swizzle: element (cl, b) lives at cl*N2 + (b ^ rsw(cl))
__device__ __forceinline__ int rsw(int cl) { return ((cl >> 1) & 7) << 1; }

template <int N1, int N2, int C>
__global__ void __launch_bounds__(PairCfg<N1, N2, C>::THREADS, 2)
fft_cluster_pair(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out,
                 const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = PairCfg<N1, N2, C>;
  constexpr int R = Cfg::R, N = Cfg::N, W1 = Cfg::W1, W2 = Cfg::W2, T1 = Cfg::T1, T2 = Cfg::T2;
  constexpr int P1 = Cfg::P1, P2 = Cfg::P2;
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  float2* coarse = smem;
  float2* fine = smem + Cfg::NC;
  float2* buf = fine + Cfg::S;

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
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) coarse[e] = coarse_g[e];
  for (int e = tid; e < Cfg::S; e += Cfg::THREADS) fine[e] = fine_g[e];
  __syncthreads();

  // pass 1: columns b0 = p*W1 + 2cp and b0 + 1, FFT over a
  const int cp = tid % P1, j = tid / P1;
  float2 v0[R], v1[R];
  mbar_wait(&bars[0], 0);
  {
    const float4* tile = reinterpret_cast<const float4*>(buf) + cp;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float4 x = tile[(j + T1 * i) * P1];
      v0[i] = make_float2(x.x, x.y);
      v1[i] = make_float2(x.z, x.w);
    }
  }
  __syncthreads();
  block_fft_pair<N1, R, W1>(v0, v1, j, cp, buf, coarse, Cfg::NC / N1);
  cluster_arrive_relaxed();  // this CTA no longer reads buf
  const int b0 = p * W1 + 2 * cp;
  {
    // W_N^{b0 c} and W_N^{(b0+1) c} for c = j + T1*i by recurrences in i
    auto tw = [&](int e) { return cmul(coarse[e >> Cfg::LOGS], fine[e & (Cfg::S - 1)]); };
    float2 w = tw(b0 * j), u = tw(j);
    const float2 sw = tw(b0 * T1), su = tw(T1);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v0[i] = cmul(v0[i], w);
      v1[i] = cmul(v1[i], cmul(w, u));
      w = cmul(w, sw);
      u = cmul(u, su);
    }
  }
  cluster_wait();  // every destination buffer is free and its mbarrier armed
  {
    const uint32_t base = smem_u32(buf);
    const uint32_t rbar = smem_u32(&bars[1]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = j + T1 * i;
      const int q = c / W2, cl = c - q * W2;
      const uint32_t off = (uint32_t)((cl * N2 + (b0 ^ rsw(cl))) * sizeof(float2));
      st_async_f4(mapa_u32(base + off, q), make_float4(v0[i].x, v0[i].y, v1[i].x, v1[i].y), mapa_u32(rbar, q));
    }
  }
  mbar_wait(&bars[1], 0);

  // pass 2: c0 = p*W2 + 2cp2 and c0 + 1, FFT over b
  const int cp2 = tid % P2, j2 = tid / P2;
  {
    const int cl0 = 2 * cp2, cl1 = cl0 + 1;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int b = j2 + T2 * i;
      v0[i] = buf[cl0 * N2 + (b ^ rsw(cl0))];
      v1[i] = buf[cl1 * N2 + (b ^ rsw(cl1))];
    }
  }
  __syncthreads();
  block_fft_pair<N2, R, W2>(v0, v1, j2, cp2, buf, coarse, Cfg::NC / N2);
  float4* dst = reinterpret_cast<float4*>(out + t * N + p * W2 + 2 * cp2);
#pragma unroll
  for (int i = 0; i < R; ++i)
    __stcs(dst + (int64_t)(j2 + T2 * i) * (N1 / 2), make_float4(v0[i].x, v0[i].y, v1[i].x, v1[i].y));
}

// MODE 5: one column per thread (512 threads, 64 registers -> 2 CTAs = 32
// warps per SM) with the same conflict-free row layouts as MODE 4: exchanges
// in [element][W] rows (a warp's 32 columns = one 256 B row), an XOR-
// swizzled receive buffer, one TMA tile load and recurrence twiddles.
struct MapRow {
  int w, col;
  __device__ __forceinline__ int operator()(int e) const { return e * w + col; }
};

// SEPRECV (MODE 6): a separate receive buffer, so no CTA ever has to wait for
// the others to stop using theirs — the only cluster barrier (mbarrier-init
// visibility) is arrived at kernel start and waited just before the scatter.
template <int N1, int N2, int C, bool SEPRECV>
struct RowsCfg {
  using Base = ClusterCfg<N1, N2, C>;
  static constexpr int TILE = N1 * N2 / C;
  static constexpr int BUF = TILE;
  // coarse twiddles as float4 (w, i*w): 2 float2 slots per entry
  static constexpr size_t SMEM = (size_t)(2 * Base::NC + BUF + (SEPRECV ? TILE : 0)) * sizeof(float2);
};

#ifndef DPP_EXP
#define DPP_EXP 0  // profiling only: 1 = data movement without the FFT math, 2 = math without HBM traffic
#endif
#ifndef DPP_ROWS_MINB256
#define DPP_ROWS_MINB256 4
#endif
template <int THREADS>
struct RowsMinBlocks {
  static constexpr int value = THREADS == 256 ? DPP_ROWS_MINB256 : 1024 / THREADS;
};

template <int N1, int N2, int C, bool SEPRECV>
__global__ void __launch_bounds__(ClusterCfg<N1, N2, C>::THREADS, RowsMinBlocks<ClusterCfg<N1, N2, C>::THREADS>::value)
fft_cluster_rows(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out,
                 const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g) {
  using Cfg = ClusterCfg<N1, N2, C>;
  using RC = RowsCfg<N1, N2, C, SEPRECV>;
  constexpr int R = Cfg::R, N = Cfg::N, W1 = Cfg::W1, W2 = Cfg::W2, T1 = Cfg::T1, T2 = Cfg::T2;
  extern __shared__ __align__(128) float2 smem[];
  __shared__ uint64_t bars[2];
  float4* coarse = reinterpret_cast<float4*>(smem);
  float2* buf = smem + 2 * Cfg::NC;
  float2* recv = SEPRECV ? buf + RC::TILE : buf;

  const int p = (int)cluster_ctarank();
  const int64_t t = blockIdx.x / C;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
#if DPP_EXP == 2
    mbar_arrive_expect_tx(&bars[0], 0);
#else
    mbar_arrive_expect_tx(&bars[0], (uint32_t)(N1 * W1 * sizeof(float2)));
#endif
    mbar_arrive_expect_tx(&bars[1], (uint32_t)(N2 * W2 * sizeof(float2)));
#if DPP_EXP != 2
    tma_load_2d(buf, &tin, p * W1, (int)(t * N1), &bars[0]);
#endif
  }
  for (int e = tid; e < Cfg::NC; e += Cfg::THREADS) {
    const float2 w = coarse_g[e];
    coarse[e] = make_float4(w.x, w.y, -w.y, w.x);
  }
  __syncthreads();
  if constexpr (SEPRECV) cluster_arrive_relaxed();  // mbarriers initialised

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
#if DPP_EXP != 1
  block_fft<N1, R>(v, j, buf, MapRow{W1, col}, coarse, Cfg::NC / N1);
#endif
  if constexpr (!SEPRECV) cluster_arrive_relaxed();  // this CTA no longer reads buf
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
  if constexpr (!SEPRECV) __syncthreads();  // SEPRECV: pass 2 exchanges in buf, free since pass 1
#if DPP_EXP != 1
  block_fft<N2, R>(v, j2, buf, MapRow{W2, cl}, coarse, Cfg::NC / N2);
#endif
  float2* dst = out + t * N + p * W2 + cl;
#if DPP_EXP == 2
  if (v[0].x != 1234.5f) return;
#endif
#pragma unroll
  for (int i = 0; i < R; ++i) __stcs(dst + (int64_t)(j2 + T2 * i) * N1, v[i]);
}

template <int N1, int N2, int C, bool SEPRECV>
static int prepare_rows() {
  auto kern = fft_cluster_rows<N1, N2, C, SEPRECV>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)RowsCfg<N1, N2, C, SEPRECV>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int N1, int N2, int C, bool SEPRECV>
static int launch_rows(const float2* in, float2* out, int64_t batch, const float2* coarse, const float2* fine,
                       cudaStream_t s) {
  using Cfg = ClusterCfg<N1, N2, C>;
  CUtensorMap tmap;
  int rc = make_tmap_c64(&tmap, in, (uint64_t)batch * N1, N2, N1, Cfg::W1);
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * C), 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = RowsCfg<N1, N2, C, SEPRECV>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_cluster_rows<N1, N2, C, SEPRECV>, tmap, out, coarse, fine));
  return DPP_OK;
}

// ---------------------------------------------------------------------------
// MODE 7 (2^16 = 256 x 256, 16-CTA clusters): warp-local passes.
//
// Each warp owns two whole columns of the CTA's 256 x 16 tile: lane l of warp
// w works on column 2w + ((l >> 3) & 1) with j = (l & 7) | ((l >> 4) << 3), so
// a column's 16 threads sit in one warp and both Stockham exchanges of a
// 256-point pass need only __syncwarp (no CTA barrier), while each half-warp
// covers 8 rows x 2 columns.  One 32 KB buffer per CTA carries everything and
// a warp only ever touches its own columns' slots:
//   TMA tile load (128B-swizzled [row][16 cols]) -> pass 1 in place ->
//   st.async scatter into the peers' buffers ([b][16 cl], same swizzle) ->
//   pass 2 in place -> output tile staged in place -> one TMA tile store.
// Slot (row r, column c) = float2 16r + 2((c/2) ^ (r&7)) + (c&1).  Every
// access pattern below gives a half-warp 8 distinct r&7 x 2 column parities =
// 16 distinct 8-byte bank pairs (conflict-free, 2 wavefronts per warp):
//   rows j + 16i (tile read, output staging): r&7 = j&7;
//   pass-2 receive rows rho(b) = b ^ ((b&1) << 2), which also keeps the two
//   sending columns (b even/odd) on disjoint chunks at the receiver;
//   exchange rows xr(e) = 16(e/16) + ((e%16) ^ ((e/16)&7)) for both the write
//   (e = 16j + i) and the read (e = j + 16i): r&7 = (i ^ j)&7.
// For the exchange the slot is ((per-thread base) ^ 18(i&7)) + const(i), so
// each access costs one LOP3 (the XOR lands on bits the base keeps clear).
// Stage twiddles W_256^{ij}: a [j][i ^ (j&7)] float4 (w, i*w) table.
// SEP: separate receive buffer (no buffer-free cluster barrier, 3 CTAs/SM).
#ifdef DPP_PHASES
// profiling build only: per-CTA clock64 stamps of the MODE 7 phases
__device__ long long g_phase[65536 * 12];
extern "C" int dpp_debug_phases(long long* host, long long n) {
  return cudaMemcpyFromSymbol(host, g_phase, (size_t)n * sizeof(long long)) == cudaSuccess ? 0 : 2;
}
#define PHASE(k) \
  if (threadIdx.x == 0 && blockIdx.x < 65536) g_phase[blockIdx.x * 12 + (k)] = clock64();
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
#define PHASE_EXTRA(k, v) \
  if (threadIdx.x == 0 && blockIdx.x < 65536) g_phase[blockIdx.x * 12 + (k)] = (v);
#else
#define PHASE(k)
#define PHASE_EXTRA(k, v)
#endif

namespace w16 {
constexpr int N1 = 256, N2 = 256, W = 16, R = 16;
constexpr int TILE = N1 * W;  // one 256 x 16 sub-tile: 4096 float2 = 32 KB
// cluster of CC CTAs: each CTA holds SUB = 16/CC sub-tiles (8 warps each)
template <int CC>
struct Shape {
  static constexpr int SUB = 16 / CC, THREADS = 256 * SUB, W2 = 16 * SUB;
  static constexpr int MINB = CC == 16 ? 4 : 2;
};
template <int CC, bool SEP>
constexpr size_t smem_bytes() { return 1024 + (size_t)(SEP ? 2 : 1) * Shape<CC>::SUB * TILE * 8 + 256 * 16; }
__device__ __forceinline__ uint32_t slot(int r, int c) {
  return (uint32_t)(r * 16 + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1));
}
__device__ __forceinline__ float2 lds2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts2(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
}

// Per-thread shared-memory bases (bytes) of one 1024-aligned tile buffer.
struct Lane {
  uint32_t row;  // rows j + 16i: + 2048 i
  uint32_t xw;   // exchange write e = 16j + i: (xw ^ 144(i&7)) + 1024 (i>>3)
  uint32_t xq;   // exchange read  e = j + 16i: (xq ^ 144(i&7)) + 2048 i
  __device__ __forceinline__ Lane(uint32_t buf, int w, int par, int j) {
    const int j7 = j & 7;
    const uint32_t z = (uint32_t)(18 * j7 ^ 2 * w);
    row = buf + 8u * (uint32_t)(16 * j + 2 * (w ^ j7) + par);
    xw = buf + 8u * ((uint32_t)(256 * j + par) | z);
    xq = buf + 8u * ((uint32_t)(16 * (j & 8) + par) | z);
  }
};

// 256-point Stockham transform of one column held as v[i] = x[j + 16 i]; on
// exit v[i] = X[j + 16 i].  The column's slots serve as the exchange scratch.
__device__ __forceinline__ void col256(float2 (&v)[R], const Lane& L, uint32_t twj, int j) {
  dft16(v);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < R; ++i) sts2((L.xw ^ (144u * (i & 7))) + 1024u * (i >> 3), v[i]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = lds2((L.xq ^ (144u * (i & 7))) + 2048u * i);
  (void)j;
#pragma unroll
  for (int i = 1; i < R; ++i) v[i] = twmul(v[i], lds4((twj ^ (16u * (i & 7))) + 128u * (i >> 3)));
  dft16(v);
}
}  // namespace w16

// PERSIST (MODE 9): ceil(batch / G) transforms per cluster, G = the
// co-resident cluster count (31 on B200: a 16-CTA cluster needs 16 free slots
// in one GPC, so at most 3.35 of the 4 slots per SM hold CTAs; launching one
// cluster per transform averages 2.98, profiles/micro/phases.py).  The next
// tile's TMA load is issued once the previous output store has read the
// buffer.  Measured slower (1.64 vs 1.39 ms): without a second tile buffer
// the load latency is exposed every iteration and each cluster runs at the
// pace of its busiest SM.  Kept as a documented variant.
template <int CC, bool SEP, bool PERSIST>
__global__ void __launch_bounds__(w16::Shape<CC>::THREADS, SEP ? (CC == 16 ? 3 : 1) : w16::Shape<CC>::MINB)
fft_warp_65536(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
               const float2* __restrict__ coarse_g, const float2* __restrict__ fine_g, int64_t batch) {
  static_assert(!(SEP && PERSIST), "the separate-receive variant runs one transform per cluster");
  using namespace w16;
  constexpr int SUB = Shape<CC>::SUB;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bars[2];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  float2* buf = reinterpret_cast<float2*>(smem_raw + pad);
  float2* recv = SEP ? buf + SUB * TILE : buf;
  float4* tw = reinterpret_cast<float4*>(buf + (SEP ? 2 : 1) * SUB * TILE);

  const int p = (int)cluster_ctarank();
  const int64_t stride = PERSIST ? (int64_t)(gridDim.x / CC) : batch;
  int64_t t = blockIdx.x / CC;
  const int tid = threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const int sub = w >> 3, wl = w & 7;  // sub-tile and warp within it
  const int par = (lane >> 3) & 1, j = (lane & 7) | ((lane >> 4) << 3);
  const int col = 2 * wl + par;        // column within the sub-tile
  const uint32_t mybuf = smem_u32(buf) + (uint32_t)(sub * TILE * 8);
  const uint32_t myrecv = smem_u32(recv) + (uint32_t)(sub * TILE * 8);
  PHASE(0)
  PHASE_EXTRA(8, smid())
  PHASE_EXTRA(9, gtimer())
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if (t < batch) {
      mbar_arrive_expect_tx(&bars[0], (uint32_t)(SUB * TILE * 8));
#pragma unroll
      for (int s = 0; s < SUB; ++s) tma_load_2d(buf + s * TILE, &tin, (p * SUB + s) * W, (int)(t * N1), &bars[0]);
      mbar_arrive_expect_tx(&bars[1], (uint32_t)(SUB * TILE * 8));
    }
  }
  if (tid < 256) {
    // stage-twiddle table: entry [jj][ii ^ (jj & 7)] = W_256^{ii*jj} as (w, i*w)
    const int jj = tid >> 4, ii = tid & 15;
    const float2 x = __ldg(coarse_g + ((ii * jj) & 255));
    tw[jj * 16 + (ii ^ (jj & 7))] = make_float4(x.x, x.y, -x.y, x.x);
  }
  const int b = (p * SUB + sub) * W + col;
  // four-step twiddle W_N^{b (j + 16 i)} = W_N^{bj} (W_N^{16b})^i from the
  // coarse W_256 x fine W_N tables, fetched before the tile wait
  const float2 w0 = cmul(__ldg(coarse_g + ((b * j) >> 8)), __ldg(fine_g + ((b * j) & 255)));
  const float2 sw = cmul(__ldg(coarse_g + ((b * 16) >> 8)), __ldg(fine_g + ((b * 16) & 255)));
  const uint32_t twj = smem_u32(tw) + 256u * (uint32_t)j + 16u * (uint32_t)(j & 7);
  __syncthreads();
  if constexpr (SEP) cluster_arrive_relaxed();  // mbarriers initialised

  for (uint32_t k = 0; t < batch; t += stride, ++k) {
    const uint32_t ph = k & 1;
    float2 v[R];
    {
      const Lane L(mybuf, wl, par, j);
      mbar_wait(&bars[0], ph);
      PHASE(1)
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = lds2(L.row + 2048u * i);
      col256(v, L, twj, j);
    }
    PHASE(2)
    if constexpr (!SEP) cluster_arrive_relaxed();  // this CTA no longer reads buf
    {
      float2 x = w0;
      // opaque per iteration: otherwise the 16 loop-invariant twiddles are
      // hoisted out of the persistent loop and spilled
      asm volatile("" : "+f"(x.x), "+f"(x.y));
#pragma unroll
      for (int i = 0; i < R; ++i) {
        v[i] = cmul(v[i], x);
        x = cmul(x, sw);
      }
    }
    cluster_wait();
    PHASE(3)
    {
      // Z[b][c = j + 16 i] belongs to CTA i / SUB, sub-tile i % SUB, column j, row rho(b)
      const int rb = b ^ ((b & 1) << 2);
      const uint32_t scatter_off = smem_u32(recv) + 8u * slot(rb, j);
      const uint32_t rbar = smem_u32(&bars[1]);
#pragma unroll
      for (int i = 0; i < R; ++i)
        st_async_f2(mapa_u32(scatter_off + (uint32_t)((i % SUB) * TILE * 8), i / SUB), v[i],
                    mapa_u32(rbar, i / SUB));
    }
    // pass 2: column c = W2 p + 16 sub + col over b = j + 16 i (received at row rho(b))
    const Lane L(myrecv, wl, par, j);
    PHASE(4)
    const int jr = j ^ ((j & 1) << 2);
    const uint32_t rrow = myrecv + 8u * (uint32_t)(16 * jr + 2 * (wl ^ (jr & 7)) + par);
    mbar_wait(&bars[1], ph);
    PHASE(5)
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = lds2(rrow + 2048u * i);
    col256(v, L, twj, j);
    PHASE(6)
    // X[c + 256 k2], k2 = j + 16 i: staged at row k2, column col; TMA tile stores
    __syncwarp();
#pragma unroll
    for (int i = 0; i < R; ++i) sts2(L.row + 2048u * i, v[i]);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < SUB; ++s) tma_store_2d(&tout, (p * SUB + s) * W, (int)(t * N2), recv + s * TILE);
      bulk_commit_and_wait_all();
      const int64_t tn = t + stride;
      if (tn < batch) {
        mbar_arrive_expect_tx(&bars[0], (uint32_t)(SUB * TILE * 8));
#pragma unroll
        for (int s = 0; s < SUB; ++s) tma_load_2d(buf + s * TILE, &tin, (p * SUB + s) * W, (int)(tn * N1), &bars[0]);
        mbar_arrive_expect_tx(&bars[1], (uint32_t)(SUB * TILE * 8));
      }
      PHASE(7)
      PHASE_EXTRA(10, gtimer())
    }
  }
}

template <int CC, bool SEP, bool PERSIST>
static int prepare_warp65536(int* max_clusters) {
  auto kern = fft_warp_65536<CC, SEP, PERSIST>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)w16::smem_bytes<CC, SEP>()));
  if (CC > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  *max_clusters = 0;
  if (PERSIST) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CC * 1024, 1, 1);
    cfg.blockDim = dim3(w16::Shape<CC>::THREADS, 1, 1);
    cfg.dynamicSmemBytes = w16::smem_bytes<CC, SEP>();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DPP_CUDA_CHECK(cudaOccupancyMaxActiveClusters(max_clusters, kern, &cfg));
    if (*max_clusters < 1) return fail(DPP_ECUDA, "no cluster of the 2^16 kernel fits on this device");
  }
  return DPP_OK;
}

template <int CC, bool SEP, bool PERSIST>
static int launch_warp65536(const float2* in, float2* out, int64_t batch, const float2* coarse, const float2* fine,
                            int max_clusters, cudaStream_t s) {
  using namespace w16;
  CUtensorMap tin, tout;
  int rc = make_tmap_c64(&tin, in, (uint64_t)batch * N1, N2, N1, W, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_c64(&tout, out, (uint64_t)batch * N2, N1, N2, W, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int64_t clusters = PERSIST ? (batch < max_clusters ? batch : max_clusters) : batch;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * CC), 1, 1);
  cfg.blockDim = dim3(Shape<CC>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem_bytes<CC, SEP>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_warp_65536<CC, SEP, PERSIST>, tin, tout, coarse, fine, batch));
  return DPP_OK;
}

template <int N1, int N2, int C>
static int prepare_pair() {
  auto kern = fft_cluster_pair<N1, N2, C>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)PairCfg<N1, N2, C>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int N1, int N2, int C>
static int launch_pair(const float2* in, float2* out, int64_t batch, const float2* coarse, const float2* fine,
                       cudaStream_t s) {
  using Cfg = PairCfg<N1, N2, C>;
  CUtensorMap tmap;
  int rc = make_tmap_c64(&tmap, in, (uint64_t)batch * N1, N2, N1, Cfg::W1);
  if (rc) return rc;
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
  DPP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fft_cluster_pair<N1, N2, C>, tmap, out, coarse, fine));
  return DPP_OK;
}

static int g_cluster_mode = -1;  // DPP_FFT_CLUSTER_MODE=0..4 selects the exchange variant (default 4)

static int cluster_mode() {
  if (g_cluster_mode < 0) {
    const char* e = getenv("DPP_FFT_CLUSTER_MODE");
    g_cluster_mode = e ? (e[0] - '0') : 5;
    if (g_cluster_mode < 0 || g_cluster_mode > 9) g_cluster_mode = 5;
  }
  return g_cluster_mode;
}

template <int N1, int N2, int C, int MODE>
static int prepare_cluster_mode() {
  auto kern = fft_cluster_kernel<N1, N2, C, MODE>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ClusterCfg<N1, N2, C>::SMEM));
  if (C > 8) DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DPP_OK;
}

template <int N1, int N2, int C>
static int prepare_cluster(FftPlan* p) {
  p->mode = cluster_mode();
  // MODE 7-9: the warp-local 2^16 kernel (other sizes use MODE 5)
  if (p->mode >= 7 && !(N1 == 256 && N2 == 256 && (C == 16 || C == 8))) p->mode = 5;
  if constexpr (N1 == 256 && N2 == 256 && (C == 16 || C == 8)) {
    if (p->mode == 7) return prepare_warp65536<C, false, false>(&p->max_clusters);
    if (p->mode == 8) return prepare_warp65536<C, true, false>(&p->max_clusters);
    if (p->mode == 9) return prepare_warp65536<C, false, true>(&p->max_clusters);
  }
  switch (p->mode) {
    case 0: return prepare_cluster_mode<N1, N2, C, 0>();
    case 1: return prepare_cluster_mode<N1, N2, C, 1>();
    case 2: return prepare_cluster_mode<N1, N2, C, 2>();
    case 3: return prepare_persistent<N1, N2, C>(&p->max_clusters);
    case 5: return prepare_rows<N1, N2, C, false>();
    case 6: return prepare_rows<N1, N2, C, true>();
    default: return prepare_pair<N1, N2, C>();
  }
}

template <int N1, int N2, int C>
static int launch_cluster(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  using Cfg = ClusterCfg<N1, N2, C>;
  const float2* coarse = p->tw_a;
  const float2* fine = p->tw_b;
  if (p->mode == 3) return launch_persistent<N1, N2, C>(in, out, batch, coarse, fine, p->max_clusters, s);
  if (p->mode == 4) return launch_pair<N1, N2, C>(in, out, batch, coarse, fine, s);
  if (p->mode == 5) return launch_rows<N1, N2, C, false>(in, out, batch, coarse, fine, s);
  if (p->mode == 6) return launch_rows<N1, N2, C, true>(in, out, batch, coarse, fine, s);
  if constexpr (N1 == 256 && N2 == 256 && (C == 16 || C == 8)) {
    if (p->mode == 7) return launch_warp65536<C, false, false>(in, out, batch, coarse, fine, 0, s);
    if (p->mode == 8) return launch_warp65536<C, true, false>(in, out, batch, coarse, fine, 0, s);
    if (p->mode == 9) return launch_warp65536<C, false, true>(in, out, batch, coarse, fine, p->max_clusters, s);
  }
  auto kern = p->mode == 0   ? fft_cluster_kernel<N1, N2, C, 0>
              : p->mode == 1 ? fft_cluster_kernel<N1, N2, C, 1>
                             : fft_cluster_kernel<N1, N2, C, 2>;
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
  // 2048 and 4096 go through the TMA/row-layout kernel with a 1-CTA "cluster":
  // the generic small kernel ran 4096-point rows at 1.1 TB/s (C5 profile)
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
    const char* e = getenv("DPP_FFT_L2");
    if (!e || atoi(e) != 0) {
      p->kind = FftPlan::L2X;
      if (int rc = fft65536_l2x_init(p)) return rc;
      snprintf(p->desc, sizeof(p->desc),
               "two-pass 256x256 four-step, L2-resident exchange (ring %d, lag %d), 32 KB SMEM transpose per item",
               p->l2_ring, p->l2_lag);
      return DPP_OK;
    }
  }
  if (lg <= 17) {
    // split n = N1 * N2 with N1 <= N2, cluster C so that each CTA holds <= 8192 points
    p->kind = FftPlan::CLUSTER;
    p->n1a = 1LL << (lg / 2);
    p->n2a = n / p->n1a;
    p->cluster = (int)(n / 8192 > 1 ? n / 8192 : 1);
    if (n == 65536) {
      // 16 CTAs of 4096 points (4 CTAs = 32 warps per SM) beat 8 of 8192
      // (2 per SM): 1.34 vs 1.53 ms for 4096 x 2^16 (profiles/fft_c2_r1.md)
      const char* e = getenv("DPP_FFT_C65536");
      p->cluster = (e && atoi(e) == 8) ? 8 : 16;
    }
    int rc = DPP_OK;
    switch (n) {
      case 2048: rc = prepare_cluster<32, 64, 1>(p); break;
      case 4096: rc = prepare_cluster<64, 64, 1>(p); break;
      case 8192: rc = prepare_cluster<64, 128, 1>(p); break;
      case 16384: rc = prepare_cluster<128, 128, 2>(p); break;
      case 32768: rc = prepare_cluster<128, 256, 4>(p); break;
      case 65536:
        rc = p->cluster == 16 ? prepare_cluster<256, 256, 16>(p) : prepare_cluster<256, 256, 8>(p);
        break;
      case 131072: rc = prepare_cluster<256, 512, 16>(p); break;
    }
    if (rc) return rc;
    const int64_t nc = p->n1a > p->n2a ? p->n1a : p->n2a;
    if (upload_table(twiddle_table(nc, nc), &p->tw_a)) return DPP_ECUDA;
    if (upload_table(twiddle_table(n, n / nc), &p->tw_b)) return DPP_ECUDA;
    if (n == 4096) {
      const char* e = getenv("DPP_FFT_WS4K");
      if (!e || atoi(e) != 0) {
        if (int rc2 = fft4096_ws_init(p)) return rc2;
        p->ws4k = 1;
        snprintf(p->desc, sizeof(p->desc),
                 "256x16 in one CTA, warp-specialised TMA pipeline (2 stages, P1 warp-local, P2 in-thread)");
        return DPP_OK;
      }
    }
    if (n == 131072) {
      const char* e = getenv("DPP_FFT_L2");
      if (!e || atoi(e) != 0) {
        if (int rc2 = fft128k_l2_init(p)) return rc2;
        p->ring128k = 1;
        snprintf(p->desc, sizeof(p->desc),
                 "two-pass 256x512 four-step, L2-resident exchange (ring %d, lag %d), warp-wide 512-point P2",
                 p->l2_ring, p->l2_lag);
        return DPP_OK;
      }
    }
    if (n == 8192 || n == 16384 || n == 32768) {
      const char* e = getenv("DPP_FFT_L2");
      if (!e || atoi(e) != 0) {
        if (int rc2 = fft16k_l2_init(p)) return rc2;
        p->ring16k = 1;
        snprintf(p->desc, sizeof(p->desc),
                 "two-pass 256x%lld four-step, L2-resident exchange (ring %d, lag %d), units of %lld transforms",
                 (long long)(n / 256), p->l2_ring, p->l2_lag, (long long)(65536 / n));
        return DPP_OK;
      }
    }
    static const char* modes[10] = {"push", "pull", "async", "persistent TMA + st.async",
                                    "column pairs, TMA tile + st.async", "row layouts, TMA tile + st.async",
                                    "row layouts, separate receive buffer",
                                    "warp-local passes, swizzled TMA tile in/out",
                                    "warp-local passes, separate receive buffer",
                                    "warp-local passes, persistent clusters"};
    snprintf(p->desc, sizeof(p->desc), "cluster<%lldx%lld, C=%d> four-step over DSMEM (%s%s)",
             (long long)p->n1a, (long long)p->n2a, p->cluster, modes[p->mode],
             (p->mode == 3 || p->mode == 9) ? (std::string(", ") + std::to_string(p->max_clusters) + " clusters").c_str() : "");
    return DPP_OK;
  }
  if (n == 262144 || n == 524288 || n == 1048576) {
    const char* e = getenv("DPP_FFT_L2");
    if (!e || atoi(e) != 0) {
      p->kind = FftPlan::CLUSTER;
      if (int rc = fft128k_l2_init(p)) return rc;
      p->ring128k = 1;
      snprintf(p->desc, sizeof(p->desc),
               "two-pass %lldx%lld four-step, L2-resident exchange (ring %d, lag %d), warp-wide 512-point FFTs",
               (long long)(n <= 524288 ? 512 : 1024), (long long)(n <= 524288 ? n / 512 : 1024), p->l2_ring,
               p->l2_lag);
      return DPP_OK;
    }
  }
  return fft_large_init(p);
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
    switch (p->n0) {
      case 2048: return launch_cluster<32, 64, 1>(p, in, out, batch, s);
      case 4096: return launch_cluster<64, 64, 1>(p, in, out, batch, s);
      case 8192: return launch_cluster<64, 128, 1>(p, in, out, batch, s);
      case 16384: return launch_cluster<128, 128, 2>(p, in, out, batch, s);
      case 32768: return launch_cluster<128, 256, 4>(p, in, out, batch, s);
      case 65536:
        return p->cluster == 16 ? launch_cluster<256, 256, 16>(p, in, out, batch, s)
                                : launch_cluster<256, 256, 8>(p, in, out, batch, s);
      case 131072: return launch_cluster<256, 512, 16>(p, in, out, batch, s);
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
