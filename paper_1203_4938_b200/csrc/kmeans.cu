// GPU k-means codebook trainer following the reference
// algorithm /root/reference/pkg/src/dpp/apps/imgc.py:221-273:
//   k-means++ seeding driven by the caller's RNG stream (first pick index and
//   one uniform per further centroid, as numpy's Generator.choice consumes
//   them), then <= max_iter Lloyd iterations (assign to nearest centroid,
//   centroid = member mean, empty cluster -> farthest point from its assigned
//   centroid, stop when assignments repeat), binary64 throughout.
// Parity with the host trainer is tolerance-based (the reference's GEMM-based
// distances and sequential cumsum are CPU/BLAS dependent), see tests.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace dpp {

constexpr int KD = 16;  // block vectors are 16-dim

// The trainer keeps its points as structure of arrays, coordinate m of point
// i at soa[m n + i]: a warp's loads of one coordinate are 256 contiguous
// bytes (the caller's (n, 16) rows made every per-thread load a 128-byte
// stride: the k-means++ pass ran at a third of HBM bandwidth).
// (also the binary32 rows the tensor-core Lloyd assignment searches with)
__global__ void __launch_bounds__(256) to_soa(const double* __restrict__ pts, int64_t n, double* __restrict__ soa,
                                              float* __restrict__ rows32) {
  __shared__ double t[16][257];
  const int64_t i0 = (int64_t)blockIdx.x * 256;
  for (int e = threadIdx.x; e < 256 * KD; e += 256) {  // coalesced row-major read
    const int64_t r = i0 + e / KD;
    const double v = r < n ? pts[i0 * KD + e] : 0.0;
    t[e % KD][e / KD] = v;
    if (r < n) rows32[i0 * KD + e] = (float)v;
  }
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  if (i < n)
#pragma unroll
    for (int m = 0; m < KD; ++m) soa[m * n + i] = t[m][threadIdx.x];
}

__device__ __forceinline__ double dist2_soa(const double* __restrict__ soa, int64_t n, int64_t i,
                                            const double* c) {
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < KD; ++m) {
    const double d = soa[m * n + i] - c[m];
    s = fma(d, d, s);
  }
  return s;
}

// d2[i] = min(d2[i], |p_i - c|^2) (or init when first); per-block partial sums
__global__ void kpp_update(const double* __restrict__ pts, int64_t n, const double* __restrict__ c,
                           double* __restrict__ d2, double* __restrict__ block_sums, int first) {
  __shared__ double cs[KD];
  __shared__ double red[32];
  if (threadIdx.x < KD) cs[threadIdx.x] = c[threadIdx.x];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    const double d = dist2_soa(pts, n, i, cs);
    v = first ? d : fmin(d2[i], d);
    d2[i] = v;
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
  }
}

// k-means++ draw, one CTA of PICK_T threads (log-depth; a single thread walking
// the 16k block sums of a 4M-point frame took milliseconds per draw):
//   total = sum of the block sums, target = u * total (or the caller's target);
//   block = the first whose inclusive prefix exceeds target (else the last),
//   pick  = the first point of that block whose inclusive prefix exceeds target
//           (else the block's last point) — numpy's searchsorted(cdf, u, 'right')
//           as imgc.py:241-248 draws it, over d2 in index order.
constexpr int PICK_T = 1024;

// inclusive CTA-wide scan of one double per thread; *total = the CTA sum
__device__ double cta_scan_incl(double v, double* ws, double* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) ws[w] = v;
  __syncthreads();
  if (w == 0) {
    double s = lane < nw ? ws[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    ws[lane] = s;
  }
  __syncthreads();
  if (w > 0) v += ws[w - 1];
  *total = ws[nw - 1];
  __syncthreads();
  return v;
}

// USE_U: target = u * total (degenerate total <= 0: uniform pick u * n);
// otherwise `val` is the target itself (shard-local draw)
template <bool USE_U>
__global__ void __launch_bounds__(PICK_T) kpp_pick(const double* __restrict__ d2, int64_t n,
                                                   const double* __restrict__ block_sums, int nblocks, int block,
                                                   double val, const double* __restrict__ pts,
                                                   double* __restrict__ centroid, int64_t* __restrict__ pick_out) {
  __shared__ double ws[32];
  __shared__ int first_t;
  __shared__ int blk_s;
  __shared__ int64_t pick_s;
  __shared__ double acc_s;
  const int tid = threadIdx.x;
  const int per = (nblocks + PICK_T - 1) / PICK_T;
  const int b0 = min(nblocks, tid * per), b1 = min(nblocks, b0 + per);
  double loc = 0.0;
  for (int b = b0; b < b1; ++b) loc += block_sums[b];
  double total;
  const double incl = cta_scan_incl(loc, ws, &total);
  if (tid == 0) {
    first_t = PICK_T;
    pick_s = -1;
  }
  __syncthreads();
  double target = val;
  if (USE_U) {
    if (total <= 0.0) {
      if (tid == 0) {
        int64_t pk = (int64_t)(val * (double)n);
        pick_s = pk < n ? pk : n - 1;
      }
      __syncthreads();
      goto copy;
    }
    target = val * total;
  }
  // the first block whose prefix exceeds target lies in the first such thread's range
  if (b1 > b0 && (incl > target || b1 == nblocks)) atomicMin(&first_t, tid);
  __syncthreads();
  if (tid == first_t) {
    double acc = incl - loc;
    int b = b0;
    for (; b < b1 - 1; ++b) {
      if (acc + block_sums[b] > target) break;
      acc += block_sums[b];
    }
    blk_s = b;
    acc_s = acc;
  }
  __syncthreads();
  {
    const int64_t lo = (int64_t)blk_s * block, hi = lo + block < n ? lo + block : n;
    const double v = tid < hi - lo ? d2[lo + tid] : 0.0;
    double unused;
    const double pin = acc_s + cta_scan_incl(v, ws, &unused);
    if (tid == 0) first_t = PICK_T;
    __syncthreads();
    if (tid < hi - lo && pin > target) atomicMin(&first_t, tid);
    __syncthreads();
    if (tid == 0) pick_s = first_t < PICK_T ? lo + first_t : hi - 1;
    __syncthreads();
  }
copy:
  if (tid == 0) *pick_out = pick_s;
  if (tid < KD) centroid[tid] = pts[tid * n + pick_s];
}

// total of the block sums (the shard's d2 total for the all-reduce)
__global__ void __launch_bounds__(PICK_T) kpp_total(const double* __restrict__ block_sums, int nblocks,
                                                    double* __restrict__ total) {
  __shared__ double ws[32];
  const int per = (nblocks + PICK_T - 1) / PICK_T;
  const int b0 = min(nblocks, (int)threadIdx.x * per), b1 = min(nblocks, b0 + per);
  double loc = 0.0;
  for (int b = b0; b < b1; ++b) loc += block_sums[b];
  double t;
  cta_scan_incl(loc, ws, &t);
  if (threadIdx.x == 0) *total = t;
}

// shard accumulator for the all-reduce: [k*16 sums][k counts][changed][sse] in binary64
__global__ void pack_acc(const double* __restrict__ sums, const unsigned long long* __restrict__ counts,
                         const unsigned long long* __restrict__ changed, const double* __restrict__ sse, int k,
                         double* __restrict__ acc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * KD) acc[e] = sums[e];
  else if (e < k * KD + k) acc[e] = (double)counts[e - k * KD];
  else if (e == k * KD + k) acc[e] = (double)*changed;
  else if (e == k * KD + k + 1) acc[e] = *sse;
}

int vq_assign_tc(const float* vecs, int64_t n, const float* cents, int k, uint8_t* idx, cudaStream_t s);

// binary64 centroids -> the binary32 codebook of the tensor-core search
__global__ void cents_to_f32(const double* __restrict__ c, int k, float* __restrict__ c32) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * KD) c32[e] = (float)c[e];
}

// Lloyd update after the assignment: the nearest centroid of every point
// comes from the encoder's tensor-core search (vq_assign_tc: binary16-split scores
// on tcgen05, exact binary32 re-check of near ties, strict <, first index —
// SURVEY §8(f) row 2's "GEMM distances on tensor cores"); this pass counts
// changed assignments, adds the binary64 distance to the chosen centroid
// (the reference's trace formula) and accumulates binary64 per-cluster sums
// and counts in shared memory, flushed once per persistent block.
constexpr int PPT = 2;
__global__ void __launch_bounds__(256) lloyd_assign(const double* __restrict__ pts, int64_t n,
                                                    const double* __restrict__ cents, int k,
                                                    const uint8_t* __restrict__ nearest,
                                                    int32_t* __restrict__ assign, double* __restrict__ sums,
                                                    unsigned long long* __restrict__ counts,
                                                    unsigned long long* __restrict__ changed,
                                                    double* __restrict__ sse) {
  extern __shared__ __align__(16) double sh[];
  double* sc = sh;                  // k * KD centroids
  double* ssum = sh + k * KD;       // k * KD partial sums
  unsigned int* scnt = reinterpret_cast<unsigned int*>(ssum + k * KD);
  for (int e = threadIdx.x; e < k * KD; e += blockDim.x) {
    sc[e] = cents[e];
    ssum[e] = 0.0;
  }
  for (int e = threadIdx.x; e < k; e += blockDim.x) scnt[e] = 0;
  __syncthreads();
  double local_sse = 0.0;
  unsigned nchanged = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = nearest[i];
    const double* c = sc + j * KD;
    double d = 0.0;
#pragma unroll
    for (int m = 0; m < KD; ++m) {
      const double p = pts[m * n + i];
      const double t = p - c[m];
      d = fma(t, t, d);
      atomicAdd(&ssum[j * KD + m], p);
    }
    local_sse += d;
    nchanged += assign[i] != j;
    assign[i] = j;
    atomicAdd(&scnt[j], 1u);
  }
  for (int o = 16; o > 0; o >>= 1) {
    local_sse += __shfl_xor_sync(0xffffffffu, local_sse, o);
    nchanged += __shfl_xor_sync(0xffffffffu, nchanged, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sse, local_sse);
    if (nchanged) atomicAdd(changed, (unsigned long long)nchanged);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * KD; e += blockDim.x)
    if (ssum[e] != 0.0) atomicAdd(&sums[e], ssum[e]);
  for (int e = threadIdx.x; e < k; e += blockDim.x)
    if (scnt[e]) atomicAdd(&counts[e], (unsigned long long)scnt[e]);
}

// one Lloyd assignment: binary32 codebook, tensor-core nearest centroid,
// binary64 update pass (shared by the single-GPU trainer and the shards)
static int lloyd_pass(const double* soa, const float* rows32, int64_t n, const double* cents, float* cents32, int k,
                      uint8_t* nearest, int32_t* assign, double* sums, unsigned long long* counts,
                      unsigned long long* changed, double* sse, cudaStream_t s);

// launch geometry and shared memory of lloyd_assign: at most the resident blocks
static inline int lloyd_blocks(int64_t n) {
  static int resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lloyd_assign, 256,
                                                      (size_t)256 * KD * 2 * sizeof(double) + 256 * 4) != cudaSuccess ||
        per < 1)
      per = 1;
    resident = per * sms;
  }
  const int64_t need = (n + 255) / 256;
  return (int)(need < resident ? need : resident);
}
static inline size_t lloyd_smem(int k) { return (size_t)k * KD * 2 * sizeof(double) + k * sizeof(unsigned int); }

__global__ void lloyd_means(double* __restrict__ cents, const double* __restrict__ sums,
                            const unsigned long long* __restrict__ counts, int k) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * KD && counts[e / KD]) cents[e] = sums[e] / (double)counts[e / KD];
}

// farthest point from its assigned centroid (for empty-cluster reseeding);
// `base` = global index of the shard's first point
__global__ void far_point(const double* __restrict__ pts, int64_t n, const double* __restrict__ cents,
                          const int32_t* __restrict__ assign, unsigned long long* __restrict__ best,
                          int64_t base = 0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = dist2_soa(pts, n, i, cents + (int64_t)assign[i] * KD);
  // pack (distance as f32 bits, inverted index): atomicMax picks the largest
  // distance and, among equal ones, the lowest index (np.argmax)
  atomicMax(best, ((unsigned long long)__float_as_uint((float)d) << 32) | (0xffffffffu - (uint32_t)(base + i)));
}

static int lloyd_pass(const double* soa, const float* rows32, int64_t n, const double* cents, float* cents32, int k,
                      uint8_t* nearest, int32_t* assign, double* sums, unsigned long long* counts,
                      unsigned long long* changed, double* sse, cudaStream_t s) {
  static int attr = 0;
  if (!attr) {
    DPP_CUDA_CHECK(cudaFuncSetAttribute(lloyd_assign, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)lloyd_smem(256)));
    attr = 1;
  }
  DPP_CUDA_CHECK(cudaMemsetAsync(sums, 0, (size_t)k * KD * sizeof(double), s));
  DPP_CUDA_CHECK(cudaMemsetAsync(counts, 0, k * sizeof(unsigned long long), s));
  DPP_CUDA_CHECK(cudaMemsetAsync(changed, 0, sizeof(unsigned long long), s));
  DPP_CUDA_CHECK(cudaMemsetAsync(sse, 0, sizeof(double), s));
  cents_to_f32<<<(k * KD + 255) / 256, 256, 0, s>>>(cents, k, cents32);
  if (int rc = vq_assign_tc(rows32, n, cents32, k, nearest, s)) return rc;
  lloyd_assign<<<lloyd_blocks(n), 256, lloyd_smem(k), s>>>(soa, n, cents, k, nearest, assign, sums, counts, changed,
                                                           sse);
  DPP_LAUNCH_CHECK("lloyd_assign");
  return DPP_OK;
}

// one shard of a row-sharded k-means (multi-GPU): the
// device buffers of the single-GPU trainer for this rank's points; the
// driver (paper_1203_4938_b200/kmeans.py, kmeans_sharded) combines shards
// with one all-reduce per seeding step / Lloyd iteration
struct KmShard {
  const double* pts = nullptr;  // the caller's (n, 16) rows
  double* soa = nullptr;        // the trainer's copy, coordinate-major
  float* rows32 = nullptr;      // binary32 rows for the tensor-core search
  float* cents32 = nullptr;
  uint8_t* nearest = nullptr;
  int64_t n = 0;
  int k = 0, nb = 0;
  cudaStream_t s = nullptr;
  double *d2 = nullptr, *bsum = nullptr, *sums = nullptr, *sse = nullptr, *total = nullptr;
  int32_t* assign = nullptr;
  unsigned long long *counts = nullptr, *changed = nullptr, *far = nullptr;
  int64_t* pick = nullptr;
  void release() {
    for (void* ptr : {(void*)soa, (void*)rows32, (void*)cents32, (void*)nearest, (void*)d2, (void*)bsum, (void*)sums, (void*)sse, (void*)total, (void*)assign,
                      (void*)counts, (void*)changed, (void*)far, (void*)pick})
      if (ptr) cudaFree(ptr);
  }
};

}  // namespace dpp

struct dpp_kmeans_shard {
  dpp::KmShard impl;
};

extern "C" {

int dpp_kmeans_shard_create(dpp_kmeans_shard** shard, const double* pts, int64_t n, int k, void* stream) {
  using namespace dpp;
  if (!shard) return fail(DPP_EINVAL, "NULL shard pointer");
  *shard = nullptr;
  if (n < 0 || n > 0x7fffffffLL) return fail(DPP_EINVAL, "shard of %lld points", (long long)n);
  if (k < 1 || k > 256) return fail(DPP_EINVAL, "codebook size must be in 1..256");
  auto* h = new dpp_kmeans_shard();
  KmShard& m = h->impl;
  m.pts = pts;
  m.n = n;
  m.k = k;
  m.nb = (int)((n + 255) / 256);
  m.s = static_cast<cudaStream_t>(stream);
  const size_t nn = (size_t)(n > 0 ? n : 1), nbb = (size_t)(m.nb > 0 ? m.nb : 1);
  bool ok = cudaMalloc(&m.soa, nn * KD * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&m.rows32, nn * KD * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&m.cents32, (size_t)k * KD * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&m.nearest, nn) == cudaSuccess &&
            cudaMalloc(&m.d2, nn * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&m.bsum, nbb * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&m.sums, (size_t)k * KD * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&m.sse, sizeof(double)) == cudaSuccess && cudaMalloc(&m.total, sizeof(double)) == cudaSuccess &&
            cudaMalloc(&m.assign, nn * sizeof(int32_t)) == cudaSuccess &&
            cudaMalloc(&m.counts, k * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&m.changed, sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&m.far, sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&m.pick, sizeof(int64_t)) == cudaSuccess;
  if (ok && n > 0) {
    to_soa<<<m.nb, 256, 0, m.s>>>(pts, n, m.soa, m.rows32);
    ok = cudaGetLastError() == cudaSuccess;
  }
  if (!ok || cudaMemsetAsync(m.assign, 0xff, nn * sizeof(int32_t), m.s) != cudaSuccess) {
    m.release();
    delete h;
    return fail(DPP_ECUDA, "k-means shard allocation failed");
  }
  *shard = h;
  return DPP_OK;
}

// k-means++ step on the shard: d2 = min(d2, |p - centroid|^2) (first: init);
// *total (host) = the shard's sum of d2 in block order
int dpp_kmeans_shard_seed(dpp_kmeans_shard* shard, const double* centroid, int first, double* total) {
  using namespace dpp;
  if (!shard || !centroid || !total) return fail(DPP_EINVAL, "NULL argument to dpp_kmeans_shard_seed");
  KmShard& m = shard->impl;
  if (m.n == 0) {
    *total = 0.0;
    return DPP_OK;
  }
  kpp_update<<<m.nb, 256, 0, m.s>>>(m.soa, m.n, centroid, m.d2, m.bsum, first);
  kpp_total<<<1, PICK_T, 0, m.s>>>(m.bsum, m.nb, m.total);
  DPP_LAUNCH_CHECK("k-means++ shard update");
  DPP_CUDA_CHECK(cudaMemcpyAsync(total, m.total, sizeof(double), cudaMemcpyDeviceToHost, m.s));
  DPP_CUDA_CHECK(cudaStreamSynchronize(m.s));
  return DPP_OK;
}

// the shard's pick for a local target (local_index < 0), or the given local
// index (degenerate all-zero d2: uniform pick); copies the point to
// centroid_out (device, 16 doubles) and returns the local index
int dpp_kmeans_shard_pick(dpp_kmeans_shard* shard, double target, int64_t local_index, double* centroid_out,
                          int64_t* picked) {
  using namespace dpp;
  if (!shard || !centroid_out || !picked) return fail(DPP_EINVAL, "NULL argument to dpp_kmeans_shard_pick");
  KmShard& m = shard->impl;
  if (m.n == 0) return fail(DPP_EINVAL, "pick from an empty shard");
  if (local_index >= 0) {
    if (local_index >= m.n) return fail(DPP_EINVAL, "local index %lld outside the shard", (long long)local_index);
    DPP_CUDA_CHECK(cudaMemcpyAsync(centroid_out, m.pts + local_index * KD, KD * sizeof(double),
                                   cudaMemcpyDeviceToDevice, m.s));
    *picked = local_index;
    return DPP_OK;
  }
  kpp_pick<false><<<1, PICK_T, 0, m.s>>>(m.d2, m.n, m.bsum, m.nb, 256, target, m.soa, centroid_out, m.pick);
  DPP_LAUNCH_CHECK("k-means++ shard pick");
  DPP_CUDA_CHECK(cudaMemcpyAsync(picked, m.pick, sizeof(int64_t), cudaMemcpyDeviceToHost, m.s));
  DPP_CUDA_CHECK(cudaStreamSynchronize(m.s));
  return DPP_OK;
}

// Lloyd assignment on the shard: acc (device, k*16 + k + 2 doubles) =
// [per-cluster coordinate sums][counts][assignments changed][sum of squared distances]
int dpp_kmeans_shard_assign(dpp_kmeans_shard* shard, const double* cents, double* acc) {
  using namespace dpp;
  if (!shard || !cents || !acc) return fail(DPP_EINVAL, "NULL argument to dpp_kmeans_shard_assign");
  KmShard& m = shard->impl;
  const int k = m.k;
  const int tot = k * KD + k + 2;
  if (m.n == 0) {
    DPP_CUDA_CHECK(cudaMemsetAsync(acc, 0, tot * sizeof(double), m.s));
    return DPP_OK;
  }
  if (int rc = lloyd_pass(m.soa, m.rows32, m.n, cents, m.cents32, k, m.nearest, m.assign, m.sums, m.counts,
                          m.changed, m.sse, m.s))
    return rc;
  pack_acc<<<(tot + 255) / 256, 256, 0, m.s>>>(m.sums, m.counts, m.changed, m.sse, k, acc);
  DPP_LAUNCH_CHECK("lloyd shard assign");
  return DPP_OK;
}

// farthest point of the shard from its assigned centroid, packed as in
// far_point with global indices (base = the shard's first global index);
// *packed (device int64) receives the shard maximum (0 for an empty shard)
int dpp_kmeans_shard_far(dpp_kmeans_shard* shard, const double* cents, int64_t base, int64_t* packed) {
  using namespace dpp;
  if (!shard || !cents || !packed) return fail(DPP_EINVAL, "NULL argument to dpp_kmeans_shard_far");
  KmShard& m = shard->impl;
  DPP_CUDA_CHECK(cudaMemsetAsync(packed, 0, sizeof(int64_t), m.s));
  if (m.n == 0) return DPP_OK;
  far_point<<<m.nb, 256, 0, m.s>>>(m.soa, m.n, cents, m.assign, reinterpret_cast<unsigned long long*>(packed), base);
  DPP_LAUNCH_CHECK("far point");
  return DPP_OK;
}

// an empty cluster reseeded at a point of this shard: the point joins it
int dpp_kmeans_shard_set_assign(dpp_kmeans_shard* shard, int64_t local_index, int cluster) {
  using namespace dpp;
  if (!shard || local_index < 0 || local_index >= shard->impl.n)
    return fail(DPP_EINVAL, "bad dpp_kmeans_shard_set_assign arguments");
  KmShard& m = shard->impl;
  int32_t c = cluster;
  DPP_CUDA_CHECK(cudaMemcpyAsync(m.assign + local_index, &c, sizeof(int32_t), cudaMemcpyHostToDevice, m.s));
  DPP_CUDA_CHECK(cudaStreamSynchronize(m.s));
  return DPP_OK;
}

void dpp_kmeans_shard_destroy(dpp_kmeans_shard* shard) {
  if (!shard) return;
  shard->impl.release();
  delete shard;
}

int dpp_kmeans(const double* pts, int64_t n, int k, int64_t first_pick, const double* uniforms, int max_iter,
               float* centroids_out, double* trace, int* iterations, void* stream) {
  using namespace dpp;
  auto s = static_cast<cudaStream_t>(stream);
  if (n < 1) return fail(DPP_EINVAL, "no blocks to cluster");
  if (k < 1 || k > 256) return fail(DPP_EINVAL, "codebook size must be in 1..256");
  if (k > n) return fail(DPP_EINVAL, "codebook size %d exceeds %lld training blocks", k, (long long)n);
  if (n > 0x7fffffffLL) return fail(DPP_EINVAL, "too many training blocks");
  const int T = 256;
  const int nb = (int)((n + T - 1) / T);
  double *soa = nullptr, *d2 = nullptr, *bsum = nullptr, *cents = nullptr, *sums = nullptr, *sse = nullptr;
  float *rows32 = nullptr, *cents32 = nullptr;
  uint8_t* nearest = nullptr;
  int32_t* assign = nullptr;
  unsigned long long *counts = nullptr, *changed = nullptr, *far = nullptr;
  int64_t* pick = nullptr;
  // every exit path (errors included) returns the scratch to the pool
  struct Release {
    std::vector<void*> ptrs;
    cudaStream_t s;
    ~Release() {
      for (void* ptr : ptrs)
        if (ptr) cudaFreeAsync(ptr, s);
    }
  } release{{}, s};
  auto alloc = [&](auto** ptr, size_t bytes) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, s);
    release.ptrs.push_back(*ptr);
    return e;
  };
  DPP_CUDA_CHECK(alloc(&soa, n * KD * sizeof(double)));
  DPP_CUDA_CHECK(alloc(&rows32, n * KD * sizeof(float)));
  DPP_CUDA_CHECK(alloc(&cents32, (size_t)k * KD * sizeof(float)));
  DPP_CUDA_CHECK(alloc(&nearest, (size_t)n));
  DPP_CUDA_CHECK(alloc(&d2, n * sizeof(double)));
  DPP_CUDA_CHECK(alloc(&bsum, nb * sizeof(double)));
  DPP_CUDA_CHECK(alloc(&cents, (size_t)k * KD * sizeof(double)));
  DPP_CUDA_CHECK(alloc(&sums, (size_t)k * KD * sizeof(double)));
  DPP_CUDA_CHECK(alloc(&sse, sizeof(double)));
  DPP_CUDA_CHECK(alloc(&assign, n * sizeof(int32_t)));
  DPP_CUDA_CHECK(alloc(&counts, k * sizeof(unsigned long long)));
  DPP_CUDA_CHECK(alloc(&changed, sizeof(unsigned long long)));
  DPP_CUDA_CHECK(alloc(&far, sizeof(unsigned long long)));
  DPP_CUDA_CHECK(alloc(&pick, sizeof(int64_t)));

  to_soa<<<nb, T, 0, s>>>(pts, n, soa, rows32);
  // k-means++ seeding
  DPP_CUDA_CHECK(cudaMemcpyAsync(cents, pts + first_pick * KD, KD * sizeof(double), cudaMemcpyDeviceToDevice, s));
  for (int j = 1; j < k; ++j) {
    kpp_update<<<nb, T, 0, s>>>(soa, n, cents + (j - 1) * KD, d2, bsum, j == 1);
    kpp_pick<true><<<1, PICK_T, 0, s>>>(d2, n, bsum, nb, T, uniforms[j - 1], soa, cents + j * KD, pick);
  }
  DPP_LAUNCH_CHECK("k-means++ seeding");

  // Lloyd
  DPP_CUDA_CHECK(cudaMemsetAsync(assign, 0xff, n * sizeof(int32_t), s));  // -1: every point "changes"
  std::vector<unsigned long long> hcounts(k);
  int it = 0;
  // first assignment
  auto assign_pass = [&](unsigned long long* h_changed, double* h_sse) -> int {
    if (int rc = lloyd_pass(soa, rows32, n, cents, cents32, k, nearest, assign, sums, counts, changed, sse, s))
      return rc;
    DPP_CUDA_CHECK(cudaMemcpyAsync(h_changed, changed, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    DPP_CUDA_CHECK(cudaMemcpyAsync(h_sse, sse, sizeof(double), cudaMemcpyDeviceToHost, s));
    DPP_CUDA_CHECK(cudaMemcpyAsync(hcounts.data(), counts, k * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    DPP_CUDA_CHECK(cudaStreamSynchronize(s));
    return DPP_OK;
  };
  unsigned long long h_changed = 0;
  double h_sse = 0.0;
  if (int rc = assign_pass(&h_changed, &h_sse)) return rc;
  for (; it < max_iter; ++it) {
    // centroid = member mean; empty cluster -> farthest point (in index order)
    lloyd_means<<<(k * KD + 255) / 256, 256, 0, s>>>(cents, sums, counts, k);
    for (int j = 0; j < k; ++j) {
      if (hcounts[j]) continue;
      DPP_CUDA_CHECK(cudaMemsetAsync(far, 0, sizeof(unsigned long long), s));
      far_point<<<nb, T, 0, s>>>(soa, n, cents, assign, far);
      unsigned long long hf = 0;
      DPP_CUDA_CHECK(cudaMemcpyAsync(&hf, far, sizeof(hf), cudaMemcpyDeviceToHost, s));
      DPP_CUDA_CHECK(cudaStreamSynchronize(s));
      const int32_t idx = (int32_t)(0xffffffffu - (uint32_t)(hf & 0xffffffffu));
      DPP_CUDA_CHECK(cudaMemcpyAsync(cents + (int64_t)j * KD, pts + (int64_t)idx * KD, KD * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
      DPP_CUDA_CHECK(cudaMemcpyAsync(assign + idx, &j, sizeof(int32_t), cudaMemcpyHostToDevice, s));
      DPP_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    if (int rc = assign_pass(&h_changed, &h_sse)) return rc;
    if (trace) trace[it] = h_sse;
    if (h_changed == 0) { ++it; break; }
  }
  if (iterations) *iterations = it;
  // binary64 -> binary32 centroids
  std::vector<double> hc((size_t)k * KD);
  DPP_CUDA_CHECK(cudaMemcpyAsync(hc.data(), cents, hc.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  DPP_CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<float> hf(hc.size());
  for (size_t e = 0; e < hc.size(); ++e) hf[e] = (float)hc[e];
  DPP_CUDA_CHECK(cudaMemcpyAsync(centroids_out, hf.data(), hf.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  DPP_CUDA_CHECK(cudaStreamSynchronize(s));
  return DPP_OK;
}

}  // extern "C"
