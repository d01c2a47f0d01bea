// Block-compression node for sm_100a (apps/imgc.py of the reference).
//
// Everything here is bit-exact with the reference on the same inputs: binary32
// arithmetic is written with __f*_rn intrinsics (no FMA contraction, left to
// right as the kernel-language bodies evaluate, kernel/interp.py:348-358), the
// block statistics use binary64 with numpy's 8-accumulator pairwise order for
// 16-wide reductions (r_m = a_m + a_{m+8}, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))),
// and quantisers use round-half-even rint before clipping (imgc.py:375, 400-401).
#include <cstdint>
#include <cstring>

#include <cuda_fp16.h>

#include "common.cuh"
#include "tma.cuh"

namespace dpp {

// BT.601 constants as the kernel bodies spell them (imgc.py:131-134); each
// literal parses to the same binary32 as the reference's float32(float(text)).
#define K_YR 0.299f
#define K_YG 0.587f
#define K_YB 0.114f
#define K_BR 0.168736f
#define K_BG 0.331264f
#define K_RG 0.418688f
#define K_RB 0.081312f

struct YCC {
  float y, cb, cr;
};

// imgc.py:132-134: yl = 0.299f*r + 0.587f*g + 0.114f*b;
// cb = 128 - 0.168736f*r - 0.331264f*g + 0.5f*b; cr = 128 + 0.5f*r - 0.418688f*g - 0.081312f*b
__device__ __forceinline__ YCC ycc(float r, float g, float b) {
  YCC o;
  o.y = __fadd_rn(__fadd_rn(__fmul_rn(K_YR, r), __fmul_rn(K_YG, g)), __fmul_rn(K_YB, b));
  o.cb = __fadd_rn(__fsub_rn(__fsub_rn(128.0f, __fmul_rn(K_BR, r)), __fmul_rn(K_BG, g)), __fmul_rn(0.5f, b));
  o.cr = __fsub_rn(__fsub_rn(__fadd_rn(128.0f, __fmul_rn(0.5f, r)), __fmul_rn(K_RG, g)), __fmul_rn(K_RB, b));
  return o;
}
__device__ __forceinline__ float luma(float r, float g, float b) {
  return __fadd_rn(__fadd_rn(__fmul_rn(K_YR, r), __fmul_rn(K_YG, g)), __fmul_rn(K_YB, b));
}

// numpy pairwise sum of 16 (binary32 / binary64)
__device__ __forceinline__ float pw16f(const float (&a)[16]) {
  float r[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) r[m] = __fadd_rn(a[m], a[m + 8]);
  return __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                   __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
}
__device__ __forceinline__ double pw16d(const double (&a)[16]) {
  double r[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) r[m] = __dadd_rn(a[m], a[m + 8]);
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

// clip(rint(x), 0, 255) -> u8 (numpy rint is round-half-even)
__device__ __forceinline__ uint8_t q8f(float x) { return (uint8_t)fminf(fmaxf(rintf(x), 0.f), 255.f); }
__device__ __forceinline__ uint8_t q8d(double x) { return (uint8_t)fmin(fmax(rint(x), 0.0), 255.0); }

// squared distance exactly as dot(d, d) of vq_program (imgc.py:176-177,
// interp.py:417-419): d = b - c in binary32, products, pairwise-16 sum.
__device__ __forceinline__ float vq_dist(const float (&b)[16], const float4* c) {
  float p[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 cv = c[q];
    float d0 = __fsub_rn(b[4 * q + 0], cv.x), d1 = __fsub_rn(b[4 * q + 1], cv.y);
    float d2 = __fsub_rn(b[4 * q + 2], cv.z), d3 = __fsub_rn(b[4 * q + 3], cv.w);
    p[4 * q + 0] = __fmul_rn(d0, d0);
    p[4 * q + 1] = __fmul_rn(d1, d1);
    p[4 * q + 2] = __fmul_rn(d2, d2);
    p[4 * q + 3] = __fmul_rn(d3, d3);
  }
  return pw16f(p);
}

// The same distance with sm_100 packed binary32 pairs (FADD2/FMUL2, each lane
// IEEE round-to-nearest, no contraction): bit-identical, 25 instead of 47 FP
// instructions.  Components are paired so that every pairwise step of the
// reduction is a lane-wise add: pair k of a vector is
//   k=0..3: (v0,v2) (v1,v3) (v4,v6) (v5,v7);  k=4..7: the same +8.
// Then R = P[k] + P[k+4] gives (r0,r2) (r1,r3) (r4,r6) (r5,r7),
// R0+R1 = (r0+r1, r2+r3), R2+R3 = (r4+r5, r6+r7), and two scalar adds finish
// ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)).
__device__ __forceinline__ int vq_pair_src(int k, int half) {  // component of pair k, lane half
  const int base = (k & 4) ? 8 : 0, kk = k & 3;
  return base + (kk >> 1) * 4 + (kk & 1) + half * 2;
}
__device__ __forceinline__ void vq_pack(const float (&v)[16], float2 (&pv)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) pv[k] = make_float2(v[vq_pair_src(k, 0)], v[vq_pair_src(k, 1)]);
}
__device__ __forceinline__ float vq_dist_pairs(const float2 (&b)[8], const float2* c) {
  float2 p[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float2 cv = c[k];
    const float2 d = __fadd2_rn(b[k], make_float2(-cv.x, -cv.y));
    p[k] = __fmul2_rn(d, d);
  }
  // NOTE: ptxas fuses an FMUL2 feeding an FADD2 into FFMA2 even for explicit
  // add.rn/mul.rn.f32x2 and -fmad=false (checked in SASS), which would break
  // bit-exactness; the reduction therefore stays scalar (FADD is never fused
  // with a packed multiply).  31 FP instructions per centroid instead of 47.
  const float r0 = __fadd_rn(p[0].x, p[4].x), r2 = __fadd_rn(p[0].y, p[4].y);
  const float r1 = __fadd_rn(p[1].x, p[5].x), r3 = __fadd_rn(p[1].y, p[5].y);
  const float r4 = __fadd_rn(p[2].x, p[6].x), r6 = __fadd_rn(p[2].y, p[6].y);
  const float r5 = __fadd_rn(p[3].x, p[7].x), r7 = __fadd_rn(p[3].y, p[7].y);
  return __fadd_rn(__fadd_rn(__fadd_rn(r0, r1), __fadd_rn(r2, r3)), __fadd_rn(__fadd_rn(r4, r5), __fadd_rn(r6, r7)));
}
// codebook -> shared memory in pair order (8 float2 per centroid)
__device__ __forceinline__ void vq_stage_codebook(const float* cbk, int ncb, float2* s) {
  for (int e = threadIdx.x; e < ncb * 8; e += blockDim.x) {
    const int j = e >> 3, k = e & 7;
    s[e] = make_float2(cbk[j * 16 + vq_pair_src(k, 0)], cbk[j * 16 + vq_pair_src(k, 1)]);
  }
}

// "float best = 3.402823e38f" (imgc.py:173) parses to 0x7f7ffffd, not FLT_MAX
#define VQ_BEST_INIT __int_as_float(0x7f7ffffd)

// ---------------------------------------------------------------------------
// drop-in nodes

__global__ void ycbcr_kernel(const uchar4* __restrict__ rgba, float* __restrict__ yl,
                             float* __restrict__ cb, float* __restrict__ cr, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uchar4 p = rgba[i];
  const YCC o = ycc((float)p.x, (float)p.y, (float)p.z);
  yl[i] = o.y;
  cb[i] = o.cb;
  cr[i] = o.cr;
}

// avg[i] = (b.s0 + b.s1 + ... + b.sf) * 0.0625f  (imgc.py:143-148), sequential sum
__global__ void boxdown_kernel(const float4* __restrict__ blk, float* __restrict__ avg, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 v = blk[4 * i + q];
    acc = q == 0 ? v.x : __fadd_rn(acc, v.x);
    acc = __fadd_rn(acc, v.y);
    acc = __fadd_rn(acc, v.z);
    acc = __fadd_rn(acc, v.w);
  }
  avg[i] = __fmul_rn(acc, 0.0625f);
}

// gradient_program(width, height), imgc.py:155-166.  fault[0] collects the
// first work-item whose dx read leaves the chunk, fault[1] the same for dy.
__global__ void gradient_kernel(const float* __restrict__ lum, float* __restrict__ dx,
                                float* __restrict__ dy, int64_t width, int64_t height,
                                int64_t n, unsigned long long* fault) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t x = i % width, y = i / width;
  const float li = lum[i];
  float vx = 0.f, vy = 0.f;
  if (x < width - 1) {
    if (i + 1 < n) vx = __fsub_rn(lum[i + 1], li);
    else if (fault) atomicMin(&fault[0], (unsigned long long)i);
  }
  if (y < height - 1) {
    if (i + width < n) vy = __fsub_rn(lum[i + width], li);
    else if (fault) atomicMin(&fault[1], (unsigned long long)i);
  }
  dx[i] = vx;
  dy[i] = vy;
}

// vq_program(codebook_size), imgc.py:169-185: the chunk's cbk stream holds the
// codebook (tiled per chunk by the reference host, imgc.py:419).
__global__ void vqnearest_kernel(const float* __restrict__ blk, const float* __restrict__ cbk,
                                 int32_t* __restrict__ idx, int64_t n, int ncb) {
  extern __shared__ float2 scp[];
  vq_stage_codebook(cbk, ncb, scp);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float b[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 v = reinterpret_cast<const float4*>(blk)[4 * i + q];
    b[4 * q] = v.x; b[4 * q + 1] = v.y; b[4 * q + 2] = v.z; b[4 * q + 3] = v.w;
  }
  float2 bp[8];
  vq_pack(b, bp);
  float best = VQ_BEST_INIT;
  int bj = 0;
  for (int j = 0; j < ncb; ++j) {
    const float d = vq_dist_pairs(bp, scp + 8 * j);
    if (d < best) { best = d; bj = j; }
  }
  idx[i] = bj;
}

// ---------------------------------------------------------------------------
// fused encoder: one thread per 4x4 block

struct EncodeArgs {
  const uint8_t* px;
  int64_t height, width, row_stride, image_stride;
  const float* codebook;
  int ncb;
  int64_t codebook_stride;
  double sigma_min;
  uint8_t* records;
  uint8_t* cb_plane;
  uint8_t* cr_plane;
  float* block_grad;
  float* norm32;
  double* norm64;  // STATS variant only
  // planar records (graph node outputs mu / sig / idx): when set, the
  // tensor-core encoder writes the three record bytes to these planes
  // instead of the interleaved `records` run
  uint8_t* mu_plane;
  uint8_t* sig_plane;
  uint8_t* idx_plane;
  // CH = 0 (the k-means trainer's Lloyd assignment, csrc/kmeans.cu): the
  // blocks are given as normalised binary32 16-vectors, vecs[k][16], and only
  // idx_plane is written
  const float* vecs = nullptr;
  // CH = 1 on the tensor-core encoder: pixel rows of each tile staged by TMA
  // (launch_encode_tc sets it when every tile is one 512 x 4 pixel box)
  int px_tma = 0;
};

template <int CH>
__device__ __forceinline__ void load_rgb(const uint8_t* row, int64_t x, float& r, float& g, float& b) {
  if constexpr (CH == 1) {
    r = g = b = (float)row[x];
  } else {
    const uint8_t* p = row + x * CH;
    r = (float)p[0];
    g = (float)p[1];
    b = (float)p[2];
  }
}

// Binary64 block mean and standard deviation exactly as numpy computes
// blocks.mean(axis=1) / blocks.std(axis=1) (imgc.py:384-386): pairwise-8
// sums, x / 16 (== x * 0.0625, a power of two: the same rounding); on return
// bd[i] = y_i - mean, the centred block.
__device__ __forceinline__ void block_moments(const float (&yv)[16], double (&bd)[16], double& mean, double& sd) {
  double sq[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) bd[i] = (double)yv[i];
  mean = __dmul_rn(pw16d(bd), 0.0625);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    bd[i] = __dsub_rn(bd[i], mean);
    sq[i] = __dmul_rn(bd[i], bd[i]);
  }
  sd = __dsqrt_rn(__dmul_rn(pw16d(sq), 0.0625));
}

// a / b correctly rounded in binary64 from one shared reciprocal (Markstein's
// theorem): with y = RN(1/b) and q = RN(a*y) — within one ulp of a/b — the
// residual r = a - b*q is exact under FMA and RN(q + r*y) = RN(a/b).  The 16
// divisions of a block by the same deviation then cost 3 DFMA each instead of
// a full __ddiv_rn (reciprocal iteration, scaling checks and a slow path).
__device__ __forceinline__ double div_rn_rcp(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, y, q);
}

// Rounding-tie exceptions of the two binary64 quantisers:
// a value whose fractional part is within 1e-9 of one half is where a
// different rounding rule or a last-bit difference in the statistics could
// change rint(); counted so parity reports can state them.
__device__ __forceinline__ bool near_half(double x) { return fabs(__dsub_rn(x, floor(x)) - 0.5) < 1e-9; }

template <int CH>
__global__ void __launch_bounds__(256) ties_kernel(const EncodeArgs a, unsigned long long* ties) {
  const int64_t img = blockIdx.y;
  const int64_t bw = a.width / 4, nblocks = bw * (a.height / 4);
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool tm = false, ts = false;
  if (k < nblocks) {
    // block row / column in 32 bits (the entry points reject images of
    // 2^32 blocks or more): a 64-bit division per block was ~3% of the encoder
    const uint32_t k32 = (uint32_t)k, bw32 = (uint32_t)bw;
    const uint32_t by32 = k32 / bw32;
    const int64_t by = by32, bx = k32 - by32 * bw32;
    const uint8_t* base = a.px + img * a.image_stride;
    float yv[16];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float R, G, B;
        load_rgb<CH>(base + (4 * by + r) * a.row_stride, 4 * bx + c, R, G, B);
        yv[4 * r + c] = luma(R, G, B);
      }
    double bd[16], mean, sd;
    block_moments(yv, bd, mean, sd);
    tm = near_half(mean);
    ts = near_half(__dmul_rn(sd, 4.0));
  }
  const unsigned cm = __popc(__ballot_sync(0xffffffffu, tm)), cs = __popc(__ballot_sync(0xffffffffu, ts));
  if ((threadIdx.x & 31) == 0) {
    if (cm) atomicAdd(ties, (unsigned long long)cm);
    if (cs) atomicAdd(ties + 1, (unsigned long long)cs);
  }
}

// STATS = true: the k-means training pass — only block_grad and the binary64
// normalised blocks (imgc.py:378-388), no chroma, VQ or records.
// Forward block transform of block k of image img (imgc.py:358-401 steps 1-4
// for one block): pixels -> Y/Cb/Cr (binary32), chroma planes, optional
// gradient filter, binary64 mean/std, normalised block.  Returns false in
// STATS mode (outputs written, nothing left to quantise).
// Gray input (CH = 1, R = G = B = v): Y, Cb, Cr of a pixel are functions of
// its byte alone, so a 256-entry table of the reference's binary32 results
// (the same ycc() evaluation, once per value) replaces 9 FMUL + 8 FADD + I2F
// per pixel with one LDS.128.
__device__ __forceinline__ void gray_lut_fill(float4* lut, int tid, int nthreads) {
  for (int v = tid; v < 256; v += nthreads) {
    const YCC o = ycc((float)v, (float)v, (float)v);
    lut[v] = make_float4(o.y, o.cb, o.cr, 0.f);
  }
}

template <int CH, bool STATS>
__device__ __forceinline__ bool block_front(const EncodeArgs& a, int64_t img, int64_t k, float (&nb)[16],
                                            double& mean, double& sd, const float4* lut = nullptr,
                                            bool aligned4 = false, const uint32_t* pre = nullptr) {
  const int64_t bw = a.width / 4, bh = a.height / 4, nblocks = bw * bh;
  {
    // block row / column in 32 bits (the entry points reject images of
    // 2^32 blocks or more): a 64-bit division per block was ~3% of the encoder
    const uint32_t k32 = (uint32_t)k, bw32 = (uint32_t)bw;
    const uint32_t by32 = k32 / bw32;
    const int64_t by = by32, bx = k32 - by32 * bw32;
    const uint8_t* base = a.px + img * a.image_stride;
    float yv[16];
    float cbs = 0.f, crs = 0.f;
    if (CH == 1 && lut) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint8_t* row = base + (4 * by + r) * a.row_stride + 4 * bx;
        uint32_t w;
        if (pre) {
          w = pre[r];  // loaded one tile ahead by the caller
        } else if (aligned4) {
          w = __ldg(reinterpret_cast<const unsigned int*>(row));
        } else {
          w = (uint32_t)row[0] | (uint32_t)row[1] << 8 | (uint32_t)row[2] << 16 | (uint32_t)row[3] << 24;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 e = lut[(w >> (8 * c)) & 255u];
          yv[4 * r + c] = e.x;
          cbs = (r == 0 && c == 0) ? e.y : __fadd_rn(cbs, e.y);
          crs = (r == 0 && c == 0) ? e.z : __fadd_rn(crs, e.z);
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint8_t* row = base + (4 * by + r) * a.row_stride;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float R, G, B;
          load_rgb<CH>(row, 4 * bx + c, R, G, B);
          const YCC o = ycc(R, G, B);
          yv[4 * r + c] = o.y;
          cbs = (r == 0 && c == 0) ? o.cb : __fadd_rn(cbs, o.cb);
          crs = (r == 0 && c == 0) ? o.cr : __fadd_rn(crs, o.cr);
        }
      }
    }
    if constexpr (!STATS) {
      a.cb_plane[img * nblocks + k] = q8f(__fmul_rn(cbs, 0.0625f));
      a.cr_plane[img * nblocks + k] = q8f(__fmul_rn(crs, 0.0625f));
    }

    if (a.block_grad) {
      // forward differences with clamped borders (imgc.py:158-161), hypot
      // in binary64 rounded once (numpy float32 hypot), pairwise-16 mean
      float right[4], below[4];
      const int64_t xr = 4 * bx + 4, yb = 4 * by + 4;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        right[r] = 0.f;
        if (xr < a.width) {
          float R, G, B;
          load_rgb<CH>(base + (4 * by + r) * a.row_stride, xr, R, G, B);
          right[r] = luma(R, G, B);
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        below[c] = 0.f;
        if (yb < a.height) {
          float R, G, B;
          load_rgb<CH>(base + yb * a.row_stride, 4 * bx + c, R, G, B);
          below[c] = luma(R, G, B);
        }
      }
      float mag[16];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float l = yv[4 * r + c];
          float gx = 0.f, gy = 0.f;
          if (4 * bx + c < a.width - 1) gx = __fsub_rn(c < 3 ? yv[4 * r + c + 1] : right[r], l);
          if (4 * by + r < a.height - 1) gy = __fsub_rn(r < 3 ? yv[4 * (r + 1) + c] : below[c], l);
          const double dxd = (double)gx, dyd = (double)gy;
          mag[4 * r + c] = __double2float_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(dxd, dxd), __dmul_rn(dyd, dyd))));
        }
      }
      // x / 16 and x * 0.0625 are the same real number: identical roundings
      a.block_grad[img * nblocks + k] = __fmul_rn(pw16f(mag), 0.0625f);
    }

    // block statistics in binary64 (imgc.py:384-388)
    double bd[16];
    block_moments(yv, bd, mean, sd);
    const double safe = fmax(sd, a.sigma_min);  // np.maximum(sigmas, sigma_min)
    const double rsafe = __drcp_rn(safe);
    if constexpr (STATS) {
      // training rows for the k-means trainer: normalised blocks in binary64
      double* dst = a.norm64 + (img * nblocks + k) * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[i] = div_rn_rcp(bd[i], safe, rsafe);
      return false;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) nb[i] = __double2float_rn(div_rn_rcp(bd[i], safe, rsafe));
    if (a.norm32) {
      float4* dst = reinterpret_cast<float4*>(a.norm32 + (img * nblocks + k) * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float4(nb[4 * q], nb[4 * q + 1], nb[4 * q + 2], nb[4 * q + 3]);
    }
  }
  return true;
}

template <int CH, bool STATS = false>
__global__ void __launch_bounds__(256) encode_kernel(const EncodeArgs a) {
  __shared__ float2 scp[256 * 8];
  __shared__ uint8_t srec[256 * 3];
  const int64_t img = blockIdx.y;
  if constexpr (!STATS) {
    vq_stage_codebook(a.codebook + img * a.codebook_stride, a.ncb, scp);
    __syncthreads();
  }
  const int64_t nblocks = (a.width / 4) * (a.height / 4);
  const int64_t k0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t k = k0 + threadIdx.x;
  float nb[16];
  double mean, sd;
  if (k < nblocks && block_front<CH, STATS>(a, img, k, nb, mean, sd)) {
    // exact nearest centroid (vq_program semantics: strict <, first index wins)
    float2 bp[8];
    vq_pack(nb, bp);
    float best = VQ_BEST_INIT;
    int bj = 0;
    for (int j = 0; j < a.ncb; ++j) {
      const float d = vq_dist_pairs(bp, scp + 8 * j);
      if (d < best) { best = d; bj = j; }
    }
    const int t = threadIdx.x;
    srec[3 * t + 0] = q8d(mean);
    srec[3 * t + 1] = q8d(__dmul_rn(sd, 4.0));  // sd / 0.25 is exact
    srec[3 * t + 2] = (uint8_t)bj;
    if (a.idx_plane) {
      a.mu_plane[img * nblocks + k] = srec[3 * t];
      a.sig_plane[img * nblocks + k] = srec[3 * t + 1];
      a.idx_plane[img * nblocks + k] = srec[3 * t + 2];
    }
  }
  if constexpr (!STATS) {
    if (a.idx_plane) return;
    __syncthreads();
    // records of this CTA are one contiguous run: write it with coalesced bytes
    const int64_t nrec = (nblocks - k0 < (int64_t)blockDim.x ? nblocks - k0 : (int64_t)blockDim.x) * 3;
    uint8_t* rec = a.records + (img * nblocks + k0) * 3;
    for (int e = threadIdx.x; e < nrec; e += blockDim.x) rec[e] = srec[e];
  }
}

// ---------------------------------------------------------------------------
// Tensor-core pruned EXACT vector quantisation (tcgen05, kind::f16).
//
// The exact search costs 31 binary32 ops per (block, centroid).  Here a
// 128-block tile is multiplied against the whole 256-entry codebook on the
// 5th-gen tensor cores (binary16 hi + lo split of both operands, three MMAs
// n_hi.c_hi + n_hi.c_lo + n_lo.c_hi, fp32 accumulation in TMEM), plus one bias
// MMA (a constant A column against the per-centroid |c_j|^2/2 + 8), so TMEM holds
//   v_j = |c_j|^2/2 + 8 - n.c_j  =  (D_j - |n|^2)/2 + 8  (+- DELTA/2)
// which is >= D_j/2 >= 0 for every normalised block (|n|^2 <= 16).  The rank
// phase (ws::rank_chunk) finds the minimum and counts the scores within the
// band of it; when the minimum is alone there, the approximate argmin IS the
// reference's index; otherwise the block is re-checked with the reference's
// exact binary32 distance over every centroid whose score is within the band,
// in index order with strict <, so ties resolve to the first index exactly
// like vq_program (imgc.py:175-178).  DELTA bounds |s_j - (D^fp32_j - |n|^2)|:
// the split's truncation (2^-22 relative per operand, the same 22 bits as a
// 3xTF32 split), fp32 accumulation, the fp32 norm, and the reference's own
// rounding of D (<= 7u*D); see DESIGN.md.  It is scaled by the codebook's
// largest norm and checked empirically in tests; a codebook outside the
// binary16 split's range sends every block to the exact path.
namespace tc {
constexpr int M = 128;      // blocks per tile (TMEM lanes)
constexpr int NCB = 256;    // centroids (padded; TMEM columns)
constexpr float BIAS = 8.f;  // >= |n|^2 / 2 for every normalised block
// shared-memory matrix descriptor, layout SWIZZLE_NONE: lbo = byte offset of
// the next K core matrix, sbo = byte offset of the next 8-row group (0: every
// group reads the same rows)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  return d;                            // base offset 0, layout SWIZZLE_NONE
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
}  // namespace tc

// Encoder (round 2): one CTA per SM, 16 warps in FOUR identical groups of
// 128 threads; group g takes local tiles i = g, g + 4, ... (128 blocks each,
// one block per thread) and runs every phase of its tile itself:
//   front: pixels -> Y/Cb/Cr (gray: table), chroma bytes, binary64
//     statistics, normalised block -> the group's A buffer (-n as binary16
//     hi + lo) and its exact binary32 copy; the record bytes mu / sigma stay
//     in the thread's registers;
//   MMA: one elected thread issues the 3 x binary16 + bias MMAs of the whole
//     codebook (N = 256) into TMEM slot i & 1 (256 columns) once the group
//     two tiles back has read that slot, and commits mma_done[i & 1];
//   rank: tcgen05.ld of the row's 256 scores (32 per chunk), chunk minimum
//     and threshold count on the FMA pipe, TMEM slot released, the exact
//     re-check of the rare ambiguous block, the record written.
// The front of a tile is a long binary64 latency chain; four groups keep
// four such chains (and the short rank phases) in flight per SM partition
// where a front / epilogue split kept two, with the two TMEM slots shared
// by the groups in tile order.  Images are processed one after another with
// every CTA striding over the image's tiles; the codebook (B operand) is
// restaged between images after a CTA-wide barrier.

namespace ws {
constexpr int THREADS = 512;
// Operands in binary16, split hi + lo (x = hi + lo + e, |e| <= 2^-22 |x|: the
// same 22 significant bits as the tf32 split, at twice the tensor-core rate;
// tcgen05 kind::f16 keeps binary16 subnormals, profiles/micro/f16_subnormal.cu).
// K-major canonical layout without swizzle: 8-row groups of four 16-byte
// K-chunks (8 halves: hi k 0..7, hi 8..15, lo 0..7, lo 8..15), 512 B per group.
__device__ __forceinline__ uint32_t off16(int row, int k) {
  return (uint32_t)((row >> 3) * 512 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}
constexpr size_t A_BYTES = tc::M * 64;                      // 8 KB per buffer (hi | lo halves)
constexpr size_t B_BYTES = tc::NCB * 64;                    // 16 KB: codebook hi | lo halves
constexpr size_t B_OFF = 0;
constexpr size_t A_OFF = B_OFF + B_BYTES;                   // A buffers, one per group
constexpr size_t AX_OFF = A_OFF + 4 * A_BYTES;              // exact binary32 blocks, 128 x 16 per group
constexpr size_t CBX_OFF = AX_OFF + 4 * tc::M * 64;         // exact binary32 codebook, 256 x 16
constexpr size_t CN_OFF = CBX_OFF + tc::NCB * 64;           // |c_j|^2
constexpr size_t ABIAS_OFF = CN_OFF + tc::NCB * 4;          // 8 rows x [1 1 0 ... 0] (16 halves)
constexpr size_t BBIAS_OFF = ABIAS_OFF + 256;               // per centroid [hi lo 0 ... 0] of |c|^2/2 + 8
constexpr size_t LUT_OFF = BBIAS_OFF + tc::NCB * 32;        // gray table, 256 x float4
constexpr size_t PX_OFF = LUT_OFF + 256 * 16;                // gray pixels: 2 boxes of 4 x 512 per group
constexpr size_t PX_BYTES = 4 * 512;
constexpr size_t SMEM = PX_OFF + 4 * 2 * PX_BYTES;
// kind::f16 (binary16 A and B, fp32 accumulate), M = 128, N = 256 (the whole
// codebook in one instruction), K = 16 per instruction
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(tc::NCB >> 3) << 17) | ((uint32_t)(tc::M >> 4) << 24);
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
// x -> (hi, lo) binary16 halves; |x - hi - lo| <= 2^-22 |x| (v - hi is exact in binary32)
__device__ __forceinline__ void split16(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(__fsub_rn(v, __half2float(hi)));
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float m;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(a), "f"(b), "f"(c));  // FMNMX3
  return m;
}
// Rank one 32-column chunk of a row's scores v_j (j = j0 .. j0 + 31) on the
// FMA pipe.  cm = the chunk minimum; every score below thr = RN(cm + band)
// gets t_j = 1, every other t_j = 0 — FFMA.SAT(v_j, -2^60, 2^60 thr) is
// exactly 0 or 1 because the fused product-sum differs from 0 by >= 2^27
// unless v_j == thr (then 0): thr >= band >= 2^-14 has ulp >= 2^-37.  acc =
// sum t_j (1024 + j) is exact in binary32 (<= 32 * 1279 < 2^24): acc < 2048
// means the minimum is the only score of the chunk below thr, and then
// acc - 1024 is its column.  2 FMA-pipe ops per score (immediate forms) and
// 1/2 ALU op (3-input min), where a best / runner-up tournament on integer
// keys costs 3.5 ALU ops per score.
__device__ __forceinline__ void rank_chunk(const uint32_t (&r)[32], int j0, float band60, float& cm, float& acc) {
  float m[11];
#pragma unroll
  for (int e = 0; e < 10; ++e)
    m[e] = fmin3(__uint_as_float(r[3 * e]), __uint_as_float(r[3 * e + 1]), __uint_as_float(r[3 * e + 2]));
  m[10] = fminf(__uint_as_float(r[30]), __uint_as_float(r[31]));
  cm = fmin3(fmin3(fmin3(m[0], m[1], m[2]), fmin3(m[3], m[4], m[5]), fmin3(m[6], m[7], m[8])), m[9], m[10]);
  const float beta = fmaf(cm, 0x1p60f, band60);  // 2^60 RN(cm + band): power-of-two scaling is exact
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    float t;
    asm("fma.rn.sat.f32 %0, %1, 0fDD800000, %2;" : "=f"(t) : "f"(__uint_as_float(r[e])), "f"(beta));  // -2^60
    a[e & 3] = fmaf(t, (float)(1024 + j0 + e), a[e & 3]);
  }
  acc = (a[0] + a[1]) + (a[2] + a[3]);
}
}  // namespace ws

template <int CH>
__global__ void __launch_bounds__(ws::THREADS, 1) encode_ws_kernel(const EncodeArgs a, int64_t batch,
                                                                   float delta_scale, unsigned long long* ambiguous,
                                                                   const __grid_constant__ CUtensorMap tpx) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  uint8_t* sB = tsm + ws::B_OFF;
  float* scn = reinterpret_cast<float*>(tsm + ws::CN_OFF);  // |c_j|^2
  float4* lut = reinterpret_cast<float4*>(tsm + ws::LUT_OFF);
  // mma_done per GROUP: a barrier shared by the two groups of a TMEM slot
  // would let a group's parity wait see the other group's completed phase
  __shared__ __align__(8) uint64_t mma_done[4], tmem_free[2];
  __shared__ __align__(8) uint64_t px_full[4][2];  // a.px_tma: pixel box of the group's tile landed
  __shared__ uint32_t tmem_base_s;
  __shared__ unsigned int cmax_bits;
  __shared__ unsigned long long zero_key;  // (exact distance of the zero block, index) minimum
  __shared__ int wide_cb;  // codebook outside the binary16 split's range: every block takes the exact path
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp >> 2;      // group: local tiles grp, grp + 4, ...
  const int row = tid & 127;      // tile row (block) = TMEM lane of this thread
  const bool aligned4 = (((uintptr_t)a.px | (uintptr_t)a.row_stride | (uintptr_t)a.image_stride) & 3) == 0;
  uint8_t* sA = tsm + ws::A_OFF + grp * ws::A_BYTES;
  float* sAX = reinterpret_cast<float*>(tsm + ws::AX_OFF) + grp * tc::M * 16;  // exact blocks of this group
  const float* sCBX = reinterpret_cast<const float*>(tsm + ws::CBX_OFF);

  auto stage_codebook = [&](int64_t img) {
    const float* cbk = a.codebook + img * a.codebook_stride;
    if (tid == 0) {
      cmax_bits = 0;
      zero_key = ~0ull;
      wide_cb = 0;
    }
    __syncthreads();
    for (int e = tid; e < tc::NCB * 16; e += ws::THREADS) {
      const int j = e >> 4, k = e & 15;
      const float c = j < a.ncb ? cbk[j * 16 + k] : 0.f;
      __half hi, lo;
      ws::split16(c, hi, lo);
      *reinterpret_cast<__half*>(sB + ws::off16(j, k)) = hi;
      *reinterpret_cast<__half*>(sB + ws::off16(j, 16 + k)) = lo;
      reinterpret_cast<float*>(tsm + ws::CBX_OFF)[e] = c;
      if (!(fabsf(c) <= 0x1p14f)) wide_cb = 1;  // outside the binary16 split's range (or NaN)
    }
    __syncthreads();
    for (int j = tid; j < tc::NCB; j += ws::THREADS) {
      float s = 0.f;
      if (j < a.ncb)
        for (int k = 0; k < 16; ++k) s = fmaf(cbk[j * 16 + k], cbk[j * 16 + k], s);
      scn[j] = j < a.ncb ? s : 1e30f;
      // bias B operand: |c_j|^2/2 + 8 as binary16 hi + lo (padding centroids
      // get the largest finite score so they never win)
      const float bv = j < a.ncb ? fmaf(0.5f, s, tc::BIAS) : 60000.f;
      if (!(bv <= 0x1p15f)) wide_cb = 1;
      __half bh, bl;
      ws::split16(bv, bh, bl);
      uint8_t* brow = tsm + ws::BBIAS_OFF + (j >> 3) * 256 + (j & 7) * 16;  // K-chunks at +0, +128
      *reinterpret_cast<uint4*>(brow) = make_uint4(__half_as_ushort(bh) | ((uint32_t)__half_as_ushort(bl) << 16), 0u,
                                                   0u, 0u);
      *reinterpret_cast<uint4*>(brow + 128) = make_uint4(0u, 0u, 0u, 0u);
      if (j < a.ncb) {
        atomicMax(&cmax_bits, __float_as_uint(s));  // s >= 0: bit order = value order
        // a constant block normalises to exactly 0: its index is the exact
        // (reference-order) argmin of |c_j|^2, strict <, first index
        float c[16];
        for (int k = 0; k < 16; ++k) c[k] = cbk[j * 16 + k];
        float2 zp[8], cp[8];
        const float zero16[16] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        vq_pack(zero16, zp);
        vq_pack(c, cp);
        const float d = vq_dist_pairs(zp, cp);
        if (d < VQ_BEST_INIT) atomicMin(&zero_key, ((unsigned long long)__float_as_uint(d) << 32) | (unsigned)j);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
  };

  if (tid < 128)  // bias A operand: 8 rows x [1 1 0 ... 0] halves (one 8-row group, sbo = 0)
    reinterpret_cast<__half*>(tsm + ws::ABIAS_OFF)[tid] = __float2half_rn((tid < 64 && (tid & 7) < 2) ? 1.f : 0.f);
  if (CH == 1) gray_lut_fill(lut, tid, ws::THREADS);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(&mma_done[q], 1);
    for (int q = 0; q < 2; ++q) mbar_init(&tmem_free[q], 4);
    for (int q = 0; q < 8; ++q) mbar_init(&px_full[q >> 1][q & 1], 1);
    fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  const int64_t nblocks = (a.width / 4) * (a.height / 4);
  const int64_t ntiles = (nblocks + tc::M - 1) / tc::M;
  // u counts this CTA's local tiles over all images (every group steps it by
  // one per tile of every group, so all threads agree on the barrier phases):
  // tile u belongs to group u & 3 and uses TMEM slot u & 1 for the
  // (u >> 1)-th time
  uint32_t u0 = 0;
  uint32_t gtiles = 0;  // tiles this group has run (mma_done[grp] phases, px_full buffer gtiles & 1)
  const bool px_tma = CH == 1 && a.px_tma;
  uint32_t* spx = reinterpret_cast<uint32_t*>(tsm + ws::PX_OFF) + grp * (2 * ws::PX_BYTES / 4);
  // the group's i-th tile of image img: one 512 x 4 pixel box (tiles never
  // straddle block rows when px_tma is set)
  auto px_issue = [&](int64_t img, int64_t i, int buf) {
    const int64_t bw = a.width / 4;
    const int64_t k0 = (blockIdx.x + (int64_t)gridDim.x * i) * tc::M, by = k0 / bw;
    mbar_arrive_expect_tx(&px_full[grp][buf], (uint32_t)ws::PX_BYTES);
    tma_load_3d(spx + buf * (ws::PX_BYTES / 4), &tpx, (int)(k0 - by * bw), (int)(4 * by), (int)img,
                &px_full[grp][buf]);
  };
  unsigned long long namb = 0;
  for (int64_t img = 0; img < batch; ++img) {
    stage_codebook(img);
    const float cmax = sqrtf(__uint_as_float(cmax_bits));
    // band half-width: 1.5e-3 at |c| <= 4 (the normalised-block scale), growing
    // with the distance magnitude (4 + |c|max)^2 for larger codebook vectors
    const float delta2 = 2.f * delta_scale * 1.5e-3f * fmaxf(1.f, (4.f + cmax) * (4.f + cmax) / 64.f);
    const int zero_idx = zero_key == ~0ull ? 0 : (int)(zero_key & 0xffffffffu);
    const int64_t nlocal = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    // the group's first two tiles of this image (every earlier box was consumed)
    if (px_tma && row == 0)
      for (int q = 0; q < 2; ++q)
        if (grp + 4 * q < nlocal) px_issue(img, grp + 4 * q, (gtiles + q) & 1);
    for (int64_t i = grp; i < nlocal; i += 4) {
      const uint32_t u = u0 + (uint32_t)i;
      const int slot = u & 1;
      const uint32_t use = u >> 1;
      const uint32_t tmem = tmem_base_s + 256u * slot;
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // lanes 32 (w % 4) ..
      const int64_t t = blockIdx.x + (int64_t)gridDim.x * i;
      const int64_t k = t * tc::M + row;
      const bool active = k < nblocks;
      // ---------------------------------------------------------------- front
      float nb[16];
      double mean = 0.0, sd = 0.0;
      if (active) {
        if constexpr (CH == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(a.vecs + k * 16) + q);
            nb[4 * q] = f.x;
            nb[4 * q + 1] = f.y;
            nb[4 * q + 2] = f.z;
            nb[4 * q + 3] = f.w;
          }
        } else if (px_tma) {
          const int buf = gtiles & 1;
          mbar_wait(&px_full[grp][buf], (gtiles >> 1) & 1);
          uint32_t w4[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) w4[r] = spx[buf * (ws::PX_BYTES / 4) + r * tc::M + row];
          block_front<CH, false>(a, img, k, nb, mean, sd, lut, aligned4, w4);
        } else {
          block_front<CH, false>(a, img, k, nb, mean, sd, CH == 1 ? lut : nullptr, aligned4);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) nb[e] = 0.f;
      }
      bool zero = true;
#pragma unroll
      for (int e = 0; e < 16; ++e) zero = zero && nb[e] == 0.f;
      const uint8_t mu = q8d(mean), sg = q8d(__dmul_rn(sd, 4.0));  // sd / 0.25 is exact
      // the group's A buffer: its previous reader (the MMA of tile u - 4) was
      // waited for by this group's own rank phase
#pragma unroll
      for (int q = 0; q < 2; ++q) {  // K-chunks of 8: hi at chunk q, lo at chunk 2 + q
        __half2 hh[4], ll[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __half h0, l0, h1, l1;
          ws::split16(-nb[8 * q + 2 * e], h0, l0);
          ws::split16(-nb[8 * q + 2 * e + 1], h1, l1);
          hh[e] = __halves2half2(h0, h1);
          ll[e] = __halves2half2(l0, l1);
        }
        *reinterpret_cast<uint4*>(sA + ws::off16(row, 8 * q)) = *reinterpret_cast<uint4*>(hh);
        *reinterpret_cast<uint4*>(sA + ws::off16(row, 16 + 8 * q)) = *reinterpret_cast<uint4*>(ll);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)  // the exact block for the re-check
        *reinterpret_cast<float4*>(sAX + row * 16 + 4 * q) =
            make_float4(nb[4 * q], nb[4 * q + 1], nb[4 * q + 2], nb[4 * q + 3]);
      fence_proxy_async_smem();
      ws::named_sync(1 + grp, 128);
      // the pixel box is consumed: refill it with the group's tile i + 8
      if (px_tma && row == 0 && i + 8 < nlocal) px_issue(img, i + 8, gtiles & 1);
      // ------------------------------------------------------------------ MMA
      if (row == 0) {
        // TMEM slot: free once tile u - 2 (another group) has read its scores
        mbar_wait(&tmem_free[slot], (use & 1) ^ 1);
        tc::fence_after();
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        // hi.hi, hi.lo, lo.hi over K = 0..15 (hi chunks at +0, lo chunks at +256)
        ws::mma(tmem, tc::sdesc(a0, 128, 512), tc::sdesc(b0, 128, 512), 0u);
        ws::mma(tmem, tc::sdesc(a0, 128, 512), tc::sdesc(b0 + 256, 128, 512), 1u);
        ws::mma(tmem, tc::sdesc(a0 + 256, 128, 512), tc::sdesc(b0, 128, 512), 1u);
        // + |c_j|^2/2 + 8: A = [1 1 0 ... 0] in every row, B = [hi lo 0 ... 0]
        ws::mma(tmem, tc::sdesc(smem_u32(tsm + ws::ABIAS_OFF), 128, 0),
                tc::sdesc(smem_u32(tsm + ws::BBIAS_OFF), 128, 256), 1u);
        tc::commit(&mma_done[grp]);
      }
      // ----------------------------------------------------------------- rank
      mbar_wait(&mma_done[grp], gtiles & 1);
      ++gtiles;
      tc::fence_after();
      // chunks of 32 columns: chunk minimum + count / column of the scores
      // within `band` of it; across chunks keep the smallest minimum and its
      // chunk's count.  A block is ambiguous when the smallest chunk holds a
      // second score below min + band or another chunk's minimum lies within
      // band of it (conservative when an earlier pair of chunk minima was
      // close and a later chunk undercuts both: a re-check, never a miss).
      const float band = 0.5f * delta2 * (1.f + 0x1p-9f);
      const float band60 = band * 0x1p60f;
      float gm = __int_as_float(0x7f800000), gacc = 0.f;
      bool close = false;
      // TMEM loads are short (tens of cycles): one 32-column chunk in flight
#pragma unroll
      for (int c = 0; c < tc::NCB / 32; ++c) {
        uint32_t r[32];
        ws::ld32_nowait(taddr + c * 32, r);
        ws::ld_wait();
        if (c == tc::NCB / 32 - 1) {
          // every score of this tile is in registers: the slot goes to tile u + 2
          tc::fence_before();
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_free[slot])) : "memory");
        }
        float cm, cacc;
        ws::rank_chunk(r, c * 32, band60, cm, cacc);
        close = close || fabsf(cm - gm) <= band;
        gacc = cm < gm ? cacc : gacc;
        gm = fminf(gm, cm);
      }
      const int i1 = (int)gacc - 1024;
      const float v1 = gm;
      const float quant = __int_as_float((__float_as_int(fabsf(v1)) & 0x7F800000)) * 0x1p-15f;  // 2^8 ulps of v1
      const bool amb = active && !zero && (close || gacc >= 2048.f || wide_cb);
      int bj = zero ? zero_idx : i1;
      unsigned amb_lanes = __ballot_sync(0xffffffffu, amb);
      // rare (~0.05 % of blocks): the whole warp re-checks one ambiguous block
      // at a time — each lane rescores 8 centroids on the CUDA cores (fp32,
      // error << DELTA) and runs the reference's exact distance on those inside
      // the band; a lexicographic (distance, index) warp minimum reproduces
      // "strict <, first index wins" over all 256.  The block and the codebook
      // come from their exact binary32 copies.
      while (amb_lanes) {
        const int src = __ffs(amb_lanes) - 1;
        amb_lanes &= amb_lanes - 1;
        const int srow = (row & ~31) + src;
        float nv[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 x = *reinterpret_cast<const float4*>(sAX + srow * 16 + 4 * q);
          nv[4 * q] = x.x;
          nv[4 * q + 1] = x.y;
          nv[4 * q + 2] = x.z;
          nv[4 * q + 3] = x.w;
        }
        // the band in the old score scale s = |c|^2 - 2 n.c = 2 (v - 8); a wide
        // codebook re-checks every centroid
        const float lim = wide_cb ? __int_as_float(0x7f800000)
                                  : __shfl_sync(0xffffffffu, 2.f * (v1 + quant - tc::BIAS) + delta2, src);
        float2 bp[8];
        vq_pack(nv, bp);
        float best = VQ_BEST_INIT;
        int bx = 0x7fffffff;
#pragma unroll 1
        for (int j = lane; j < a.ncb; j += 32) {
          float c[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 x = *reinterpret_cast<const float4*>(sCBX + j * 16 + 4 * q);
            c[4 * q] = x.x;
            c[4 * q + 1] = x.y;
            c[4 * q + 2] = x.z;
            c[4 * q + 3] = x.w;
          }
          float dotv = 0.f;
#pragma unroll
          for (int e = 0; e < 16; ++e) dotv = fmaf(nv[e], c[e], dotv);
          if (fmaf(-2.f, dotv, scn[j]) <= lim) {
            float2 cp[8];
            vq_pack(c, cp);
            const float d = vq_dist_pairs(bp, cp);
            if (d < best) { best = d; bx = j; }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float od = __shfl_xor_sync(0xffffffffu, best, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bx, o);
          if (od < best || (od == best && oj < bx)) { best = od; bx = oj; }
        }
        if (lane == src) {
          bj = bx == 0x7fffffff ? 0 : bx;
          ++namb;
        }
      }
      // every thread writes its own block's record: three byte stores per
      // warp instruction cover 96 contiguous bytes (interleaved) or 32 per
      // plane
      if (CH == 0) {
        if (active) a.idx_plane[k] = (uint8_t)bj;
      } else if (active) {
        const int64_t gk = img * nblocks + k;
        if (a.idx_plane) {
          a.mu_plane[gk] = mu;
          a.sig_plane[gk] = sg;
          a.idx_plane[gk] = (uint8_t)bj;
        } else {
          uint8_t* rec = a.records + gk * 3;
          rec[0] = mu;
          rec[1] = sg;
          rec[2] = (uint8_t)bj;
        }
      }
    }
    u0 += (uint32_t)nlocal;
    // every MMA of this image has been waited for by its group and every
    // group has finished reading A/B: the codebook may be replaced
    __syncthreads();
  }
  if (ambiguous && namb) atomicAdd(ambiguous, namb);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_s));
}

// DPP_IMGC_VQ=exact selects the CUDA-core brute force (1), default tensor cores (0)
static int vq_mode() {
  const char* e = getenv("DPP_IMGC_VQ");  // read per call: tests flip it at run time
  return (e && e[0] == 'e') ? 1 : 0;
}

static int launch_encode_tc(const EncodeArgs& a, int channels, int64_t batch, int64_t nblocks, float delta_scale,
                            unsigned long long* ambiguous, cudaStream_t s) {
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (sm_count <= 0) sm_count = 148;
  }
  // one CTA per SM (all 512 TMEM columns); every CTA takes every image's tiles
  // in a stride of the grid, so a grid larger than one image's tiles idles
  const int64_t ntiles = (nblocks + tc::M - 1) / tc::M;
  const int64_t want = (ntiles + 3) / 4;  // every group of a CTA busy
  dim3 grid((unsigned)(want < sm_count ? want : sm_count));
  const size_t smem = ws::SMEM;
  // gray pixels by TMA: every tile one 512 x 4 box (block rows a multiple of
  // the 128-block tile), 16-byte aligned rows and images
  EncodeArgs b = a;
  CUtensorMap tpx;
  std::memset(&tpx, 0, sizeof(tpx));
  const int64_t istride = batch > 1 ? a.image_stride : a.row_stride * a.height;
  b.px_tma = channels == 1 && (a.width / 4) % tc::M == 0 && ((uintptr_t)a.px % 16) == 0 && a.row_stride % 16 == 0 &&
             istride % 16 == 0 && batch <= 65535;
  if (b.px_tma) {
    const uint64_t dims[3] = {(uint64_t)(a.width / 4), (uint64_t)a.height, (uint64_t)(batch > 0 ? batch : 1)};
    const uint64_t strides[2] = {(uint64_t)a.row_stride, (uint64_t)istride};
    const uint32_t box[3] = {(uint32_t)tc::M, 4, 1};
    if (make_tmap_u8_3d(&tpx, a.px, dims, strides, box, true)) b.px_tma = 0;
  }
  switch (channels) {
#define TC_CASE(CHN)                                                                                        \
  case CHN:                                                                                                 \
    DPP_CUDA_CHECK(cudaFuncSetAttribute(encode_ws_kernel<CHN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        (int)smem));                                                        \
    encode_ws_kernel<CHN><<<grid, ws::THREADS, smem, s>>>(b, batch, delta_scale, ambiguous, tpx);         \
    break;
    TC_CASE(0)
    TC_CASE(1)
    TC_CASE(3)
    TC_CASE(4)
#undef TC_CASE
  }
  DPP_LAUNCH_CHECK("encode_ws_kernel");
  return DPP_OK;
}

// Nearest centroid of n normalised binary32 16-vectors (the encoder's search:
// 3 x binary16 tensor-core scores, exact binary32 re-check of the ambiguous ones,
// strict <, first index) — the Lloyd assignment of the k-means trainer.
int vq_assign_tc(const float* vecs, int64_t n, const float* cents, int k, uint8_t* idx, cudaStream_t s) {
  if (n <= 0) return DPP_OK;
  EncodeArgs a{};
  a.vecs = vecs;
  a.height = 4 * n;  // n "blocks" of one 4-wide column
  a.width = 4;
  a.codebook = cents;
  a.ncb = k;
  a.idx_plane = idx;
  return launch_encode_tc(a, 0, 1, n, 1.0f, nullptr, s);
}

// ---------------------------------------------------------------------------
// decoder (imgc.py:426-439): one thread per pixel, binary64 like numpy

__global__ void decode_kernel(const uint8_t* __restrict__ records, const uint8_t* __restrict__ cbp,
                              const uint8_t* __restrict__ crp, const float* __restrict__ codebook,
                              int64_t height, int64_t width, uint8_t* __restrict__ rgb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= height * width) return;
  const int64_t y = i / width, x = i - y * width;
  const int64_t bw = width / 4;
  const int64_t k = (y / 4) * bw + x / 4;
  const int pos = (int)((y & 3) * 4 + (x & 3));
  const double mean = (double)records[3 * k];
  const double sigma = __dmul_rn((double)records[3 * k + 1], 0.25);
  const double cval = (double)codebook[records[3 * k + 2] * 16 + pos];
  const double l = __dadd_rn(mean, __dmul_rn(sigma, cval));
  const double cb = __dsub_rn((double)cbp[k], 128.0);
  const double cr = __dsub_rn((double)crp[k], 128.0);
  const double r = __dadd_rn(l, __dmul_rn(1.402, cr));
  const double g = __dsub_rn(__dsub_rn(l, __dmul_rn(0.344136, cb)), __dmul_rn(0.714136, cr));
  const double b = __dadd_rn(l, __dmul_rn(1.772, cb));
  rgb[3 * i + 0] = q8d(r);
  rgb[3 * i + 1] = q8d(g);
  rgb[3 * i + 2] = q8d(b);
}

static unsigned grid1(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace dpp

extern "C" {

int dpp_imgc_ycbcr(const uint8_t* rgba, float* yl, float* cb, float* cr, int64_t pixels, void* stream) {
  if (pixels < 0) return dpp::fail(DPP_EINVAL, "pixels must be >= 0");
  if (pixels == 0) return DPP_OK;
  dpp::ycbcr_kernel<<<dpp::grid1(pixels, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uchar4*>(rgba), yl, cb, cr, pixels);
  DPP_LAUNCH_CHECK("ycbcr_kernel");
  return DPP_OK;
}

int dpp_imgc_boxdown(const float* blk, float* avg, int64_t blocks, void* stream) {
  if (blocks < 0) return dpp::fail(DPP_EINVAL, "blocks must be >= 0");
  if (blocks == 0) return DPP_OK;
  dpp::boxdown_kernel<<<dpp::grid1(blocks, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(blk), avg, blocks);
  DPP_LAUNCH_CHECK("boxdown_kernel");
  return DPP_OK;
}

int dpp_imgc_gradient(const float* lum, float* dx, float* dy, int64_t width, int64_t height,
                      int64_t items, int64_t* fault_item, void* stream) {
  if (width < 1 || height < 1 || items < 0) return dpp::fail(DPP_EINVAL, "bad gradient geometry");
  if (fault_item) *fault_item = -1;
  if (items == 0) return DPP_OK;
  if (items >= width * height) {
    // whole frames: every guarded read stays inside the chunk, nothing to report
    dpp::gradient_kernel<<<dpp::grid1(items, 256), 256, 0, (cudaStream_t)stream>>>(lum, dx, dy, width, height,
                                                                                    items, nullptr);
    DPP_LAUNCH_CHECK("gradient_kernel");
    return DPP_OK;
  }
  unsigned long long* fault = nullptr;
  DPP_CUDA_CHECK(cudaMallocAsync(&fault, 2 * sizeof(unsigned long long), (cudaStream_t)stream));
  DPP_CUDA_CHECK(cudaMemsetAsync(fault, 0xff, 2 * sizeof(unsigned long long), (cudaStream_t)stream));
  dpp::gradient_kernel<<<dpp::grid1(items, 256), 256, 0, (cudaStream_t)stream>>>(lum, dx, dy, width, height,
                                                                                  items, fault);
  DPP_LAUNCH_CHECK("gradient_kernel");
  unsigned long long h[2];
  DPP_CUDA_CHECK(cudaMemcpyAsync(h, fault, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  DPP_CUDA_CHECK(cudaFreeAsync(fault, (cudaStream_t)stream));
  DPP_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  // the interpreter evaluates the dx statement for every lane before dy
  const unsigned long long none = ~0ULL;
  const unsigned long long bad = h[0] != none ? h[0] : h[1];
  if (bad != none) {
    const int64_t i = (int64_t)bad;
    const int64_t at = h[0] != none ? i + 1 : i + width;
    if (fault_item) *fault_item = i;
    return dpp::fail(DPP_EINVAL, "index %lld out of range for point 'lum' (0..%lld)", (long long)at,
                     (long long)(items - 1));
  }
  return DPP_OK;
}

int dpp_imgc_vqnearest(const float* blk, const float* cbk, int32_t* idx, int64_t items, int64_t cbk_items,
                       int codebook_size, void* stream) {
  if (items < 0 || codebook_size < 0 || codebook_size > 4096)
    return dpp::fail(DPP_EINVAL, "bad vqnearest arguments");
  if (items == 0) return DPP_OK;
  if (codebook_size > cbk_items)
    return dpp::fail(DPP_EINVAL, "index %lld out of range for point 'cbk' (0..%lld)", (long long)cbk_items,
                     (long long)(cbk_items - 1));
  const size_t smem = (size_t)codebook_size * 16 * sizeof(float);
  if (smem > 48 * 1024)
    DPP_CUDA_CHECK(cudaFuncSetAttribute(dpp::vqnearest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  dpp::vqnearest_kernel<<<dpp::grid1(items, 256), 256, smem, (cudaStream_t)stream>>>(blk, cbk, idx, items,
                                                                                     codebook_size);
  DPP_LAUNCH_CHECK("vqnearest_kernel");
  return DPP_OK;
}

static int encode_common(const uint8_t* px, int channels, int64_t height, int64_t width, int64_t row_stride,
                         int64_t image_stride, int64_t batch, const float* codebook, int n_cb,
                         int64_t codebook_stride, double sigma_min, uint8_t* records, uint8_t* mu_plane,
                         uint8_t* sig_plane, uint8_t* idx_plane, uint8_t* cb_plane, uint8_t* cr_plane,
                         float* block_grad, float* norm32, void* stream) {
  if (height % 4 || width % 4 || height < 4 || width < 4)
    return dpp::fail(DPP_EINVAL, "dimensions must be multiples of 4, got %lldx%lld", (long long)width,
                     (long long)height);
  if ((height / 4) * (width / 4) > 0xffffffffLL)
    return dpp::fail(DPP_EINVAL, "%lldx%lld has 2^32 or more 4x4 blocks", (long long)width, (long long)height);
  if (n_cb < 1 || n_cb > 256) return dpp::fail(DPP_EINVAL, "codebook size must be in 1..256");
  if (channels != 1 && channels != 3 && channels != 4)
    return dpp::fail(DPP_EINVAL, "channels must be 1, 3 or 4, got %d", channels);
  if (row_stride < width * channels) return dpp::fail(DPP_EINVAL, "row stride too small");
  if (batch < 0 || batch > 65535) return dpp::fail(DPP_EINVAL, "batch must be in 0..65535");
  if (batch == 0) return DPP_OK;
  if (!(sigma_min > 0.0)) return dpp::fail(DPP_EINVAL, "sigma_min must be > 0");
  if (!px || !codebook || !cb_plane || !cr_plane || (!records && !(mu_plane && sig_plane && idx_plane)))
    return dpp::fail(DPP_EINVAL, "NULL data pointer");
  dpp::EncodeArgs a{px,      height,   width,      row_stride, image_stride, codebook, n_cb,
                    codebook_stride, sigma_min, records,  cb_plane,   cr_plane, block_grad, norm32,
                    nullptr, mu_plane, sig_plane, idx_plane};
  const int64_t nblocks = (height / 4) * (width / 4);
  auto s = (cudaStream_t)stream;
  if (dpp::vq_mode() == 1) {
    dim3 grid(dpp::grid1(nblocks, 256), (unsigned)batch);
    switch (channels) {
      case 1: dpp::encode_kernel<1><<<grid, 256, 0, s>>>(a); break;
      case 3: dpp::encode_kernel<3><<<grid, 256, 0, s>>>(a); break;
      default: dpp::encode_kernel<4><<<grid, 256, 0, s>>>(a); break;
    }
    DPP_LAUNCH_CHECK("encode_kernel");
    return DPP_OK;
  }
  return dpp::launch_encode_tc(a, channels, batch, nblocks, 1.0f, nullptr, s);
}

int dpp_imgc_encode(const uint8_t* px, int channels, int64_t height, int64_t width, int64_t row_stride,
                    int64_t image_stride, int64_t batch, const float* codebook, int n_cb,
                    int64_t codebook_stride, double sigma_min, uint8_t* records, uint8_t* cb_plane, uint8_t* cr_plane,
                    float* block_grad, float* norm32, void* stream) {
  return encode_common(px, channels, height, width, row_stride, image_stride, batch, codebook, n_cb, codebook_stride,
                       sigma_min, records, nullptr, nullptr, nullptr, cb_plane, cr_plane, block_grad, norm32, stream);
}

int dpp_imgc_encode_planar(const uint8_t* px, int channels, int64_t height, int64_t width, int64_t row_stride,
                           int64_t image_stride, int64_t batch, const float* codebook, int n_cb,
                           int64_t codebook_stride, double sigma_min, uint8_t* mu_plane, uint8_t* sig_plane,
                           uint8_t* idx_plane, uint8_t* cb_plane, uint8_t* cr_plane, void* stream) {
  if (!mu_plane || !sig_plane || !idx_plane) return dpp::fail(DPP_EINVAL, "NULL record plane");
  return encode_common(px, channels, height, width, row_stride, image_stride, batch, codebook, n_cb, codebook_stride,
                       sigma_min, nullptr, mu_plane, sig_plane, idx_plane, cb_plane, cr_plane, nullptr, nullptr,
                       stream);
}

// Test hook: the tensor-core encoder with a scaled pruning band and a count of
// blocks that needed the exact re-check (device counter, accumulated).
int dpp_imgc_encode_tc_debug(const uint8_t* px, int channels, int64_t height, int64_t width, const float* codebook,
                             int n_cb, uint8_t* records, uint8_t* cb_plane, uint8_t* cr_plane, float delta_scale,
                             unsigned long long* ambiguous, void* stream) {
  if (height % 4 || width % 4 || n_cb < 1 || n_cb > 256) return dpp::fail(DPP_EINVAL, "bad geometry");
  if ((height / 4) * (width / 4) > 0xffffffffLL)
    return dpp::fail(DPP_EINVAL, "%lldx%lld has 2^32 or more 4x4 blocks", (long long)width, (long long)height);
  dpp::EncodeArgs a{px, height, width, width * channels, height * width * channels, codebook, n_cb, 0, 0.25,
                    records, cb_plane, cr_plane, nullptr, nullptr, nullptr};
  return dpp::launch_encode_tc(a, channels, 1, (height / 4) * (width / 4), delta_scale, ambiguous,
                               (cudaStream_t)stream);
}

int dpp_imgc_block_stats(const uint8_t* px, int channels, int64_t height, int64_t width, int64_t row_stride,
                         int64_t image_stride, int64_t batch, double sigma_min, double* norm64,
                         float* block_grad, void* stream) {
  if (height % 4 || width % 4 || height < 4 || width < 4)
    return dpp::fail(DPP_EINVAL, "dimensions must be multiples of 4, got %lldx%lld", (long long)width,
                     (long long)height);
  if ((height / 4) * (width / 4) > 0xffffffffLL)
    return dpp::fail(DPP_EINVAL, "%lldx%lld has 2^32 or more 4x4 blocks", (long long)width, (long long)height);
  if (channels != 1 && channels != 3 && channels != 4)
    return dpp::fail(DPP_EINVAL, "channels must be 1, 3 or 4, got %d", channels);
  if (!norm64 || !block_grad) return dpp::fail(DPP_EINVAL, "norm64 and block_grad are required");
  if (batch < 0 || batch > 65535) return dpp::fail(DPP_EINVAL, "batch must be in 0..65535");
  if (batch == 0) return DPP_OK;
  dpp::EncodeArgs a{px, height, width, row_stride, image_stride, nullptr, 0, 0, sigma_min,
                    nullptr, nullptr, nullptr, block_grad, nullptr, norm64};
  const int64_t nblocks = (height / 4) * (width / 4);
  dim3 grid(dpp::grid1(nblocks, 256), (unsigned)batch);
  auto s = (cudaStream_t)stream;
  switch (channels) {
    case 1: dpp::encode_kernel<1, true><<<grid, 256, 0, s>>>(a); break;
    case 3: dpp::encode_kernel<3, true><<<grid, 256, 0, s>>>(a); break;
    default: dpp::encode_kernel<4, true><<<grid, 256, 0, s>>>(a); break;
  }
  DPP_LAUNCH_CHECK("encode_kernel<stats>");
  return DPP_OK;
}

int dpp_imgc_rounding_ties(const uint8_t* px, int channels, int64_t height, int64_t width, int64_t row_stride,
                           int64_t image_stride, int64_t batch, unsigned long long* ties, void* stream) {
  if (height % 4 || width % 4 || height < 4 || width < 4)
    return dpp::fail(DPP_EINVAL, "dimensions must be multiples of 4, got %lldx%lld", (long long)width,
                     (long long)height);
  if ((height / 4) * (width / 4) > 0xffffffffLL)
    return dpp::fail(DPP_EINVAL, "%lldx%lld has 2^32 or more 4x4 blocks", (long long)width, (long long)height);
  if (channels != 1 && channels != 3 && channels != 4)
    return dpp::fail(DPP_EINVAL, "channels must be 1, 3 or 4, got %d", channels);
  if (!ties) return dpp::fail(DPP_EINVAL, "ties is required");
  if (batch < 0 || batch > 65535) return dpp::fail(DPP_EINVAL, "batch must be in 0..65535");
  if (batch == 0) return DPP_OK;
  dpp::EncodeArgs a{px, height, width, row_stride, image_stride, nullptr, 0, 0, 0.25,
                    nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const int64_t nblocks = (height / 4) * (width / 4);
  dim3 grid(dpp::grid1(nblocks, 256), (unsigned)batch);
  auto s = (cudaStream_t)stream;
  switch (channels) {
    case 1: dpp::ties_kernel<1><<<grid, 256, 0, s>>>(a, ties); break;
    case 3: dpp::ties_kernel<3><<<grid, 256, 0, s>>>(a, ties); break;
    default: dpp::ties_kernel<4><<<grid, 256, 0, s>>>(a, ties); break;
  }
  DPP_LAUNCH_CHECK("ties_kernel");
  return DPP_OK;
}

int dpp_imgc_decode(const uint8_t* records, const uint8_t* cb_plane, const uint8_t* cr_plane,
                    const float* codebook, int n_cb, int64_t height, int64_t width, uint8_t* rgb,
                    void* stream) {
  if (height % 4 || width % 4) return dpp::fail(DPP_EINVAL, "dimensions must be multiples of 4");
  if (n_cb < 1 || n_cb > 256) return dpp::fail(DPP_EINVAL, "codebook size must be in 1..256");
  const int64_t n = height * width;
  if (n == 0) return DPP_OK;
  dpp::decode_kernel<<<dpp::grid1(n, 256), 256, 0, (cudaStream_t)stream>>>(records, cb_plane, cr_plane,
                                                                           codebook, height, width, rgb);
  DPP_LAUNCH_CHECK("decode_kernel");
  return DPP_OK;
}

}  // extern "C"
