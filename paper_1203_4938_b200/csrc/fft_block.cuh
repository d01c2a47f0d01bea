// Block-level Stockham FFT building block shared by the 1-D and 2-D kernels.
#pragma once

#include "common.cuh"

namespace dpp {

// ---------------------------------------------------------------------------
// Block-level Stockham FFT.
//
// Size-M transform computed by T = M/R threads.  On entry thread j holds
// v[i] = x[j + T*i]; on exit v[i] = X[j + T*i] (natural order, strided).
// Pass with current sub-transform size Ns (Govindaraju et al. 2008):
//   twiddle v[i] *= W_{Ns*R}^{i*(j mod Ns)}; DFT_R; write to
//   (j div Ns)*Ns*R + (j mod Ns) + i*Ns; read back v[i] = buf[j + T*i].
// When log2 M is not a multiple of log2 R, one leading radix-2^(rem) pass is
// done on the registers as it arrives from memory (no exchange before it).
// `map` turns a logical element index into a shared-memory offset; `tw` is a
// W_{M*tw_step} table so that W_M^e = tw[e*tw_step].

struct MapIdentity {
  __device__ __forceinline__ int operator()(int e) const { return e; }
};
struct MapPad16 {  // one float2 of padding per 16 elements: breaks stride-16 bank aliasing
  __device__ __forceinline__ int operator()(int e) const { return e + (e >> 4); }
};

// twiddle multiply from a table entry: float2 = w (rotation built on the fly),
// float4 = (w, i*w) precomputed so the product is exactly FMUL2 + FFMA2
__device__ __forceinline__ float2 twmul(float2 v, float2 w) { return cmul(v, w); }
__device__ __forceinline__ float2 twmul(float2 v, float4 w) {
  return cmul_pre(v, make_float2(w.x, w.y), make_float2(w.z, w.w));
}

template <int M, int R, class Map, class TW>
__device__ __forceinline__ void block_fft(float2 (&v)[R], int j, float2* buf, Map map,
                                          const TW* tw, int tw_step) {
  constexpr int T = M / R;
  constexpr int LOGM = ilog2(M);
  constexpr int LOGR = ilog2(R);
  constexpr int REM = LOGM % LOGR;
  constexpr int NPASS = LOGM / LOGR;
  constexpr int NS0 = 1 << REM;
  if constexpr (REM != 0) {
    constexpr int r = 1 << REM;
    constexpr int S = R / r;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float2 u[r];
#pragma unroll
      for (int q = 0; q < r; ++q) u[q] = v[s + q * S];
      dft_r<r>(u);
      const int jp = j + T * s;
#pragma unroll
      for (int q = 0; q < r; ++q) buf[map(jp * r + q)] = u[q];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = buf[map(j + T * i)];
    __syncthreads();
  }
#pragma unroll
  for (int pass = 0; pass < NPASS; ++pass) {
    const int ns = NS0 << (LOGR * pass);
    const int jm = j & (ns - 1);
    if (ns > 1) {
      const int unit = jm * (M / (ns * R));
#pragma unroll
      for (int i = 1; i < R; ++i) v[i] = twmul(v[i], tw[(i * unit) * tw_step]);
    }
    dft_r<R>(v);
    if (ns * R < M) {
      const int base = (j - jm) * R + jm;
#pragma unroll
      for (int i = 0; i < R; ++i) buf[map(base + i * ns)] = v[i];
      __syncthreads();
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = buf[map(j + T * i)];
      __syncthreads();
    }
  }
}

}  // namespace dpp

namespace dpp {

// ---------------------------------------------------------------------------
// Column-pair variant: each thread runs the same Stockham schedule on TWO
// adjacent columns (v0 = column 2cp, v1 = column 2cp+1).  Exchanges use a
// row-major [element][W] layout, so every shared-memory access is one
// 16-byte LDS.128/STS.128 of a column pair and a half-warp (16 column pairs)
// covers one contiguous 256-byte row: conflict-free without padding, and
// half the shared-memory instructions of the single-column form.
template <int M, int R, int W>
__device__ __forceinline__ void block_fft_pair(float2 (&v0)[R], float2 (&v1)[R], int j, int cp, float2* buf,
                                               const float2* tw, int tw_step) {
  constexpr int T = M / R;
  constexpr int LOGM = ilog2(M);
  constexpr int LOGR = ilog2(R);
  constexpr int REM = LOGM % LOGR;
  constexpr int NPASS = LOGM / LOGR;
  constexpr int NS0 = 1 << REM;
  float4* row = reinterpret_cast<float4*>(buf) + cp;  // element e of the pair at row[e * (W / 2)]
  constexpr int RS = W / 2;
  if constexpr (REM != 0) {
    constexpr int r = 1 << REM;
    constexpr int S = R / r;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float2 u0[r], u1[r];
#pragma unroll
      for (int q = 0; q < r; ++q) {
        u0[q] = v0[s + q * S];
        u1[q] = v1[s + q * S];
      }
      dft_r<r>(u0);
      dft_r<r>(u1);
      const int jp = j + T * s;
#pragma unroll
      for (int q = 0; q < r; ++q) row[(jp * r + q) * RS] = make_float4(u0[q].x, u0[q].y, u1[q].x, u1[q].y);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float4 t = row[(j + T * i) * RS];
      v0[i] = make_float2(t.x, t.y);
      v1[i] = make_float2(t.z, t.w);
    }
    __syncthreads();
  }
#pragma unroll
  for (int pass = 0; pass < NPASS; ++pass) {
    const int ns = NS0 << (LOGR * pass);
    const int jm = j & (ns - 1);
    if (ns > 1) {
      const int unit = jm * (M / (ns * R));
#pragma unroll
      for (int i = 1; i < R; ++i) {
        const float2 w = tw[(i * unit) * tw_step];
        v0[i] = cmul(v0[i], w);
        v1[i] = cmul(v1[i], w);
      }
    }
    dft_r<R>(v0);
    dft_r<R>(v1);
    if (ns * R < M) {
      const int base = (j - jm) * R + jm;
#pragma unroll
      for (int i = 0; i < R; ++i) row[(base + i * ns) * RS] = make_float4(v0[i].x, v0[i].y, v1[i].x, v1[i].y);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const float4 t = row[(j + T * i) * RS];
        v0[i] = make_float2(t.x, t.y);
        v1[i] = make_float2(t.z, t.w);
      }
      __syncthreads();
    }
  }
}

}  // namespace dpp
