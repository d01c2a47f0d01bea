// 2-D column pass through the L2 exchange ring (columns of R = 256 * B rows,
// B = 16: 4096-row images, B = 64: 16384-row images).
//
// The column FFT of length R for a tile of 16 adjacent columns is a four-step
// with r = 256 b + a (a < 256, b < B) and k = k1 + B k2:
//   P1(u, g): rows r = 256 b + a for the A = 4096 / (16 B) values a in
//             [A g, A g + A) and every b — one 3-D TMA box (16 x A x B) —
//             B-point FFTs over b (B = 16: one sequence per thread, no
//             exchange; B = 64: 4 lanes per sequence, one in-warp exchange),
//             twiddle W_R^{a k1}, written to the ring slot of unit u as
//             S[k1][a][16 columns] (128B-swizzled rows).
//   P2(u, k1): the 32 KB block S[k1] by one bulk copy, 256-point FFTs over a
//             (exactly the 1-D kernel's P2, csrc/fft_l2.cu), output rows
//             k1 + B k2 by one 3-D TMA store (16 x 1 x 256).
// A unit u is one (image, 16-column tile); P1 and P2 each have B items per
// unit, ordered, published and waited for exactly like the 1-D kernel's
// transforms (same producer / compute-warp structure, same deadlock argument).
// In place: P2(u) writes unit u's columns only after every P1(u) has read them.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "l2ring.cuh"
#include "tma.cuh"

namespace dpp {
namespace colring {

using namespace ring;

constexpr int CW = 8;
constexpr int THREADS = (CW + 1) * 32;
constexpr int TILE = 4096;
constexpr int S = 2;

struct Args {
  float2* scratch;
  int* ctrl;
  const float2* twr;   // W_R^m, m < R
  const float4* tw256; // W256^m as (w, i*w), m < 256
  int units, tiles_per_image, lag, ring;
  float alpha;         // SPEC: spectrum_u8 scale
  int np, col0, tb;    // PEER: ranks, first column of this rank's block, output to the row slabs
  const float2* twlo;  // TW: W_N^m for m < 16384 ...
  const float2* twhi;  //     ... and W_N^(16384 h): W_N^m = twlo[m & 16383] * twhi[m >> 14]
  float2* side = nullptr;  // SPEC on a pair array (non-null): column 0 of each half, raw, for spectrum_pair_fixup
};

// TW (1-D transforms above 2^17, csrc/fft_large.cu): the four-step twiddle
// W_N^{r k1} of the column-length (row r) x row-length (column k1) split,
// applied to the loaded values before the column FFT
__device__ __forceinline__ float2 tw_big(const Args& a, uint32_t m) {
  return cmul(__ldg(a.twlo + (m & 16383u)), __ldg(a.twhi + (m >> 14)));
}
template <bool TW>
__device__ __forceinline__ void p1_twiddle(float2 (&v)[16], const Args& a, uint32_t m0, uint32_t step) {
  if constexpr (TW) {
    float2 w = tw_big(a, m0);
    const float2 st = tw_big(a, step);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = cmul(v[j], w);
      w = cmul(w, st);
    }
  }
}

// PEER: one tensor map per rank (row slabs in, row slabs or the local column slab out)
struct Maps8 {
  CUtensorMap m[8];
};
template <bool PEER>
struct MapSet {
  using type = CUtensorMap;
};
template <>
struct MapSet<true> {
  using type = Maps8;
};
__device__ __forceinline__ const CUtensorMap* map_at(const CUtensorMap& m, int) { return &m; }
__device__ __forceinline__ const CUtensorMap* map_at(const Maps8& m, int j) { return &m.m[j]; }

// XP (the first pass of the two-pass large 1-D transform, csrc/fft_large.cu):
// the ring slot is laid out S[column][k1 / 16][a][k1 % 16] instead of
// S[k1][a][column], so a P2 block is one column's 16 consecutive k1 over all
// a, and its output (16 k1 x 256 k2 of ONE column) is a 128-byte-row box of
// the transposed result T[column][k1 + B k2]: (col, a, k1) sits at
// 4096 (col B/16 + k1/16) + swz(a, k1 % 16) of the slot.

// P1, B = 16: thread = one (column, a) sequence over b; no exchange
template <bool TW = false, bool XP = false>
__device__ __forceinline__ void p1_b16(float2 (&v)[16], uint32_t b, int warp, int lane, int g, float2* slot,
                                       const Args& a, uint64_t keep_pol, int colbase = 0) {
  const int col = lane & 15, alo = 2 * warp + (lane >> 4);
  const int ar = 16 * g + alo;
#pragma unroll
  for (int bb = 0; bb < 16; ++bb) v[bb] = lds64(b + 8u * swz(16 * bb + alo, col));
  {
    const uint32_t kc = (uint32_t)(colbase + col);  // rows 256 bb + ar
    p1_twiddle<TW>(v, a, (uint32_t)ar * kc, 256u * kc);
  }
  dft16c(v);  // v[k1]
  const float2 wa = __ldg(a.twr + ar);  // W_R^a
  float2 w = wa;
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
    v[k1] = cmul(v[k1], w);
    w = cmul(w, wa);
  }
  if constexpr (XP) {
    // one 128-byte row: k1 = 0..15 of (col, a), four whole 32-byte sectors;
    // k1 = 4 g .. 4 g + 3 lands in sector g ^ ((a & 7) >> 1), chunk pair
    // swapped when a is odd (the 128B swizzle)
    float2* dst = slot + 4096 * col + 16 * ar;
    const bool odd = ar & 1;
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4)
      st_l2_hint4(dst + 4 * (g4 ^ ((ar & 7) >> 1)), odd ? v[4 * g4 + 2] : v[4 * g4], odd ? v[4 * g4 + 3] : v[4 * g4 + 1],
                  odd ? v[4 * g4] : v[4 * g4 + 2], odd ? v[4 * g4 + 1] : v[4 * g4 + 3], keep_pol);
  } else {
    float2* dst = slot + swz(ar, col);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) st_l2_hint(dst + 4096 * k1, v[k1], keep_pol);
  }
}

// P1, B = 64: four lanes per (column, a) sequence; b = 4 b1 + b0 with b1 in
// registers, k1 = m0 + 16 m1.  Exchange slot of (b0, m0): row 4 beta + a_lo,
// beta = g(m0) ^ b0, g(m0) = 4 m0 | ((m0 >> 2) & 1): both the write (fixed m0)
// and the read (fixed b0) give a half-warp 2 distinct row parities x 8 columns
// = 16 distinct bank pairs.
__device__ __forceinline__ int gbeta(int m0) { return (m0 << 2) | ((m0 >> 2) & 1); }

template <bool TW = false, bool XP = false>
__device__ __forceinline__ void p1_b64(float2 (&v)[16], uint32_t b, int warp, int lane, int g, float2* slot,
                                       const Args& a, uint64_t keep_pol, int colbase = 0) {
  const int alo = warp >> 1, col = 8 * (warp & 1) + (lane & 7), b0 = lane >> 3;
#pragma unroll
  for (int b1 = 0; b1 < 16; ++b1) v[b1] = lds64(b + 8u * swz(16 * b1 + 4 * b0 + alo, col));
  {
    const uint32_t kc = (uint32_t)(colbase + col);  // rows 256 (4 b1 + b0) + 4 g + alo
    p1_twiddle<TW>(v, a, (uint32_t)(256 * b0 + 4 * g + alo) * kc, 1024u * kc);
  }
  dft16c(v);  // v[m0]
  {
    const float2 wb = __ldg(a.twr + 256 * b0);  // W64^b0 = W_R^{256 b0}
    float2 w = wb;
#pragma unroll
    for (int m0 = 1; m0 < 16; ++m0) {
      v[m0] = cmul(v[m0], w);
      w = cmul(w, wb);
    }
  }
  __syncwarp();
#pragma unroll
  for (int m0 = 0; m0 < 16; ++m0) sts64(b + 8u * swz(4 * (gbeta(m0) ^ b0) + alo, col), v[m0]);
  __syncwarp();
  const int j = b0;  // after the exchange this lane owns m0 = 4 j + i
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) v[4 * i + c] = lds64(b + 8u * swz(4 * (gbeta(4 * j + i) ^ c) + alo, col));
#pragma unroll
  for (int i = 0; i < 4; ++i) dft4c(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);  // v[4 i + m1]
  // W_R^{a k1}, a = 4 g + a_lo, k1 = 4 j + i + 16 m1
  const int ar = 4 * g + alo;
  const float2 s1 = __ldg(a.twr + ar), s16 = __ldg(a.twr + 16 * ar);
  float2 wi = __ldg(a.twr + 4 * ar * j);
  float2* base = slot + swz(ar, col);
  if constexpr (XP) {
    // k1 = 4 j + i + 16 m1: this lane holds k1 % 16 = 4 j .. 4 j + 3 of every
    // m1 — one whole 32-byte sector of row (col, m1, a): sector j ^ ((a & 7)
    // >> 1), chunk pair swapped when a is odd
    float2 wv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      wv[i] = wi;
      wi = cmul(wi, s1);
    }
    const bool odd = ar & 1;
#pragma unroll
    for (int m1 = 0; m1 < 4; ++m1) {
      float2 e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        e[i] = cmul(v[4 * i + m1], wv[i]);
        wv[i] = cmul(wv[i], s16);
      }
      st_l2_hint4(slot + 4096 * (4 * col + m1) + 16 * ar + 4 * (j ^ ((ar & 7) >> 1)), odd ? e[2] : e[0],
                  odd ? e[3] : e[1], odd ? e[0] : e[2], odd ? e[1] : e[3], keep_pol);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 w = wi;
#pragma unroll
      for (int m1 = 0; m1 < 4; ++m1) {
        st_l2_hint(base + 4096 * (4 * j + i + 16 * m1), cmul(v[4 * i + m1], w), keep_pol);
        w = cmul(w, s16);
      }
      wi = cmul(wi, s1);
    }
  }
}

// P1 for B = 4 and 8 (1024- and 2048-row images): S = 16 / B whole sequences
// per thread, in registers (the B = 16 pattern with A = 16 S a-values per
// item): thread (col, t) owns a = t + 16 s, s < S.
// TW: tile row A bb + t + 16 s is row 256 bb + ar of the column (the box
// takes rows A g .. A g + A of each 256-row block), twiddled by W_N^{row kc}.
template <int B, bool TW = false>
__device__ __forceinline__ void p1_bsmall(float2 (&v)[16], uint32_t b, int warp, int lane, int g, float2* slot,
                                          const Args& a, uint64_t keep_pol, int colbase = 0) {
  constexpr int S = 16 / B, A = 16 * S;
  const int col = lane & 15, t = 2 * warp + (lane >> 4);
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int bb = 0; bb < B; ++bb) v[s * B + bb] = lds64(b + 8u * swz(A * bb + t + 16 * s, col));
  if constexpr (TW) {
    const uint32_t kc = (uint32_t)(colbase + col);
    const float2 st = tw_big(a, 256u * kc);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float2 w = tw_big(a, (uint32_t)(A * g + t + 16 * s) * kc);
#pragma unroll
      for (int bb = 0; bb < B; ++bb) {
        v[s * B + bb] = cmul(v[s * B + bb], w);
        w = cmul(w, st);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    if constexpr (B == 8) {
      float2 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) u[q] = v[s * 8 + q];
      dft8(u);
#pragma unroll
      for (int q = 0; q < 8; ++q) v[s * 8 + q] = u[q];
    } else {
      dft4c(v[s * 4], v[s * 4 + 1], v[s * 4 + 2], v[s * 4 + 3]);
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int ar = A * g + t + 16 * s;
    const float2 wa = __ldg(a.twr + ar);  // W_R^a
    float2 w = wa;
#pragma unroll
    for (int k1 = 1; k1 < B; ++k1) {
      v[s * B + k1] = cmul(v[s * B + k1], w);
      w = cmul(w, wa);
    }
    float2* dst = slot + swz(ar, col);
#pragma unroll
    for (int k1 = 0; k1 < B; ++k1) st_l2_hint(dst + 4096 * k1, v[s * B + k1], keep_pol);
  }
}

// P1 for B = 32 and 128: L = B / 16 lanes per (column, a) sequence, the
// B = 64 pattern above with general L (b = L b1 + b0, k1 = m0 + 16 m1, lane j
// owns m0 = Q j + ii, Q = 16 / L; exchange slot beta = gL(m0) ^ b0 with
// gL(m0) = L m0 | ((m0 / Q) & (L/2 - 1)), as in csrc/fft16k_l2.cu).
template <int L>
__device__ __forceinline__ int gbetaL(int m0) {
  constexpr int Q = 16 / L;
  return L * m0 | ((m0 / Q) & (L / 2 - 1));
}
template <int L>
__device__ __forceinline__ void dftLc(float2* v) {
  if constexpr (L == 2) {
    const float2 t = v[0];
    v[0] = make_float2(t.x + v[1].x, t.y + v[1].y);
    v[1] = make_float2(t.x - v[1].x, t.y - v[1].y);
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
// TW: tile row 16 b1 + A b0 + alo is row 256 (L b1 + b0) + ar of the column.
template <int L, bool TW = false, bool XP = false>
__device__ __forceinline__ void p1_bL(float2 (&v)[16], uint32_t b, int warp, int lane, int g, float2* slot,
                                      const Args& a, uint64_t keep_pol, int colbase = 0) {
  constexpr int A = 16 / L, Q = 16 / L;  // a values per item (A * L = 16), m0 values per lane
  // 256 threads = 16 columns x A a-values x L lanes
  constexpr int SPW = 32 / L;  // sequences per warp
  const int b0 = lane / SPW;
  const int rest = warp * SPW + lane % SPW;  // 0 .. 256 / L - 1: (a, column) of the sequence
  const int col = rest & 15, alo = (rest >> 4) & (A - 1);
#pragma unroll
  for (int b1 = 0; b1 < 16; ++b1) v[b1] = lds64(b + 8u * swz(16 * b1 + A * b0 + alo, col));
  {
    const uint32_t kc = (uint32_t)(colbase + col);
    p1_twiddle<TW>(v, a, (uint32_t)(256 * b0 + A * g + alo) * kc, 256u * L * kc);
  }
  dft16c(v);  // v[m0]
  {
    const float2 wb = __ldg(a.twr + 256 * b0);  // W_B^b0 = W_R^{256 b0}
    float2 w = wb;
#pragma unroll
    for (int m0 = 1; m0 < 16; ++m0) {
      v[m0] = cmul(v[m0], w);
      w = cmul(w, wb);
    }
  }
  __syncwarp();
#pragma unroll
  for (int m0 = 0; m0 < 16; ++m0) sts64(b + 8u * swz(A * (gbetaL<L>(m0) ^ b0) + alo, col), v[m0]);
  __syncwarp();
  const int j = b0;  // after the exchange this lane owns m0 = Q j + ii
#pragma unroll
  for (int ii = 0; ii < Q; ++ii)
#pragma unroll
    for (int c = 0; c < L; ++c) v[L * ii + c] = lds64(b + 8u * swz(A * (gbetaL<L>(Q * j + ii) ^ c) + alo, col));
#pragma unroll
  for (int ii = 0; ii < Q; ++ii) dftLc<L>(v + L * ii);  // v[L ii + m1]
  // W_R^{a k1}, a = A g + alo, k1 = Q j + ii + 16 m1
  const int ar = A * g + alo;
  const float2 s1 = __ldg(a.twr + ar), s16 = __ldg(a.twr + 16 * ar);
  float2 wi = __ldg(a.twr + Q * ar * j);
  if constexpr (XP) {
    // this lane holds k1 % 16 = Q j .. Q j + Q - 1 of every m1: whole 32-byte
    // sectors (Q = 8: two) or one 16-byte chunk (Q = 2) of row (col, m1, a)
    float2 wv[Q];
#pragma unroll
    for (int ii = 0; ii < Q; ++ii) {
      wv[ii] = wi;
      wi = cmul(wi, s1);
    }
    const bool odd = ar & 1;
#pragma unroll
    for (int m1 = 0; m1 < L; ++m1) {
      float2 e[Q];
#pragma unroll
      for (int ii = 0; ii < Q; ++ii) {
        e[ii] = cmul(v[L * ii + m1], wv[ii]);
        wv[ii] = cmul(wv[ii], s16);
      }
      float2* row = slot + 4096 * (col * L + m1) + 16 * ar;
      if constexpr (Q >= 4) {
#pragma unroll
        for (int h = 0; h < Q / 4; ++h)
          st_l2_hint4(row + 4 * ((Q * j / 4 + h) ^ ((ar & 7) >> 1)), odd ? e[4 * h + 2] : e[4 * h],
                      odd ? e[4 * h + 3] : e[4 * h + 1], odd ? e[4 * h] : e[4 * h + 2],
                      odd ? e[4 * h + 1] : e[4 * h + 3], keep_pol);
      } else {
        st_l2_hint2(row + 2 * (j ^ (ar & 7)), e[0], e[1], keep_pol);
      }
    }
  } else {
    float2* base = slot + swz(ar, col);
#pragma unroll
    for (int ii = 0; ii < Q; ++ii) {
      float2 w = wi;
#pragma unroll
      for (int m1 = 0; m1 < L; ++m1) {
        st_l2_hint(base + 4096 * (Q * j + ii + 16 * m1), cmul(v[L * ii + m1], w), keep_pol);
        w = cmul(w, s16);
      }
      wi = cmul(wi, s1);
    }
  }
}

// SPEC: the C5 chain's spectrum_u8 node fused into the output: P2 stages
// u8 = spectrum(X) (a 16 x 256 byte tile per stage) and TMA-stores bytes.
//
// PEER (row-sharded C3): the all-to-all is fused into this pass.
// Rank j holds rows [j R/P, (j+1) R/P) = b in [j B/P, (j+1) B/P) of every
// image in its own row slab; the P1 box is P sub-boxes, one TMA load from each
// rank's slab (peer-mapped: NVLink reads), landing at 1024-byte-aligned
// offsets of the stage so the 128B swizzle is unchanged.  P2 either stores
// the 256 output rows of its k1 as P sub-boxes into the ranks' row slabs
// (tb: natural row-sharded output, in place is safe because column block q is
// touched by rank q only) or one box into the local R x (C/P) column slab.
template <int B, bool DISCARD, bool SPEC = false, bool PEER = false, bool TW = false, bool XP = false>
__global__ void __launch_bounds__(THREADS, 3)
fft_cols_l2w(const __grid_constant__ typename MapSet<PEER>::type tin,
             const __grid_constant__ typename MapSet<PEER>::type tout, const Args a) {
  constexpr int A = TILE / (16 * B);  // a values per P1 item
  constexpr int LOGB = B == 4 ? 2 : (B == 8 ? 3 : (B == 16 ? 4 : (B == 32 ? 5 : (B == 64 ? 6 : 7))));
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  __shared__ int s_tick[S];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int total = 2 * B * a.units;
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
  const int R = 256 * B;

  if (warp == CW) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    const uint64_t stream_pol = policy_evict_first();
    int head = 0, i = 0;
    auto publish = [&](int k) {
      const int s = k % S;
      int pass, u;
      decode(s_tick[s] >> LOGB, a.units, a.lag, pass, u);
      const int g = s_tick[s] & (B - 1);
      if (pass == 1) {
        red_release_add(cnt1 + u, 1);
      } else {
        if (u + a.ring < a.units) red_release_add(cnt2 + u, 1);  // lines discarded by the compute warps
        const int img = u / a.tiles_per_image, ct = u - img * a.tiles_per_image;
        if constexpr (PEER) {
          if (a.tb) {
            const int kk = 256 / a.np;
            for (int j = 0; j < a.np; ++j)
              tma_store_3d(map_at(tout, j), a.col0 + 16 * ct, g, img * kk, smem + s * TILE + j * (TILE / a.np));
          } else {
            tma_store_3d(map_at(tout, 0), 16 * ct, g, img * 256, smem + s * TILE);
          }
        } else if constexpr (XP) {
          // P2 block g = (column, k1 / 16): row img C + 16 ct + column of T, viewed [k2][k1]
          const int C = 16 * a.tiles_per_image;
          tma_store_3d(&tout, 16 * (g % (B / 16)), 0, img * C + 16 * ct + g / (B / 16), smem + s * TILE);
        } else if (SPEC && a.side) {
          // pair array: column tile ct of half h is image 2 img + h's columns
          // c0 .. c0 + 15
          const int half = a.tiles_per_image / 2, h = ct >= half, c0 = 16 * (ct - h * half);
          tma_store_3d(&tout, c0, g, (2 * img + h) * 256,
                       reinterpret_cast<const uint8_t*>(smem + S * TILE) + s * 4096);
        } else {
          tma_store_3d(&tout, 16 * ct, g, img * 256,
                       SPEC ? reinterpret_cast<const void*>(reinterpret_cast<const uint8_t*>(smem + S * TILE) +
                                                            s * 4096)
                            : reinterpret_cast<const void*>(smem + s * TILE));
        }
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
      decode(tick >> LOGB, a.units, a.lag, pass, u);
      const int g = tick & (B - 1);
      const int* dep = pass == 2 ? cnt1 + u : (u >= a.ring ? cnt2 + (u - a.ring) : nullptr);
      if (dep) {
        while (ld_acquire(dep) < B) {
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
        const int img = u / a.tiles_per_image, ct = u - img * a.tiles_per_image;
        if constexpr (PEER) {
          const int nb = B / a.np;
          for (int j = 0; j < a.np; ++j)
            tma_load_3d(buf + j * (TILE / a.np), map_at(tin, j), a.col0 + 16 * ct, A * g, img * nb, &full[s]);
        } else {
          tma_load_3d(buf, &tin, 16 * ct, A * g, img * B, &full[s]);
        }
      } else {
        fence_proxy_async_global();
        bulk_g2s(buf, a.scratch + (size_t)(u & (a.ring - 1)) * (16 * R) + 4096 * g, TILE * sizeof(float2),
                 &full[s]);
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
  // P2 = the 1-D kernel's P2 (warp w owns columns 2w, 2w+1; half-warp = 8 rows
  // x 2 columns; XOR-immediate exchange addresses), see csrc/fft_l2.cu.
  const int col = 2 * warp + (lane & 1);
  const int idx = lane >> 1;
  const int q = idx & 7, p = lane & 1;
  const uint32_t x9 = 16u * (uint32_t)((9 * q) ^ warp);
  const uint32_t offA = 128u * idx + 16u * (uint32_t)(warp ^ q) + 8u * p;
  const uint32_t offW = 2048u * idx + 8u * p + x9;
  const uint32_t offR = 1024u * (idx >> 3) + 8u * p + x9;
  const uint32_t sbase = smem_u32(smem);
  const uint64_t keep_pol = policy_evict_last();
  const float4 t1 = __ldg(a.tw256 + idx);
  const float2 w1 = make_float2(t1.x, t1.y);  // W256^idx
  float2 v[16];
  for (int i = 0;; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const int tick = s_tick[s];
    if (tick < 0) break;
    int pass, u;
    decode(tick >> LOGB, a.units, a.lag, pass, u);
    const int g = tick & (B - 1);
    const uint32_t b = sbase + (uint32_t)s * (TILE * 8);
    float2* slot = a.scratch + (size_t)(u & (a.ring - 1)) * (16 * R);
    if (pass == 1) {
      const int colbase = TW ? 16 * (u - (u / a.tiles_per_image) * a.tiles_per_image) : 0;
      if constexpr (B == 16)
        p1_b16<TW, XP>(v, b, warp, lane, g, slot, a, keep_pol, colbase);
      else
        if constexpr (B == 64)
          p1_b64<TW, XP>(v, b, warp, lane, g, slot, a, keep_pol, colbase);
        else if constexpr (B < 16)
          p1_bsmall<B, TW>(v, b, warp, lane, g, slot, a, keep_pol, colbase);
        else
          p1_bL<B / 16, TW, XP>(v, b, warp, lane, g, slot, a, keep_pol, colbase);
    } else {
      if (DISCARD) discard_l2(slot + 4096 * g + 16 * (tid & 255));
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
      dft16c(v);
      if constexpr (SPEC) {
        if (a.side) {
          // pair array (fft4096_ws<PAIR> rows): the column is column c of one
          // image's half spectrum (the mirrored half is spectrum_pair_mirror's).
          // Column 0 of each half carries the packed DC / Nyquist columns: raw
          // values to the side buffer for spectrum_pair_fixup.
          const int half = a.tiles_per_image / 2;
          const int img = u / a.tiles_per_image, ct = u - img * a.tiles_per_image, h = ct >= half;
          if (col == 0 && ct - h * half == 0) {
            float2* sd = a.side + (size_t)(2 * img + h) * R + g;
#pragma unroll
            for (int d1 = 0; d1 < 16; ++d1) sd[B * (idx + 16 * d1)] = v[d1];
          }
        }
        {
          uint8_t* o = reinterpret_cast<uint8_t*>(smem + S * TILE) + s * 4096 + 16 * idx + col;
#pragma unroll
          for (int d1 = 0; d1 < 16; ++d1) o[256 * d1] = spectrum_u8_one(v[d1].x, v[d1].y, a.alpha);  // row k2
        }
      } else {
        __syncwarp();
#pragma unroll
        for (int d1 = 0; d1 < 16; ++d1) sts64(bA + 2048 * d1, v[d1]);  // output row k2 = idx + 16 d1
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive1(&done[s]);
  }
}

}  // namespace colring

// ---------------------------------------------------------------------------
// host side

static int g_col_discard = -1;

static size_t colring_smem(bool spec = false) {
  return (size_t)colring::S * (colring::TILE * sizeof(float2) + (spec ? 4096 : 0));
}

template <int B>
static int colring_prepare(int* ctas) {
  const size_t smem = colring_smem();
  DPP_CUDA_CHECK(cudaFuncSetAttribute(colring::fft_cols_l2w<B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  DPP_CUDA_CHECK(cudaFuncSetAttribute(colring::fft_cols_l2w<B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  DPP_CUDA_CHECK(cudaFuncSetAttribute(colring::fft_cols_l2w<B, true, false, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if constexpr (B == 16 || B == 64)  // the fused spectrum (4096 / 16384 rows)
    DPP_CUDA_CHECK(cudaFuncSetAttribute(colring::fft_cols_l2w<B, true, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)colring_smem(true)));
  // the four-step twiddle (every ring length)
  DPP_CUDA_CHECK(cudaFuncSetAttribute(colring::fft_cols_l2w<B, true, false, false, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if constexpr (B >= 16) {  // transposed output (first pass of the two-pass large 1-D transform)
    DPP_CUDA_CHECK(cudaFuncSetAttribute(colring::fft_cols_l2w<B, true, false, false, false, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  int per_sm = 0, dev = 0, sms = 0;
  DPP_CUDA_CHECK(
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, colring::fft_cols_l2w<B, true>, colring::THREADS, smem));
  DPP_CUDA_CHECK(cudaGetDevice(&dev));
  DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(DPP_ECUDA, "fft_cols_l2w does not fit on an SM");
  *ctas = per_sm * sms;
  return DPP_OK;
}

// Set up the column ring for an n0-row, n1-column rank-2 plan; returns
// DPP_ENOTSUP (plan falls back to the cluster column kernel) when the shape
// has no ring schedule.
int fft2d_colring_init(FftPlan* p) {
  const int64_t R = p->n0;
  if (!(R == 1024 || R == 2048 || R == 4096 || R == 8192 || R == 16384 || R == 32768) || p->n1 % 16)
    return DPP_ENOTSUP;
  g_col_discard = 1;
  const int B = (int)(R / 256);
  int rc = B == 4    ? colring_prepare<4>(&p->col_ring_ctas)
           : B == 8  ? colring_prepare<8>(&p->col_ring_ctas)
           : B == 16 ? colring_prepare<16>(&p->col_ring_ctas)
                   : B == 32 ? colring_prepare<32>(&p->col_ring_ctas)
                             : B == 64 ? colring_prepare<64>(&p->col_ring_ctas)
                                       : colring_prepare<128>(&p->col_ring_ctas);
  if (rc) return rc;
  p->l2_lag = ring_stress() ? 2 : 768 / B;
  int ring = 1;
  while (ring < 2 * p->l2_lag + 8) ring <<= 1;
  p->l2_ring = ring;
  const int64_t units = p->batch * (p->n1 / 16);
  if (units > 0x7fffffff / (2 * B)) return fail(DPP_EINVAL, "2-D batch too large for the column ring");
  std::vector<float2> twr((size_t)R);
  for (int64_t m = 0; m < R; ++m) {
    const double ang = -2.0 * M_PI * (double)m / (double)R;
    twr[(size_t)m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  std::vector<float4> t256(256);
  for (int m = 0; m < 256; ++m) {
    const double ang = -2.0 * M_PI * (double)m / 256.0;
    const float c = (float)std::cos(ang), s = (float)std::sin(ang);
    t256[(size_t)m] = make_float4(c, s, -s, c);
  }
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_tw, 256 * sizeof(float4) + (size_t)R * sizeof(float2)));
  DPP_CUDA_CHECK(cudaMemcpy(p->l2_tw, t256.data(), 256 * sizeof(float4), cudaMemcpyHostToDevice));
  DPP_CUDA_CHECK(cudaMemcpy(reinterpret_cast<float2*>(p->l2_tw + 256), twr.data(), (size_t)R * sizeof(float2),
                            cudaMemcpyHostToDevice));
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_scratch, (size_t)ring * 16 * R * sizeof(float2)));
  p->l2_ctrl_bytes = (32 + 2 * (size_t)(units > 0 ? units : 1)) * sizeof(int);
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_ctrl, p->l2_ctrl_bytes));
  DPP_CUDA_CHECK(cudaEventCreateWithFlags(&p->l2_done, cudaEventDisableTiming));
  p->col_ring = 1;
  return DPP_OK;
}

// The DC / Nyquist columns of a pair array's spectra: side holds the column
// FFT of (A'[r][0]) = (A[r][0], A[r][N/2]) per image, C[k] = P[k] + i Q[k]
// with P, Q the (Hermitian) spectra of the two real columns; separated as in
// the row pass and written to columns 0 and C/2.
__global__ void __launch_bounds__(256) spectrum_pair_fixup(const float2* __restrict__ side, uint8_t* __restrict__ out,
                                                           int rows, int cols, int64_t n, float alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t img = i / rows;
  const int k = (int)(i - img * rows);
  const float2 z = side[i], zm = side[img * rows + ((rows - k) & (rows - 1))];
  uint8_t* o = out + (size_t)i * cols;
  o[0] = spectrum_u8_one(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y), alpha);
  o[cols / 2] = spectrum_u8_one(0.5f * (z.y + zm.y), 0.5f * (zm.x - z.x), alpha);
}

// The mirrored half of pair spectra: out[k][x] = out[(-k) mod R][C - x] for
// x = C/2 + 1 .. C - 1 (|X[-k][C-x]| = |X[k][x]| for a real image).  One
// thread per 16-byte output chunk q = C/32 + m of row k: byte i is column
// c = C - 16q - i of row -k, i.e. byte 16 - i of source chunk a = C/16 - 1 - q
// (i >= 1) and byte 0 of chunk a + 1 (i = 0).  (Written in the column ring's
// epilogue instead, the mirror starts one byte past a 16-byte boundary — TMA
// rejects it — and per-row byte-split stores cost 1 ms per 64 images.)  Byte 0
// of chunk C/32 is column C/2: spectrum_pair_fixup, which runs after this.
__global__ void __launch_bounds__(256) spectrum_pair_mirror(uint8_t* __restrict__ out, int rows, int cols,
                                                            int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cq = cols / 32;
  const int64_t row = i / cq;
  const int q = cq + (int)(i - row * cq), a = 2 * cq - 1 - q;
  const int64_t img = row / rows;
  const int k = (int)(row - img * rows);
  const uint8_t* src = out + ((size_t)img * rows + ((rows - k) & (rows - 1))) * cols;
  const uint4 lo = *reinterpret_cast<const uint4*>(src + 16 * a);
  const uint32_t b0 = src[16 * (a + 1)];
  uint4 w;
  w.x = __byte_perm(b0, lo.w, 0x5670);  // [b0, lo15, lo14, lo13]
  w.y = __byte_perm(lo.w, lo.z, 0x5670);
  w.z = __byte_perm(lo.z, lo.y, 0x5670);
  w.w = __byte_perm(lo.y, lo.x, 0x5670);  // [lo4, lo3, lo2, lo1]
  *reinterpret_cast<uint4*>(out + ((size_t)img * rows + k) * cols + 16 * q) = w;
}

// spec_out != nullptr: fused spectrum_u8 — the column pass writes u8 spectra there.
// side != nullptr (with spec_out): `data` is a pair array of `batch` pairs of
// real images (fft4096_ws<PAIR>); 2 batch spectra are written, side is scratch
// of 2 batch R complex values.
int fft2d_colring_execute(const FftPlan* p, float2* data, int64_t batch, cudaStream_t s, uint8_t* spec_out,
                          float alpha, float2* dst, const float2* twlo, const float2* twhi, bool xp, float2* side) {
  if (!dst) dst = data;
  const int64_t R = p->n0, C = p->n1;
  const int B = (int)(R / 256);
  const int64_t units = batch * (C / 16);
  if (units == 0) return DPP_OK;
  CUtensorMap tin, tout;
  {
    const uint64_t dims[3] = {(uint64_t)C, 256, (uint64_t)(B * batch)};
    const uint64_t strides[2] = {(uint64_t)C * 8, (uint64_t)C * 8 * 256};
    const uint32_t box[3] = {16, (uint32_t)(colring::TILE / (16 * B)), (uint32_t)B};
    if (int rc = make_tmap_c64_3d(&tin, data, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  }
  if (xp) {
    // transposed output T (C rows of R = 256 B per image), a row viewed [k2][k1]
    if (spec_out || twlo || B < 16)
      return fail(DPP_ENOTSUP, "transposed column pass needs 4096 .. 32768 rows, no fused epilogue");
    if (dst == data) return fail(DPP_EINVAL, "transposed column pass cannot run in place");
    const uint64_t dims[3] = {(uint64_t)B, 256, (uint64_t)C * batch};
    const uint64_t strides[2] = {(uint64_t)B * 8, (uint64_t)R * 8};
    const uint32_t box[3] = {16, 256, 1};
    if (int rc = make_tmap_c64_3d(&tout, dst, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  } else if (spec_out) {
    if (side && (C != 4096 || twlo)) return fail(DPP_EINVAL, "pair spectra need 4096-column pair arrays");
    const uint64_t dims[3] = {(uint64_t)C, (uint64_t)B, (uint64_t)(256 * batch * (side ? 2 : 1))};
    const uint64_t strides[2] = {(uint64_t)C, (uint64_t)C * B};
    const uint32_t box[3] = {16, 1, 256};
    if (int rc = make_tmap_u8_3d(&tout, spec_out, dims, strides, box)) return rc;
  } else {
    const uint64_t dims[3] = {(uint64_t)C, (uint64_t)B, (uint64_t)(256 * batch)};
    const uint64_t strides[2] = {(uint64_t)C * 8, (uint64_t)C * 8 * B};
    const uint32_t box[3] = {16, 1, 256};
    if (int rc = make_tmap_c64_3d(&tout, dst, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  }
  colring::Args a;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw;
  a.twr = reinterpret_cast<const float2*>(p->l2_tw + 256);
  a.units = (int)units;
  a.tiles_per_image = (int)(C / 16);
  a.lag = (int)(units < p->l2_lag ? units : p->l2_lag);
  a.ring = p->l2_ring;
  a.alpha = alpha;
  a.np = 1;
  a.col0 = a.tb = 0;
  a.twlo = twlo;
  a.twhi = twhi;
  a.side = spec_out ? side : nullptr;
  DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
  DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)units) * sizeof(int), s));
  const int64_t items = 2 * (int64_t)B * units;
  const unsigned grid = (unsigned)(items < p->col_ring_ctas ? items : p->col_ring_ctas);
  const size_t smem = colring_smem(spec_out != nullptr);
  if (spec_out && B != 16 && B != 64) return fail(DPP_ENOTSUP, "fused spectrum needs 4096 or 16384 rows");

  if (xp) {
    switch (B) {
      case 16: colring::fft_cols_l2w<16, true, false, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      case 32: colring::fft_cols_l2w<32, true, false, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      case 64: colring::fft_cols_l2w<64, true, false, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      default: colring::fft_cols_l2w<128, true, false, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a);
    }
  } else if (twlo) {
    switch (B) {
      case 4: colring::fft_cols_l2w<4, true, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      case 8: colring::fft_cols_l2w<8, true, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      case 16: colring::fft_cols_l2w<16, true, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      case 32: colring::fft_cols_l2w<32, true, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      case 64: colring::fft_cols_l2w<64, true, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
      default: colring::fft_cols_l2w<128, true, false, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a);
    }
  } else if (spec_out) {
    if (B == 16)
      colring::fft_cols_l2w<16, true, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a);
    else
      colring::fft_cols_l2w<64, true, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a);
  } else {
#define COLRING_PLAIN(BB)                                                                  \
  case BB:                                                                                 \
    if (g_col_discard)                                                                     \
      colring::fft_cols_l2w<BB, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a);  \
    else                                                                                   \
      colring::fft_cols_l2w<BB, false><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); \
    break;
    switch (B) {
      COLRING_PLAIN(4)
      COLRING_PLAIN(8)
      COLRING_PLAIN(16)
      COLRING_PLAIN(32)
      COLRING_PLAIN(64)
      COLRING_PLAIN(128)
    }
#undef COLRING_PLAIN
  }
  DPP_LAUNCH_CHECK("fft_cols_l2w");
  DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
  if (spec_out && side) {
    const int64_t nm = 2 * batch * R * (C / 32), n = 2 * batch * R;
    spectrum_pair_mirror<<<(unsigned)((nm + 255) / 256), 256, 0, s>>>(spec_out, (int)R, (int)C, nm);
    DPP_LAUNCH_CHECK("spectrum_pair_mirror");
    spectrum_pair_fixup<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(side, spec_out, (int)R, (int)C, n, alpha);
    DPP_LAUNCH_CHECK("spectrum_pair_fixup");
  }
  return DPP_OK;
}

// Row-sharded 2-D column pass with the exchange fused in (PEER kernel above).
// slabs[j]: rank j's batch x (R/np) x C row slab (already row-transformed;
// device pointers valid in this process — peer-mapped for j != rank).
// tb: outs[j] = rank j's row slab of the result (may equal slabs[j]);
// otherwise outs[0] = this rank's batch x R x (C/np) column slab.
int fft2d_colring_execute_peer(const FftPlan* p, const float2* const* slabs, float2* const* outs, int np, int rank,
                               int tb, int64_t batch, cudaStream_t s) {
  const int64_t R = p->n0, C = p->n1;
  const int B = (int)(R / 256);
  if (!p->col_ring) return fail(DPP_ENOTSUP, "row-sharded column pass needs the column ring (n0 = 1024 .. 32768, rows a multiple of 16 columns)");
  if (np < 1 || np > 8 || (np & (np - 1)) || B % np)
    return fail(DPP_EINVAL, "rank count %d must be a power of two <= 8 dividing %d", np, B);
  if (rank < 0 || rank >= np) return fail(DPP_EINVAL, "rank %d outside 0..%d", rank, np - 1);
  if (C % (16 * np)) return fail(DPP_EINVAL, "%lld columns do not split into 16-column tiles over %d ranks",
                                 (long long)C, np);
  if (batch < 0 || batch > p->batch) return fail(DPP_EINVAL, "batch %lld outside the planned 0..%lld",
                                                 (long long)batch, (long long)p->batch);
  for (int j = 0; j < np; ++j)
    if (!slabs[j] || (tb ? !outs[j] : !outs[0])) return fail(DPP_EINVAL, "NULL slab pointer");
  const int64_t w = C / np;
  const int64_t units = batch * (w / 16);
  if (units == 0) return DPP_OK;
  const int nb = B / np, kk = 256 / np;
  colring::Maps8 tin, tout;
  std::memset(&tin, 0, sizeof(tin));
  std::memset(&tout, 0, sizeof(tout));
  for (int j = 0; j < np; ++j) {
    const uint64_t dims[3] = {(uint64_t)C, 256, (uint64_t)nb * batch};
    const uint64_t strides[2] = {(uint64_t)C * 8, (uint64_t)C * 8 * 256};
    const uint32_t box[3] = {16, (uint32_t)(colring::TILE / (16 * B)), (uint32_t)nb};
    if (int rc = make_tmap_c64_3d(&tin.m[j], slabs[j], dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  }
  if (tb) {
    for (int j = 0; j < np; ++j) {
      const uint64_t dims[3] = {(uint64_t)C, (uint64_t)B, (uint64_t)kk * batch};
      const uint64_t strides[2] = {(uint64_t)C * 8, (uint64_t)C * 8 * B};
      const uint32_t box[3] = {16, 1, (uint32_t)kk};
      if (int rc = make_tmap_c64_3d(&tout.m[j], outs[j], dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
    }
  } else {
    const uint64_t dims[3] = {(uint64_t)w, (uint64_t)B, (uint64_t)(256 * batch)};
    const uint64_t strides[2] = {(uint64_t)w * 8, (uint64_t)w * 8 * B};
    const uint32_t box[3] = {16, 1, 256};
    if (int rc = make_tmap_c64_3d(&tout.m[0], outs[0], dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  }
  colring::Args a;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw;
  a.twr = reinterpret_cast<const float2*>(p->l2_tw + 256);
  a.units = (int)units;
  a.tiles_per_image = (int)(w / 16);
  a.lag = (int)(units < p->l2_lag ? units : p->l2_lag);
  a.ring = p->l2_ring;
  a.alpha = 0.f;
  a.twlo = a.twhi = nullptr;
  a.np = np;
  a.col0 = (int)(rank * w);
  a.tb = tb ? 1 : 0;
  DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
  DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)units) * sizeof(int), s));
  const int64_t items = 2 * (int64_t)B * units;
  const unsigned grid = (unsigned)(items < p->col_ring_ctas ? items : p->col_ring_ctas);
  const size_t smem = colring_smem(false);
  switch (B) {
    case 4: colring::fft_cols_l2w<4, true, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
    case 8: colring::fft_cols_l2w<8, true, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
    case 16: colring::fft_cols_l2w<16, true, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
    case 32: colring::fft_cols_l2w<32, true, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
    case 64: colring::fft_cols_l2w<64, true, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a); break;
    default: colring::fft_cols_l2w<128, true, false, true><<<grid, colring::THREADS, smem, s>>>(tin, tout, a);
  }
  DPP_LAUNCH_CHECK("fft_cols_l2w<peer>");
  DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
  return DPP_OK;
}

}  // namespace dpp
