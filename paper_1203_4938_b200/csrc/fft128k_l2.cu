// 1-D FFT node, n = 2^17 = 256 x 512: two-pass four-step through the L2
// exchange ring (the 2^16 kernel's schedule, csrc/fft_l2.cu), one transform
// per unit, 32 items per pass.  n = 512 a + b (a < 256, b < 512),
// k = k1 + 256 k2.
//
//   P1(u, g), g < 32: columns b in [16 g, 16 g + 16) of the [a][b] view (one
//       2-D TMA box, 128B-swizzled): the 2^16 kernel's warp-local 256-point
//       FFTs over a, twiddle W_n^{b k1}, stored to ring slot u as 32 blocks
//       S[k1 / 8] of 512 rows b x 8 columns k1 % 8, element (b, c) at
//       8 b + (c ^ ((b >> 1) & 7)) — the XOR makes the P2 reads conflict-free.
//   P2(u, g2), g2 < 32: block S[g2] by one bulk copy; warp w owns k1 = 8 g2 + w
//       (one 512-point sequence per warp, lane b0 holding b = 32 b1 + b0):
//       16-point FFT over b1, twiddle W_512^{b0 m0}, an in-warp exchange so
//       that lane (m0, l0) holds c = 2 l1 + l0, 16-point FFT over l1,
//       twiddle W_32^{l0 m1} and the last radix-2 with the partner lane
//       (shuffle): k2 = m0 + 16 m1 + 256 m2.  Output rows k2 (8 columns k1)
//       staged 64B-swizzled and written by two 2-D TMA stores (8 x 256).
// Two named barriers per P2 item: the stage is reused for the exchange and
// the output only after every warp has its inputs / finished its exchange.
//
// n = 2^18 = 512 x 512 (LOGN = 18, 64 items per pass): P1 is the same
// warp-wide 512-point FFT down 8 columns of the [a][b] view (two 2-D TMA
// boxes of 8 x 256, 64B-swizzled), twiddle W_n^{b k1}, stored straight from
// registers into the P2 block layout above; P2 is the 2^17 P2 with 512 output
// columns.
//
// n = 2^19 = 512 x 1024 (LOGN = 19, 128 items per pass): P1 as for 2^18 on
// rows of 1024; P2 blocks are 4 columns k1 x 1024 rows b (element (b, c) at
// 4 b + (c ^ ((b >> 2) & 3))), and each 1024-point sequence is split over a
// warp pair by one decimation-in-frequency step: warp e of the pair FFTs
// (x[j] + x[j+512]) (e = 0) or (x[j] - x[j+512]) W_1024^j (e = 1) with the
// 512-point warp FFT, giving X[2 k' + e] — no exchange between the two warps.
// Output tile 1024 rows x 4 columns, 32B-swizzled, four 2-D TMA stores (4 x 256).
//
// n = 2^20 = 1024 x 1024 (LOGN = 20, 256 items per pass): P1 loads 4 columns
// x 1024 rows (four 32B-swizzled boxes) and runs the same warp-pair
// decimation-in-frequency 1024-point FFT down each column, twiddle
// W_n^{b k1}, stores into the 4-column P2 blocks; P2 is the 2^19 P2.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "l2ring.cuh"
#include "tma.cuh"

namespace dpp {
namespace ring128k {

using namespace ring;

constexpr int CW = 8;
constexpr int THREADS = (CW + 1) * 32;
constexpr int TILE = 4096;
constexpr int S = 2;

struct Args {
  float2* scratch;
  int* ctrl;
  const float2* twn;    // W_n^m, m < n
  const float4* tw256;  // W256^m as (w, i*w)
  int units, lag, ring;
};

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// One 512-point FFT per warp: on entry lane b0 holds v[b1] = x[32 b1 + b0];
// on exit lane (m0 = lane >> 1, m2 = lane & 1) holds v[m1] = X[m0 + 16 m1 +
// 256 m2].  rx: this warp's 4 KB exchange region; pwb -> W_512^lane, pw32 -> W_32.
__device__ __forceinline__ void fft512_warp(float2 (&v)[16], uint32_t rx, int lane, const float2* pwb,
                                            const float2* pw32) {
  dft16c(v);  // v[m0]
  {
    const float2 wb = __ldg(pwb);
    float2 w = wb;
#pragma unroll
    for (int m0 = 1; m0 < 16; ++m0) {
      v[m0] = cmul(v[m0], w);
      w = cmul(w, wb);
    }
  }
#pragma unroll
  for (int m0 = 0; m0 < 16; ++m0) sts64(rx + 8u * (32 * m0 + (lane ^ (2 * (m0 & 7)))), v[m0]);
  __syncwarp();
  const int m0r = lane >> 1, l0 = lane & 1;
#pragma unroll
  for (int l1 = 0; l1 < 16; ++l1) v[l1] = lds64(rx + 8u * (32 * m0r + ((2 * l1 + l0) ^ (2 * (m0r & 7)))));
  dft16c(v);  // v[m1] = F_l0[m1]
  if (l0) {
    const float2 w32 = __ldg(pw32);
    float2 w = w32;
#pragma unroll
    for (int m1 = 1; m1 < 16; ++m1) {
      v[m1] = cmul(v[m1], w);
      w = cmul(w, w32);
    }
  }
#pragma unroll
  for (int m1 = 0; m1 < 16; ++m1) {
    const float px = __shfl_xor_sync(0xffffffffu, v[m1].x, 1);
    const float py = __shfl_xor_sync(0xffffffffu, v[m1].y, 1);
    v[m1] = l0 ? make_float2(px - v[m1].x, py - v[m1].y) : make_float2(v[m1].x + px, v[m1].y + py);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(THREADS, 3)
fft_ring512_l2w(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, const Args a) {
  constexpr int N = 1 << LOGN;
  constexpr int LOGI = LOGN == 17 ? 5 : (LOGN == 18 ? 6 : (LOGN == 19 ? 7 : 8)), ITEMS = 1 << LOGI;  // per pass
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  __shared__ int s_tick[S];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int total = 2 * ITEMS * a.units;
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

  if (warp == CW) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    const uint64_t stream_pol = policy_evict_first();
    int head = 0, i = 0;
    auto publish = [&](int k) {
      const int s = k % S;
      int pass, u;
      decode(s_tick[s] >> LOGI, a.units, a.lag, pass, u);
      if (pass == 1) {
        red_release_add(cnt1 + u, 1);
      } else {
        if (u + a.ring < a.units) red_release_add(cnt2 + u, 1);
        const int g2 = s_tick[s] & (ITEMS - 1);
        if constexpr (LOGN >= 19) {
          // four 256-row tiles: output rows k2 = 2 k'' + e, tile (e, k'' >> 8)
#pragma unroll
          for (int t4 = 0; t4 < 4; ++t4)
            tma_store_3d(&tout, 4 * g2, t4 >> 1, 512 * u + 256 * (t4 & 1), smem + s * TILE + t4 * (TILE / 4));
        } else {
          tma_store_2d_hint(&tout, 8 * g2, 512 * u, smem + s * TILE, stream_pol);
          tma_store_2d_hint(&tout, 8 * g2, 512 * u + 256, smem + s * TILE + TILE / 2, stream_pol);
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
      decode(tick >> LOGI, a.units, a.lag, pass, u);
      const int g = tick & (ITEMS - 1);
      const int* dep = pass == 2 ? cnt1 + u : (u >= a.ring ? cnt2 + (u - a.ring) : nullptr);
      if (dep) {
        while (ld_acquire(dep) < ITEMS) {
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
        if constexpr (LOGN == 17) {
          tma_load_2d_hint(buf, &tin, 16 * g, 256 * u, &full[s], stream_pol);
        } else if constexpr (LOGN == 20) {
#pragma unroll
          for (int h = 0; h < 4; ++h)
            tma_load_2d_hint(buf + h * (TILE / 4), &tin, 4 * g, 1024 * u + 256 * h, &full[s], stream_pol);
        } else {
          tma_load_2d_hint(buf, &tin, 8 * g, 512 * u, &full[s], stream_pol);
          tma_load_2d_hint(buf + TILE / 2, &tin, 8 * g, 512 * u + 256, &full[s], stream_pol);
        }
      } else {
        fence_proxy_async_global();
        bulk_g2s(buf, a.scratch + (size_t)(u & (a.ring - 1)) * N + 4096 * g, TILE * sizeof(float2), &full[s]);
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
  const uint32_t sbase = smem_u32(smem);
  const uint64_t keep_pol = policy_evict_last();
  float2 v[16];
  for (int i = 0;; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const int tick = s_tick[s];
    if (tick < 0) break;
    int pass, u;
    decode(tick >> LOGI, a.units, a.lag, pass, u);
    const int g = tick & (ITEMS - 1);
    const uint32_t b = sbase + (uint32_t)s * (TILE * 8);
    float2* slot = a.scratch + (size_t)(u & (a.ring - 1)) * N;
    if (pass == 1 && LOGN == 17) {
      // P1 (the 2^16 kernel's mapping): column col = 2w + (lane & 1), row part idx = lane >> 1
      const int col = 2 * warp + (lane & 1);
      const int idx = lane >> 1;
      const int q = idx & 7, p = lane & 1;
      const uint32_t x9 = 16u * (uint32_t)((9 * q) ^ warp);
      const uint32_t offA = 128u * idx + 16u * (uint32_t)(warp ^ q) + 8u * p;
      const uint32_t offW = 2048u * idx + 8u * p + x9;
      const uint32_t offR = 1024u * (idx >> 3) + 8u * p + x9;
      const float4 t1 = __ldg(a.tw256 + idx);
      const float2 w1 = make_float2(t1.x, t1.y);  // W256^idx
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
      dft16c(v);  // v[c1] = Y[b][k1 = idx + 16 c1], b = 16 g + col
      const int bb = 16 * g + col;
      float2 w = __ldg(a.twn + bb * idx);
      const float2 step = __ldg(a.twn + 16 * bb);
      v[0] = cmul(v[0], w);
#pragma unroll
      for (int c1 = 1; c1 < 16; ++c1) {
        w = cmul(w, step);
        v[c1] = cmul(v[c1], w);
      }
      // k1 = idx + 16 c1 -> block (idx >> 3) + 2 c1, column idx & 7
      float2* dst = slot + 4096 * (idx >> 3) + 8 * bb + ((idx & 7) ^ ((bb >> 1) & 7));
#pragma unroll
      for (int c1 = 0; c1 < 16; ++c1) st_l2_hint(dst + 8192 * c1, v[c1], keep_pol);
    } else if (pass == 1 && LOGN == 20) {
      // P1, n = 2^20: warp pair p owns column b = 4 g + p of the 1024 x 4 tile
      // (four 256-row quarters, 32B-swizzled); warp e of the pair takes the
      // DIF half: a = 32 a1 + lane paired with a + 512
      const int p = warp >> 1, e = warp & 1;
      const int bb = 4 * g + p;
      float2 wj = __ldg(a.twn + (N / 1024) * lane);  // W_1024^{lane}, then x W_32 per a1
      const float2 w32s = __ldg(a.twn + N / 32);
#pragma unroll
      for (int a1 = 0; a1 < 16; ++a1) {
        const int r = 32 * (a1 & 7) + lane;  // row inside quarter a1 >> 3 (and + 2 for a + 512)
        const uint32_t ad = b + 8192u * (uint32_t)(a1 >> 3) + 32u * (uint32_t)r +
                            16u * (uint32_t)((p >> 1) ^ ((r >> 2) & 1)) + 8u * (uint32_t)(p & 1);
        const float2 lo = lds64(ad), hi = lds64(ad + 16384u);
        if (e) {
          v[a1] = cmul(make_float2(lo.x - hi.x, lo.y - hi.y), wj);
          wj = cmul(wj, w32s);
        } else {
          v[a1] = make_float2(lo.x + hi.x, lo.y + hi.y);
        }
      }
      bar_compute();  // every warp holds its half-column: the stage is free for the exchange
      fft512_warp(v, b + 8u * 512 * (uint32_t)warp, lane, a.twn + (N / 512) * lane, a.twn + N / 32);
      // lane (m0, m2) of warp e holds k1 = 2 (m0 + 16 m1 + 256 m2) + e; twiddle W_n^{b k1}
      const int m0r = lane >> 1, l0 = lane & 1;
      const int kb = 2 * m0r + e;  // < 32
      float2 w = __ldg(a.twn + bb * (kb + 512 * l0));
      const float2 step = __ldg(a.twn + 32 * bb);
      v[0] = cmul(v[0], w);
#pragma unroll
      for (int m1 = 1; m1 < 16; ++m1) {
        w = cmul(w, step);
        v[m1] = cmul(v[m1], w);
      }
      // 4-column blocks: k1 >> 2 = (kb >> 2) + 8 m1 + 128 m2, k1 & 3 = kb & 3
      float2* dst = slot + 4096 * ((kb >> 2) + 128 * l0) + 4 * bb + ((kb & 3) ^ ((bb >> 2) & 3));
#pragma unroll
      for (int m1 = 0; m1 < 16; ++m1) st_l2_hint(dst + 32768 * m1, v[m1], keep_pol);
    } else if (pass == 1) {
      // P1, n = 2^18: warp w owns column b = 8 g + w of the 512 x 8 tile
      // (two 256-row halves, 64B-swizzled), lane b0 holds a = 32 a1 + b0
      const int bb = 8 * g + warp;
#pragma unroll
      for (int a1 = 0; a1 < 16; ++a1) {
        const int r = 32 * (a1 & 7) + lane;  // row inside half a1 >> 3
        v[a1] = lds64(b + 16384u * (uint32_t)(a1 >> 3) + 64u * (uint32_t)r +
                      16u * (uint32_t)((warp >> 1) ^ ((r >> 1) & 3)) + 8u * (uint32_t)(warp & 1));
      }
      bar_compute();  // every warp holds its column: the stage is free for the exchange
      fft512_warp(v, b + 8u * 512 * (uint32_t)warp, lane, a.twn + (N / 512) * lane, a.twn + N / 32);
      // lane (m0, m2) holds k1 = m0 + 16 m1 + 256 m2; twiddle W_n^{b k1}
      const int m0r = lane >> 1, l0 = lane & 1;
      const int k1b = m0r + 256 * l0;
      float2 w = __ldg(a.twn + bb * k1b);
      const float2 step = __ldg(a.twn + 16 * bb);
      v[0] = cmul(v[0], w);
#pragma unroll
      for (int m1 = 1; m1 < 16; ++m1) {
        w = cmul(w, step);
        v[m1] = cmul(v[m1], w);
      }
      if constexpr (LOGN == 18) {
        // k1 >> 3 = (m0 >> 3) + 2 m1 + 32 m2, k1 & 7 = m0 & 7
        float2* dst = slot + 4096 * ((m0r >> 3) + 32 * l0) + 8 * bb + ((m0r & 7) ^ ((bb >> 1) & 7));
#pragma unroll
        for (int m1 = 0; m1 < 16; ++m1) st_l2_hint(dst + 8192 * m1, v[m1], keep_pol);
      } else {
        // 4-column blocks: k1 >> 2 = (m0 >> 2) + 4 m1 + 64 m2, k1 & 3 = m0 & 3
        float2* dst = slot + 4096 * ((m0r >> 2) + 64 * l0) + 4 * bb + ((m0r & 3) ^ ((bb >> 2) & 3));
#pragma unroll
        for (int m1 = 0; m1 < 16; ++m1) st_l2_hint(dst + 16384 * m1, v[m1], keep_pol);
      }
    } else if (LOGN >= 19) {
      // P2, n = 2^19, 2^20: warp pair p = k1 % 4 of the block, warp e = w & 1 of the pair
      discard_l2(slot + 4096 * g + 16 * (tid & 255));
      const int p = warp >> 1, e = warp & 1;
      const uint32_t rd = b + 8u * (uint32_t)(4 * lane + (p ^ ((lane >> 2) & 3)));
      float2 wj = __ldg(a.twn + (N / 1024) * lane);  // W_1024^{lane}, then x W_32 per b1
      const float2 w32s = __ldg(a.twn + N / 32);
#pragma unroll
      for (int b1 = 0; b1 < 16; ++b1) {
        const float2 lo = lds64(rd + 8u * 128 * b1), hi = lds64(rd + 8u * 128 * b1 + 16384u);
        if (e) {
          v[b1] = cmul(make_float2(lo.x - hi.x, lo.y - hi.y), wj);
          wj = cmul(wj, w32s);
        } else {
          v[b1] = make_float2(lo.x + hi.x, lo.y + hi.y);
        }
      }
      bar_compute();  // every warp holds its half-sequence: the stage is free for the exchange
      fft512_warp(v, b + 8u * 512 * (uint32_t)warp, lane, a.twn + (N / 512) * lane, a.twn + N / 32);
      bar_compute();  // every exchange read is done: the stage takes the output tile
      // X[k1 + (n/1024) k2], k2 = 2 k' + e, k' = m0 + 16 m1 + 256 m2: this warp's
      // outputs are the parity-e rows — tile (e, m2), row r = m0 + 16 m1, column p,
      // 32B-swizzled (chunk ^= (r >> 2) & 1); a 3-D TMA store puts row r of tile
      // (e, h) at k2 = 2 (256 h + r) + e
      const int m0r = lane >> 1, l0 = lane & 1;
      const uint32_t ob = b + 8192u * (uint32_t)(2 * e + l0) + 8u * (uint32_t)(p & 1);
#pragma unroll
      for (int m1 = 0; m1 < 16; ++m1) {
        const int r = m0r + 16 * m1;
        sts64(ob + 32u * (uint32_t)r + 16u * (uint32_t)((p >> 1) ^ ((r >> 2) & 1)), v[m1]);
      }
    } else {
      // P2 (2^17, 2^18): warp = k1 % 8, lane b0 holds b = 32 b1 + b0
      discard_l2(slot + 4096 * g + 16 * (tid & 255));
      const uint32_t rd = b + 8u * (uint32_t)(8 * lane + (warp ^ ((lane >> 1) & 7)));
#pragma unroll
      for (int b1 = 0; b1 < 16; ++b1) v[b1] = lds64(rd + 8u * 256 * b1);
      bar_compute();  // every warp holds its sequence: the stage is free for the exchange
      fft512_warp(v, b + 8u * 512 * (uint32_t)warp, lane, a.twn + (N / 512) * lane, a.twn + N / 32);
      bar_compute();  // every exchange read is done: the stage takes the output tile
      // X[k1 + R k2] (R = n / 512 columns), k2 = m0 + 16 m1 + 256 m2: row
      // r = m0 + 16 m1 of half m2, column warp, 64B-swizzled (chunk ^= (r >> 1) & 3)
      const int m0r = lane >> 1, l0 = lane & 1;
      const uint32_t ob = b + 16384u * (uint32_t)l0 + 8u * (uint32_t)(warp & 1);
#pragma unroll
      for (int m1 = 0; m1 < 16; ++m1) {
        const int r = m0r + 16 * m1;
        sts64(ob + 64u * (uint32_t)r + 16u * (uint32_t)((warp >> 1) ^ ((r >> 1) & 3)), v[m1]);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive1(&done[s]);
  }
}

}  // namespace ring128k

static int g_r512_ctas[4] = {0, 0, 0, 0};

// n = 2^17 (256 x 512) and 2^18 (512 x 512)
int fft128k_l2_init(FftPlan* p) {
  using namespace ring128k;
  const int64_t N = p->n0;
  if (N < (1 << 17) || N > (1 << 20) || (N & (N - 1)))
    return fail(DPP_EINVAL, "the 512-point ring is for n = 2^17 .. 2^20");
  const int slot = N == (1 << 17) ? 0 : (N == (1 << 18) ? 1 : (N == (1 << 19) ? 2 : 3));
  const size_t smem = (size_t)S * TILE * sizeof(float2);
  if (!g_r512_ctas[slot]) {
    const void* fns[4] = {(const void*)fft_ring512_l2w<17>, (const void*)fft_ring512_l2w<18>,
                          (const void*)fft_ring512_l2w<19>, (const void*)fft_ring512_l2w<20>};
    const void* fn = fns[slot];
    DPP_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, dev = 0, sms = 0;
    DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, THREADS, smem));
    DPP_CUDA_CHECK(cudaGetDevice(&dev));
    DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1) return fail(DPP_ECUDA, "fft_ring512_l2w does not fit on an SM");
    g_r512_ctas[slot] = per_sm * sms;
  }
  // units are whole transforms (1 or 2 MB): the 2^16 kernel's 24 MB lag and 64 MB ring
  const int lags[4] = {24, 16, 8, 4}, rings[4] = {64, 32, 16, 8};
  p->l2_lag = ring_stress() ? 2 : lags[slot];
  p->l2_ring = ring_stress() ? 4 : rings[slot];
  if (p->l2_ring <= p->l2_lag) p->l2_ring = p->l2_lag + 1;
  int r = 1;
  while (r < p->l2_ring) r <<= 1;
  p->l2_ring = r;
  std::vector<float2> twn((size_t)N);
  for (int64_t m = 0; m < N; ++m) {
    const double ang = -2.0 * M_PI * (double)m / (double)N;
    twn[(size_t)m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  std::vector<float4> t256(256);
  for (int m = 0; m < 256; ++m) {
    const double ang = -2.0 * M_PI * (double)m / 256.0;
    const float c = (float)std::cos(ang), s = (float)std::sin(ang);
    t256[(size_t)m] = make_float4(c, s, -s, c);
  }
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_tw, 256 * sizeof(float4) + (size_t)N * sizeof(float2)));
  DPP_CUDA_CHECK(cudaMemcpy(p->l2_tw, t256.data(), 256 * sizeof(float4), cudaMemcpyHostToDevice));
  DPP_CUDA_CHECK(cudaMemcpy(reinterpret_cast<float2*>(p->l2_tw + 256), twn.data(), (size_t)N * sizeof(float2),
                            cudaMemcpyHostToDevice));
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_scratch, (size_t)p->l2_ring * N * sizeof(float2)));
  const int64_t units = p->batch > 0 ? p->batch : 1;
  p->l2_ctrl_bytes = (32 + 2 * (size_t)units) * sizeof(int);
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_ctrl, p->l2_ctrl_bytes));
  DPP_CUDA_CHECK(cudaEventCreateWithFlags(&p->l2_done, cudaEventDisableTiming));
  return DPP_OK;
}

int fft128k_l2_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  using namespace ring128k;
  if (batch <= 0) return DPP_OK;
  const int lg = p->n0 == (1 << 17) ? 17 : (p->n0 == (1 << 18) ? 18 : (p->n0 == (1 << 19) ? 19 : 20));
  const int items = 32 << (lg - 17);
  if (batch > 0x7fffffff / (2 * items)) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  CUtensorMap tin, tout;
  if (lg == 20) {
    // input as 1024 rows a x 1024 columns b, boxes of 4 columns x 256 rows (32B swizzle)
    if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 1024, 1024, 256, 4, CU_TENSOR_MAP_SWIZZLE_32B)) return rc;
  } else if (lg >= 18) {
    // input as 512 rows a x n/512 columns b, boxes of 8 columns x 256 rows (64B swizzle)
    if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 512, (uint64_t)(p->n0 / 512), 256, 8,
                               CU_TENSOR_MAP_SWIZZLE_64B))
      return rc;
  } else {
    if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 256, 512, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B))
      return rc;
  }
  if (lg >= 19) {
    // output rows k2 = 2 k'' + e (1024 per transform) x n/1024 columns k1 as a 3-D view
    // {k1, e, k''}; boxes of 4 columns x 1 parity x 256 rows
    const uint64_t cols = (uint64_t)(p->n0 / 1024);
    const uint64_t dims[3] = {cols, 2, (uint64_t)batch * 512};
    const uint64_t strides[2] = {cols * 8, cols * 16};
    const uint32_t box[3] = {4, 1, 256};
    if (int rc = make_tmap_c64_3d(&tout, out, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_32B)) return rc;
  } else {
    // output as rows k2 (512 per transform) x n/512 columns k1, boxes of 8 columns x 256 rows
    if (int rc = make_tmap_c64(&tout, out, (uint64_t)batch * 512, (uint64_t)(p->n0 / 512), 256, 8,
                               CU_TENSOR_MAP_SWIZZLE_64B))
      return rc;
  }
  Args a;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw;
  a.twn = reinterpret_cast<const float2*>(p->l2_tw + 256);
  a.units = (int)batch;
  a.lag = (int)(batch < p->l2_lag ? batch : p->l2_lag);
  a.ring = p->l2_ring;
  DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
  DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)batch) * sizeof(int), s));
  const int64_t total = 2 * (int64_t)items * batch;
  const int ctas = g_r512_ctas[lg - 17];
  const unsigned grid = (unsigned)(total < ctas ? total : ctas);
  const size_t smem = (size_t)S * TILE * sizeof(float2);
  if (lg == 20)
    fft_ring512_l2w<20><<<grid, THREADS, smem, s>>>(tin, tout, a);
  else if (lg == 19)
    fft_ring512_l2w<19><<<grid, THREADS, smem, s>>>(tin, tout, a);
  else if (lg == 18)
    fft_ring512_l2w<18><<<grid, THREADS, smem, s>>>(tin, tout, a);
  else
    fft_ring512_l2w<17><<<grid, THREADS, smem, s>>>(tin, tout, a);
  DPP_LAUNCH_CHECK("fft_ring512_l2w");
  DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
  return DPP_OK;
}

}  // namespace dpp
