// FFT node, n = 2^16: two-pass four-step with the intermediate kept in L2.
//
// Same mathematics as the cluster kernel (fft.cu, n = N2*a + b, k = c + N1*d,
// N1 = N2 = 256), but the exchange between the two 256-point passes goes
// through a small ring of scratch slots that lives in L2 instead of through
// distributed shared memory inside a 16-CTA cluster.  Measured in round 1
// (profiles/r1_fft_c2_structure.md): the 16-CTA DSMEM all-to-all alone caps the
// data movement at 78% of HBM, cluster packing leaves ~3 CTAs per SM, and
// every CTA spends half its life waiting on cluster peers.  Here every work
// item is an independent 256-thread CTA:
//
//   P1(t, g)  pass 1 of transform t on columns b in [16g, 16g+16):
//             16 coalesced 128 B row reads per warp instruction pair (LDG.64,
//             HBM, evict-first) -> radix-16 over a1 -> W256 twiddle -> one
//             conflict-free SMEM transpose -> radix-16 over a0 -> W_N^{bc}
//             (per-thread recurrence) -> scratch S[c>>4][b][c&15] (128 B rows).
//   P2(t, g)  pass 2 of transform t on c in [16g, 16g+16): reads the 32 KB
//             block S[g] (L2 hits) -> radix-16 -> W256 -> SMEM transpose ->
//             radix-16 -> X[c + 256 d] (128 B rows, streaming stores).
//
// Each point crosses HBM exactly twice (read x, write X: the 16 B compulsory
// traffic) and shared memory twice (16 B), against 80 B of SMEM/DSMEM traffic
// per point in the cluster kernel.
//
// Ordering.  CTAs take tickets from a global counter; tickets map to items
// in the order P1(0..L-1), then P1(L+m), P2(m) alternating, then the last
// P2s, so P2(t) is issued 2L+1 item groups after P1(t).  P2(t) waits (thread
// 0 spins on an acquire load) until the 16 P1 items of t have published
// (release add); P1(t) waits until P2(t-R) has released ring slot t mod R.
// Every wait is on a strictly smaller ticket, held by a CTA that is already
// resident, so the schedule cannot deadlock.  With L = 40 and R = 96 the
// waits are almost never taken.  Scratch reads bypass L1 (ld.global.cg); the
// read-out slot lines are discarded from L2 (discard.global.L2) so dirty
// scratch never costs an HBM write-back.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft_plan.cuh"
#include "tma.cuh"
#include "fft_block.cuh"
#include "l2ring.cuh"

namespace dpp {

namespace l2x {

constexpr int N = 65536;
constexpr int THREADS = 256;
constexpr int ITEMS = 16;  // items per pass per transform
using namespace ring;

struct Ctrl {
  int* ticket;  // [0]
  int* cnt1;    // [batch] P1 items published per transform
  int* cnt2;    // [batch] P2 items that released their ring slot
};

// W_256^e as (w, i*w) for cmul_pre
__device__ __forceinline__ float2 twp(float2 v, const float4* tab, int e) {
  const float4 w = __ldg(tab + e);
  return cmul_pre(v, make_float2(w.x, w.y), make_float2(w.z, w.w));
}

template <bool DISCARD>
__global__ void __launch_bounds__(THREADS, 4)
fft65536_l2x(const float2* __restrict__ in, float2* __restrict__ out, float2* __restrict__ scratch,
             int* __restrict__ ctrl, int batch, int lag, int ring, const float4* __restrict__ tw256,
             const float4* __restrict__ twn) {
  __shared__ float2 buf[16 * 16 * 16];
  __shared__ int s_ticket;
  const int tid = threadIdx.x;
  if (tid == 0) s_ticket = atomicAdd(ctrl, 1);
  __syncthreads();
  const int ticket = s_ticket;
  int* cnt1 = ctrl + 32;
  int* cnt2 = cnt1 + batch;
  int pass, t;
  decode(ticket >> 4, batch, lag, pass, t);
  const int g = ticket & 15;
  const int lo = tid & 15;   // lane within the half-warp
  const int hi = tid >> 4;   // half-warp index 0..15
  float2* slot = scratch + (size_t)(t % ring) * N;
  float2 v[16];

  if (pass == 1) {
    // stage A: thread (b_lo = lo, a0 = hi) loads a = 16 a1 + a0, column b = 16 g + lo
    const float2* src = in + (size_t)t * N + 16 * g + lo + 256 * hi;
#pragma unroll
    for (int a1 = 0; a1 < 16; ++a1) v[a1] = ld_stream(src + 4096 * a1);
    dft16(v);  // v[c0] = sum_a1 x W16^{a1 c0}
#pragma unroll
    for (int c0 = 1; c0 < 16; ++c0) v[c0] = twp(v[c0], tw256, hi * c0);
    // transpose: (b_lo, a0 | c0) -> (c0, b_lo | a0); slot (a0, c0, b_lo ^ c0)
#pragma unroll
    for (int c0 = 0; c0 < 16; ++c0) buf[(hi * 16 + c0) * 16 + (lo ^ c0)] = v[c0];
    __syncthreads();
    // stage B: thread (c0 = lo, b_lo = hi)
#pragma unroll
    for (int a0 = 0; a0 < 16; ++a0) v[a0] = buf[(a0 * 16 + lo) * 16 + (hi ^ lo)];
    dft16(v);  // v[c1] = Z[b][c0 + 16 c1]
    // four-step twiddle W_N^{b c}, c = c0 + 16 c1: base W^{b c0}, step W^{16 b}
    const int b = 16 * g + hi;
    const float4 wb = __ldg(twn + b * lo);
    const float4 ws = __ldg(twn + 16 * b);
    const float2 step = make_float2(ws.x, ws.y);
    float2 w = make_float2(wb.x, wb.y);
    v[0] = cmul_pre(v[0], w, make_float2(wb.z, wb.w));
#pragma unroll
    for (int c1 = 1; c1 < 16; ++c1) {
      w = cmul(w, step);
      v[c1] = cmul(v[c1], w);
    }
    if (t >= ring) {
      if (tid == 0) wait_count(cnt2 + (t - ring), ITEMS);
      __syncthreads();
    }
    // S[c1][b][c0]
    float2* dst = slot + b * 16 + lo;
#pragma unroll
    for (int c1 = 0; c1 < 16; ++c1) st_l2(dst + 4096 * c1, v[c1]);
    __syncthreads();
    if (tid == 0) red_release_add(cnt1 + t, 1);
  } else {
    if (tid == 0) wait_count(cnt1 + t, ITEMS);
    __syncthreads();
    // stage A: thread (c_lo = lo, b0 = hi) loads b = 16 b1 + b0 of S[g]
    const float2* src = slot + 4096 * g + 16 * hi + lo;
#pragma unroll
    for (int b1 = 0; b1 < 16; ++b1) v[b1] = ld_l2(src + 256 * b1);
    dft16(v);  // v[d0]
#pragma unroll
    for (int d0 = 1; d0 < 16; ++d0) v[d0] = twp(v[d0], tw256, hi * d0);
    // transpose: (c_lo, b0 | d0) -> (c_lo, d0 | b0); slot (b0, d0, c_lo)
#pragma unroll
    for (int d0 = 0; d0 < 16; ++d0) buf[(hi * 16 + d0) * 16 + lo] = v[d0];
    __syncthreads();
    if constexpr (DISCARD) discard_l2(slot + 4096 * g + 16 * tid);
#pragma unroll
    for (int b0 = 0; b0 < 16; ++b0) v[b0] = buf[(b0 * 16 + hi) * 16 + lo];
    if (t + ring < batch) {  // someone reuses this slot: publish "read out" after every discard
      __syncthreads();
      if (tid == 0) red_release_add(cnt2 + t, 1);
    }
    dft16(v);  // v[d1]: X[c + 256 (d0 + 16 d1)], c = 16 g + c_lo, d0 = hi
    float2* dst = out + (size_t)t * N + 16 * g + lo + 256 * hi;
#pragma unroll
    for (int d1 = 0; d1 < 16; ++d1) st_stream(dst + 4096 * d1, v[d1]);
  }
}


// ---------------------------------------------------------------------------
// v2 (default): persistent CTAs with a two-stage TMA prefetch ring.
//
// Profiling v1 (profiles/r1_fft_l2x.md) showed the non-persistent form
// latency-bound (IPC 1.2, long-scoreboard stalls on the 16 LDGs every item
// waits for).  Here each CTA loops over tickets and, while it computes item
// i out of stage i&1, the TMA engine is already filling stage (i+1)&1 with the
// next item: P1 tiles by one 2-D tensor load (256 rows x 128 B), P2 blocks by
// one 32 KB bulk copy from the L2 ring.  The stage buffer doubles as the
// transpose buffer once its contents are in registers.
//
// Deadlock freedom with prefetch: a P2 item's dependency (its 16 P1 items)
// is only POLLED when prefetching; if unmet, the issue is deferred to the
// start of that item's iteration, when the CTA holds no unfinished item.  The
// P1 slot-reuse wait happens while processing (deps on smaller tickets only).
constexpr int STAGE = 4096;  // float2 per stage (32 KB)
constexpr int P1_WARPS = THREADS / 32;

struct L2pArgs {
  float2* out;
  float2* scratch;
  int* ctrl;
  const float4* tw256;
  const float4* twn;
  int batch, lag, ring;
};


// thread 0 only: start loading item `tick` into stage s; returns false (and
// issues nothing) when !blocking and the item's producers are not finished
__device__ __forceinline__ bool issue_item(const CUtensorMap* tin, const L2pArgs& a, int tick, float2* buf,
                                           uint64_t* bar, bool blocking) {
  int pass, t;
  decode(tick >> 4, a.batch, a.lag, pass, t);
  const int g = tick & 15;
  if (pass == 1) {
    mbar_arrive_expect_tx(bar, STAGE * sizeof(float2));
    tma_load_2d(buf, tin, 16 * g, t * 256, bar);
    return true;
  }
  const int* cnt1 = a.ctrl + 32;
  if (blocking)
    wait_count(cnt1 + t, ITEMS * P1_WARPS);
  else if (ld_acquire(cnt1 + t) < ITEMS * P1_WARPS)
    return false;
  fence_proxy_async_global();
  mbar_arrive_expect_tx(bar, STAGE * sizeof(float2));
  bulk_g2s(buf, a.scratch + (size_t)(t % a.ring) * N + 4096 * g, STAGE * sizeof(float2), bar);
  return true;
}

template <bool DISCARD>
__global__ void __launch_bounds__(THREADS, 3)
fft65536_l2p(const __grid_constant__ CUtensorMap tin, const L2pArgs a) {
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ uint64_t bars[2];
  __shared__ int s_tick[2];
  __shared__ int s_def[2];
  float4* tw = reinterpret_cast<float4*>(smem + 2 * STAGE);
  const int tid = threadIdx.x;
  const int lo = tid & 15, hi = tid >> 4;
  const int total = 2 * ITEMS * a.batch;
  int* cnt1 = a.ctrl + 32;
  int* cnt2 = cnt1 + a.batch;
  tw[tid] = a.tw256[tid];
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    for (int s = 0; s < 2; ++s) {
      const int tick = atomicAdd(a.ctrl, 1);
      s_tick[s] = tick;
      s_def[s] = tick < total ? !issue_item(&tin, a, tick, smem + s * STAGE, &bars[s], s == 0) : 0;
    }
  }
  __syncthreads();
  float2 v[16];
  for (int i = 0;; ++i) {
    const int s = i & 1;
    const int tick = s_tick[s];
    if (tick >= total) break;
    float2* buf = smem + s * STAGE;
    if (tid == 0 && s_def[s]) issue_item(&tin, a, tick, buf, &bars[s], true);
    int pass, t;
    decode(tick >> 4, a.batch, a.lag, pass, t);
    const int g = tick & 15;
    float2* slot = a.scratch + (size_t)(t % a.ring) * N;
    mbar_wait(&bars[s], (i >> 1) & 1);
    if (DISCARD && pass == 2) discard_l2(slot + 4096 * g + 16 * tid);
    // stage A (both passes): thread (lo, hi) holds column lo, rows 16 j + hi
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = buf[(16 * j + hi) * 16 + lo];
    dft16(v);
#pragma unroll
    for (int k = 1; k < 16; ++k) v[k] = twmul(v[k], tw[hi * k]);
    __syncthreads();  // stage contents consumed
    if (pass == 2 && tid == 0 && t + a.ring < a.batch) red_release_add(cnt2 + t, 1);
    if (pass == 1) {
      // (b_lo, a0 | c0) -> (c0, b_lo | a0); slot (a0, c0, b_lo ^ c0)
#pragma unroll
      for (int k = 0; k < 16; ++k) buf[(hi * 16 + k) * 16 + (lo ^ k)] = v[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = buf[(k * 16 + lo) * 16 + (hi ^ lo)];
    } else {
      // (c_lo, b0 | d0) -> (c_lo, d0 | b0); slot (b0, d0, c_lo)
#pragma unroll
      for (int k = 0; k < 16; ++k) buf[(hi * 16 + k) * 16 + lo] = v[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = buf[(k * 16 + hi) * 16 + lo];
    }
    fence_proxy_async_smem();  // generic accesses of buf before the TMA refill
    __syncthreads();           // buf free
    if (tid == 0) {
      const int next = atomicAdd(a.ctrl, 1);
      s_tick[s] = next;
      s_def[s] = next < total ? !issue_item(&tin, a, next, buf, &bars[s], false) : 0;
    }
    dft16(v);
    if (pass == 1) {
      // W_N^{b c}, b = 16 g + hi, c = lo + 16 c1
      const int b = 16 * g + hi;
      const float4 wb = __ldg(a.twn + b * lo);
      const float4 ws = __ldg(a.twn + 16 * b);
      const float2 step = make_float2(ws.x, ws.y);
      float2 w = make_float2(wb.x, wb.y);
      v[0] = cmul_pre(v[0], w, make_float2(wb.z, wb.w));
#pragma unroll
      for (int c1 = 1; c1 < 16; ++c1) {
        w = cmul(w, step);
        v[c1] = cmul(v[c1], w);
      }
      if (t >= a.ring) wait_count(cnt2 + (t - a.ring), ITEMS);
      float2* dst = slot + b * 16 + lo;
#pragma unroll
      for (int c1 = 0; c1 < 16; ++c1) st_l2(dst + 4096 * c1, v[c1]);
      __syncwarp();
      if ((tid & 31) == 0) red_release_add(cnt1 + t, 1);
    } else {
      float2* dst = a.out + (size_t)t * N + 16 * g + lo + 256 * hi;
#pragma unroll
      for (int d1 = 0; d1 < 16; ++d1) st_stream(dst + 4096 * d1, v[d1]);
    }
  }
}

// ---------------------------------------------------------------------------
// v3 (default): warp-specialised, warp-local passes.
//
// v2 still stalled on CTA barriers around the SMEM transposes, on the
// release fences after the scratch stores and on L1 invalidations from the
// acquire polls (profiles/r1_fft_l2x.md).  v3 moves all of that off the
// compute warps:
//   * one PRODUCER warp (lane 0) takes tickets, polls dependencies, issues
//     the TMA loads into an S-stage ring (full[s] mbarriers), and after the
//     compute warps finish an item (done[s], 8 arrivals) publishes it: P1 ->
//     release-add cnt1[t]; P2 -> discard the scratch lines, release the ring
//     slot (cnt2[t]) and TMA-store the output tile.  While it waits for a
//     dependency it keeps publishing finished items, so it can never hold up
//     the items the dependency is waiting for.
//   * 8 COMPUTE warps; warp w owns columns 2w, 2w+1 of the 256 x 16 tile, so
//     both radix-16 exchanges of a 256-point pass are warp-local
//     (__syncwarp, in place in the warp's own slots) — no CTA barrier at all.
// Tile layout (both passes, input and output tiles): 128B-swizzled rows,
// complex (r, c) at r*16 + 2*((c>>1) ^ (r&7)) + (c&1) — what TMA SWIZZLE_128B
// produces/consumes, and P1 writes its scratch rows in the same order so the
// P2 block arrives by a plain bulk copy already swizzled.  Every warp access
// below touches 8 chunks x 2 parities twice: 2 wavefronts per 256 B, the
// minimum.
namespace l2w {
using namespace ring;

constexpr int CW = 8;
constexpr int THREADS = (CW + 1) * 32;
constexpr int TILE = 4096;

struct Args {
  float2* scratch;
  int* ctrl;
  const float4* tw256;   // [k][idx] = W256^{k*idx} as (w, i*w)
  const float2* tw4096;  // W4096^e, e < 256
  const float2* tw65536; // W65536^e, e < 256
  int batch, lag, ring;
};


#ifndef DPP_L2_PF
#define DPP_L2_PF 0  // L2 prefetch distance in item-times (measured: no gain, profiles/r1_fft_l2.md)
#endif
// LDG2: P2 reads its block straight from L2 into registers (ld.global.cg)
// instead of a bulk copy into the stage: 16 B/point less shared-memory
// traffic, the L2 latency exposed to the compute warps instead
template <int S, int MINB, bool DISCARD, int PF = DPP_L2_PF, bool LDG2 = false>
__global__ void __launch_bounds__(THREADS, MINB)
fft65536_l2w(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, const Args a) {
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  __shared__ int s_tick[S];
  float4* tw = reinterpret_cast<float4*>(smem + S * TILE);
  float2* t4096 = reinterpret_cast<float2*>(tw + 256);
  float2* t65536 = t4096 + 256;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int total = 2 * l2x::ITEMS * a.batch;
  int* cnt1 = a.ctrl + 32;
  int* cnt2 = cnt1 + a.batch;
  for (int e = tid; e < 256; e += THREADS) {
    tw[e] = a.tw256[e];
    t4096[e] = a.tw4096[e];
    t65536[e] = a.tw65536[e];
  }
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
      int pass, t;
      l2x::decode(s_tick[s] >> 4, a.batch, a.lag, pass, t);
      const int g = s_tick[s] & 15;
      if (pass == 1) {
        l2x::red_release_add(cnt1 + t, 1);
      } else {
        if (t + a.ring < a.batch) l2x::red_release_add(cnt2 + t, 1);  // lines discarded by the compute warps
        tma_store_2d_hint(&tout, 16 * g, t * 256, smem + s * TILE, stream_pol);
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
      int pass, t;
      l2x::decode(tick >> 4, a.batch, a.lag, pass, t);
      const int g = tick & 15;
      if (PF > 0) {
        // tickets are consumed at ~gridDim.x per item time: warm L2 with the P1
        // tile PF item-times ahead (whichever CTA takes that ticket then loads
        // it from L2 instead of HBM; P2 blocks are in L2 already)
        const int ft = tick + PF * (int)gridDim.x;
        if (ft < total) {
          int fp, fu;
          l2x::decode(ft >> 4, a.batch, a.lag, fp, fu);
          if (fp == 1) tma_prefetch_2d(&tin, 16 * (ft & 15), fu * 256);
        }
      }
      const int* dep = pass == 2 ? cnt1 + t : (t >= a.ring ? cnt2 + (t - a.ring) : nullptr);
      if (dep) {
        while (l2x::ld_acquire(dep) < l2x::ITEMS) {
          if (head < i && mbar_try(&done[head % S], (head / S) & 1)) {
            publish(head);
            ++head;
          } else {
            __nanosleep(32);
          }
        }
      }
      bulk_wait_read0();  // the stage's previous output tile has left shared memory
      s_tick[s] = tick;
      float2* buf = smem + s * TILE;
      if (LDG2 && pass == 2) {
        mbar_arrive1(&full[s]);  // the compute warps load the block themselves
        continue;
      }
      mbar_arrive_expect_tx(&full[s], TILE * sizeof(float2));
      if (pass == 1) {
        tma_load_2d_hint(buf, &tin, 16 * g, t * 256, &full[s], stream_pol);
      } else {
        l2x::fence_proxy_async_global();
        bulk_g2s(buf, a.scratch + (size_t)(t & (a.ring - 1)) * l2x::N + 4096 * g, TILE * sizeof(float2), &full[s]);
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
  // a half-warp = 8 rows x 2 columns: 16 distinct 8-byte bank pairs.  All
  // tile addresses are a per-thread base (+ an XOR pattern) + immediates:
  //   tile rows r = 16 j + idx:        base + offA + 2048 j
  //   exchange write (idx | k):        ((base + offW) ^ 144 (k&7)) + 1024 (k>>3)
  //   exchange read  (k | idx):        ((base + offR) ^ 144 (k&7)) + 2048 k
  // (derived from swz(); the XOR only touches address bits 4..9 and every
  // stage is 1024-byte aligned).
  const int col = 2 * warp + (lane & 1);
  const int idx = lane >> 1;
  const int q = idx & 7, p = lane & 1;
  const uint32_t x9 = 16u * (uint32_t)((9 * q) ^ warp);
  const uint32_t offA = 128u * idx + 16u * (uint32_t)(warp ^ q) + 8u * p;
  const uint32_t offW = 2048u * idx + 8u * p + x9;
  const uint32_t offR = 1024u * (idx >> 3) + 8u * p + x9;
  const uint32_t sbase = smem_u32(smem);
  const uint64_t keep_pol = policy_evict_last();
  const float2 w1 = make_float2(tw[16 + idx].x, tw[16 + idx].y);  // W256^idx
  float2 v[16];
  for (int i = 0;; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const int tick = s_tick[s];
    if (tick < 0) break;
    int pass, t;
    l2x::decode(tick >> 4, a.batch, a.lag, pass, t);
    const int g = tick & 15;
    const uint32_t b = sbase + (uint32_t)s * (TILE * 8);
    float2* slot = a.scratch + (size_t)(t & (a.ring - 1)) * l2x::N;
    const uint32_t bA = b + offA;
    if (LDG2 && pass == 2) {
      const float2* pa = slot + 4096 * g + (offA >> 3);  // the block has the tile's layout
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = ld_l2(pa + 256 * j);
    } else {
      // the P2 block is in shared memory: drop its scratch lines (no HBM write-back)
      if (DISCARD && pass == 2) l2x::discard_l2(slot + 4096 * g + 16 * (tid & 255));
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = lds64(bA + 2048 * j);
    }
    dft16c(v);
    if (LDG2 && DISCARD && pass == 2) {
      asm volatile("bar.sync 1, 256;" ::: "memory");  // every warp's loads have returned
      l2x::discard_l2(slot + 4096 * g + 16 * (tid & 255));
    }
    float2 wk = w1;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      // W256^{idx k} by recurrence from the per-thread constant W256^idx: FMA-pipe
      // work instead of 15 LDS.128 per item (shared memory is the busier pipe)
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
    if (pass == 1) {
      // W_N^{b c}, b = 16 g + col, c = idx + 16 c1
      const int bb = 16 * g + col;
      float2 w = cmul(t4096[g * idx], t65536[col * idx]);
      const float2 step = t4096[bb];
      v[0] = cmul(v[0], w);
#pragma unroll
      for (int c1 = 1; c1 < 16; ++c1) {
        w = cmul(w, step);
        v[c1] = cmul(v[c1], w);
      }
      float2* dst = slot + swz(bb, idx);
#pragma unroll
      for (int c1 = 0; c1 < 16; ++c1) st_l2_hint(dst + 4096 * c1, v[c1], keep_pol);
    } else {
      __syncwarp();
      // output tile row d = idx + 16 d1, column col
#pragma unroll
      for (int d1 = 0; d1 < 16; ++d1) sts64(bA + 2048 * d1, v[d1]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive1(&done[s]);
  }
}

}  // namespace l2w

std::vector<float4> rot_table(int64_t n, int64_t count) {
  std::vector<float4> t((size_t)count);
  for (int64_t e = 0; e < count; ++e) {
    const double a = -2.0 * M_PI * (double)e / (double)n;
    const float c = (float)std::cos(a), s = (float)std::sin(a);
    t[(size_t)e] = make_float4(c, s, -s, c);
  }
  return t;
}

}  // namespace l2x

static int g_discard = -1;
static int g_l2_version = 0;
static int g_l2p_ctas = 0;

static int l2p_prepare() {
  using namespace l2x;
  const size_t smem = 2 * STAGE * sizeof(float2) + 256 * sizeof(float4);
  for (auto kern : {fft65536_l2p<true>, fft65536_l2p<false>})
    DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0, dev = 0, sms = 0;
  DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft65536_l2p<true>, THREADS, smem));
  DPP_CUDA_CHECK(cudaGetDevice(&dev));
  DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(DPP_ECUDA, "fft65536_l2p does not fit on an SM");
  g_l2p_ctas = per_sm * sms;
  return DPP_OK;
}

static int l2p_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  using namespace l2x;
  CUtensorMap tmap;
  if (int rc = make_tmap_c64(&tmap, in, (uint64_t)batch * 256, 256, 256, 16)) return rc;
  L2pArgs a;
  a.out = out;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw;
  a.twn = p->l2_tw + 256;
  a.batch = (int)batch;
  a.lag = (int)(batch < p->l2_lag ? batch : p->l2_lag);
  a.ring = p->l2_ring;
  const int64_t items = 2 * ITEMS * batch;
  const unsigned grid = (unsigned)(items < g_l2p_ctas ? items : g_l2p_ctas);
  const size_t smem = 2 * STAGE * sizeof(float2) + 256 * sizeof(float4);
  if (g_discard)
    fft65536_l2p<true><<<grid, THREADS, smem, s>>>(tmap, a);
  else
    fft65536_l2p<false><<<grid, THREADS, smem, s>>>(tmap, a);
  DPP_LAUNCH_CHECK("fft65536_l2p");
  return DPP_OK;
}


#ifndef DPP_L2W_S
#define DPP_L2W_S 2  // default schedule: stages per CTA
#endif
#ifndef DPP_L2W_MINB
#define DPP_L2W_MINB 3  // and CTAs per SM
#endif
static int g_l2w_cfg = 0;  // 0: S=2 x 3 CTAs/SM, 1: S=3 x 2 CTAs/SM
static int g_l2w_ldg2 = 0;  // DPP_L2_P2LDG=1: P2 blocks loaded by the compute warps (A/B variant)
static int g_l2w_ctas = 0;

template <int S, int MINB, bool D>
static int l2w_prepare_one(size_t smem) {
  auto kern = l2x::l2w::fft65536_l2w<S, MINB, D>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return DPP_OK;
}

static size_t l2w_smem(int S) { return (size_t)S * l2x::l2w::TILE * sizeof(float2) + 8192; }

static int l2w_prepare() {
  if (const char* e = getenv("DPP_FFT_L2_CFG")) g_l2w_cfg = atoi(e) == 1 ? 1 : 0;
  if (const char* e = getenv("DPP_L2_P2LDG")) g_l2w_ldg2 = atoi(e) != 0;
  const int S = g_l2w_cfg ? 3 : DPP_L2W_S;
  const size_t smem = l2w_smem(S);
  {
    auto k2 = l2x::l2w::fft65536_l2w<DPP_L2W_S, DPP_L2W_MINB, true, DPP_L2_PF, true>;
    DPP_CUDA_CHECK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l2w_smem(DPP_L2W_S)));
  }
  int rc = g_l2w_cfg ? (l2w_prepare_one<3, 2, true>(smem) || l2w_prepare_one<3, 2, false>(smem))
                     : (l2w_prepare_one<DPP_L2W_S, DPP_L2W_MINB, true>(smem) || l2w_prepare_one<DPP_L2W_S, DPP_L2W_MINB, false>(smem));
  if (rc) return DPP_ECUDA;
  int per_sm = 0, dev = 0, sms = 0;
  if (g_l2w_cfg)
    DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, l2x::l2w::fft65536_l2w<3, 2, true>,
                                                                 l2x::l2w::THREADS, smem));
  else
    DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, l2x::l2w::fft65536_l2w<DPP_L2W_S, DPP_L2W_MINB, true>,
                                                                 l2x::l2w::THREADS, smem));
  DPP_CUDA_CHECK(cudaGetDevice(&dev));
  DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(DPP_ECUDA, "fft65536_l2w does not fit on an SM");
  g_l2w_ctas = per_sm * sms;
  return DPP_OK;
}

static int l2w_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  CUtensorMap tin, tout;
  if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  if (int rc = make_tmap_c64(&tout, out, (uint64_t)batch * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  l2x::l2w::Args a;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw + 256 + 4096;
  a.tw4096 = reinterpret_cast<const float2*>(p->l2_tw + 256 + 4096 + 256);
  a.tw65536 = reinterpret_cast<const float2*>(p->l2_tw + 256 + 4096 + 256 + 128);
  a.batch = (int)batch;
  a.lag = (int)(batch < p->l2_lag ? batch : p->l2_lag);
  a.ring = p->l2_ring;
  const int64_t items = 2 * l2x::ITEMS * batch;
  const unsigned grid = (unsigned)(items < g_l2w_ctas ? items : g_l2w_ctas);
  const int S = g_l2w_cfg ? 3 : DPP_L2W_S;
  const size_t smem = l2w_smem(S);
  if (g_l2w_cfg) {
    if (g_discard) l2x::l2w::fft65536_l2w<3, 2, true><<<grid, l2x::l2w::THREADS, smem, s>>>(tin, tout, a);
    else l2x::l2w::fft65536_l2w<3, 2, false><<<grid, l2x::l2w::THREADS, smem, s>>>(tin, tout, a);
  } else if (g_l2w_ldg2) {
    l2x::l2w::fft65536_l2w<DPP_L2W_S, DPP_L2W_MINB, true, DPP_L2_PF, true><<<grid, l2x::l2w::THREADS, smem, s>>>(
        tin, tout, a);
  } else {
    if (g_discard) l2x::l2w::fft65536_l2w<DPP_L2W_S, DPP_L2W_MINB, true><<<grid, l2x::l2w::THREADS, smem, s>>>(tin, tout, a);
    else l2x::l2w::fft65536_l2w<DPP_L2W_S, DPP_L2W_MINB, false><<<grid, l2x::l2w::THREADS, smem, s>>>(tin, tout, a);
  }
  DPP_LAUNCH_CHECK("fft65536_l2w");
  return DPP_OK;
}

int fft65536_l2x_init(FftPlan* p) {
  using namespace l2x;
  if (g_discard < 0) {
    const char* e = getenv("DPP_FFT_L2_DISCARD");
    g_discard = e ? atoi(e) != 0 : 1;
  }
  if (g_l2_version == 0) {
    const char* e = getenv("DPP_FFT_L2");
    g_l2_version = e ? atoi(e) : 3;
    if (g_l2_version < 1 || g_l2_version > 3) g_l2_version = 3;
    if (g_l2_version == 2)
      if (int rc = l2p_prepare()) return rc;
    if (g_l2_version == 3)
      if (int rc = l2w_prepare()) return rc;
  }
  p->l2_lag = 48;
  p->l2_ring = 128;
  if (const char* e = getenv("DPP_FFT_L2_LAG")) p->l2_lag = atoi(e);
  if (const char* e = getenv("DPP_FFT_L2_RING")) p->l2_ring = atoi(e);
  if (p->l2_ring <= p->l2_lag) p->l2_ring = p->l2_lag + 1;
  {  // a power of two (slot = t & (ring - 1))
    int r = 1;
    while (r < p->l2_ring) r <<= 1;
    p->l2_ring = r;
  }
  const auto t256 = rot_table(256, 256);
  const auto tn = rot_table(N, 4096);
  std::vector<float4> all(t256);
  all.insert(all.end(), tn.begin(), tn.end());
  // v3 tables: W256^{k*idx} k-major, then W4096^e and W65536^e (e < 256) as float2 pairs
  for (int k = 0; k < 16; ++k)
    for (int i = 0; i < 16; ++i) all.push_back(t256[(k * i) & 255]);
  const auto t4096 = rot_table(4096, 256);
  const auto t65536 = rot_table(N, 256);
  for (const auto* tab : {&t4096, &t65536})
    for (int e = 0; e < 256; e += 2)
      all.push_back(make_float4((*tab)[e].x, (*tab)[e].y, (*tab)[e + 1].x, (*tab)[e + 1].y));
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_tw, all.size() * sizeof(float4)));
  DPP_CUDA_CHECK(cudaMemcpy(p->l2_tw, all.data(), all.size() * sizeof(float4), cudaMemcpyHostToDevice));
  const size_t ring = (size_t)p->l2_ring * N * sizeof(float2);
  const size_t ctrl = (32 + 2 * (size_t)(p->batch > 0 ? p->batch : 1)) * sizeof(int);
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_scratch, ring));
  DPP_CUDA_CHECK(cudaMalloc(&p->l2_ctrl, ctrl));
  DPP_CUDA_CHECK(cudaEventCreateWithFlags(&p->l2_done, cudaEventDisableTiming));
  p->l2_ctrl_bytes = ctrl;
  return DPP_OK;
}

int fft65536_l2x_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s) {
  using namespace l2x;
  if (batch <= 0) return DPP_OK;
  if (g_l2_version >= 2) {
    if (batch > 0x7fffffff / (2 * ITEMS)) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
    DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
    DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)batch) * sizeof(int), s));
    if (int rc = g_l2_version == 3 ? l2w_execute(p, in, out, batch, s) : l2p_execute(p, in, out, batch, s))
      return rc;
    DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
    return DPP_OK;
  }
  if (batch > 0x7fffffff / (2 * ITEMS)) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  // the ring and counters belong to the plan: order this launch after the
  // previous one even when callers use different streams
  DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
  DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)batch) * sizeof(int), s));
  const int lag = (int)(batch < p->l2_lag ? batch : p->l2_lag);
  const float4* tw256 = p->l2_tw;
  const float4* twn = p->l2_tw + 256;
  const unsigned grid = (unsigned)(2 * ITEMS * batch);
  if (g_discard)
    fft65536_l2x<true><<<grid, THREADS, 0, s>>>(in, out, p->l2_scratch, p->l2_ctrl, (int)batch, lag, p->l2_ring,
                                                 tw256, twn);
  else
    fft65536_l2x<false><<<grid, THREADS, 0, s>>>(in, out, p->l2_scratch, p->l2_ctrl, (int)batch, lag,
                                                  p->l2_ring, tw256, twn);
  DPP_LAUNCH_CHECK("fft65536_l2x");
  DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
  return DPP_OK;
}

}  // namespace dpp
