// Session-5 C2 A/B variants of csrc/fft_l2.cu (NOT built into the library).
// Each V_* macro selects one measured change; results in profiles/r2_c2_diagnosis.md.
// Build one:  mkdir -p alt/v && cp profiles/micro/fft_l2_variants.cu alt/v/fft_l2.cu &&
//   python profiles/micro/build_variant.py NAME alt/v/fft_l2.cu -DV_SW=1   (then profiles/micro/sess_ab_c2.sh alt/NAME.so)
// Session-5 C2 A/B variants of csrc/fft_l2.cu (NOT built into the library).
// Each V_* macro selects one measured change; results in profiles/r2_c2_diagnosis.md.
// Build one:  mkdir -p alt/v && cp profiles/micro/fft_l2_variants.cu alt/v/fft_l2.cu &&
//   python profiles/micro/build_variant.py NAME alt/v/fft_l2.cu -DV_SW=1   (then profiles/micro/sess_ab_c2.sh alt/NAME.so)
// FFT node, n = 2^16 (the C2 headline): two-pass four-step with the
// intermediate kept in L2.
//
// n = 256 a + b, k = c + 256 d (N1 = N2 = 256): pass 1 (P1) runs the 256-point
// column FFTs over a and applies W_N^{bc}; pass 2 (P2) runs the 256-point row
// FFTs over b.  Work items are 32 KB tiles:
//
//   P1(t, g)  the 16 columns b in [16g, 16g+16) of transform t (256 rows x
//             128 B, one 2-D TMA load, 128B-swizzled) -> column FFTs ->
//             W_N^{bc} -> a scratch ring slot, S[c>>4][b][c&15] (evict-last
//             stores, swizzled so the P2 block needs no transpose).
//   P2(t, g)  the 32 KB block S[g] (one bulk copy from L2) -> row FFTs ->
//             X[16g + c_lo + 256 d] by one 2-D TMA store.
//
// Each point crosses HBM exactly twice (read x, write X: the 16 B compulsory
// traffic); the exchange lives in L2 and is discarded after the P2 read
// (discard.global.L2), so dirty scratch never costs an HBM write-back.
//
// Ordering.  CTAs take tickets from a global counter; tickets map to items in
// the order P1(0..L-1), then P1(L+m), P2(m) alternating, then the last P2s, so
// P2(t) is issued 2L+1 item groups after P1(t).  P2(t) waits (acquire) until
// the 16 P1 items of t have published (release add); P1(t) waits until P2(t-R)
// has released ring slot t mod R.  Every wait is on a strictly smaller ticket,
// held by a CTA that is already resident, so the schedule cannot deadlock for
// any grid.  Lag L = 48, ring R = 128 slots (64 MB of scratch address space).
#include <cmath>
#include <vector>

#include "common.cuh"
#ifndef V_S
#define V_S 2
#endif
#ifndef V_MINB
#define V_MINB 3
#endif
#ifndef V_NOSLEEP
#define V_NOSLEEP 0
#endif
#ifndef V_DISC
#define V_DISC true
#endif
#ifndef V_RING
#define V_RING 128
#endif
#ifndef V_DIRECT
#define V_DIRECT 0
#endif
#ifndef V_SW
#define V_SW 0
#endif
#ifndef V_LAG
#define V_LAG 48
#endif
#ifndef V_DEFER
#define V_DEFER 0
#endif
#ifndef V_CWREL
#define V_CWREL 0
#endif
#ifndef V_TPF
#define V_TPF 0
#endif
#include "fft_plan.cuh"
#include "tma.cuh"
#include "l2ring.cuh"

namespace dpp {

namespace l2x {

constexpr int N = 65536;
constexpr int ITEMS = 16;  // items per pass per transform
using namespace ring;

// ---------------------------------------------------------------------------
// The kernel: warp-specialised, warp-local passes.
//
// Round-1 measurements (profiles/r1_fft_l2.md): a non-persistent version
// (item CTAs, LDG/STG) was latency-bound, a persistent one with CTA barriers
// stalled on the SMEM transposes and the release fences.  v3 moves all of
// that off the compute warps:
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
constexpr int THREADS = (CW + 1 + V_SW) * 32;
constexpr int TILE = 4096;

struct Args {
  float2* scratch;
  int* ctrl;
  const float4* tw256;   // [k][idx] = W256^{k*idx} as (w, i*w)
  const float2* tw4096;  // W4096^e, e < 256
  const float2* tw65536; // W65536^e, e < 256
  int batch, lag, ring;
  float2* out;  // V_DIRECT
};


template <int S, int MINB, bool DISCARD>
__global__ void __launch_bounds__(THREADS, MINB)
fft65536_l2w(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, const Args a) {
  extern __shared__ __align__(1024) float2 smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  __shared__ __align__(8) uint64_t ready[S];  // V_SW: producer -> store warp
  __shared__ __align__(8) uint64_t freed[S];  // V_SW: store warp -> producer (stage read out)
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
      mbar_init(&ready[s], 1);
      mbar_init(&freed[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

#if V_SW
  if (warp == CW + 1) {
    // ---------------------------------------------------------- store warp
    // issues the P2 output stores, so the producer's gpu-scope release never
    // has a bulk store of its own thread in flight
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    for (int k = 0;; ++k) {
      const int s = k % S;
      mbar_wait(&ready[s], (k / S) & 1);
      const int tick = s_tick[s];
      if (tick < 0) break;
      int pass, t;
      l2x::decode(tick >> 4, a.batch, a.lag, pass, t);
      if (pass == 2) {
        tma_store_2d_hint(&tout, 16 * (tick & 15), t * 256, smem + s * TILE, pol);
        bulk_commit();
        bulk_wait_read0();
      }
      mbar_arrive1(&freed[s]);
    }
    bulk_wait0();
    return;
  }
  if (warp == CW) {
    if (lane != 0) return;
    const uint64_t stream_pol = policy_evict_first();
    int head = 0, i = 0;
    auto publish = [&](int k) {
      const int s = k % S;
      int pass, t;
      l2x::decode(s_tick[s] >> 4, a.batch, a.lag, pass, t);
      if (pass == 1) l2x::red_release_add(cnt1 + t, 1);
      else if (t + a.ring < a.batch) l2x::red_release_add(cnt2 + t, 1);
      mbar_arrive1(&ready[s]);
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
        if (i >= S) mbar_wait(&freed[s], ((i - S) / S) & 1);
        s_tick[s] = -1;
        mbar_arrive1(&full[s]);
        break;
      }
      int pass, t;
      l2x::decode(tick >> 4, a.batch, a.lag, pass, t);
      const int g = tick & 15;
      const int* dep = pass == 2 ? cnt1 + t : (t >= a.ring ? cnt2 + (t - a.ring) : nullptr);
      if (dep) {
        while (l2x::ld_acquire(dep) < l2x::ITEMS) {
          if (head < i && mbar_try(&done[head % S], (head / S) & 1)) {
            publish(head);
            ++head;
          } else if (!V_NOSLEEP) {
            __nanosleep(32);
          }
        }
      }
      if (i >= S) mbar_wait(&freed[s], ((i - S) / S) & 1);  // item i - S has left the stage
      s_tick[s] = tick;
      float2* buf = smem + s * TILE;
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
    // the store warp's end marker: stage i % S holds s_tick = -1 (item i - S has been freed)
    mbar_arrive1(&ready[i % S]);
    return;
  }
#endif
  if (warp == CW) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    const uint64_t stream_pol = policy_evict_first();
    int head = 0, i = 0;
    int next_tick = V_TPF ? atomicAdd(a.ctrl, 1) : 0;
    auto publish = [&](int k) {
      const int s = k % S;
      int pass, t;
      l2x::decode(s_tick[s] >> 4, a.batch, a.lag, pass, t);
      const int g = s_tick[s] & 15;
      if (pass == 1) {
        if (!V_CWREL) l2x::red_release_add(cnt1 + t, 1);
      } else {
        if (!V_CWREL && t + a.ring < a.batch) l2x::red_release_add(cnt2 + t, 1);  // lines discarded by the compute warps
        if (!V_DIRECT) {
          tma_store_2d_hint(&tout, 16 * g, t * 256, smem + s * TILE, stream_pol);
          bulk_commit();
        }
      }
    };
#if V_DEFER
    // the gpu-scope release of a finished item is issued after the next load
    // (its stage-bound part — the P2 output store — first), so the fence no
    // longer sits between a stage becoming free and its refill
    int dpass = 0, dt = 0;
    bool dpend = false;
    auto release = [&](int pass, int t) {
      if (pass == 1) l2x::red_release_add(cnt1 + t, 1);
      else if (t + a.ring < a.batch) l2x::red_release_add(cnt2 + t, 1);
    };
    auto flush = [&]() {
      if (dpend) release(dpass, dt);
      dpend = false;
    };
    for (;; ++i) {
      const int s = i % S;
      while (head <= i - S) {
        mbar_wait(&done[head % S], (head / S) & 1);
        flush();
        const int hs = head % S;
        l2x::decode(s_tick[hs] >> 4, a.batch, a.lag, dpass, dt);
        if (dpass == 2) {
          tma_store_2d_hint(&tout, 16 * (s_tick[hs] & 15), dt * 256, smem + hs * TILE, stream_pol);
          bulk_commit();
        }
        dpend = true;
        ++head;
      }
      const int tick = atomicAdd(a.ctrl, 1);
      if (tick >= total) {
        flush();
        s_tick[s] = -1;
        mbar_arrive1(&full[s]);
        break;
      }
      int pass, t;
      l2x::decode(tick >> 4, a.batch, a.lag, pass, t);
      const int g = tick & 15;
      const int* dep = pass == 2 ? cnt1 + t : (t >= a.ring ? cnt2 + (t - a.ring) : nullptr);
      if (dep && l2x::ld_acquire(dep) < l2x::ITEMS) {
        flush();  // the dependency may be this CTA's own deferred item
        while (l2x::ld_acquire(dep) < l2x::ITEMS) {
          if (head < i && mbar_try(&done[head % S], (head / S) & 1)) {
            publish(head);
            ++head;
          } else if (!V_NOSLEEP) {
            __nanosleep(32);
          }
        }
      }
      bulk_wait_read0();  // the stage's previous output tile has left shared memory
      s_tick[s] = tick;
      float2* buf = smem + s * TILE;
      mbar_arrive_expect_tx(&full[s], TILE * sizeof(float2));
      if (pass == 1) {
        tma_load_2d_hint(buf, &tin, 16 * g, t * 256, &full[s], stream_pol);
      } else {
        l2x::fence_proxy_async_global();
        bulk_g2s(buf, a.scratch + (size_t)(t & (a.ring - 1)) * l2x::N + 4096 * g, TILE * sizeof(float2), &full[s]);
      }
      flush();
    }
#else
    for (;; ++i) {
      const int s = i % S;
      while (head <= i - S) {
        mbar_wait(&done[head % S], (head / S) & 1);
        publish(head);
        ++head;
      }
      int tick;
      if (V_TPF) {
        tick = next_tick;
        if (tick < total) next_tick = atomicAdd(a.ctrl, 1);
      } else {
        tick = atomicAdd(a.ctrl, 1);
      }
      if (tick >= total) {
        s_tick[s] = -1;
        mbar_arrive1(&full[s]);
        break;
      }
      int pass, t;
      l2x::decode(tick >> 4, a.batch, a.lag, pass, t);
      const int g = tick & 15;
      const int* dep = pass == 2 ? cnt1 + t : (t >= a.ring ? cnt2 + (t - a.ring) : nullptr);
      if (dep) {
        while (l2x::ld_acquire(dep) < l2x::ITEMS * (V_CWREL ? CW : 1)) {
          if (head < i && mbar_try(&done[head % S], (head / S) & 1)) {
            publish(head);
            ++head;
          } else if (!V_NOSLEEP) {
            __nanosleep(32);
          }
        }
      }
      bulk_wait_read0();  // the stage's previous output tile has left shared memory
      s_tick[s] = tick;
      float2* buf = smem + s * TILE;
      mbar_arrive_expect_tx(&full[s], TILE * sizeof(float2));
      if (pass == 1) {
        tma_load_2d_hint(buf, &tin, 16 * g, t * 256, &full[s], stream_pol);
      } else {
        l2x::fence_proxy_async_global();
        bulk_g2s(buf, a.scratch + (size_t)(t & (a.ring - 1)) * l2x::N + 4096 * g, TILE * sizeof(float2), &full[s]);
      }
    }
#endif
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
    // the P2 block is in shared memory: drop its scratch lines (no HBM write-back)
    if (DISCARD && pass == 2) l2x::discard_l2(slot + 4096 * g + 16 * (tid & 255));
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = lds64(bA + 2048 * j);
    dft16c(v);
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
      if (V_DIRECT) {
        // X[16 g + col + 256 d], d = idx + 16 d1, straight from registers
        float2* o = a.out + (size_t)t * l2x::N + 16 * g + col + 256 * idx;
#pragma unroll
        for (int d1 = 0; d1 < 16; ++d1) st_stream(o + 4096 * d1, v[d1]);
      } else {
      __syncwarp();
      // output tile row d = idx + 16 d1, column col
#pragma unroll
      for (int d1 = 0; d1 < 16; ++d1) sts64(bA + 2048 * d1, v[d1]);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive1(&done[s]);
      if (V_CWREL) {
        if (pass == 1) l2x::red_release_add(a.ctrl + 32 + t, 1);
        else if (t + a.ring < a.batch) l2x::red_release_add(a.ctrl + 32 + a.batch + t, 1);
      }
    }
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

static int g_l2_ctas = 0;
static constexpr size_t L2_SMEM = V_S * 4096 * sizeof(float2) + 8192;

static int l2_prepare() {
  auto kw = l2x::l2w::fft65536_l2w<V_S, V_MINB, V_DISC>;
  DPP_CUDA_CHECK(cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L2_SMEM));
  int per_sm = 0, dev = 0, sms = 0;
  DPP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kw, l2x::l2w::THREADS, L2_SMEM));
  DPP_CUDA_CHECK(cudaGetDevice(&dev));
  DPP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(DPP_ECUDA, "the 2^16 ring kernel does not fit on an SM");
  g_l2_ctas = per_sm * sms;
  return DPP_OK;
}

int fft65536_l2x_init(FftPlan* p) {
  using namespace l2x;
  if (g_l2_ctas == 0)
    if (int rc = l2_prepare()) return rc;
  p->l2_lag = ring_stress() ? 2 : V_LAG;
  p->l2_ring = ring_stress() ? 4 : V_RING;  // a power of two (slot = t & (ring - 1)), > lag
  // tables: W256^{k*idx} k-major (16 x 16 float4 (w, i*w)), then W4096^e and
  // W65536^e (e < 256) as float2 pairs
  const auto t256 = rot_table(256, 256);
  std::vector<float4> all;
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
  if (batch > 0x7fffffff / (2 * ITEMS)) return fail(DPP_EINVAL, "batch %lld too large", (long long)batch);
  if ((size_t)(32 + 2 * batch) * sizeof(int) > p->l2_ctrl_bytes)
    return fail(DPP_EINVAL, "batch %lld exceeds the plan's batch", (long long)batch);
  CUtensorMap tin, tout;
  if (int rc = make_tmap_c64(&tin, in, (uint64_t)batch * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  if (int rc = make_tmap_c64(&tout, out, (uint64_t)batch * 256, 256, 256, 16, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  l2w::Args a;
  a.scratch = p->l2_scratch;
  a.ctrl = p->l2_ctrl;
  a.tw256 = p->l2_tw;
  a.tw4096 = reinterpret_cast<const float2*>(p->l2_tw + 256);
  a.tw65536 = reinterpret_cast<const float2*>(p->l2_tw + 256 + 128);
  a.batch = (int)batch;
  a.out = out;
  a.lag = (int)(batch < p->l2_lag ? batch : p->l2_lag);
  a.ring = p->l2_ring;
  const int64_t items = 2 * ITEMS * batch;
  const unsigned grid = (unsigned)(items < g_l2_ctas ? items : g_l2_ctas);
  // the ring and counters belong to the plan: order this launch after the
  // previous one even when callers use different streams
  DPP_CUDA_CHECK(cudaStreamWaitEvent(s, p->l2_done, 0));
  DPP_CUDA_CHECK(cudaMemsetAsync(p->l2_ctrl, 0, (32 + 2 * (size_t)batch) * sizeof(int), s));
  l2w::fft65536_l2w<V_S, V_MINB, V_DISC><<<grid, l2w::THREADS, L2_SMEM, s>>>(tin, tout, a);
  DPP_LAUNCH_CHECK("fft65536_l2w");
  DPP_CUDA_CHECK(cudaEventRecord(p->l2_done, s));
  return DPP_OK;
}

}  // namespace dpp
