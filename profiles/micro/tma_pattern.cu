// HBM access-pattern microbenchmark for the L2-ring FFT kernels: a persistent
// TMA copy (load a box into a shared-memory stage, TMA-store it to the same
// coordinates of the output) over 2 GiB of complex64, with the box shapes the
// ring kernels use, timed with CUDA events.  No math, no L2 exchange, no
// cross-CTA dependencies — the ceiling the pattern itself allows.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_pattern tma_pattern.cu -lcuda
//   ./tma_pattern
//
// modes (rows of 256 complex = 2 KB, i.e. one 2^16 transform = 256 rows):
//   c2     box 16 cols x 256 rows (128 B x 256 at 2 KB stride, 32 KB), SWIZZLE_128B
//          — the C2 P1 load / P2 store pattern
//   contig box 256 cols x 16 rows (16 contiguous rows, 32 KB)
//   w32    box 32 cols x 256 rows (256 B x 256 at 2 KB stride, 64 KB)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

#define CK(x)                                                                        \
  do {                                                                               \
    auto e_ = (x);                                                                   \
    if (e_ != 0) {                                                                   \
      fprintf(stderr, "%s:%d: error %d\n", __FILE__, __LINE__, (int)e_);             \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(32) copy_kernel(const __grid_constant__ CUtensorMap tin,
                                                  const __grid_constant__ CUtensorMap tout, int ntiles,
                                                  int tile_bytes, int cols_per_tile, int rows_per_tile,
                                                  int tiles_per_band) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto coords = [&](int tile, int& x, int& y) {
    const int band = tile / tiles_per_band, g = tile - band * tiles_per_band;
    x = g * cols_per_tile;
    y = band * rows_per_tile;
  };
  auto load = [&](int s, int tile) {
    int x, y;
    coords(tile, x, y);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(tile_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(su32(smem + (size_t)s * tile_bytes)),
        "l"(&tin), "r"(x), "r"(y), "r"(su32(&full[s]))
        : "memory");
  };
  const int first = blockIdx.x, step = gridDim.x;
  for (int k = 0; k < S; ++k)
    if (first + k * step < ntiles) load(k, first + k * step);
  for (int j = 0;; ++j) {
    const int tile = first + j * step;
    if (tile >= ntiles) break;
    const int s = j % S;
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
            su32(&full[s])),
        "r"((j / S) & 1)
        : "memory");
    int x, y;
    coords(tile, x, y);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tout),
                 "r"(x), "r"(y), "r"(su32(smem + (size_t)s * tile_bytes))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage stored one iteration ago (its store had this iteration's wait to drain)
    if (j >= 1) {
      const int pt = first + (j - 1 + S) * step;
      if (pt < ntiles) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        load((j - 1) % S, pt);
      }
    }
  }
  // the last stage's refill never happens (no tile j - 1 + S beyond the end)
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled enc;

template <int S>
static int launch(const CUtensorMap& ti, const CUtensorMap& to, int grid, size_t sm, int ntiles, int tile_bytes,
                  int bc, int br, int tpb) {
  CK(cudaFuncSetAttribute(copy_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  copy_kernel<S><<<grid, 32, sm>>>(ti, to, ntiles, tile_bytes, bc, br, tpb);
  return 0;
}

static int tmap(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, uint32_t br, uint32_t bc,
                CUtensorMapSwizzle sw) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 8};
  const cuuint32_t box[2] = {bc, br};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main() {
  CK(cuInit(0));
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  const uint64_t cols = 256, rows = (1ull << 28) / cols;  // 2^28 complex = 2 GiB
  void *in, *out;
  CK(cudaMalloc(&in, rows * cols * 8));
  CK(cudaMalloc(&out, rows * cols * 8));
  CK(cudaMemset(in, 1, rows * cols * 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  struct Mode {
    const char* name;
    uint32_t br, bc;
    CUtensorMapSwizzle sw;
  } modes[] = {{"c2", 256, 16, CU_TENSOR_MAP_SWIZZLE_128B},
               {"contig", 16, 256, CU_TENSOR_MAP_SWIZZLE_NONE},
               {"w32", 256, 32, CU_TENSOR_MAP_SWIZZLE_NONE},
               {"c2_128r", 128, 16, CU_TENSOR_MAP_SWIZZLE_128B}};
  struct Cfg {
    int ctas_per_sm, stages;
  } cfgs[] = {{3, 2}, {1, 6}, {2, 3}};
  for (auto& m : modes) {
    CUtensorMap ti, to;
    CK(tmap(&ti, in, rows, cols, m.br, m.bc, m.sw));
    CK(tmap(&to, out, rows, cols, m.br, m.bc, m.sw));
    const int tile_bytes = (int)(m.br * m.bc * 8);
    const int tiles_per_band = (int)(cols / m.bc);
    const int ntiles = (int)(rows / m.br) * tiles_per_band;
    for (auto& c : cfgs) {
      const int stages = tile_bytes > 32768 ? c.stages / 2 : c.stages;
      if (stages < 2) continue;  // the refill order below needs two stages
      const size_t sm = (size_t)stages * tile_bytes;
      if (sm > 200 * 1024 / c.ctas_per_sm + 1024) continue;
      auto (*k)(const CUtensorMap&, const CUtensorMap&, int, size_t, int, int, int, int, int) -> int = nullptr;
      switch (stages) {
        case 2: k = launch<2>; break;
        case 3: k = launch<3>; break;
        case 6: k = launch<6>; break;
        default: continue;
      }
      const int grid = sms * c.ctas_per_sm;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e30f, tot = 0;
      for (int it = 0; it < 8; ++it) {
        cudaEventRecord(e0);
        CK(k(ti, to, grid, sm, ntiles, tile_bytes, (int)m.bc, (int)m.br, tiles_per_band));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2) {
          tot += ms;
          if (ms < best) best = ms;
        }
      }
      CK(cudaGetLastError());
      const double bytes = 2.0 * rows * cols * 8;
      printf("{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"stages\": %d, \"tile_kb\": %d, \"ms_best\": %.4f, "
             "\"ms_mean\": %.4f, \"GBps\": %.1f}\n",
             m.name, c.ctas_per_sm, stages, tile_bytes / 1024, best, tot / 6, bytes / best / 1e6);
    }
  }
  return 0;
}
