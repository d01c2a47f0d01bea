// Plan object behind the opaque dpp_fft_plan handle.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

struct dpp_fft_plan;  // public opaque name (include/dpp_b200.h)

namespace dpp {

struct FftPlan {
  enum Kind { SMALL = 1, CLUSTER = 2, L2X = 3, LARGE = 4 };
  int rank = 1;
  int64_t n0 = 0, n1 = 0, batch = 0;  // rank 1: n0 points; rank 2: n0 rows x n1 cols
  int device = 0;
  // 1-D schedule along a row (rank 1: the transform; rank 2: the row pass)
  int kind = 0;
  int64_t n1a = 0, n2a = 0;  // cluster split n = n1a * n2a
  int cluster = 1;
  int mode = 3;              // cluster exchange variant (fft.cu)
  int max_clusters = 0;      // co-resident clusters for the persistent variant
  float2* tw_a = nullptr;    // coarse twiddles (W_n for SMALL, W_max(n1a,n2a) for CLUSTER)
  float2* tw_b = nullptr;    // fine twiddles W_n^lo
  // rank 2: column pass schedule
  FftPlan* rows = nullptr;   // 1-D plan along n1 (row pass)
  int col_kind = 0;
  int64_t col_split = 0;     // column length n0 = col_split * (n0 / col_split)
  int col_cluster = 1;
  int col_width = 0;         // columns per tile
  float2* ctw_a = nullptr;
  float2* ctw_b = nullptr;
  // L2X (n = 2^16 two-pass, fft_l2.cu): scratch ring, ticket/counters, tables
  int l2_lag = 0, l2_ring = 0;
  float4* l2_tw = nullptr;
  float2* l2_scratch = nullptr;
  int* l2_ctrl = nullptr;
  size_t l2_ctrl_bytes = 0;
  cudaEvent_t l2_done = nullptr;
  // rank 2: column pass through the L2 ring (fft2d_l2.cu) instead of the cluster kernel
  int col_ring = 0, col_ring_ctas = 0;
  // rank 1, n = 2^14: L2-ring kernel for batches of 4 (fft16k_l2.cu), cluster kernel for the rest
  int ring16k = 0;
  // rank 1, n = 4096: warp-specialised single-CTA kernel (fft4k.cu)
  int ws4k = 0;
  // rank 1, n = 2^17: L2-ring kernel, one transform per unit (fft128k_l2.cu)
  int ring128k = 0;
  // rank 1, n > 2^17 (fft_large.cu): transpose, row pass (rows), twiddled column ring (cols)
  FftPlan* cols = nullptr;
  // two-pass schedule (n = A x Bc, both 4096 or 16384): xcols = A-point column
  // ring with transposed output (replaces transpose + row pass)
  FftPlan* xcols = nullptr;
  float2* big_tw = nullptr;       // W_N^m, m < 16384, then W_N^(16384 h)
  float2* big_scratch = nullptr;  // in-place calls: big_chunk transforms at a time
  int64_t big_chunk = 0;
  char desc[256] = {0};
};

int fft1d_plan_init(FftPlan* p);
int fft1d_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft2d_plan_init(FftPlan* p);
bool fft2d_shape_supported(int64_t n0, int64_t n1);
int fft2d_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft2d_columns_execute(const FftPlan* p, float2* data, int64_t batch, cudaStream_t s);
void fft_plan_release(FftPlan* p);
int fft65536_l2x_init(FftPlan* p);
int fft65536_l2x_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft2d_colring_init(FftPlan* p);
int fft2d_colring_execute(const FftPlan* p, float2* data, int64_t batch, cudaStream_t s,
                          uint8_t* spec_out = nullptr, float alpha = 0.f, float2* dst = nullptr,
                          const float2* twlo = nullptr, const float2* twhi = nullptr, bool xp = false,
                          float2* side = nullptr);
int fft_large_init(FftPlan* p);
int fft_twiddle_slab(float2* data, int64_t rows, int64_t cols, int64_t c0, int64_t n, cudaStream_t s);
int fft_large_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft2d_colring_execute_peer(const FftPlan* p, const float2* const* slabs, float2* const* outs, int np, int rank,
                               int tb, int64_t batch, cudaStream_t s);
int fft16k_l2_init(FftPlan* p);
int fft16k_l2_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft128k_l2_init(FftPlan* p);
int fft128k_l2_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft4096_ws_init(FftPlan* p);
int fft4096_ws_execute(const FftPlan* p, const float2* in, float2* out, int64_t batch, cudaStream_t s);
int fft4096_ws_execute_u8(const FftPlan* p, const uint8_t* in, float2* out, int64_t batch, cudaStream_t s);
int fft4096_ws_execute_u8_pair(const FftPlan* p, const uint8_t* in, float2* out, int64_t npairs, int rows,
                               cudaStream_t s);
int leaf_execute(int k, const float* x, float* y, int64_t items, cudaStream_t s);

}  // namespace dpp
