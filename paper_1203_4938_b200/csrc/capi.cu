// extern "C" surface of libdpp_b200.so (declared in include/dpp_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "common.cuh"
#include "fft_plan.cuh"

// The plan owns mutable device state (L2 exchange rings, their counters, the
// large-size scratch) that consecutive executions reuse in stream order: each
// execution waits for the previous one's completion event and records its
// own.  `mu` makes that wait/launch/record sequence atomic across host
// threads, so one plan can be shared by threads and streams.
struct dpp_fft_plan {
  dpp::FftPlan impl;
  std::mutex mu;
};

namespace {
// Executions may come from threads that never touched the runtime (no current
// context: the driver-API tensor-map encode would fail with
// CUDA_ERROR_INVALID_CONTEXT): make the plan's device current for the call
// and restore the caller's device afterwards.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

namespace dpp {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

void fft_plan_release(FftPlan* p) {
  if (!p) return;
  if (p->tw_a) cudaFree(p->tw_a);
  if (p->tw_b) cudaFree(p->tw_b);
  if (p->ctw_a) cudaFree(p->ctw_a);
  if (p->ctw_b) cudaFree(p->ctw_b);
  p->tw_a = p->tw_b = p->ctw_a = p->ctw_b = nullptr;
  if (p->l2_tw) cudaFree(p->l2_tw);
  if (p->l2_scratch) cudaFree(p->l2_scratch);
  if (p->l2_ctrl) cudaFree(p->l2_ctrl);
  if (p->l2_done) cudaEventDestroy(p->l2_done);
  p->l2_tw = nullptr;
  p->l2_scratch = nullptr;
  p->l2_ctrl = nullptr;
  p->l2_done = nullptr;
  if (p->rows) {
    fft_plan_release(p->rows);
    delete p->rows;
    p->rows = nullptr;
  }
  if (p->xcols) {
    fft_plan_release(p->xcols);
    delete p->xcols;
    p->xcols = nullptr;
  }
  if (p->cols) {
    fft_plan_release(p->cols);
    delete p->cols;
    p->cols = nullptr;
  }
  if (p->big_tw) cudaFree(p->big_tw);
  if (p->big_scratch) cudaFree(p->big_scratch);
  p->big_tw = p->big_scratch = nullptr;
}

}  // namespace dpp

extern "C" {

int dpp_abi_version(void) { return DPP_ABI_VERSION; }

const char* dpp_last_error(void) { return dpp::g_last_error; }

int dpp_fft_plan_create(dpp_fft_plan** plan, int rank, int64_t n0, int64_t n1, int64_t batch,
                        size_t* workspace_bytes) {
  if (!plan) return dpp::fail(DPP_EINVAL, "plan pointer is NULL");
  *plan = nullptr;
  if (rank != 1 && rank != 2) return dpp::fail(DPP_EINVAL, "rank must be 1 or 2, got %d", rank);
  if (batch < 0) return dpp::fail(DPP_EINVAL, "batch must be >= 0, got %lld", (long long)batch);
  auto* h = new (std::nothrow) dpp_fft_plan();
  if (!h) return dpp::fail(DPP_EINVAL, "out of host memory");
  h->impl.rank = rank;
  h->impl.n0 = n0;
  h->impl.n1 = rank == 2 ? n1 : 1;
  h->impl.batch = batch;
  cudaGetDevice(&h->impl.device);
  const int rc = rank == 1 ? dpp::fft1d_plan_init(&h->impl) : dpp::fft2d_plan_init(&h->impl);
  if (rc != DPP_OK) {
    dpp::fft_plan_release(&h->impl);
    delete h;
    return rc;
  }
  if (workspace_bytes) *workspace_bytes = 0;
  *plan = h;
  return DPP_OK;
}

int dpp_fft_plan_supported(int rank, int64_t n0, int64_t n1) {
  if (rank == 1) return n0 >= 2 && (n0 & (n0 - 1)) == 0 && n0 <= (1LL << 30);
  if (rank == 2) return dpp::fft2d_shape_supported(n0, n1) ? 1 : 0;
  return 0;
}

int dpp_fft_plan_describe(const dpp_fft_plan* plan, char* buf, size_t len) {
  if (!plan || !buf || len == 0) return dpp::fail(DPP_EINVAL, "bad describe arguments");
  snprintf(buf, len, "%s", plan->impl.desc);
  return DPP_OK;
}

int dpp_fft_c2c_forward_batch(const dpp_fft_plan* plan, const float* in, float* out, int64_t batch,
                              void* workspace, void* stream) {
  (void)workspace;
  if (!plan) return dpp::fail(DPP_EINVAL, "plan is NULL");
  if (batch < 0 || batch > plan->impl.batch)
    return dpp::fail(DPP_EINVAL, "batch %lld outside the planned 0..%lld", (long long)batch,
                     (long long)plan->impl.batch);
  if (batch > 0 && (!in || !out)) return dpp::fail(DPP_EINVAL, "NULL data pointer");
  auto s = static_cast<cudaStream_t>(stream);
  const auto* src = reinterpret_cast<const float2*>(in);
  auto* dst = reinterpret_cast<float2*>(out);
  std::lock_guard<std::mutex> g(const_cast<dpp_fft_plan*>(plan)->mu);
  DeviceScope dev_scope(plan->impl.device);
  return plan->impl.rank == 1 ? dpp::fft1d_execute(&plan->impl, src, dst, batch, s)
                              : dpp::fft2d_execute(&plan->impl, src, dst, batch, s);
}

int dpp_fft_c2c_forward(const dpp_fft_plan* plan, const float* in, float* out, void* workspace,
                        void* stream) {
  if (!plan) return dpp::fail(DPP_EINVAL, "plan is NULL");
  return dpp_fft_c2c_forward_batch(plan, in, out, plan->impl.batch, workspace, stream);
}

int dpp_fft_c2c_columns(const dpp_fft_plan* plan, float* data, int64_t batch, void* stream) {
  if (!plan) return dpp::fail(DPP_EINVAL, "plan is NULL");
  if (plan->impl.rank != 2) return dpp::fail(DPP_EINVAL, "column pass needs a rank-2 plan");
  if (batch < 0 || batch > plan->impl.batch)
    return dpp::fail(DPP_EINVAL, "batch %lld outside the planned 0..%lld", (long long)batch,
                     (long long)plan->impl.batch);
  std::lock_guard<std::mutex> g(const_cast<dpp_fft_plan*>(plan)->mu);
  DeviceScope dev_scope(plan->impl.device);
  return dpp::fft2d_columns_execute(&plan->impl, reinterpret_cast<float2*>(data), batch,
                                    static_cast<cudaStream_t>(stream));
}

int dpp_fft_twiddle(float* data, int64_t rows, int64_t cols, int64_t col0, int64_t n, void* stream) {
  if (rows * cols > 0 && !data) return dpp::fail(DPP_EINVAL, "NULL data pointer");
  return dpp::fft_twiddle_slab(reinterpret_cast<float2*>(data), rows, cols, col0, n,
                               static_cast<cudaStream_t>(stream));
}

int dpp_fft2d_u8_spectrum(const dpp_fft_plan* plan, const uint8_t* in, uint8_t* out, float alpha, float* work,
                          int64_t batch, void* stream) {
  if (!plan) return dpp::fail(DPP_EINVAL, "plan is NULL");
  const dpp::FftPlan& p = plan->impl;
  if (p.rank != 2) return dpp::fail(DPP_EINVAL, "the fused u8 -> 2-D FFT -> spectrum path needs a rank-2 plan");
  if (batch < 0 || batch > p.batch)
    return dpp::fail(DPP_EINVAL, "batch %lld outside the planned 0..%lld", (long long)batch, (long long)p.batch);
  // the spectrum epilogue exists for the 4096- and 16384-row rings only:
  // reject everything else before the row pass is launched
  if (!p.rows || !p.rows->ws4k || !p.col_ring || (p.n0 != 4096 && p.n0 != 16384))
    return dpp::fail(DPP_ENOTSUP,
                     "no fused schedule for %lld x %lld (needs 4096 or 16384 rows of 4096 columns and a ring "
                     "column pass)",
                     (long long)p.n0, (long long)p.n1);
  if (batch == 0) return DPP_OK;
  if (!in || !out || !work) return dpp::fail(DPP_EINVAL, "NULL data pointer");
  auto s = static_cast<cudaStream_t>(stream);
  auto* w = reinterpret_cast<float2*>(work);
  std::lock_guard<std::mutex> g(const_cast<dpp_fft_plan*>(plan)->mu);
  DeviceScope dev_scope(plan->impl.device);
  // real images in pairs: one complex transform per pair (z = a + i b, the
  // half spectra separated in the row pass), each spectrum written with its
  // mirror; an odd last image takes the single-image schedule
  const int64_t npairs = batch / 2, img = p.n0 * p.n1;
  if (npairs) {
    float2* side = w + npairs * img;  // 2 npairs n0 values; work holds batch images
    if (int rc = dpp::fft4096_ws_execute_u8_pair(p.rows, in, w, npairs, (int)p.n0, s)) return rc;
    if (int rc = dpp::fft2d_colring_execute(&p, w, npairs, s, out, alpha, nullptr, nullptr, nullptr, false, side))
      return rc;
  }
  if (batch & 1) {
    const int64_t off = 2 * npairs * img;
    if (int rc = dpp::fft4096_ws_execute_u8(p.rows, in + off, w, p.n0, s)) return rc;
    return dpp::fft2d_colring_execute(&p, w, 1, s, out + off, alpha);
  }
  return DPP_OK;
}

int dpp_fft2d_columns_sharded(const dpp_fft_plan* plan, const float* const* slabs, float* const* outs, int nranks,
                              int rank, int transpose_back, int64_t batch, void* stream) {
  if (!plan || !slabs || !outs) return dpp::fail(DPP_EINVAL, "NULL argument to dpp_fft2d_columns_sharded");
  if (plan->impl.rank != 2) return dpp::fail(DPP_EINVAL, "the sharded column pass needs a rank-2 plan");
  std::lock_guard<std::mutex> g(const_cast<dpp_fft_plan*>(plan)->mu);
  DeviceScope dev_scope(plan->impl.device);
  return dpp::fft2d_colring_execute_peer(&plan->impl, reinterpret_cast<const float2* const*>(slabs),
                                         reinterpret_cast<float2* const*>(outs), nranks, rank, transpose_back, batch,
                                         static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// SURVEY §8(b) `dpp_fft2d_c2c_fwd_sharded`: the whole row-sharded transform in
// one call over a peer group (the mapped slabs and flag arrays of every rank)

struct dpp_peer_group {
  int nranks = 0, rank = 0;
  float* slabs[8] = {nullptr};
  int* flags[8] = {nullptr};
  double timeout_s = 30.0;
  int epoch = 0;
  std::mutex mu;
};

int dpp_peer_group_create(dpp_peer_group** group, int nranks, int rank, float* const* slabs, int* const* flags,
                          double timeout_s) {
  if (!group) return dpp::fail(DPP_EINVAL, "NULL group pointer");
  *group = nullptr;
  if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || !slabs || !flags)
    return dpp::fail(DPP_EINVAL, "bad peer group (%d ranks, rank %d)", nranks, rank);
  auto* g = new (std::nothrow) dpp_peer_group();
  if (!g) return dpp::fail(DPP_EINVAL, "out of host memory");
  g->nranks = nranks;
  g->rank = rank;
  g->timeout_s = timeout_s > 0 ? timeout_s : 30.0;
  for (int j = 0; j < nranks; ++j) {
    if (!slabs[j] || !flags[j]) {
      delete g;
      return dpp::fail(DPP_EINVAL, "NULL slab or flag pointer for rank %d", j);
    }
    g->slabs[j] = slabs[j];
    g->flags[j] = flags[j];
  }
  *group = g;
  return DPP_OK;
}

void dpp_peer_group_destroy(dpp_peer_group* group) { delete group; }

int dpp_fft2d_c2c_fwd_sharded(const dpp_fft_plan* plan, dpp_peer_group* group, const float* rows_in, float* out,
                              int transpose_back, int64_t batch, void* stream) {
  if (!plan || !group) return dpp::fail(DPP_EINVAL, "NULL plan or peer group");
  const dpp::FftPlan& p = plan->impl;
  if (p.rank != 2 || !p.rows) return dpp::fail(DPP_EINVAL, "the sharded transform needs a rank-2 plan");
  if (batch < 0 || batch > p.batch)
    return dpp::fail(DPP_EINVAL, "batch %lld outside the planned 0..%lld", (long long)batch, (long long)p.batch);
  if (!transpose_back && !out) return dpp::fail(DPP_EINVAL, "column-slab output needs `out`");
  if (batch == 0) return DPP_OK;
  const int P = group->nranks;
  if (p.n0 % P) return dpp::fail(DPP_EINVAL, "%lld rows do not split over %d ranks", (long long)p.n0, P);
  auto s = static_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> g(const_cast<dpp_fft_plan*>(plan)->mu);
  std::lock_guard<std::mutex> gg(group->mu);
  DeviceScope dev_scope(p.device);
  float2* slab = reinterpret_cast<float2*>(group->slabs[group->rank]);
  const float2* src = rows_in ? reinterpret_cast<const float2*>(rows_in) : slab;
  // 1. row pass of this rank's rows into its (peer-visible) slab
  if (int rc = dpp::fft1d_execute(p.rows, src, slab, batch * (p.n0 / P), s)) return rc;
  // 2. every slab is row-transformed
  if (int rc = dpp_peer_barrier(group->flags, P, group->rank, ++group->epoch, group->timeout_s, stream)) return rc;
  // 3. column pass with the exchange fused in
  float* col_out[8] = {reinterpret_cast<float*>(out)};
  if (int rc = dpp::fft2d_colring_execute_peer(&p, reinterpret_cast<const float2* const*>(group->slabs),
                                               reinterpret_cast<float2* const*>(transpose_back ? group->slabs
                                                                                               : col_out),
                                               P, group->rank, transpose_back, batch, s))
    return rc;
  // 4. no rank reuses its slab while peers still read or write it
  return dpp_peer_barrier(group->flags, P, group->rank, ++group->epoch, group->timeout_s, stream);
}

void dpp_fft_plan_destroy(dpp_fft_plan* plan) {
  if (!plan) return;
  dpp::fft_plan_release(&plan->impl);
  delete plan;
}

int dpp_fft_leaf(int k, const float* x, float* y, int64_t items, void* stream) {
  if (items < 0) return dpp::fail(DPP_EINVAL, "items must be >= 0");
  return dpp::leaf_execute(k, x, y, items, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
