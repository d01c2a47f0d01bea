/*
 * dpp_b200.h — C ABI of the B200 (sm_100a) FFT and block-compression nodes.
 *
 * This is the drop-in boundary.  The reference (arXiv 1203.4938 platform,
 * package `dpp`) has no FFI: its per-node execution point is the Python call
 *   _run_instance(kernel, items, inputs, outputs, parallelism, budget, record)
 *   (/root/reference/pkg/src/dpp/engine.py:218-235)
 * which hands flat little-endian scalar buffers to the lockstep
 * interpreter run_lanes (kernel/interp.py:471-485).  Every function below
 * replaces that call for one node kind, taking the same flat buffers as
 * device pointers plus the caller's cudaStream_t (passed as void*).  The host
 * binding is ctypes (paper_1203_4938_b200/_lib.py); INTEGRATION.md shows the
 * stub a maintainer of the reference would add.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers owned by the caller (PyTorch
 *    allocates).  No entry point allocates device memory except plan
 *    creation (twiddle tables; for n = 2^16 also the L2 exchange ring,
 *    128 slots x 512 KB, and its counters), freed by *_destroy.
 *  - Every launch is asynchronous on `stream` (cudaStream_t; NULL = legacy).
 *  - Return 0 (DPP_OK) or an error code; dpp_last_error() returns the
 *    thread-local message of the last failure.  Host mapping:
 *      DPP_EINVAL  -> PlanError / ValueError       (errors.py:62, fft.py:134-139)
 *      DPP_ECUDA   -> EngineRuntimeError (DeviceError)   (errors.py:66-81)
 *      DPP_ENCCL   -> EngineRuntimeError (DeviceError)
 *  - Entry points are re-entrant; plans are immutable after creation and may
 *    be shared by threads (engine.py:292-317 runs chunks on thread pools).
 *    Executions of one plan that owns an exchange ring are ordered on the
 *    device (each launch waits on an event recorded by the previous one),
 *    whatever streams the callers use.
 *  - Complex data is interleaved (re, im) binary32, exactly the reference's
 *    complex64 view (fft.py:160-163).
 */
#ifndef DPP_B200_H
#define DPP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPP_ABI_VERSION 1

#define DPP_OK 0
#define DPP_EINVAL 1
#define DPP_ECUDA 2
#define DPP_ENCCL 3
#define DPP_ENOTSUP 4

/* Library identity / diagnostics. */
int dpp_abi_version(void);
const char* dpp_last_error(void);

/* ------------------------------------------------------------------------
 * FFT node
 * ------------------------------------------------------------------------ */

typedef struct dpp_fft_plan dpp_fft_plan;

/* Create a forward, unnormalised complex-to-complex plan.
 *   rank 1: `batch` contiguous transforms of n0 points (n1 ignored).
 *   rank 2: `batch` contiguous n0 x n1 row-major 2-D transforms (n0 256..32768).
 * Sizes must be powers of two >= 2 (same rule as FftPlan, fft.py:133-139);
 * rank 1 up to 2^30 (above 2^20: two HBM passes for 2^22 .. 2^30, three for
 * 2^21; in-place calls stage
 * through a plan-owned scratch of <= 256 MB or one transform, allocated on
 * the first in-place call); in and out must be equal or disjoint.
 * *workspace_bytes receives the scratch the execute call needs (may be 0).
 * Replaces: apps/fft.py:150-174 `fft` (host bit-reversal fft.py:159, leaf
 * DFT node fft.py:162, host binary64 butterflies fft.py:165-173). */
int dpp_fft_plan_create(dpp_fft_plan** plan, int rank, int64_t n0, int64_t n1,
                        int64_t batch, size_t* workspace_bytes);

/* 1 when dpp_fft_plan_create would accept (rank, n0, n1), else 0.  Pure
 * shape rules: no device, no allocation (plan-time validation in the graph
 * engine, engine.py:82-135, must not touch a GPU). */
int dpp_fft_plan_supported(int rank, int64_t n0, int64_t n1);

/* Human-readable kernel schedule of a plan (for logs and bench lines). */
int dpp_fft_plan_describe(const dpp_fft_plan* plan, char* buf, size_t len);

/* Execute: in/out hold batch * n0 (* n1) complex64; in == out is allowed.
 * `workspace` is reserved (pass NULL): scratch is plan-owned. */
int dpp_fft_c2c_forward(const dpp_fft_plan* plan, const float* in, float* out,
                        void* workspace, void* stream);

/* Same plan, different batch count (<= the planned batch). */
int dpp_fft_c2c_forward_batch(const dpp_fft_plan* plan, const float* in, float* out,
                              int64_t batch, void* workspace, void* stream);

/* Column pass only of a rank-2 plan, in place: for each of `batch` n0 x n1
 * row-major arrays, the n0-point FFT of every column.  The row-sharded 2-D
 * transform runs it on the column slab each rank holds after the all-to-all
 * (SURVEY §8(e) C3). */
int dpp_fft_c2c_columns(const dpp_fft_plan* plan, float* data, int64_t batch, void* stream);

/* Four-step twiddle of the row-sharded 1-D transform, in place: for a
 * rows x cols row-major complex64 block whose first column is global column
 * col0 of an R x C view of an n-point signal, data[r][c] *= W_n^{r (col0 + c)}
 * (angles in binary64 from the exact integer phase).  The sharded 1-D FFT
 * (distributed.fft1d_row_sharded; the reference's fft() for any power of two,
 * apps/fft.py:150-174) applies it to each rank's column slab between the
 * column FFTs and the all-to-all back to row slabs. */
int dpp_fft_twiddle(float* data, int64_t rows, int64_t cols, int64_t col0, int64_t n, void* stream);

/* C5 fusion: to_complex -> 2-D FFT -> spectrum_u8 in two passes.  in: batch
 * n0 x n1 u8 images; out: batch n0 x n1 u8 spectra (the spectrum_u8 node's
 * arithmetic); work: batch * n0 * n1 complex64 (the row-pass result).  Needs
 * n1 = 4096 and n0 in {4096, 16384} (DPP_ENOTSUP otherwise: run the three
 * nodes separately).  The executor uses it when the graph has exactly that
 * chain with no other consumer of the intermediate edges.  Images go in
 * pairs, one complex transform of z = a + i b per pair with the two real
 * spectra separated in the row pass (X[k] = (Z[k] + conj Z[-k]) / 2) and
 * each written together with its point mirror; the spectra therefore differ
 * from the three separate nodes by float32 rounding (a count of off-by-one
 * bytes, within the adapter's tolerance) and are exactly point-symmetric.
 * An odd last image runs the single-image schedule. */
int dpp_fft2d_u8_spectrum(const dpp_fft_plan* plan, const uint8_t* in, uint8_t* out, float alpha, float* work,
                          int64_t batch, void* stream);

void dpp_fft_plan_destroy(dpp_fft_plan* plan);

/* Row-sharded 2-D transform (SURVEY §8(b) `dpp_fft2d_c2c_fwd_sharded`, §8(e)
 * C3) with the all-to-all fused into the column pass: no NCCL on the data
 * path.  The reference has no 2-D node; the oracle is the row-then-column
 * composition of apps/fft.py:150-174.  Each of `nranks` processes (one per
 * GPU) holds rows [rank*n0/P, (rank+1)*n0/P) of every image in a
 * batch x (n0/P) x n1 row slab and has already run the row pass
 * (dpp_fft_c2c_forward_batch of a rank-1 n1 plan) on it; after a
 * dpp_peer_barrier, rank q computes the n0-point FFTs of columns
 * [q*n1/P, (q+1)*n1/P), reading every rank's slab directly (peer-mapped
 * pointers, slabs[j] for rank j, NVLink loads).  transpose_back != 0: the
 * results are stored into every rank's row slab outs[j] (natural row-sharded
 * layout; outs may equal slabs); else into this rank's batch x n0 x (n1/P)
 * column slab outs[0].  A second dpp_peer_barrier must follow before any rank
 * reuses its slabs.  plan: rank 2, n0 x n1, n0 in 1024 .. 32768
 * (DPP_ENOTSUP otherwise); nranks a power of two <= 8 dividing n0/256;
 * n1 a multiple of 16*nranks. */
int dpp_fft2d_columns_sharded(const dpp_fft_plan* plan, const float* const* slabs, float* const* outs,
                              int nranks, int rank, int transpose_back, int64_t batch, void* stream);

/* CUDA IPC for the peer-mapped slabs: handle (64 bytes) and byte offset of
 * `ptr` inside its allocation; open maps a peer allocation's base into this
 * process (peer access enabled lazily); close unmaps it. */
int dpp_ipc_get_handle(const void* ptr, void* handle, uint64_t* offset);
int dpp_ipc_open(const void* handle, void** base);
int dpp_ipc_close(void* base);

/* Stream-ordered barrier over peer-mapped int32[8] flag arrays (flags[j] =
 * rank j's, zero-initialised; epoch increases by one per barrier): stores
 * epoch into slot `rank` of every array (system-scope release) and waits for
 * every slot of its own (acquire).  Traps after timeout_s instead of hanging. */
int dpp_peer_barrier(int* const* flags, int nranks, int rank, int epoch, double timeout_s, void* stream);

/* The whole row-sharded transform in one call (SURVEY §8(b)
 * `dpp_fft2d_c2c_fwd_sharded`; the peer group replaces the NCCL communicator
 * of that sketch: no collective library on the data path).  A group holds
 * every rank's peer-mapped row slab (batch x n0/P x n1 complex64) and flag
 * array (int32[8], zeroed) — slabs[rank]/flags[rank] are this rank's own —
 * and the barrier epoch.  The call: row pass of rows_in (NULL: the slab
 * already holds the rows) into slabs[rank], barrier, fused column/exchange
 * pass, barrier.  transpose_back != 0: the result is this rank's rows in
 * slabs[rank] (`out` unused); else this rank's batch x n0 x (n1/P) column
 * slab in `out`.  All ranks call it with the same plan shape and batch. */
typedef struct dpp_peer_group dpp_peer_group;
int dpp_peer_group_create(dpp_peer_group** group, int nranks, int rank, float* const* slabs, int* const* flags,
                          double timeout_s);
void dpp_peer_group_destroy(dpp_peer_group* group);
int dpp_fft2d_c2c_fwd_sharded(const dpp_fft_plan* plan, dpp_peer_group* group, const float* rows_in, float* out,
                              int transpose_back, int64_t batch, void* stream);

/* The reference's quadratic oracle naive_dft (apps/fft.py:32-42) on the
 * device: binary64 accumulation, rounded to complex64; `batch` signals of n. */
int dpp_naive_dft(const float* x, float* y, int64_t n, int64_t batch, void* stream);

/* Leaf DFT node dft{2,4,8} (apps/fft.py:86-123): one dense 2^k-point DFT per
 * work-item over float{2^(k+1)} vectors whose lanes sit at bit-reversed
 * offsets.  Arithmetic is the generated body's exactly: binary32, terms in
 * source order, left-to-right, no contraction -> bit-identical to the
 * reference engine.  x, y: items * 2^(k+1) floats. */
int dpp_fft_leaf(int k, const float* x, float* y, int64_t items, void* stream);

/* ------------------------------------------------------------------------
 * Block-compression node (apps/imgc.py)
 * ------------------------------------------------------------------------ */

/* Drop-in replacements of the four reference nodes, same io, bit-exact.
 *   ycbcr     imgc.py:128-140   rgba: pixels*4 u8 -> yl, cb, cr: pixels f32
 *   boxdown   imgc.py:143-152   blk: blocks*16 f32 -> avg: blocks f32
 *   gradient  imgc.py:155-166   lum: items f32 -> dx, dy: items f32
 *             (width/height are the constants baked into the generated body;
 *              items is the chunk's work-item count; a read past the chunk
 *              is a fault exactly as the interpreter's bounds check,
 *              kernel/interp.py:222-284: DPP_EINVAL + first faulting item)
 *   vqnearest imgc.py:169-185   blk, cbk: items*16 f32 -> idx: items i32
 *             (the chunk's cbk holds codebook_size centroids, as the
 *              reference tiles it per chunk, imgc.py:406-423) */
int dpp_imgc_ycbcr(const uint8_t* rgba, float* yl, float* cb, float* cr,
                   int64_t pixels, void* stream);
int dpp_imgc_boxdown(const float* blk, float* avg, int64_t blocks, void* stream);
int dpp_imgc_gradient(const float* lum, float* dx, float* dy, int64_t width,
                      int64_t height, int64_t items, int64_t* fault_item, void* stream);
int dpp_imgc_vqnearest(const float* blk, const float* cbk, int32_t* idx, int64_t items,
                       int64_t cbk_items, int codebook_size, void* stream);

/* Fused encoder: forward block transform + quantisation + ordering in one
 * kernel per tile (imgc.py:343-403 steps 1,2,5 and the quantisers, with the
 * codebook as input).
 *   px          batch images, each height x width pixels of `channels` u8
 *               (1 = gray meaning R=G=B, 3 = RGB, 4 = RGBA with A ignored),
 *               rows `row_stride` bytes apart, images `image_stride` apart.
 *   codebook    per image n_cb x 16 f32 (codebook_stride floats apart; 0 =
 *               one codebook shared by every image).
 *   sigma_min   deviation floor of the normalisation (imgc.py:345, 387; 0.25).
 *   records     per image 3 * blocks u8, interleaved (mean, sigma idx, index)
 *               in raster block order (imgc.py:295-305).
 *   cb_plane, cr_plane   per image (h/4) x (w/4) u8.
 *   block_grad  nullable; per image blocks f32 mean gradient magnitude
 *               (imgc.py:378-381), the k-means training filter.
 *   norm32      nullable; per image blocks x 16 normalised f32 blocks
 *               (imgc.py:396, the vq input).
 * Output strides per image: 3*blocks, blocks, blocks, blocks*16. */
int dpp_imgc_encode(const uint8_t* px, int channels, int64_t height, int64_t width,
                    int64_t row_stride, int64_t image_stride, int64_t batch,
                    const float* codebook, int n_cb, int64_t codebook_stride, double sigma_min,
                    uint8_t* records, uint8_t* cb_plane, uint8_t* cr_plane,
                    float* block_grad, float* norm32, void* stream);

/* Same encoder with the three record bytes written as planes (per block:
 * mu_plane[k], sig_plane[k], idx_plane[k]; strides per image = blocks), the
 * layout of the graph node's mu / sig / idx outputs, so a device-resident
 * edge needs no de-interleaving pass. */
int dpp_imgc_encode_planar(const uint8_t* px, int channels, int64_t height, int64_t width,
                           int64_t row_stride, int64_t image_stride, int64_t batch,
                           const float* codebook, int n_cb, int64_t codebook_stride, double sigma_min,
                           uint8_t* mu_plane, uint8_t* sig_plane, uint8_t* idx_plane,
                           uint8_t* cb_plane, uint8_t* cr_plane, void* stream);

/* The encoder's nearest-centroid search runs on the tensor cores (tcgen05
 * kind::tf32, 3xTF32 split) with an exact binary32 re-check of every
 * centroid inside the error band, so the output is identical to the
 * brute-force search (environment DPP_IMGC_VQ=exact selects the latter).
 * Test hook: the tensor-core encoder for one gray/RGB/RGBA image with the
 * pruning band scaled by delta_scale; *ambiguous (device counter) is
 * incremented by the number of blocks that needed the exact re-check. */
int dpp_imgc_encode_tc_debug(const uint8_t* px, int channels, int64_t height, int64_t width,
                             const float* codebook, int n_cb, uint8_t* records, uint8_t* cb_plane,
                             uint8_t* cr_plane, float delta_scale, unsigned long long* ambiguous,
                             void* stream);

/* Training pass of the codec (imgc.py:378-388): per block the mean gradient
 * magnitude (block_grad, the k-means training filter) and the binary64
 * normalised block (norm64, blocks x 16) — the k-means input. */
int dpp_imgc_block_stats(const uint8_t* px, int channels, int64_t height, int64_t width,
                         int64_t row_stride, int64_t image_stride, int64_t batch, double sigma_min,
                         double* norm64, float* block_grad, void* stream);

/* Parity report of the codec's two binary64 quantisers (imgc.py:398-401,
 * SURVEY §8(d) C4): adds to ties[0] the number of blocks whose mean, and to
 * ties[1] the number whose sigma / 0.25, lies within 1e-9 of a half-integer
 * (the values where rint() depends on the last bits).  Same statistics code
 * as the encoder; ties is a device array of two counters. */
int dpp_imgc_rounding_ties(const uint8_t* px, int channels, int64_t height, int64_t width,
                           int64_t row_stride, int64_t image_stride, int64_t batch,
                           unsigned long long* ties, void* stream);

/* k-means codebook trainer (imgc.py:221-273) on device: k-means++ seeding
 * from the caller's RNG stream (index of the first pick and a HOST array of
 * k-1 uniforms in [0,1), as numpy's Generator.choice consumes them), then
 * <= max_iter Lloyd iterations in binary64.  pts: n x 16 doubles (device);
 * centroids_out: k x 16 floats (device); trace: nullable host array of
 * max_iter per-iteration SSE values; *iterations = iterations run. */
int dpp_kmeans(const double* pts, int64_t n, int k, int64_t first_pick, const double* uniforms,
               int max_iter, float* centroids_out, double* trace, int* iterations, void* stream);

/* The same trainer over points sharded across ranks (one process per GPU,
 * SURVEY §8(f) row 2 multi-GPU): each rank wraps its contiguous slice of the
 * training blocks in a shard; the driver (kmeans.py, kmeans_sharded) does one
 * small all-reduce per k-means++ step and one per Lloyd iteration.
 *   seed:   d2 = min(d2, |p - centroid|^2) (first != 0: initialise);
 *           *total (host) = the shard's d2 sum in block order.
 *   pick:   the point whose inclusive d2 prefix first exceeds `target`
 *           (searchsorted 'right', imgc.py:245), or local_index when >= 0;
 *           copied to centroid_out (device, 16 doubles); *picked = its index.
 *   assign: nearest centroid (first minimum) per point; acc (device,
 *           k*16 + k + 2 doubles) = [coordinate sums][counts][changed][SSE].
 *   far:    *packed (device int64) = max over the shard of
 *           (f32 bits of the distance to the assigned centroid) << 32 |
 *           (0xffffffff - global index), base = the shard's first index.
 *   set_assign: the reseeded point joins `cluster`. */
typedef struct dpp_kmeans_shard dpp_kmeans_shard;
int dpp_kmeans_shard_create(dpp_kmeans_shard** shard, const double* pts, int64_t n, int k, void* stream);
int dpp_kmeans_shard_seed(dpp_kmeans_shard* shard, const double* centroid, int first, double* total);
int dpp_kmeans_shard_pick(dpp_kmeans_shard* shard, double target, int64_t local_index, double* centroid_out,
                          int64_t* picked);
int dpp_kmeans_shard_assign(dpp_kmeans_shard* shard, const double* cents, double* acc);
int dpp_kmeans_shard_far(dpp_kmeans_shard* shard, const double* cents, int64_t base, int64_t* packed);
int dpp_kmeans_shard_set_assign(dpp_kmeans_shard* shard, int64_t local_index, int cluster);
void dpp_kmeans_shard_destroy(dpp_kmeans_shard* shard);

/* C5 chain adapters (node bodies in apps/chain.py):
 *   to_complex:  y[i] = ((float)x[i], 0)          n u8 -> n complex64 (n % 4 == 0)
 *   spectrum_u8: y[i] = (u8)clamp(floor(alpha*log(1+|z[i]|)), 0, 255)   (n even) */
int dpp_u8_to_complex(const uint8_t* x, float* y, int64_t n, void* stream);
int dpp_spectrum_u8(const float* z, uint8_t* y, int64_t n, float alpha, void* stream);

/* Inverse (imgc.py:426-439), for round-trip tests on device. */
int dpp_imgc_decode(const uint8_t* records, const uint8_t* cb_plane, const uint8_t* cr_plane,
                    const float* codebook, int n_cb, int64_t height, int64_t width,
                    uint8_t* rgb, void* stream);

/* ------------------------------------------------------------------------
 * JIT of kernel-language node bodies
 * ------------------------------------------------------------------------ */

/* A node body with no hand-written implementation is translated to CUDA C
 * (paper_1203_4938_b200/kernel/codegen.py: the reference evaluator's
 * semantics, kernel/interp.py) and compiled here with NVRTC for sm_100a
 * (cubin, -fmad=false).  Replaces: engine.plan's compile_kernel + the
 * interpreter run_lanes (/root/reference/pkg/src/dpp/engine.py:82-135,
 * kernel/interp.py:471-485) for such nodes.  Compiling needs no GPU.
 *   log: nullable buffer for the NVRTC log (log_len bytes). */
typedef struct dpp_jit_kernel dpp_jit_kernel;
int dpp_jit_compile(const char* source, const char* name, dpp_jit_kernel** kernel, char* log,
                    size_t log_len);

/* Launch `items` work-items (256 threads per CTA) on `stream`.  params: the
 * generated kernel's 64-bit parameter block (point pointers, element
 * counts, items, global size, first work-item id, fault word, detail). */
int dpp_jit_launch(dpp_jit_kernel* kernel, const uint64_t* params, int nparams, int64_t items,
                   void* stream);
void dpp_jit_destroy(dpp_jit_kernel* kernel);

#ifdef __cplusplus
}
#endif

#endif /* DPP_B200_H */
