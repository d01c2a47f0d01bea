// Peer memory plumbing for the row-sharded 2-D FFT: CUDA IPC
// handles so every rank maps every other rank's row slab (NVLink loads and
// TMA stores straight into peer HBM, no staging copies, no NCCL on the data
// path), and a stream-ordered flag barrier between the row pass and the fused
// column/exchange pass (csrc/fft2d_l2.cu, PEER).
#include <cuda.h>

#include <cstring>

#include "common.cuh"

namespace dpp {
namespace {

struct PeerFlags {
  int* f[8];
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Rank `rank` stores epoch into slot `rank` of every rank's flag array, then
// waits until every rank has stored it into its own array.  System-scope
// release/acquire orders all earlier stream work (the row pass, or the fused
// pass's peer TMA stores) before the peers proceed.  A peer that never arrives
// traps the kernel after `timeout_ns` instead of hanging the GPU.
__global__ void peer_barrier_kernel(PeerFlags fl, int np, int rank, int epoch, uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  asm volatile("fence.sc.sys;" ::: "memory");
  for (int j = 0; j < np; ++j)
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(fl.f[j] + rank), "r"(epoch) : "memory");
  const uint64_t t0 = globaltimer();
  for (int j = 0; j < np; ++j) {
    for (;;) {
      int v;
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(fl.f[rank] + j) : "memory");
      if (v - epoch >= 0) break;
      if (globaltimer() - t0 > timeout_ns) asm volatile("trap;");
      __nanosleep(256);
    }
  }
}

CUresult (*g_addr_range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;

}  // namespace
}  // namespace dpp

extern "C" {

int dpp_ipc_get_handle(const void* ptr, void* handle, uint64_t* offset) {
  using namespace dpp;
  if (!ptr || !handle || !offset) return fail(DPP_EINVAL, "NULL argument to dpp_ipc_get_handle");
  if (!g_addr_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(DPP_ECUDA, "cuMemGetAddressRange entry point unavailable");
    g_addr_range = reinterpret_cast<decltype(g_addr_range)>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (g_addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(DPP_EINVAL, "pointer %p is not device memory", ptr);
  cudaIpcMemHandle_t h;
  DPP_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<CUdeviceptr>(ptr) - base;
  return DPP_OK;
}

int dpp_ipc_open(const void* handle, void** base) {
  using namespace dpp;
  if (!handle || !base) return fail(DPP_EINVAL, "NULL argument to dpp_ipc_open");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  DPP_CUDA_CHECK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return DPP_OK;
}

int dpp_ipc_close(void* base) {
  using namespace dpp;
  if (!base) return DPP_OK;
  DPP_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return DPP_OK;
}

int dpp_peer_barrier(int* const* flags, int nranks, int rank, int epoch, double timeout_s, void* stream) {
  using namespace dpp;
  if (!flags || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks)
    return fail(DPP_EINVAL, "bad dpp_peer_barrier arguments (%d ranks, rank %d)", nranks, rank);
  PeerFlags fl;
  std::memset(&fl, 0, sizeof(fl));
  for (int j = 0; j < nranks; ++j) {
    if (!flags[j]) return fail(DPP_EINVAL, "NULL flag array for rank %d", j);
    fl.f[j] = flags[j];
  }
  const uint64_t tmo = (uint64_t)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
  peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(fl, nranks, rank, epoch, tmo);
  DPP_LAUNCH_CHECK("peer_barrier");
  return DPP_OK;
}

}  // extern "C"
