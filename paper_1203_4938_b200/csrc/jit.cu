// JIT for kernel-language node bodies: CUDA C generated
// by paper_1203_4938_b200/kernel/codegen.py is compiled here with NVRTC for
// sm_100a (cubin, no FMA contraction) and launched through the driver API.
//
// NVRTC is loaded with dlopen (no link-time dependency): compiling needs no
// GPU, so the CPU test suite can check every generated kernel compiles; the
// module is loaded into the current context on first launch.
#include <cuda.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace dpp {
namespace {

typedef int nvrtcResult_;
typedef struct _nvrtcProgram* nvrtcProgram_;
struct Nvrtc {
  nvrtcResult_ (*create)(nvrtcProgram_*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_ (*compile)(nvrtcProgram_, int, const char* const*);
  nvrtcResult_ (*log_size)(nvrtcProgram_, size_t*);
  nvrtcResult_ (*log)(nvrtcProgram_, char*);
  nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t*);
  nvrtcResult_ (*cubin)(nvrtcProgram_, char*);
  nvrtcResult_ (*destroy)(nvrtcProgram_*);
  bool ok = false;
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                           "/usr/local/cuda/lib64/libnvrtc.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
    n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
    n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
    n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
  });
  return n;
}

// driver API through the runtime's entry-point query (no link-time libcuda:
// the library must load on machines without a GPU driver)
struct Drv {
  CUresult (*ctx_current)(CUcontext*) = nullptr;
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*get_fn)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  CUresult (*unload)(CUmodule) = nullptr;
  CUresult (*err)(CUresult, const char**) = nullptr;
  bool ok = false;
};

Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* sym, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(sym, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    d.ok = get("cuCtxGetCurrent", (void**)&d.ctx_current) && get("cuModuleLoadData", (void**)&d.load) &&
           get("cuModuleGetFunction", (void**)&d.get_fn) && get("cuLaunchKernel", (void**)&d.launch) &&
           get("cuModuleUnload", (void**)&d.unload) && get("cuGetErrorString", (void**)&d.err);
  });
  return d;
}

}  // namespace
}  // namespace dpp

struct dpp_jit_kernel {
  std::string name;
  std::vector<char> cubin;
  std::mutex mu;
  std::vector<std::pair<CUcontext, CUfunction>> fns;  // per context
  std::vector<CUmodule> mods;
};

extern "C" {

int dpp_jit_compile(const char* source, const char* name, dpp_jit_kernel** kernel, char* log, size_t log_len) {
  using namespace dpp;
  if (!source || !name || !kernel) return fail(DPP_EINVAL, "NULL argument to dpp_jit_compile");
  Nvrtc& nv = nvrtc();
  if (!nv.ok) return fail(DPP_ENOTSUP, "NVRTC (libnvrtc.so.12) is not available");
  nvrtcProgram_ prog = nullptr;
  if (nv.create(&prog, source, "dpp_node.cu", 0, nullptr, nullptr) != 0)
    return fail(DPP_ECUDA, "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17", "-lineinfo"};
  const int rc = nv.compile(prog, 4, opts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  std::string lg(ls, '\0');
  if (ls) nv.log(prog, &lg[0]);
  if (log && log_len) {
    std::strncpy(log, lg.c_str(), log_len - 1);
    log[log_len - 1] = 0;
  }
  if (rc != 0) {
    nv.destroy(&prog);
    return fail(DPP_EINVAL, "NVRTC compile of %s failed: %.800s", name, lg.c_str());
  }
  size_t cs = 0;
  nv.cubin_size(prog, &cs);
  auto* k = new dpp_jit_kernel();
  k->name = name;
  k->cubin.resize(cs);
  nv.cubin(prog, k->cubin.data());
  nv.destroy(&prog);
  *kernel = k;
  return DPP_OK;
}

int dpp_jit_launch(dpp_jit_kernel* kernel, const uint64_t* params, int nparams, int64_t items, void* stream) {
  using namespace dpp;
  if (!kernel || !params || nparams <= 0) return fail(DPP_EINVAL, "bad dpp_jit_launch arguments");
  if (items <= 0) return DPP_OK;
  cudaFree(nullptr);  // make the runtime's primary context current on this thread
  Drv& d = drv();
  if (!d.ok) return fail(DPP_ECUDA, "CUDA driver entry points unavailable");
  CUcontext ctx = nullptr;
  if (d.ctx_current(&ctx) != CUDA_SUCCESS || !ctx) return fail(DPP_ECUDA, "no current CUDA context");
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> g(kernel->mu);
    for (auto& e : kernel->fns)
      if (e.first == ctx) fn = e.second;
    if (!fn) {
      CUmodule mod = nullptr;
      if (d.load(&mod, kernel->cubin.data()) != CUDA_SUCCESS)
        return fail(DPP_ECUDA, "cuModuleLoadData failed for %s", kernel->name.c_str());
      if (d.get_fn(&fn, mod, kernel->name.c_str()) != CUDA_SUCCESS)
        return fail(DPP_ECUDA, "cuModuleGetFunction(%s) failed", kernel->name.c_str());
      kernel->mods.push_back(mod);
      kernel->fns.emplace_back(ctx, fn);
    }
  }
  const unsigned grid = (unsigned)((items + 255) / 256);
  void* args[] = {const_cast<uint64_t*>(params)};
  const CUresult r = d.launch(fn, grid, 1, 1, 256, 1, 1, 0, (CUstream)stream, args, nullptr);
  if (r != CUDA_SUCCESS) {
    const char* msg = nullptr;
    d.err(r, &msg);
    return fail(DPP_ECUDA, "cuLaunchKernel(%s): %s", kernel->name.c_str(), msg ? msg : "?");
  }
  return DPP_OK;
}

void dpp_jit_destroy(dpp_jit_kernel* kernel) {
  if (!kernel) return;
  if (!kernel->mods.empty() && dpp::drv().ok)
    for (CUmodule m : kernel->mods) dpp::drv().unload(m);
  delete kernel;
}

}  // extern "C"
