#include "dyn.hpp"

#include <dlfcn.h>

#include <mutex>

#include "ir.hpp"

namespace sfx {

#define SFX_STR2(x) #x
#define SFX_STR(x) SFX_STR2(x)

namespace {

void* open_first(const char* const* names) {
  for (const char* const* n = names; *n; ++n)
    if (void* h = dlopen(*n, RTLD_NOW | RTLD_LOCAL)) return h;
  return nullptr;
}

}  // namespace

const Driver& driver() {
  static Driver d;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libcuda.so.1", "libcuda.so", nullptr};
    void* h = open_first(names);
    if (!h) {
      err = "CUDA driver (libcuda.so.1) not available: no GPU on this host";
      return;
    }
#define SFX_BIND(name)                                                        \
  d.name = reinterpret_cast<decltype(d.name)>(dlsym(h, SFX_STR(name)));       \
  if (!d.name) err = std::string("libcuda missing symbol ") + SFX_STR(name);
    SFX_BIND(cuInit)
    SFX_BIND(cuDeviceGet)
    SFX_BIND(cuDeviceGetAttribute)
    SFX_BIND(cuDevicePrimaryCtxRetain)
    SFX_BIND(cuCtxSetCurrent)
    SFX_BIND(cuCtxGetCurrent)
    SFX_BIND(cuMemAlloc)
    SFX_BIND(cuMemFree)
    SFX_BIND(cuMemHostAlloc)
    SFX_BIND(cuMemFreeHost)
    SFX_BIND(cuMemcpyHtoDAsync)
    SFX_BIND(cuMemcpyDtoHAsync)
    SFX_BIND(cuMemcpyDtoDAsync)
    SFX_BIND(cuMemsetD32Async)
    SFX_BIND(cuStreamSynchronize)
    SFX_BIND(cuStreamCreate)
    SFX_BIND(cuStreamDestroy)
    SFX_BIND(cuStreamWaitEvent)
    SFX_BIND(cuEventCreate)
    SFX_BIND(cuEventDestroy)
    SFX_BIND(cuEventRecord)
    SFX_BIND(cuEventSynchronize)
    SFX_BIND(cuEventElapsedTime)
    SFX_BIND(cuModuleLoadData)
    SFX_BIND(cuModuleUnload)
    SFX_BIND(cuModuleGetFunction)
    SFX_BIND(cuLaunchKernel)
    SFX_BIND(cuLaunchKernelEx)
    SFX_BIND(cuFuncGetAttribute)
    SFX_BIND(cuFuncSetAttribute)
    SFX_BIND(cuGetErrorName)
    SFX_BIND(cuStreamBeginCapture)
    SFX_BIND(cuStreamEndCapture)
    SFX_BIND(cuGraphInstantiateWithFlags)
    SFX_BIND(cuGraphLaunch)
    SFX_BIND(cuGraphExecDestroy)
    SFX_BIND(cuGraphDestroy)
    SFX_BIND(cuIpcGetMemHandle)
    SFX_BIND(cuIpcOpenMemHandle)
    SFX_BIND(cuIpcCloseMemHandle)
    SFX_BIND(cuMemcpyHtoD)
    SFX_BIND(cuStreamWriteValue32)
    SFX_BIND(cuStreamWaitValue32)
    SFX_BIND(cuStreamIsCapturing)
    SFX_BIND(cuMemcpyDtoH)
#undef SFX_BIND
    if (err.empty()) {
      CUresult r = d.cuInit(0);
      if (r != CUDA_SUCCESS) err = "cuInit failed (" + std::to_string(static_cast<int>(r)) + ")";
    }
  });
  if (!err.empty()) throw Error(SFX_ERR_CUDA, err);
  return d;
}

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    // the toolkit's NVRTC first (12.9, sm_100a SASS), by absolute path so a
    // different NVRTC already mapped into the process (e.g. torch's) is not reused
    const char* names[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so", nullptr};
    void* h = open_first(names);
    if (!h) {
      err = "NVRTC (libnvrtc.so.12) not available";
      return;
    }
#define SFX_BIND(name)                                                  \
  n.name = reinterpret_cast<decltype(n.name)>(dlsym(h, SFX_STR(name))); \
  if (!n.name) err = std::string("libnvrtc missing symbol ") + SFX_STR(name);
    SFX_BIND(nvrtcCreateProgram)
    SFX_BIND(nvrtcCompileProgram)
    SFX_BIND(nvrtcGetProgramLogSize)
    SFX_BIND(nvrtcGetProgramLog)
    SFX_BIND(nvrtcGetCUBINSize)
    SFX_BIND(nvrtcGetCUBIN)
    SFX_BIND(nvrtcDestroyProgram)
    SFX_BIND(nvrtcGetErrorString)
    SFX_BIND(nvrtcVersion)
#undef SFX_BIND
  });
  if (!err.empty()) throw Error(SFX_ERR_COMPILE, err);
  return n;
}

void check_cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* name = nullptr;
  const Driver& d = driver();
  if (d.cuGetErrorName) d.cuGetErrorName(r, &name);
  throw Error(SFX_ERR_CUDA, std::string(what) + " failed: " + (name ? name : std::to_string(static_cast<int>(r))));
}

std::string library_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&library_dir), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash);
  }
  return ".";
}

}  // namespace sfx
