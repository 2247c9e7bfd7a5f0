// Lazily-bound CUDA driver, NVRTC and NCCL entry points.  libsfx.so has no
// link-time dependency on libcuda/libnvrtc/libnccl so that it loads (and its
// symbols can be checked, and kernels can be generated and compiled to sm_100a
// cubins) on a machine without a GPU driver.
#pragma once

#include <cuda.h>
#include <nvrtc.h>

#include <string>

namespace sfx {

struct Driver {
#define SFX_DRV(name) decltype(&::name) name = nullptr;
  SFX_DRV(cuInit)
  SFX_DRV(cuDeviceGet)
  SFX_DRV(cuDeviceGetAttribute)
  SFX_DRV(cuDevicePrimaryCtxRetain)
  SFX_DRV(cuCtxSetCurrent)
  SFX_DRV(cuCtxGetCurrent)
  SFX_DRV(cuMemAlloc)
  SFX_DRV(cuMemFree)
  SFX_DRV(cuMemHostAlloc)
  SFX_DRV(cuMemFreeHost)
  SFX_DRV(cuMemcpyHtoDAsync)
  SFX_DRV(cuMemcpyDtoHAsync)
  SFX_DRV(cuMemcpyDtoDAsync)
  SFX_DRV(cuMemsetD32Async)
  SFX_DRV(cuStreamSynchronize)
  SFX_DRV(cuStreamCreate)
  SFX_DRV(cuStreamDestroy)
  SFX_DRV(cuStreamWaitEvent)
  SFX_DRV(cuEventCreate)
  SFX_DRV(cuEventDestroy)
  SFX_DRV(cuEventRecord)
  SFX_DRV(cuEventSynchronize)
  SFX_DRV(cuEventElapsedTime)
  SFX_DRV(cuModuleLoadData)
  SFX_DRV(cuModuleUnload)
  SFX_DRV(cuModuleGetFunction)
  SFX_DRV(cuLaunchKernel)
  SFX_DRV(cuLaunchKernelEx)
  SFX_DRV(cuFuncGetAttribute)
  SFX_DRV(cuFuncSetAttribute)
  SFX_DRV(cuGetErrorName)
  SFX_DRV(cuStreamBeginCapture)
  SFX_DRV(cuStreamEndCapture)
  SFX_DRV(cuGraphInstantiateWithFlags)
  SFX_DRV(cuGraphLaunch)
  SFX_DRV(cuGraphExecDestroy)
  SFX_DRV(cuGraphDestroy)
  SFX_DRV(cuIpcGetMemHandle)
  SFX_DRV(cuIpcOpenMemHandle)
  SFX_DRV(cuIpcCloseMemHandle)
  SFX_DRV(cuMemcpyHtoD)
  SFX_DRV(cuStreamWriteValue32)
  SFX_DRV(cuStreamWaitValue32)
  SFX_DRV(cuStreamIsCapturing)
  SFX_DRV(cuMemcpyDtoH)
#undef SFX_DRV
};

struct Nvrtc {
#define SFX_RTC(name) decltype(&::name) name = nullptr;
  SFX_RTC(nvrtcCreateProgram)
  SFX_RTC(nvrtcCompileProgram)
  SFX_RTC(nvrtcGetProgramLogSize)
  SFX_RTC(nvrtcGetProgramLog)
  SFX_RTC(nvrtcGetCUBINSize)
  SFX_RTC(nvrtcGetCUBIN)
  SFX_RTC(nvrtcDestroyProgram)
  SFX_RTC(nvrtcGetErrorString)
  SFX_RTC(nvrtcVersion)
#undef SFX_RTC
};

const Driver& driver();  // throws sfx::Error(SFX_ERR_CUDA) if libcuda is unavailable
const Nvrtc& nvrtc();    // throws sfx::Error(SFX_ERR_COMPILE) if libnvrtc is unavailable
void check_cu(CUresult r, const char* what);

// Directory holding libsfx.so (for the in-tree kernel cache).
std::string library_dir();

}  // namespace sfx
