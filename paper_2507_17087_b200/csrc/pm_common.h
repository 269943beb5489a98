// Shared plumbing of libmapple_b200: error reporting and lazily resolved
// CUDA driver entry points (resolved through the runtime, so the library
// loads on machines without libcuda -- the CPU build/test container).
#pragma once

// tiles per CTA of the partition scatter (partition_device.cuh keeps the same default for
// NVRTC, and mapping.cpp passes this value to every NVRTC compile)
#ifndef PM_SCATTER_TILES
#define PM_SCATTER_TILES 2
#endif

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/mapple_b200.h"

namespace pm {

void set_error(const char* fmt, ...);

#define PM_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::pm::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                      __FILE__, __LINE__);                                       \
      return PM_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define PM_CU_TRY(expr)                                                          \
  do {                                                                           \
    CUresult _r = (expr);                                                        \
    if (_r != CUDA_SUCCESS) {                                                    \
      ::pm::set_error("%s failed: CUresult %d (%s:%d)", #expr, (int)_r,          \
                      __FILE__, __LINE__);                                       \
      return PM_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

struct Driver {
  decltype(&cuModuleLoadData) moduleLoadData = nullptr;
  decltype(&cuModuleUnload) moduleUnload = nullptr;
  decltype(&cuModuleGetFunction) moduleGetFunction = nullptr;
  decltype(&cuLaunchKernel) launchKernel = nullptr;
  decltype(&cuFuncSetAttribute) funcSetAttribute = nullptr;
  decltype(&cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
  decltype(&cuCtxGetCurrent) ctxGetCurrent = nullptr;
  bool ok = false;
};

// Resolve once; returns nullptr (with pm_last_error set) when no driver.
const Driver* driver();

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

int num_sms();

}  // namespace pm
