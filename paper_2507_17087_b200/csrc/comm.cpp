// NVLink peer-memory plumbing for the mapped executors.
//
// The executors move operand panels between GPUs with the copy engines
// (cudaMemcpy2DAsync on peer pointers over NVLink / NVSwitch), so transfers
// never compete with the tensor-core kernels for SMs.  Peer pointers come
// from CUDA IPC handles exchanged once through torch.distributed.

#include <cstring>

#include "pm_common.h"

extern "C" {

int pm_ipc_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return pm::set_error("pm_ipc_handle: null"), PM_ERR_INVALID;
  void* base = nullptr;
  size_t size = 0;
  // find the allocation that contains ptr (the caching allocator sub-allocates)
  CUdeviceptr b = 0;
  size_t sz = 0;
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return pm::set_error("cuMemGetAddressRange unavailable"), PM_ERR_CUDA;
    get_range = reinterpret_cast<GetRange>(p);
  }
  PM_CU_TRY(get_range(&b, &sz, (CUdeviceptr)ptr));
  base = (void*)b;
  size = sz;
  (void)size;
  cudaIpcMemHandle_t h;
  PM_CUDA_TRY(cudaIpcGetMemHandle(&h, base));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((const char*)ptr - (const char*)base);
  return PM_OK;
}

int pm_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return pm::set_error("pm_ipc_open: null"), PM_ERR_INVALID;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  PM_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return PM_OK;
}

int pm_ipc_close(void* base) {
  PM_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return PM_OK;
}

int pm_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                    int64_t height, void* stream) {
  if (width <= 0 || height <= 0) return PM_OK;
  PM_CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                                (size_t)height, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return PM_OK;
}

}  // extern "C"
