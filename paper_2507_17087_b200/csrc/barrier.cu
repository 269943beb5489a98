// Stream-ordered barrier among the GPUs of a box through peer memory (NVLink),
// replacing a 4-byte NCCL all-reduce where an executor only needs ordering
// (Cannon / 2.5D shift rounds): every GPU pushes its barrier epoch into each
// peer's flag slot with a system-scope release store and spins until every peer
// has pushed the same epoch into its own flags (acquire).  The epoch lives in
// device memory and is advanced by the kernel itself, so the barrier can be
// captured in a CUDA graph and replayed.  Work stream-ordered before the
// barrier on one GPU happens-before work stream-ordered after it on every GPU.

#include <cuda_runtime.h>

#include "pm_common.h"

namespace pm {
namespace {

__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(int32_t* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(32) k_peer_barrier(const pm_peer_barrier_view v) {
  const int q = threadIdx.x;
  int e = 0;
  if (q == 0) {
    e = *v.epoch + 1;
    *v.epoch = e;
  }
  e = __shfl_sync(0xffffffffu, e, 0);
  if (q < v.world && q != v.rank) {
    __threadfence_system();
    st_release_sys(v.peer_slot[q], e);
    while (ld_acquire_sys(v.my_flags + q) < e) __nanosleep(64);
  }
  __syncwarp();
}

}  // namespace
}  // namespace pm

extern "C" int pm_peer_barrier(const pm_peer_barrier_view* v, void* stream) {
  if (!v || !v->my_flags || !v->epoch || v->world < 1 || v->world > PM_BARRIER_MAX_RANKS ||
      v->rank < 0 || v->rank >= v->world)
    return pm::set_error("pm_peer_barrier: bad view"), PM_ERR_INVALID;
  for (int q = 0; q < v->world; ++q)
    if (q != v->rank && !v->peer_slot[q])
      return pm::set_error("pm_peer_barrier: missing peer slot %d", q), PM_ERR_INVALID;
  if (v->world == 1) return PM_OK;
  pm::k_peer_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(*v);
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}
