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

// Copies then a barrier, in one launch (the Cannon / 2.5D shift rounds): every CTA
// copies its share of the blocks with 16-byte loads / stores (peer or local memory),
// fences and takes a ticket; the last CTA resets the ticket and runs the barrier.
// Replaces copy-engine pulls + a separate barrier kernel where the blocks are small
// and the round is latency-bound (configs[0]: 1 MiB blocks on a 2x2 grid).
struct CopySet {
  pm_peer_copy c[PM_PEER_COPY_MAX];
  int n;
};

__global__ void __launch_bounds__(256) k_peer_copy_barrier(const pm_peer_barrier_view v,
                                                           const CopySet cs,
                                                           unsigned* __restrict__ ticket) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (int k = 0; k < cs.n; ++k) {
    const int4* __restrict__ src = reinterpret_cast<const int4*>(cs.c[k].src);
    int4* __restrict__ dst = reinterpret_cast<int4*>(cs.c[k].dst);
    const long long words = cs.c[k].bytes / 16;
    for (long long w = gt; w < words; w += gs) dst[w] = __ldcg(src + w);
  }
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) *ticket = 0u;
  if (threadIdx.x >= 32 || v.world <= 1) return;
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

extern "C" int pm_peer_copy_barrier(const pm_peer_barrier_view* v, const pm_peer_copy* copies,
                                    int32_t n, uint32_t* ticket, void* stream) {
  if (!v || !v->epoch || !ticket || n < 0 || n > PM_PEER_COPY_MAX || (n > 0 && !copies) ||
      v->world < 1 || v->world > PM_BARRIER_MAX_RANKS || v->rank < 0 || v->rank >= v->world)
    return pm::set_error("pm_peer_copy_barrier: bad arguments"), PM_ERR_INVALID;
  if (v->world > 1) {  // the same view checks as pm_peer_barrier
    if (!v->my_flags) return pm::set_error("pm_peer_copy_barrier: bad view"), PM_ERR_INVALID;
    for (int q = 0; q < v->world; ++q)
      if (q != v->rank && !v->peer_slot[q])
        return pm::set_error("pm_peer_copy_barrier: missing peer slot %d", q), PM_ERR_INVALID;
  }
  pm::CopySet cs{};
  long long words = 0;
  for (int k = 0; k < n; ++k) {
    const pm_peer_copy& c = copies[k];
    if (c.bytes < 0 || c.bytes % 16 || (((uintptr_t)c.dst | (uintptr_t)c.src) & 15) ||
        (c.bytes && (!c.dst || !c.src)))
      return pm::set_error("pm_peer_copy_barrier: copies must be 16-byte aligned multiples"),
             PM_ERR_INVALID;
    cs.c[k] = c;
    words += c.bytes / 16;
  }
  cs.n = n;
  long long blocks = (words + 256 * 4 - 1) / (256 * 4);
  const long long cap = (long long)pm::num_sms();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  pm::k_peer_copy_barrier<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(*v, cs, ticket);
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

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
