// K2 -- stable ownership partition of mapped points.
//
// Reference semantics: expand_shards / shard_policy (tasksim/sim.py:67-120)
// split an index launch into one leaf per distinct processor, each leaf
// keeping its points in launch order; proc_counts (cli.py:154-164) counts
// them.  On the GPU that is a stable counting sort of point indices by
// processor id (stable_partition.cuh).  Traffic: the 4 B/pt processor id is
// read by the histogram and by the scatter, the 4 B/pt index written once.

#include <cuda_runtime.h>

#include <cstdint>

#include "pm_common.h"
#include "stable_partition.cuh"

namespace pm {
namespace {

struct ProcKey {
  const int* __restrict__ proc;
  int nbins;
  unsigned long long* bad;
  bool vec_ok;  // proc is 16-byte aligned: keys4() may use vector loads
  static constexpr bool kVec4 = true;
  static constexpr bool kPeek = false;
  __device__ __forceinline__ void uniform(long long, int, int) const {}
  __device__ __forceinline__ int check(int b, long long i) const {
    if (b < 0 || b >= nbins) {
      atomicMin(bad, (unsigned long long)i);
      return -1;
    }
    return b;
  }
  __device__ __forceinline__ int operator()(long long i) const { return check(__ldg(proc + i), i); }
  // L2 prefetch of the 128-byte line holding item i (the histogram pass prefetches the
  // tile a CTA that starts about one CTA lifetime later will read)
  __device__ __forceinline__ void prefetch(long long i, long long n) const {
    if (i < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(proc + i));
  }
  // four consecutive ids (i % 4 == 0) packed as int8 bins
  static constexpr bool kRaw4 = true;
  __device__ __forceinline__ int4 raw4(long long i) const {
    return __ldg(reinterpret_cast<const int4*>(proc + i));
  }
  __device__ __forceinline__ int pack4(int4 v, long long i) const {
    return (check(v.x, i) & 0xFF) | ((check(v.y, i + 1) & 0xFF) << 8) |
           ((check(v.z, i + 2) & 0xFF) << 16) | ((check(v.w, i + 3) & 0xFF) << 24);
  }
  __device__ __forceinline__ int keys4(long long i) const { return pack4(raw4(i), i); }
};

struct PermSink {
  int* __restrict__ perm;
  __device__ __forceinline__ void put(int, long long pos, long long i) const { perm[pos] = (int)i; }
  __device__ __forceinline__ void put_run(int, long long pos, long long i, int count) const {
    pmdev::store_iota(perm + pos, (int)i, count);
  }
};

// `bad` is an unsigned atomicMin target that starts at UINT64_MAX; report
// "no bad id" as -1 (same bit pattern) -- nothing to do.
}  // namespace
}  // namespace pm

extern "C" {

size_t pm_partition_scratch_bytes(int64_t n, int32_t nbins) {
  return pm::part_scratch_bytes(n, nbins);
}

int pm_partition(const int32_t* proc, int64_t n, int32_t nbins, int64_t* counts,
                 int64_t* offsets, int32_t* perm, int64_t* bad, void* scratch,
                 size_t scratch_bytes, void* stream) {
  if (n < 0 || !counts || !offsets || !bad || (n > 0 && !proc))
    return pm::set_error("pm_partition: bad arguments"), PM_ERR_INVALID;
  if (n >= (1LL << 31))
    return pm::set_error("pm_partition: int32 permutation needs n < 2^31"), PM_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  PM_CUDA_TRY(cudaMemsetAsync(bad, 0xFF, sizeof(int64_t), s));
  pm::ProcKey key{proc, nbins, reinterpret_cast<unsigned long long*>(bad),
                  ((uintptr_t)proc % 16) == 0};
  pm::PermSink sink{perm};
  return pm::stable_partition(key, sink, perm != nullptr, n, nbins,
                              reinterpret_cast<long long*>(counts),
                              reinterpret_cast<long long*>(offsets), scratch, scratch_bytes, s);
}

}  // extern "C"
