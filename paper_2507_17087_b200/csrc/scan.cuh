// Device-wide exclusive scan of int64 (in place), used by K2 and K3.
// Reduce-then-scan over 2048-element blocks, recursing on the block sums.
#pragma once

#include <cuda_runtime.h>

#include "pm_common.h"

namespace pm {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr long long kScanBlock = kScanThreads * kScanItems;

inline size_t scan_scratch_bytes(long long len) {
  size_t bytes = 64;  // grand total + padding
  while (len > kScanBlock) {
    len = (len + kScanBlock - 1) / kScanBlock;
    bytes += (size_t)len * 8 + 64;
  }
  return bytes;
}

__device__ __forceinline__ long long warp_incl_scan(long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    long long u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

// Exclusive scan of this thread's value across the block; *total = block sum.
__device__ __forceinline__ long long block_excl_scan(long long v, long long* total) {
  __shared__ long long warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long incl = warp_incl_scan(v);
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    long long s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < kScanThreads / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  long long base = warp ? warp_sums[warp - 1] : 0;
  *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();
  return base + incl - v;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const long long* __restrict__ x, long long len, long long* __restrict__ sums) {
  const long long base = blockIdx.x * kScanBlock + (long long)threadIdx.x * kScanItems;
  long long s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    if (base + j < len) s += x[base + j];
  long long total;
  block_excl_scan(s, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_apply(long long* __restrict__ x, long long len, const long long* __restrict__ offs,
             long long* __restrict__ grand_total) {
  const long long base = blockIdx.x * kScanBlock + (long long)threadIdx.x * kScanItems;
  long long v[kScanItems];
  long long s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = (base + j < len) ? x[base + j] : 0;
    s += v[j];
  }
  long long total;
  long long run = block_excl_scan(s, &total) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (base + j < len) x[base + j] = run;
    run += v[j];
  }
  if (grand_total && threadIdx.x == 0) *grand_total = total;
}

// Apply pass that finds its own block offset: the sum of the block sums before it
// (read straight from L2 -- at most kScanLookback of them), so a scan of up to
// kScanBlock * kScanLookback elements is two launches with no recursion; the last
// block writes the grand total.
constexpr long long kScanLookback = 4096;

__global__ void __launch_bounds__(kScanThreads)
k_scan_apply_lb(long long* __restrict__ x, long long len, const long long* __restrict__ sums,
                long long* __restrict__ grand_total) {
  __shared__ long long s_off;
  long long pre = 0;
  for (long long b = threadIdx.x; b < blockIdx.x; b += kScanThreads) pre += __ldg(sums + b);
  long long dummy;
  pre = block_excl_scan(pre, &dummy);  // the block-wide sum lands in dummy
  if (threadIdx.x == 0) s_off = dummy;
  __syncthreads();
  const long long off = s_off;
  const long long base = blockIdx.x * kScanBlock + (long long)threadIdx.x * kScanItems;
  long long v[kScanItems];
  long long sm = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = (base + j < len) ? x[base + j] : 0;
    sm += v[j];
  }
  long long total;
  long long run = block_excl_scan(sm, &total) + off;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (base + j < len) x[base + j] = run;
    run += v[j];
  }
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) *grand_total = off + total;
}

// In-place exclusive scan; the grand total lands in *(long long*)scratch.
inline int exclusive_scan_i64(long long* x, long long len, void* scratch, cudaStream_t s) {
  long long* total = reinterpret_cast<long long*>(scratch);
  char* cur = reinterpret_cast<char*>(scratch) + 64;
  if (len <= 0) {
    PM_CUDA_TRY(cudaMemsetAsync(total, 0, 8, s));
    return PM_OK;
  }
  if (len <= kScanBlock) {
    k_scan_apply<<<1, kScanThreads, 0, s>>>(x, len, nullptr, total);
    PM_CUDA_TRY(cudaGetLastError());
    return PM_OK;
  }
  const long long nblk = (len + kScanBlock - 1) / kScanBlock;
  long long* sums = reinterpret_cast<long long*>(cur);
  cur += nblk * 8 + 64;
  k_scan_reduce<<<(unsigned)nblk, kScanThreads, 0, s>>>(x, len, sums);
  PM_CUDA_TRY(cudaGetLastError());
  if (nblk <= kScanLookback) {
    k_scan_apply_lb<<<(unsigned)nblk, kScanThreads, 0, s>>>(x, len, sums, total);
    PM_CUDA_TRY(cudaGetLastError());
    return PM_OK;
  }
  // recurse: scan the block sums, total goes to the same grand-total slot
  {
    // the recursive call needs its own total slot followed by its levels; we
    // reuse `total` by laying the deeper levels after `sums`
    long long* deeper_total = total;
    char* deeper = cur - 64;  // recursion writes its total at deeper, levels after
    int rc = exclusive_scan_i64(sums, nblk, deeper, s);
    if (rc) return rc;
    PM_CUDA_TRY(cudaMemcpyAsync(deeper_total, deeper, 8, cudaMemcpyDeviceToDevice, s));
  }
  k_scan_apply<<<(unsigned)nblk, kScanThreads, 0, s>>>(x, len, sums, nullptr);
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

}  // namespace
}  // namespace pm
