// Generic stable counting partition used by K2 (points by processor) and K3
// (halo transfer entries by (src, dst) pair).
//
// Items are indexed 0..n-1; `Key::operator()(i)` returns the bin of item i or
// -1 (no output).  `Sink::put(bin, pos, i)` writes item i at output position
// pos (see partition_device.cuh for the full Key / Sink concepts).
//
//   k_part_hist     one CTA per tile: warp-aggregated (match.any) shared
//                   atomics; hist written bin-major hist[b * ntiles + t]
//   exclusive scan  of hist -> first output slot of every (bin, tile)
//   k_part_scatter  per tile, 256 items per round; lanes grouped by bin with
//                   match.any, rank = popc(peers below), per-warp counts
//                   (round-tagged) in shared memory give the prefix across
//                   warps; a running per-bin count carries across rounds.
//                   Output order inside a bin = item order (stable).
#pragma once

#include <cuda_runtime.h>

#include "partition_device.cuh"
#include "pm_common.h"
#include "scan.cuh"

namespace pm {
namespace {

using pmdev::kPartThreads;
using pmdev::kPartWarps;

inline int part_tile(int nbins) {
  int m = (nbins + 255) / 256;
  return 2048 * (m < 1 ? 1 : m);
}

inline size_t small_scratch_bytes(long long n, int nbins);

inline size_t part_scratch_bytes(long long n, int nbins) {
  if (n <= 0 || nbins <= 0) return 256;
  const long long tile = part_tile(nbins);
  const long long ntiles = (n + tile - 1) / tile;
  const long long len = ntiles * nbins;
  const size_t big = (size_t)(len * 8) + scan_scratch_bytes(len) + 256;
  const size_t small = small_scratch_bytes(n, nbins);
  return big > small ? big : small;
}

template <class Key>
__global__ void __launch_bounds__(kPartThreads)
k_part_hist(Key key, long long n, int nbins, int tile, long long ntiles,
            long long* __restrict__ hist) {
  extern __shared__ int h[];
  for (int b = threadIdx.x; b < nbins; b += kPartThreads) h[b] = 0;
  __syncthreads();
  const long long start = (long long)blockIdx.x * tile;
  const int lane = threadIdx.x & 31;
  for (int off = threadIdx.x; off < tile; off += kPartThreads) {
    const long long i = start + off;
    const int b = i < n ? key(i) : -1;
    if (__any_sync(0xffffffffu, b >= 0)) {
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      if (b >= 0 && lane == __ffs(peers) - 1) atomicAdd(&h[b], __popc(peers));
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += kPartThreads)
    hist[(long long)b * ntiles + blockIdx.x] = h[b];
}

template <class Key, class Sink>
__global__ void __launch_bounds__(kPartThreads)
k_part_scatter(Key key, Sink sink, long long n, int nbins, int tile, long long ntiles,
               const long long* __restrict__ pos0) {
  extern __shared__ int sm[];
  int* run = sm;         // [nbins]
  int* wc = sm + nbins;  // [kPartWarps][nbins], (round << 16) | count
  for (int b = threadIdx.x; b < nbins; b += kPartThreads) run[b] = 0;
  for (int b = threadIdx.x; b < kPartWarps * nbins; b += kPartThreads) wc[b] = -1;
  __syncthreads();
  const long long t = blockIdx.x;
  const long long start = t * tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const int rounds = tile / kPartThreads;
  for (int r = 0; r < rounds; ++r) {
    const long long i = start + (long long)r * kPartThreads + threadIdx.x;
    const int b = i < n ? key(i) : -1;
    const bool any = __any_sync(0xffffffffu, b >= 0);
    int rank = 0, cnt = 0;
    if (any) {
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      rank = __popc(peers & below);
      cnt = __popc(peers);
      if (b >= 0 && rank == 0) wc[warp * nbins + b] = (r << 16) | cnt;
    }
    __syncthreads();
    if (b >= 0) {
      int pre = 0;
      for (int w = 0; w < warp; ++w) {
        const int v = wc[w * nbins + b];
        if ((v >> 16) == r) pre += v & 0xFFFF;
      }
      sink.put(b, pos0[(long long)b * ntiles + t] + run[b] + pre + rank, i);
    }
    __syncthreads();
    if (b >= 0 && rank == 0) atomicAdd(&run[b], cnt);
  }
}

__global__ void k_part_bin_totals(const long long* __restrict__ scanned, long long ntiles,
                                  int nbins, const long long* __restrict__ total,
                                  long long* __restrict__ counts, long long* __restrict__ offsets) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  const long long lo = scanned[(long long)b * ntiles];
  const long long hi = (b + 1 < nbins) ? scanned[(long long)(b + 1) * ntiles] : *total;
  counts[b] = hi - lo;
  offsets[b] = lo;
}

// ---- fast path for up to kSmallBins bins: chunked, atomic-free -------------------
// (device bodies in partition_device.cuh, shared with the NVRTC fused kernels)
using pmdev::kIPT;
using pmdev::kSmallBins;
using pmdev::kSmallTile;

// scratch: hist[nbins][ntiles] int64 | tile_info[ntiles] int32 (256-aligned) | scan temp
inline size_t small_info_bytes(long long ntiles) {
  return (size_t)((ntiles * 4 + 255) / 256 * 256);
}
inline size_t small_scan_offset(long long ntiles, int nbins) {
  return (size_t)(ntiles * nbins * 8) + small_info_bytes(ntiles);
}
inline size_t small_scratch_bytes(long long n, int nbins) {
  const long long ntiles = (n + kSmallTile - 1) / kSmallTile;
  const long long len = ntiles * nbins;
  return small_scan_offset(ntiles, nbins) + scan_scratch_bytes(len) + 256;
}

// (2 or 4 tiles per CTA measured no faster: 1.39 / 1.39 vs 1.38 ms, tools/k2_hist_ab.sh)
template <class Key>
__global__ void __launch_bounds__(kPartThreads)
k_small_hist(Key key, long long n, int nbins, long long ntiles, long long* __restrict__ hist) {
  extern __shared__ __align__(16) int smem_words[];
  pmdev::small_hist_body(key, n, nbins, ntiles, hist, smem_words, (long long)blockIdx.x);
}

// Histogram pass for keys whose ids are a plain int32 array (Key::kRaw4): one WARP per
// 4096-id tile, so no CTA-wide barrier ever holds a load back -- each lane keeps
// kHistBatch 16-byte loads in flight, run-length counts them into its warp's shared
// histogram, and the warp writes the tile's histogram column and summary itself.
#ifndef PM_HIST_BATCH
#define PM_HIST_BATCH 8
#endif
constexpr int kHistBatch = PM_HIST_BATCH;

template <class Key>
__global__ void __launch_bounds__(kPartThreads)
k_small_hist_warp(Key key, long long n, int nbins, long long ntiles,
                  long long* __restrict__ hist) {
  extern __shared__ __align__(16) int smem_words[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long tile = (long long)blockIdx.x * kPartWarps + warp;
  if (tile >= ntiles) return;  // whole warps only: nothing below synchronises the CTA
  int* hw = smem_words + warp * nbins;
  for (int b = lane; b < nbins; b += 32) hw[b] = 0;
  __syncwarp();
  const long long base = tile * kSmallTile;
  int run_bin = -1, run = 0;
  auto add = [&](int b) {
    if (b != run_bin) {
      if (run_bin >= 0) atomicAdd(hw + run_bin, run);
      run_bin = b;
      run = 0;
    }
    ++run;
  };
  if (base + kSmallTile <= n && key.vec_ok) {
    // lane l reads ids base + 4 (32 k + l) .. + 3, k = 0 .. 31
#pragma unroll 1
    for (int k0 = 0; k0 < kSmallTile / 128; k0 += kHistBatch) {
      int4 raw[kHistBatch];
#pragma unroll
      for (int u = 0; u < kHistBatch; ++u)
        raw[u] = key.raw4(base + 4 * (32LL * (k0 + u) + lane));
#pragma unroll
      for (int u = 0; u < kHistBatch; ++u) {
        const int packed = key.pack4(raw[u], base + 4 * (32LL * (k0 + u) + lane));
#pragma unroll
        for (int q = 0; q < 4; ++q) add((int)(signed char)(packed >> (8 * q)));
      }
    }
  } else {
    for (int k = lane; k < kSmallTile; k += 32) {
      const long long i = base + k;
      add(i < n ? key(i) : -1);
    }
  }
  if (run_bin >= 0) atomicAdd(hw + run_bin, run);
  __syncwarp();
  int only = -1;
  bool any = false;
  for (int b0 = 0; b0 < nbins; b0 += 32) {
    const int b = b0 + lane;
    const int v = b < nbins ? hw[b] : 0;
    if (b < nbins) hist[(long long)b * ntiles + tile] = v;
    const unsigned full = __ballot_sync(0xffffffffu, v == kSmallTile);
    any |= __ballot_sync(0xffffffffu, v != 0) != 0;
    if (full) only = b0 + __ffs(full) - 1;
  }
  if (lane == 0) {
    // the last (possibly partial) tile always takes the general path
    const int info = tile + 1 == ntiles ? pmdev::kTileMixed
                     : only >= 0        ? only
                     : any              ? pmdev::kTileMixed
                                        : pmdev::kTileEmpty;
    const_cast<int*>(pmdev::tile_info_of(hist, nbins, ntiles))[tile] = info;
  }
}

// (min 6 CTAs / SM: the uniform-tile copy is a pure store stream, occupancy-bound)
// kScatterTiles tiles per CTA (partition_device.cuh small_scatter_tiles)
template <class Key, class Sink>
__global__ void __launch_bounds__(kPartThreads, 6)
k_small_scatter(Key key, Sink sink, long long n, int nbins, long long ntiles,
                const long long* __restrict__ pos0) {
  extern __shared__ __align__(16) int smem_words[];
  pmdev::small_scatter_tiles<pmdev::kScatterTiles>(key, sink, n, nbins, ntiles, pos0, smem_words,
                                                   (long long)blockIdx.x * pmdev::kScatterTiles);
}
inline unsigned small_scatter_grid(long long ntiles) {
  return (unsigned)((ntiles + pmdev::kScatterTiles - 1) / pmdev::kScatterTiles);
}

inline size_t small_hist_smem(int nbins) {
  return sizeof(int) * (size_t)nbins * kPartWarps;
}
inline size_t small_scatter_smem(int nbins) {
  return sizeof(int) * ((size_t)nbins * kPartThreads + kSmallBins + 1) + 2 * kSmallTile +
         kSmallTile;
}

// counts/offsets always; the scatter only when `scatter` is true.
template <class Key, class Sink>
int stable_partition_small(Key key, Sink sink, bool scatter, long long n, int nbins,
                           long long* counts, long long* offsets, void* scratch,
                           size_t scratch_bytes, cudaStream_t s) {
  if (scratch_bytes < small_scratch_bytes(n, nbins))
    return set_error("partition: scratch too small"), PM_ERR_INVALID;
  const long long ntiles = (n + kSmallTile - 1) / kSmallTile;
  if (ntiles > 0x7FFFFFFFLL) return set_error("partition: too many tiles"), PM_ERR_UNSUPPORTED;
  const long long len = ntiles * nbins;
  long long* hist = reinterpret_cast<long long*>(scratch);
  void* scan_tmp = reinterpret_cast<char*>(scratch) + small_scan_offset(ntiles, nbins);
  const size_t smem_h = small_hist_smem(nbins), smem_s = small_scatter_smem(nbins);
  if (smem_h > 48 * 1024)
    PM_CUDA_TRY(cudaFuncSetAttribute(k_small_hist<Key>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
  if (smem_s > 48 * 1024)
    PM_CUDA_TRY(cudaFuncSetAttribute(k_small_scatter<Key, Sink>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
  bool per_warp = false;
  if constexpr (Key::kVec4 && Key::kRaw4) {
    static const bool cta_per_tile = getenv("PM_HIST_CTA") != nullptr;  // A/B knob
    per_warp = !cta_per_tile;
    if (per_warp)
      k_small_hist_warp<Key><<<(unsigned)((ntiles + kPartWarps - 1) / kPartWarps), kPartThreads,
                               smem_h, s>>>(key, n, nbins, ntiles, hist);
  }
  if (!per_warp)
    k_small_hist<Key><<<(unsigned)ntiles, kPartThreads, smem_h, s>>>(key, n, nbins, ntiles,
                                                                         hist);
  PM_CUDA_TRY(cudaGetLastError());
  int rc = exclusive_scan_i64(hist, len, scan_tmp, s);
  if (rc) return rc;
  k_part_bin_totals<<<(nbins + 255) / 256, 256, 0, s>>>(
      hist, ntiles, nbins, reinterpret_cast<const long long*>(scan_tmp), counts, offsets);
  PM_CUDA_TRY(cudaGetLastError());
  if (scatter) {
    k_small_scatter<Key, Sink><<<small_scatter_grid(ntiles), kPartThreads, smem_s, s>>>(
        key, sink, n, nbins, ntiles, hist);
    PM_CUDA_TRY(cudaGetLastError());
  }
  return PM_OK;
}

// The scatter pass alone, reusing the scanned histogram and tile summary a
// previous counting call (`scatter` false, same key / n / nbins) left in scratch.
template <class Key, class Sink>
int stable_partition_small_scatter(Key key, Sink sink, long long n, int nbins, void* scratch,
                                   size_t scratch_bytes, cudaStream_t s) {
  if (nbins < 1 || nbins > kSmallBins)
    return set_error("partition: scatter-only pass needs 1..%d bins", kSmallBins),
           PM_ERR_UNSUPPORTED;
  if (n <= 0) return PM_OK;
  if (scratch_bytes < small_scratch_bytes(n, nbins))
    return set_error("partition: scratch too small"), PM_ERR_INVALID;
  const long long ntiles = (n + kSmallTile - 1) / kSmallTile;
  const size_t smem_s = small_scatter_smem(nbins);
  if (smem_s > 48 * 1024)
    PM_CUDA_TRY(cudaFuncSetAttribute(k_small_scatter<Key, Sink>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
  k_small_scatter<Key, Sink><<<small_scatter_grid(ntiles), kPartThreads, smem_s, s>>>(
      key, sink, n, nbins, ntiles, reinterpret_cast<const long long*>(scratch));
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

// counts/offsets always; the scatter only when `scatter` is true.
template <class Key, class Sink>
int stable_partition(Key key, Sink sink, bool scatter, long long n, int nbins, long long* counts,
                     long long* offsets, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (nbins > 0 && nbins <= kSmallBins && n > 0)
    return stable_partition_small(key, sink, scatter, n, nbins, counts, offsets, scratch,
                                  scratch_bytes, s);
  if (nbins <= 0 || nbins > 4096) return set_error("partition: 1..4096 bins"), PM_ERR_INVALID;
  if (scratch_bytes < part_scratch_bytes(n, nbins))
    return set_error("partition: scratch too small"), PM_ERR_INVALID;
  if (n <= 0) {
    PM_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(long long) * nbins, s));
    PM_CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(long long) * nbins, s));
    return PM_OK;
  }
  const int tile = part_tile(nbins);
  const long long ntiles = (n + tile - 1) / tile;
  if (ntiles > 0x7FFFFFFFLL) return set_error("partition: too many tiles"), PM_ERR_UNSUPPORTED;
  const long long len = ntiles * nbins;
  long long* hist = reinterpret_cast<long long*>(scratch);
  void* scan_tmp = reinterpret_cast<char*>(scratch) + len * 8;
  k_part_hist<Key><<<(unsigned)ntiles, kPartThreads, sizeof(int) * nbins, s>>>(key, n, nbins, tile,
                                                                             ntiles, hist);
  PM_CUDA_TRY(cudaGetLastError());
  int rc = exclusive_scan_i64(hist, len, scan_tmp, s);
  if (rc) return rc;
  k_part_bin_totals<<<(nbins + 255) / 256, 256, 0, s>>>(
      hist, ntiles, nbins, reinterpret_cast<const long long*>(scan_tmp), counts, offsets);
  PM_CUDA_TRY(cudaGetLastError());
  if (scatter) {
    const size_t smem = sizeof(int) * (size_t)nbins * (1 + kPartWarps);
    if (smem > 48 * 1024)
      PM_CUDA_TRY(cudaFuncSetAttribute(k_part_scatter<Key, Sink>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_part_scatter<Key, Sink><<<(unsigned)ntiles, kPartThreads, smem, s>>>(key, sink, n, nbins,
                                                                          tile, ntiles, hist);
    PM_CUDA_TRY(cudaGetLastError());
  }
  return PM_OK;
}

}  // namespace
}  // namespace pm
