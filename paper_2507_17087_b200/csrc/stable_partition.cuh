// Generic stable counting partition used by K2 (points by processor) and K3
// (halo transfer entries by (src, dst) pair).
//
// Items are indexed 0..n-1; `Key::operator()(i)` returns the bin of item i or
// -1 (no output).  `Sink::put(pos, i)` writes item i at output position pos.
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

#include <type_traits>

#include "pm_common.h"
#include "scan.cuh"

namespace pm {
namespace {

constexpr int kPartThreads = 256;
constexpr int kPartWarps = kPartThreads / 32;

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
      sink.put(pos0[(long long)b * ntiles + t] + run[b] + pre + rank, i);
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
//
// Thread t of a tile owns the contiguous items [t*IPT, (t+1)*IPT); item order
// inside a tile is therefore (thread, item), the input order.  Counts live in
// lane-private shared memory cells cnt[bin][thread] (bank = thread % 32, no
// conflicts, no atomics).  The scatter scans cnt along threads for every bin
// and each thread then writes its items at base + prefix + running count.
constexpr int kSmallBins = 64;
constexpr int kIPT = 16;                          // items per thread
constexpr int kSmallTile = kPartThreads * kIPT;   // 4096 items per tile

inline size_t small_scratch_bytes(long long n, int nbins) {
  const long long ntiles = (n + kSmallTile - 1) / kSmallTile;
  const long long len = ntiles * nbins;
  return (size_t)(len * 8) + scan_scratch_bytes(len) + 256;
}

// Phase A of both kernels: keys evaluated in coalesced order (item
// base + t + 256 m), stored as int8 bins in shared memory.
template <class Key, class = void>
struct HasKeys4 : std::false_type {};
template <class Key>
struct HasKeys4<Key, decltype(void(&Key::keys4))> : std::true_type {};

template <class Key>
__device__ __forceinline__ void small_keys(Key& key, long long base, long long n,
                                           signed char* __restrict__ sbin) {
  if constexpr (HasKeys4<Key>::value) {
    // 4 consecutive keys per 16-byte load (e.g. processor ids in HBM)
#pragma unroll
    for (int m = 0; m < kIPT / 4; ++m) {
      const int off = (m * kPartThreads + threadIdx.x) * 4;
      const long long i = base + off;
      int packed;
      if (i + 3 < n && key.vec_ok) {
        packed = key.keys4(i);
      } else {
        packed = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          packed |= ((i + q < n ? key(i + q) : -1) & 0xFF) << (8 * q);
      }
      *reinterpret_cast<int*>(sbin + off) = packed;
    }
  } else {
#pragma unroll 4
    for (int m = 0; m < kIPT; ++m) {
      const int off = m * kPartThreads + threadIdx.x;
      const long long i = base + off;
      sbin[off] = (signed char)(i < n ? key(i) : -1);
    }
  }
}

template <class Key>
__global__ void __launch_bounds__(kPartThreads)
k_small_hist(Key key, long long n, int nbins, long long ntiles, long long* __restrict__ hist) {
  extern __shared__ __align__(16) int smem_words[];  // int8 bins[4096] | cnt[nbins][256]
  signed char* sbin = reinterpret_cast<signed char*>(smem_words);
  int* cnt = smem_words + kSmallTile / 4;
  for (int b = 0; b < nbins; ++b) cnt[b * kPartThreads + threadIdx.x] = 0;
  const long long base = (long long)blockIdx.x * kSmallTile;
  small_keys(key, base, n, sbin);
  __syncthreads();
  // count this thread's 16 contiguous bins (one 16-byte shared load)
  const int4 w = reinterpret_cast<const int4*>(sbin)[threadIdx.x];
  const signed char* bb = reinterpret_cast<const signed char*>(&w);
  int run_bin = -1, run = 0;
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int b = bb[j];
    if (b != run_bin) {
      if (run_bin >= 0) cnt[run_bin * kPartThreads + threadIdx.x] += run;
      run_bin = b;
      run = 0;
    }
    ++run;
  }
  if (run_bin >= 0) cnt[run_bin * kPartThreads + threadIdx.x] += run;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = warp; b < nbins; b += kPartWarps) {
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kPartThreads / 32; ++k) sum += cnt[b * kPartThreads + k * 32 + lane];
#pragma unroll
    for (int d = 16; d; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
    if (lane == 0) hist[(long long)b * ntiles + blockIdx.x] = sum;
  }
}

template <class Key, class Sink>
__global__ void __launch_bounds__(kPartThreads)
k_small_scatter(Key key, Sink sink, long long n, int nbins, long long ntiles,
                const long long* __restrict__ pos0) {
  // shared: bins[4096] int8 | stage[4096] int16 | cnt[nbins][256] | start[nbins + 1]
  extern __shared__ __align__(16) int smem_words[];
  signed char* sbin = reinterpret_cast<signed char*>(smem_words);
  short* stage = reinterpret_cast<short*>(sbin + kSmallTile);
  int* cnt = reinterpret_cast<int*>(stage + kSmallTile);
  int* start = cnt + nbins * kPartThreads;
  for (int b = 0; b < nbins; ++b) cnt[b * kPartThreads + threadIdx.x] = 0;
  const long long base = (long long)blockIdx.x * kSmallTile;
  small_keys(key, base, n, sbin);
  __syncthreads();
  const int4 w = reinterpret_cast<const int4*>(sbin)[threadIdx.x];
  const signed char* bb = reinterpret_cast<const signed char*>(&w);
  int bins[kIPT];
#pragma unroll
  for (int j = 0; j < kIPT; ++j) bins[j] = bb[j];
  int run_bin = -1, run = 0;
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    if (bins[j] != run_bin) {
      if (run_bin >= 0) cnt[run_bin * kPartThreads + threadIdx.x] += run;
      run_bin = bins[j];
      run = 0;
    }
    ++run;
  }
  if (run_bin >= 0) cnt[run_bin * kPartThreads + threadIdx.x] += run;
  __syncthreads();
  // exclusive scan of each bin's row along the threads; row totals -> start[]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = warp; b < nbins; b += kPartWarps) {
    int* row = cnt + b * kPartThreads;
    int v[kPartThreads / 32];
    int s = 0;
#pragma unroll
    for (int k = 0; k < kPartThreads / 32; ++k) {
      v[k] = row[lane * (kPartThreads / 32) + k];
      s += v[k];
    }
    int incl = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += u;
    }
    int run_pre = incl - s;
#pragma unroll
    for (int k = 0; k < kPartThreads / 32; ++k) {
      row[lane * (kPartThreads / 32) + k] = run_pre;
      run_pre += v[k];
    }
    if (lane == 31) start[b] = incl;  // bin total in this tile
  }
  __syncthreads();
  if (warp == 0) {  // start[b] = exclusive prefix of the bin totals (nbins <= 64)
    const int t0 = lane < nbins ? start[lane] : 0;
    const int t1 = lane + 32 < nbins ? start[lane + 32] : 0;
    int a = t0, c = t1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int ua = __shfl_up_sync(0xffffffffu, a, d), uc = __shfl_up_sync(0xffffffffu, c, d);
      if (lane >= d) { a += ua; c += uc; }
    }
    const int tot0 = __shfl_sync(0xffffffffu, a, 31);
    const int tot1 = __shfl_sync(0xffffffffu, c, 31);
    if (lane < nbins) start[lane] = a - t0;
    if (lane + 32 < nbins) start[lane + 32] = tot0 + c - t1;
    if (lane == 0) start[nbins] = tot0 + tot1;
  }
  __syncthreads();
  // a tile whose items all share one bin (block mappings: the common case)
  // maps item k to output k of that bin's segment -- write it straight out
  int only = -1;
  for (int b = 0; b < nbins; ++b)
    if (start[b + 1] - start[b] == kSmallTile) only = b;
  if (only >= 0) {
    const long long p0 = pos0[(long long)only * ntiles + blockIdx.x];
#pragma unroll 4
    for (int k = threadIdx.x; k < kSmallTile; k += kPartThreads) sink.put(p0 + k, base + k);
    return;
  }
  // stable local positions; stage the item offsets in output order
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int b = bins[j];
    if (b < 0) continue;
    int* c = cnt + b * kPartThreads + threadIdx.x;
    const int r = *c;
    *c = r + 1;
    stage[start[b] + r] = (short)(threadIdx.x * kIPT + j);
  }
  __syncthreads();
  // coalesced write-out, one bin segment per warp at a time
  for (int b = warp; b < nbins; b += kPartWarps) {
    const int lo = start[b], hi = start[b + 1];
    if (lo == hi) continue;
    const long long p0 = pos0[(long long)b * ntiles + blockIdx.x] - lo;
    for (int k = lo + lane; k < hi; k += 32) sink.put(p0 + k, base + stage[k]);
  }
}

inline size_t small_hist_smem(int nbins) {
  return sizeof(int) * (size_t)nbins * kPartThreads + kSmallTile;
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
  void* scan_tmp = reinterpret_cast<char*>(scratch) + len * 8;
  const size_t smem_h = small_hist_smem(nbins), smem_s = small_scatter_smem(nbins);
  if (smem_h > 48 * 1024)
    PM_CUDA_TRY(cudaFuncSetAttribute(k_small_hist<Key>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
  if (smem_s > 48 * 1024)
    PM_CUDA_TRY(cudaFuncSetAttribute(k_small_scatter<Key, Sink>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
  k_small_hist<Key><<<(unsigned)ntiles, kPartThreads, smem_h, s>>>(key, n, nbins, ntiles, hist);
  PM_CUDA_TRY(cudaGetLastError());
  int rc = exclusive_scan_i64(hist, len, scan_tmp, s);
  if (rc) return rc;
  k_part_bin_totals<<<(nbins + 255) / 256, 256, 0, s>>>(
      hist, ntiles, nbins, reinterpret_cast<const long long*>(scan_tmp), counts, offsets);
  PM_CUDA_TRY(cudaGetLastError());
  if (scatter) {
    k_small_scatter<Key, Sink><<<(unsigned)ntiles, kPartThreads, smem_s, s>>>(key, sink, n,
                                                                             nbins, ntiles, hist);
    PM_CUDA_TRY(cudaGetLastError());
  }
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
