// Device half of the small-bin stable counting partition (<= 64 bins).
//
// Self-contained (no includes, no host code) so the same text is compiled
// twice: statically by nvcc for K2 / K3 (stable_partition.cuh) and, embedded
// as a string, by NVRTC next to a generated mapping program for the fused
// map + partition kernels (mapping.cpp) -- there the key of a point is its
// processor id computed in registers, so no id array is ever read.
//
// Key concept:  int operator()(long long i)  -> bin of item i, or -1 (no output)
//               static constexpr bool kVec4; if true also
//               bool vec_ok; int keys4(long long i) -> 4 int8 bins of items i..i+3
//               void prefetch(long long i, long long n): L2 prefetch of item i's key
//               static constexpr bool kRaw4; if true also int4 raw4(long long i) (the
//               16-byte load alone) and int pack4(int4, long long i) (keys4 of it)
//               void uniform(long long base, int count, int bin): the scatter
//               skipped evaluating items [base, base + count), all in `bin`
//               static constexpr bool kPeek; if true also int peek(long long i):
//               the bin without side effects or checks (histogram fast path)
// Sink concept: void put(int bin, long long pos, long long i)
//               void put_run(int bin, long long pos, long long i, int count): the
//               whole CTA stores items i .. i + count - 1 at pos .. pos + count - 1
//
// Thread t of a 4096-item tile owns the contiguous items [16 t, 16 t + 16);
// counts live in lane-private shared cells cnt[bin][thread] (bank = thread %
// 32: no conflicts, no atomics).  The scatter scans cnt along the threads of
// every bin and each thread writes its items at base + prefix + running count.
#pragma once

namespace pmdev {

constexpr int kPartThreads = 256;
constexpr int kPartWarps = kPartThreads / 32;
constexpr int kSmallBins = 64;
constexpr int kIPT = 16;                          // items per thread
constexpr int kSmallTile = kPartThreads * kIPT;   // 4096 items per tile

#ifndef PM_IOTA_CS
#define PM_IOTA_CS 1
#endif

// dst[k] = v0 + k for k < count, by the whole CTA: 16-byte streaming stores
// between a scalar head (to 16-byte alignment) and tail.
__device__ __forceinline__ void store_iota(int* dst, int v0, int count) {
  int head = (int)((4 - (((unsigned long long)dst >> 2) & 3)) & 3);
  if (head > count) head = count;
  if ((int)threadIdx.x < head) dst[threadIdx.x] = v0 + (int)threadIdx.x;
  const int nvec = (count - head) >> 2;
  int4* body = reinterpret_cast<int4*>(dst + head);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const int e = v0 + head + 4 * v;
#if PM_IOTA_CS
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(body + v), "r"(e),
                 "r"(e + 1), "r"(e + 2), "r"(e + 3) : "memory");
#else
    body[v] = make_int4(e, e + 1, e + 2, e + 3);
#endif
  }
  for (int k = head + 4 * nvec + threadIdx.x; k < count; k += blockDim.x) dst[k] = v0 + k;
}

// Phase A of both passes: keys evaluated in coalesced order (item base + t +
// 256 m), stored as int8 bins in shared memory.
template <class Key>
__device__ __forceinline__ void small_keys(const Key& key, long long base, long long n,
                                           signed char* __restrict__ sbin) {
  if constexpr (Key::kVec4) {
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

// Histogram pass: order is irrelevant, so every thread run-length counts the
// keys it evaluates (coalesced order) and flushes a run into its warp's
// shared histogram with one atomic when the bin changes -- block mappings
// flush once per thread.  shared: h[kPartWarps][nbins]
//
// Scratch layout shared with the host (stable_partition.cuh): hist[nbins][ntiles]
// (int64, scanned in place into output slots), then tile_info[ntiles] (int32):
// the single bin of a full tile, kTileEmpty (no output) or kTileMixed.
constexpr int kTileMixed = -1;
constexpr int kTileEmpty = -2;
__device__ __forceinline__ const int* tile_info_of(const long long* hist, int nbins,
                                                   long long ntiles) {
  return reinterpret_cast<const int*>(hist + (long long)nbins * ntiles);
}

// Histogram-pass L2 prefetch distance in tiles (kVec4 keys): ~600 tiles = 4 CTAs per SM
// ahead, 9.8 MB of ids in flight; 1.55 -> 1.41 ms on 1.07e9 ids (tools/k2_prefetch_ab.sh)
#ifndef PM_HIST_PREFETCH_TILES
#define PM_HIST_PREFETCH_TILES 600
#endif

template <class Key>
__device__ __forceinline__ void small_hist_body(const Key& key, long long n, int nbins,
                                                long long ntiles, long long* __restrict__ hist,
                                                int* smem_words, long long tile) {
  int* h = smem_words;
  __shared__ int s_only, s_any;
  if (threadIdx.x == 0) s_only = kTileMixed, s_any = 0;
  for (int b = threadIdx.x; b < kPartWarps * nbins; b += kPartThreads) h[b] = 0;
  __syncthreads();
  const long long base = tile * kSmallTile;
  int* hw = h + (threadIdx.x >> 5) * nbins;
  int run_bin = -1, run = 0;
  auto add = [&](int b) {
    if (b != run_bin) {
      if (run_bin >= 0) atomicAdd(hw + run_bin, run);
      run_bin = b;
      run = 0;
    }
    ++run;
  };
  if constexpr (Key::kVec4) {
#if PM_HIST_PREFETCH_TILES > 0
    // one L2 prefetch per 128-byte line of the tile PM_HIST_PREFETCH_TILES ahead: a CTA
    // lives a few microseconds, so that tile's CTA finds its ids in L2
    if (threadIdx.x < kSmallTile / 32)
      key.prefetch(base + (long long)PM_HIST_PREFETCH_TILES * kSmallTile + 32 * threadIdx.x, n);
#endif
    if (base + kSmallTile <= n && key.vec_ok) {
      // all four 16-byte loads first, then the counting: the loads are in flight
      // together (interleaved with the counting, ptxas issued them one at a time)
      int packed[kIPT / 4];
      if constexpr (Key::kRaw4) {
        int4 raw[kIPT / 4];
#pragma unroll
        for (int m = 0; m < kIPT / 4; ++m)
          raw[m] = key.raw4(base + (long long)(m * kPartThreads + threadIdx.x) * 4);
#pragma unroll
        for (int m = 0; m < kIPT / 4; ++m)
          packed[m] = key.pack4(raw[m], base + (long long)(m * kPartThreads + threadIdx.x) * 4);
      } else {
#pragma unroll
        for (int m = 0; m < kIPT / 4; ++m)
          packed[m] = key.keys4(base + (long long)(m * kPartThreads + threadIdx.x) * 4);
      }
#pragma unroll
      for (int m = 0; m < kIPT / 4; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q) add((int)(signed char)(packed[m] >> (8 * q)));
    } else {
#pragma unroll
      for (int m = 0; m < kIPT / 4; ++m) {
        const long long i = base + (long long)(m * kPartThreads + threadIdx.x) * 4;
        if (i + 3 < n && key.vec_ok) {
          const int packed = key.keys4(i);
#pragma unroll
          for (int q = 0; q < 4; ++q) add((int)(signed char)(packed >> (8 * q)));
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) add(i + q < n ? key(i + q) : -1);
        }
      }
    }
  } else if (base + kSmallTile <= n) {  // full tile: no bounds checks
    if constexpr (Key::kPeek) {
      // unchecked evaluation; a failing / out-of-range item (bin outside
      // [0, nbins)) is only flagged here and re-evaluated with reporting below
      bool bad = false;
#pragma unroll 4
      for (int m = 0; m < kIPT; ++m) {
        const int r = key.peek(base + m * kPartThreads + threadIdx.x);
        const bool ok = (unsigned)r < (unsigned)nbins;
        bad |= !ok;
        add(ok ? r : -1);
      }
      if (bad)
        for (int m = 0; m < kIPT; ++m) (void)key(base + m * kPartThreads + threadIdx.x);
    } else {
#pragma unroll 4
      for (int m = 0; m < kIPT; ++m) add(key(base + m * kPartThreads + threadIdx.x));
    }
  } else {
#pragma unroll 4
    for (int m = 0; m < kIPT; ++m) {
      const long long i = base + m * kPartThreads + threadIdx.x;
      add(i < n ? key(i) : -1);
    }
  }
  if (run_bin >= 0) atomicAdd(hw + run_bin, run);
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += kPartThreads) {
    int sum = 0;
#pragma unroll
    for (int w = 0; w < kPartWarps; ++w) sum += h[w * nbins + b];
    hist[(long long)b * ntiles + tile] = sum;
    if (sum) s_any = 1;
    if (sum == kSmallTile) s_only = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the last (possibly partial) tile always takes the general path
    const int info = tile + 1 == ntiles ? kTileMixed
                     : s_only >= 0       ? s_only
                     : s_any             ? kTileMixed
                                         : kTileEmpty;
    const_cast<int*>(tile_info_of(hist, nbins, ntiles))[tile] = info;
  }
}

// Histogram pass for keys that can prove a whole tile's bin without evaluating
// its points (Key::tile_bin(base, count) -> the bin, or -1 if not proven; the
// generated mapping programs do it by interval arithmetic over the tile's
// coordinate box).  Grid-stride over groups of 256 tiles: every thread tries
// to prove one tile and, on success, writes its histogram column and tile_info
// (a uniform tile: pass 2 writes its indices without evaluating anything);
// the CTA then histograms the unproven tiles of the group point by point.
// The last (possibly partial) tile always takes the general path.
template <class Key>
__device__ __forceinline__ void small_hist_proof(const Key& key, long long n, int nbins,
                                                 long long ntiles, long long* __restrict__ hist,
                                                 int* smem_words) {
  __shared__ int s_todo[kPartThreads];
  int* info = const_cast<int*>(tile_info_of(hist, nbins, ntiles));
  const long long ngroups = (ntiles + kPartThreads - 1) / kPartThreads;
  for (long long g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const long long t = g * kPartThreads + threadIdx.x;
    int b = -1;
    if (t + 1 < ntiles) b = key.tile_bin(t * kSmallTile, kSmallTile);
    if (b >= nbins) b = -1;
    if (b >= 0) {
      for (int q = 0; q < nbins; ++q) hist[(long long)q * ntiles + t] = q == b ? kSmallTile : 0;
      info[t] = b;
    }
    s_todo[threadIdx.x] = t < ntiles && b < 0;
    __syncthreads();
    for (int j = 0; j < kPartThreads; ++j)
      if (s_todo[j]) small_hist_body(key, n, nbins, ntiles, hist, smem_words, g * kPartThreads + j);
    __syncthreads();
  }
}

// shared: int8 bins[4096] | int16 stage[4096] | cnt[nbins][256] | start[nbins + 1]
// pos0[b * ntiles + t] = first output slot of (bin b, tile t) (scanned histogram)
template <class Key, class Sink>
__device__ __forceinline__ void small_scatter_body(const Key& key, const Sink& sink, long long n,
                                                   int nbins, long long ntiles,
                                                   const long long* __restrict__ pos0,
                                                   int* smem_words, long long tile) {
  signed char* sbin = reinterpret_cast<signed char*>(smem_words);
  short* stage = reinterpret_cast<short*>(sbin + kSmallTile);
  int* cnt = reinterpret_cast<int*>(stage + kSmallTile);
  int* start = cnt + nbins * kPartThreads;
  const long long base = tile * kSmallTile;
  // The histogram pass left a summary of every tile (tile_info): a tile with no
  // output at all (every key -1: e.g. interior cells of a halo launch) is
  // skipped; a full tile whose 4096 items all share one bin (block mappings,
  // the common case) is a straight copy of consecutive indices -- in neither
  // case is a key evaluated or read.
  const int info = __ldg(tile_info_of(pos0, nbins, ntiles) + tile);
  if (info == kTileEmpty) return;
  if (info >= 0) {
    const int only = info;
    const long long p0 = pos0[(long long)only * ntiles + tile];
    key.uniform(base, kSmallTile, only);
    sink.put_run(only, p0, base, kSmallTile);
    return;
  }
  for (int b = 0; b < nbins; ++b) cnt[b * kPartThreads + threadIdx.x] = 0;
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
    const long long p0 = pos0[(long long)only * ntiles + tile];
#pragma unroll 4
    for (int k = threadIdx.x; k < kSmallTile; k += kPartThreads) sink.put(only, p0 + k, base + k);
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
    const long long p0 = pos0[(long long)b * ntiles + tile] - lo;
    for (int k = lo + lane; k < hi; k += 32) sink.put(b, p0 + k, base + stage[k]);
  }
}

// The scatter over kTiles consecutive tiles (first_tile ..) per CTA.  The prologue
// fetches every tile's summary and -- in parallel, not after it -- all nbins candidate
// output starts, so a uniform tile's stores wait for one load latency instead of two
// dependent ones, once per kTiles tiles.  Mixed tiles take the general body.
#ifndef PM_SCATTER_TILES
#define PM_SCATTER_TILES 2
#endif
constexpr int kScatterTiles = PM_SCATTER_TILES;

template <int kTiles, class Key, class Sink>
__device__ __forceinline__ void small_scatter_tiles(const Key& key, const Sink& sink, long long n,
                                                    int nbins, long long ntiles,
                                                    const long long* __restrict__ pos0,
                                                    int* smem_words, long long first_tile) {
  __shared__ int s_info[kTiles];
  __shared__ long long s_p0[kTiles][kSmallBins];
  const int* tile_info = tile_info_of(pos0, nbins, ntiles);
  const int per = nbins + 1;
  if (kTiles * per <= kPartThreads) {
    const int j = threadIdx.x / per, q = threadIdx.x - j * per;
    const long long t = first_tile + j;
    if (j < kTiles) {
      if (q == nbins) s_info[j] = t < ntiles ? __ldg(tile_info + t) : kTileEmpty;
      else if (t < ntiles) s_p0[j][q] = __ldg(pos0 + (long long)q * ntiles + t);
    }
  } else if (threadIdx.x < kTiles) {
    const long long t = first_tile + threadIdx.x;
    const int info = t < ntiles ? __ldg(tile_info + t) : kTileEmpty;
    s_info[threadIdx.x] = info;
    if (info >= 0) s_p0[threadIdx.x][info] = __ldg(pos0 + (long long)info * ntiles + t);
  }
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < kTiles; ++j) {
    const long long t = first_tile + j;
    const int info = s_info[j];
    if (info == kTileEmpty) continue;
    if (info >= 0) {
      key.uniform(t * kSmallTile, kSmallTile, info);
      sink.put_run(info, s_p0[j][info], t * kSmallTile, kSmallTile);
      continue;
    }
    small_scatter_body(key, sink, n, nbins, ntiles, pos0, smem_words, t);
    __syncthreads();  // shared memory is reused by the next mixed tile
  }
}

}  // namespace pmdev
