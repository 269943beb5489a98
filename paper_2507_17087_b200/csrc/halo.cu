// K3 -- halo transfer lists of a cell-owned grid.
//
// For every cell c, dimension n and direction s in {-1, +1} (one "slot"
// c * 2R + 2n + (s > 0)), the slot emits an entry (src = owner(c),
// dst = owner of the first cell c + s*j*e_n, 1 <= j <= h_n, whose owner
// differs) if such a cell exists inside the grid.  For a block partition this
// is exactly the set of cells within h_n of an internal face, counted on both
// sides and clipped to the adjacent block -- the quantity the reference's
// oracle_boundary_count enumerates (commvol.py:136-168) and surface_volume
// closes (commvol.py:94-96).  Entries are grouped by key src * P + dst with
// cells ascending (stable_partition.cuh), which is the send list of every
// (src, dst) pair.  The owner grid is read once from HBM; neighbour reads hit
// L1/L2.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "pm_common.h"
#include "stable_partition.cuh"

namespace pm {
namespace {

// I: index arithmetic type -- 32-bit whenever the slot count allows (integer
// division by the runtime extents dominates the key's cost)
template <typename I>
struct HaloKey {
  const int* __restrict__ owner;
  long long ext[3];
  long long stride[3];
  int halo[3];
  int rank;
  int nprocs;
  bool vec_ok;  // 2-D grid: the 4 slots of a cell are 4 consecutive items -> keys4
  bool unit_halo;     // 2-D with h = (1, 1)
  bool small_pairs;   // nprocs^2 < 128: keys fit the int8 lanes of keys4
  double inv_cols;    // 1 / ext[1]
  unsigned div_m, div_s;  // magic multiplier / shift for n / ext[1] (32-bit keys)
  bool div_one;           // ext[1] == 1
  static constexpr bool kVec4 = true;
  static constexpr bool kPeek = false;
  static constexpr bool kRaw4 = false;
  __device__ __forceinline__ void uniform(long long, int, int) const {}
  __device__ __forceinline__ void prefetch(long long, long long) const {}
  // the four slots (up, down, left, right) of cell i / 4 of a 2-D grid: one index
  // decomposition and one owner load per cell, neighbours from L1/L2
  __device__ __forceinline__ int keys4(long long i) const {
    const I cell = (I)i >> 2;
    const I cols = (I)ext[1];
    I r;
    if constexpr (sizeof(I) == 4) {
      // row = cell / cols by multiply-high with the host's magic number (exact for
      // every 32-bit numerator; branch-free round-up method)
      if (div_one) {
        r = cell;
      } else {
        const unsigned t = __umulhi(div_m, cell);
        r = (t + ((cell - t) >> 1)) >> div_s;
      }
    } else {
      // 64-bit slot space: double reciprocal, corrected to the exact quotient
      r = (I)((double)cell * inv_cols);
      if (r * cols > cell) --r;
      else if ((r + 1) * cols <= cell) ++r;
    }
    const I c = cell - r * cols;
    const int o = __ldg(owner + cell);
    if (o < 0 || o >= nprocs) return -1;  // all four slots empty (0xFF bytes)
    if (unit_halo) {  // h = (1, 1): the four direct neighbours
      const int qs[4] = {r > 0 ? __ldg(owner + (cell - cols)) : o,
                         (long long)r + 1 < ext[0] ? __ldg(owner + (cell + cols)) : o,
                         c > 0 ? __ldg(owner + (cell - 1)) : o,
                         (long long)c + 1 < ext[1] ? __ldg(owner + (cell + 1)) : o};
      int packed = 0;
#pragma unroll
      for (int dd = 0; dd < 4; ++dd) {
        const int q = qs[dd];
        const int key = (q == o || q < 0 || q >= nprocs) ? -1 : o * nprocs + q;
        packed |= (key & 0xFF) << (8 * dd);
      }
      return packed;
    }
    int packed = 0;
#pragma unroll
    for (int dd = 0; dd < 4; ++dd) {
      const int n = dd >> 1;
      const int dir = (dd & 1) ? 1 : -1;
      const long long x = n == 0 ? (long long)r : (long long)c;
      const long long st = n == 0 ? (long long)cols : 1;
      int key = -1;
      for (int j = 1; j <= halo[n]; ++j) {
        const long long y = x + dir * j;
        if (y < 0 || y >= ext[n]) break;
        const int q = __ldg(owner + (long long)cell + (long long)dir * j * st);
        if (q != o) {
          key = (q < 0 || q >= nprocs) ? -1 : o * nprocs + q;
          break;
        }
      }
      packed |= (key & 0xFF) << (8 * dd);
    }
    return packed;
  }
  __device__ __forceinline__ int operator()(long long i) const {
    const I slots = (I)(2 * rank);
    const I cell = (I)i / slots;
    const int dd = (int)((I)i - cell * slots);
    const int n = dd >> 1;
    const int dir = (dd & 1) ? 1 : -1;
    const int h = halo[n];
    if (h <= 0) return -1;
    const I x = (cell / (I)stride[n]) % (I)ext[n];
    const int o = __ldg(owner + cell);
    if (o < 0 || o >= nprocs) return -1;
    for (int j = 1; j <= h; ++j) {
      const long long y = (long long)x + dir * j;
      if (y < 0 || y >= ext[n]) return -1;
      const int q = __ldg(owner + (long long)cell + (long long)dir * j * stride[n]);
      if (q != o) return (q < 0 || q >= nprocs) ? -1 : o * nprocs + q;
    }
    return -1;
  }
};

struct HaloSink {
  long long* __restrict__ cells;
  signed char* __restrict__ dims;
  int slots;
  __device__ __forceinline__ void put_run(int b, long long pos, long long i, int count) const {
    for (int k = threadIdx.x; k < count; k += blockDim.x) put(b, pos + k, i + k);
  }
  __device__ __forceinline__ void put(int, long long pos, long long i) const {
    const long long c = i / slots;
    cells[pos] = c;
    if (dims) dims[pos] = (signed char)(i - c * slots);
  }
};

template <typename I>
bool make_key(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
              int32_t nprocs, HaloKey<I>* k, long long* ncells) {
  if (rank < 1 || rank > 3 || nprocs < 1 || nprocs > 64 || !ext || !halo) return false;
  *k = HaloKey<I>{};
  k->owner = owner;
  k->rank = rank;
  k->nprocs = nprocs;
  k->vec_ok = rank == 2;
  k->small_pairs = nprocs * nprocs < 128;
  long long st = 1;
  for (int m = rank - 1; m >= 0; --m) {
    if (ext[m] < 1 || halo[m] < 0) return false;
    k->ext[m] = ext[m];
    k->stride[m] = st;
    k->halo[m] = halo[m];
    st *= ext[m];
  }
  *ncells = st;
  if (rank == 2) {
    k->unit_halo = halo[0] == 1 && halo[1] == 1;
    k->inv_cols = 1.0 / (double)ext[1];
    // n / d = (t + ((n - t) >> 1)) >> (l - 1), t = umulhi(m, n), l = ceil(log2 d),
    // m = floor(2^32 (2^l - d) / d) + 1  (d >= 2; valid for all 32-bit n)
    const unsigned long long d = (unsigned long long)ext[1];
    k->div_one = d == 1;
    if (d >= 2 && d <= 0xFFFFFFFFull) {
      unsigned l = 0;
      while ((1ull << l) < d) ++l;
      k->div_m = (unsigned)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
      k->div_s = l - 1;
    }
  }
  return true;
}

// ---- K3 by compaction (transfer.halo_lists) ---------------------------------------
//
// Halo entries are sparse (cells next to an ownership boundary), so instead of a
// per-(pair, tile) histogram the lists are built in three steps:
//   k_halo_count    per 8192-slot tile: number of entries; per-pair totals by
//                   shared then global atomics (non-empty tiles only)
//   exclusive scan  of the tile counts -> each tile's first output slot
//   k_halo_compact  non-empty tiles only: warp-shuffle + shared-memory prefix
//                   sums place every entry (pair key, slot index) in slot order
// then K2 stably partitions the compacted keys by pair and k_halo_gather emits
// (cell, dim) in that order -- the same lists as the single-pass partition.
constexpr int kHaloTile = 8192;  // slots per tile: 8 rounds of 256 threads x 4
constexpr int kHaloRounds = kHaloTile / (4 * kPartThreads);

template <class Key>
__device__ __forceinline__ void halo_keys4(const Key& key, long long i0, long long n, int (&k)[4]) {
  if (key.vec_ok && key.small_pairs && i0 + 3 < n) {
    const int packed = key.keys4(i0);
#pragma unroll
    for (int q = 0; q < 4; ++q) k[q] = (int)(signed char)(packed >> (8 * q));
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) k[q] = i0 + q < n ? key(i0 + q) : -1;
  }
}

template <class Key>
__global__ void __launch_bounds__(kPartThreads)
k_halo_count(Key key, long long n, int npairs, long long* __restrict__ tile_cnt,
             unsigned long long* __restrict__ pair_cnt) {
  extern __shared__ int sp[];  // [npairs]
  __shared__ int s_tot;
  for (int b = threadIdx.x; b < npairs; b += kPartThreads) sp[b] = 0;
  if (threadIdx.x == 0) s_tot = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kHaloTile;
  int c = 0;
  for (int r = 0; r < kHaloRounds; ++r) {
    int k[4];
    halo_keys4(key, base + (long long)r * 4 * kPartThreads + 4 * threadIdx.x, n, k);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (k[q] >= 0) {
        ++c;
        atomicAdd(&sp[k[q]], 1);
      }
  }
  for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_tot, c);
  __syncthreads();
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = s_tot;
  if (s_tot)
    for (int b = threadIdx.x; b < npairs; b += kPartThreads)
      if (sp[b]) atomicAdd(pair_cnt + b, (unsigned long long)sp[b]);
}

template <class Key>
__global__ void __launch_bounds__(kPartThreads)
k_halo_compact(Key key, long long n, long long ntiles, const long long* __restrict__ tile_off,
               const long long* __restrict__ total, long long cap, int* __restrict__ out_key,
               long long* __restrict__ out_slot) {
  const long long t = blockIdx.x;
  const long long lo = tile_off[t], hi = t + 1 < ntiles ? tile_off[t + 1] : *total;
  if (lo == hi) return;
  __shared__ int s_warp[kPartWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long base = t * kHaloTile;
  long long running = lo;
  for (int r = 0; r < kHaloRounds; ++r) {
    const long long i0 = base + (long long)r * 4 * kPartThreads + 4 * threadIdx.x;
    int k[4];
    halo_keys4(key, i0, n, k);
    const int c = (k[0] >= 0) + (k[1] >= 0) + (k[2] >= 0) + (k[3] >= 0);
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += u;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kPartWarps; ++w) {
      const int v = s_warp[w];
      before += w < warp ? v : 0;
      all += v;
    }
    long long pos = running + before + incl - c;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (k[q] >= 0) {
        if (pos < cap) {
          out_key[pos] = k[q];
          out_slot[pos] = i0 + q;
        }
        ++pos;
      }
    running += all;
    __syncthreads();
  }
}

__global__ void k_halo_gather(const int* __restrict__ perm, const long long* __restrict__ slot,
                              long long n, int slots, long long* __restrict__ cells,
                              signed char* __restrict__ dims) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const long long s = slot[perm[j]];
    const long long c = s / slots;
    cells[j] = c;
    if (dims) dims[j] = (signed char)(s - c * slots);
  }
}

// ---- 2-D, h = (1, 1), cols % 4 == 0: column strips with a rolling row window -------
//
// The common stencil case.  A block owns a strip of kStripCells columns (4 cells per
// thread, one 16-byte load per row) and walks kStripRows rows down it, keeping the
// rows above and below in registers, so every owner is read from HBM once (plus one
// halo row per strip); the left / right neighbours come from the adjacent lanes by
// shuffle.  Most 4-cell groups have no entry at all and cost one comparison.  A tile
// is one row segment of the strip, tile index row * nseg + seg (row-major = slot
// order); the compaction revisits only strips holding entries.
constexpr int kStripCells = 4 * kPartThreads;  // 1024 columns per strip
constexpr int kStripRows = 64;                 // rows per block (one mask bit each)
#ifndef PM_STRIP_BATCH
#define PM_STRIP_BATCH 4
#endif
#ifndef PM_STRIP_MINB
#define PM_STRIP_MINB 4
#endif
#ifndef PM_STRIP_PREFETCH
#define PM_STRIP_PREFETCH 4
#endif
constexpr int kStripBatch = PM_STRIP_BATCH;    // rows of loads in flight per thread
static_assert(kStripRows % kStripBatch == 0, "the unclamped walk takes whole batches");


struct Strip2D {
  const int* __restrict__ owner;
  long long rows, cols;
  int nseg;
  int nprocs;

  __device__ __forceinline__ int4 row(long long r, long long c0) const {
    return __ldg(reinterpret_cast<const int4*>(owner + r * cols + c0));
  }
  // keys of the 16 slots (cell, dd) of the 4 cells cur; returns the number of entries
  __device__ __forceinline__ int keys(const int4& up, const int4& cur, const int4& dn, int lf,
                                      int rt, int (&k)[16]) const {
    const int a = cur.x;
    if (((cur.y ^ a) | (cur.z ^ a) | (cur.w ^ a) | (up.x ^ a) | (up.y ^ a) | (up.z ^ a) |
         (up.w ^ a) | (dn.x ^ a) | (dn.y ^ a) | (dn.z ^ a) | (dn.w ^ a) | (lf ^ a) | (rt ^ a)) == 0)
      return 0;
    const int o[4] = {cur.x, cur.y, cur.z, cur.w};
    const int q[4][4] = {{up.x, dn.x, lf, cur.y},
                         {up.y, dn.y, cur.x, cur.z},
                         {up.z, dn.z, cur.y, cur.w},
                         {up.w, dn.w, cur.z, rt}};
    int n = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int dd = 0; dd < 4; ++dd) {
        const int qq = q[j][dd];
        const bool e = qq != o[j] && (unsigned)qq < (unsigned)nprocs &&
                       (unsigned)o[j] < (unsigned)nprocs;
        k[j * 4 + dd] = e ? o[j] * nprocs + qq : -1;
        n += e;
      }
    return n;
  }
};

// Walks the block's rows; calls f(i, up, cur, dn, lf, rt) for row r0 + i, i < nr.
// Lanes past the last column re-read the last group (the caller masks them with
// `active`); the column left of column 0 is column 0 itself and the column right of
// the last is the last (= no entry).  Blocks touching the first or last grid row
// (kClamp) also clamp row indices: the row above row 0 is row 0, the row below the
// last row the last row.  All lanes of every warp call f.
template <bool kClamp, class F>
__device__ __forceinline__ void strip_walk(const Strip2D& h, long long r0, int nr, long long c0,
                                           F&& f) {
  const int lane = threadIdx.x & 31;
  const long long cc = c0 < h.cols ? c0 : h.cols - 4;
  const bool has_rt = c0 + 4 < h.cols;
  const int* col = h.owner + cc;
  const int* edge = h.owner + (lane == 0 ? (cc > 0 ? cc - 1 : 0) : min(cc + 4, h.cols - 1));
  const bool edge_lane = lane == 0 || lane == 31;
  const size_t st = (size_t)h.cols;
  const unsigned last = (unsigned)(h.rows - 1), ur0 = (unsigned)r0;
  int4 cur = __ldg(reinterpret_cast<const int4*>(col + (size_t)ur0 * st));
  int4 up = __ldg(reinterpret_cast<const int4*>(col + (size_t)(ur0 ? ur0 - 1 : 0) * st));
  const int* pr = col + (size_t)(ur0 + 1) * st;  // row r0 + i + 1 (unclamped walk)
  const int* pe = edge + (size_t)ur0 * st;       // edge column of row r0 + i
#pragma unroll 1
  for (int i = 0; i < nr; i += kStripBatch) {
    int4 nx[kStripBatch];
    int ed[kStripBatch];
#pragma unroll
    for (int u = 0; u < kStripBatch; ++u) {
      if constexpr (kClamp) {
        const unsigned r = min(ur0 + i + u, last);
        nx[u] = __ldg(reinterpret_cast<const int4*>(col + (size_t)min(r + 1, last) * st));
        ed[u] = edge_lane ? __ldg(edge + (size_t)r * st) : 0;
      } else {
        nx[u] = __ldg(reinterpret_cast<const int4*>(pr + u * st));
        ed[u] = edge_lane ? __ldg(pe + u * st) : 0;
      }
    }
    if constexpr (!kClamp) {
#if PM_STRIP_PREFETCH > 0
      // L2 prefetch PM_STRIP_PREFETCH rows past this batch (one lane per 128-byte line):
      // more bytes in flight than the register window holds, at no register cost
      if ((lane & 7) == 0 && i + kStripBatch + PM_STRIP_PREFETCH < nr) {
#pragma unroll
        for (int u = 0; u < kStripBatch; ++u)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pr + (PM_STRIP_PREFETCH + u) * st));
      }
#endif
      pr += kStripBatch * st;
      pe += kStripBatch * st;
    }
#pragma unroll
    for (int u = 0; u < kStripBatch; ++u) {
      const int4 dn = nx[u];
      int lf = __shfl_up_sync(0xffffffffu, cur.w, 1);
      int rt = __shfl_down_sync(0xffffffffu, cur.x, 1);
      if (lane == 0) lf = ed[u];
      if (lane == 31) rt = ed[u];
      if (!has_rt) rt = cur.w;
      if (kClamp ? i + u < nr : true) f(i + u, up, cur, dn, lf, rt);  // block-uniform
      up = cur;
      cur = dn;
    }
  }
}

// interior row blocks (rows r0 - 1 .. r0 + kStripRows exist) walk unclamped
template <class F>
__device__ __forceinline__ void strip_rows(const Strip2D& h, long long r0, int nr, long long c0,
                                           F&& f) {
  if (r0 > 0 && r0 + kStripRows < h.rows)
    strip_walk<false>(h, r0, kStripRows, c0, f);
  else
    strip_walk<true>(h, r0, nr, c0, f);
}

inline size_t pad256(size_t b) { return (b + 255) / 256 * 256; }

__global__ void __launch_bounds__(kPartThreads, PM_STRIP_MINB)
k_halo2d_count(Strip2D h, int npairs, long long* __restrict__ tile_cnt,
               unsigned long long* __restrict__ pair_cnt, unsigned long long* __restrict__ warp_rows,
               unsigned short* __restrict__ warp_pre, unsigned* __restrict__ wl_count,
               unsigned* __restrict__ wl, unsigned* __restrict__ lane_mask) {
  extern __shared__ int sp[];  // [npairs]
  __shared__ int s_row[kStripRows][kPartWarps];
  __shared__ unsigned s_mask[kStripRows / 32][kPartWarps];
  __shared__ int s_any, s_done;
  for (int b = threadIdx.x; b < npairs; b += kPartThreads) sp[b] = 0;
  if (threadIdx.x == 0) s_any = 0, s_done = 0;
  __syncthreads();
  const int seg = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long r0 = (long long)blockIdx.y * kStripRows;
  const int nr = (int)min((long long)kStripRows, h.rows - r0);
  const long long c0 = (long long)seg * kStripCells + 4 * threadIdx.x;
  const bool active = c0 < h.cols;
  unsigned groups = 0;  // bit g: this thread's cells hold entries in rows 8g .. 8g + 7
  strip_rows(h, r0, nr, c0, [&](int i, const int4& up, const int4& cur, const int4& dn, int lf,
                                int rt) {
    int k[16];
    const int n = active ? h.keys(up, cur, dn, lf, rt, k) : 0;
    if (n) {
      groups |= 1u << (i >> 3);
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (k[q] >= 0) atomicAdd(&sp[k[q]], 1);
    }
    const int tot = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0) s_row[i][warp] = tot;
  });
  if (groups) s_any = 1;
  // per 8-row group, the lanes of this warp holding entries: the compaction loads only
  // theirs (written only for warps with entries -- the only ones it reads)
  if (__any_sync(0xffffffffu, groups != 0)) {
    unsigned* lm = lane_mask + (((long long)blockIdx.y * h.nseg + seg) * kPartWarps + warp) * 8;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const unsigned m = __ballot_sync(0xffffffffu, groups >> g & 1);
      if (lane == g) lm[g] = m;
    }
  }
  // the last warp to finish does the block's epilogue; the others leave at once (a
  // block-wide barrier here kept 7 warps waiting for the slowest one)
  __threadfence_block();
  __syncwarp();  // every lane's shared atomics / s_any store precede lane 0's ticket
  int last = 0;
  if (lane == 0) last = atomicAdd(&s_done, 1) == kPartWarps - 1;
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence_block();
  // per tile (row): its entry count; per warp: which rows hold its entries and, in
  // non-empty tiles, its first entry within the tile
  const long long blk = (long long)blockIdx.y * h.nseg + seg;
#pragma unroll
  for (int q = 0; q < kStripRows / 32; ++q) {
    const int i = 32 * q + lane;
    int c[kPartWarps];
    int all = 0;
#pragma unroll
    for (int w = 0; w < kPartWarps; ++w) {
      c[w] = i < nr ? s_row[i][w] : 0;
      all += c[w];
    }
    if (i < nr) {
      tile_cnt[(r0 + i) * h.nseg + seg] = all;
      if (all) {
        int before = 0;
#pragma unroll
        for (int w = 0; w < kPartWarps; ++w) {
          warp_pre[((r0 + i) * h.nseg + seg) * kPartWarps + w] = (unsigned short)before;
          before += c[w];
        }
      }
    }
#pragma unroll
    for (int w = 0; w < kPartWarps; ++w) {
      const unsigned m = __ballot_sync(0xffffffffu, c[w] != 0);
      if (lane == w) s_mask[q][w] = m;
    }
  }
  __syncwarp();
  if (lane < kPartWarps) {
    unsigned long long rows_hit = 0;
#pragma unroll
    for (int q = 0; q < kStripRows / 32; ++q)
      rows_hit |= (unsigned long long)s_mask[q][lane] << (32 * q);
    warp_rows[blk * kPartWarps + lane] = rows_hit;
    // the compaction's work list: the units holding entries
    if (rows_hit) wl[atomicAdd(wl_count, 1u)] = (unsigned)(blk * kPartWarps + lane);
  }
  if (s_any)
    for (int b = lane; b < npairs; b += 32)
      if (sp[b]) atomicAdd(pair_cnt + b, (unsigned long long)sp[b]);
}

// Persistent compaction over the count pass's work list (one item per (row block,
// strip, warp) unit holding entries).  The unit's entries sit, per 8-row group, in the
// cells of the lanes of that group's lane mask, in the rows of its row mask: one
// (row, lane) combination per thread, row-major, so a vertical cut (one lane, every
// row) fills a warp with 32 rows at once and a horizontal cut (every lane, one row)
// with 32 lanes.  Each thread loads its four cells and their neighbours and computes
// their entries; a segmented warp scan over the threads of one row (plus the part of
// that row placed by the previous iteration) gives each entry its slot-order position.
// Entries past `cap` are dropped.
__global__ void __launch_bounds__(256)
k_halo2d_compact(Strip2D h, const long long* __restrict__ tile_off,
                 const unsigned long long* __restrict__ warp_rows,
                 const unsigned short* __restrict__ warp_pre, const unsigned* __restrict__ wl_count,
                 const unsigned* __restrict__ wl, const unsigned* __restrict__ lane_mask,
                 long long cap, int* __restrict__ out_key, long long* __restrict__ out_slot) {
  const int lane = threadIdx.x & 31;
  const unsigned lanes_le = 0xffffffffu >> (31 - lane);
  const unsigned nitems = *wl_count;
  const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
  const size_t st = (size_t)h.cols;
  for (unsigned it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nitems; it += nwarps) {
    const unsigned unit = wl[it];
    const long long blk = unit / kPartWarps;
    const int warp = (int)(unit % kPartWarps);
    const long long rb = blk / h.nseg;
    const int seg = (int)(blk - rb * h.nseg);
    const unsigned long long rows = warp_rows[unit];
    const unsigned my_lm = lane < 8 ? lane_mask[(long long)unit * 8 + lane] : 0u;
    // combinations per 8-row group and their running start (every lane holds all 8)
    int start[9];
    start[0] = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const unsigned lm = __shfl_sync(0xffffffffu, my_lm, g);
      start[g + 1] = start[g] + __popc((unsigned)(rows >> (8 * g)) & 0xFFu) * __popc(lm);
    }
    const int n = start[8];
    int carry_ri = -1;
    long long carry = 0;  // entries of row carry_ri placed by the previous iteration
    for (int g0 = 0; g0 < n; g0 += 32) {
      const int g = g0 + lane;
      const bool valid = g < n;
      int grp = 0;
#pragma unroll
      for (int q = 1; q < 8; ++q) grp += g >= start[q];
      const unsigned lm = __shfl_sync(0xffffffffu, my_lm, grp);
      int ri = 1 << 20;
      int c = 0;
      int k[16];
      long long slot0 = 0, row_first = 0;
      if (valid) {
        const int p = __popc(lm);
        const int local = g - start[grp];
        const unsigned grows = (unsigned)(rows >> (8 * grp)) & 0xFFu;
        ri = 8 * grp + (int)__fns(grows, 0, local / p + 1);
        const int ln = (int)__fns(lm, 0, local % p + 1);
        const long long r = rb * kStripRows + ri;
        const long long c0 = (long long)seg * kStripCells + 4 * (warp * 32 + ln);
        const long long ru = r > 0 ? r - 1 : 0, rd = r + 1 < h.rows ? r + 1 : r;
        const int4 up = __ldg(reinterpret_cast<const int4*>(h.owner + ru * st + c0));
        const int4 cur = __ldg(reinterpret_cast<const int4*>(h.owner + r * st + c0));
        const int4 dn = __ldg(reinterpret_cast<const int4*>(h.owner + rd * st + c0));
        const int lf = c0 > 0 ? __ldg(h.owner + r * st + c0 - 1) : cur.x;
        const int rt = c0 + 4 < h.cols ? __ldg(h.owner + r * st + c0 + 4) : cur.w;
        const long long t = r * h.nseg + seg;
        row_first = __ldg(tile_off + t) + __ldg(warp_pre + t * kPartWarps + warp);
        slot0 = (r * h.cols + c0) * 4;
        c = h.keys(up, cur, dn, lf, rt, k);
      }
      int incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += u;
      }
      // segmented: the first thread of each row's run is a head
      const int prev_ri = __shfl_up_sync(0xffffffffu, ri, 1);
      const bool head = lane == 0 || ri != prev_ri;
      const unsigned heads = __ballot_sync(0xffffffffu, head);
      const int hl = 31 - __clz(heads & lanes_le);
      const int seg_base = __shfl_sync(0xffffffffu, incl - c, hl);
      long long excl = incl - c - seg_base;
      if (ri == carry_ri) excl += carry;  // the row continues from the previous iteration
      if (c) {
        long long pos = row_first + excl;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (k[q] >= 0) {
            if (pos < cap) {
              out_key[pos] = k[q];
              out_slot[pos] = slot0 + q;
            }
            ++pos;
          }
      }
      // carry into the next iteration: the row of lane 31 and what is placed of it so far
      carry_ri = __shfl_sync(0xffffffffu, ri, 31);
      carry = __shfl_sync(0xffffffffu, excl + c, 31);
    }
  }
}

// ---- grouping of the compacted entries by (src, dst) pair ---------------------------
//
// A stable counting sort of the compacted keys (slot order) with small tiles (1024
// entries per CTA, so even a few hundred thousand entries fill the GPU): per-tile key
// histogram, one scan of the key-major [pair][tile] histogram, then a scatter that
// ranks equal keys within a warp by match.any and across warps / rounds through
// shared memory, writing each entry's (cell, dim) at its grouped position.
constexpr int kGroupTile = 4 * kPartThreads;

__global__ void __launch_bounds__(kPartThreads)
k_group_hist(const int* __restrict__ keys, long long cap, const long long* __restrict__ total,
             int npairs, long long ntiles, long long* __restrict__ hist) {
  __shared__ int sh[64];
  for (int b = threadIdx.x; b < npairs; b += kPartThreads) sh[b] = 0;
  __syncthreads();
  const long long n = min(cap, *total);
  const long long base = (long long)blockIdx.x * kGroupTile;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long i = base + q * kPartThreads + threadIdx.x;
    if (i < n) atomicAdd(&sh[__ldg(keys + i)], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < npairs; b += kPartThreads)
    hist[(long long)b * ntiles + blockIdx.x] = sh[b];
}

__global__ void __launch_bounds__(kPartThreads)
k_group_scatter(const int* __restrict__ keys, const long long* __restrict__ slots, long long cap,
                const long long* __restrict__ total, int npairs, long long ntiles,
                const long long* __restrict__ off, int nslots, long long* __restrict__ cells,
                signed char* __restrict__ dims, const long long* __restrict__ grand,
                long long* __restrict__ pair_counts, long long* __restrict__ pair_offsets) {
  __shared__ int wc[kPartWarps][64];
  __shared__ long long run[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x < npairs) {  // k_part_bin_totals, folded in
    const int b = threadIdx.x;
    const long long lo = off[(long long)b * ntiles];
    const long long hi = b + 1 < npairs ? off[(long long)(b + 1) * ntiles] : *grand;
    pair_counts[b] = hi - lo;
    pair_offsets[b] = lo;
  }
  for (int b = threadIdx.x; b < npairs; b += kPartThreads)
    run[b] = off[(long long)b * ntiles + blockIdx.x];
  const long long n = min(cap, *total);
  const long long base = (long long)blockIdx.x * kGroupTile;
  const unsigned lt = (1u << lane) - 1;
  for (int q = 0; q < 4; ++q) {
    wc[warp][lane] = 0;
    wc[warp][lane + 32] = 0;
    __syncwarp();
    const long long i = base + q * kPartThreads + threadIdx.x;
    const int key = i < n ? __ldg(keys + i) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && lane == __ffs(peers) - 1) wc[warp][key] = __popc(peers);
    __syncthreads();
    if (key >= 0) {
      long long pos = run[key] + __popc(peers & lt);
      for (int w = 0; w < warp; ++w) pos += wc[w][key];
      const long long sl = __ldg(slots + i);
      const long long c = sl / nslots;
      cells[pos] = c;
      if (dims) dims[pos] = (signed char)(sl - c * nslots);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < npairs; b += kPartThreads) {
      int add = 0;
#pragma unroll
      for (int w = 0; w < kPartWarps; ++w) add += wc[w][b];
      run[b] += add;
    }
    __syncthreads();
  }
}

bool make_strip2d(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
                  int32_t nprocs, Strip2D* h) {
  if (rank != 2 || halo[0] != 1 || halo[1] != 1 || ext[1] % 4 != 0 || ext[1] < 4 || ext[0] < 1 ||
      (uintptr_t)owner % 16 != 0 || nprocs < 1 || nprocs > 64)
    return false;
  const long long nseg = (ext[1] + kStripCells - 1) / kStripCells;
  if (ext[1] > 0x7FFFFFFF || (ext[0] + kStripRows - 1) / kStripRows > 65535) return false;
  h->owner = owner;
  h->rows = ext[0];
  h->cols = ext[1];
  h->nseg = (int)nseg;
  h->nprocs = nprocs;
  return true;
}

// tile scratch: offsets int64 [ntiles] | scan temp
size_t halo_tile_bytes(long long ntiles) {
  return (size_t)(((ntiles * 8 + 255) / 256) * 256) + scan_scratch_bytes(ntiles);
}

// strip kernels: tile scratch | per-(row block, strip, warp) row masks | per-(tile, warp)
// first entry (written for non-empty tiles only) | work list count | work list
size_t strip_mask_bytes(const Strip2D& h) {
  return pad256((size_t)((h.rows + kStripRows - 1) / kStripRows) * h.nseg * kPartWarps * 8);
}
size_t strip_pre_bytes(const Strip2D& h) {
  return pad256((size_t)h.rows * h.nseg * kPartWarps * 2);
}
size_t strip_tile_bytes(const Strip2D& h) {
  return pad256(halo_tile_bytes(h.rows * h.nseg)) + strip_mask_bytes(h) + strip_pre_bytes(h) +
         256 + strip_mask_bytes(h) / 2 + strip_mask_bytes(h) * 4;
}
unsigned long long* strip_warp_rows(const Strip2D& h, void* scratch) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(scratch) +
                                               pad256(halo_tile_bytes(h.rows * h.nseg)));
}
unsigned short* strip_warp_pre(const Strip2D& h, void* scratch) {
  return reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(strip_warp_rows(h, scratch)) +
                                           strip_mask_bytes(h));
}
unsigned* strip_wl_count(const Strip2D& h, void* scratch) {
  return reinterpret_cast<unsigned*>(reinterpret_cast<char*>(strip_warp_pre(h, scratch)) +
                                     strip_pre_bytes(h));
}
unsigned* strip_wl(const Strip2D& h, void* scratch) { return strip_wl_count(h, scratch) + 64; }
unsigned* strip_lane_mask(const Strip2D& h, void* scratch) {
  return reinterpret_cast<unsigned*>(reinterpret_cast<char*>(strip_wl(h, scratch)) +
                                     strip_mask_bytes(h) / 2);
}

template <class Key>
int halo_count(const Key& key, long long n, int npairs, long long* pair_cnt, void* scratch,
               size_t bytes, long long* total_out, cudaStream_t s) {
  const long long ntiles = (n + kHaloTile - 1) / kHaloTile;
  if (bytes < halo_tile_bytes(ntiles)) return set_error("pm_halo_count: scratch too small"),
                                               PM_ERR_INVALID;
  PM_CUDA_TRY(cudaMemsetAsync(pair_cnt, 0, sizeof(long long) * npairs, s));
  if (ntiles == 0) {
    if (total_out) PM_CUDA_TRY(cudaMemsetAsync(total_out, 0, 8, s));
    return PM_OK;
  }
  long long* tile = reinterpret_cast<long long*>(scratch);
  void* scan_tmp = reinterpret_cast<char*>(scratch) + ((ntiles * 8 + 255) / 256) * 256;
  k_halo_count<Key><<<(unsigned)ntiles, kPartThreads, sizeof(int) * npairs, s>>>(
      key, n, npairs, tile, reinterpret_cast<unsigned long long*>(pair_cnt));
  PM_CUDA_TRY(cudaGetLastError());
  int rc = exclusive_scan_i64(tile, ntiles, scan_tmp, s);
  if (rc || !total_out) return rc;
  PM_CUDA_TRY(cudaMemcpyAsync(total_out, scan_tmp, 8, cudaMemcpyDeviceToDevice, s));
  return PM_OK;
}

template <class Key>
int halo_compact(const Key& key, long long n, void* scratch, int* keys, long long* slots_out,
                 long long cap, cudaStream_t s) {
  const long long ntiles = (n + kHaloTile - 1) / kHaloTile;
  if (ntiles == 0) return PM_OK;
  const long long* tile = reinterpret_cast<const long long*>(scratch);
  const long long* total = reinterpret_cast<const long long*>(
      reinterpret_cast<char*>(scratch) + ((ntiles * 8 + 255) / 256) * 256);
  k_halo_compact<Key><<<(unsigned)ntiles, kPartThreads, 0, s>>>(key, n, ntiles, tile, total, cap,
                                                               keys, slots_out);
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

}  // namespace
}  // namespace pm

extern "C" {

size_t pm_halo_scratch_bytes(const int64_t* ext, int32_t rank, int32_t nprocs) {
  if (!ext || rank < 1 || rank > 3 || nprocs < 1) return 256;
  long long cells = 1;
  for (int m = 0; m < rank; ++m) cells *= ext[m];
  return pm::part_scratch_bytes(cells * 2 * rank, nprocs * nprocs);
}

int pm_halo_lists(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
                  int32_t nprocs, int64_t* pair_counts, int64_t* pair_offsets, int64_t* cells,
                  int8_t* dims, void* scratch, size_t scratch_bytes, void* stream) {
  long long ncells = 0;
  pm::HaloKey<unsigned long long> key64;
  if (!owner || !pair_counts || !pair_offsets ||
      !pm::make_key(owner, ext, rank, halo, nprocs, &key64, &ncells))
    return pm::set_error("pm_halo_lists: bad arguments (rank 1..3, nprocs 1..64)"),
           PM_ERR_INVALID;
  pm::HaloSink sink{reinterpret_cast<long long*>(cells), reinterpret_cast<signed char*>(dims),
                    2 * rank};
  const long long items = ncells * 2 * rank;
  if (items <= (1LL << 32)) {  // 32-bit slot arithmetic (item indices < 2^32)
    pm::HaloKey<unsigned> key32;
    pm::make_key(owner, ext, rank, halo, nprocs, &key32, &ncells);
    return pm::stable_partition(key32, sink, cells != nullptr, items, nprocs * nprocs,
                                reinterpret_cast<long long*>(pair_counts),
                                reinterpret_cast<long long*>(pair_offsets), scratch,
                                scratch_bytes, (cudaStream_t)stream);
  }
  return pm::stable_partition(key64, sink, cells != nullptr, items, nprocs * nprocs,
                              reinterpret_cast<long long*>(pair_counts),
                              reinterpret_cast<long long*>(pair_offsets), scratch, scratch_bytes,
                              (cudaStream_t)stream);
}

size_t pm_halo_tile_scratch_bytes(const int64_t* ext, int32_t rank) {
  if (!ext || rank < 1 || rank > 3) return 256;
  long long cells = 1;
  for (int m = 0; m < rank; ++m) cells *= ext[m];
  long long ntiles = (cells * 2 * rank + pm::kHaloTile - 1) / pm::kHaloTile;
  size_t bytes = pm::halo_tile_bytes(ntiles);
  if (rank == 2 && ext[0] >= 1 && ext[1] >= 4) {  // the strip kernels' layout
    pm::Strip2D h{};
    h.rows = ext[0];
    h.nseg = (int)((ext[1] + pm::kStripCells - 1) / pm::kStripCells);
    bytes = std::max(bytes, pm::strip_tile_bytes(h));
  }
  return bytes;
}

int pm_halo_count(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
                  int32_t nprocs, int64_t* pair_counts, void* tile_scratch, size_t bytes,
                  int64_t* total, void* stream) {
  long long ncells = 0;
  pm::HaloKey<unsigned long long> key64;
  if (!owner || !pair_counts || !tile_scratch ||
      !pm::make_key(owner, ext, rank, halo, nprocs, &key64, &ncells))
    return pm::set_error("pm_halo_count: bad arguments (rank 1..3, nprocs 1..64)"),
           PM_ERR_INVALID;
  const long long items = ncells * 2 * rank;
  auto* pc = reinterpret_cast<long long*>(pair_counts);
  pm::Strip2D h2;
  if (pm::make_strip2d(owner, ext, rank, halo, nprocs, &h2)) {
    const long long ntiles = h2.rows * h2.nseg;
    if (bytes < pm::strip_tile_bytes(h2))
      return pm::set_error("pm_halo_count: scratch too small"), PM_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    PM_CUDA_TRY(cudaMemsetAsync(pc, 0, sizeof(long long) * nprocs * nprocs, s));
    PM_CUDA_TRY(cudaMemsetAsync(pm::strip_wl_count(h2, tile_scratch), 0, 4, s));
    long long* tile = reinterpret_cast<long long*>(tile_scratch);
    const dim3 grid((unsigned)h2.nseg, (unsigned)((h2.rows + pm::kStripRows - 1) / pm::kStripRows));
    pm::k_halo2d_count<<<grid, pm::kPartThreads, sizeof(int) * nprocs * nprocs, s>>>(
        h2, nprocs * nprocs, tile, reinterpret_cast<unsigned long long*>(pc),
        pm::strip_warp_rows(h2, tile_scratch), pm::strip_warp_pre(h2, tile_scratch),
        pm::strip_wl_count(h2, tile_scratch), pm::strip_wl(h2, tile_scratch),
        pm::strip_lane_mask(h2, tile_scratch));
    PM_CUDA_TRY(cudaGetLastError());
    void* scan_tmp = reinterpret_cast<char*>(tile_scratch) + ((ntiles * 8 + 255) / 256) * 256;
    int rc = pm::exclusive_scan_i64(tile, ntiles, scan_tmp, s);
    if (rc || !total) return rc;
    PM_CUDA_TRY(cudaMemcpyAsync(total, scan_tmp, 8, cudaMemcpyDeviceToDevice, s));
    return PM_OK;
  }
  if (items <= (1LL << 32)) {
    pm::HaloKey<unsigned> key32;
    pm::make_key(owner, ext, rank, halo, nprocs, &key32, &ncells);
    return pm::halo_count(key32, items, nprocs * nprocs, pc, tile_scratch, bytes,
                          reinterpret_cast<long long*>(total), (cudaStream_t)stream);
  }
  return pm::halo_count(key64, items, nprocs * nprocs, pc, tile_scratch, bytes,
                        reinterpret_cast<long long*>(total), (cudaStream_t)stream);
}

int pm_halo_compact(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
                    int32_t nprocs, void* tile_scratch, int32_t* keys, int64_t* slots, int64_t cap,
                    void* stream) {
  long long ncells = 0;
  pm::HaloKey<unsigned long long> key64;
  if (!owner || !tile_scratch || !keys || !slots ||
      !pm::make_key(owner, ext, rank, halo, nprocs, &key64, &ncells))
    return pm::set_error("pm_halo_compact: bad arguments"), PM_ERR_INVALID;
  const long long items = ncells * 2 * rank;
  auto* so = reinterpret_cast<long long*>(slots);
  pm::Strip2D h2;
  if (pm::make_strip2d(owner, ext, rank, halo, nprocs, &h2)) {
    const long long* tile = reinterpret_cast<const long long*>(tile_scratch);
    // persistent warps over the work list
    pm::k_halo2d_compact<<<(unsigned)(pm::num_sms() * 8), 256, 0, (cudaStream_t)stream>>>(
        h2, tile, pm::strip_warp_rows(h2, tile_scratch), pm::strip_warp_pre(h2, tile_scratch),
        pm::strip_wl_count(h2, tile_scratch), pm::strip_wl(h2, tile_scratch),
        pm::strip_lane_mask(h2, tile_scratch), cap, keys, so);
    PM_CUDA_TRY(cudaGetLastError());
    return PM_OK;
  }
  if (items <= (1LL << 32)) {
    pm::HaloKey<unsigned> key32;
    pm::make_key(owner, ext, rank, halo, nprocs, &key32, &ncells);
    return pm::halo_compact(key32, items, tile_scratch, keys, so, cap, (cudaStream_t)stream);
  }
  return pm::halo_compact(key64, items, tile_scratch, keys, so, cap, (cudaStream_t)stream);
}

size_t pm_halo_group_scratch_bytes(int64_t cap, int32_t nprocs) {
  const long long ntiles = (cap + pm::kGroupTile - 1) / pm::kGroupTile;
  const long long len = std::max(1LL, ntiles * nprocs * nprocs);
  return pm::pad256((size_t)len * 8) + pm::scan_scratch_bytes(len);
}

int pm_halo_group(const int32_t* keys, const int64_t* slots, int64_t cap, const int64_t* total,
                  int32_t rank, int32_t nprocs, int64_t* pair_counts, int64_t* pair_offsets,
                  int64_t* cells, int8_t* dims, void* scratch, size_t scratch_bytes,
                  void* stream) {
  if (cap < 0 || rank < 1 || rank > 3 || nprocs < 1 || nprocs > 8 || !total || !pair_counts ||
      !pair_offsets || !scratch || (cap > 0 && (!keys || !slots || !cells)))
    return pm::set_error("pm_halo_group: bad arguments (nprocs 1..8)"), PM_ERR_INVALID;
  if (scratch_bytes < pm_halo_group_scratch_bytes(cap, nprocs))
    return pm::set_error("pm_halo_group: scratch too small"), PM_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int npairs = nprocs * nprocs;
  const long long ntiles = std::max(1LL, (long long)((cap + pm::kGroupTile - 1) / pm::kGroupTile));
  const long long len = ntiles * npairs;
  long long* hist = reinterpret_cast<long long*>(scratch);
  void* scan_tmp = reinterpret_cast<char*>(scratch) + pm::pad256((size_t)len * 8);
  auto* tot = reinterpret_cast<const long long*>(total);
  pm::k_group_hist<<<(unsigned)ntiles, pm::kPartThreads, 0, s>>>(keys, cap, tot, npairs, ntiles,
                                                                hist);
  PM_CUDA_TRY(cudaGetLastError());
  int rc = pm::exclusive_scan_i64(hist, len, scan_tmp, s);
  if (rc) return rc;
  if (cells) {  // the scatter's block 0 also writes the per-pair counts / offsets
    pm::k_group_scatter<<<(unsigned)ntiles, pm::kPartThreads, 0, s>>>(
        keys, reinterpret_cast<const long long*>(slots), cap, tot, npairs, ntiles, hist, 2 * rank,
        reinterpret_cast<long long*>(cells), reinterpret_cast<signed char*>(dims),
        reinterpret_cast<const long long*>(scan_tmp), reinterpret_cast<long long*>(pair_counts),
        reinterpret_cast<long long*>(pair_offsets));
    PM_CUDA_TRY(cudaGetLastError());
    return PM_OK;
  }
  pm::k_part_bin_totals<<<1, 64, 0, s>>>(hist, ntiles, npairs,
                                         reinterpret_cast<const long long*>(scan_tmp),
                                         reinterpret_cast<long long*>(pair_counts),
                                         reinterpret_cast<long long*>(pair_offsets));
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

int pm_halo_gather(const int32_t* perm, const int64_t* slots, int64_t n, int32_t rank,
                   int64_t* cells, int8_t* dims, void* stream) {
  if (n < 0 || rank < 1 || rank > 3 || (n > 0 && (!perm || !slots || !cells)))
    return pm::set_error("pm_halo_gather: bad arguments"), PM_ERR_INVALID;
  if (n == 0) return PM_OK;
  long long blocks = (n + 255) / 256;
  const long long cap = (long long)pm::num_sms() * 8;
  if (blocks > cap) blocks = cap;
  pm::k_halo_gather<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      perm, reinterpret_cast<const long long*>(slots), n, 2 * rank,
      reinterpret_cast<long long*>(cells), reinterpret_cast<signed char*>(dims));
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

}  // extern "C"
