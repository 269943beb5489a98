// K5 -- 5-point Jacobi sweep of a block-mapped 2-D grid with the halo exchange
// fused in (BASELINE configs[4]; the paper's stencil workload).
//
// Each GPU owns one rectangle of the global grid (from the Mapple block
// mapping, K1 + K2).  A sweep reads buffer `in` and writes `out`:
//   out[i][j] = 0.25 * (in[i-1][j] + in[i+1][j] + in[i][j-1] + in[i][j+1])
// for interior cells of the global grid; global boundary cells are copied
// (Dirichlet).  Cells just outside the rectangle are read straight from the
// neighbouring GPU's `in` buffer over NVLink (peer pointers, L2-bypassing
// loads) -- no halo buffers, no copies, no NCCL.
//
// Left / right neighbours exchange columns through column strips: the first and
// last column of every rectangle are computed by dedicated CTAs (launched last) that
// read the neighbour's adjacent column as a contiguous strip -- 16-byte NVLink loads
// of 4 rows -- and publish their own column into a strip for the next sweep, so no
// tile waits on a left / right neighbour and no tile does per-row scalar peer loads.
//
// Cross-GPU ordering, per neighbour (flags pushed into the reader's memory; flag =
// sweeps the writer has completed):
//   publish  sweep s's kernel starts only after all CTAs of sweep s-1 finished
//            (stream order), so its first CTA publishes "s sweeps done" with a
//            system-scope release store into each neighbour's flag slot -- no
//            per-CTA ticket atomics or fences;
//   RAW      a first / last row tile waits until the up / down neighbour has
//            published s (finished sweep s-1), a column-strip CTA until every
//            neighbour has; other tiles never wait;
//   WAR      with three rotating buffers (and column strips) a neighbour reads
//            the buffer / strip I write at sweep s during its sweep s-2.  My
//            sweep s-1 row-edge tiles (up / down) or strip CTAs (left / right)
//            already waited for that neighbour's flag >= s-1, i.e. for its sweep
//            s-2 to finish, so the WAR order is implied and not checked.
// Launch order: column-strip CTAs, the middle tile rows, then the first / last tile
// rows, so the tiles that wait on flags usually find them set.
//
// Traffic: 8 B per cell per sweep from HBM (read in, write out); vertical
// neighbours are reused through L1 inside a 16-row tile.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "pm_common.h"

namespace pm {
namespace {

constexpr int TC = 512;   // cols per tile (128 threads x float4)
constexpr int kThreads = 128;

__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(int32_t* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ float ld_peer(const float* p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float4 ld_peer4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.sys.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_flag(const int32_t* f, int target) {
  if (ld_acquire_sys(f) >= target) return;
  while (ld_acquire_sys(f) < target) __nanosleep(256);
}

// value of global cell (my-local coords i, j may be one step outside the rectangle)
__device__ __forceinline__ float fetch(const pm_stencil_view& v, int64_t i, int64_t j) {
  if (i >= 0 && i < v.rows && j >= 0 && j < v.cols) return __ldg(v.in + i * v.pitch + j);
  if (i < 0) return ld_peer(v.nbr[0] + (v.nbr_rows[0] - 1) * v.nbr_pitch[0] + j);
  if (i >= v.rows) return ld_peer(v.nbr[1] + j);
  if (j < 0) return ld_peer(v.nbr[2] + i * v.nbr_pitch[2] + (v.nbr_cols[2] - 1));
  return ld_peer(v.nbr[3] + i * v.nbr_pitch[3]);
}

// The first / last column of the rectangle when a left / right neighbour exists: one
// thread per 4 rows reads the neighbour's published column strip with one 16-byte
// NVLink load, computes the 4 cells and publishes them into its own strip for the
// next sweep.  These CTAs (launched after every tile) are the only ones that wait for
// the left / right neighbours; the tiles leave those cells to them.
constexpr int kStripRowsPerCta = 4 * kThreads;
#ifndef PM_STRIPS_FIRST
#define PM_STRIPS_FIRST 1
#endif

__device__ __noinline__ void column_strip(const pm_stencil_view& v, int sweep, int side, int blk) {
  if (threadIdx.x == 0 && sweep > 0) {
    for (int d = 0; d < 4; ++d)
      if (v.nbr[d]) wait_flag(v.my_flags + v.nbr_rank[d], sweep);
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blk * kStripRowsPerCta + 4 * threadIdx.x;
  if (i0 >= v.rows) return;
  const int64_t j = side ? v.cols - 1 : 0;
  const float4 nb = ld_peer4(v.nbr_col[side] + i0);  // the neighbour's adjacent column
  const float nbv[4] = {nb.x, nb.y, nb.z, nb.w};
  float res[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = i0 + q;
    if (i >= v.rows) break;
    const int64_t gi = v.grow0 + i;
    const float mid = __ldg(v.in + i * v.pitch + j);
    if (gi == 0 || gi == v.grows - 1) {
      res[q] = mid;  // Dirichlet row
    } else {
      const float up = fetch(v, i - 1, j), dn = fetch(v, i + 1, j);
      const float in_side = fetch(v, i, side ? j - 1 : j + 1);  // the inner neighbour
      res[q] = 0.25f * ((up + dn) + (nbv[q] + in_side));
    }
    v.out[i * v.pitch + j] = res[q];
  }
  float* pub = v.col_out[side];
  if (pub) {
    if (i0 + 4 <= v.rows) {
      *reinterpret_cast<float4*>(pub + i0) = make_float4(res[0], res[1], res[2], res[3]);
    } else {
      for (int q = 0; i0 + q < v.rows; ++q) pub[i0 + q] = res[q];
    }
  }
}

template <int TR>
__global__ void __launch_bounds__(kThreads, 5)
k_jacobi(const __grid_constant__ pm_stencil_view v, int sweep, int tiles_r, int tiles_c, int n_interior) {
  // column-strip CTAs first (few; they spin on the left / right flags at most while the
  // tiles stream, so the sweep has no serial tail), interior tiles next, edge tiles
  // last (index order = launch order)
  const int per = (int)((v.rows + kStripRowsPerCta - 1) / kStripRowsPerCta);
  const int nstrip = (v.nbr[2] ? per : 0) + (v.nbr[3] ? per : 0);
  const int b = PM_STRIPS_FIRST ? ((int)blockIdx.x - nstrip + (int)gridDim.x) % (int)gridDim.x
                                : (int)blockIdx.x;
  const int ntiles = tiles_r * tiles_c;
  const bool has_nbr = v.nbr[0] || v.nbr[1] || v.nbr[2] || v.nbr[3];
  if (has_nbr && blockIdx.x == 0 && threadIdx.x == 0 && sweep > 0) {
    // every CTA of sweep - 1 has finished: tell the neighbours
    __threadfence_system();
    for (int d = 0; d < 4; ++d)
      if (v.nbr[d]) st_release_sys(v.nbr_flag_slot[d], sweep);
  }
  if (b >= ntiles) {
    const int k = b - ntiles;
    const int side = (v.nbr[2] && k < per) ? 0 : 1;
    column_strip(v, sweep, side, (v.nbr[2] && k < per) ? k : k - (v.nbr[2] ? per : 0));
    return;
  }
  // middle tile rows in row-major order (the first / last tile column included: they
  // wait for nothing, and a tail of edge-column tiles alone hits few DRAM channels --
  // their segments are a power-of-two pitch apart), then the first and last tile rows
  // (which wait for the up / down neighbours)
  int tr, tc;
  if (b < n_interior) {  // n_interior = (tiles_r - 2) * tiles_c
    tr = 1 + b / tiles_c;
    tc = b % tiles_c;
  } else {
    const int e = b - n_interior;
    tr = e < tiles_c ? 0 : tiles_r - 1;
    tc = e < tiles_c ? e : e - tiles_c;
  }
  const bool edge_r0 = tr == 0, edge_r1 = tr == tiles_r - 1;
  const bool edge_c0 = tc == 0, edge_c1 = tc == tiles_c - 1;
  const bool interior = !(edge_r0 || edge_r1 || edge_c0 || edge_c1);
  if ((edge_r0 && v.nbr[0]) || (edge_r1 && v.nbr[1])) {
    // RAW: the first / last row tiles read the up / down neighbour's rows of sweep - 1
    // (the left / right columns are the strip CTAs')
    if (threadIdx.x == 0 && sweep > 0) {
      if (edge_r0 && v.nbr[0]) wait_flag(v.my_flags + v.nbr_rank[0], sweep);
      if (edge_r1 && v.nbr[1]) wait_flag(v.my_flags + v.nbr_rank[1], sweep);
    }
    __syncthreads();
  }
  // cells of a column a strip CTA computes (left / right neighbour present)
  const bool skip_x = v.nbr[2] != nullptr, skip_w = v.nbr[3] != nullptr;

  const int64_t r0 = (int64_t)tr * TR;
  const int64_t c = (int64_t)tc * TC + threadIdx.x * 4;
  if (!(edge_r0 || edge_r1) && (v.pitch & 3) == 0 && (v.cols & 3) == 0) {
    // rows r0-1 .. r0+TR all inside the rectangle and no Dirichlet row (only the
    // first / last row tiles can hold one): rolling float4 window, 8 rows of loads
    // in flight per thread (in/out never alias).  Interior tiles take every
    // neighbour locally; in the first / last column tile the thread at the
    // rectangle's left / right edge reads that column from the neighbour over
    // NVLink (or keeps a Dirichlet column of the global grid).
    if (c >= v.cols) return;
    const float* __restrict__ p = v.in + (r0 - 1) * v.pitch + c;
    float* __restrict__ po = v.out + r0 * v.pitch + c;
    const int64_t pitch = v.pitch;
    const bool left_edge = !interior && c == 0, right_edge = !interior && c + 4 == v.cols;
    const bool g_first = left_edge && v.gcol0 == 0;
    const bool g_last = right_edge && v.gcol0 + v.cols == v.gcols;
    const bool own_x = !(left_edge && skip_x), own_w = !(right_edge && skip_w);
    float4 up = __ldg(reinterpret_cast<const float4*>(p));
    float4 mid = __ldg(reinterpret_cast<const float4*>(p + pitch));
    for (int r8 = 0; r8 < TR; r8 += 8) {
      float4 dn[8];
      float lf[8], rt[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float* row = p + (int64_t)(r8 + u + 1) * pitch;
        dn[u] = __ldg(reinterpret_cast<const float4*>(row + pitch));
        lf[u] = left_edge ? 0.f : __ldg(row - 1);
        rt[u] = right_edge ? 0.f : __ldg(row + 4);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 o;
        o.x = 0.25f * ((up.x + dn[u].x) + (lf[u] + mid.y));
        o.y = 0.25f * ((up.y + dn[u].y) + (mid.x + mid.z));
        o.z = 0.25f * ((up.z + dn[u].z) + (mid.y + mid.w));
        o.w = 0.25f * ((up.w + dn[u].w) + (mid.z + rt[u]));
        if (g_first) o.x = mid.x;  // Dirichlet columns
        if (g_last) o.w = mid.w;
        float* dst = po + (int64_t)(r8 + u) * pitch;
        if (own_x && own_w) {
          __stcs(reinterpret_cast<float4*>(dst), o);
        } else {  // the strip CTA writes the neighbour-facing cell
          if (own_x) dst[0] = o.x;
          dst[1] = o.y;
          dst[2] = o.z;
          if (own_w) dst[3] = o.w;
        }
        up = mid;
        mid = dn[u];
      }
    }
  } else if ((v.pitch & 3) == 0 && c + 4 <= v.cols) {
    // edge tile, full vector: same rolling window, rows / columns just outside
    // the rectangle come from the neighbours over NVLink
    auto row4 = [&](int64_t i) -> float4 {
      if (i >= 0 && i < v.rows) return *reinterpret_cast<const float4*>(v.in + i * v.pitch + c);
      const float* q = nullptr;
      if (i < 0 && v.nbr[0]) q = v.nbr[0] + (v.nbr_rows[0] - 1) * v.nbr_pitch[0] + c;
      if (i >= v.rows && v.nbr[1]) q = v.nbr[1] + c;
      if (!q) return make_float4(0.f, 0.f, 0.f, 0.f);  // global boundary: unused
      return ld_peer4(q);  // 16-byte aligned: pitch % 4 == 0 on every GPU, c % 4 == 0
    };
    const bool own_x = !(c == 0 && skip_x), own_w = !(c + 4 == v.cols && skip_w);
    const int64_t r1 = min(r0 + TR, v.rows);
    float4 up = row4(r0 - 1), mid = row4(r0);
    const bool g_first = v.gcol0 + c == 0, g_last = v.gcol0 + c + 3 == v.gcols - 1;
    for (int64_t i8 = r0; i8 < r1; i8 += 8) {
      // issue the batch's loads first (peer loads included) so their NVLink
      // latencies overlap instead of serialising row by row
      float4 dn[8];
      float lf[8], rt[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = i8 + u;
        dn[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        lf[u] = rt[u] = 0.f;
        if (i >= r1) continue;
        dn[u] = row4(i + 1);
        if (c > 0) lf[u] = __ldg(v.in + i * v.pitch + c - 1);
        if (c + 4 < v.cols) rt[u] = __ldg(v.in + i * v.pitch + c + 4);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = i8 + u;
        if (i >= r1) break;
        float4 o;
        o.x = 0.25f * ((up.x + dn[u].x) + (lf[u] + mid.y));
        o.y = 0.25f * ((up.y + dn[u].y) + (mid.x + mid.z));
        o.z = 0.25f * ((up.z + dn[u].z) + (mid.y + mid.w));
        o.w = 0.25f * ((up.w + dn[u].w) + (mid.z + rt[u]));
        const int64_t gi = v.grow0 + i;
        if (gi == 0 || gi == v.grows - 1) {
          o = mid;  // Dirichlet rows
        } else {
          if (g_first) o.x = mid.x;  // Dirichlet columns
          if (g_last) o.w = mid.w;
        }
        float* dst = v.out + i * v.pitch + c;
        if (own_x && own_w) {
          __stcs(reinterpret_cast<float4*>(dst), o);
        } else {  // the strip CTA writes the neighbour-facing cell
          if (own_x) dst[0] = o.x;
          dst[1] = o.y;
          dst[2] = o.z;
          if (own_w) dst[3] = o.w;
        }
        up = mid;
        mid = dn[u];
      }
    }
  } else if (c < v.cols) {
    const int64_t r1 = min(r0 + TR, v.rows);
    const bool vec = (c + 4 <= v.cols) && ((v.pitch & 3) == 0);
    for (int64_t i = r0; i < r1; ++i) {
      const int64_t gi = v.grow0 + i;
      float res[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t j = c + q;
        if (j >= v.cols) { res[q] = 0.f; continue; }
        if ((j == 0 && skip_x) || (j == v.cols - 1 && skip_w)) {  // a strip CTA's cell
          res[q] = __int_as_float(0x7fc00000);
          continue;
        }
        const int64_t gj = v.gcol0 + j;
        if (gi == 0 || gj == 0 || gi == v.grows - 1 || gj == v.gcols - 1) {
          res[q] = __ldg(v.in + i * v.pitch + j);  // Dirichlet boundary
        } else {
          const float up = fetch(v, i - 1, j), dn = fetch(v, i + 1, j);
          const float lf = fetch(v, i, j - 1), rt = fetch(v, i, j + 1);
          res[q] = 0.25f * ((up + dn) + (lf + rt));
        }
      }
      float* o = v.out + i * v.pitch + c;
      const bool strip_cell = (c == 0 && skip_x) || (c + 4 >= v.cols && skip_w);
      if (vec && !strip_cell) {
        *reinterpret_cast<float4*>(o) = make_float4(res[0], res[1], res[2], res[3]);
      } else {
        for (int q = 0; q < 4 && c + q < v.cols; ++q)
          if (!((c + q == 0 && skip_x) || (c + q == v.cols - 1 && skip_w))) o[q] = res[q];
      }
    }
  }
}

}  // namespace
}  // namespace pm

extern "C" int pm_stencil_sweep(const pm_stencil_view* v, int32_t sweep, void* stream) {
  if (!v || !v->in || !v->out || v->rows <= 0 || v->cols <= 0 || v->pitch < v->cols || sweep < 0)
    return pm::set_error("pm_stencil_sweep: bad view"), PM_ERR_INVALID;
  static int tr_env = [] {
    const char* e = getenv("PM_STENCIL_TR");
    return e ? atoi(e) : 16;
  }();
  const int TR = (tr_env == 32 || tr_env == 64 || tr_env == 128) ? tr_env : 16;
  const int tiles_r = (int)((v->rows + TR - 1) / TR);
  const int tiles_c = (int)((v->cols + pm::TC - 1) / pm::TC);
  const int n_interior = std::max(tiles_r - 2, 0) * tiles_c;
  const int per = (int)((v->rows + pm::kStripRowsPerCta - 1) / pm::kStripRowsPerCta);
  if ((v->nbr[2] && !v->nbr_col[0]) || (v->nbr[3] && !v->nbr_col[1]) ||
      (((uintptr_t)v->nbr_col[0] | (uintptr_t)v->nbr_col[1] | (uintptr_t)v->col_out[0] |
        (uintptr_t)v->col_out[1]) & 15))
    return pm::set_error("pm_stencil_sweep: left / right neighbours need 16-byte aligned "
                         "column strips"), PM_ERR_INVALID;
  const int total = tiles_r * tiles_c + (v->nbr[2] ? per : 0) + (v->nbr[3] ? per : 0);
  cudaStream_t s = (cudaStream_t)stream;
  switch (TR) {
    case 16: pm::k_jacobi<16><<<total, pm::kThreads, 0, s>>>(*v, sweep, tiles_r, tiles_c, n_interior); break;
    case 32: pm::k_jacobi<32><<<total, pm::kThreads, 0, s>>>(*v, sweep, tiles_r, tiles_c, n_interior); break;
    case 128: pm::k_jacobi<128><<<total, pm::kThreads, 0, s>>>(*v, sweep, tiles_r, tiles_c, n_interior); break;
    default: pm::k_jacobi<64><<<total, pm::kThreads, 0, s>>>(*v, sweep, tiles_r, tiles_c, n_interior); break;
  }
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}
