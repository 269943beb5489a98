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
// Cross-GPU ordering, per neighbour (flags pushed into the reader's memory; flag =
// sweeps the writer has completed):
//   publish  sweep s's kernel starts only after all CTAs of sweep s-1 finished
//            (stream order), so its first CTA publishes "s sweeps done" with a
//            system-scope release store into each neighbour's flag slot -- no
//            per-CTA ticket atomics or fences;
//   RAW      a tile touching my rectangle's edge waits until that neighbour
//            has published s (finished sweep s-1); interior tiles never wait;
//   WAR      with three rotating buffers a neighbour reads the buffer I write
//            at sweep s during its sweep s-2.  My sweep s-1 edge tiles on that
//            side already waited for the neighbour's flag >= s-1, i.e. for its
//            sweep s-2 to finish, so the WAR order is implied and not checked.
// Tiles are launched interior-first so edge tiles usually find the flag set.
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

template <int TR>
__global__ void __launch_bounds__(kThreads)
k_jacobi(const pm_stencil_view v, int sweep, int tiles_r, int tiles_c, int n_interior) {
  // interior tiles first, edge tiles last (block index order = launch order)
  const int b = blockIdx.x;
  int tr, tc;
  if (b < n_interior) {
    const int ic = tiles_c - 2;
    tr = 1 + b / ic;
    tc = 1 + b % ic;
  } else {
    // the ring of edge tiles: top row, bottom row, then left/right of the rest
    int e = b - n_interior;
    const int per_mid = tiles_c > 1 ? 2 : 1;
    if (e < tiles_c) {
      tr = 0;
      tc = e;
    } else if (tiles_r > 1 && e < 2 * tiles_c) {
      tr = tiles_r - 1;
      tc = e - tiles_c;
    } else {
      e -= (tiles_r > 1 ? 2 : 1) * tiles_c;
      tr = 1 + e / per_mid;
      tc = (e % per_mid == 0) ? 0 : tiles_c - 1;
    }
  }
  const bool edge_r0 = tr == 0, edge_r1 = tr == tiles_r - 1;
  const bool edge_c0 = tc == 0, edge_c1 = tc == tiles_c - 1;
  const bool interior = !(edge_r0 || edge_r1 || edge_c0 || edge_c1);
  const bool has_nbr = v.nbr[0] || v.nbr[1] || v.nbr[2] || v.nbr[3];
  if (has_nbr && b == 0 && threadIdx.x == 0 && sweep > 0) {
    // every CTA of sweep - 1 has finished: tell the neighbours
    __threadfence_system();
    for (int d = 0; d < 4; ++d)
      if (v.nbr[d]) st_release_sys(v.nbr_flag_slot[d], sweep);
  }
  if (!interior && has_nbr) {
    // RAW: edge tiles read neighbour cells produced by their sweep - 1
    if (threadIdx.x == 0) {
      const bool need[4] = {edge_r0, edge_r1, edge_c0, edge_c1};
      for (int d = 0; d < 4; ++d)
        if (v.nbr[d] && need[d]) wait_flag(v.my_flags + v.nbr_rank[d], sweep);
    }
    __syncthreads();
  }

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
    const float* pl = left_edge && v.nbr[2]
                          ? v.nbr[2] + r0 * v.nbr_pitch[2] + (v.nbr_cols[2] - 1) : nullptr;
    const float* pr = right_edge && v.nbr[3] ? v.nbr[3] + r0 * v.nbr_pitch[3] : nullptr;
    const bool g_first = left_edge && v.gcol0 == 0;
    const bool g_last = right_edge && v.gcol0 + v.cols == v.gcols;
    float4 up = __ldg(reinterpret_cast<const float4*>(p));
    float4 mid = __ldg(reinterpret_cast<const float4*>(p + pitch));
    for (int r8 = 0; r8 < TR; r8 += 8) {
      float4 dn[8];
      float lf[8], rt[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float* row = p + (int64_t)(r8 + u + 1) * pitch;
        dn[u] = __ldg(reinterpret_cast<const float4*>(row + pitch));
        lf[u] = left_edge ? (pl ? ld_peer(pl + (int64_t)(r8 + u) * v.nbr_pitch[2]) : 0.f)
                          : __ldg(row - 1);
        rt[u] = right_edge ? (pr ? ld_peer(pr + (int64_t)(r8 + u) * v.nbr_pitch[3]) : 0.f)
                           : __ldg(row + 4);
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
        __stcs(reinterpret_cast<float4*>(po + (int64_t)(r8 + u) * pitch), o);
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
      return make_float4(ld_peer(q), ld_peer(q + 1), ld_peer(q + 2), ld_peer(q + 3));
    };
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
        else if (v.nbr[2]) lf[u] = ld_peer(v.nbr[2] + i * v.nbr_pitch[2] + (v.nbr_cols[2] - 1));
        if (c + 4 < v.cols) rt[u] = __ldg(v.in + i * v.pitch + c + 4);
        else if (v.nbr[3]) rt[u] = ld_peer(v.nbr[3] + i * v.nbr_pitch[3]);
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
        __stcs(reinterpret_cast<float4*>(v.out + i * v.pitch + c), o);
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
      if (vec) {
        *reinterpret_cast<float4*>(o) = make_float4(res[0], res[1], res[2], res[3]);
      } else {
        for (int q = 0; q < 4 && c + q < v.cols; ++q) o[q] = res[q];
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
  const int n_interior = std::max(tiles_r - 2, 0) * std::max(tiles_c - 2, 0);
  const int total = tiles_r * tiles_c;
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
