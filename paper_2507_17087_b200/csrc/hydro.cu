// K7 -- PENNANT-style Lagrangian staggered-grid hydrodynamics (the paper's
// PENNANT workload, after Ferenbaugh 2015) on an unstructured
// quadrilateral mesh, with the shared-point exchange fused over NVLink.
//
// Zones are placed by a Mapple mapping of the zone launch; each point belongs
// to one GPU.  A zone reads its 4 points' state -- (x, y, u, v), one 16-byte
// record per point -- through per-rank pointer tables (peer loads over NVLink for
// points owned by another GPU) and deposits its corner forces with 8-byte float2 atomics straight into the
// owning GPU's force array -- Legion PENNANT's master/ghost point exchange
// and its point-force reduction become the cross-GPU corners of the zone
// kernel, with no copy pass.  Corners shared by consecutive zones of a warp are summed
// with shuffles first (about 2 atomics per zone on a row-numbered mesh).
//
//   k_hydro_zones   one thread per zone: area (shoelace), PdV energy update
//                   with the previous step's pressure, EOS (gamma-law gas),
//                   artificial viscosity q = cq rho (dA/dt)^2 / A under
//                   compression, edge pressure forces -> 4 corner forces
//   k_hydro_points  one thread per local point: a = F / m, wall boundary
//                   conditions, velocity / position update, force reset
//
// Point references are int32: (rank << 27) | slot.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "pm_common.h"

namespace pm {
namespace {

struct HydroArgs {
  pm_hydro_view v;
};

__device__ __forceinline__ int rk(int ref) { return (int)((unsigned)ref >> 27); }
__device__ __forceinline__ int sl(int ref) { return ref & ((1 << 27) - 1); }

// one zone: area, PdV energy update, EOS, artificial viscosity and the 4 corner forces
// (st[k]: the (x, y, u, v) of the zone's point k; f[k]: point k's corner force)
__device__ __forceinline__ void hydro_zone(const pm_hydro_view& v, const float4 (&st)[4],
                                           float zm, float ze, float za, float zpe,
                                           float2 (&f)[4], float& e_out, float& a_out,
                                           float& pe_out) {
  float area = 0.f, dadt = 0.f;
  float nx[4], ny[4];  // edge k (point k -> k+1) outward normal scaled by its length
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int k1 = (k + 1) & 3;
    area += st[k].x * st[k1].y - st[k1].x * st[k].y;
    nx[k] = st[k1].y - st[k].y;
    ny[k] = st[k].x - st[k1].x;
    dadt += (st[k].z + st[k1].z) * nx[k] + (st[k].w + st[k1].w) * ny[k];
  }
  area *= 0.5f;
  dadt *= 0.5f;
  // PdV work of the last step's pressure over this step's volume change
  const float e = ze - zpe * (area - za) / zm;
  const float rho = zm / area;
  const float p = (v.gamma - 1.0f) * rho * e;
  const float q = dadt < 0.f ? v.cq * rho * dadt * dadt / area : 0.f;
  const float pe = p + q;
  e_out = e;
  a_out = area;
  pe_out = pe;
  // corner force of point k = half of each adjacent edge's pressure force
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int km = (k + 3) & 3;
    f[k] = make_float2(0.5f * pe * (nx[km] + nx[k]), 0.5f * pe * (ny[km] + ny[k]));
  }
}

// deposit a corner force in the owner's memory: one 8-byte vector atomic (sm_90+ float2
// atomicAdd) into this GPU's points; two 4-byte float atomics -- the form NVLink peer
// atomics natively support -- into a peer's
__device__ __forceinline__ void deposit(const pm_hydro_view& v, int ref, float2 f) {
  const int r = rk(ref), s = sl(ref);
  if (r == v.rank) {
    atomicAdd(reinterpret_cast<float2*>(v.fxy[r]) + s, f);
  } else {
    atomicAdd(v.fxy[r] + 2 * s, f.x);
    atomicAdd(v.fxy[r] + 2 * s + 1, f.y);
  }
}

__device__ __forceinline__ float4 point_state(const pm_hydro_view& v, int ref) {
  // point state is read-only during this phase (also on the peers): one 16-byte
  // non-coherent load of (x, y, u, v)
  return __ldg(reinterpret_cast<const float4*>(v.pst[rk(ref)]) + sl(ref));
}

#ifndef PM_HYDRO_WARP_COMBINE
#define PM_HYDRO_WARP_COMBINE 1
#endif

// One zone per thread.  Consecutive zones of a row share an edge: corners 1 and 2 of
// zone z are corners 0 and 3 of zone z + 1 whenever the mesh numbers zones along rows
// (checked per pair at run time, so any z2p is handled).  Each lane hands its corners
// 1 / 2 to the next lane, which adds them to its corners 0 / 3 when the point refs
// match: about 2 force atomics per zone instead of 4 on the L2 atomic units.
__global__ void __launch_bounds__(256)
k_hydro_zones(const __grid_constant__ HydroArgs a) {
  const pm_hydro_view& v = a.v;
  const long long z = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nz = v.n_zones;
  const bool live = z < nz;
#if !PM_HYDRO_WARP_COMBINE
  if (!live) return;
#endif
  int ref[4] = {-1, -1, -1, -1};
  float2 f[4];
  if (live) {
    float4 st[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) ref[k] = __ldg(v.z2p + k * nz + z);
#pragma unroll
    for (int k = 0; k < 4; ++k) st[k] = point_state(v, ref[k]);
    float e, ar, pe;
    hydro_zone(v, st, __ldg(v.zm + z), v.ze[z], v.za[z], v.zpe[z], f, e, ar, pe);
    v.ze[z] = e;
    v.za[z] = ar;
    v.zpe[z] = pe;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) f[k] = make_float2(0.f, 0.f);
  }
#if PM_HYDRO_WARP_COMBINE
  const unsigned all = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int r1 = __shfl_up_sync(all, ref[1], 1), r2 = __shfl_up_sync(all, ref[2], 1);
  const float g1x = __shfl_up_sync(all, f[1].x, 1), g1y = __shfl_up_sync(all, f[1].y, 1);
  const float g2x = __shfl_up_sync(all, f[2].x, 1), g2y = __shfl_up_sync(all, f[2].y, 1);
  const bool take0 = live && lane > 0 && r1 == ref[0];
  const bool take3 = live && lane > 0 && r2 == ref[3];
  if (take0) f[0].x += g1x, f[0].y += g1y;
  if (take3) f[3].x += g2x, f[3].y += g2y;
  const bool gave1 = __shfl_down_sync(all, take0, 1) && lane < 31;
  const bool gave2 = __shfl_down_sync(all, take3, 1) && lane < 31;
  if (!live) return;
  deposit(v, ref[0], f[0]);
  if (!gave1) deposit(v, ref[1], f[1]);
  if (!gave2) deposit(v, ref[2], f[2]);
  deposit(v, ref[3], f[3]);
#else
#pragma unroll
  for (int k = 0; k < 4; ++k) deposit(v, ref[k], f[k]);
#endif
}

__device__ __forceinline__ float4 hydro_move(float4 q, float2 f, float m, int bc, float dt) {
  const float rm = 1.0f / m;
  const float ax = (bc & 1) ? 0.f : f.x * rm;
  const float ay = (bc & 2) ? 0.f : f.y * rm;
  const float u1 = q.z + dt * ax, w1 = q.w + dt * ay;
  return make_float4(q.x + dt * 0.5f * (q.z + u1), q.y + dt * 0.5f * (q.w + w1), u1, w1);
}

__global__ void __launch_bounds__(256)
k_hydro_points(const __grid_constant__ HydroArgs a) {
  const pm_hydro_view& v = a.v;
  const int me = v.rank;
  float4* st = reinterpret_cast<float4*>(v.pst[me]);
  float2* f = reinterpret_cast<float2*>(v.fxy[me]);
  const float dt = v.dt;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // two points per thread: 16-byte accesses to every array but the masses (8 bytes) and
  // the wall flags (2 bytes); the tail goes point by point
  const long long nv = v.n_points >> 1;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nv; g += stride) {
    const float2 m2 = __ldg(reinterpret_cast<const float2*>(v.pm) + g);
    const char2 b2 = __ldg(reinterpret_cast<const char2*>(v.pbc) + g);
    const float4 ff = __ldcs(reinterpret_cast<const float4*>(f) + g);  // fx0 fy0 fx1 fy1
    const float4 q0 = st[2 * g], q1 = st[2 * g + 1];
    st[2 * g] = hydro_move(q0, make_float2(ff.x, ff.y), m2.x, b2.x, dt);
    st[2 * g + 1] = hydro_move(q1, make_float2(ff.z, ff.w), m2.y, b2.y, dt);
    reinterpret_cast<float4*>(f)[g] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long n = 2 * nv + (long long)blockIdx.x * blockDim.x + threadIdx.x; n < v.n_points;
       n += stride) {
    st[n] = hydro_move(st[n], f[n], v.pm[n], v.pbc[n], dt);
    f[n] = make_float2(0.f, 0.f);
  }
}

}  // namespace
}  // namespace pm

extern "C" {

int pm_hydro_step(const pm_hydro_view* view, int32_t phase, void* stream) {
  if (!view || view->rank < 0 || view->rank >= PM_HYDRO_MAX_RANKS || view->n_zones < 0 ||
      view->n_points < 0 || !(view->dt > 0.0f))
    return pm::set_error("pm_hydro_step: bad view"), PM_ERR_INVALID;
  if (view->n_points >= (1LL << 27))
    return pm::set_error("pm_hydro_step: > 2^27 points per GPU"), PM_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  pm::HydroArgs a{*view};
  if (phase == 0) {
    if (view->n_zones == 0) return PM_OK;
    // one zone per thread (two per thread, with vector zone loads and eight gathers in
    // flight, was slower: 1.21 vs 0.96 ms at 67M zones)
    // (two vertically stacked zones per thread over a row-pair zone numbering -- 6 gathers
    // and 1.5 atomics per zone -- measured slower: 1.10 vs 0.92 ms, tools/hydro_ab2.sh)
    pm::k_hydro_zones<<<(unsigned)((view->n_zones + 255) / 256), 256, 0, s>>>(a);
  } else if (phase == 1) {
    if (view->n_points == 0) return PM_OK;
    // one thread per two points, no grid-stride persistence (0.53 vs 0.61 ms at 67M
    // points with 8 CTAs per SM looping)
    long long blocks = (view->n_points / 2 + 255) / 256 + 1;
    if (const char* c = getenv("PM_HYDRO_POINT_CTAS"))
      if (atoll(c) > 0 && atoll(c) < blocks) blocks = atoll(c);
    if (blocks > 0x7FFFFFFFLL) blocks = 0x7FFFFFFFLL;
    pm::k_hydro_points<<<(unsigned)blocks, 256, 0, s>>>(a);
  } else {
    return pm::set_error("pm_hydro_step: phase 0 (zones) or 1 (points)"), PM_ERR_INVALID;
  }
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

}  // extern "C"
