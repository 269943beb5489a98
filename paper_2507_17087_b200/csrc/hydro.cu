// K7 -- PENNANT-style Lagrangian staggered-grid hydrodynamics (the paper's
// PENNANT workload, after Ferenbaugh 2015) on an unstructured
// quadrilateral mesh, with the shared-point exchange fused over NVLink.
//
// Zones are placed by a Mapple mapping of the zone launch; each point belongs
// to one GPU.  A zone reads its 4 points' positions and velocities through
// per-rank pointer tables (peer loads over NVLink for points owned by another
// GPU) and deposits its corner forces with 8-byte float2 atomics straight into the
// owning GPU's force array -- Legion PENNANT's master/ghost point exchange
// and its point-force reduction become the cross-GPU corners of the zone
// kernel, with no copy pass.
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

#include "pm_common.h"

namespace pm {
namespace {

struct HydroArgs {
  pm_hydro_view v;
};

__device__ __forceinline__ int rk(int ref) { return (int)((unsigned)ref >> 27); }
__device__ __forceinline__ int sl(int ref) { return ref & ((1 << 27) - 1); }

__global__ void __launch_bounds__(256)
k_hydro_zones(const __grid_constant__ HydroArgs a) {
  const pm_hydro_view& v = a.v;
  const long long z = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nz = v.n_zones;
  if (z >= nz) return;
  int ref[4];
  float x[4], y[4], u[4], w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) ref[k] = __ldg(v.z2p + k * nz + z);
  // point state is read-only during this phase (also on the peers): non-coherent loads
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = rk(ref[k]), s = sl(ref[k]);
    x[k] = __ldg(v.px[r] + s);
    y[k] = __ldg(v.py[r] + s);
    u[k] = __ldg(v.ux[r] + s);
    w[k] = __ldg(v.uy[r] + s);
  }
  float area = 0.f, dadt = 0.f;
  float nx[4], ny[4];  // edge k (point k -> k+1) outward normal scaled by its length
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int k1 = (k + 1) & 3;
    area += x[k] * y[k1] - x[k1] * y[k];
    nx[k] = y[k1] - y[k];
    ny[k] = x[k] - x[k1];
    dadt += (u[k] + u[k1]) * nx[k] + (w[k] + w[k1]) * ny[k];
  }
  area *= 0.5f;
  dadt *= 0.5f;
  const float zm = __ldg(v.zm + z);
  // PdV work of the last step's pressure over this step's volume change
  const float e = v.ze[z] - v.zpe[z] * (area - v.za[z]) / zm;
  const float rho = zm / area;
  const float p = (v.gamma - 1.0f) * rho * e;
  const float q = dadt < 0.f ? v.cq * rho * dadt * dadt / area : 0.f;
  const float pe = p + q;
  v.ze[z] = e;
  v.za[z] = area;
  v.zpe[z] = pe;
  // corner force of point k = half of each adjacent edge's pressure force, deposited
  // in the owner's memory: one 8-byte vector atomic (sm_90+ float2 atomicAdd) into
  // this GPU's points; two 4-byte float atomics -- the form NVLink peer atomics
  // natively support -- into a peer's
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int km = (k + 3) & 3;
    const int r = rk(ref[k]), s = sl(ref[k]);
    const float fx = 0.5f * pe * (nx[km] + nx[k]), fy = 0.5f * pe * (ny[km] + ny[k]);
    if (r == v.rank) {
      atomicAdd(reinterpret_cast<float2*>(v.fxy[r]) + s, make_float2(fx, fy));
    } else {
      atomicAdd(v.fxy[r] + 2 * s, fx);
      atomicAdd(v.fxy[r] + 2 * s + 1, fy);
    }
  }
}

__global__ void __launch_bounds__(256)
k_hydro_points(const __grid_constant__ HydroArgs a) {
  const pm_hydro_view& v = a.v;
  const int me = v.rank;
  float *px = v.px[me], *py = v.py[me], *ux = v.ux[me], *uy = v.uy[me];
  float2* f = reinterpret_cast<float2*>(v.fxy[me]);
  const float dt = v.dt;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // four points per thread: 16-byte loads / stores of every array (all base
  // pointers are 16-byte aligned allocations; the tail goes point by point)
  const long long nv = v.n_points >> 2;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nv; g += stride) {
    const float4 m4 = __ldg(reinterpret_cast<const float4*>(v.pm) + g);
    const char4 b4 = __ldg(reinterpret_cast<const char4*>(v.pbc) + g);
    const float4 fa = reinterpret_cast<const float4*>(f)[2 * g];      // fx0 fy0 fx1 fy1
    const float4 fb = reinterpret_cast<const float4*>(f)[2 * g + 1];  // fx2 fy2 fx3 fy3
    float4 u = reinterpret_cast<float4*>(ux)[g], w = reinterpret_cast<float4*>(uy)[g];
    float4 x = reinterpret_cast<float4*>(px)[g], y = reinterpret_cast<float4*>(py)[g];
    const float fxs[4] = {fa.x, fa.z, fb.x, fb.z}, fys[4] = {fa.y, fa.w, fb.y, fb.w};
    const float ms[4] = {m4.x, m4.y, m4.z, m4.w};
    const int bcs[4] = {b4.x, b4.y, b4.z, b4.w};
    float* uu = &u.x;
    float* ww = &w.x;
    float* xx = &x.x;
    float* yy = &y.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float rm = 1.0f / ms[j];
      const float ax = (bcs[j] & 1) ? 0.f : fxs[j] * rm;
      const float ay = (bcs[j] & 2) ? 0.f : fys[j] * rm;
      const float u1 = uu[j] + dt * ax, w1 = ww[j] + dt * ay;
      xx[j] += dt * 0.5f * (uu[j] + u1);
      yy[j] += dt * 0.5f * (ww[j] + w1);
      uu[j] = u1;
      ww[j] = w1;
    }
    reinterpret_cast<float4*>(ux)[g] = u;
    reinterpret_cast<float4*>(uy)[g] = w;
    reinterpret_cast<float4*>(px)[g] = x;
    reinterpret_cast<float4*>(py)[g] = y;
    reinterpret_cast<float4*>(f)[2 * g] = make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(f)[2 * g + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long n = 4 * nv + (long long)blockIdx.x * blockDim.x + threadIdx.x; n < v.n_points;
       n += stride) {
    const float rm = 1.0f / v.pm[n];
    const int bc = v.pbc[n];
    const float2 fn = f[n];
    float ax = fn.x * rm, ay = fn.y * rm;
    if (bc & 1) ax = 0.f;
    if (bc & 2) ay = 0.f;
    const float u0 = ux[n], w0 = uy[n];
    const float u1 = u0 + dt * ax, w1 = w0 + dt * ay;
    px[n] += dt * 0.5f * (u0 + u1);
    py[n] += dt * 0.5f * (w0 + w1);
    ux[n] = u1;
    uy[n] = w1;
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
    pm::k_hydro_zones<<<(unsigned)((view->n_zones + 255) / 256), 256, 0, s>>>(a);
  } else if (phase == 1) {
    if (view->n_points == 0) return PM_OK;
    long long blocks = (view->n_points / 4 + 255) / 256 + 1;
    const long long cap = (long long)pm::num_sms() * 8;
    if (blocks > cap) blocks = cap;
    pm::k_hydro_points<<<(unsigned)blocks, 256, 0, s>>>(a);
  } else {
    return pm::set_error("pm_hydro_step: phase 0 (zones) or 1 (points)"), PM_ERR_INVALID;
  }
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

}  // extern "C"
