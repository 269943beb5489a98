// K6 -- circuit simulation (the paper's Circuit workload, PAPER.md:495,
// after Bauer et al. 2012 / the Legion circuit example) with the node
// exchange fused into the kernels over NVLink.
//
// A piece of the circuit (its nodes and the wires whose in-node it owns) lives
// on the GPU its Mapple mapping assigns it to.  A wire's out-node may belong
// to a piece on another GPU: its voltage is read and its charge deposited
// directly in that GPU's memory through CUDA IPC pointers (peer loads and
// peer float atomics over NVLink), so there is no ghost-copy pass and no
// separate reduction -- the "halo" is exactly the cross-GPU wires.
//
//   k_circuit_wires  (calc_new_currents + distribute_charge)  one thread per
//                    wire; `steps` fixed-point iterations of the implicit
//                    segment update in registers (FP32-pipe bound), then the
//                    two charge deposits
//   k_circuit_nodes  (update_voltages)  one thread per local node
//
// Node references are int32: (rank << 27) | slot in that rank's node arrays.

#include <cuda_runtime.h>

#include <cstdint>

#include "pm_common.h"

namespace pm {
namespace {

constexpr int kSeg = PM_CIRCUIT_SEGMENTS;

struct CircuitArgs {
  pm_circuit_view v;
};

__device__ __forceinline__ float* node_ptr(float* const* tab, int ref) {
  return tab[(unsigned)ref >> 27] + (ref & ((1 << 27) - 1));
}

#ifndef PM_CIRCUIT_MINB
#define PM_CIRCUIT_MINB 8  // 64 registers: 8 CTAs / SM (measured 3.16 -> 2.96 ms per iteration)
#endif
#ifndef PM_CIRCUIT_UNROLL
#define PM_CIRCUIT_UNROLL 1
#endif
#define PM_STR2(x) #x
#define PM_STR(x) PM_STR2(x)

__global__ void __launch_bounds__(128, PM_CIRCUIT_MINB)
k_circuit_wires(const __grid_constant__ CircuitArgs a) {
  const pm_circuit_view& v = a.v;
  const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= v.n_wires) return;
  const long long nw = v.n_wires;
  const int in_ref = v.in_ref[w], out_ref = v.out_ref[w];
  const float rdt = 1.0f / v.dt, dt = v.dt;
  const float L = v.inductance[w];
  const float rR = 1.0f / v.resistance[w];
  const float rC = 1.0f / v.capacitance[w];
  float tv[kSeg + 1], ov[kSeg + 1], ti[kSeg], oi[kSeg];
  tv[0] = ov[0] = *node_ptr(v.volt, in_ref);
  tv[kSeg] = ov[kSeg] = *node_ptr(v.volt, out_ref);
#pragma unroll
  for (int s = 0; s < kSeg - 1; ++s) tv[s + 1] = ov[s + 1] = v.wire_volt[s * nw + w];
#pragma unroll
  for (int s = 0; s < kSeg; ++s) ti[s] = oi[s] = v.current[s * nw + w];
  // dV = R I + L dI/dt  =>  I = (dV - L (I - I_old) / dt) / R
  //                        = dV / R + kr I_old - kr I,  kr = L / (dt R)
  // V_seg = V_seg_old + dt (I_in - I_out) / C
  // rearranged so one step is 10 x (FADD + 2 FFMA) + 9 x (FADD + FFMA) = 48 FP32 ops
  const float kr = L * rdt * rR;
  const float dtrC = dt * rC;
  float ci[kSeg];
#pragma unroll
  for (int s = 0; s < kSeg; ++s) ci[s] = kr * oi[s];
  _Pragma(PM_STR(unroll PM_CIRCUIT_UNROLL))
  for (int it = 0; it < v.steps; ++it) {
#pragma unroll
    for (int s = 0; s < kSeg; ++s) ti[s] = fmaf(tv[s + 1] - tv[s], rR, fmaf(-kr, ti[s], ci[s]));
#pragma unroll
    for (int s = 0; s < kSeg - 1; ++s) tv[s + 1] = fmaf(dtrC, ti[s] - ti[s + 1], ov[s + 1]);
  }
#pragma unroll
  for (int s = 0; s < kSeg; ++s) v.current[s * nw + w] = ti[s];
#pragma unroll
  for (int s = 0; s < kSeg - 1; ++s) v.wire_volt[s * nw + w] = tv[s + 1];
  // distribute_charge: straight into the owning GPU's charge array
  atomicAdd(node_ptr(v.charge, in_ref), -dt * ti[0]);
  atomicAdd(node_ptr(v.charge, out_ref), dt * ti[kSeg - 1]);
}

__global__ void __launch_bounds__(256)
k_circuit_nodes(const __grid_constant__ CircuitArgs a) {
  const pm_circuit_view& v = a.v;
  const int rank = v.rank;
  float* volt = v.volt[rank];
  float* charge = v.charge[rank];
  for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < v.n_nodes;
       n += (long long)gridDim.x * blockDim.x) {
    const float c = charge[n];
    volt[n] = (volt[n] + c / v.node_cap[n]) * (1.0f - v.leakage[n]);
    charge[n] = 0.0f;
  }
}

}  // namespace
}  // namespace pm

extern "C" {

int pm_circuit_step(const pm_circuit_view* view, int32_t phase, void* stream) {
  if (!view || view->rank < 0 || view->rank >= PM_CIRCUIT_MAX_RANKS || view->n_wires < 0 ||
      view->n_nodes < 0 || view->steps < 0 || !(view->dt > 0.0f))
    return pm::set_error("pm_circuit_step: bad view"), PM_ERR_INVALID;
  if (view->n_nodes >= (1LL << 27))
    return pm::set_error("pm_circuit_step: > 2^27 nodes per GPU"), PM_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  pm::CircuitArgs a{*view};
  if (phase == 0) {
    if (view->n_wires == 0) return PM_OK;
    const long long blocks = (view->n_wires + 127) / 128;
    pm::k_circuit_wires<<<(unsigned)blocks, 128, 0, s>>>(a);
  } else if (phase == 1) {
    if (view->n_nodes == 0) return PM_OK;
    long long blocks = (view->n_nodes + 255) / 256;
    const long long cap = (long long)pm::num_sms() * 8;
    if (blocks > cap) blocks = cap;
    pm::k_circuit_nodes<<<(unsigned)blocks, 256, 0, s>>>(a);
  } else {
    return pm::set_error("pm_circuit_step: phase 0 (wires) or 1 (nodes)"), PM_ERR_INVALID;
  }
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

}  // extern "C"
