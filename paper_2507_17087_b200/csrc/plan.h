// Internal: the loaded form of a point program (pm_plan).
#pragma once

#include <mutex>
#include <string>

#include "pm_common.h"

struct pm_plan {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;  // pm_map_points (K1)
  int n_coords = 0;
  int implicit = 0;
  int device = 0;
  int n_regs = 0;
  std::string src;          // generated K1 source (the fused module extends it)
  std::string probe_src;    // failure probe (pm_map_probe), compiled on first use
  CUmodule probe_mod = nullptr;
  CUfunction probe_fn = nullptr;
  // fused map + partition kernels (K1 + K2 in two passes), built on first use
  std::mutex fused_mu;
  bool fused_ready = false;
  CUmodule fused_mod = nullptr;
  CUfunction fn_hist = nullptr, fn_scatter = nullptr, fn_scatter_peer = nullptr;
};

namespace pm {
// Compile + load the fused module of `plan` (idempotent, thread-safe).
int plan_fused(pm_plan* plan);
}  // namespace pm
