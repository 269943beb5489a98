// Error reporting and driver entry points shared by all libmapple_b200 units.
#include <mutex>

#include "pm_common.h"

namespace pm {

namespace {
thread_local char g_err[8192] = "";
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

template <typename F>
static bool resolve(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p) {
    return false;
  }
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Driver* driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = resolve("cuModuleLoadData", &d.moduleLoadData) &&
           resolve("cuModuleUnload", &d.moduleUnload) &&
           resolve("cuModuleGetFunction", &d.moduleGetFunction) &&
           resolve("cuLaunchKernel", &d.launchKernel) &&
           resolve("cuFuncSetAttribute", &d.funcSetAttribute) &&
           resolve("cuTensorMapEncodeTiled", &d.tensorMapEncodeTiled) &&
           resolve("cuCtxGetCurrent", &d.ctxGetCurrent);
  });
  if (!d.ok) {
    set_error("CUDA driver entry points unavailable (no GPU driver?)");
    return nullptr;
  }
  return &d;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

}  // namespace pm

extern "C" {
int pm_abi_version(void) { return PM_ABI_VERSION; }
const char* pm_last_error(void) { return pm::g_err; }
}
