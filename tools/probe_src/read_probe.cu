// HBM read ceiling probe: every thread sums `iters` 16-byte loads (grid-stride), one int
// out per thread-block.  Built by tools/read_probe.py with nvcc; not part of the library.
#include <cuda_runtime.h>
extern "C" __global__ void __launch_bounds__(256) k_read(const int4* __restrict__ p, long long n4,
                                                         int* out) {
  int acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) out[blockIdx.x] = acc;
}
extern "C" __global__ void __launch_bounds__(256) k_read_unroll(const int4* __restrict__ p,
                                                                long long n4, int* out) {
  // 4 independent loads in flight per thread per iteration
  int acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n4; i += stride) acc ^= p[i].x;
  if (acc == 0x7fffffff) out[blockIdx.x] = acc;
}
extern "C" int launch(int which, const void* p, long long n4, int* out, long long blocks,
                      cudaStream_t s) {
  if (which == 0) k_read<<<(unsigned)blocks, 256, 0, s>>>((const int4*)p, n4, out);
  else k_read_unroll<<<(unsigned)blocks, 256, 0, s>>>((const int4*)p, n4, out);
  return (int)cudaGetLastError();
}
