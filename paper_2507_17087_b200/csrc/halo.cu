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

#include <cstdint>

#include "pm_common.h"
#include "stable_partition.cuh"

namespace pm {
namespace {

struct HaloKey {
  const int* __restrict__ owner;
  long long ext[3];
  long long stride[3];
  int halo[3];
  int rank;
  int nprocs;
  static constexpr bool kVec4 = false;
  static constexpr bool kPeek = false;
  __device__ __forceinline__ void uniform(long long, int, int) const {}
  __device__ __forceinline__ int operator()(long long i) const {
    const int slots = 2 * rank;
    const long long cell = i / slots;
    const int dd = (int)(i - cell * slots);
    const int n = dd >> 1;
    const int dir = (dd & 1) ? 1 : -1;
    const int h = halo[n];
    if (h <= 0) return -1;
    const long long x = (cell / stride[n]) % ext[n];
    const int o = __ldg(owner + cell);
    if (o < 0 || o >= nprocs) return -1;
    for (int j = 1; j <= h; ++j) {
      const long long y = x + dir * j;
      if (y < 0 || y >= ext[n]) return -1;
      const int q = __ldg(owner + cell + (long long)dir * j * stride[n]);
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

bool make_key(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
              int32_t nprocs, HaloKey* k, long long* ncells) {
  if (rank < 1 || rank > 3 || nprocs < 1 || nprocs > 64 || !ext || !halo) return false;
  *k = HaloKey{};
  k->owner = owner;
  k->rank = rank;
  k->nprocs = nprocs;
  long long st = 1;
  for (int m = rank - 1; m >= 0; --m) {
    if (ext[m] < 1 || halo[m] < 0) return false;
    k->ext[m] = ext[m];
    k->stride[m] = st;
    k->halo[m] = halo[m];
    st *= ext[m];
  }
  *ncells = st;
  return true;
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
  pm::HaloKey key;
  long long ncells = 0;
  if (!owner || !pair_counts || !pair_offsets ||
      !pm::make_key(owner, ext, rank, halo, nprocs, &key, &ncells))
    return pm::set_error("pm_halo_lists: bad arguments (rank 1..3, nprocs 1..64)"),
           PM_ERR_INVALID;
  pm::HaloSink sink{reinterpret_cast<long long*>(cells), reinterpret_cast<signed char*>(dims),
                    2 * rank};
  return pm::stable_partition(key, sink, cells != nullptr, ncells * 2 * rank, nprocs * nprocs,
                              reinterpret_cast<long long*>(pair_counts),
                              reinterpret_cast<long long*>(pair_offsets), scratch, scratch_bytes,
                              (cudaStream_t)stream);
}

}  // extern "C"
