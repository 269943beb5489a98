// K1+K2 fused -- map an index launch and partition it by processor without
// materialising the processor ids.
//
// Pass 1 (pm_map_hist) evaluates the point program and histograms the ids
// per 4096-point tile (0 B/pt of HBM in implicit mode); the per-(bin, tile)
// counts are scanned into output slots.  Pass 2 (pm_map_scatter) evaluates
// the program again and writes every point's index at its stable slot -- the
// only per-point HBM traffic (4 B/pt, +4 B/pt when the ids are also wanted).
// K1 then K2 would move 4 (write ids) + 4 (hist read) + 4 + 4 (scatter read +
// write) = 16 B/pt.  Between the passes the caller may exchange the counts
// (sharded launches, distmap.py): pass 2 can then write each processor's
// points straight into the buffer of the GPU that hosts it, over NVLink.
//
// Reference semantics: cmd_map's loop (cli.py:149-170) + expand_shards'
// leaves (tasksim/sim.py:67-120) = a stable partition of launch points by
// processor; failures report the lowest failing point like pm_map_batch.

#include "plan.h"
#include "stable_partition.cuh"

namespace {

int check_common(const pm_plan* plan, const int32_t* points, int64_t n, int64_t first,
                 int32_t nbins, const uint64_t* status, size_t scratch_bytes) {
  if (!plan || !status || n < 0 || first < 0)
    return pm::set_error("map_partition: bad arguments"), PM_ERR_INVALID;
  if (nbins < 1 || nbins > pm::kSmallBins)
    return pm::set_error("map_partition: 1..%d processors", pm::kSmallBins), PM_ERR_UNSUPPORTED;
  if (!plan->implicit && plan->n_coords > 0 && n > 0 && !points)
    return pm::set_error("map_partition: explicit plan needs points"), PM_ERR_INVALID;
  if (first + n >= (1LL << 47))
    return pm::set_error("map_partition: index too large"), PM_ERR_UNSUPPORTED;
  if ((n + pm::kSmallTile - 1) / pm::kSmallTile > 0x7FFFFFFFLL)
    return pm::set_error("map_partition: too many tiles"), PM_ERR_UNSUPPORTED;
  if (scratch_bytes < pm::small_scratch_bytes(n, nbins))
    return pm::set_error("map_partition: scratch too small"), PM_ERR_INVALID;
  return PM_OK;
}

int set_smem(CUfunction f, size_t bytes) {
  if (bytes <= 48 * 1024) return PM_OK;
  PM_CU_TRY(pm::driver()->funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                           (int)bytes));
  return PM_OK;
}

}  // namespace

extern "C" {

size_t pm_map_partition_scratch_bytes(int64_t n, int32_t nbins) {
  return pm::small_scratch_bytes(n, nbins);
}

int pm_map_hist(pm_plan* plan, const int32_t* points, int64_t n, int64_t first, int32_t nbins,
                int64_t* counts, int64_t* offsets, uint64_t* status, void* scratch,
                size_t scratch_bytes, void* stream) {
  int rc = check_common(plan, points, n, first, nbins, status, scratch_bytes);
  if (rc) return rc;
  if (!counts || !offsets) return pm::set_error("pm_map_hist: null counts"), PM_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    PM_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * nbins, s));
    PM_CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(int64_t) * nbins, s));
    return PM_OK;
  }
  if ((rc = pm::plan_fused(plan))) return rc;
  const pm::Driver* d = pm::driver();
  long long ntiles = (n + pm::kSmallTile - 1) / pm::kSmallTile;
  const long long len = ntiles * nbins;
  long long* hist = reinterpret_cast<long long*>(scratch);
  void* scan_tmp = reinterpret_cast<char*>(scratch) + pm::small_scan_offset(ntiles, nbins);
  const size_t smem = pm::small_hist_smem(nbins);
  if ((rc = set_smem(plan->fn_hist, smem))) return rc;
  const int32_t* pts = points;
  long long nn = n, ff = first;
  int nb = nbins;
  void* args[] = {(void*)&pts, (void*)&nn, (void*)&ff, (void*)&nb, (void*)&ntiles,
                  (void*)&hist, (void*)&status};
  // grid-stride over groups of 256 tiles (tiles proven uniform cost one thread each)
  long long groups = (ntiles + pm::kPartThreads - 1) / pm::kPartThreads;
  const long long cap = (long long)pm::num_sms() * 8;
  if (groups > cap) groups = cap;
  PM_CU_TRY(d->launchKernel(plan->fn_hist, (unsigned)groups, 1, 1, pm::kPartThreads, 1, 1,
                            (unsigned)smem, (CUstream)s, args, nullptr));
  if ((rc = pm::exclusive_scan_i64(hist, len, scan_tmp, s))) return rc;
  pm::k_part_bin_totals<<<(nbins + 255) / 256, 256, 0, s>>>(
      hist, ntiles, nbins, reinterpret_cast<const long long*>(scan_tmp),
      reinterpret_cast<long long*>(counts), reinterpret_cast<long long*>(offsets));
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

int pm_map_scatter(pm_plan* plan, const int32_t* points, int64_t n, int64_t first, int32_t nbins,
                   int32_t* out_proc, int32_t* perm, const int64_t* bin_dst, int64_t index_base,
                   uint64_t* status, void* scratch, size_t scratch_bytes, void* stream) {
  int rc = check_common(plan, points, n, first, nbins, status, scratch_bytes);
  if (rc) return rc;
  if (!perm && !bin_dst) return pm::set_error("pm_map_scatter: no destination"), PM_ERR_INVALID;
  if (index_base < 0 || index_base + n > 0x7FFFFFFFLL)
    return pm::set_error("pm_map_scatter: int32 indices need index_base + n < 2^31"),
           PM_ERR_UNSUPPORTED;
  if (n == 0) return PM_OK;
  if ((rc = pm::plan_fused(plan))) return rc;
  const pm::Driver* d = pm::driver();
  long long ntiles = (n + pm::kSmallTile - 1) / pm::kSmallTile;
  const long long* pos0 = reinterpret_cast<const long long*>(scratch);
  CUfunction f = bin_dst ? plan->fn_scatter_peer : plan->fn_scatter;
  const size_t smem = pm::small_scatter_smem(nbins);
  if ((rc = set_smem(f, smem))) return rc;
  const int32_t* pts = points;
  long long nn = n, ff = first, base = index_base;
  int nb = nbins;
  const void* dst = bin_dst ? (const void*)bin_dst : (const void*)perm;
  void* args[] = {(void*)&pts, (void*)&nn, (void*)&ff, (void*)&nb, (void*)&ntiles,
                  (void*)&pos0, (void*)&status, (void*)&out_proc, (void*)&dst, (void*)&base};
  // (the NVRTC text and this file see the same PM_SCATTER_TILES default)
  PM_CU_TRY(d->launchKernel(f, pm::small_scatter_grid(ntiles), 1, 1, pm::kPartThreads, 1, 1,
                            (unsigned)smem, (CUstream)stream, args, nullptr));
  return PM_OK;
}

}  // extern "C"
