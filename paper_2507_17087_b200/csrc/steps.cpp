// Step programs: the mapped executors' per-step schedules as data, run by one C call.
//
// A mapped multiply (SUMMA / PUMMA panels, Johnson / COSMA grids, Cannon / 2.5D
// rounds) is, per GPU and per step, a fixed list of operations over fixed device
// pointers: copy-engine pulls of peer panels on a few copy lanes, waits of the
// compute stream on those pulls, tcgen05 GEMM launches (possibly reduce-adding
// into a peer's C), peer-memory barriers.  The host-side planners (Python here;
// any host through this ABI) build that list once; pm_steps_run replays it with
// no per-op host round trips: lanes fork from the compute stream at the step's
// start (so a step's pulls follow the previous step's GEMMs -- the WAR order on
// the operand buffers) and join back at its end.  Capturable into a CUDA graph.

#include <cstring>
#include <mutex>
#include <vector>

#include "pm_common.h"

struct pm_steps {
  std::vector<pm_step_op> ops;
  std::vector<pm_peer_copy> copies;      // COPY_BARRIER payloads (ops point into it)
  cudaStream_t lanes[PM_STEP_LANES] = {};
  cudaEvent_t start = nullptr;
  std::vector<cudaEvent_t> done;         // per op (PULL)
  int used[PM_STEP_LANES] = {};
  int last[PM_STEP_LANES];               // last PULL op per lane
  int device = 0;
};

extern "C" {

void pm_steps_destroy(pm_steps* s) {
  if (!s) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(s->device);
  for (auto e : s->done)
    if (e) cudaEventDestroy(e);
  if (s->start) cudaEventDestroy(s->start);
  for (auto l : s->lanes)
    if (l) cudaStreamDestroy(l);
  cudaSetDevice(cur);
  delete s;
}

int pm_steps_create(const pm_step_op* ops, int32_t n, pm_steps** out) {
  if (!out || n < 0 || (n > 0 && !ops)) return pm::set_error("pm_steps_create: bad arguments"),
                                               PM_ERR_INVALID;
  *out = nullptr;
  pm_steps* s = new pm_steps();
  cudaGetDevice(&s->device);
  for (int l = 0; l < PM_STEP_LANES; ++l) s->last[l] = -1;
  size_t ncopy = 0;
  for (int i = 0; i < n; ++i) {
    const pm_step_op& o = ops[i];
    switch (o.kind) {
      case PM_STEP_PULL:
        if (o.lane < -1 || o.lane >= PM_STEP_LANES) {
          delete s;
          return pm::set_error("pm_steps_create: op %d: lane %d", i, o.lane), PM_ERR_INVALID;
        }
        break;
      case PM_STEP_WAIT:
        if (o.lane < 0 || o.lane >= i || ops[o.lane].kind != PM_STEP_PULL || ops[o.lane].lane < 0) {
          delete s;
          return pm::set_error("pm_steps_create: op %d waits for %d, not an earlier lane pull", i,
                               o.lane), PM_ERR_INVALID;
        }
        break;
      case PM_STEP_GEMM_BF16: case PM_STEP_GEMM_TF32: case PM_STEP_MEMSET: case PM_STEP_FORK:
        break;
      case PM_STEP_BARRIER:
        if (!o.barrier) {
          delete s;
          return pm::set_error("pm_steps_create: op %d: null barrier", i), PM_ERR_INVALID;
        }
        break;
      case PM_STEP_COPY_BARRIER:
        if (!o.barrier || !o.ticket || o.n_copies < 0 || o.n_copies > PM_PEER_COPY_MAX ||
            (o.n_copies && !o.copies)) {
          delete s;
          return pm::set_error("pm_steps_create: op %d: bad copy barrier", i), PM_ERR_INVALID;
        }
        ncopy += o.n_copies;
        break;
      default:
        delete s;
        return pm::set_error("pm_steps_create: op %d: unknown kind %d", i, o.kind), PM_ERR_INVALID;
    }
  }
  s->ops.assign(ops, ops + n);
  s->copies.reserve(ncopy);
  for (auto& o : s->ops)  // own the copy lists
    if (o.kind == PM_STEP_COPY_BARRIER) {
      const size_t at = s->copies.size();
      s->copies.insert(s->copies.end(), o.copies, o.copies + o.n_copies);
      o.copies = s->copies.data() + at;
    }
  s->done.assign(n, nullptr);
  cudaError_t e = cudaEventCreateWithFlags(&s->start, cudaEventDisableTiming);
  for (int i = 0; i < n && e == cudaSuccess; ++i) {
    const pm_step_op& o = s->ops[i];
    if (o.kind == PM_STEP_PULL && o.lane >= 0) {
      e = cudaEventCreateWithFlags(&s->done[i], cudaEventDisableTiming);
      s->used[o.lane] = 1;
      s->last[o.lane] = i;
    }
  }
  for (int l = 0; l < PM_STEP_LANES && e == cudaSuccess; ++l)
    if (s->used[l]) e = cudaStreamCreateWithFlags(&s->lanes[l], cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    pm_steps_destroy(s);
    return pm::set_error("pm_steps_create: %s", cudaGetErrorString(e)), PM_ERR_CUDA;
  }
  *out = s;
  return PM_OK;
}

int pm_steps_run(pm_steps* s, void* stream) {
  if (!s) return pm::set_error("pm_steps_run: null program"), PM_ERR_INVALID;
  cudaStream_t cs = (cudaStream_t)stream;
  bool forked = false;
  for (size_t i = 0; i < s->ops.size(); ++i) {
    const pm_step_op& o = s->ops[i];
    int rc = PM_OK;
    switch (o.kind) {
      case PM_STEP_PULL: {
        cudaStream_t st = cs;
        if (o.lane >= 0) {
          if (!forked) {  // the lanes start after everything already on the compute stream
            PM_CUDA_TRY(cudaEventRecord(s->start, cs));
            for (int l = 0; l < PM_STEP_LANES; ++l)
              if (s->used[l]) PM_CUDA_TRY(cudaStreamWaitEvent(s->lanes[l], s->start, 0));
            forked = true;
          }
          st = s->lanes[o.lane];
        }
        if (o.width > 0 && o.height > 0)
          PM_CUDA_TRY(cudaMemcpy2DAsync(o.dst, (size_t)o.dpitch, o.src, (size_t)o.spitch,
                                        (size_t)o.width, (size_t)o.height,
                                        cudaMemcpyDeviceToDevice, st));
        if (o.lane >= 0) PM_CUDA_TRY(cudaEventRecord(s->done[i], st));
        break;
      }
      case PM_STEP_WAIT:
        PM_CUDA_TRY(cudaStreamWaitEvent(cs, s->done[o.lane], 0));
        break;
      case PM_STEP_GEMM_BF16:
        rc = pm_gemm_bf16(o.src, o.lda, o.b, o.ldb, o.dst, o.ldc, o.m, o.n, o.k, o.c_bf16,
                          o.accumulate, stream);
        break;
      case PM_STEP_GEMM_TF32:
        rc = pm_gemm_tf32(static_cast<const float*>(o.src), o.lda,
                          static_cast<const float*>(o.b), o.ldb, static_cast<float*>(o.dst),
                          o.ldc, o.m, o.n, o.k, o.accumulate, stream);
        break;
      case PM_STEP_MEMSET:
        PM_CUDA_TRY(cudaMemsetAsync(o.dst, 0, (size_t)o.width, cs));
        break;
      case PM_STEP_BARRIER:
        rc = pm_peer_barrier(static_cast<const pm_peer_barrier_view*>(o.barrier), stream);
        break;
      case PM_STEP_COPY_BARRIER:
        rc = pm_peer_copy_barrier(static_cast<const pm_peer_barrier_view*>(o.barrier), o.copies,
                                  o.n_copies, o.ticket, stream);
        break;
      case PM_STEP_FORK:  // later lane pulls follow everything queued so far on cs
        PM_CUDA_TRY(cudaEventRecord(s->start, cs));
        for (int l = 0; l < PM_STEP_LANES; ++l)
          if (s->used[l]) PM_CUDA_TRY(cudaStreamWaitEvent(s->lanes[l], s->start, 0));
        forked = true;
        break;
    }
    if (rc) return rc;
  }
  if (forked)  // join: the next step (and the caller) see every pull of this one
    for (int l = 0; l < PM_STEP_LANES; ++l)
      if (s->used[l] && s->last[l] >= 0) PM_CUDA_TRY(cudaStreamWaitEvent(cs, s->done[s->last[l]], 0));
  return PM_OK;
}

}  // extern "C"
