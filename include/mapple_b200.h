/*
 * mapple_b200.h -- C ABI of the B200-native Mapple mapping/execution library.
 *
 * Plain C types only (no torch, no CUDA headers needed by callers: streams are
 * passed as `void*` = cudaStream_t/CUstream, device buffers as raw pointers).
 * Every device buffer is owned by the caller; the library never allocates or
 * frees caller memory (transient scratch is passed in explicitly).  All
 * launches are stream-ordered; no entry point synchronises the device except
 * where documented.  Return value: PM_OK (0) or a PM_ERR_* code with a
 * thread-local message in pm_last_error().
 *
 * Reference interfaces each entry point replaces (paths under the reference
 * root, pkg/src/procmap/):
 *   pm_plan_create / pm_plan_destroy
 *       <- compile_mapper() / MappingFunction (dsl/interp.py:366-433): the
 *          per-ispace prefix is evaluated on the host and the per-point suffix
 *          is lowered to a pm_program (paper_2507_17087_b200/dsl/lower.py).
 *   pm_map_batch
 *       <- the per-point loop `fn(pt, ispace)` of cmd_map (cli.py:155-161)
 *          and shard_policy (tasksim/sim.py:78); MappingFunction.__call__
 *          (dsl/interp.py:401-418) + ProcSpace.resolve (spaces.py:185-213).
 *   pm_partition
 *       <- expand_shards / shard_policy ownership leaves (tasksim/sim.py:67-120)
 *          and proc_counts (cli.py:154-164): a stable partition of points by
 *          processor.
 *   pm_halo_lists
 *       <- oracle_boundary_count (commvol.py:136-168): per-(src,dst) halo
 *          transfer lists of a block-mapped grid whose totals equal the count.
 *   pm_gemm_bf16
 *       <- the per-processor tile product of the paper's matmul workloads
 *          (PAPER.md:493); no reference code exists.
 */
#ifndef MAPPLE_B200_H
#define MAPPLE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM_ABI_VERSION 1

/* status codes */
#define PM_OK 0
#define PM_ERR_INVALID 1     /* bad argument / malformed program            */
#define PM_ERR_CUDA 2        /* CUDA runtime or driver failure               */
#define PM_ERR_NVRTC 3       /* JIT compilation of the point program failed  */
#define PM_ERR_UNSUPPORTED 4 /* shape / size outside what the kernel handles */

/* point-program opcodes (dsl/lower.py OP_*) */
enum pm_opcode {
  PM_OP_CONST = 0,  /* dst = imm (128-bit: lo | hi << 64)                 */
  PM_OP_COORD = 1,  /* dst = point coordinate `lo`                        */
  PM_OP_ADD = 2,    /* dst = a + b                                        */
  PM_OP_SUB = 3,    /* dst = a - b                                        */
  PM_OP_MUL = 4,    /* dst = a * b                                        */
  PM_OP_DIV = 5,    /* dst = floor(a / b); c = 1: a >= 0 and b > 0 proven;
                       site >= 0: fail(site) when b == 0                  */
  PM_OP_MOD = 6,    /* dst = a - b * floor(a / b); flags as PM_OP_DIV     */
  PM_OP_GT = 7,     /* dst = a > b                                        */
  PM_OP_LT = 8,     /* dst = a < b                                        */
  PM_OP_EQ = 9,     /* dst = a == b                                       */
  PM_OP_SELECT = 10,/* dst = a ? b : c                                    */
  PM_OP_MOV = 11,   /* dst = a                                            */
  PM_OP_CHECK = 12, /* fail(site) unless lo <= a < hi                     */
  PM_OP_FAIL = 13,  /* fail(site)                                         */
  PM_OP_IF = 14,    /* if (a != 0) {                                      */
  PM_OP_ELSE = 15,  /* } else {                                           */
  PM_OP_ENDIF = 16, /* }                                                  */
  PM_OP_RET = 17    /* processor id = a                                   */
};

typedef struct pm_insn {
  int32_t op, dst, a, b, c, site;
  int64_t lo, hi;
} pm_insn;

typedef struct pm_program {
  int32_t n_insns;
  const pm_insn* insns;
  int32_t n_regs;
  const uint8_t* reg_width; /* per register: 0 = int32, 1 = int64, 2 = int128 */
  int32_t n_coords;         /* rank of an iteration point                      */
  int32_t implicit;         /* 1: points are the row-major ispace enumeration  */
  const int64_t* extents;   /* n_coords ispace extents (implicit mode)         */
} pm_program;

typedef struct pm_plan pm_plan;

int pm_abi_version(void);
const char* pm_last_error(void);

/* CUDA C++ source of the specialised point kernel (for inspection/tests).
 * Writes at most `cap` bytes (NUL-terminated) and the full length to *len. */
int pm_codegen(const pm_program* prog, char* buf, size_t cap, size_t* len);

/* JIT-compile the point program for the current device (NVRTC, sm_100a) and
 * load it.  Needs a GPU only for the final module load; with `load == 0` the
 * program is compiled to a cubin and discarded (a CPU-side build check). */
int pm_compile_check(const pm_program* prog);
int pm_plan_create(const pm_program* prog, pm_plan** out);
void pm_plan_destroy(pm_plan* plan);

/* Map n points.  points: NULL in implicit mode (point i is the row-major
 * point `first + i` of the ispace) or n * n_coords int32 row-major.
 * out_proc[i] = node * procs_per_node + proc, or -1 where the point failed.
 * status (device, 8 bytes, caller initialises to UINT64_MAX): atomicMin of
 * ((first + i) << 16 | site) over failing points -- the lowest failing index
 * and the site it failed at. */
int pm_map_batch(const pm_plan* plan, const int32_t* points, int64_t n, int64_t first,
                 int32_t* out_proc, uint64_t* status, void* stream);

/* Failure probe for exact error messages
 *   <- the reference formats the operand values into the message of the
 *      exception it raises at the failing point ("index (3, 8) out of range for
 *      shape (2, 2)", spaces.py:215-221 re-wrapped at dsl/interp.py:255-258;
 *      "index 5 out of range for tuple of rank 2", dsl/interp.py:212-213;
 *      "dimension 3 out of range for rank 2", dsl/interp.py:247-248).
 * Re-evaluates the single point `index` (a launch index as reported in the
 * status word: implicit mode = row-major linear index; explicit mode = the row
 * of `points`) with a diagnostic twin of the plan's kernel, compiled on first
 * use.  Device outputs: site[0] = the failing site (-1 if the point maps),
 * site[1] = the result; dump[2 r], dump[2 r + 1] = register r at the failure as
 * the low / high 64-bit words of its sign-extended 128-bit value, for
 * r < pm_plan_regs(plan). */
int pm_plan_regs(const pm_plan* plan);
int pm_compile_check_probe(const pm_program* prog);  /* NVRTC build of the probe (no GPU) */
int pm_map_probe(pm_plan* plan, const int32_t* points, int64_t index, int64_t* dump,
                 int32_t* site, void* stream);

/* Fused map + partition (K1 + K2 without materialising the processor ids)
 *   <- cmd_map's loop (cli.py:149-170) feeding expand_shards / shard_policy
 *      (tasksim/sim.py:67-120): the stable partition of launch points
 *      [first, first + n) by processor id, ids in [0, nbins), nbins <= 64.
 * Pass 1, pm_map_hist: counts[b], offsets[b] (exclusive prefix) per processor;
 *   the per-tile histogram stays in `scratch` for pass 2.
 * Pass 2, pm_map_scatter: with the same n / first / nbins / scratch, writes
 *   point index (index_base + i) at its stable slot: perm[offsets[b] + r] or,
 *   when bin_dst != NULL, ((int32_t*)bin_dst[2 b])[offsets[b] + r + bin_dst[2 b + 1]]
 *   (bin_dst: device array of nbins (pointer, element shift) pairs; the pointers
 *   may be peer-GPU memory).  out_proc (nullable) receives the processor ids.
 * Failures: as pm_map_batch (status, caller-initialised to UINT64_MAX); a
 *   failing point is left out of the partition.  Explicit mode: `points` as in
 *   pm_map_batch, indexed by i.  scratch: pm_map_partition_scratch_bytes(). */
size_t pm_map_partition_scratch_bytes(int64_t n, int32_t nbins);
int pm_compile_check_fused(const pm_program* prog);
int pm_map_hist(pm_plan* plan, const int32_t* points, int64_t n, int64_t first, int32_t nbins,
                int64_t* counts, int64_t* offsets, uint64_t* status, void* scratch,
                size_t scratch_bytes, void* stream);
int pm_map_scatter(pm_plan* plan, const int32_t* points, int64_t n, int64_t first, int32_t nbins,
                   int32_t* out_proc, int32_t* perm, const int64_t* bin_dst, int64_t index_base,
                   uint64_t* status, void* scratch, size_t scratch_bytes, void* stream);

/* Stable partition of n processor ids in [0, nbins):
 *   counts[b]  = #points with id b                    (int64, device)
 *   offsets[b] = exclusive prefix of counts           (int64, device)
 *   perm[...]  = point indices grouped by id, each group in input order.
 * ids outside [0, nbins) are an error (PM_ERR_INVALID is reported via
 * `bad`, a device int64 set to the first offending index, or -1).
 * scratch: pm_partition_scratch_bytes(n, nbins) bytes of device memory. */
size_t pm_partition_scratch_bytes(int64_t n, int32_t nbins);
int pm_partition(const int32_t* proc, int64_t n, int32_t nbins, int64_t* counts,
                 int64_t* offsets, int32_t* perm, int64_t* bad, void* scratch,
                 size_t scratch_bytes, void* stream);

/* Halo transfer lists of a 2D/3D grid owned cell-by-cell (owner = int32 proc
 * id per cell, row-major, extents ext[0..rank-1]).  A cell c of owner P is
 * sent to Q != P along dim n / direction s when the first cell of a different
 * owner among c + s*j*e_n (1 <= j <= halo[n]) is owned by Q; one entry per
 * (cell, dim, direction).  Totals equal oracle_boundary_count for block
 * partitions.  Output grouped by key = src * nprocs + dst, cells ascending:
 *   pair_counts[nprocs*nprocs], pair_offsets[nprocs*nprocs] (int64, device),
 *   cells[...] (int64 linear cell index), dims[...] (int8: 2*n + (s > 0)).
 * Pass cells == NULL to count only.  scratch: pm_halo_scratch_bytes(). */
size_t pm_halo_scratch_bytes(const int64_t* ext, int32_t rank, int32_t nprocs);
int pm_halo_lists(const int32_t* owner, const int64_t* ext, int32_t rank,
                  const int32_t* halo, int32_t nprocs, int64_t* pair_counts,
                  int64_t* pair_offsets, int64_t* cells, int8_t* dims, void* scratch,
                  size_t scratch_bytes, void* stream);
/* The same lists by compaction (what transfer.halo_lists uses; halo entries are
 * sparse, so no per-(pair, tile) histogram is built):
 *   pm_halo_count    pair_counts[nprocs^2] and, in tile_scratch
 *                    (pm_halo_tile_scratch_bytes), each 8192-slot tile's output
 *                    offset (and, after the scan, the total entry count);
 *   pm_halo_compact  every entry as (pair key, slot index = cell * 2R + 2n + (s>0))
 *                    in slot order into keys / slots [cap] (entries past cap dropped);
 *   (pm_partition of keys into nprocs^2 bins -> perm, counts, offsets)
 *   pm_halo_gather   cells[j] / dims[j] of slots[perm[j]] (dims nullable). */
size_t pm_halo_tile_scratch_bytes(const int64_t* ext, int32_t rank);
int pm_halo_count(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
                  int32_t nprocs, int64_t* pair_counts, void* tile_scratch, size_t bytes,
                  int64_t* total /* nullable: device copy of the entry count */, void* stream);
int pm_halo_compact(const int32_t* owner, const int64_t* ext, int32_t rank, const int32_t* halo,
                    int32_t nprocs, void* tile_scratch, int32_t* keys, int64_t* slots, int64_t cap,
                    void* stream);
/* Grouping without a permutation array: the stable partition of the compacted
 * keys (only the first *total of the cap items; total = the device-side entry
 * count, e.g. the sum of pair_counts) writes each entry's cells[] / dims[]
 * at its grouped position, and pair_counts / pair_offsets.  No host
 * synchronisation is needed between count, compaction and grouping when the
 * caller sizes keys / slots / cells / dims with a capacity `cap` (entries
 * past it are dropped; compare the returned total with cap).
 * scratch: pm_halo_group_scratch_bytes(cap, nprocs). */
size_t pm_halo_group_scratch_bytes(int64_t cap, int32_t nprocs);
int pm_halo_group(const int32_t* keys, const int64_t* slots, int64_t cap, const int64_t* total,
                  int32_t rank, int32_t nprocs, int64_t* pair_counts, int64_t* pair_offsets,
                  int64_t* cells, int8_t* dims, void* scratch, size_t scratch_bytes,
                  void* stream);
int pm_halo_gather(const int32_t* perm, const int64_t* slots, int64_t n, int32_t rank,
                   int64_t* cells, int8_t* dims, void* stream);

/* C[M,N] (+)= A[M,K] * B[K,N] on the tcgen05 tensor cores, bf16 inputs, fp32
 * accumulation.  A is row-major (K contiguous, lda >= K); B is given
 * transposed as Bt[N,K] row-major (K contiguous, ldb >= K).  C is row-major
 * fp32 (ldc >= N) or bf16 when c_bf16 != 0; accumulate != 0 adds into C.
 * accumulate: 0 = overwrite, 1 = C += AB, 2 = C += AB with element-wise atomic
 * reduce-add (TMA .add; C may be a peer GPU's IPC-mapped buffer, several GPUs may add
 * concurrently; fp32 only).  lda, ldb % 8 == 0, 16-byte aligned A, Bt. */
int pm_gemm_bf16(const void* A, int64_t lda, const void* Bt, int64_t ldb, void* C,
                 int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t c_bf16,
                 int32_t accumulate, void* stream);

/* Same on fp32 operands through the TF32 tensor-core path (tcgen05 kind::tf32,
 * fp32 accumulation): A[M,K], Bt[N,K], C[M,N] fp32 row-major; lda, ldb % 4 == 0.
 * Used for the fp32 Cannon configuration (BASELINE configs[0]). */
int pm_gemm_tf32(const float* A, int64_t lda, const float* Bt, int64_t ldb, float* C, int64_t ldc,
                 int64_t M, int64_t N, int64_t K, int32_t accumulate, void* stream);

/* NVLink peer memory for the mapped executors (replaces the Legion/Realm
 * data movement the paper's runs used; the reference
 * package models it only as element counts, commvol.py:1-17).
 *   pm_ipc_handle: 64-byte CUDA IPC handle of the allocation holding ptr and
 *                  ptr's byte offset inside it;
 *   pm_ipc_open / pm_ipc_close: map / unmap a peer's allocation;
 *   pm_copy2d_async: pitched copy-engine copy (peer or local), stream-ordered. */
int pm_ipc_handle(const void* ptr, void* handle_out, int64_t* offset_out);
int pm_ipc_open(const void* handle, void** base_out);
int pm_ipc_close(void* base);
int pm_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                    int64_t height, void* stream);

/* Stream-ordered barrier among the box's GPUs through peer memory (no NCCL):
 * each GPU pushes its next epoch (*epoch + 1, advanced on the device, so the
 * barrier is CUDA-graph capturable) into peer_slot[q] = &flags_q[rank] with a
 * system-scope release store and waits until my_flags[q] reaches it for every
 * peer q (acquire).  Replaces the per-round 4-byte NCCL all-reduce of the
 * Cannon / 2.5D shifts (the orderings the reference's algorithms need between
 * rounds).  Flags and epoch start at zero and only grow. */
#define PM_BARRIER_MAX_RANKS 16
typedef struct pm_peer_barrier_view {
  int32_t* my_flags;                         /* [world] local, pushed by peers   */
  int32_t* peer_slot[PM_BARRIER_MAX_RANKS];  /* &peer q's my_flags[rank]         */
  int32_t* epoch;                            /* local device counter             */
  int32_t world, rank;
} pm_peer_barrier_view;
int pm_peer_barrier(const pm_peer_barrier_view* view, void* stream);
/* Up to PM_PEER_COPY_MAX contiguous copies (peer or local, 16-byte aligned, bytes a
 * multiple of 16) done by the SMs, then the same barrier, in one launch: a Cannon /
 * 2.5D shift round when its blocks are small and the round latency-bound.  `ticket`:
 * a device uint32, zero at first use (the kernel leaves it zero). */
#define PM_PEER_COPY_MAX 4
typedef struct pm_peer_copy {
  void* dst;
  const void* src;
  int64_t bytes;
} pm_peer_copy;
int pm_peer_copy_barrier(const pm_peer_barrier_view* view, const pm_peer_copy* copies,
                         int32_t n, uint32_t* ticket, void* stream);

/* One 5-point Jacobi sweep of this GPU's rectangle of a block-mapped grid
 * (the paper's stencil workload; ownership from the Mapple
 * block mapping, halo totals = surface_volume, commvol.py:94-96).  Neighbour
 * cells are read straight from the neighbours' `in` buffers (peer pointers);
 * ordering with the neighbours uses flags each GPU pushes into the others'
 * `my_flags` with system-scope release stores (see csrc/stencil.cu).  Three
 * rotating buffers per GPU; `sweep` counts from 0. */
typedef struct pm_stencil_view {
  float* out;
  const float* in;
  int64_t rows, cols, pitch; /* my rectangle (elements) and its row pitch      */
  int64_t grow0, gcol0;      /* global origin of the rectangle                 */
  int64_t grows, gcols;      /* global extents                                 */
  const float* nbr[4];       /* up, down, left, right neighbour `in` or NULL   */
  int64_t nbr_pitch[4];
  int64_t nbr_rows[4], nbr_cols[4];
  int32_t* my_flags;         /* [world] sweep-done flags pushed by neighbours  */
  int32_t* nbr_flag_slot[4]; /* &neighbour.my_flags[my rank] (peer pointers)   */
  int32_t nbr_rank[4];
  uint32_t* ticket;          /* unused (kept for the struct layout)           */
  float* col_out[2];         /* my first / last column of `out`, contiguous    */
                             /* (read by the left / right neighbour)           */
  const float* nbr_col[2];   /* left neighbour's last column of its `in` strip,*/
                             /* right neighbour's first column (peer pointers) */
} pm_stencil_view;
int pm_stencil_sweep(const pm_stencil_view* view, int32_t sweep, void* stream);

/* One phase of a circuit-simulation iteration (the paper's Circuit workload,
 * PAPER.md:495, after the Legion circuit example of Bauer et al. 2012; no
 * reference code, SURVEY.md §8c "parity unpinned").  Pieces are placed by a
 * Mapple mapping; node arrays are per GPU; a node reference is
 * (rank << 27) | slot, resolved through the per-rank pointer tables (peer
 * pointers for other GPUs, CUDA IPC).  Wire state is structure-of-arrays:
 * current[s * n_wires + w] (s < SEGMENTS), wire_volt[s * n_wires + w]
 * (s < SEGMENTS - 1).
 *   phase 0: calc_new_currents (`steps` iterations) + distribute_charge
 *            (float atomics into the owning GPU's charge, peer or local);
 *   phase 1: update_voltages of this GPU's nodes (charge -> voltage, leakage,
 *            charge reset).
 * Phases of different GPUs must be separated by a barrier (the executor
 * orders them with a stream-ordered NCCL all-reduce). */
#define PM_CIRCUIT_SEGMENTS 10
#define PM_CIRCUIT_MAX_RANKS 16
typedef struct pm_circuit_view {
  int64_t n_wires, n_nodes;  /* this GPU's wires / nodes                       */
  const int32_t* in_ref;     /* [n_wires] node references                      */
  const int32_t* out_ref;
  const float* inductance;   /* [n_wires]                                      */
  const float* resistance;
  const float* capacitance;
  float* current;            /* [SEGMENTS][n_wires]                            */
  float* wire_volt;          /* [SEGMENTS - 1][n_wires]                        */
  const float* node_cap;     /* [n_nodes] this GPU's nodes                     */
  const float* leakage;
  float* volt[PM_CIRCUIT_MAX_RANKS];   /* per rank: its node voltages / charges */
  float* charge[PM_CIRCUIT_MAX_RANKS];
  int32_t rank, steps;
  float dt;
} pm_circuit_view;
int pm_circuit_step(const pm_circuit_view* view, int32_t phase, void* stream);

/* Step programs: a mapped executor's per-step schedule as data, replayed by one
 * call (the C-ABI form of the executors, SURVEY §8(b) pm_run_*: the planners --
 * executors/summa.py plan_panels, grid3d.py, cannon.py cannon_schedule -- build
 * the op list once over fixed device / peer pointers; any host can build one).
 *   PM_STEP_PULL          pitched copy-engine copy dst <- src (dpitch / spitch /
 *                         width bytes x height rows, peer or local) on copy lane
 *                         `lane` (0..PM_STEP_LANES-1), or on the compute stream
 *                         when lane == -1;
 *   PM_STEP_WAIT          the compute stream waits for the lane pull at op index
 *                         `lane` (an earlier PM_STEP_PULL with lane >= 0);
 *   PM_STEP_GEMM_BF16     pm_gemm_bf16(src = A, lda, b = Bt, ldb, dst = C, ldc, m, n,
 *                         k, c_bf16, accumulate) on the compute stream;
 *   PM_STEP_GEMM_TF32     pm_gemm_tf32(src, lda, b, ldb, dst, ldc, m, n, k, accumulate);
 *   PM_STEP_MEMSET        zero `width` bytes at dst (compute stream);
 *   PM_STEP_BARRIER       pm_peer_barrier(barrier);
 *   PM_STEP_COPY_BARRIER  pm_peer_copy_barrier(barrier, copies, n_copies, ticket);
 *   PM_STEP_FORK          the lanes (re)start after everything queued so far on the
 *                         compute stream (later lane pulls follow e.g. a GEMM that
 *                         read the buffers they overwrite).
 * pm_steps_run: the lanes fork from `stream` at the first lane pull (after
 * everything already queued on it) or at a PM_STEP_FORK, and join back at the end
 * of the step; no
 * host synchronisation; capturable in a CUDA graph.  The program keeps its own
 * copy of the ops (and copy lists) but not of the memory they point to. */
#define PM_STEP_LANES 4
enum {
  PM_STEP_PULL = 0, PM_STEP_WAIT = 1, PM_STEP_GEMM_BF16 = 2, PM_STEP_GEMM_TF32 = 3,
  PM_STEP_MEMSET = 4, PM_STEP_BARRIER = 5, PM_STEP_COPY_BARRIER = 6, PM_STEP_FORK = 7
};
typedef struct pm_step_op {
  int32_t kind, lane;
  void* dst;
  const void* src;
  const void* b;
  int64_t dpitch, spitch, width, height;
  int64_t lda, ldb, ldc, m, n, k;
  int32_t c_bf16, accumulate;
  const void* barrier;            /* pm_peer_barrier_view*                     */
  const pm_peer_copy* copies;
  int32_t n_copies;
  uint32_t* ticket;
} pm_step_op;
typedef struct pm_steps pm_steps;
int pm_steps_create(const pm_step_op* ops, int32_t n, pm_steps** out);
int pm_steps_run(pm_steps* program, void* stream);
void pm_steps_destroy(pm_steps* program);

/* One phase of a PENNANT-style Lagrangian hydro step (the paper's PENNANT
 * workload, after Ferenbaugh 2015; no reference code, parity
 * against oracle/hydro.py).  Quadrilateral zones with counter-clockwise point
 * references (rank << 27) | slot, z2p[k * n_zones + z]; points per GPU.
 *   phase 0: zones -- area, PdV energy update with the previous pressure,
 *            gamma-law EOS, artificial viscosity, corner forces deposited with
 *            float2 atomics into the owning GPU's fxy (peer or local);
 *   phase 1: this GPU's points -- acceleration, wall conditions (pbc bit 0:
 *            x fixed, bit 1: y fixed), velocity / position update, force reset.
 * Phases of different GPUs must be separated by a barrier. */
#define PM_HYDRO_MAX_RANKS 16
typedef struct pm_hydro_view {
  int64_t n_zones, n_points;
  const int32_t* z2p;        /* [4][n_zones] point references                  */
  const float* zm;           /* [n_zones] zone mass                            */
  float* ze;                 /* specific internal energy                       */
  float* za;                 /* area after the last step                       */
  float* zpe;                /* p + q of the last step (0 before the first)    */
  const float* pm;           /* [n_points] point mass                          */
  const int8_t* pbc;         /* [n_points] wall flags                          */
  float* pst[PM_HYDRO_MAX_RANKS];     /* per point (x, y, u, v): 16 bytes  */
  float* fxy[PM_HYDRO_MAX_RANKS];     /* interleaved (fx, fy) per point  */
  int32_t rank;
  float dt, gamma, cq;
} pm_hydro_view;
int pm_hydro_step(const pm_hydro_view* view, int32_t phase, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MAPPLE_B200_H */
