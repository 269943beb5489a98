// K4 -- tile GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// C[M,N] (+)= A[M,K] * B[K,N], bf16 in, fp32 accumulate, B given as Bt[N,K]
// (both operands K-major).  This is the per-processor tile product of the
// mapped matmul workloads; the reference has no numeric code
// for it.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A tile 128x64 and B tile 256x64 per k-block
//               (128-byte swizzle) into a kStages-deep shared-memory ring
//   warp 1      MMA issuer: one elected thread issues 4 x tcgen05.mma
//               (M=128, N=256, K=16) per k-block into a TMEM accumulator and
//               commits the stage back to the producer
//   warp 2      TMEM allocator (512 columns = 2 accumulators x 256 fp32)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns at a time,
//               convert, store to global; the second accumulator lets the
//               MMA of tile i+1 overlap the epilogue of tile i
// Tiles are walked in M-grouped order so CTAs running at the same time share
// A row-panels and B column-panels in L2.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "pm_common.h"

namespace pm {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle atom row
constexpr int UMMA_K = 16;
constexpr int kStages = 4;
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr uint32_t kTmemCols = 512;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = kStages * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// ---- PTX helpers -------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Shared-memory matrix descriptor for a K-major tile whose rows are 128-byte
// swizzled (TMA SWIZZLE_128B): 8-row groups are 1024 bytes apart (SBO).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);       // start address
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO
  d |= (uint64_t)1 << 46;                        // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// kind::tf32 instruction descriptor: D=f32, A=B=tf32 (format 2), both K-major.
__host__ __device__ constexpr uint32_t make_idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// kind::f16 instruction descriptor: D=f32, A=B=bf16, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Params {
  int M, N, K;
  int tiles_m, tiles_n, k_blocks;
  float* c32;
  __nv_bfloat16* c16;
  long long ldc;
  int accumulate;
  int group_m;  // tile raster: group_m M-tiles advance together across N
  int debug_nostore;  // experiments only (PM_GEMM_NOSTORE): skip the C stores
  int tma_store;      // epilogue through smem + TMA bulk store (map_c valid)
  int* tile_counter;  // dynamic tile scheduler ticket (zeroed before each launch)
  int ticket_end;     // draws per launch (tiles + one terminal draw per pair): the
                      // draw ticket_end - 1 is the last and zeroes the counter
  int k_split;        // 1-SM kernel: K slices per output tile (<= 1: none); > 1 adds
                      // every slice's partial product into C with vector red.add
  int wave_slack;     // wave barrier: proceed when all but this many tiles of the
                      // previous wave have issued their last load
  int wave_sync;      // wide kernel: a tile of wave w (= ticket / pairs) starts loading
                      // only once every tile of wave w - 1 has issued its last load
                      // (tile_counter[1] counts them): the co-resident tiles then walk K
                      // in step and share their A / B panels in L2
};

__device__ __forceinline__ void tile_coords(int t, const Params& p, int& tm, int& tn) {
  // grouped raster: kGroupM M-tiles advance together across N
  const int per_group = p.group_m * p.tiles_n;
  const int g = t / per_group;
  const int first_m = g * p.group_m;
  const int gm = min(p.group_m, p.tiles_m - first_m);
  const int r = t - g * per_group;
  tm = first_m + r % gm;
  tn = r / gm;
}

// TF32 = true: fp32 operands on the tensor cores (kind::tf32, 32 fp32 = one
// 128-byte swizzle row per k-block, UMMA K = 8); same smem bytes per stage.
template <bool TF32>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_1sm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
           const Params p) {
  constexpr int BKE = TF32 ? 32 : BK;  // elements per 128-byte k-block row
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ksplit = p.k_split > 1 ? p.k_split : 1;
  const int kb_per = (p.k_blocks + ksplit - 1) / ksplit;  // k-blocks per slice
  const int ntiles = p.tiles_m * p.tiles_n * ksplit;      // (output tile, K slice) items

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int tm, tn;
        tile_coords(t / ksplit, p, tm, tn);
        const int kb0 = (t % ksplit) * kb_per, kb1 = min(p.k_blocks, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(&map_a, &full[stage], sa + stage * A_BYTES, kb * BKE, tm * BM);
          tma_load_2d(&map_b, &full[stage], sb + stage * B_BYTES, kb * BKE, tn * BN);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = TF32 ? make_idesc_tf32(BM, BN) : make_idesc(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb0 = (t % ksplit) * kb_per, kb1 = min(p.k_blocks, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sb + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            const uint64_t ad = smem_desc_sw128(a0 + k * UMMA_K * 2);
            const uint64_t bd = smem_desc_sw128(b0 + k * UMMA_K * 2);
            if constexpr (TF32)
              tc_mma_tf32(d_tmem, ad, bd, idesc, ((kb - kb0) | k) != 0);
            else
              tc_mma(d_tmem, ad, bd, idesc, ((kb - kb0) | k) != 0);
          }
          tc_commit(&empty[stage]);  // smem slot free once these MMAs retire
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else if (warp >= kEpiWarp0) {
    const int ew = warp - kEpiWarp0;  // TMEM lanes 32*ew .. 32*ew+31
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      int tm, tn;
      tile_coords(t / ksplit, p, tm, tn);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * BM + ew * 32 + lane;
      const bool row_ok = row < p.M;
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + ch * 32, v);
        const int col0 = tn * BN + ch * 32;
        if (!row_ok || col0 >= p.N) continue;
        const bool full_cols = col0 + 32 <= p.N;
        if (p.c32) {
          float* dst = p.c32 + (long long)row * p.ldc + col0;
          if (ksplit > 1) {  // slices of one tile add concurrently: vector reduction-adds
            if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + j),
                             "f"(__uint_as_float(v[j])), "f"(__uint_as_float(v[j + 1])),
                             "f"(__uint_as_float(v[j + 2])), "f"(__uint_as_float(v[j + 3]))
                             : "memory");
            } else {
              for (int j = 0; j < 32 && col0 + j < p.N; ++j)
                atomicAdd(dst + j, __uint_as_float(v[j]));
            }
          } else if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                     __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
              if (p.accumulate) {
                const float4 c = *reinterpret_cast<const float4*>(dst + j);
                o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
              }
              *reinterpret_cast<float4*>(dst + j) = o;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
              float o = __uint_as_float(v[j]);
              if (p.accumulate) o += dst[j];
              dst[j] = o;
            }
          }
        } else {
          __nv_bfloat16* dst = p.c16 + (long long)row * p.ldc + col0;
          if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint32_t w[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float x0 = __uint_as_float(v[j + 2 * q]), x1 = __uint_as_float(v[j + 2 * q + 1]);
                if (p.accumulate) {
                  x0 += __bfloat162float(dst[j + 2 * q]);
                  x1 += __bfloat162float(dst[j + 2 * q + 1]);
                }
                __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
                w[q] = *reinterpret_cast<uint32_t*>(&h);
              }
              *reinterpret_cast<uint4*>(dst + j) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
              float o = __uint_as_float(v[j]);
              if (p.accumulate) o += __bfloat162float(dst[j]);
              dst[j] = __float2bfloat16_rn(o);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

// ---- 2-CTA variant: UMMA 256x256 issued by the pair's leader ------------------
//
// A CTA pair (cluster of 2 on one TPC) owns a 256 x 256 output tile.  Each
// CTA stages its 128 rows of A and its 128 rows of Bt (half of N) per k-block;
// the leader's single thread issues tcgen05.mma.cta_group::2 (M=256, N=256,
// K=16), which reads both CTAs' shared memory and accumulates each CTA's 128
// rows into that CTA's TMEM.  Per SM this halves the operand bytes read from
// shared memory per MMA (64 B/clk instead of 96), the limit of the 1-CTA
// kernel (ncu: tensor pipe 76% active).
namespace two {

constexpr int kStages2 = 6;
constexpr int A2_BYTES = 128 * BK * 2;  // 16 KB: this CTA's 128 rows of A
constexpr int B2_BYTES = 128 * BK * 2;  // 16 KB: this CTA's 128 rows of Bt
constexpr int STAGE2 = A2_BYTES + B2_BYTES;
constexpr int SMEM2 = kStages2 * STAGE2 + 1024 + 512;
constexpr int TM = 256, TN = 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

__device__ __forceinline__ void tma_load_2sm(const CUtensorMap* map, uint32_t bar_cluster,
                                             void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void mma2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit2(uint64_t* bar) {
  // arrive on the barrier at this smem offset in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_gemm_bf16_2sm(const __grid_constant__ CUtensorMap map_a,
                const __grid_constant__ CUtensorMap map_b, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages2 * A2_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages2 * STAGE2);
  uint64_t* full = bars;                  // leader's are used (count 2)
  uint64_t* empty = bars + kStages2;      // per CTA, signalled by the leader's commit
  uint64_t* tfull = bars + 2 * kStages2;  // per CTA, signalled by the leader's commit
  uint64_t* tempty = bars + 2 * kStages2 + 2;  // leader's are used (count 8)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kStages2 + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int tiles_m = (p.M + TM - 1) / TM;
  const int tiles_n = (p.N + TN - 1) / TN;
  const int ntiles = tiles_m * tiles_n;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  auto coords = [&](int t, int& tm, int& tn) {
    const int per_group = p.group_m * tiles_n;
    const int g = t / per_group;
    const int first_m = g * p.group_m;
    const int gm = min(p.group_m, tiles_m - first_m);
    const int r = t - g * per_group;
    tm = first_m + r % gm;
    tn = r / gm;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        int tm, tn;
        coords(t, tm, tn);
        const int am = tm * TM + crank * 128;
        const int bn = tn * TN + crank * 128;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = full0 + stage * 8;
          if (leader) {
            mbar_expect_tx(&full[stage], 2 * STAGE2);
          } else {
            mbar_arrive_cluster(fb);
          }
          tma_load_2sm(&map_a, fb, sa + stage * A2_BYTES, kb * BK, am);
          tma_load_2sm(&map_b, fb, sb + stage * B2_BYTES, kb * BK, bn);
          if (++stage == kStages2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc(TM, TN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < ntiles; t += npairs, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + stage * A2_BYTES);
          const uint32_t b0 = smem_u32(sb + stage * B2_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            mma2(d_tmem, smem_desc_sw128(a0 + k * UMMA_K * 2), smem_desc_sw128(b0 + k * UMMA_K * 2),
                 idesc, (kb | k) != 0);
          }
          commit2(&empty[stage]);
          if (++stage == kStages2) { stage = 0; phase ^= 1; }
        }
        commit2(&tfull[acc]);
      }
    }
  } else if (warp >= kEpiWarp0) {
    const int ew = warp - kEpiWarp0;
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    int it = 0;
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      int tm, tn;
      coords(t, tm, tn);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * TM + crank * 128 + ew * 32 + lane;
      const bool row_ok = row < p.M;
#pragma unroll 1
      for (int ch = 0; ch < TN / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * TN + ch * 32, v);
        const int col0 = tn * TN + ch * 32;
        if (!row_ok || col0 >= p.N) continue;
        const bool full_cols = col0 + 32 <= p.N;
        if (p.c32) {
          float* dst = p.c32 + (long long)row * p.ldc + col0;
          if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                     __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
              if (p.accumulate) {
                const float4 c = *reinterpret_cast<const float4*>(dst + j);
                o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
              }
              *reinterpret_cast<float4*>(dst + j) = o;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
              float o = __uint_as_float(v[j]);
              if (p.accumulate) o += dst[j];
              dst[j] = o;
            }
          }
        } else {
          __nv_bfloat16* dst = p.c16 + (long long)row * p.ldc + col0;
          if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint32_t w[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float x0 = __uint_as_float(v[j + 2 * q]), x1 = __uint_as_float(v[j + 2 * q + 1]);
                if (p.accumulate) {
                  x0 += __bfloat162float(dst[j + 2 * q]);
                  x1 += __bfloat162float(dst[j + 2 * q + 1]);
                }
                __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
                w[q] = *reinterpret_cast<uint32_t*>(&h);
              }
              *reinterpret_cast<uint4*>(dst + j) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
              float o = __uint_as_float(v[j]);
              if (p.accumulate) o += __bfloat162float(dst[j]);
              dst[j] = __float2bfloat16_rn(o);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

}  // namespace two

// ---- wide 2-CTA variant: pair tile 512 x 256, CTA tile 256 x 256 ------------
//
// Same pairing as `two`, but every k-step issues two UMMA 256x256 (rows
// 0..255 and 256..511 of the pair tile) sharing the B half in shared memory,
// accumulating into the two 256-column halves of TMEM.  Per MAC this reads
// 25% fewer operand bytes from L2 than the 256x256 pair tile (ncu: the
// 256x256 kernel moved 2x the L2 bytes of cuBLAS for 16384^3), which is what
// bounds the clock under the 1 kW power cap.  With all 512 TMEM columns in
// use the accumulator is not double-buffered; instead 8 epilogue warps drain
// the two halves in parallel and the MMA of the next tile starts on a half as
// soon as that half is drained.
namespace wide {

using namespace two;

constexpr int kStagesW = 4;
constexpr int AW_BYTES = 256 * BK * 2;  // 32 KB: this CTA's 2 x 128 rows of A
constexpr int BW_BYTES = 128 * BK * 2;  // 16 KB: this CTA's 128 rows of Bt
constexpr int STAGEW = AW_BYTES + BW_BYTES;
constexpr int EPI_BUF = 32 * 32 * 4;    // per epilogue warp: one 32x32 fp32 box
constexpr int kEpiWarps = 8;
constexpr int SMEMW = kStagesW * STAGEW + kEpiWarps * EPI_BUF + 1024 + 512;
constexpr int WM = 512, WN = 256;
constexpr int kThreadsW = 384;  // warps 0-3 control, 4-7 drain half 0, 8-11 drain half 1
constexpr int kQ = 4;           // tile-queue slots
// consumers of every tile-queue slot: the non-leader producer, the leader's
// MMA thread and the 8 epilogue warps of each CTA
constexpr int kQConsumers = 1 + 1 + 2 * kEpiWarps;

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y,
                                             bool add) {
  if (add) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];"
        ::"l"(map), "r"(smem_u32(src)), "r"(x), "r"(y) : "memory");
  } else {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 ::"l"(map), "r"(smem_u32(src)), "r"(x), "r"(y) : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// One warp's 32 rows x 32 columns through shared memory and a TMA store.
// fp32: 128-byte rows, SWIZZLE_128B (16-byte chunk c of row r at c ^ (r & 7));
// bf16: 64-byte rows, SWIZZLE_64B (chunk c at c ^ ((r >> 1) & 3)).
__device__ __forceinline__ void store_chunk_tma(const CUtensorMap* map_c, bool f32, bool add,
                                                uint8_t* buf, int lane, int row0, int col0,
                                                const uint32_t (&v)[32]) {
  if (lane == 0) bulk_wait_read0();  // previous store out of this buffer has read it
  __syncwarp();
  if (f32) {
    uint8_t* rowp = buf + lane * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t a = smem_u32(rowp + ((c ^ (lane & 7)) << 4));
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v[4 * c]),
                   "r"(v[4 * c + 1]), "r"(v[4 * c + 2]), "r"(v[4 * c + 3])
                   : "memory");
    }
  } else {
    uint8_t* rowp = buf + lane * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[8 * c + 2 * q]),
                                                 __uint_as_float(v[8 * c + 2 * q + 1]));
        w[q] = *reinterpret_cast<uint32_t*>(&h);
      }
      const uint32_t a = smem_u32(rowp + ((c ^ ((lane >> 1) & 3)) << 4));
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]),
                   "r"(w[2]), "r"(w[3])
                   : "memory");
    }
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) tma_store_2d(map_c, buf, col0, row0, add);
}

__device__ __forceinline__ void store_chunk(const Params& p, int row, int col0,
                                            const uint32_t (&v)[32]) {
  if (row >= p.M || col0 >= p.N || p.debug_nostore) return;
  const bool full_cols = col0 + 32 <= p.N;
  if (p.c32) {
    float* dst = p.c32 + (long long)row * p.ldc + col0;
    if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                               __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        if (p.accumulate) {
          const float4 c = *reinterpret_cast<const float4*>(dst + j);
          o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
        }
        *reinterpret_cast<float4*>(dst + j) = o;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
        float o = __uint_as_float(v[j]);
        if (p.accumulate) o += dst[j];
        dst[j] = o;
      }
    }
  } else {
    __nv_bfloat16* dst = p.c16 + (long long)row * p.ldc + col0;
    if (full_cols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float x0 = __uint_as_float(v[j + 2 * q]), x1 = __uint_as_float(v[j + 2 * q + 1]);
          if (p.accumulate) {
            x0 += __bfloat162float(dst[j + 2 * q]);
            x1 += __bfloat162float(dst[j + 2 * q + 1]);
          }
          __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
          w[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(dst + j) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
        float o = __uint_as_float(v[j]);
        if (p.accumulate) o += __bfloat162float(dst[j]);
        dst[j] = __float2bfloat16_rn(o);
      }
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsW, 1)
k_gemm_bf16_wide(const __grid_constant__ CUtensorMap map_a,
                 const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_c, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStagesW * AW_BYTES;
  uint8_t* epi = smem + kStagesW * STAGEW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + kEpiWarps * EPI_BUF);
  uint64_t* full = bars;                    // leader's (count 2)
  uint64_t* empty = bars + kStagesW;        // per CTA (leader's commit)
  uint64_t* tfull = bars + 2 * kStagesW;    // per CTA (leader's commit)
  uint64_t* tempty = bars + 2 * kStagesW + 1;  // [2] leader's, count 16 each
  uint64_t* qfull = bars + 2 * kStagesW + 3;   // [kQ] per CTA: tile index published
  uint64_t* qempty = qfull + kQ;               // [kQ] leader's: all consumers read it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(qempty + kQ);
  int* tileq = reinterpret_cast<int*>(tmem_holder + 4);  // [kQ] tile ring

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int tiles_m = (p.M + WM - 1) / WM;
  const int tiles_n = (p.N + WN - 1) / WN;
  const int ntiles = tiles_m * tiles_n;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStagesW; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 16);  // 8 epilogue warps x 2 CTAs per TMEM half
    mbar_init(&tempty[1], 16);
    for (int i = 0; i < kQ; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], kQConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // Dynamic tile scheduler: the leader's producer draws tiles from a global
  // ticket and publishes them through a kQ-slot ring in both CTAs; every role
  // of both CTAs walks the same sequence.  Tiles therefore run in raster order
  // of their start time, so the tiles resident at any moment stay contiguous
  // in the grouped raster and share A/B panels in L2 -- with a static
  // round-robin the pairs drift apart over ~100 waves and L2 reuse collapses
  // (ncu: 211 GB DRAM reads for one 32768^3 launch).
  const uint32_t qempty0 = mapa_shared(smem_u32(&qempty[0]), 0);
  int q_slot = 0;
  uint32_t q_phase = 0;
  auto next_tile = [&]() -> int {  // consumers: wait, read, release the slot
    mbar_wait_cluster(&qfull[q_slot], q_phase);
    const int t = *(volatile int*)&tileq[q_slot];
    mbar_arrive_cluster(qempty0 + q_slot * 8);
    if (++q_slot == kQ) { q_slot = 0; q_phase ^= 1; }
    return t;
  };
  auto publish_tile = [&]() -> int {  // leader producer: draw and publish
    mbar_wait(&qempty[q_slot], q_phase ^ 1);
    const int t = atomicAdd(p.tile_counter, 1);
    if (t == p.ticket_end - 1) atomicExch(p.tile_counter, 0);  // every pair has drawn
    tileq[q_slot] = t;
    const uint32_t peer_q = mapa_shared(smem_u32(&tileq[q_slot]), 1);
    asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(peer_q), "r"(t) : "memory");
    mbar_arrive(&qfull[q_slot]);
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                     mapa_shared(smem_u32(&qfull[q_slot]), 1))
                 : "memory");
    if (++q_slot == kQ) { q_slot = 0; q_phase ^= 1; }
    return t;
  };

  auto coords = [&](int t, int& tm, int& tn) {
    const int per_group = p.group_m * tiles_n;
    const int g = t / per_group;
    const int first_m = g * p.group_m;
    const int gm = min(p.group_m, tiles_m - first_m);
    const int r = t - g * per_group;
    tm = first_m + r % gm;
    tn = r / gm;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (;;) {
        const int t = leader ? publish_tile() : next_tile();
        if (t >= ntiles) break;
        int tm, tn;
        coords(t, tm, tn);
        const int am = tm * WM + crank * 128;
        const int bn = tn * WN + crank * 128;
        if (p.wave_sync && leader) {
          // wave barrier: every tile of the previous wave has issued its last load.  A
          // hint, not a correctness condition: a pair gives up after 2 ms (e.g. when
          // another kernel keeps some pairs from being resident), so it cannot hang
          const int need = (t / npairs) * npairs - p.wave_slack;
          volatile int* done = p.tile_counter + 1;
          if (*done < need) {
            unsigned long long t0, t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            do {
              __nanosleep(128);
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            } while (*done < need && t1 - t0 < 2000000ull);
          }
        }
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = full0 + stage * 8;
          if (leader) {
            mbar_expect_tx(&full[stage], 2 * STAGEW);
          } else {
            mbar_arrive_cluster(fb);
          }
          uint8_t* a = sa + stage * AW_BYTES;
          tma_load_2sm(&map_a, fb, a, kb * BK, am);
          tma_load_2sm(&map_a, fb, a + AW_BYTES / 2, kb * BK, am + 256);
          tma_load_2sm(&map_b, fb, sb + stage * BW_BYTES, kb * BK, bn);
          if (++stage == kStagesW) { stage = 0; phase ^= 1; }
        }
        if (p.wave_sync && leader) atomicAdd(p.tile_counter + 1, 1);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc(256, WN);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        if (next_tile() >= ntiles) break;
        const uint32_t tphase = it & 1;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + stage * AW_BYTES);
          const uint32_t b0 = smem_u32(sb + stage * BW_BYTES);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (kb == 0) {  // this half of TMEM must be drained by the epilogue
              mbar_wait(&tempty[h], tphase ^ 1);
              tc_fence_after();
            }
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              mma2(tmem_base + h * WN, smem_desc_sw128(a0 + h * (AW_BYTES / 2) + k * UMMA_K * 2),
                   smem_desc_sw128(b0 + k * UMMA_K * 2), idesc, (kb | k) != 0);
            }
          }
          commit2(&empty[stage]);
          if (++stage == kStagesW) { stage = 0; phase ^= 1; }
        }
        commit2(&tfull[0]);
      }
    }
  } else if (warp >= 4) {
    // all 8 epilogue warps drain TMEM half 0 first, then half 1 (warp j of a lane
    // quarter takes column chunks 4j .. 4j + 3 of each half): half 0 is free for the
    // next tile's MMAs after half of the drain time
    const int j = (warp - 4) >> 2;  // column half of each TMEM half drained by this warp
    const int q = warp & 3;         // TMEM lane quarter this warp may access
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    for (int it = 0;; ++it) {
      int t = 0;
      if (lane == 0) t = next_tile();
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) break;
      int tm, tn;
      coords(t, tm, tn);
      mbar_wait(&tfull[0], it & 1);
      tc_fence_after();
      uint8_t* buf = epi + (warp - 4) * EPI_BUF;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int row0 = tm * WM + h * 256 + crank * 128 + q * 32;
#pragma unroll 1
        for (int ch = 4 * j; ch < 4 * j + WN / 64; ++ch) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + h * WN + ch * 32, v);
          if (p.tma_store) {
            if (!p.debug_nostore)
              store_chunk_tma(&map_c, p.c32 != nullptr, p.accumulate != 0, buf, lane, row0,
                              tn * WN + ch * 32, v);
          } else {
            store_chunk(p, row0 + lane, tn * WN + ch * 32, v);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + 8 * h);
      }
    }
    if (lane == 0) {
      // the TMA stores / reduce-adds (async proxy, possibly into a peer GPU's C) have
      // completed; publish them at system scope before the kernel retires, so work
      // ordered after this kernel on any GPU (e.g. a stream-ordered NCCL barrier)
      // observes them
      bulk_wait0();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence_system();
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

}  // namespace wide

int make_map(const Driver* d, CUtensorMap* map, const void* base, long long rows, long long cols,
             long long ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = d->tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                       const_cast<void*>(base), dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: CUresult %d", (int)r);
    return PM_ERR_CUDA;
  }
  return PM_OK;
}

int make_map_f32(const Driver* d, CUtensorMap* map, const void* base, long long rows,
                 long long cols, long long ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = d->tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                       const_cast<void*>(base), dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(f32) failed: CUresult %d", (int)r);
    return PM_ERR_CUDA;
  }
  return PM_OK;
}

}  // namespace gemm
}  // namespace pm

extern "C" int pm_gemm_tf32(const float* A, int64_t lda, const float* Bt, int64_t ldb, float* C,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t accumulate,
                            void* stream) {
  using namespace pm::gemm;
  if (!A || !Bt || !C || M <= 0 || N <= 0 || K <= 0 || lda < K || ldb < K || ldc < N)
    return pm::set_error("pm_gemm_tf32: bad arguments"), PM_ERR_INVALID;
  if ((lda % 4) || (ldb % 4) || ((uintptr_t)A % 16) || ((uintptr_t)Bt % 16))
    return pm::set_error("pm_gemm_tf32: A/Bt need 16-byte aligned rows (ld % 4 == 0)"),
           PM_ERR_UNSUPPORTED;
  if (M > (1LL << 31) || N > (1LL << 31) || K > (1LL << 31))
    return pm::set_error("pm_gemm_tf32: dimension too large"), PM_ERR_UNSUPPORTED;
  const pm::Driver* d = pm::driver();
  if (!d) return PM_ERR_CUDA;
  CUtensorMap ma, mb;
  int rc = make_map_f32(d, &ma, A, M, K, lda, BM);
  if (rc) return rc;
  rc = make_map_f32(d, &mb, Bt, N, K, ldb, BN);
  if (rc) return rc;
  Params p{};
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.tiles_n = (int)((N + BN - 1) / BN);
  p.k_blocks = (int)((K + 31) / 32);
  p.c32 = C;
  p.ldc = ldc;
  p.accumulate = accumulate != 0;
  p.group_m = 8;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return pm::set_error("pm_gemm_tf32: device id"), PM_ERR_UNSUPPORTED;
  if (!attr_done[dev]) {
    PM_CUDA_TRY(cudaFuncSetAttribute(k_gemm_1sm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SMEM_BYTES));
    attr_done[dev] = true;
  }
  const long long tiles = (long long)p.tiles_m * p.tiles_n;
  // few output tiles (small products, e.g. Cannon's 512^3 blocks): split K over the idle
  // SMs, every slice reduction-adding into C (zeroed first unless accumulating)
  const int sms = pm::num_sms();
  int ks = 1;
  if (tiles * 2 <= sms && p.k_blocks >= 8) {
    ks = (int)std::min<long long>(sms / tiles, p.k_blocks / 4);
    const int kb_per = (p.k_blocks + ks - 1) / ks;
    ks = (p.k_blocks + kb_per - 1) / kb_per;  // no empty slice
  }
  if (ks > 1) {
    p.k_split = ks;
    if (!p.accumulate)
      PM_CUDA_TRY(cudaMemset2DAsync(C, ldc * sizeof(float), 0, N * sizeof(float), M,
                                    (cudaStream_t)stream));
  }
  const long long ntiles = tiles * ks;
  int grid = sms;
  if (ntiles < grid) grid = (int)ntiles;
  k_gemm_1sm<true><<<grid, kThreads, SMEM_BYTES, (cudaStream_t)stream>>>(ma, mb, p);
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}

namespace pm::gemm {
// Scheduler tickets (4-byte counters, one per 128-byte line): per (device,
// stream) for eager launches, fresh for each captured launch.  Never freed --
// library scratch that lives as long as the process, like the module state.
static int tile_ticket(int dev, void* stream, int** out) {
  static std::mutex mu;
  static std::map<std::pair<int, void*>, int*> per_stream;
  static int* pool[64] = {nullptr};
  static int pool_used[64] = {0};
  constexpr int kPool = 256;
  std::lock_guard<std::mutex> lock(mu);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PM_CUDA_TRY(cudaStreamIsCapturing((cudaStream_t)stream, &cs));
  const bool captured = cs != cudaStreamCaptureStatusNone;
  if (!captured) {
    auto it = per_stream.find({dev, stream});
    if (it != per_stream.end()) return *out = it->second, PM_OK;
  }
  if (!pool[dev] || pool_used[dev] == kPool) {
    // a new block (cudaMalloc is legal during a capture only in relaxed mode;
    // every launch zeroes its ticket with a stream-ordered memset, so the block
    // needs no initialisation)
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    PM_CUDA_TRY(cudaThreadExchangeStreamCaptureMode(&mode));
    cudaError_t e = cudaMalloc(&pool[dev], kPool * 128);
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (e != cudaSuccess)
      return pm::set_error("tile ticket allocation: %s", cudaGetErrorString(e)), PM_ERR_CUDA;
    pool_used[dev] = 0;
  }
  int* t = pool[dev] + 32 * pool_used[dev]++;
  if (!captured) per_stream[{dev, stream}] = t;
  return *out = t, PM_OK;
}
}  // namespace pm::gemm

extern "C" int pm_gemm_bf16(const void* A, int64_t lda, const void* Bt, int64_t ldb, void* C,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t c_bf16,
                            int32_t accumulate, void* stream) {
  using namespace pm::gemm;
  if (!A || !Bt || !C || M <= 0 || N <= 0 || K <= 0 || lda < K || ldb < K || ldc < N)
    return pm::set_error("pm_gemm_bf16: bad arguments"), PM_ERR_INVALID;
  if ((lda % 8) || (ldb % 8) || ((uintptr_t)A % 16) || ((uintptr_t)Bt % 16))
    return pm::set_error("pm_gemm_bf16: A/Bt need 16-byte aligned rows (ld % 8 == 0)"),
           PM_ERR_UNSUPPORTED;
  if (M > (1LL << 31) || N > (1LL << 31) || K > (1LL << 31))
    return pm::set_error("pm_gemm_bf16: dimension too large"), PM_ERR_UNSUPPORTED;
  const pm::Driver* d = pm::driver();
  if (!d) return PM_ERR_CUDA;
  // kernel choice: 0 = 1-CTA 128x256, 1 = CTA pair 256x256, 2 = CTA pair 512x256
  int kind = M <= 128 ? 0 : (M >= 1024 && N >= 256) ? 2 : 1;
  if (const char* k = getenv("PM_GEMM_KERNEL")) kind = atoi(k);
  // accumulate == 2: element-wise atomic reduce-add (TMA .add), e.g. several
  // GPUs adding partial products into one C over NVLink
  const bool atomic_add = accumulate == 2;
  if (atomic_add) {
    if (c_bf16) return pm::set_error("pm_gemm_bf16: atomic accumulate needs fp32 C"), PM_ERR_UNSUPPORTED;
    kind = 2;
  }
  const bool pair = kind != 0;
  CUtensorMap ma, mb;
  int rc = make_map(d, &ma, A, M, K, lda, BM);
  if (rc) return rc;
  rc = make_map(d, &mb, Bt, N, K, ldb, pair ? 128 : BN);
  if (rc) return rc;
  Params p{};
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.tiles_n = (int)((N + BN - 1) / BN);
  p.k_blocks = (int)((K + BK - 1) / BK);
  p.c32 = c_bf16 ? nullptr : reinterpret_cast<float*>(C);
  p.c16 = c_bf16 ? reinterpret_cast<__nv_bfloat16*>(C) : nullptr;
  p.ldc = ldc;
  p.accumulate = accumulate != 0;
  // raster group (M-tiles per group): long K panels do not fit L2, so narrow
  // groups re-read less from HBM (sustained sweep: K=32768 g2 1270 TF/s vs g6
  // 1151; K=16384 g4 best)
  // wide kernel with the wave barrier (default): the co-resident tiles walk K in step,
  // so a 4-row raster group shares A panels across ~18 tiles and B panels across 4 while
  // they are in L2 (32768^3: 97 -> 52 GB DRAM reads, +9% clock under the power cap,
  // 1290 -> 1412 TF/s sustained, cuBLAS 1328); without it narrow groups re-read less
  // (reduce-adding launches -- C in a peer's memory -- measured the same with and without
  // it, and with half a wave of slack: Johnson (1,1,2) / (1,2,2) within +-2% run to run,
  // tools/grid3d_ab2.sh)
  // Not for reduce-adding launches (C in a peer's memory: the 3-D / 2.5D fused
  // reduce-scatter): wave-aligned tiles would all drain over NVLink at once -- interleaved
  // single launches into a peer, 16384^3 6.76 -> 6.32 ms and 16384x32768x16384 13.34 ->
  // 12.71 ms without it (tools/remote_add_probe.py); PM_GEMM_ADD_WAVE=1 keeps it
  static const bool add_wave = getenv("PM_GEMM_ADD_WAVE") != nullptr;
  const bool wave = kind == 2 && (!atomic_add || add_wave) &&
                    !(getenv("PM_GEMM_WAVESYNC") && atoi(getenv("PM_GEMM_WAVESYNC")) == 0);
  p.group_m = kind == 2 ? (wave ? 4 : (K >= 24576 ? 2 : 4)) : 8;
  if (const char* g = getenv("PM_GEMM_GROUP")) p.group_m = atoi(g) > 0 ? atoi(g) : p.group_m;
  p.debug_nostore = getenv("PM_GEMM_NOSTORE") ? 1 : 0;
  static bool attr_done[64] = {false};
  static std::mutex init_mu;
  std::lock_guard<std::mutex> init_lock(init_mu);  // the per-device statics below
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return pm::set_error("pm_gemm_bf16: device id"), PM_ERR_UNSUPPORTED;
  if (!attr_done[dev]) {
    PM_CUDA_TRY(cudaFuncSetAttribute(k_gemm_1sm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SMEM_BYTES));
    PM_CUDA_TRY(cudaFuncSetAttribute(k_gemm_1sm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SMEM_BYTES));
    PM_CUDA_TRY(cudaFuncSetAttribute(two::k_gemm_bf16_2sm,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, two::SMEM2));
    PM_CUDA_TRY(cudaFuncSetAttribute(wide::k_gemm_bf16_wide,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, wide::SMEMW));
    attr_done[dev] = true;
  }
  if (pair) {
    // persistent grid = the number of CTA pairs that can be co-resident
    const bool use_wide = kind == 2;
    static int max_pairs[64][2] = {{0}};
    int& mp = max_pairs[dev][use_wide];
    if (!mp) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = 2;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.gridDim = dim3(2 * (pm::num_sms() / 2));
      cfg.blockDim = dim3(use_wide ? wide::kThreadsW : kThreads);
      cfg.dynamicSmemBytes = use_wide ? wide::SMEMW : two::SMEM2;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int n = 0;
      cudaError_t e = use_wide ? cudaOccupancyMaxActiveClusters(&n, wide::k_gemm_bf16_wide, &cfg)
                               : cudaOccupancyMaxActiveClusters(&n, two::k_gemm_bf16_2sm, &cfg);
      if (e != cudaSuccess || n <= 0) n = pm::num_sms() / 2;
      mp = n;
      if (getenv("PM_GEMM_DEBUG")) fprintf(stderr, "pm_gemm: %d co-resident CTA pairs\n", n);
    }
    const long long tm = use_wide ? wide::WM : two::TM, tn = use_wide ? wide::WN : two::TN;
    const long long pairs_needed = ((M + tm - 1) / tm) * ((N + tn - 1) / tn);
    long long pairs = mp;
    if (pairs_needed < pairs) pairs = pairs_needed;
    if (use_wide) {
      CUtensorMap mc;
      std::memset(&mc, 0, sizeof(mc));
      const int esize = c_bf16 ? 2 : 4;
      p.tma_store = ((ldc * esize) % 16 == 0) && ((uintptr_t)C % 16 == 0) &&
                    !(accumulate && c_bf16) && !getenv("PM_GEMM_DIRECT_STORE");
      if (atomic_add && !p.tma_store)
        return pm::set_error("pm_gemm_bf16: atomic accumulate needs ldc %% 4 == 0 and a "
                             "16-byte aligned C"), PM_ERR_UNSUPPORTED;
      if (p.tma_store) {
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)(ldc * esize)};
        cuuint32_t box[2] = {32, 32};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = d->tensorMapEncodeTiled(
            &mc, c_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C,
            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            c_bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
          return pm::set_error("cuTensorMapEncodeTiled(C) failed: %d", (int)r), PM_ERR_CUDA;
      }
      // tile-scheduler ticket: one counter per (device, stream) -- launches on
      // one stream are serialised, so they may share it -- and a dedicated one
      // for every launch captured into a CUDA graph (a replay then never shares
      // its ticket with an eager launch).  The kernel's last draw zeroes it
      // again (self-resetting); the stream-ordered memset keeps a launch safe
      // even after an aborted one.
      rc = tile_ticket(dev, stream, &p.tile_counter);
      if (rc) return rc;
      p.ticket_end = (int)(pairs_needed + pairs);
      p.wave_sync = wave ? 1 : 0;
      p.wave_slack = getenv("PM_GEMM_WAVE_SLACK") ? atoi(getenv("PM_GEMM_WAVE_SLACK")) : 0;
      PM_CUDA_TRY(cudaMemsetAsync(p.tile_counter, 0, 2 * sizeof(int), (cudaStream_t)stream));
      wide::k_gemm_bf16_wide<<<(unsigned)(2 * pairs), wide::kThreadsW, wide::SMEMW,
                               (cudaStream_t)stream>>>(ma, mb, mc, p);
    } else {
      two::k_gemm_bf16_2sm<<<(unsigned)(2 * pairs), kThreads, two::SMEM2,
                             (cudaStream_t)stream>>>(ma, mb, p);
    }
    PM_CUDA_TRY(cudaGetLastError());
    return PM_OK;
  }
  const long long ntiles = (long long)p.tiles_m * p.tiles_n;
  int grid = pm::num_sms();
  if (ntiles < grid) grid = (int)ntiles;
  k_gemm_1sm<false><<<grid, kThreads, SMEM_BYTES, (cudaStream_t)stream>>>(ma, mb, p);
  PM_CUDA_TRY(cudaGetLastError());
  return PM_OK;
}
