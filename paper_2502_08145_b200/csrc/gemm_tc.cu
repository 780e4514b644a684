// gemm_tc.cu — the three local products of Algorithm 1 on the sm_100a tensor cores.
//
//   line 3  O^  = I  x W     -> op NN: A K-major,  B MN-major
//   line 11  dI^ = dO x W^T   -> op NT: A K-major,  B K-major
//   line 13  dW  = I^T x dO   -> op TN: A MN-major, B MN-major
//
// The paper tuned cuBLAS/rocBLAS NN/NT/TN modes because its
// TN kernel ran at 6% of peak.  On tcgen05 the operand major is two bits of the
// instruction descriptor, so all three products are one kernel template that
// stages operands with TMA in the layout they already have in HBM — no
// transposes, no mode tuner.
//
// Two kernels:
//   gemm_bf16_tcgen05       1-CTA reference variant (AXONN_GEMM_VARIANT=single):
//     warp 0 TMA producer, warp 1 MMA issuer (tcgen05.mma 128x256x16), warp 2
//     TMEM allocator (two 128x256 fp32 accumulators), warps 4..7 epilogue;
//     BM=128, BN=256, BK=64, 4 stages.
//   gemm_bf16_tcgen05_pair  the product path (below): CTA pairs
//     (cta_group::2), 512x256 or 256x256 pair tiles, dynamic tile scheduling,
//     a stream-K tail for partial waves (SkParams), an 8-warp epilogue that
//     releases the accumulator as soon as it is in registers (both sub-tiles
//     first in the 4-stage variant, with setmaxnreg), TMA-store or fused
//     NVLink epilogues (EpiTarget: red.add pair, multimem.red, exchange,
//     scatter, ...), an optional memory-bound side task for the idle helper
//     warps (SideSum), and programmatic dependent launch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "gemm.h"
#include "ptx.cuh"

namespace axonn {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int THREADS = 256;
constexpr int SMEM_A = BM * BK * 2;  // 16 KiB
constexpr int SMEM_B = BN * BK * 2;  // 32 KiB
constexpr int STAGE_BYTES = SMEM_A + SMEM_B;
constexpr int TMEM_COLS = 2 * BN;    // two fp32 accumulators
constexpr int MN_CHUNK = 64;         // MN-major operands: 64-element (128 B) chunks
constexpr int MN_CHUNK_BYTES = MN_CHUNK * BK * 2;  // 8 KiB, the LBO of MN-major tiles
constexpr int GROUP_M = 16;          // tile raster: bands of 16 M-tiles for L2 reuse
constexpr size_t SMEM_BYTES = 1024 /*align*/ + STAGES * STAGE_BYTES + 256 /*barriers*/;

struct TileCoord {
  int m0, n0;
};

__device__ __forceinline__ TileCoord tile_coord(int t, int tiles_m, int tiles_n) {
  const int per_group = GROUP_M * tiles_n;
  const int g = t / per_group;
  const int first_m = g * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int r = t - g * per_group;
  return {(first_m + r % gm) * BM, (r / gm) * BN};
}


__device__ __forceinline__ TileCoord tile_coord_g(int t, int tiles_m, int tiles_n, int group_m,
                                                  int bm, int bn) {
  if (group_m < 0) {  // bands of -group_m N-tiles, M fastest... transposed raster
    const int gn_sz = -group_m;
    const int per_group = gn_sz * tiles_m;
    const int g = t / per_group;
    const int first_n = g * gn_sz;
    const int gn = min(tiles_n - first_n, gn_sz);
    const int r = t - g * per_group;
    return {(r / gn) * bm, (first_n + r % gn) * bn};
  }
  const int per_group = group_m * tiles_n;
  const int g = t / per_group;
  const int first_m = g * group_m;
  const int gm = min(tiles_m - first_m, group_m);
  const int r = t - g * per_group;
  return {(first_m + r % gm) * bm, (r / gm) * bn};
}

// A_MN / B_MN: 0 = operand stored K-major in HBM, 1 = stored MN-major.
template <int A_MN, int B_MN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, __nv_bfloat16* __restrict__ C,
                      int64_t ldc, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * SMEM_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * SMEM_B);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const TileCoord tc = tile_coord(t, tiles_m, tiles_n);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          const int k0 = kb * BK;
          uint8_t* a_dst = sA + stage * SMEM_A;
          uint8_t* b_dst = sB + stage * SMEM_B;
          if (A_MN == 0) {
            ptx::tma_load_2d(a_dst, &tmA, &full[stage], k0, tc.m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / MN_CHUNK; ++c)
              ptx::tma_load_2d(a_dst + c * MN_CHUNK_BYTES, &tmA, &full[stage], tc.m0 + c * MN_CHUNK, k0);
          }
          if (B_MN == 0) {
            ptx::tma_load_2d(b_dst, &tmB, &full[stage], k0, tc.n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / MN_CHUNK; ++c)
              ptx::tma_load_2d(b_dst + c * MN_CHUNK_BYTES, &tmB, &full[stage], tc.n0 + c * MN_CHUNK, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(sA + stage * SMEM_A);
          const uint32_t b_base = ptx::smem_u32(sB + stage * SMEM_B);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: advance 16 elements = 32 B inside the 128-B swizzle row.
            // MN-major: advance 16 K-rows = two 1024-B swizzle atoms.
            const uint64_t ad = A_MN ? ptx::sdesc_sw128(a_base + kk * 2048, MN_CHUNK_BYTES, 1024)
                                     : ptx::sdesc_sw128(a_base + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::sdesc_sw128(b_base + kk * 2048, MN_CHUNK_BYTES, 1024)
                                     : ptx::sdesc_sw128(b_base + kk * 32, 16, 1024);
            ptx::umma_f16(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          ptx::umma_commit(&empty[stage]);  // smem slot free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit(&tfull[acc]);      // accumulator complete
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // --------------------------------------------------------- epilogue
    const int e = warp - 4;  // TMEM lanes 32e .. 32e+31 (warp % 4 == e)
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec_ok = ((ldc & 7) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const TileCoord tc = tile_coord(t, tiles_m, tiles_n);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int row = tc.m0 + 32 * e + lane;
      __nv_bfloat16* crow = C + static_cast<int64_t>(row) * ldc;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * e) << 16) +
                               static_cast<uint32_t>(acc * BN + c * 32);
        ptx::tmem_ld_32x32b_x32(taddr, v);
        ptx::tmem_wait_ld();
        const int col0 = tc.n0 + c * 32;
        if (row < M && col0 < N) {
          if (vec_ok && col0 + 32 <= N) {
            uint4* dst = reinterpret_cast<uint4*>(crow + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 w;
              w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
              w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
              w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
              w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
              dst[q] = w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (col0 + q < N) crow[col0 + q] = __float2bfloat16_rn(__uint_as_float(v[q]));
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, TMEM_COLS);
}


// ===================================================================== 2-CTA
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// (256*MT) x 256 tile; CTA r owns rows [r*128*MT, (r+1)*128*MT) of it.  Per
// 64-wide K block each CTA stages its 128*MT rows of A and 128 rows (N/2) of
// B; the leader issues MT tcgen05.mma.cta_group::2 (M=256, N=256, K=16) per
// K=16 step — MMA mt reads rows [mt*128, mt*128+128) of both CTAs' A and both
// halves of B — accumulating into TMEM columns [mt*256, mt*256+256).
//   MT = 1: 256x256 tile, 5 stages of 32 KiB, two accumulators (the epilogue
//           of tile i overlaps the main loop of tile i+1);
//   MT = 2: 512x256 tile, 4 stages of 48 KiB (DEEP; 3 with AXONN_MT2_DEEP=0),
//           one accumulator filling all 512 TMEM columns: 33% more flops per
//           byte staged from L2 and a quarter fewer operand-panel reads per
//           GEMM, which lowers L2/DRAM traffic and power (the B200 runs
//           power-capped under this load).
template <int MT, int DEEP = 0>
struct PairCfg {
  static constexpr int ROWS_CTA = 128 * MT;
  static constexpr int BM = 256 * MT;
  static constexpr int BN = 256;
  // DEEP (MT = 2 only): a 4th operand stage in place of the second epilogue
  // staging box, so the next tile's first 4 K-blocks (not 3) accumulate into
  // sub-tile 0 while the epilogue still drains sub-tile 1
  static constexpr int STAGES = MT == 1 ? 5 : (DEEP ? 4 : 3);
  static constexpr int ACC = 2 / MT;                // accumulator buffers in TMEM
  static constexpr int SMEM_A = ROWS_CTA * BK * 2;
  static constexpr int SMEM_B = 128 * BK * 2;
  static constexpr int STAGE_BYTES = SMEM_A + SMEM_B;
  static constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, each owning half the columns
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  // per warp: 32 x 64 bf16 staging boxes; with two, the TMA store of one overlaps filling the other
  static constexpr int EPI_BOXES = DEEP ? 1 : 2;
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_BOXES * 32 * 64 * 2;
  // + the kXSum unit ring (256 entries) and its counters
  static constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + 256 + 1024 + 32;
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// ------------------------------------------------------------ stream-K tail
// When a launch's tiles do not fill whole waves of CTA pairs (e.g. the C2 proj
// dW: 128 tiles of 512x256 over 74 pairs, 1.73 waves), the first
// `sk_tiles` = (tiles mod pairs) + pairs tiles in raster order are split along K:
// their sk_tiles x num_kb K-blocks are dealt out evenly, pair c taking the
// contiguous range [u0, u1) (at least one tile's worth, so a tile has at most
// two pieces).  Pair c processes, in order: the HEAD of the tile its range
// ends in (K-blocks [0, h): the contributor, fp32 partial sums to a
// workspace), the whole tiles inside its range, and the TAIL of the tile its
// range starts in (K-blocks [t0, num_kb): the finisher, which adds pair c-1's
// partial sums before the epilogue proper).  Every pair then draws the
// remaining tiles (whole waves) from the dynamic tile counter.
//
// No pair ever waits on a pair that has not started: the contributor claims
// its HEAD (claim 0 -> 1) when its producer reaches it (its first item); a
// finisher that finds the claim still 0 takes the whole tile itself (0 -> 2,
// role WHOLE) and the contributor, seeing 2, skips its HEAD and resets the
// claim.  A finisher therefore only waits on a running pair, so a grid that
// is not fully resident still completes.  Claims and ready flags return to 0
// by the end of every launch.  The sums are deterministic: fixed split points
// and one fixed addition order (partial of K-blocks [0, t0) + the rest).
struct SkParams {
  int sk_tiles = 0;         // tiles [0, sk_tiles) split along K; 0 = off
  int units = 0;            // sk_tiles * num_kb
  float4* ws = nullptr;     // per SK tile: 2 CTAs x MT x 8 warps x 4 x 8 x 32 float4
  int* claim = nullptr;     // per SK tile
  int* ready = nullptr;     // per SK tile x 2 CTAs x 8 epilogue warps
};

enum : int { kRoleFull = 0, kRoleHead = 1, kRoleTail = 2, kRoleWhole = 3 };

__host__ __device__ __forceinline__ int item_tile(int it) { return it & 0x0FFFFFFF; }
__host__ __device__ __forceinline__ int item_role(int it) { return static_cast<int>(static_cast<unsigned>(it) >> 28); }
__host__ __device__ __forceinline__ int make_item(int tile, int role) { return tile | (role << 28); }

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys_i(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_i(int* p, int v) {
  asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ldcg_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_cg_f4(const float4* p) {  // L2 only: written by another SM
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t addf(uint32_t a, float b) {
  return __float_as_uint(__uint_as_float(a) + b);
}

// the idx-th stream-K item of the pair owning K-block range [u0, u1)
// (HEAD, whole tiles, TAIL), or -1 past the end
__host__ __device__ __forceinline__ int sk_static_item(int u0, int u1, int kb, int idx) {
  int n = 0;
  if (u1 % kb) {
    if (idx == n) return make_item(u1 / kb, kRoleHead);
    ++n;
  }
  const int f0 = (u0 + kb - 1) / kb, f1 = u1 / kb;
  if (f1 > f0) {
    if (idx < n + (f1 - f0)) return make_item(f0 + idx - n, kRoleFull);
    n += f1 - f0;
  }
  if (u0 % kb) {
    if (idx == n) return make_item(u0 / kb, kRoleTail);
  }
  return -1;
}

// K-block range of an item for the pair owning [u0, u1)
__host__ __device__ __forceinline__ void item_kb(int it, int u0, int u1, int kb, int* kb0,
                                                 int* kb1) {
  const int t = item_tile(it), r = item_role(it);
  *kb0 = r == kRoleTail ? u0 - t * kb : 0;
  *kb1 = r == kRoleHead ? u1 - t * kb : kb;
}

// OUTF = 1: fp32 output (the dW GEMM when gradients are reduced in fp32,
// SURVEY.md §8(f) f-4): the accumulator is stored without rounding.
template <int A_MN, int B_MN, int MT, int OUTF, int DEEP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<MT, DEEP>::THREADS, 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmC, int use_tma_store,
                           void* __restrict__ Cv, int64_t ldc, int M, int N, int K,
                           int split_release,
                           int group_m, const __grid_constant__ EpiTarget epi,
                           int* __restrict__ tile_counter, const __grid_constant__ SkParams sk,
                           const __grid_constant__ SideSum side) {
  using Cfg = PairCfg<MT, DEEP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::SMEM_A;
  uint8_t* sEpi = sB + Cfg::STAGES * Cfg::SMEM_B;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + Cfg::EPI_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* tq_full = tempty + 2;     // tile queue (dynamic scheduling), both CTAs
  uint64_t* tq_empty = tq_full + 4;   // consumer releases, counted on the leader
  int* tq = reinterpret_cast<int*>(tq_empty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + 4);
  // kXSum: ring of finished output units (epilogue warps push, helper warps
  // 2 and 3 sum them), 256 entries; then the per-helper heads, the tail and
  // the count of epilogue warps that are done
  int* xring = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full) + 256);
  unsigned* xhead = reinterpret_cast<unsigned*>(xring + 256);  // [2]
  unsigned* xtail = xhead + 2;
  unsigned* xfin = xhead + 3;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;
  const int tiles_m = (M + Cfg::BM - 1) / Cfg::BM;
  const int tiles_n = (N + Cfg::BN - 1) / Cfg::BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (K + BK - 1) / BK;
  const bool dynamic = tile_counter != nullptr;
  // stream-K (dynamic scheduling only): this pair's K-block range
  const bool skon = dynamic && sk.sk_tiles > 0;
  const int sk_u0 = skon ? static_cast<int>(static_cast<long long>(sk.units) * cluster / nclusters) : 0;
  const int sk_u1 = skon ? static_cast<int>(static_cast<long long>(sk.units) * (cluster + 1) / nclusters) : 0;

  // Work sequence.  Static: cluster c takes tiles c, c + nclusters, ...
  // Dynamic: the leader's producer decides the next item — its stream-K
  // items first (above), then tiles in raster order from a global counter
  // when its cluster is ready for one — and publishes it to both CTAs'
  // 4-entry queues; the other consumers (peer producer, MMA, every epilogue
  // warp of both CTAs) read their own copy and release the slot on the leader.
  // Keeping the tiles in flight a compact band of the raster keeps the
  // operand panels they share resident in L2 across the whole K loop.
  // An item is a tile index with its stream-K role in bits 28..31; -1 ends.
  auto consume_tile = [&](int seq, bool arrive) -> int {
    if (!dynamic) {
      const int t = cluster + seq * nclusters;
      return t < num_tiles ? t : -1;
    }
    const int slot = seq & 3;
    ptx::mbar_wait_cluster(&tq_full[slot], (seq >> 2) & 1);
    const int t = *reinterpret_cast<volatile int*>(&tq[slot]);
    if (arrive) ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tq_empty[slot]), 0));
    return t;
  };
  int sk_idx = 0;  // leader producer: next stream-K item of this pair
  auto next_item = [&]() -> int {
    while (skon) {
      const int it = sk_static_item(sk_u0, sk_u1, num_kb, sk_idx);
      if (it < 0) break;
      ++sk_idx;
      const int t = item_tile(it);
      if (item_role(it) == kRoleHead) {
        if (atomicCAS(&sk.claim[t], 0, 1) == 0) return it;
        atomicExch(&sk.claim[t], 0);  // the finisher took the whole tile
        continue;
      }
      if (item_role(it) == kRoleTail)
        return atomicCAS(&sk.claim[t], 0, 2) == 0 ? make_item(t, kRoleWhole) : it;
      return it;
    }
    int t = atomicAdd(tile_counter, 1) + sk.sk_tiles;
    return t < num_tiles ? t : -1;
  };
  auto produce_tile = [&](int seq) -> int {  // leader producer
    if (!dynamic) {
      const int t = cluster + seq * nclusters;
      return t < num_tiles ? t : -1;
    }
    const int slot = seq & 3;
    ptx::mbar_wait_cluster(&tq_empty[slot], ((seq >> 2) & 1) ^ 1);
    const int t = next_item();
    tq[slot] = t;
    ptx::st_shared_cluster_u32(ptx::mapa_shared(ptx::smem_u32(&tq[slot]), 1), static_cast<uint32_t>(t));
    ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tq_full[slot]), 0));
    ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tq_full[slot]), 1));
    return t;
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (use_tma_store) ptx::prefetch_tmap(&tmC);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * Cfg::EPI_WARPS);  // every epilogue warp of the pair
    }
    for (int q = 0; q < 4; ++q) {
      ptx::mbar_init(&tq_full[q], 1);
      ptx::mbar_init(&tq_empty[q], 2 + 2 * Cfg::EPI_WARPS);  // MMA, peer producer, epilogues
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  if (warp == 3) {
    for (int i = lane; i < 256; i += 32) xring[i] = 0;
    if (lane < 4) xhead[lane] = 0;  // heads, tail, finished count
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the next kernel may be scheduled now (its
  // CTAs take SMs as ours exit and run their prologue); this one touches no
  // global memory before the previous kernel in the stream has completed.
  // Both are no-ops without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // kLoadAll: the epilogue warpgroups take registers from warpgroup 0
  // (producer, MMA issuer, helpers) within the CTA's launch allocation of
  // 384 x 168: 128 x 56 + 256 x 224 = 64512 (setmaxnreg.inc would wait
  // forever for registers the CTA does not have, so the host only launches
  // this variant when the kernel was compiled to 168 registers)
  constexpr bool kLoadAll = MT == 2 && !OUTF && DEEP;
  // side task (SideSum): the epoch of this call, read before any CTA can
  // have advanced it (the last helper warp out does, after every CTA started)
  const int side_p = side.n16 > 0 ? *reinterpret_cast<const volatile int*>(side.par) : 0;

  // kExchange / kXSum: the call counter picks the receive set (device-side
  // double buffering); kXSum: the flag epoch of this call
  const bool xsum = epi.mode == kXSum;
  const int xcalls = (epi.mode == kExchange || xsum) && epi.par
                         ? *reinterpret_cast<const volatile int*>(epi.par) : 0;
  const unsigned long long* xbase = (xcalls & 1) ? epi.peer_alt : epi.peer;
  const int xepoch = xcalls + 1;
  const int xupr = (N + 127) / 128;
  // kXSum: sum output unit u (32 rows x 128 columns) with the whole warp:
  // slot 0 + slot 1 of our receive set (own partial; the peer's, landed over
  // NVLink) in fp32, one RNE rounding, to the output; mark it done
  auto xsum_unit = [&](int uu) {
    const int r0 = (uu / xupr) * 32, c0 = (uu % xupr) * 128;
    const char* s0 = reinterpret_cast<const char*>(xbase[epi.me]);
    const char* s1 = s0 + static_cast<uint64_t>(epi.slice) * 2;
#pragma unroll 8
    for (int i = 0; i < 16; ++i) {
      const int v = lane + 32 * i;
      const int row = r0 + (v >> 4), col = c0 + (v & 15) * 8;
      if (row < M && col < N) {
        const uint64_t off = (static_cast<uint64_t>(row) * N + col) * 2;
        uint4 a, b;
        asm volatile("ld.global.cg.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(s0 + off) : "memory");
        asm volatile("ld.global.cg.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(s1 + off) : "memory");
        *reinterpret_cast<uint4*>(epi.peer[2] + off) = ptx::add_bf16x8(a, b);
      }
    }
    __syncwarp();
    if (lane == 0) reinterpret_cast<int*>(epi.peer[5])[uu] = xepoch;
  };

  if (warp < 4) {
  // warpgroup 0: producer, MMA issuer, helpers (kLoadAll: 56 registers each;
  // the CTA keeps its launch allocation, 384 x 168: 128 x 56 + 256 x 224)
  if constexpr (kLoadAll) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int seq = 0;; ++seq) {
        const int it = leader ? produce_tile(seq) : consume_tile(seq, true);
        if (it < 0) break;
        int kb0, kb1;
        item_kb(it, sk_u0, sk_u1, num_kb, &kb0, &kb1);
        const TileCoord tc = tile_coord_g(item_tile(it), tiles_m, tiles_n, group_m, Cfg::BM, Cfg::BN);
        const int am = tc.m0 + Cfg::ROWS_CTA * static_cast<int>(rank);  // this CTA's A rows
        const int bn = tc.n0 + 128 * static_cast<int>(rank);            // this CTA's half of N
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          uint8_t* a_dst = sA + stage * Cfg::SMEM_A;
          uint8_t* b_dst = sB + stage * Cfg::SMEM_B;
          if (A_MN == 0) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)  // 128-row boxes, 16 KiB apart
              ptx::tma_load_2d_2sm(a_dst + mt * 16384, &tmA, &full[stage], k0, am + 128 * mt);
          } else {
#pragma unroll
            for (int c = 0; c < Cfg::ROWS_CTA / MN_CHUNK; ++c)
              ptx::tma_load_2d_2sm(a_dst + c * MN_CHUNK_BYTES, &tmA, &full[stage],
                                   am + c * MN_CHUNK, k0);
          }
          if (B_MN == 0) {
            ptx::tma_load_2d_2sm(b_dst, &tmB, &full[stage], k0, bn);
          } else {
            ptx::tma_load_2d_2sm(b_dst, &tmB, &full[stage], bn, k0);
            ptx::tma_load_2d_2sm(b_dst + MN_CHUNK_BYTES, &tmB, &full[stage], bn + MN_CHUNK, k0);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();  // lanes 1..31 park here (converged) until lane 0 is done
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(256, Cfg::BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      // the K-block `kb` staged in slot `st`, sub-tiles [mt0, mt1) of the accumulator
      auto issue = [&](uint32_t d_tmem, int st, int kb, int mt0, int mt1) {
        const uint32_t a_base = ptx::smem_u32(sA + st * Cfg::SMEM_A);
        const uint32_t b_base = ptx::smem_u32(sB + st * Cfg::SMEM_B);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t bd = B_MN ? ptx::sdesc_sw128(b_base + kk * 2048, MN_CHUNK_BYTES, 1024)
                                   : ptx::sdesc_sw128(b_base + kk * 32, 16, 1024);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            if (mt < mt0 || mt >= mt1) continue;
            // rows [mt*128, mt*128+128) of each CTA's A start 16 KiB apart in
            // both majors (128 rows x 128 B, or two 8-KiB MN chunks)
            const uint32_t ab = a_base + mt * 16384;
            const uint64_t ad = A_MN ? ptx::sdesc_sw128(ab + kk * 2048, MN_CHUNK_BYTES, 1024)
                                     : ptx::sdesc_sw128(ab + kk * 32, 16, 1024);
            ptx::umma_f16_2sm(d_tmem + mt * Cfg::BN, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
        }
      };
      auto advance = [&](int& st, uint32_t& ph) {
        if (++st == Cfg::STAGES) {
          st = 0;
          ph ^= 1;
        }
      };
      for (int seq = 0;; ++seq) {
        const int it = consume_tile(seq, true);
        if (it < 0) break;
        int kb0, kb1;
        item_kb(it, sk_u0, sk_u1, num_kb, &kb0, &kb1);
        const int nkb = kb1 - kb0;  // K-blocks of this item (kb below counts from 0)
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * MT * Cfg::BN);
        int kb = 0;
        if (MT == 2) {
          // One accumulator (all 512 columns), released per sub-tile: while the
          // epilogue still drains sub-tile 1 of the previous tile, the first
          // STAGES staged K-blocks already accumulate into sub-tile 0.
          ptx::mbar_wait(&tempty[0], acc_phase ^ 1);
          if (!split_release) ptx::mbar_wait(&tempty[1], acc_phase ^ 1);
          ptx::tc_fence_after();
          const int pro = !split_release ? 0 : nkb < Cfg::STAGES ? nkb : Cfg::STAGES;
          int st2 = stage;
          uint32_t ph2 = phase;
          for (int j = 0; j < pro; ++j) {
            ptx::mbar_wait(&full[st2], ph2);
            ptx::tc_fence_after();
            issue(d_tmem, st2, j, 0, 1);
            advance(st2, ph2);
          }
          if (split_release) {
            ptx::mbar_wait(&tempty[1], acc_phase ^ 1);
            ptx::tc_fence_after();
          }
          for (; kb < pro; ++kb) {
            issue(d_tmem, stage, kb, 1, 2);
            ptx::umma_commit_2sm(&empty[stage], 0x3);  // frees the slot in both CTAs
            advance(stage, phase);
          }
        } else {
          ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
          ptx::tc_fence_after();
        }
        for (; kb < nkb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          issue(d_tmem, stage, kb, 0, MT);
          ptx::umma_commit_2sm(&empty[stage], 0x3);  // frees the slot in both CTAs
          advance(stage, phase);
        }
        ptx::umma_commit_2sm(&tfull[acc], 0x3);      // both CTAs' accumulators ready
        if (++acc == Cfg::ACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 2 || warp == 3) {
    if (side.n16 > 0) {
      // ---------------------------------------------- side task (SideSum)
      const int want = side_p + 1;
      if (blockIdx.x == 0 && warp == 3 && lane == 0) {  // CTA 0 meets the peer
        if (side.arrive_peer) {
          // our previous kernels' writes to the peer (the producing GEMM's
          // partial) happen before this release; the peer's before our acquire
          asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(side.arrive_peer), "r"(want)
                       : "memory");
          long long spins = 0;
          while (ld_acquire_sys_i(side.arrive_own) - want < 0) {
            __nanosleep(128);
            if (++spins > (1LL << 27)) __trap();  // the peer never arrived: fail loudly
          }
        }
        st_release_gpu(side.go, want);
      }
      if (lane == 0)
        while (ld_acquire_gpu(side.go) - want < 0) __nanosleep(256);
      __syncwarp();
      const uint4* r = reinterpret_cast<const uint4*>((side_p & 1) ? side.recv1 : side.recv0);
      uint4* o = reinterpret_cast<uint4*>(side.out);
      const long long n16 = side.n16;
      const long long stride = static_cast<long long>(gridDim.x) * 64;
      long long i = static_cast<long long>(blockIdx.x) * 64 + (warp - 2) * 32 + lane;
      for (; i + 3 * stride < n16; i += 4 * stride) {  // 8 loads in flight per thread
        uint4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = ldcg_u4(r + i + u * stride);
          b[u] = ldcg_u4(r + n16 + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) o[i + u * stride] = ptx::add_bf16x8(a[u], b[u]);
      }
      for (; i < n16; i += stride) o[i] = ptx::add_bf16x8(ldcg_u4(r + i), ldcg_u4(r + n16 + i));
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        if (atomicAdd(side.fin, 1u) == 2 * gridDim.x - 1) {  // every helper warp is done
          *side.fin = 0;
          *side.par = want;  // the producing GEMM's next call takes the other receive set
          __threadfence();
        }
      }
    }
    // ------------------------------------------------ kXSum helpers (both CTAs)
    // Helper c sums ring slots c, c + 2, ... in order once the peer's flag for
    // the unit is up.  It never holds the epilogue back for long: when the
    // ring backs up (the peer lags) or the epilogue is done and the wait
    // budget is spent, the unit is left to the sweep kernel.
    if (xsum) {
      const int c = warp - 2;
      int end_budget = 400;  // polls of ~0.2 us once every epilogue warp is done
      for (unsigned k = 0;; ++k) {
        const unsigned sl = 2 * k + c;
        int entry = 0;
        bool stop = false;
        for (;;) {
          entry = *reinterpret_cast<volatile int*>(&xring[sl & 255]);
          if ((entry & 255) == static_cast<int>((sl >> 8) % 255 + 1)) break;
          if (*reinterpret_cast<volatile unsigned*>(xfin) == Cfg::EPI_WARPS &&
              *reinterpret_cast<volatile unsigned*>(xtail) <= sl) {
            stop = true;
            break;
          }
          __nanosleep(64);
        }
        if (stop) break;
        __threadfence_block();  // the pushing warp's fence precedes its ring store
        const int uu = entry >> 8;
        bool ok = false;
        for (;;) {
          const int f = ld_acquire_sys_i(reinterpret_cast<const int*>(epi.peer[3]) + uu);
          ok = __all_sync(0xffffffffu, f == xepoch);
          if (ok) break;
          const unsigned tail = *reinterpret_cast<volatile unsigned*>(xtail);
          const bool done = *reinterpret_cast<volatile unsigned*>(xfin) == Cfg::EPI_WARPS;
          if (tail - sl > 192 || (done && --end_budget < 0)) break;
          __nanosleep(200);
        }
        if (ok) xsum_unit(uu);
        __syncwarp();
        if (lane == 0) *reinterpret_cast<volatile unsigned*>(&xhead[c]) = k + 1;
      }
    }
    __syncwarp();
  }
  } else {
    // warpgroups 1 and 2: the epilogue (kLoadAll: 224 registers each)
    if constexpr (kLoadAll) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
    // ------------------------------------------------ epilogue (both CTAs)
    // TMEM -> registers (thread = row) -> bf16 -> XOR-swizzled smem -> 16-B
    // vectors with 8 consecutive threads covering one 128-B row segment, so
    // every global store / NVLink write is a full line.
    const int ew = warp - 4;          // epilogue warp 0..7
    const int e = ew & 3;             // TMEM lane quarter (warp % 4)
    const int chalf = ew >> 2;        // which 128 columns of the tile this warp stores
    constexpr int ELEM = OUTF ? 4 : 2;        // bytes per output element
    constexpr int CCOLS = 128 / ELEM;         // columns per staged chunk (128-B rows)
    constexpr int UCOLS = 16 / ELEM;          // columns per 16-B unit
    constexpr int NCH = 128 / CCOLS;          // chunks per warp (its 128 columns)
    char* const Cb = static_cast<char*>(Cv);
    __nv_bfloat16* const C = static_cast<__nv_bfloat16*>(Cv);
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec_ok =
        ((ldc * ELEM) % 16 == 0) && ((reinterpret_cast<uintptr_t>(Cv) & 15) == 0);
    uint8_t* stage_base = sEpi + ew * (Cfg::EPI_BOXES * 32 * 64 * 2);
    // kExchange double buffering: the receive buffers of this call (parity
    // counter written in stream order by the previous call's barrier kernel)
    int nstore = 0;  // TMA stores issued by this warp (alternate staging boxes)
    for (int seq = 0;; ++seq) {
      const int t = consume_tile(seq, false);
      __syncwarp();
      if (dynamic && lane == 0)
        ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tq_empty[seq & 3]), 0));
      if (t < 0) break;
      const int role = item_role(t);
      const TileCoord tc = tile_coord_g(item_tile(t), tiles_m, tiles_n, group_m, Cfg::BM, Cfg::BN);
      // stream-K: this warp's workspace units (32 lanes x 16 B, coalesced) and ready flag
      const size_t ws_warp = ((static_cast<size_t>(item_tile(t)) * 2 + rank) * MT * 8 + ew) * (4 * 8 * 32) + lane;
      auto ws_unit = [&](int mt, int q, int j) -> float4* {
        return sk.ws + ws_warp + static_cast<size_t>(mt) * (8 * 4 * 8 * 32) + (q * 8 + j) * 32;
      };
      int* const ready = sk.ready + (item_tile(t) * 2 + static_cast<int>(rank)) * 8 + ew;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if (role == kRoleTail) {  // the contributor's partial sums have landed
        if (lane == 0)
          while (ld_acquire_gpu(ready) == 0) __nanosleep(100);
        __syncwarp();
      }
      // bf16: this warp's share of sub-tile mt goes TMEM -> registers
      // (RNE-packed; + the stream-K partial sums on a TAIL) and the sub-tile
      // is released at once, so the MMA warp resumes before the staging and
      // stores.  kLoadAll (the 4-stage 512x256 pipeline): both sub-tiles are
      // loaded and released before any store (the epilogue warps hold 128
      // packed registers; setmaxnreg above), so the next tile's MMAs never
      // wait for sub-tile 0's stores.
      auto load_pack = [&](int mt, uint32_t (&pkd)[OUTF ? 1 : NCH][32]) {
        if constexpr (!OUTF) {
          const uint32_t col_base = static_cast<uint32_t>((acc * MT + mt) * Cfg::BN);
#pragma unroll
          for (int ci = 0; ci < NCH; ++ci) {
            uint32_t v0[32], v1[32];
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * e) << 16) + col_base +
                                   static_cast<uint32_t>((chalf * NCH + ci) * CCOLS);
            ptx::tmem_ld_32x32b_x32(taddr, v0);
            ptx::tmem_ld_32x32b_x32(taddr + 32, v1);
            ptx::tmem_wait_ld();
            if (role == kRoleTail) {  // finisher: + the partial sums of K-blocks [0, t0)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 w0 = ld_cg_f4(ws_unit(mt, 2 * ci, j));
                const float4 w1 = ld_cg_f4(ws_unit(mt, 2 * ci + 1, j));
                v0[4 * j] = addf(v0[4 * j], w0.x);
                v0[4 * j + 1] = addf(v0[4 * j + 1], w0.y);
                v0[4 * j + 2] = addf(v0[4 * j + 2], w0.z);
                v0[4 * j + 3] = addf(v0[4 * j + 3], w0.w);
                v1[4 * j] = addf(v1[4 * j], w1.x);
                v1[4 * j + 1] = addf(v1[4 * j + 1], w1.y);
                v1[4 * j + 2] = addf(v1[4 * j + 2], w1.z);
                v1[4 * j + 3] = addf(v1[4 * j + 3], w1.w);
              }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              pkd[ci][i] = ptx::pack_bf16x2(v0[2 * i], v0[2 * i + 1]);
              pkd[ci][16 + i] = ptx::pack_bf16x2(v1[2 * i], v1[2 * i + 1]);
            }
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_leader(&tempty[MT == 2 ? mt : acc]);
        }
      };
      uint32_t pkall[kLoadAll ? 2 : 1][OUTF ? 1 : NCH][32];
      if constexpr (kLoadAll) {
        if (role != kRoleHead) {
          load_pack(0, pkall[0]);
          load_pack(1, pkall[1]);
        }
      }
#pragma unroll (kLoadAll ? 2 : 1)
      for (int mt = 0; mt < MT; ++mt) {
        const int row0 = tc.m0 + Cfg::ROWS_CTA * static_cast<int>(rank) + 128 * mt + 32 * e;
        const uint32_t col_base = static_cast<uint32_t>((acc * MT + mt) * Cfg::BN);
        if (role == kRoleHead) {
          // contributor: fp32 partial sums of K-blocks [0, h) to the workspace
#pragma unroll 1
          for (int q = 0; q < 4; ++q) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(32 * e) << 16) + col_base +
                                        static_cast<uint32_t>(chalf * 128 + q * 32),
                                    v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *ws_unit(mt, q, j) = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                               __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0 && (MT == 2 || mt == MT - 1)) ptx::mbar_arrive_leader(&tempty[MT == 2 ? mt : acc]);
          continue;
        }
        uint32_t pk_one[OUTF ? 1 : NCH][32];
        if constexpr (!kLoadAll) load_pack(mt, pk_one);
        uint32_t(&pk)[OUTF ? 1 : NCH][32] = kLoadAll ? pkall[kLoadAll ? mt : 0] : pk_one;
#pragma unroll (OUTF ? 1 : NCH)
        for (int ci = 0; ci < NCH; ++ci) {
          const int c = chalf * NCH + ci;
          const bool tma = use_tma_store && epi.mode == kStore;
          uint8_t* stage =
              stage_base + (tma && Cfg::EPI_BOXES == 2 ? (nstore & 1) * (32 * 64 * 2) : 0);
          const uint32_t stage_u32 = ptx::smem_u32(stage);
          if (tma) {
            // the store issued EPI_BOXES chunks ago read this box: make sure it is done
            if (lane == 0) {
              if (Cfg::EPI_BOXES == 2)
                ptx::tma_store_wait_read_le1();
              else
                ptx::tma_store_wait_read();
            }
            __syncwarp();
          }
          if constexpr (OUTF) {
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * e) << 16) + col_base +
                                   static_cast<uint32_t>(c * CCOLS);
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(taddr, v);
            ptx::tmem_wait_ld();
            if (role == kRoleTail) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 w = ld_cg_f4(ws_unit(mt, ci, j));
                v[4 * j] = addf(v[4 * j], w.x);
                v[4 * j + 1] = addf(v[4 * j + 1], w.y);
                v[4 * j + 2] = addf(v[4 * j + 2], w.z);
                v[4 * j + 3] = addf(v[4 * j + 3], w.w);
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 16-B unit = 4 fp32 columns
              const uint32_t a = stage_u32 + lane * 128 + ((j ^ (lane & 7)) << 4);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v[4 * j]),
                           "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                           : "memory");
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 16-B unit = 8 bf16 columns
              const uint32_t a = stage_u32 + lane * 128 + ((j ^ (lane & 7)) << 4);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[ci][4 * j]),
                           "r"(pk[ci][4 * j + 1]), "r"(pk[ci][4 * j + 2]), "r"(pk[ci][4 * j + 3])
                           : "memory");
            }
          }
          if (tma) {
            // the staged chunk is exactly TMA's 128-B-swizzled 32-row box
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&tmC, stage, tc.n0 + c * CCOLS, row0);
              ptx::tma_store_commit();
            }
            ++nstore;
            continue;
          }
          __syncwarp();
          const int u = lane & 7;
          const int gcol = tc.n0 + c * CCOLS + u * UCOLS;
          if (epi.mode == kPairSum) {
            // 2-rank all-reduce completed in the epilogue (see gemm.h): no
            // pass over the output after the GEMM, no barrier
            const int ccol0 = tc.n0 + c * CCOLS;
            if (row0 < M && ccol0 < N) {
#pragma unroll 2
              for (int it = 0; it < 8; ++it) {  // our partial -> the peer's receive buffer
                const int r = it * 4 + (lane >> 3);
                const int grow = row0 + r;
                if (grow < M && gcol < N) {
                  uint4 w;
                  const uint32_t a = stage_u32 + r * 128 + ((u ^ (r & 7)) << 4);
                  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "r"(a) : "memory");
                  *reinterpret_cast<uint4*>(epi.peer[1] + (static_cast<uint64_t>(grow) * N + gcol) * 2) = w;
                }
              }
              ptx::fence_sys();
              __syncwarp();
              uint32_t ticket = 0;
              const uint64_t chunk = static_cast<uint64_t>(row0 / 32) * epi.slice + ccol0 / CCOLS;
              if (lane == 0) ticket = ptx::atom_add_acqrel_sys(epi.mc + 4 * chunk, 1u);
              ticket = __shfl_sync(0xffffffffu, ticket, 0);
              if (ticket & 1u) {  // second to arrive: the peer's partial has landed here
                ptx::fence_sys();
#pragma unroll 2
                for (int it = 0; it < 8; ++it) {
                  const int r = it * 4 + (lane >> 3);
                  const int grow = row0 + r;
                  if (grow < M && gcol < N) {
                    uint4 w;
                    const uint32_t a = stage_u32 + r * 128 + ((u ^ (r & 7)) << 4);
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "r"(a) : "memory");
                    const uint64_t off = (static_cast<uint64_t>(grow) * N + gcol) * 2;
                    uint4 p;  // written by the peer over NVLink: bypass L1
                    asm volatile("ld.volatile.global.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(p.x), "=r"(p.y), "=r"(p.z), "=r"(p.w)
                                 : "l"(epi.peer[0] + off) : "memory");
                    const uint4 f = ptx::add_bf16x8(w, p);
                    *reinterpret_cast<uint4*>(epi.peer[2] + off) = f;
                    *reinterpret_cast<uint4*>(epi.peer[3] + off) = f;
                  }
                }
                ptx::fence_sys();
                __syncwarp();
                if (lane == 0) {
                  ptx::red_add_release_sys(epi.peer[4], 1u);
                  ptx::red_add_release_sys(epi.peer[5], 1u);
                }
              }
            }
            __syncwarp();
            continue;
          }
#pragma unroll 2
          for (int it = 0; it < 8; ++it) {
            const int r = it * 4 + (lane >> 3);
            uint4 w;
            const uint32_t a = stage_u32 + r * 128 + ((u ^ (r & 7)) << 4);
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                         : "r"(a)
                         : "memory");
            const int grow = row0 + r;
            if (grow < M && gcol < N) {
              if (epi.mode == kMcRed) {
                // fused 2-rank all-reduce (host guarantees N % 8 == 0, ldc % 8 == 0)
                ptx::multimem_red_add_bf16x8(
                    epi.mc + (static_cast<uint64_t>(grow) * ldc + gcol) * 2, w);
              } else if (epi.mode == kExchange || epi.mode == kXSum) {
                // all-reduce by exchange: this 16-B vector to slot `me` of every rank
                const long long f = static_cast<long long>(grow) * N + gcol;
                const uint64_t off =
                    static_cast<uint64_t>(static_cast<long long>(epi.me) * epi.slice + f) * ELEM;
                for (int q = 0; q < epi.P; ++q) *reinterpret_cast<uint4*>(xbase[q] + off) = w;
              } else if (epi.mode == kRedPair) {
                const uint64_t off = (static_cast<uint64_t>(grow) * ldc + gcol) * 2;
                ptx::red_add_bf16x8(epi.mc + off, w);
                ptx::red_add_bf16x8_sys(epi.peer[0] + off, w);
              } else if (epi.mode == kRedLocal) {
                ptx::red_add_bf16x8(epi.mc + (static_cast<uint64_t>(grow) * ldc + gcol) * 2, w);
              } else if (epi.mode == kScatter) {
                // fused reduce-scatter: this 16-B vector goes to its owner's slot
                const long long f = static_cast<long long>(grow) * N + gcol;
                const int o = static_cast<int>(f / epi.slice);
                const long long off =
                    static_cast<long long>(epi.me) * epi.slice + (f - o * epi.slice);
                *reinterpret_cast<uint4*>(epi.peer[o] + static_cast<uint64_t>(off) * ELEM) = w;
              } else if (vec_ok && gcol + UCOLS <= N) {
                *reinterpret_cast<uint4*>(Cb + (static_cast<int64_t>(grow) * ldc + gcol) * ELEM) = w;
              } else if (OUTF) {
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
                float* dst = reinterpret_cast<float*>(Cb) + static_cast<int64_t>(grow) * ldc + gcol;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (gcol + q < N) dst[q] = __uint_as_float(ws[q]);
              } else {
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
                __nv_bfloat16* dst = C + static_cast<int64_t>(grow) * ldc + gcol;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  if (gcol + q < N) {
                    const uint16_t bits = static_cast<uint16_t>(ws[q >> 1] >> (16 * (q & 1)));
                    dst[q] = __ushort_as_bfloat16(bits);
                  }
                }
              }
            }
          }
          __syncwarp();
        }
        if (OUTF && MT == 2) {
          // this warp's share of sub-tile mt is out of TMEM: release it (the
          // MMA warp starts the next tile on sub-tile 0 before sub-tile 1 is free)
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_leader(&tempty[mt]);
        }
      }
      if (xsum && role != kRoleHead) {
        // kXSum: this tile's partial (both copies) is performed system-wide
        // before the peer's flags for its units go up; the units then go to
        // the helper warps (epi.mc bit 0, experiments: all to the sweep;
        // bit 1: no fence, timing only)
        if (!(epi.mc & 2)) ptx::fence_sys();
        __syncwarp();
        if (lane == 0) {
#pragma unroll 1
          for (int mt = 0; mt < MT; ++mt) {
            const int row0 = tc.m0 + Cfg::ROWS_CTA * static_cast<int>(rank) + 128 * mt + 32 * e;
            const int col0 = tc.n0 + chalf * 128;
            if (row0 >= M || col0 >= N) continue;
            const int uu = (row0 / 32) * xupr + col0 / 128;
            st_relaxed_sys_i(reinterpret_cast<int*>(epi.peer[4]) + uu, xepoch);
            if (epi.mc & 1) continue;
            // slot s of the ring: helper s & 1 consumes it; wait until that
            // helper is done with slot s - 256 (helpers never wait long)
            const unsigned sl = atomicAdd(xtail, 1u);
            while (static_cast<int>((sl >> 1) - *reinterpret_cast<volatile unsigned*>(&xhead[sl & 1])) >= 128)
              __nanosleep(64);
            *reinterpret_cast<volatile int*>(&xring[sl & 255]) =
                uu * 256 + static_cast<int>((sl >> 8) % 255 + 1);  // round stamp 1..255
          }
        }
        __syncwarp();
      }
      if (role == kRoleHead) {
        // every lane's partial sums are written before the flag is raised
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(ready, 1);
      } else if (role == kRoleTail && lane == 0) {
        *ready = 0;  // back to 0 for the next launch (the only reader is done)
        if (rank == 0 && ew == 0) sk.claim[item_tile(t)] = 0;
      }
      if (OUTF && MT != 2 && role != kRoleHead) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_leader(&tempty[acc]);
      }
      if (++acc == Cfg::ACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (xsum && lane == 0) atomicAdd(xfin, 1u);  // this warp pushes no more units
    if (epi.mode != kStore) ptx::fence_sys();  // remote writes performed before the kernel retires
    if (use_tma_store && lane == 0) ptx::tma_store_wait_all();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_2sm(tmem_base, TMEM_COLS);
  // the last CTA out returns the tile counter (and the exit count) to 0 for
  // the slot's next launch: no memset between launches
  if (dynamic && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(reinterpret_cast<unsigned*>(tile_counter + 1), 1u) == gridDim.x - 1) {
      tile_counter[0] = 0;
      tile_counter[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D bf16 tensor map over a row-major matrix: `inner` contiguous elements per
// row, `outer` rows, row stride `ld` elements; box box_inner x box_outer with
// 128-byte swizzle; out-of-bounds elements read as zero.
bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_inner, uint32_t box_outer, bool f32 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  static const int promo = [] {
    const char* v = std::getenv("AXONN_L2_PROMOTION");  // 0 none, 1 64B, 2 128B, 3 256B
    return v && *v ? std::atoi(v) : 3;
  }();
  const CUtensorMapL2promotion p =
      promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
      : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
      : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, p,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int A_MN, int B_MN>
cudaError_t launch_single(const CUtensorMap& ma, const CUtensorMap& mb, void* C, int64_t ldc,
                          int M, int N, int K, int num_sms, cudaStream_t stream) {
  auto kern = gemm_bf16_tcgen05<A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SMEM_BYTES));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  kern<<<grid, THREADS, SMEM_BYTES, stream>>>(ma, mb, static_cast<__nv_bfloat16*>(C), ldc, M, N,
                                              K);
  return cudaGetLastError();
}

int env_int(const char* name, int dflt);

// Dynamic tile scheduling: a ring of global counter pairs (tile counter, CTAs
// finished), zeroed once; the last CTA of every launch resets its pair, so
// consecutive GEMMs have no memset between them (which would also break the
// programmatic dependent launch).  A slot is reused only after kSlots further
// launches, so launches on different streams never share a live counter
// unless more than kSlots GEMMs are in flight at once.  AXONN_SCHED=static
// disables it.  Called under the library mutex.
int* next_tile_counter(cudaStream_t stream) {
  static const bool dyn = [] {
    const char* v = std::getenv("AXONN_SCHED");
    return !(v && std::strcmp(v, "static") == 0);
  }();
  if (!dyn) return nullptr;
  constexpr int kSlots = 16384;
  static int* ring = nullptr;
  static int next = 0;
  if (!ring) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return nullptr;  // first use inside a capture: static scheduling for this launch
    if (cudaMalloc(&ring, 2 * kSlots * sizeof(int)) != cudaSuccess) {
      ring = nullptr;
      return nullptr;
    }
    if (cudaMemset(ring, 0, 2 * kSlots * sizeof(int)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return nullptr;
  }
  int* c = ring + 2 * next;
  next = (next + 1) % kSlots;
  return c;
}

// Stream-K tail (see SkParams): split the first (tiles mod pairs) + pairs
// tiles along K when whole-tile waves would leave more than AXONN_SK_LOSS
// percent (default 4) of the pairs idle, the tiles fill at least one wave and
// K is long enough to split (>= 16 K-blocks).  Workspaces come from a ring of
// kSkSlots (zeroed once; every launch leaves its flags at 0), so launches on
// different streams share a slot only when more than kSkSlots stream-K GEMMs
// are in flight at once.  AXONN_SK=0 disables it.  Called under the library
// mutex.
long long g_sk_launches = 0;

SkParams stream_k_plan(int tiles, int pairs, int num_kb, int mt, cudaStream_t stream) {
  static const bool on = env_int("AXONN_SK", 1) != 0;
  static const int loss_pct = env_int("AXONN_SK_LOSS", 4);
  SkParams p;
  if (!on || pairs < 1 || tiles < pairs || tiles % pairs == 0 || num_kb < 16) return p;
  const int waves = (tiles + pairs - 1) / pairs;
  if (100LL * (static_cast<long long>(waves) * pairs - tiles) <= static_cast<long long>(loss_pct) * waves * pairs)
    return p;
  const int sk_tiles = tiles % pairs + pairs;
  constexpr int kSkSlots = 4;
  constexpr int kMaxSkTiles = 160;  // > 2 x pairs on any sm_100 part (<= 160 SMs)
  if (sk_tiles > kMaxSkTiles) return p;
  struct Slot {
    float4* ws = nullptr;
    int* flags = nullptr;
  };
  static Slot slots[kSkSlots];
  static int next = 0;
  Slot& s = slots[next];
  const size_t ws_bytes = static_cast<size_t>(kMaxSkTiles) * 2 * 2 /*MT max*/ * 8 * 4 * 8 * 32 * 16;
  const size_t flag_bytes = static_cast<size_t>(kMaxSkTiles) * (1 + 16) * sizeof(int);
  if (!s.ws) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return p;  // no allocation inside a capture (the eager warm-up allocates)
    if (cudaMalloc(&s.ws, ws_bytes) != cudaSuccess) {
      s.ws = nullptr;
      return p;
    }
    if (cudaMalloc(&s.flags, flag_bytes) != cudaSuccess || cudaMemset(s.flags, 0, flag_bytes) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      cudaFree(s.ws);
      s.ws = nullptr;
      return p;
    }
  }
  next = (next + 1) % kSkSlots;
  ++g_sk_launches;
  p.sk_tiles = sk_tiles;
  p.units = sk_tiles * num_kb;
  p.ws = s.ws;
  p.claim = s.flags;
  p.ready = s.flags + kMaxSkTiles;
  (void)mt;
  return p;
}

template <int A_MN, int B_MN, int MT, int OUTF = 0, int DEEP = 0>
cudaError_t launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                        int use_tma_store, void* C, int64_t ldc, int M, int N, int K, int num_sms,
                        int group_m, const EpiTarget& epi, cudaStream_t stream,
                        const SideSum& side = SideSum()) {
  using Cfg = PairCfg<MT, DEEP>;
  auto kern = gemm_bf16_tcgen05_pair<A_MN, B_MN, MT, OUTF, DEEP>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::SMEM_BYTES));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + Cfg::BM - 1) / Cfg::BM) * ((N + Cfg::BN - 1) / Cfg::BN);
  int grid = (num_sms / 2) * 2;
  if (2 * tiles < grid) grid = 2 * tiles;
  if (grid < 2) grid = 2;
  int* counter = next_tile_counter(stream);
  // MT=2: release the accumulator per sub-tile (AXONN_SPLIT_RELEASE=0: whole tile)
  static const int split = env_int("AXONN_SPLIT_RELEASE", 1) != 0;
  const SkParams sk = counter ? stream_k_plan(tiles, grid / 2, (K + BK - 1) / BK, MT, stream)
                              : SkParams();
  // programmatic dependent launch (AXONN_PDL=0: plain stream order)
  static const bool pdl = env_int("AXONN_PDL", 1) != 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(Cfg::THREADS);
  lc.dynamicSmemBytes = Cfg::SMEM_BYTES;
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kern, ma, mb, mc, use_tma_store, C, ldc, M, N, K, split, group_m,
                            epi, counter, sk, side);
}

// MT = 2 takes the deep-pipeline configuration (4 operand stages, one
// epilogue staging box per warp) unless AXONN_MT2_DEEP=0.
template <int A_MN, int B_MN>
cudaError_t launch_pair_mt(int mt, const CUtensorMap& ma, const CUtensorMap& mb,
                           const CUtensorMap& mc, int use_tma_store, void* C, int64_t ldc, int M,
                           int N, int K, int num_sms, int group_m, const EpiTarget& epi,
                           cudaStream_t stream, const SideSum& side) {
  // the deep variant's register hand-over assumes 168 registers per thread
  static const bool deep = env_int("AXONN_MT2_DEEP", 1) != 0 && [] {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, gemm_bf16_tcgen05_pair<A_MN, B_MN, 2, 0, 1>) == cudaSuccess &&
           fa.numRegs == 168;
  }();
  if (mt == 2)
    return deep ? launch_pair<A_MN, B_MN, 2, 0, 1>(ma, mb, mc, use_tma_store, C, ldc, M, N, K,
                                                   num_sms, group_m, epi, stream, side)
                : launch_pair<A_MN, B_MN, 2, 0, 0>(ma, mb, mc, use_tma_store, C, ldc, M, N, K,
                                                   num_sms, group_m, epi, stream, side);
  return launch_pair<A_MN, B_MN, 1>(ma, mb, mc, use_tma_store, C, ldc, M, N, K, num_sms, group_m,
                                    epi, stream, side);
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

}  // namespace

thread_local cudaError_t g_launch_error = cudaSuccess;

// C[M][N] (bf16, ldc) = op(A) x op(B); see axonn_gemm in include/axonn.h.
// AXONN_GEMM_VARIANT=single selects the 1-CTA kernel (kept for A/B timing);
// the default is the CTA-pair kernel: 512x256 tiles for plain launches
// (AXONN_PAIR_MT=1: 256x256) and for fused-collective epilogues with K >= 8192,
// 256x256 for shorter fused launches.  AXONN_GROUP_M sets the raster band.
GemmStatus gemm_bf16_tc(int op, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* C, int64_t ldc, int num_sms,
                        cudaStream_t stream, const EpiTarget* epi_in, bool out_f32,
                        const SideSum* side_in) {
  const SideSum side = side_in ? *side_in : SideSum();
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return GemmStatus::kBadShape;
  if ((lda & 7) || (ldb & 7) || (reinterpret_cast<uintptr_t>(A) & 15) ||
      (reinterpret_cast<uintptr_t>(B) & 15))
    return GemmStatus::kBadAlignment;
  static const bool single_env = [] {
    const char* v = std::getenv("AXONN_GEMM_VARIANT");
    return v && std::strcmp(v, "single") == 0;
  }();
  // the 1-CTA kernel has no fp32 epilogue and no side task
  const bool single = single_env && !out_f32 && !(side_in && side_in->n16 > 0);
  // raster band: 4096 rows of tiles (AXONN_GROUP_M overrides, in tiles; < 0 = bands of N tiles)
  static const int group_m_env = env_int("AXONN_GROUP_M", 0);
  // 512x256 tiles (MT=2: less L2/DRAM traffic per flop) for plain-store
  // launches; 256x256 (MT=1: double-buffered TMEM, so the NVLink-writing
  // epilogue overlaps the next tile's main loop) for fused-collective epilogues.
  static const int mt_plain = env_int("AXONN_PAIR_MT", 2) == 1 ? 1 : 2;
  // fused epilogues: 512x256 when the K loop is long enough to amortise the
  // serialised (NVLink-writing) epilogue, else 256x256 (AXONN_PAIR_MT_FUSED=1|2 forces)
  static const int mt_fused_env = env_int("AXONN_PAIR_MT_FUSED", 0);
  const int mt_fused = mt_fused_env == 1 ? 1 : mt_fused_env == 2 ? 2 : (K >= 8192 ? 2 : 1);
  CUtensorMap ma, mb;
  const int m = static_cast<int>(M), n = static_cast<int>(N), k = static_cast<int>(K);
  // B box rows along N: 256 for the single-CTA tile, 128 (half of N) per CTA of a pair.
  const uint32_t bkrows = single ? BN : 128;
  bool ok;
  switch (op) {
    case 0:  // NN: A [M][K] (K-major), B [K][N] (N-major)
      ok = make_map(&ma, A, K, M, lda, BK, 128) && make_map(&mb, B, N, K, ldb, MN_CHUNK, BK);
      break;
    case 1:  // NT: A [M][K], B [N][K] (K-major)
      ok = make_map(&ma, A, K, M, lda, BK, 128) && make_map(&mb, B, K, N, ldb, BK, bkrows);
      break;
    case 2:  // TN: A [K][M] (M-major), B [K][N]
      ok = make_map(&ma, A, M, K, lda, MN_CHUNK, BK) && make_map(&mb, B, N, K, ldb, MN_CHUNK, BK);
      break;
    default:
      return GemmStatus::kBadOp;
  }
  if (!ok) return GemmStatus::kTensorMap;
  cudaError_t e;
  const EpiTarget epi = epi_in ? *epi_in : EpiTarget();
  const int unit = out_f32 ? 4 : 8;  // elements per 16-B epilogue unit
  if (epi.mode != kStore && (single || (N % unit) || (ldc % unit)))
    return GemmStatus::kBadAlignment;
  if (out_f32 && op != 2) return GemmStatus::kBadOp;  // fp32 output: the dW (TN) product only
  if (out_f32 && (epi.mode == kMcRed || epi.mode == kRedLocal || epi.mode == kRedPair))
    return GemmStatus::kBadAlignment;  // red.add is bf16 here
  if (epi.mode == kScatter && (ldc != N || epi.slice % unit || epi.P < 1 || epi.P > 8))
    return GemmStatus::kBadAlignment;
  if (epi.mode == kExchange && (ldc != N || epi.slice != M * N || epi.P < 1 || epi.P > 8))
    return GemmStatus::kBadAlignment;
  if (epi.mode == kXSum && (out_f32 || ldc != N || epi.slice != M * N || epi.P != 2 || !epi.par))
    return GemmStatus::kBadAlignment;
  if (side.n16 > 0 && (epi.mode == kXSum || !side.par || !side.go || !side.fin || !side.out))
    return GemmStatus::kBadAlignment;  // the helper warps run one task; the task needs its state
  if (epi.mode == kPairSum && (out_f32 || ldc != N || epi.slice != (N + 63) / 64))
    return GemmStatus::kBadAlignment;
  // MT=2's single accumulator serialises the epilogue with the next tile; on
  // short K loops that costs more than its lower L2/DRAM traffic saves
  // (AXONN_MT2_MIN_K: smallest K that takes the 512x256 tile).
  static const int mt2_min_k = env_int("AXONN_MT2_MIN_K", 0);
  const int pair_mt = epi.mode != kStore ? mt_fused : (K >= mt2_min_k ? mt_plain : 1);
  // TMA-store epilogue for plain launches when C satisfies TMA's alignment
  // (16-byte base and row pitch) AND rows end on a 16-byte boundary: the store
  // clips the inner dimension only at 16-byte granularity, so with N % 8 != 0
  // it would write up to 7 elements past column N-1 (caught by the tests' NaN
  // canary).  AXONN_TMA_STORE=0 keeps per-thread stores.
  static const bool tma_store_env = env_int("AXONN_TMA_STORE", 1) != 0;
  CUtensorMap mc;
  int use_tma_store = 0;
  const int cols16 = out_f32 ? 4 : 8;  // elements per 16 bytes of C
  if (!single && epi.mode == kStore && tma_store_env && (ldc % cols16) == 0 && (N % cols16) == 0 &&
      (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
      make_map(&mc, C, N, M, ldc, out_f32 ? 32 : 64, 32, out_f32))
    use_tma_store = 1;
  else
    std::memset(&mc, 0, sizeof mc);
  const int group_m = group_m_env != 0 ? group_m_env : (single ? 32 : 16 / pair_mt);
  if (out_f32) {
    e = pair_mt == 2 ? launch_pair<1, 1, 2, 1>(ma, mb, mc, use_tma_store, C, ldc, m, n, k, num_sms,
                                               group_m, epi, stream, side)
                     : launch_pair<1, 1, 1, 1>(ma, mb, mc, use_tma_store, C, ldc, m, n, k, num_sms,
                                               group_m, epi, stream, side);
  } else if (single) {
    e = op == 0 ? launch_single<0, 1>(ma, mb, C, ldc, m, n, k, num_sms, stream)
        : op == 1 ? launch_single<0, 0>(ma, mb, C, ldc, m, n, k, num_sms, stream)
                  : launch_single<1, 1>(ma, mb, C, ldc, m, n, k, num_sms, stream);
  } else {
    e = op == 0 ? launch_pair_mt<0, 1>(pair_mt, ma, mb, mc, use_tma_store, C, ldc, m, n, k, num_sms, group_m, epi, stream, side)
        : op == 1 ? launch_pair_mt<0, 0>(pair_mt, ma, mb, mc, use_tma_store, C, ldc, m, n, k, num_sms, group_m, epi, stream, side)
                  : launch_pair_mt<1, 1>(pair_mt, ma, mb, mc, use_tma_store, C, ldc, m, n, k, num_sms, group_m, epi, stream, side);
  }
  g_launch_error = e;
  return e == cudaSuccess ? GemmStatus::kOk : GemmStatus::kLaunch;
}

cudaError_t gemm_last_launch_error() { return g_launch_error; }

long long gemm_stream_k_launches() { return g_sk_launches; }

// The stream-K items pair `cluster` of `nclusters` processes for a launch
// whose first sk_tiles tiles (num_kb K-blocks each) are split, in processing
// order, with the same functions the kernel uses (claims aside: a TAIL whose
// contributor has not started becomes WHOLE at run time).  Host only.
int gemm_stream_k_items(int sk_tiles, int num_kb, int cluster, int nclusters, int* tile, int* role,
                        int* kb0, int* kb1, int cap) {
  const long long units = static_cast<long long>(sk_tiles) * num_kb;
  const int u0 = static_cast<int>(units * cluster / nclusters);
  const int u1 = static_cast<int>(units * (cluster + 1) / nclusters);
  int n = 0;
  for (int idx = 0;; ++idx) {
    const int it = sk_static_item(u0, u1, num_kb, idx);
    if (it < 0) break;
    if (n < cap) {
      tile[n] = item_tile(it);
      role[n] = item_role(it);
      item_kb(it, u0, u1, num_kb, &kb0[n], &kb1[n]);
    }
    ++n;
  }
  return n;
}

}  // namespace axonn
