// gemm_tc.cu - K1: bf16/fp16 GEMM on 5th-gen tensor cores with the fused
// bias / ReLU / GELU (+ residual) epilogue.
//
// What the reference describes and this kernel realises natively:
//   * multi-level tiling + scratchpad promotion (orchestrate, tiling.cpp:
//     1059-1203; measured structure SURVEY.md §3.2): the 64x64x32 block tile
//     with double-buffered shared A/B tiles becomes a 128 x BLOCK_N x 64 tile
//     fed by a STAGES-deep TMA ring (cp.async.bulk.tensor + mbarrier
//     expect_tx), honouring the interpreter's "no use before await" rule
//     (interp.cpp:314-318, 657-685) through full/empty barrier phases;
//   * the shared C tile becomes a TMEM accumulator (tcgen05.mma kind::f16,
//     fp32), double-buffered so the epilogue of tile i overlaps the MMAs of
//     tile i+1;
//   * the 16x16 fragment mapping (mmaHook, tiling.h:96) is a
//     single-thread-issued 128 x BLOCK_N x 16 UMMA;
//   * the bias+max epilogue nest (left unfused by the reference) is applied
//     to the accumulator in registers before the one global store.
//
// Warp roles (256 threads, 1 CTA per SM, persistent over output tiles):
//   warp 0  : TMA producer (one elected lane)
//   warp 1  : MMA issuer   (one lane)
//   warp 2  : TMEM allocator / deallocator
//   warps 4-7: epilogue (thread t owns accumulator row t of the tile)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "afg_internal.h"
#include "epilogue.cuh"
#include "sm100.cuh"

namespace afg {
namespace {

using namespace sm100;

constexpr int BLOCK_M = 128;
constexpr int BLOCK_K = 64;  // 64 x 16-bit = one 128-byte swizzle row
constexpr int GROUP_M = 16;  // default tile raster: 16 M-blocks share B tiles in L2

struct GemmTcArgs {
  int M, N, K;
  int ldc;
  const float* bias;
  const void* residual;
  void* C;
  int num_m_blocks, num_n_blocks;
  int group_m;  // tile raster: M-blocks per group (consecutive tiles walk M first)
  int epi;
  int tma_store;  // 1: stage C through swizzled smem + TMA bulk tensor store
  // implicit-GEMM conv (IM2COL): output pixel m = (n, p, q) over OH x OW,
  // K = KH*KW*C ordered (ky, kx, c) like the OHWI filter.
  int c_blocks, KW, dil_w, dil_h, OH, OW, stride_w, stride_h, lower_w, lower_h;
  int early_tmem;  // epilogue: issue the chunk's TMEM loads before the staging-buffer wait
  int round_sync;  // 0: off; else 1 + counter slot: producers hold tile round r+1
                   // until every CTA has issued round r (bounded wait)
};

// Round sync counters, one pair per slot (stream_slot: one per stream, so
// concurrent launches on different streams do not share one):
// [0] = CTA arrivals per tile round, [1] = kernel exits. The last CTA to exit
// resets both; the next launch on the stream touches them only after
// griddepcontrol.wait (the previous grid has completed). A wait is bounded, so
// a disturbed counter costs time, never correctness or progress.
constexpr int ROUND_SLOTS = 64;
__device__ unsigned int g_round[ROUND_SLOTS][2];

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// AFG_EPI_EARLY_TMEM (default: on for short-K problems): A/B switch of the
// epilogue's TMEM-load placement
inline int early_tmem_for(int64_t K) {
  static const int env = [] {
    const char* e = getenv("AFG_EPI_EARLY_TMEM");
    return e ? atoi(e) : -1;
  }();
  return env >= 0 ? env : (K <= 1024 ? 1 : 0);
}

// Round sync for problems of several tile rounds: the persistent clusters
// otherwise drift apart in K, and the CTAs sharing an A / B panel read it from
// DRAM at different times (16384^3: 20.3 GB DRAM read per launch, 6.59 ms;
// with the sync 8.8 GB, 5.80 ms -- the saved DRAM power shows up as clock on
// the power-capped chip). AFG_GEMM_ROUND_SYNC=0 turns it off (A/B).
// Short K (rounds of a few microseconds) loses more to the wait than it saves
// (ResNet 1x1 convs: 747 -> 681 TFLOP/s), so only K >= 4096 syncs.
inline int round_sync_for(int tiles, int64_t K, bool pair, cudaStream_t stream) {
  static const int env = [] {
    const char* e = getenv("AFG_GEMM_ROUND_SYNC");
    return e ? atoi(e) : 1;
  }();
  if (env <= 0 || K < 4096 || tiles < 4 * (pair ? num_sms() / 2 : num_sms())) return 0;
  return 1 + stream_slot(stream, 0, ROUND_SLOTS);  // 0 (off) when the slots are used up
}

// PAIR: a CTA pair (cluster of 2) computes a 256 x BLOCK_N tile with one
// cta_group::2 MMA per K step; each CTA stages its 128 rows of A and half of
// the BLOCK_N rows/columns of B (halving per-SM B traffic in smem and L2).
template <int BLOCK_N, int STAGES, bool PAIR = false, int NG = 2>
struct SmemLayout {
  static constexpr int B_ROWS = PAIR ? BLOCK_N / 2 : BLOCK_N;  // B rows staged per CTA
  static constexpr int A_BYTES = BLOCK_M * BLOCK_K * 2;
  static constexpr int B_BYTES = B_ROWS * BLOCK_K * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // C staging: NG epilogue groups x EPI_BUFS x (128 rows x 128 B); more
  // buffers per group when they fit next to the operand stages
  static constexpr int EPI_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int EPI_BUFS = EPI_OFFSET + 4 * NG * BLOCK_M * 128 + 2048 <= 232448   ? 4
                                  : EPI_OFFSET + 2 * NG * BLOCK_M * 128 + 2048 <= 232448 ? 2
                                                                                          : 1;
  static constexpr int EPI_BYTES = NG * EPI_BUFS * BLOCK_M * 128;
  // bias of the tile columns of all epilogue groups (<= max(BLOCK_N, NG * 64))
  static constexpr int BIAS_OFFSET = EPI_OFFSET + EPI_BYTES;
  static constexpr int BAR_OFFSET = BIAS_OFFSET + (BLOCK_N > NG * 64 ? BLOCK_N : NG * 64) * 4;
  static constexpr int NUM_BARS = 2 * STAGES + 4;
  static constexpr int TOTAL = BAR_OFFSET + NUM_BARS * 8 + 16 + 1024;  // +1024 align slack
};

__device__ __forceinline__ void tile_coords(int t, int nmb, int nnb, int group_m, int& mb,
                                            int& nb) {
  const int per_group = group_m * nnb;
  const int group = t / per_group;
  const int first_m = group * group_m;
  const int gsize = min(nmb - first_m, group_m);
  const int r = t - group * per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

__device__ __forceinline__ uint32_t pack_out(float a, float b, __nv_bfloat16*) { return pack_bf16(a, b); }
__device__ __forceinline__ uint32_t pack_out(float a, float b, __half*) { return pack_f16(a, b); }
__device__ __forceinline__ uint32_t pack_out_relu(float a, float b, __nv_bfloat16*) {
  return pack_bf16_relu(a, b);
}
__device__ __forceinline__ uint32_t pack_out_relu(float a, float b, __half*) {
  return pack_f16_relu(a, b);
}

template <int EPI, typename OutT>
__device__ __forceinline__ void store_chunk32(const uint32_t (&acc)[32], const GemmTcArgs& a,
                                              int row, int col0) {
  if (row >= a.M) return;
  // 16-bit C, whole chunk, no residual, bias (+ ReLU): bias added on f32x2
  // pairs and ReLU folded into the packed conversion (the halo conv's
  // epilogue; ~2 instructions per value instead of ~4)
  if constexpr (sizeof(OutT) == 2 && (EPI == AFG_EPI_BIAS || EPI == AFG_EPI_BIAS_RELU)) {
    if (a.residual == nullptr && col0 + 32 <= a.N && (a.ldc & 7) == 0) {
      const float4* b4 = reinterpret_cast<const float4*>(a.bias + col0);
      uint32_t w[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 b = __ldg(b4 + j);
        float x0, x1, x2, x3;
        f2split(fadd2(f2(__uint_as_float(acc[4 * j]), __uint_as_float(acc[4 * j + 1])), f2(b.x, b.y)), x0, x1);
        f2split(fadd2(f2(__uint_as_float(acc[4 * j + 2]), __uint_as_float(acc[4 * j + 3])), f2(b.z, b.w)), x2, x3);
        if constexpr (EPI == AFG_EPI_BIAS_RELU) {
          w[2 * j] = pack_out_relu(x0, x1, static_cast<OutT*>(nullptr));
          w[2 * j + 1] = pack_out_relu(x2, x3, static_cast<OutT*>(nullptr));
        } else {
          w[2 * j] = pack_out(x0, x1, static_cast<OutT*>(nullptr));
          w[2 * j + 1] = pack_out(x2, x3, static_cast<OutT*>(nullptr));
        }
      }
      uint4* crow4 = reinterpret_cast<uint4*>(reinterpret_cast<OutT*>(a.C) +
                                              static_cast<int64_t>(row) * a.ldc + col0);
#pragma unroll
      for (int q = 0; q < 4; ++q) crow4[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      return;
    }
  }
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]);
  if constexpr (EPI != AFG_EPI_NONE) {
    if (col0 + 32 <= a.N) {
      const float4* b4 = reinterpret_cast<const float4*>(a.bias + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 b = __ldg(b4 + j);
        v[4 * j + 0] += b.x;
        v[4 * j + 1] += b.y;
        v[4 * j + 2] += b.z;
        v[4 * j + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < a.N) v[j] += __ldg(a.bias + col0 + j);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = apply_act<EPI>(v[j]);
  }
  OutT* crow = reinterpret_cast<OutT*>(a.C) + static_cast<int64_t>(row) * a.ldc + col0;
  const bool HAS_RES = a.residual != nullptr;
  const OutT* rrow = HAS_RES ? reinterpret_cast<const OutT*>(a.residual) +
                                   static_cast<int64_t>(row) * a.ldc + col0
                             : nullptr;
  const bool full = (col0 + 32 <= a.N) && ((a.ldc & 7) == 0);
  if (full) {
    constexpr int PER16 = 16 / sizeof(OutT);  // elements per 16-byte vector
#pragma unroll
    for (int j = 0; j < 32 / PER16; ++j) {
      OutT tmp[PER16];
      if (HAS_RES) {
        *reinterpret_cast<uint4*>(tmp) = *reinterpret_cast<const uint4*>(rrow + j * PER16);
#pragma unroll
        for (int e = 0; e < PER16; ++e)
          tmp[e] = OutCvt<OutT>::to(v[j * PER16 + e] + OutCvt<OutT>::from(tmp[e]));
      } else {
#pragma unroll
        for (int e = 0; e < PER16; ++e) tmp[e] = OutCvt<OutT>::to(v[j * PER16 + e]);
      }
      *reinterpret_cast<uint4*>(crow + j * PER16) = *reinterpret_cast<uint4*>(tmp);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j < a.N) {
        float r = v[j];
        if (HAS_RES) r += OutCvt<OutT>::from(rrow[j]);
        crow[j] = OutCvt<OutT>::to(r);
      }
    }
  }
}

// act(acc + bias) (+ residual) for 32 consecutive columns of one row, in fp32.
// `sbias` (optional): the 32 bias values already staged in shared memory.
template <int EPI, typename OutT>
__device__ __forceinline__ void epi_values32(const uint32_t (&acc)[32], const GemmTcArgs& a,
                                             int row, int col0, float (&v)[32],
                                             const float* sbias = nullptr) {
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]);
  if constexpr (EPI != AFG_EPI_NONE) {
    if (col0 + 32 <= a.N) {
      // bias add and activation on f32x2 pairs (one issue slot per pair)
      const float4* b4 = reinterpret_cast<const float4*>(a.bias + col0);
      const uint32_t sb_addr = sbias ? smem_u32(sbias) : 0u;  // staged bias: LDS, not generic loads
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 b;
        if (sbias) {
          const uint4 u = ld_shared_v4(sb_addr + 16 * j);
          b = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z),
                          __uint_as_float(u.w));
        } else {
          b = __ldg(b4 + j);
        }
        uint64_t p0 = fadd2(f2(v[4 * j], v[4 * j + 1]), f2(b.x, b.y));
        uint64_t p1 = fadd2(f2(v[4 * j + 2], v[4 * j + 3]), f2(b.z, b.w));
        p0 = apply_act2<EPI>(p0);
        p1 = apply_act2<EPI>(p1);
        f2split(p0, v[4 * j], v[4 * j + 1]);
        f2split(p1, v[4 * j + 2], v[4 * j + 3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < a.N) v[j] += __ldg(a.bias + col0 + j);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = apply_act<EPI>(v[j]);
    }
  }
  if (a.residual != nullptr && row < a.M) {
    const OutT* rrow = reinterpret_cast<const OutT*>(a.residual) + static_cast<int64_t>(row) * a.ldc + col0;
    if (col0 + 32 <= a.N && (a.ldc & 7) == 0) {
      constexpr int PER16 = 16 / sizeof(OutT);
#pragma unroll
      for (int j = 0; j < 32 / PER16; ++j) {
        OutT tmp[PER16];
        *reinterpret_cast<uint4*>(tmp) = *reinterpret_cast<const uint4*>(rrow + j * PER16);
#pragma unroll
        for (int e = 0; e < PER16; ++e) v[j * PER16 + e] += OutCvt<OutT>::from(tmp[e]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < a.N) v[j] += OutCvt<OutT>::from(rrow[j]);
    }
  }
}

template <typename OutT>
__device__ __forceinline__ void epi_values32_rt(const uint32_t (&acc)[32], const GemmTcArgs& a,
                                                int row, int col0, float (&v)[32],
                                                const float* sbias = nullptr) {
  switch (a.epi) {
    case AFG_EPI_BIAS: epi_values32<AFG_EPI_BIAS, OutT>(acc, a, row, col0, v, sbias); break;
    case AFG_EPI_BIAS_RELU: epi_values32<AFG_EPI_BIAS_RELU, OutT>(acc, a, row, col0, v, sbias); break;
    case AFG_EPI_BIAS_GELU_TANH:
      epi_values32<AFG_EPI_BIAS_GELU_TANH, OutT>(acc, a, row, col0, v, sbias);
      break;
    case AFG_EPI_BIAS_GELU_ERF:
      epi_values32<AFG_EPI_BIAS_GELU_ERF, OutT>(acc, a, row, col0, v, sbias);
      break;
    default: epi_values32<AFG_EPI_NONE, OutT>(acc, a, row, col0, v); break;
  }
}



__device__ __forceinline__ void epi_bar_sync(int g) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
}

template <typename OutT>
__device__ __forceinline__ void store_chunk32_rt(const uint32_t (&acc)[32], const GemmTcArgs& a,
                                                 int row, int col0) {
  switch (a.epi) {
    case AFG_EPI_BIAS: store_chunk32<AFG_EPI_BIAS, OutT>(acc, a, row, col0); break;
    case AFG_EPI_BIAS_RELU: store_chunk32<AFG_EPI_BIAS_RELU, OutT>(acc, a, row, col0); break;
    case AFG_EPI_BIAS_GELU_TANH:
      store_chunk32<AFG_EPI_BIAS_GELU_TANH, OutT>(acc, a, row, col0);
      break;
    case AFG_EPI_BIAS_GELU_ERF: store_chunk32<AFG_EPI_BIAS_GELU_ERF, OutT>(acc, a, row, col0); break;
    default: store_chunk32<AFG_EPI_NONE, OutT>(acc, a, row, col0); break;
  }
}

template <int BLOCK_N, int STAGES, bool B_MN_MAJOR, bool AB_BF16, typename OutT, bool IM2COL,
          bool PAIR, int NG>
__global__ void __launch_bounds__(128 + 128 * NG, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const GemmTcArgs args) {
  using L = SmemLayout<BLOCK_N, STAGES, PAIR, NG>;
  constexpr int TILE_M = PAIR ? 2 * BLOCK_M : BLOCK_M;  // rows per (pair) tile
  static_assert(BLOCK_N % 64 == 0 && BLOCK_N <= 256, "BLOCK_N");
  constexpr uint32_t TMEM_COLS = 2 * BLOCK_N <= 32    ? 32
                                 : 2 * BLOCK_N <= 64  ? 64
                                 : 2 * BLOCK_N <= 128 ? 128
                                 : 2 * BLOCK_N <= 256 ? 256
                                                      : 512;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NUM_BARS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int cid = PAIR ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int ncl = PAIR ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.tma_store) tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      // PAIR: one arrival per epilogue warp of both CTAs (on the leader's)
      // a tile that is one TMA-store chunk wide (BLOCK_N = 64, 16-bit C) is
      // handled by one epilogue group, the groups alternating tiles
      const bool alt = args.tma_store && BLOCK_N * static_cast<int>(sizeof(OutT)) == 128;
      mbar_init(&tempty_bar[s], PAIR ? 8 * NG : (alt ? 128 : 128 * NG));
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    else tmem_alloc<TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // the previous kernel's outputs (our A / B / residual) are visible
  griddep_launch_dependents();

  const int num_tiles = args.num_m_blocks * args.num_n_blocks;
  const int num_kb = (args.K + BLOCK_K - 1) / BLOCK_K;

  // Registers: 56 for the TMA / MMA / TMEM warpgroup, the rest to the
  // epilogue warpgroups. With setmaxnreg in the kernel ptxas allocates the
  // launch-bound maximum (168 x 384 or 96 x 640 threads) and compiles each
  // role's code under its own budget; the split below matches those pools
  // (checked on every build by scripts/check_regs.py).
  if (warp < 4) {
  setmaxnreg_dec<56>();
  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int round = 0;
      unsigned int* ctr = args.round_sync ? g_round[args.round_sync - 1] : nullptr;
      for (int t = cid; t < num_tiles; t += ncl, ++round) {
        if (ctr && round > 0) {
          // hold this round's loads until every CTA has issued the previous
          // round's: the clusters of a wave stay in K-lockstep, so each panel
          // slice is read from DRAM once per wave (bounded: never a deadlock)
          const unsigned int want = static_cast<unsigned int>(round) * gridDim.x;
          const uint64_t t0 = global_ns();
          while (ld_acquire_gpu(&ctr[0]) < want && global_ns() - t0 < 20000) {
          }
        }
        int mb, nb;
        tile_coords(t, args.num_m_blocks, args.num_n_blocks, args.group_m, mb, nb);
        const int m0 = mb * TILE_M + static_cast<int>(rank) * BLOCK_M;
        const int n0 = nb * BLOCK_N + static_cast<int>(rank) * L::B_ROWS;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::STAGE_BYTES;
          uint8_t* sb = sa + L::A_BYTES;
          // PAIR: both CTAs' bytes complete on the leader's full barrier
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], (PAIR ? 2 : 1) * L::STAGE_BYTES);
          const uint32_t fb = PAIR ? mapa_shared(&full_bar[stage], 0) : smem_u32(&full_bar[stage]);
          auto load2d = [&](void* dst, const CUtensorMap* tm, int c0, int c1) {
            if constexpr (PAIR) tma_load_2d_pair(dst, tm, fb, c0, c1);
            else tma_load_2d(dst, tm, &full_bar[stage], c0, c1);
          };
          if constexpr (IM2COL) {
            const int q = m0 % args.OW;
            const int p = (m0 / args.OW) % args.OH;
            const int n = m0 / (args.OW * args.OH);
            const int tap = kb / args.c_blocks;
            const int cb = kb - tap * args.c_blocks;
            const int ky = tap / args.KW;
            const int kx = tap - ky * args.KW;
            if constexpr (PAIR)
              tma_load_im2col_4d_pair(sa, &tmA, fb, cb * BLOCK_K,
                                      args.lower_w + q * args.stride_w,
                                      args.lower_h + p * args.stride_h, n,
                                      static_cast<uint16_t>(kx * args.dil_w),
                                      static_cast<uint16_t>(ky * args.dil_h));
            else
              tma_load_im2col_4d(sa, &tmA, &full_bar[stage], cb * BLOCK_K,
                                 args.lower_w + q * args.stride_w, args.lower_h + p * args.stride_h,
                                 n, static_cast<uint16_t>(kx * args.dil_w),
                                 static_cast<uint16_t>(ky * args.dil_h));
          } else {
            load2d(sa, &tmA, kb * BLOCK_K, m0);
          }
          if constexpr (B_MN_MAJOR) {
#pragma unroll
            for (int j = 0; j < L::B_ROWS / 64; ++j)
              load2d(sb + j * (64 * BLOCK_K * 2), &tmB, n0 + j * 64, kb * BLOCK_K);
          } else {
            load2d(sb, &tmB, kb * BLOCK_K, n0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (ctr) atomicAdd(&ctr[0], 1u);
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer --
    // The whole warp walks the loop (barrier waits and descriptor arithmetic
    // stay warp-uniform, in uniform registers); one elected lane issues. The
    // per-MMA work is a 64-bit immediate add on each descriptor: a
    // 128 x BLOCK_N x 16 MMA lasts only BLOCK_N / 2 tensor cycles.
    if (rank == 0) {  // PAIR: the leader CTA issues for both
    const bool leader = elect_one();
    constexpr uint32_t idesc =
        idesc_f16(TILE_M, BLOCK_N, AB_BF16 ? 1u : 0u, 0u, B_MN_MAJOR ? 1u : 0u);
    const uint64_t a_desc0 = desc_kmajor_sw128(smem_u32(smem));
    const uint64_t b_desc0 = B_MN_MAJOR ? desc_mnmajor_sw128(smem_u32(smem + L::A_BYTES), 64 * BLOCK_K * 2)
                                        : desc_kmajor_sw128(smem_u32(smem + L::A_BYTES));
    constexpr uint64_t STAGE_STEP = L::STAGE_BYTES >> 4;  // descriptor units (16 B)
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++iter) {
      const int acc = iter & 1;
      const uint32_t acc_par = (iter >> 1) & 1;
      if constexpr (PAIR) mbar_wait_cluster(&tempty_bar[acc], acc_par ^ 1);
      else mbar_wait(&tempty_bar[acc], acc_par ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BLOCK_N;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage) * STAGE_STEP;
        const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage) * STAGE_STEP;
#pragma unroll
        for (int k = 0; k < BLOCK_K / 16; ++k) {
          const uint64_t boff = B_MN_MAJOR ? static_cast<uint64_t>((k * 16 * 128) >> 4)
                                           : static_cast<uint64_t>((k * 32) >> 4);
          mma_f16_ss_if<PAIR ? 2 : 1>(leader, d_tmem, ad + static_cast<uint64_t>((k * 32) >> 4),
                                      bd + boff, idesc, (kb | k) != 0 ? 1u : 0u);
        }
        if constexpr (PAIR) mma_commit_pair_if(leader, &empty_bar[stage], 3);
        else mma_commit_if(leader, &empty_bar[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if constexpr (PAIR) mma_commit_pair_if(leader, &tfull_bar[acc], 3);
      else mma_commit_if(leader, &tfull_bar[acc]);
    }
    }
  }
  } else {
    setmaxnreg_inc<NG == 2 ? 224 : 104>();
    // ----------------------------------------------------------- epilogue --
    // NG groups of 4 warps (warps 4-7, 8-11, ...); each covers TMEM lanes
    // 0-127 (warp % 4 selects the 32-lane slice); they take column chunks
    // round-robin.
    const int eg = (warp - 4) / 4;
    const int ew = warp % 4;
    const int rloc = ew * 32 + lane;
    int iter = 0;
    // this thread's last TMEM read of accumulator `acc` is done
    auto release_acc = [&](int acc) {
      tc_fence_before();
      if constexpr (PAIR) {
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&tempty_bar[acc]);
          else mbar_arrive_cluster(&tempty_bar[acc], 0);
        }
      } else {
        mbar_arrive(&tempty_bar[acc]);
      }
    };
    if (args.tma_store) {
      // C chunk of 128 rows x 128 B staged in 128B-swizzled smem (with two
      // buffers per group a chunk is written while the previous chunk's TMA
      // store still reads its buffer), then one TMA bulk tensor store by the
      // group leader.
      constexpr int CW = 128 / static_cast<int>(sizeof(OutT));  // columns per chunk
      uint8_t* stage_base = smem + L::EPI_OFFSET + eg * L::EPI_BUFS * (BLOCK_M * 128);
      int staged = 0;  // chunks this group has staged (buffer = staged & 1)
      const bool leader = ew == 0 && lane == 0;
      // the group's bias columns (chunks eg, eg + NG, ...), staged in smem once
      // per tile: thread t of the group owns column t of that list; its global
      // load is issued before the accumulator wait, so its latency hides
      constexpr int NCHUNK = BLOCK_N / CW;
      // one chunk per tile: the groups take tiles round-robin (geff = 0 for
      // all); otherwise they take chunks of every tile round-robin
      constexpr bool ALT = NCHUNK == 1;
      const int geff = ALT ? 0 : eg;
      constexpr int GCOLS = (NCHUNK + NG - 1) / NG * CW;  // bias columns per group (max)
      float* sb = reinterpret_cast<float*>(smem + L::BIAS_OFFSET) + eg * GCOLS;
      const int bcol = (geff + NG * (rloc / CW)) * CW + rloc % CW;  // tile column of my bias value
      const bool has_bias =
          args.epi != AFG_EPI_NONE && rloc < (NCHUNK - geff + NG - 1) / NG * CW && rloc < GCOLS;
      // ReLU without a residual, 16-bit C: folded into the cvt (exact)
      const bool relu_pack =
          sizeof(OutT) == 2 && args.epi == AFG_EPI_BIAS_RELU && args.residual == nullptr;
      for (int t = cid; t < num_tiles; t += ncl, ++iter) {
        if (ALT && iter % NG != eg) continue;  // another group's tile
        int mb, nb;
        tile_coords(t, args.num_m_blocks, args.num_n_blocks, args.group_m, mb, nb);
        const int gcol = nb * BLOCK_N + bcol;
        const float bias_v = has_bias && gcol < args.N ? __ldg(args.bias + gcol) : 0.0f;
        bool bias_staged = false;
        const int acc = iter & 1;
        if (args.residual != nullptr) {
          // this thread's residual row segments of the tile into L2 while the
          // tile's MMAs still run: the epilogue's loads then hit L2 instead of
          // paying DRAM latency per chunk (BERT out-projection + residual:
          // the synchronous loads added 19 us to a 35 us GEMM)
          const int prow = mb * TILE_M + static_cast<int>(rank) * BLOCK_M + rloc;
          if (prow < args.M) {
            const char* rbase = reinterpret_cast<const char*>(args.residual) +
                                (static_cast<int64_t>(prow) * args.ldc) * sizeof(OutT);
            for (int cc = geff; cc < BLOCK_N / CW; cc += NG) {
              const int n0p = nb * BLOCK_N + cc * CW;
              if (n0p < args.N)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(rbase + static_cast<int64_t>(n0p) * sizeof(OutT)));
            }
          }
        }
        mbar_wait(&tfull_bar[acc], (iter >> 1) & 1);
        tc_fence_after();
        const int m0 = mb * TILE_M + static_cast<int>(rank) * BLOCK_M;
        const int row = m0 + rloc;
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BLOCK_N;
        constexpr int NCH = BLOCK_N / CW;
        if (geff >= NCH) release_acc(acc);  // no chunk for this group: still release once
#pragma unroll 1
        for (int cc = geff; cc < NCH; cc += NG) {
          const int n0 = nb * BLOCK_N + cc * CW;
          const bool live = n0 < args.N;  // uniform across the group
          uint8_t* stage = stage_base + (staged % L::EPI_BUFS) * (BLOCK_M * 128);
          const uint32_t srow = smem_u32(stage + rloc * 128);
          if (!bias_staged) {  // readers of the previous tile's bias passed the last barrier
            if (has_bias) sb[rloc] = bias_v;
            bias_staged = true;
          }
          // the chunk's TMEM columns in one round trip (all loads, one wait),
          // issued before the wait for the staging buffer so the load latency
          // overlaps it (the short-K epilogues stalled on that barrier)
          uint32_t rr[CW / 32][32];
          if (!args.early_tmem && live) {
            if (leader) tma_store_wait_read<L::EPI_BUFS - 1>();  // last store from this buffer
            epi_bar_sync(eg);
          }
#pragma unroll
          for (int h = 0; h < CW / 32; ++h) tmem_ld32(t_row + cc * CW + h * 32, rr[h]);
          if (args.early_tmem && live) {
            if (leader) tma_store_wait_read<L::EPI_BUFS - 1>();  // last store from this buffer
            epi_bar_sync(eg);
          }
          tmem_wait_ld();
          if (cc + NG >= NCH) release_acc(acc);  // last TMEM read of the tile
#pragma unroll
          for (int h = 0; h < CW / 32; ++h) {
            if (!live) continue;
            float v[32];
            if (relu_pack)  // bias here, ReLU folded into the 16-bit conversion below
              epi_values32<AFG_EPI_BIAS, OutT>(rr[h], args, row, n0 + h * 32, v,
                                               sb + ((cc - geff) / NG) * CW + h * 32);
            else
              epi_values32_rt<OutT>(rr[h], args, row, n0 + h * 32, v,
                                    sb + ((cc - geff) / NG) * CW + h * 32);
            // 32 values -> 64 B (16-bit) or 128 B (fp32) of the 128 B row
            constexpr int QPH = 32 * static_cast<int>(sizeof(OutT)) / 16;  // 16 B chunks per half
#pragma unroll
            for (int qq = 0; qq < QPH; ++qq) {
              const int q = h * QPH + qq;
              uint32_t w[4];
              if constexpr (sizeof(OutT) == 2) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  w[k] = relu_pack ? pack_out_relu(v[qq * 8 + 2 * k], v[qq * 8 + 2 * k + 1],
                                                   static_cast<OutT*>(nullptr))
                                   : pack_out(v[qq * 8 + 2 * k], v[qq * 8 + 2 * k + 1],
                                              static_cast<OutT*>(nullptr));
              } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = __float_as_uint(v[qq * 4 + k]);
              }
              st_shared_v4(srow + ((q ^ (rloc & 7)) * 16), w[0], w[1], w[2], w[3]);
            }
          }
          if (!live) continue;
          fence_proxy_async_smem();
          epi_bar_sync(eg);
          if (leader) {
            tma_store_2d(&tmC, stage, n0, m0);
            tma_store_commit();
          }
          ++staged;
        }
      }
      // the staging smem must outlive the stores' reads; the global writes
      // themselves complete with the grid (no wait for them at the tail)
      if (leader) tma_store_wait_read<0>();
    } else {
      for (int t = cid; t < num_tiles; t += ncl, ++iter) {
        int mb, nb;
        tile_coords(t, args.num_m_blocks, args.num_n_blocks, args.group_m, mb, nb);
        const int acc = iter & 1;
        const uint32_t acc_par = (iter >> 1) & 1;
        mbar_wait(&tfull_bar[acc], acc_par);
        tc_fence_after();
        const int row = mb * TILE_M + static_cast<int>(rank) * BLOCK_M + rloc;
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BLOCK_N;
#pragma unroll 1
        for (int c = eg; c < BLOCK_N / 32; c += NG) {
          uint32_t r[32];
          tmem_ld32(t_row + c * 32, r);
          tmem_wait_ld();
          if (c + NG >= BLOCK_N / 32) release_acc(acc);
          const int col0 = nb * BLOCK_N + c * 32;
          if (col0 < args.N) store_chunk32_rt<OutT>(r, args, row, col0);
        }
      }
    }
  }

  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // the leader's MMAs into the peer's TMEM are done
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    else tmem_dealloc<TMEM_COLS>(tmem_base);
  }
  if (args.round_sync && threadIdx.x == 0) {
    unsigned int* ctr = g_round[args.round_sync - 1];
    __threadfence();
    if (atomicAdd(&ctr[1], 1u) == gridDim.x - 1) {  // last CTA out: reset for the next launch
      atomicExch(&ctr[0], 0u);
      atomicExch(&ctr[1], 0u);
      __threadfence();
    }
  }
}

// ------------------------------------------------- halo-tiled 3x3 conv (K2b) --
// 3x3 / stride 1 / pad 1 convolution (every stride-1 3x3 layer of ResNet-50)
// with the input staged ONCE per 64-channel chunk and tile instead of once per
// filter tap: a tile = R output rows x P output columns (P = power of two >=
// W + 2, R = 128 / P, so M = 128 pixels per tile, columns >= W discarded). One
// 4-D TMA tile load brings the (R + 2) x P halo of input pixels (columns from
// -1, rows from oy0 - 1; out-of-bounds rows / columns are zero-filled by the
// TMA unit = the conv padding) into 128B-swizzled smem with a row pitch of P
// pixels. Tap (ky, kx) is then the same buffer read at a pixel offset
// ky * P + kx: the UMMA descriptor start moves by (ky P + kx) 128-byte rows.
// The 128B swizzle is a function of the absolute smem address for both the TMA
// write and the MMA read, so starts that are not 1024-byte aligned need no
// base-offset correction (verified on B200: setting it to kx breaks parity).
// L2 -> smem traffic per tile drops 9 x 16 KB -> (R+2) P 128 B (4.5x at W=56)
// relative to the im2col loader, which bound the 56x56 layers.
struct HaloArgs {
  GemmTcArgs g;            // epilogue: M (output pixels), N = OC, ldc, bias, C, epi
  int H, W, C;             // input (= output) extent, channels
  int P, R;                // halo row pitch (pixels), output rows per tile
  int tiles_per_img, num_m_tiles, c_chunks;
};

// RES_B: the whole filter (9 taps x 64 channels x OC <= BLOCK_N) is loaded into
// smem once per CTA and stays resident (a single 64-channel chunk and OC block):
// the per-tile L2 traffic is then the input halo alone.
template <int BLOCK_N, bool RES_B = false>
struct HaloSmem {
  static constexpr int A_BYTES = (128 + 2 * 64) * 128;  // (R+2) x P pixels at P = 64
  static constexpr int B_STAGES = RES_B ? 9 : (BLOCK_N == 64 ? 8 : (BLOCK_N == 128 ? 6 : 4));
  static constexpr int B_BYTES = BLOCK_N * 128;  // BLOCK_N rows x 64 channels (one tap)
  static constexpr int B_OFF = 2 * A_BYTES;
  static constexpr int BAR_OFF = B_OFF + B_STAGES * B_BYTES;
  // a_full[2], a_empty[2], b_full[S], b_empty[S], tfull[2], tempty[2]
  static constexpr int NUM_BARS = 4 + 2 * B_STAGES + 4;
  static constexpr int TOTAL = BAR_OFF + NUM_BARS * 8 + 16 + 1024;
  static_assert(TOTAL <= 232448, "halo conv smem over the 227 KB opt-in limit");
};

template <int BLOCK_N, bool AB_BF16, typename OutT, bool RES_B>
__global__ void __launch_bounds__(384, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmW, const HaloArgs args) {
  using L = HaloSmem<BLOCK_N, RES_B>;
  constexpr int NS = L::B_STAGES;
  constexpr uint32_t TMEM_COLS = 2 * BLOCK_N <= 128 ? 128 : (2 * BLOCK_N <= 256 ? 256 : 512);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 2;
  uint64_t* b_full = bars + 4;
  uint64_t* b_empty = b_full + NS;
  uint64_t* tfull = b_empty + NS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NUM_BARS);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nnb = args.g.num_n_blocks;
  const int num_tiles = args.num_m_tiles * nnb;
  const int a_bytes = (args.R + 2) * args.P * 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  griddep_launch_dependents();
  // tile t: output-pixel block mt (image n, rows oy0..oy0+R-1), OC block nb
  // (nb fastest: consecutive tiles reuse the same halo in L2)
  auto coords = [&](int t, int& n, int& oy0, int& nb) {
    const int mt = t / nnb;
    nb = t - mt * nnb;
    n = mt / args.tiles_per_img;
    oy0 = (mt - n * args.tiles_per_img) * args.R;
  };

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      int ai = 0, bs = 0;
      uint32_t bph = 0;
      if constexpr (RES_B) {  // the whole filter, once
        mbar_arrive_expect_tx(&b_full[0], 9 * L::B_BYTES);
        for (int tap = 0; tap < 9; ++tap)
          tma_load_2d(smem + L::B_OFF + tap * L::B_BYTES, &tmW, &b_full[0], tap * args.C, 0);
      }
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int n, oy0, nb;
        coords(t, n, oy0, nb);
        for (int cb = 0; cb < args.c_chunks; ++cb, ++ai) {
          const int slot = ai & 1;
          mbar_wait(&a_empty[slot], ((ai >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&a_full[slot], static_cast<uint32_t>(a_bytes));
          tma_load_4d(smem + slot * L::A_BYTES, &tmX, &a_full[slot], cb * 64, -1, oy0 - 1, n);
          if constexpr (RES_B) continue;
          for (int tap = 0; tap < 9; ++tap) {
            mbar_wait(&b_empty[bs], bph ^ 1);
            mbar_arrive_expect_tx(&b_full[bs], L::B_BYTES);
            tma_load_2d(smem + L::B_OFF + bs * L::B_BYTES, &tmW, &b_full[bs],
                        tap * args.C + cb * 64, nb * BLOCK_N);
            if (++bs == NS) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------- MMA issuer (warp-uniform)
    const bool leader = elect_one();
    constexpr uint32_t idesc = idesc_f16(BLOCK_M, BLOCK_N, AB_BF16 ? 1u : 0u, 0u, 0u);
    const uint64_t a_desc0 = desc_kmajor_sw128(smem_u32(smem));
    const uint64_t b_desc0 = desc_kmajor_sw128(smem_u32(smem + L::B_OFF));
    int ai = 0, bs = 0, iter = 0;
    uint32_t bph = 0;
    if constexpr (RES_B) {
      mbar_wait(&b_full[0], 0);
      tc_fence_after();
    }
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++iter) {
      const int acc = iter & 1;
      mbar_wait(&tempty[acc], ((iter >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BLOCK_N;
      for (int cb = 0; cb < args.c_chunks; ++cb, ++ai) {
        const int slot = ai & 1;
        mbar_wait(&a_full[slot], (ai >> 1) & 1);
        tc_fence_after();
        const uint64_t a_slot = a_desc0 + static_cast<uint64_t>(slot) * (L::A_BYTES >> 4);
        for (int tap = 0; tap < 9; ++tap) {
          const int ky = tap / 3, kx = tap - 3 * (tap / 3);
          if constexpr (RES_B) {
            bs = tap;  // resident filter: tap slot
          } else {
            mbar_wait(&b_full[bs], bph);
            tc_fence_after();
          }
          // tap window: (ky * P + kx) 128-byte pixel rows into the halo
          const uint64_t ad = a_slot + static_cast<uint64_t>((ky * args.P + kx) * 8);
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(bs) * (L::B_BYTES >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_f16_ss_if(leader, d_tmem, ad + static_cast<uint64_t>(k * 2), bd + static_cast<uint64_t>(k * 2),
                          idesc, (cb | tap | k) != 0 ? 1u : 0u);
          if constexpr (!RES_B) {
            mma_commit_if(leader, &b_empty[bs]);
            if (++bs == NS) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
        mma_commit_if(leader, &a_empty[slot]);
      }
      mma_commit_if(leader, &tfull[acc]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue --
    // accumulator row m = r * P + c -> output pixel (n, oy0 + r, c) if c < W
    const int eg = (warp - 4) / 4;
    const int ew = warp % 4;
    const int m = ew * 32 + lane;
    const int r = m / args.P, c = m - r * args.P;
    int iter = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++iter) {
      int n, oy0, nb;
      coords(t, n, oy0, nb);
      const int acc = iter & 1;
      mbar_wait(&tfull[acc], (iter >> 1) & 1);
      tc_fence_after();
      const int oy = oy0 + r;
      const int out_row = (c < args.W && oy < args.H) ? (n * args.H + oy) * args.W + c : args.g.M;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BLOCK_N;
#pragma unroll 1
      for (int ch = eg; ch < BLOCK_N / 32; ch += 2) {
        uint32_t v[32];
        tmem_ld32(t_row + ch * 32, v);
        tmem_wait_ld();
        if (ch + 2 >= BLOCK_N / 32) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        const int col0 = nb * BLOCK_N + ch * 32;
        if (col0 < args.g.N) store_chunk32_rt<OutT>(v, args.g, out_row, col0);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// --------------------------------------------------------------- host side --


template <int BLOCK_N, int STAGES, bool B_MN_MAJOR, bool AB_BF16, typename OutT,
          bool IM2COL = false, bool PAIR = false, int NG = 2>
cudaError_t launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmC, const GemmTcArgs& args, cudaStream_t stream) {
  auto kern = gemm_tc_kernel<BLOCK_N, STAGES, B_MN_MAJOR, AB_BF16, OutT, IM2COL, PAIR, NG>;
  constexpr int smem = SmemLayout<BLOCK_N, STAGES, PAIR, NG>::TOTAL;
  static_assert(smem <= 232448, "gemm smem over the 227 KB opt-in limit");
  static std::atomic<uint64_t> configured{0};  // per instantiation, one bit per device
  if (cudaError_t e = ensure_smem_optin(configured, kern, smem); e != cudaSuccess) return e;
  const int tiles = args.num_m_blocks * args.num_n_blocks;
  // persistent grid (CTA pairs: clusters of 2 on one TPC, one per 2 SMs),
  // launched as a programmatic dependent of the previous kernel in the stream
  const int grid = PAIR ? 2 * std::min(tiles, num_sms() / 2) : std::min(tiles, num_sms());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128 + 128 * NG);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (PAIR) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmC, args);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int BLOCK_N, int STAGES, bool PAIR = false, int NG = 2>
cudaError_t dispatch_types(afg_dtype ab, afg_dtype c, bool b_mn_major, const CUtensorMap& tmA,
                           const CUtensorMap& tmB, const CUtensorMap& tmC, const GemmTcArgs& args,
                           cudaStream_t s) {
#define AFG_GEMM_V(MN, BF, OT) \
  launch_variant<BLOCK_N, STAGES, MN, BF, OT, false, PAIR, NG>(tmA, tmB, tmC, args, s)
  if (ab == AFG_BF16) {
    if (c == AFG_BF16) return b_mn_major ? AFG_GEMM_V(true, true, __nv_bfloat16)
                                         : AFG_GEMM_V(false, true, __nv_bfloat16);
    if (c == AFG_F32) return b_mn_major ? AFG_GEMM_V(true, true, float)
                                        : AFG_GEMM_V(false, true, float);
  } else {
    if (c == AFG_F16) return b_mn_major ? AFG_GEMM_V(true, false, __half)
                                        : AFG_GEMM_V(false, false, __half);
    if (c == AFG_F32) return b_mn_major ? AFG_GEMM_V(true, false, float)
                                        : AFG_GEMM_V(false, false, float);
  }
#undef AFG_GEMM_V
  return cudaErrorNotSupported;
}

// TMA store descriptor for C [M, N] (row pitch ldc): boxes of 128 rows x 128 B
// (64 16-bit or 32 fp32 columns), 128-byte swizzle. 0 if C is not TMA-
// addressable (then the epilogue stores straight from registers).
int make_store_map(CUtensorMap* map, void* C, afg_dtype c, int64_t M, int64_t N, int64_t ldc) {
  const int es = dtype_bytes(c);
  if ((reinterpret_cast<uintptr_t>(C) & 15) || (ldc * es) % 16 != 0) return 0;
  const CUtensorMapDataType dt = c == AFG_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : c == AFG_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  if (make_tmap_2d(map, C, dt, es, N, M, ldc, 128 / es, BLOCK_M) != AFG_OK) return 0;
  return 1;
}

// CTA-pair tiles (256 x 256) for BLOCK_N = 256 problems with K >= 768 and at
// least one full wave of pair tiles; AFG_GEMM_PAIR=0 disables them, =2 forces
// them whenever K >= 768 (A/B knobs; 2048^3 forced: 24.1 vs 22.5 us).
bool use_pair_tiles(int block_n, int64_t M, int64_t N, int64_t K) {
  static const int mode = [] {  // 0 = off, 2 = whenever K >= 768 (A/B)
    const char* e = getenv("AFG_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  const bool enabled = mode != 0;
  // short K (<= 8 k-blocks) is epilogue / HBM bound: the pair's cross-CTA
  // accumulator hand-off costs more than the halved B staging saves
  // (measured: ResNet 1x1 convs and BERT K = 768 GEMMs)
  if (!enabled || block_n != 256 || M < 256 || K < 768) return false;
  const int64_t pair_tiles = ((M + 255) / 256) * ((N + 255) / 256);
  return mode == 2 || pair_tiles >= num_sms() / 2;
}

// Four epilogue warp groups (640-thread CTA, one C staging buffer per group)
// for the short-K pair GEMM when the epilogue is GELU: its per-element math,
// not the store stream, then bounds the tile (BERT FFN1 erf-GELU 145 -> 135 us);
// bias-only epilogues keep two groups with two buffers each (102 vs 106 us).
// AFG_GEMM_EPI_GROUPS = 2 | 4 forces either.
bool four_epi_groups(afg_epilogue epi) {
  static const int forced = [] {
    const char* e = getenv("AFG_GEMM_EPI_GROUPS");
    return e ? atoi(e) : 0;
  }();
  if (forced == 2 || forced == 4) return forced == 4;
  return epi == AFG_EPI_BIAS_GELU_TANH || epi == AFG_EPI_BIAS_GELU_ERF;
}

// AFG_GEMM_SHORTK_GROUPS = 2 | 4: epilogue groups of the output-bound
// (K <= 128, BLOCK_N = 256) single-CTA GEMM
// AFG_GEMM_SHORTK_MAXK: the largest K that takes the output-bound
// configuration (2 stages, 4 epilogue groups)
int64_t shortk_max_k() {
  static const int64_t k = [] {
    const char* e = getenv("AFG_GEMM_SHORTK_MAXK");
    return e ? static_cast<int64_t>(atoi(e)) : 128;
  }();
  return k;
}

int shortk_groups() {
  static const int g = [] {
    const char* e = getenv("AFG_GEMM_SHORTK_GROUPS");
    return e ? atoi(e) : 4;
  }();
  return g;
}

}  // namespace

// Entry used by afg_gemm (api.cpp) and the conv / BERT paths.
afg_status gemm_tc(const void* A, int64_t lda, const void* B, int64_t ldb, const float* bias,
                   const void* residual, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                   afg_dtype ab, afg_dtype c, afg_layout b_layout, afg_epilogue epi,
                   cudaStream_t stream) {
  const bool b_mn_major = b_layout == AFG_B_KN;
  // BLOCK_N: 256 when N is large enough to fill it, else 128 / 64.
  static const int bn_env = [] {  // A/B knob: AFG_GEMM_BN = 64 | 128 | 256 forces BLOCK_N
    const char* e = getenv("AFG_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  int block_n = (bn_env == 64 || bn_env == 128 || bn_env == 256)
                    ? bn_env
                    : (N >= 256 ? 256 : (N > 64 ? 128 : 64));
  // 256 x 256 tiles on a CTA pair when there are enough of them to fill the GPU
  const bool pair = use_pair_tiles(block_n, M, N, K);
  // fewer 128 x 256 tiles than SMs (2048^3: 128 tiles): 128 x 128 tiles, so
  // that the SMs with two tiles overlap one tile's epilogue with the other's
  // main loop (2048^3 + GELU, L2 flushed: 32.6 -> 26.7 us)
  if (!pair && bn_env == 0 && block_n == 256 && K >= 1024 &&
      ((M + BLOCK_M - 1) / BLOCK_M) * ((N + 255) / 256) < num_sms())
    block_n = 128;
  const CUtensorMapDataType tdt =
      ab == AFG_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmA, tmB;
  afg_status st = make_tmap_2d(&tmA, A, tdt, 2, K, M, lda, BLOCK_K, BLOCK_M);
  if (st != AFG_OK) return st;
  if (b_mn_major)
    st = make_tmap_2d(&tmB, B, tdt, 2, N, K, ldb, 64, BLOCK_K);
  else
    st = make_tmap_2d(&tmB, B, tdt, 2, K, N, ldb, BLOCK_K, pair ? block_n / 2 : block_n);
  if (st != AFG_OK) return st;

  GemmTcArgs args;
  args.M = static_cast<int>(M);
  args.N = static_cast<int>(N);
  args.K = static_cast<int>(K);
  args.ldc = static_cast<int>(ldc);
  args.bias = bias;
  args.residual = residual;
  args.C = C;
  const int tile_m = pair ? 2 * BLOCK_M : BLOCK_M;
  args.num_m_blocks = static_cast<int>((M + tile_m - 1) / tile_m);
  // raster groups span 2048 rows of A (16 x 128 or 8 x 256-row pair tiles)
  static const int group_env = [] {
    const char* e = getenv("AFG_GEMM_GROUP_M");
    return e ? atoi(e) : 0;
  }();
  args.group_m = group_env > 0 ? group_env : (pair ? GROUP_M / 2 : GROUP_M);
  args.num_n_blocks = static_cast<int>((N + block_n - 1) / block_n);
  args.epi = static_cast<int>(epi);
  CUtensorMap tmC;
  static const bool no_tma_store = [] {
    const char* e = getenv("AFG_GEMM_TMA_STORE");
    return e && atoi(e) == 0;
  }();
  args.tma_store = no_tma_store ? 0 : make_store_map(&tmC, C, c, M, N, ldc);
  args.early_tmem = early_tmem_for(K);
  args.round_sync = round_sync_for(args.num_m_blocks * args.num_n_blocks, K, pair, stream);
  cudaError_t e;
  if (pair && K >= 2048)  // long K: operand stages first (6 x 32 KB, one C buffer per group)
    e = dispatch_types<256, 6, true>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else if (pair && four_epi_groups(epi))  // GELU: four epilogue groups, one C buffer each
    e = dispatch_types<256, 5, true, 4>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else if (pair)  // shorter K: the epilogue matters more (5 stages, two C buffers per group)
    e = dispatch_types<256, 5, true>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  // output-bound: 2 stages; 4 epilogue groups x 2 C buffers (ResNet 56x56
  // 64 -> 256 1x1: 103.6 -> 90.2 us vs 2 groups x 4 buffers)
  else if (block_n == 256 && K <= shortk_max_k() && shortk_groups() == 4)
    e = dispatch_types<256, 2, false, 4>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else if (block_n == 256 && K <= 128)  // output-bound: 2 stages, 4 C buffers per group
    e = dispatch_types<256, 2>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else if (block_n == 256)
    e = dispatch_types<256, 3>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else if (block_n == 128 && K <= 128)
    e = dispatch_types<128, 2>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else if (block_n == 128)
    e = dispatch_types<128, 5>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  else
    e = dispatch_types<64, 6>(ab, c, b_mn_major, tmA, tmB, tmC, args, stream);
  if (e == cudaErrorNotSupported)
    return set_error(AFG_ERR_UNSUPPORTED, "gemm_tc: unsupported (ab, c) dtype pair");
  return cuda_status(e, "gemm_tc launch");
}

// Implicit-GEMM convolution on the same pipeline: the A tile of 128 output
// pixels x 64 channels for filter tap (ky, kx) is gathered by the TMA unit in
// im2col mode (zero fill outside the padded bounding box), B is the OHWI
// filter viewed as [OC, KH*KW*C] (K-major). SPEC.md:388-452 (conv_gemm.cpp is
// a stub in the reference).
afg_status conv_tc(const void* x, const void* w, const float* bias, void* y, int64_t B,
                   int64_t H, int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                   int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t dh, int64_t dw,
                   int64_t OH, int64_t OW, afg_dtype dt, afg_dtype yt, afg_epilogue epi,
                   cudaStream_t stream) {
  const int64_t M = B * OH * OW;
  const int64_t K = KH * KW * C;
  static const int conv_bn_env = [] {  // AFG_CONV_BN = 64 | 128 | 256 (A/B)
    const char* e = getenv("AFG_CONV_BN");
    return e ? atoi(e) : 0;
  }();
  const int block_n = (conv_bn_env == 64 || conv_bn_env == 128 || conv_bn_env == 256)
                          ? conv_bn_env
                          : (OC >= 256 ? 256 : (OC > 64 ? 128 : 64));
  const CUtensorMapDataType tdt =
      dt == AFG_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  // padded bounding box: lower = -pad_begin, upper = pad_end - (K-1)*dil with
  // pad_end chosen so that the traversal yields exactly OH x OW positions.
  const int64_t pb = (OH - 1) * sh + (KH - 1) * dh + 1 - H - pt;
  const int64_t pr = (OW - 1) * sw + (KW - 1) * dw + 1 - W - pl;
  const int lower[2] = {static_cast<int>(-pl), static_cast<int>(-pt)};
  const int upper[2] = {static_cast<int>(pr - (KW - 1) * dw), static_cast<int>(pb - (KH - 1) * dh)};
  for (int i = 0; i < 2; ++i)
    if (lower[i] < -128 || lower[i] > 127 || upper[i] < -128 || upper[i] > 127)
      return set_error(AFG_ERR_UNSUPPORTED, "conv_tc: padding outside the im2col corner range");
  if (sh > 8 || sw > 8) return set_error(AFG_ERR_UNSUPPORTED, "conv_tc: stride > 8");
  CUtensorMap tmA, tmB;
  afg_status st = make_tmap_im2col_4d(&tmA, x, tdt, C, W, H, B, lower, upper,
                                      static_cast<int>(sw), static_cast<int>(sh), BLOCK_K, BLOCK_M);
  if (st != AFG_OK) return st;
  // 256 x 256 CTA-pair tiles as for plain GEMMs (each CTA gathers its own 128
  // output pixels by im2col and half of the filter rows)
  const bool pair = use_pair_tiles(block_n, M, OC, K);
  st = make_tmap_2d(&tmB, w, tdt, 2, K, OC, K, BLOCK_K, pair ? block_n / 2 : block_n);
  if (st != AFG_OK) return st;
  GemmTcArgs args{};
  args.M = static_cast<int>(M);
  args.N = static_cast<int>(OC);
  args.K = static_cast<int>(K);
  args.ldc = static_cast<int>(OC);
  args.bias = bias;
  args.residual = nullptr;
  args.C = y;
  args.num_m_blocks = static_cast<int>((M + (pair ? 2 : 1) * BLOCK_M - 1) / ((pair ? 2 : 1) * BLOCK_M));
  args.num_n_blocks = static_cast<int>((OC + block_n - 1) / block_n);
  args.group_m = pair ? GROUP_M / 2 : GROUP_M;
  args.epi = static_cast<int>(epi);
  args.c_blocks = static_cast<int>(C / BLOCK_K);
  args.KW = static_cast<int>(KW);
  args.dil_w = static_cast<int>(dw);
  args.dil_h = static_cast<int>(dh);
  args.OH = static_cast<int>(OH);
  args.OW = static_cast<int>(OW);
  args.stride_w = static_cast<int>(sw);
  args.stride_h = static_cast<int>(sh);
  args.lower_w = lower[0];
  args.lower_h = lower[1];
  cudaError_t e;
  CUtensorMap tmC;
  args.tma_store = make_store_map(&tmC, y, yt, M, OC, OC);
  args.early_tmem = early_tmem_for(K);
  args.round_sync = 0;  // measured: ResNet convs 747 -> 681 TFLOP/s with it
  const bool f32_out = yt == AFG_F32;
#define AFG_CONV_V(BN, ST)                                                                      \
  (dt == AFG_BF16                                                                               \
       ? (f32_out ? launch_variant<BN, ST, false, true, float, true>(tmA, tmB, tmC, args, stream) \
                  : launch_variant<BN, ST, false, true, __nv_bfloat16, true>(tmA, tmB, tmC, args,  \
                                                                              stream))            \
       : (f32_out ? launch_variant<BN, ST, false, false, float, true>(tmA, tmB, tmC, args, stream) \
                  : launch_variant<BN, ST, false, false, __half, true>(tmA, tmB, tmC, args, stream)))
#define AFG_CONV_P(ST)                                                                          \
  (dt == AFG_BF16                                                                               \
       ? (f32_out ? launch_variant<256, ST, false, true, float, true, true>(tmA, tmB, tmC, args,  \
                                                                          stream)               \
                  : launch_variant<256, ST, false, true, __nv_bfloat16, true, true>(              \
                        tmA, tmB, tmC, args, stream))                                           \
       : (f32_out ? launch_variant<256, ST, false, false, float, true, true>(tmA, tmB, tmC, args, \
                                                                           stream)              \
                  : launch_variant<256, ST, false, false, __half, true, true>(tmA, tmB, tmC, args, \
                                                                              stream)))
  if (pair && K >= 2048)
    e = AFG_CONV_P(6);
  else if (pair)
    e = AFG_CONV_P(5);
  else if (block_n == 256)
    e = AFG_CONV_V(256, 3);
  else if (block_n == 128)
    e = AFG_CONV_V(128, 5);
  else
    e = AFG_CONV_V(64, 6);
#undef AFG_CONV_V
#undef AFG_CONV_P
  return cuda_status(e, "conv_tc launch");
}


// Halo-tiled 3x3 / stride-1 / pad-1 conv (see conv_halo_kernel). Returns
// AFG_ERR_UNSUPPORTED when the shape does not fit (the caller then uses the
// im2col path).
afg_status conv_halo(const void* x, const void* w, const float* bias, void* y, int64_t B,
                     int64_t H, int64_t W, int64_t C, int64_t OC, afg_dtype dt, afg_dtype yt,
                     afg_epilogue epi, cudaStream_t stream) {
  static const int mode = [] {  // AFG_CONV_HALO=0 turns it off (A/B measurements)
    const char* e = getenv("AFG_CONV_HALO");
    return e ? atoi(e) : 1;
  }();
  // W < 20 (P = 16) wastes 2 of every 16 columns and, at 14x14, 2 of 16 rows
  // too: measured slower than the im2col loader there (60 vs 55 us)
  if (mode == 0 || C % 64 != 0 || W < 20 || W + 2 > 64 || (dt != AFG_BF16 && dt != AFG_F16))
    return AFG_ERR_UNSUPPORTED;
  const int P = W + 2 <= 16 ? 16 : (W + 2 <= 32 ? 32 : 64);
  const int R = 128 / P;
  const int block_n = OC >= 256 ? 256 : (OC > 64 ? 128 : 64);
  const CUtensorMapDataType tdt =
      dt == AFG_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmX, tmW;
  const uint64_t dims[4] = {static_cast<uint64_t>(C), static_cast<uint64_t>(W),
                            static_cast<uint64_t>(H), static_cast<uint64_t>(B)};
  const uint64_t strides[3] = {static_cast<uint64_t>(C) * 2, static_cast<uint64_t>(W * C) * 2,
                               static_cast<uint64_t>(H * W * C) * 2};
  const uint32_t box[4] = {64, static_cast<uint32_t>(P), static_cast<uint32_t>(R + 2), 1};
  afg_status st = make_tmap(&tmX, x, tdt, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != AFG_OK) return st;
  st = make_tmap_2d(&tmW, w, tdt, 2, 9 * C, OC, 9 * C, 64, block_n);
  if (st != AFG_OK) return st;
  HaloArgs a{};
  a.g.M = static_cast<int>(B * H * W);
  a.g.N = static_cast<int>(OC);
  a.g.K = static_cast<int>(9 * C);
  a.g.ldc = static_cast<int>(OC);
  a.g.bias = bias;
  a.g.residual = nullptr;
  a.g.C = y;
  a.g.num_n_blocks = static_cast<int>((OC + block_n - 1) / block_n);
  a.g.epi = static_cast<int>(epi);
  a.H = static_cast<int>(H);
  a.W = static_cast<int>(W);
  a.C = static_cast<int>(C);
  a.P = P;
  a.R = R;
  a.tiles_per_img = static_cast<int>((H + R - 1) / R);
  a.num_m_tiles = static_cast<int>(B) * a.tiles_per_img;
  a.c_chunks = static_cast<int>(C / 64);
  const int tiles = a.num_m_tiles * a.g.num_n_blocks;
  const int grid = std::min(tiles, num_sms());
  auto go = [&](auto kern, int smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, kern, tmX, tmW, a);
    count_launch();
    return e2 != cudaSuccess ? e2 : cudaGetLastError();
  };
  cudaError_t e;
#define AFG_HALO(BN, RB)                                                                        \
  (yt == AFG_F32                                                                               \
       ? (dt == AFG_BF16 ? go(conv_halo_kernel<BN, true, float, RB>, HaloSmem<BN, RB>::TOTAL)    \
                         : go(conv_halo_kernel<BN, false, float, RB>, HaloSmem<BN, RB>::TOTAL))  \
       : (dt == AFG_BF16                                                                       \
              ? go(conv_halo_kernel<BN, true, __nv_bfloat16, RB>, HaloSmem<BN, RB>::TOTAL)      \
              : go(conv_halo_kernel<BN, false, __half, RB>, HaloSmem<BN, RB>::TOTAL)))
  // one channel chunk and one OC block: keep the filter resident
  const bool res_b = C == 64 && OC <= block_n && block_n <= 128;
  if (block_n == 256) e = AFG_HALO(256, false);
  else if (block_n == 128) e = res_b ? AFG_HALO(128, true) : AFG_HALO(128, false);
  else e = res_b ? AFG_HALO(64, true) : AFG_HALO(64, false);
#undef AFG_HALO
  return cuda_status(e, "conv_halo launch");
}

}  // namespace afg
